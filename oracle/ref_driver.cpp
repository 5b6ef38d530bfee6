// Oracle driver — TEST INFRASTRUCTURE, not product code.
//
// Links the reference's own slapo_core (built from /root/reference/proj/src by
// oracle/Makefile) and runs the reference executor on a fixture model with a
// schedule script, dumping everything the B200 executor is checked against:
//   model.json     post-apply ModuleDef (save_model, proj/src/model_io.cpp:225)
//   outputs.bin    forward outputs of every rank   (Executor::outputs_of_rank)
//   grads.bin      param + input gradients, every rank (backward_all_ranks)
//   params.bin     worker-local param values, every rank (init_param_rank)
//   meta.json      collective count, ledger bytes, wall-clock timing
// The dump format ("SBT1") is: magic, u32 count, then per tensor
//   u32 name_len, name, u32 rank, i64 dims[rank], f64 data.
//
// Reference APIs used: toy_bert / tp_two_linear / fig3c_exact
// (proj/tests/support/fixtures.cpp:79-171), load_schedule_script
// (proj/src/script.cpp:74), Schedule::apply (proj/src/schedule.cpp:719),
// Executor (proj/include/slapo/executor.hpp:37-63), random_tensor
// (proj/src/executor.cpp:19), uniform01 (proj/include/slapo/rng.hpp:35).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "slapo/costmodel.hpp"
#include "slapo/dump.hpp"
#include "slapo/tuner.hpp"
#include "slapo/executor.hpp"
#include "slapo/model_io.hpp"
#include "slapo/rng.hpp"
#include "slapo/schedule.hpp"
#include "slapo/script.hpp"
#include "slapo/shape_inference.hpp"
#include "support/fixtures.hpp"

using namespace slapo;

namespace {

struct Named {
    std::string name;
    const TensorValue* t;
};

void write_dump(const std::string& path, const std::vector<std::pair<std::string, TensorValue>>& ts) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw Error("cannot write " + path);
    out.write("SBT1", 4);
    std::uint32_t n = static_cast<std::uint32_t>(ts.size());
    out.write(reinterpret_cast<const char*>(&n), 4);
    for (const auto& [name, t] : ts) {
        std::uint32_t len = static_cast<std::uint32_t>(name.size());
        out.write(reinterpret_cast<const char*>(&len), 4);
        out.write(name.data(), len);
        std::uint32_t rank = static_cast<std::uint32_t>(t.spec.shape.size());
        out.write(reinterpret_cast<const char*>(&rank), 4);
        for (auto d : t.spec.shape) out.write(reinterpret_cast<const char*>(&d), 8);
        out.write(reinterpret_cast<const char*>(t.data.data()), t.data.size() * 8);
    }
}

// the inverse of write_dump: tensors in file order (used for --inputs)
std::vector<TensorValue> read_dump_values(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error("cannot read " + path);
    char magic[4];
    in.read(magic, 4);
    if (std::string(magic, 4) != "SBT1") throw Error("not an SBT1 dump: " + path);
    std::uint32_t n = 0;
    in.read(reinterpret_cast<char*>(&n), 4);
    std::vector<TensorValue> res;
    for (std::uint32_t k = 0; k < n; ++k) {
        std::uint32_t len = 0, rank = 0;
        in.read(reinterpret_cast<char*>(&len), 4);
        std::string name(len, '\0');
        in.read(name.data(), len);
        in.read(reinterpret_cast<char*>(&rank), 4);
        TensorSpec spec;
        spec.dtype = Dtype::F64;
        for (std::uint32_t r = 0; r < rank; ++r) {
            std::int64_t d = 0;
            in.read(reinterpret_cast<char*>(&d), 8);
            spec.shape.push_back(d);
        }
        TensorValue t(spec);
        in.read(reinterpret_cast<char*>(t.data.data()), static_cast<std::streamsize>(t.data.size() * 8));
        res.push_back(std::move(t));
    }
    return res;
}

std::string read_file(const std::string& p) {
    std::ifstream in(p, std::ios::binary);
    if (!in) throw Error("cannot read " + p);
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

void to_f32(ModuleDef& m) {  // as combos_test.cpp:90-100
    for (auto& p : m.params) p.spec.dtype = Dtype::F32;
    if (m.forward) {
        for (auto& n : m.forward->nodes)
            if (n.kind == NodeKind::Input) n.attrs["dtype"] = std::string("f32");
    }
    for (auto& s : m.submodules) to_f32(*s.module);
}

void collect_params(const ModuleDef& m, const std::string& path, std::vector<std::pair<std::string, const ParamDef*>>& out) {
    for (const auto& p : m.params) out.push_back({join_path(path, p.name), &p});
    for (const auto& s : m.submodules) collect_params(*s.module, join_path(path, s.name), out);
}

}  // namespace

int main(int argc, char** argv) {
    std::map<std::string, std::string> a = {
        {"model", "toy_bert"}, {"layers", "2"}, {"hidden", "8"}, {"heads", "2"}, {"vocab", "28"},
        {"batch", "4"}, {"seq", "4"}, {"p", "0.1"}, {"dtype", "f64"}, {"schedule", ""},
        {"world", "1"}, {"mode", "train"}, {"seed", "123"}, {"input_seed", "9"}, {"out", ""},
        {"backward", "1"}, {"dump_params", "0"}, {"probe_rng", ""}, {"model_json", ""},
        {"tp_hidden", "8"}, {"tp_inner", "16"}, {"tp_batch", "4"}, {"repeat", "1"}, {"cli_run", ""},
        {"estimate", ""}, {"est_batch", "0"}, {"est_mem", "17179869184"}, {"est_consts", ""}, {"ckpt_container", ""},
        {"ckpt_ratio", "0"}, {"tune", ""}, {"tune_seed", "0"}, {"tune_restarts", "3"}, {"micro", "1"},
        {"cli_train", ""}, {"inputs", ""}};
    for (int i = 1; i + 1 < argc; i += 2) {
        std::string k = argv[i];
        if (k.rfind("--", 0) != 0) { std::cerr << "bad arg " << k << "\n"; return 2; }
        a[k.substr(2)] = argv[i + 1];
    }
    try {
        if (!a["probe_rng"].empty()) {
            // probe_rng "<stream_seed>,<n>": uniform01(stream, 0xd0, i) for i < n
            // (the dropout draw, proj/src/executor.cpp:801) and hash_combine.
            std::uint64_t s = std::stoull(a["probe_rng"].substr(0, a["probe_rng"].find(',')));
            std::int64_t n = std::stoll(a["probe_rng"].substr(a["probe_rng"].find(',') + 1));
            TensorValue u(TensorSpec{{n}, Dtype::F64});
            for (std::int64_t i = 0; i < n; ++i) u.data[i] = uniform01(s, 0xd0, static_cast<std::uint64_t>(i));
            write_dump(a["out"] + "/rng.bin", {{"uniform01", u}});
            return 0;
        }
        ModuleDef model;
        if (!a["model_json"].empty()) {
            model = load_model(read_file(a["model_json"]));
        } else if (a["model"] == "toy_bert") {
            testing::BertConfig cfg;
            cfg.layers = std::stoi(a["layers"]);
            cfg.hidden = std::stoll(a["hidden"]);
            cfg.heads = std::stoll(a["heads"]);
            cfg.vocab = std::stoll(a["vocab"]);
            cfg.batch = std::stoll(a["batch"]);
            cfg.seq = std::stoll(a["seq"]);
            cfg.dropout_p = std::stod(a["p"]);
            model = testing::toy_bert(cfg);
        } else if (a["model"] == "tp_two_linear") {
            model = testing::tp_two_linear(std::stoll(a["tp_hidden"]), std::stoll(a["tp_inner"]),
                                           std::stoll(a["tp_batch"]));
        } else if (a["model"] == "fig3c") {
            model = testing::fig3c_exact();
        } else {
            throw Error("unknown model " + a["model"]);
        }
        if (a["dtype"] == "f32") to_f32(model);
        int world = std::stoi(a["world"]);
        WorldConfig wc;
        wc.world_size = world;
        Schedule sch(model, wc);
        if (!a["schedule"].empty()) load_schedule_script(sch, read_file(a["schedule"]));
        ApplyResult res = sch.apply();
        const std::string out = a["out"];
        if (!out.empty()) {
            std::ofstream(out + "/model.json") << save_model(res.model);
            std::ofstream(out + "/original.json") << save_model(model);
            if (res.stages) {  // the stage plan (ApplyResult::stages, schedule.hpp:54-57)
                std::ofstream io(out + "/stages.txt");
                io << "inputs";
                for (auto& x : res.stages->model_inputs) io << " " << x;
                io << "\noutputs";
                for (auto& x : res.stages->model_outputs) io << " " << x;
                io << "\n";
                for (std::size_t i = 0; i < res.stages->stages.size(); ++i) {
                    const auto& st = res.stages->stages[i];
                    std::ofstream(out + "/stage" + std::to_string(i) + ".json") << save_model(st.module);
                    io << "stage" << i << " consumes";
                    for (auto& x : st.consumes) io << " " << x;
                    io << " produces";
                    for (auto& x : st.produces) io << " " << x;
                    io << "\n";
                }
            }
        }
        if (a["dump_params"] == "1" && !out.empty()) {
            std::vector<std::pair<std::string, const ParamDef*>> ps;
            collect_params(res.model, "", ps);
            std::vector<std::pair<std::string, TensorValue>> dump;
            for (int r = 0; r < world; ++r)
                for (auto& [name, p] : ps) dump.push_back({"r" + std::to_string(r) + ":" + name, init_param_rank(*p, r)});
            write_dump(out + "/params.bin", dump);
        }
        auto est_opts = [&](std::int64_t batch) {
            // EstimateOptions (costmodel.hpp:37-43); est_consts "flops,link,launch,optmult"
            EstimateOptions eo;
            eo.batch = batch;
            eo.world_size = world;
            eo.device_memory_bytes = std::stoll(a["est_mem"]);
            if (!a["est_consts"].empty()) {
                std::stringstream ss(a["est_consts"]);
                std::string t;
                std::vector<double> v;
                while (std::getline(ss, t, ',')) v.push_back(std::stod(t));
                eo.constants = CostConstants{v.at(0), v.at(1), v.at(2), v.at(3)};
            }
            return eo;
        };
        auto est_json = [](const CostReport& r) {
            char buf[512];
            std::snprintf(buf, sizeof(buf),
                          "{\"step_time_s\": %.17g, \"flops\": %lld, \"recompute_flops\": %lld, \"launches\": %lld, "
                          "\"collective_bytes\": %lld, \"param_bytes\": %lld, \"activation_bytes\": %lld, "
                          "\"peak_memory_bytes\": %lld, \"oom\": %d, \"throughput_samples_per_s\": %.17g}",
                          r.step_time_s, (long long)r.flops, (long long)r.recompute_flops, (long long)r.launches,
                          (long long)r.collective_bytes, (long long)r.param_bytes, (long long)r.activation_bytes,
                          (long long)r.peak_memory_bytes, r.oom ? 1 : 0, r.throughput_samples_per_s);
            return std::string(buf);
        };
        if (!a["estimate"].empty()) {
            // slapo::estimate (costmodel.cpp:258) of the post-apply model, optionally after
            // apply_checkpoint_ratio (costmodel.cpp:310); prints to_text then a JSON line
            ModuleDef m = res.model;
            if (!a["ckpt_container"].empty()) apply_checkpoint_ratio(m, a["ckpt_container"], std::stod(a["ckpt_ratio"]));
            CostReport r = estimate(m, est_opts(std::stoll(a["est_batch"])));
            std::cout << r.to_text() << est_json(r) << std::endl;
            return 0;
        }
        if (!a["tune"].empty()) {
            // slapo::exhaustive / coordinate_descent (tuner.cpp:98-180) over batch x checkpoint
            // ratio with the cost-model objective of cmd_tune (slapo_main.cpp:218-252):
            // batch in {est_batch/4, /2, x1, x2, x4}, ratio in {0, .25, .5, .75, 1}; prints the trials
            const std::int64_t b0 = std::stoll(a["est_batch"]);
            SearchSpace sp;
            SymbolicVar vb, vr;
            vb.name = "batch";
            for (std::int64_t f : {1, 2, 4, 8, 16}) vb.candidates.push_back(Expr::parse(std::to_string(b0 * f / 4)));
            vr.name = "ckpt";
            for (const char* r : {"0", "0.25", "0.5", "0.75", "1"}) vr.candidates.push_back(Expr::parse(r));
            sp.vars = {vb, vr};
            Objective obj = [&](const Assignment& as) -> TrialEval {
                ModuleDef m = res.model;
                apply_checkpoint_ratio(m, a["ckpt_container"], as.at("ckpt"));
                CostReport r = estimate(m, est_opts(static_cast<std::int64_t>(as.at("batch"))));
                return {r.oom ? 0.0 : r.throughput_samples_per_s, r};
            };
            TunerResult tr = a["tune"] == "cd" ? coordinate_descent(sp, obj, std::stoull(a["tune_seed"]),
                                                                    std::stoi(a["tune_restarts"]))
                                               : exhaustive(sp, obj);
            for (const auto& t : tr.trials)
                std::printf("trial %.17g %.17g %.17g\n", t.assignment.at("batch"), t.assignment.at("ckpt"), t.objective);
            std::printf("best %.17g %.17g %.17g all_zero %d\n", tr.best.assignment.at("batch"), tr.best.assignment.at("ckpt"),
                        tr.best.objective, tr.all_zero ? 1 : 0);
            return 0;
        }
        ExecMode mode = a["mode"] == "verify" ? ExecMode::Verify : ExecMode::Train;
        std::uint64_t seed = std::stoull(a["seed"]);
        if (!a["cli_run"].empty()) {
            // `slapo run MODEL [SCRIPT] --seed --mode --dump` (proj/tools/slapo_main.cpp:168-199):
            // default_inputs (:69-76), run_forward / run_sharded, write_tensor_dump (dump.cpp:29)
            auto specs = declared_input_specs(*model.forward);
            std::vector<TensorValue> ins;
            for (std::size_t i = 0; i < specs.size(); ++i)
                ins.push_back(random_tensor(specs[i], derive_seed(seed, "cli-input"), static_cast<std::uint64_t>(i)));
            std::vector<TensorValue> outs;
            if (a["schedule"].empty()) outs = run_forward(model, ins, mode, derive_seed(seed, "run"));
            else if (res.stages)
                outs = run_pipeline(*res.stages, ins, std::stoi(a["micro"]), mode, derive_seed(seed, "run"));
            else if (world > 1) outs = run_sharded(res.model, ins, world, mode, derive_seed(seed, "run"));
            else outs = run_forward(res.model, ins, mode, derive_seed(seed, "run"));
            write_tensor_dump(a["cli_run"], outs);
            for (const auto& t : outs) std::cout << format_tensor_text(t) << "\n";
            return 0;
        }
        if (!a["cli_train"].empty()) {
            // the training-step reference for the B200 verifier's gradient mode
            // (paper_2302_08005_b200/cli.py verify-train): `slapo run`'s inputs and seeds
            // (slapo_main.cpp:69-82,168-199) through Executor::forward + backward_all_ranks
            // (executor.cpp:285-381); per rank the outputs and every parameter gradient as
            // the reference's SLD1 tensor dumps (dump.cpp:29) plus the gradient names.
            auto specs = declared_input_specs(*model.forward);
            std::vector<TensorValue> ins;
            for (std::size_t i = 0; i < specs.size(); ++i)
                ins.push_back(random_tensor(specs[i], derive_seed(seed, "cli-input"), static_cast<std::uint64_t>(i)));
            const ModuleDef& target = a["schedule"].empty() ? model : res.model;
            const int w = a["schedule"].empty() ? 1 : world;
            Executor ex(target, mode, derive_seed(seed, "run"), w);
            ex.forward(ins);
            auto gm = ex.backward_all_ranks();
            const std::string dir = a["cli_train"];
            for (int r = 0; r < w; ++r) {
                write_tensor_dump(dir + "/outputs.r" + std::to_string(r) + ".sld1", ex.outputs_of_rank(r));
                std::vector<TensorValue> gs;
                std::ofstream names(dir + "/grads.r" + std::to_string(r) + ".names");
                for (auto& [k, v] : gm[(std::size_t)r].params) {
                    gs.push_back(v);
                    names << k << "\n";
                }
                write_tensor_dump(dir + "/grads.r" + std::to_string(r) + ".sld1", gs);
            }
            std::cout << "{\"world\": " << w << "}" << std::endl;
            return 0;
        }
        auto specs = declared_input_specs(*model.forward);
        std::vector<TensorValue> inputs;
        if (!a["inputs"].empty()) {  // explicit inputs (SBT1 dump, declared order), e.g. one micro-batch
            inputs = read_dump_values(a["inputs"]);
            if (inputs.size() != specs.size()) throw Error("--inputs: wrong number of tensors");
            for (std::size_t i = 0; i < specs.size(); ++i) {
                if (inputs[i].data.size() != static_cast<std::size_t>(specs[i].element_count()))
                    throw Error("--inputs: tensor " + std::to_string(i) + " does not match the declared shape");
                inputs[i].spec = specs[i];
                inputs[i].quantize();
            }
        } else {
            for (std::size_t i = 0; i < specs.size(); ++i)
                inputs.push_back(random_tensor(specs[i], std::stoull(a["input_seed"]), i));
        }

        int repeat = std::stoi(a["repeat"]);
        double fwd_s = 0, bwd_s = 0;
        std::vector<std::pair<std::string, TensorValue>> outs, grads;
        std::int64_t coll_fwd = 0, coll_total = 0, ledger = 0;
        for (int it = 0; it < repeat; ++it) {
            Executor ex(res.model, mode, seed, world);
            auto t0 = std::chrono::steady_clock::now();
            ex.forward(inputs);
            auto t1 = std::chrono::steady_clock::now();
            coll_fwd = ex.collective_invocations();
            ledger = ex.ledger().retained_bytes;
            std::vector<GradientMap> gm;
            if (a["backward"] == "1") gm = ex.backward_all_ranks();
            auto t2 = std::chrono::steady_clock::now();
            coll_total = ex.collective_invocations();
            fwd_s += std::chrono::duration<double>(t1 - t0).count();
            bwd_s += std::chrono::duration<double>(t2 - t1).count();
            if (it + 1 == repeat) {
                for (int r = 0; r < world; ++r) {
                    auto o = ex.outputs_of_rank(r);
                    for (std::size_t i = 0; i < o.size(); ++i)
                        outs.push_back({"r" + std::to_string(r) + ":out" + std::to_string(i), o[i]});
                }
                for (int r = 0; r < static_cast<int>(gm.size()); ++r) {
                    for (auto& [k, v] : gm[r].params) grads.push_back({"r" + std::to_string(r) + ":" + k, v});
                    for (std::size_t i = 0; i < gm[r].inputs.size(); ++i)
                        grads.push_back({"r" + std::to_string(r) + ":@input" + std::to_string(i), gm[r].inputs[i]});
                }
            }
        }
        if (!out.empty()) {
            write_dump(out + "/outputs.bin", outs);
            write_dump(out + "/grads.bin", grads);
            std::vector<std::pair<std::string, TensorValue>> ins;
            for (std::size_t i = 0; i < inputs.size(); ++i) ins.push_back({"input" + std::to_string(i), inputs[i]});
            write_dump(out + "/inputs.bin", ins);
        }
        std::ostringstream meta;
        meta << "{\"collectives_fwd\": " << coll_fwd << ", \"collectives_total\": " << coll_total
             << ", \"ledger_bytes\": " << ledger << ", \"fwd_s\": " << fwd_s / repeat
             << ", \"bwd_s\": " << bwd_s / repeat << ", \"repeat\": " << repeat << "}";
        if (!out.empty()) std::ofstream(out + "/meta.json") << meta.str() << "\n";
        std::cout << meta.str() << std::endl;
    } catch (const std::exception& e) {
        std::cerr << "oracle error: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
