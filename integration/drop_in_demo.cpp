// The drop-in in use: a program written against the reference's API (fixtures,
// Schedule, load_schedule_script, Executor) runs the same scheduled model through
// slapo::Executor (CPU, f64) and slapo::B200Executor (B200) and prints the largest
// normalised differences of outputs and gradients. Built and run by
// tests/test_integration.py.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>

#include "b200_executor.hpp"
#include "slapo/script.hpp"
#include "support/fixtures.hpp"

using namespace slapo;

static double rel(const TensorValue& a, const TensorValue& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < b.data.size(); ++i) {
        num = std::max(num, std::fabs(a.data[i] - b.data[i]));
        den = std::max(den, std::fabs(b.data[i]));
    }
    return den > 0 ? num / den : num;
}

int main(int argc, char** argv) {
    testing::BertConfig cfg;
    cfg.layers = 2;
    cfg.hidden = 32;
    cfg.heads = 4;
    cfg.vocab = 32;
    cfg.batch = 2;
    cfg.seq = 8;
    ModuleDef model = testing::toy_bert(cfg);
    Schedule sch(model, WorldConfig{});
    if (argc > 1) {
        std::ifstream f(argv[1]);
        std::stringstream ss;
        ss << f.rdbuf();
        load_schedule_script(sch, ss.str());
    }
    ApplyResult res = sch.apply();
    auto specs = declared_input_specs(*model.forward);
    std::vector<TensorValue> inputs;
    for (size_t i = 0; i < specs.size(); ++i) inputs.push_back(random_tensor(specs[i], 9, i));
    if (argc > 2 && std::string(argv[2]) == "link-only") return 0;
    Executor cpu(res.model, ExecMode::Train, 123);
    B200Executor gpu(res.model, ExecMode::Train, 123);
    auto oc = cpu.forward(inputs);
    auto og = gpu.forward(inputs);
    GradientMap gc = cpu.backward(), gg = gpu.backward();
    double eo = 0, eg = 0;
    for (size_t i = 0; i < oc.size(); ++i) eo = std::max(eo, rel(og[i], oc[i]));
    for (auto& [k, v] : gc.params) {
        if (k.size() >= 8 && k.substr(k.size() - 8) == "key.bias") continue;  // analytically zero
        eg = std::max(eg, rel(gg.params.at(k), v));
    }
    std::printf("{\"outputs\": %.3e, \"grads\": %.3e, \"n_grads\": %zu, \"collectives\": [%lld, %lld]}\n", eo, eg,
                gc.params.size(), (long long)cpu.collective_invocations(), (long long)gpu.collective_invocations());
    return 0;
}
