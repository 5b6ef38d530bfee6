// extern "C" boundary (include/slapo_b200.h). Translates handles and host
// buffers to the C++ host layer; every exception becomes a status code plus a
// thread-local message (RuleError -> 2).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <map>
#include <dlfcn.h>
#include <sstream>

#include "../../include/slapo_b200.h"
#include "host/executor.hpp"
#include "host/rng.hpp"
#include "host/schedule.hpp"
#include "host/stages.hpp"
#include "host/pipeline_exec.hpp"
#include "host/step_model.hpp"

using namespace sb;

struct sb_model {
    Module m;
};
struct sb_schedule {
    Schedule s;
};
struct sb_pipeline {
    StagePlan p;
};
struct sb_pipeline_executor {
    std::unique_ptr<PipelineExecutor> ex;
    std::vector<HostTensor> outs;
    std::vector<GradMap> grads;  // per stage
};
struct sb_executor {
    std::unique_ptr<Executor> ex;
    std::vector<GradMap> grads;
    int world = 1;
    bool nccl = false;
    int rank = 0;
    float* dloss = nullptr;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const RuleError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    } catch (...) {
        g_err = "unknown error";
        return 1;
    }
}

std::vector<std::string> csv(const char* s) {
    std::vector<std::string> out;
    if (!s) return out;
    std::string cur;
    for (const char* p = s; *p; ++p) {
        if (*p == ',') {
            if (!cur.empty()) out.push_back(cur);
            cur.clear();
        } else if (*p != ' ') {
            cur += *p;
        }
    }
    if (!cur.empty()) out.push_back(cur);
    return out;
}

void copy_out(const std::vector<double>& v, double* out, size_t cap, size_t* n) {
    if (n) *n = v.size();
    if (out && cap >= v.size()) std::memcpy(out, v.data(), v.size() * sizeof(double));
    else if (out) throw Error("output buffer too small: need " + std::to_string(v.size()) + " doubles");
}

const GradMap& gmap(sb_executor* e, int rank) {
    if (e->grads.empty()) throw Error("backward requires a completed forward run");
    if (e->nccl) {
        if (rank != e->rank) throw Error("rank lives in another process");
        return e->grads[0];
    }
    if (rank < 0 || rank >= (int)e->grads.size()) throw Error("rank out of range");
    return e->grads[(size_t)rank];
}
}  // namespace

extern "C" {

const char* sb_last_error(void) { return g_err.c_str(); }
int sb_version(void) { return 1; }

// ------------------------------------------------------------------ models
int sb_model_toy_bert(int layers, int64_t hidden, int64_t heads, int64_t vocab, int64_t batch, int64_t seq, double p,
                      sb_model** out) {
    return guard([&] {
        BertConfig c;
        c.layers = layers;
        c.hidden = hidden;
        c.heads = heads;
        c.vocab = vocab;
        c.batch = batch;
        c.seq = seq;
        c.dropout_p = p;
        *out = new sb_model{toy_bert(c)};
    });
}
int sb_model_gpt_neo(int layers, int64_t hidden, int64_t heads, int64_t vocab, int64_t batch, int64_t seq, double p,
                     sb_model** out) {
    return guard([&] {
        DecoderConfig c;
        c.layers = layers;
        c.hidden = hidden;
        c.heads = heads;
        c.vocab = vocab;
        c.batch = batch;
        c.seq = seq;
        c.dropout_p = p;
        *out = new sb_model{gpt_neo(c)};
    });
}
int sb_model_t5_ex(int enc_layers, int dec_layers, int64_t hidden, int64_t heads, int64_t vocab, int64_t batch,
                   int64_t enc_seq, int64_t dec_seq, double p, int tie_embeddings, sb_model** out) {
    return guard([&] {
        T5Config c;
        c.tie_embeddings = tie_embeddings != 0;
        c.enc_layers = enc_layers;
        c.dec_layers = dec_layers;
        c.hidden = hidden;
        c.heads = heads;
        c.vocab = vocab;
        c.batch = batch;
        c.enc_seq = enc_seq;
        c.dec_seq = dec_seq;
        c.dropout_p = p;
        *out = new sb_model{t5(c)};
    });
}
int sb_model_t5(int enc_layers, int dec_layers, int64_t hidden, int64_t heads, int64_t vocab, int64_t batch,
                int64_t enc_seq, int64_t dec_seq, double p, sb_model** out) {
    return sb_model_t5_ex(enc_layers, dec_layers, hidden, heads, vocab, batch, enc_seq, dec_seq, p, 1, out);
}
int sb_model_tp_two_linear(int64_t hidden, int64_t inner, int64_t batch, sb_model** out) {
    return guard([&] { *out = new sb_model{tp_two_linear(hidden, inner, batch)}; });
}
int sb_model_fig3c(sb_model** out) {
    return guard([&] { *out = new sb_model{fig3c_exact()}; });
}
int sb_model_ffn_stack(int n, int64_t hidden, int64_t batch, sb_model** out) {
    return guard([&] { *out = new sb_model{ffn_stack(n, hidden, batch)}; });
}
int sb_model_from_json(const char* text, sb_model** out) {
    return guard([&] { *out = new sb_model{load_model_json(text)}; });
}
int sb_model_to_json(const sb_model* m, char* buf, size_t cap, size_t* needed) {
    return guard([&] {
        std::string s = save_model_json(m->m);
        if (needed) *needed = s.size() + 1;
        if (buf && cap >= s.size() + 1) std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}
int sb_model_to_f32(sb_model* m) {
    return guard([&] { convert_to_f32(m->m); });
}
int sb_model_equal(const sb_model* a, const sb_model* b, int* eq) {
    return guard([&] { *eq = modules_equal(a->m, b->m) ? 1 : 0; });
}
int sb_estimate(const sb_model* m, int64_t batch, int world_size, int64_t device_memory_bytes, const double* constants,
                int64_t* ints, double* reals, char* text, size_t cap, size_t* needed) {
    return guard([&] {
        EstimateOptions o;
        o.batch = batch;
        o.world_size = world_size;
        o.device_memory_bytes = device_memory_bytes;
        if (constants)
            o.constants = CostConstants{constants[0], constants[1], constants[2], constants[3]};
        CostReport r = estimate(m->m, o);
        if (ints) {
            const int64_t v[8] = {r.flops, r.recompute_flops, r.launches, r.collective_bytes,
                                  r.param_bytes, r.activation_bytes, r.peak_memory_bytes, r.oom ? 1 : 0};
            std::memcpy(ints, v, sizeof(v));
        }
        if (reals) {
            reals[0] = r.step_time_s;
            reals[1] = r.throughput_samples_per_s;
        }
        std::string t = r.to_text();
        if (needed) *needed = t.size() + 1;
        if (text && cap >= t.size() + 1) std::memcpy(text, t.c_str(), t.size() + 1);
    });
}
int sb_model_apply_checkpoint_ratio(sb_model* m, const char* container, double ratio, int* count) {
    return guard([&] {
        int c = apply_checkpoint_ratio(m->m, container ? container : "", ratio);
        if (count) *count = c;
    });
}
int sb_model_free(sb_model* m) {
    delete m;
    return 0;
}
int sb_model_num_inputs(const sb_model* m, int* n) {
    return guard([&] { *n = (int)declared_inputs(*m->m.forward).size(); });
}
int sb_model_input_shape(const sb_model* m, int idx, int64_t* dims, int* ndims) {
    return guard([&] {
        auto specs = declared_inputs(*m->m.forward);
        auto& s = specs.at((size_t)idx);
        if (*ndims < (int)s.shape.size()) throw Error("dims buffer too small");
        for (size_t i = 0; i < s.shape.size(); ++i) dims[i] = s.shape[i];
        *ndims = (int)s.shape.size();
    });
}
int sb_model_random_input(const sb_model* m, int idx, uint64_t seed, uint64_t stream, double* out, size_t cap,
                          size_t* n) {
    return guard([&] {
        auto specs = declared_inputs(*m->m.forward);
        copy_out(random_tensor(specs.at((size_t)idx), seed, stream).data, out, cap, n);
    });
}
int sb_model_param_values(const sb_model* m, const char* dotted, int rank, double* out, size_t cap, size_t* n) {
    return guard([&] {
        const Param* p = m->m.resolve_param(dotted);
        if (!p) throw Error(std::string("unknown param '") + dotted + "'");
        copy_out(param_rank(*p, rank).data, out, cap, n);
    });
}

// ---------------------------------------------------------------- schedule
int sb_schedule_create(const sb_model* m, int world, sb_schedule** out) {
    return guard([&] { *out = new sb_schedule{Schedule(m->m, WorldConfig{world})}; });
}
int sb_schedule_at(const sb_schedule* s, const char* path, sb_schedule** out) {
    return guard([&] { *out = new sb_schedule{s->s.at(path)}; });
}
int sb_schedule_trace(sb_schedule* s, int flatten, const char* leaves) {
    return guard([&] {
        TraceSpec t;
        t.flatten = flatten != 0;
        t.leaves = csv(leaves);
        s->s.trace(t);
    });
}
int sb_schedule_replace(sb_schedule* s, const char* lib, const char* pattern) {
    return guard([&] {
        if (pattern && *pattern) s->s.replace_at(lib, pattern);
        else s->s.replace_with(lib);
    });
}
int sb_schedule_shard(sb_schedule* s, const char* params, int axis) {
    return guard([&] { s->s.shard(csv(params), axis); });
}
int sb_schedule_sync(sb_schedule* s, const char* type) {
    return guard([&] { s->s.sync(type); });
}
int sb_schedule_checkpoint(sb_schedule* s, const char* pattern) {
    return guard([&] {
        if (pattern && *pattern) s->s.checkpoint_at(pattern);
        else s->s.checkpoint();
    });
}
int sb_schedule_define_pattern(sb_schedule* s, const char* name, const char* graph_json) {
    return guard([&] { s->s.define_pattern(name, parse_graph_json(graph_json)); });
}
int sb_schedule_fuse(sb_schedule* s, const char* pattern, const char* backend) {
    return guard([&] { s->s.fuse_at(pattern, backend ? backend : "composed"); });
}
int sb_schedule_pipeline_split(sb_schedule* s, const char* after) {
    return guard([&] { s->s.pipeline_split(after); });
}
int sb_schedule_find(sb_schedule* s, const char* glob, int* count) {
    return guard([&] { *count = (int)s->s.find(std::string(glob)).size(); });
}
int sb_schedule_load_script(sb_schedule* s, const char* text) {
    return guard([&] { load_schedule_script(s->s, text); });
}
int sb_schedule_num_warnings(const sb_schedule* s, int* n) {
    return guard([&] { *n = (int)s->s.warnings().size(); });
}
int sb_schedule_apply(const sb_schedule* s, sb_model** out) {
    return guard([&] { *out = new sb_model{s->s.apply().model}; });
}
static void put_names(const std::vector<std::string>& v, char* buf, size_t cap, size_t* needed) {
    std::string t;
    for (auto& x : v) t += x + "\n";
    if (needed) *needed = t.size() + 1;
    if (buf && cap >= t.size() + 1) std::memcpy(buf, t.c_str(), t.size() + 1);
}
int sb_schedule_apply_pipeline(const sb_schedule* s, sb_pipeline** out) {
    return guard([&] {
        ApplyResult r = s->s.apply();
        *out = new sb_pipeline{build_stage_plan(r.model, r.pipeline_splits)};
    });
}
int sb_pipeline_num_stages(const sb_pipeline* p, int* n) {
    return guard([&] { *n = (int)p->p.stages.size(); });
}
int sb_pipeline_stage(const sb_pipeline* p, int i, sb_model** out) {
    return guard([&] { *out = new sb_model{p->p.stages.at((size_t)i).module}; });
}
int sb_pipeline_stage_io(const sb_pipeline* p, int i, int which, char* buf, size_t cap, size_t* needed) {
    return guard([&] {
        if (i < 0) put_names(which ? p->p.model_outputs : p->p.model_inputs, buf, cap, needed);
        else put_names(which ? p->p.stages.at((size_t)i).produces : p->p.stages.at((size_t)i).consumes, buf, cap, needed);
    });
}
int sb_pipeline_free(sb_pipeline* p) {
    delete p;
    return 0;
}
int sb_schedule_free(sb_schedule* s) {
    delete s;
    return 0;
}

// ---------------------------------------------------------------- executor
static DT dt_of(int d) {
    if (d == 0) return sbk::F32;
    if (d == 1) return sbk::BF16;
    throw Error("dtype must be 0 (fp32) or 1 (bf16)");
}
int sb_executor_create(const sb_model* m, int train, uint64_t seed, int world, int dtype, int fused, sb_executor** out) {
    return guard([&] {
        auto* e = new sb_executor;
        try {
            e->ex = std::make_unique<Executor>(m->m, train != 0, seed, world, dt_of(dtype), CommConfig{}, fused != 0);
        } catch (...) {
            delete e;
            throw;
        }
        e->world = world;
        *out = e;
    });
}
int sb_nccl_unique_id(void* out128) {
    return guard([&] {
        void* h = sb::nccl_handle();
        if (!h) throw Error("NCCL not available");
        auto f = (ncclResult_t(*)(ncclUniqueId*))dlsym(h, "ncclGetUniqueId");
        ncclUniqueId id;
        if (!f || f(&id) != ncclSuccess) throw Error("ncclGetUniqueId failed");
        std::memcpy(out128, &id, sizeof(id));
    });
}
int sb_executor_create_nccl(const sb_model* m, int train, uint64_t seed, int world, int rank, const void* uid, int dtype,
                            int fused, sb_executor** out) {
    return guard([&] {
        CommConfig c;
        c.nccl = true;
        c.rank = rank;
        c.unique_id.assign((const char*)uid, (const char*)uid + 128);
        auto* e = new sb_executor;
        try {
            e->ex = std::make_unique<Executor>(m->m, train != 0, seed, world, dt_of(dtype), c, fused != 0);
        } catch (...) {
            delete e;
            throw;
        }
        e->world = world;
        e->nccl = true;
        e->rank = rank;
        *out = e;
    });
}
// Host-only lowering (no device): the per-rank plan summary as JSON.
int sb_plan_describe(const sb_model* m, int train, uint64_t seed, int world, int rank, int dtype, int fused, char* buf,
                     size_t cap) {
    return guard([&] {
        LowerOptions lo;
        lo.rank = rank;
        lo.world = world;
        lo.train = train != 0;
        lo.seed = seed;
        lo.cdt = dt_of(dtype);
        lo.fused_kernels = fused != 0;
        Plan P = lower(m->m, lo);
        std::map<std::string, int> kinds;
        int folded = 0, bias_on = 0;
        for (auto& op : P.fwd) {
            kinds[k_str(op.k)]++;
            folded += op.dgelu_fused;
            bias_on += op.has_bias && op.bias_on;
        }
        std::ostringstream o;
        o << "{\"ops\": " << P.fwd.size() << ", \"regions\": " << P.regions.size() << ", \"ledger_bytes\": "
          << P.ledger_bytes << ", \"collectives_fwd\": " << P.collectives_fwd << ", \"gelu_folded\": " << folded
          << ", \"bias_added\": " << bias_on << ", \"params\": " << P.params.size() << ", \"structure\": \""
          << P.structure() << "\", \"kinds\": {";
        bool first = true;
        for (auto& [k, c] : kinds) {
            o << (first ? "" : ", ") << "\"" << k << "\": " << c;
            first = false;
        }
        o << "}}";
        std::string s = o.str();
        if (cap < s.size() + 1) throw Error("buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}
int sb_executor_free(sb_executor* e) {
    if (e && e->dloss) cudaFree(e->dloss);
    delete e;
    return 0;
}
int sb_executor_set_nan_guard(sb_executor* e, int on) {
    return guard([&] { e->ex->set_nan_guard(on != 0); });
}
int sb_executor_forward(sb_executor* e, const double* const* inputs, int n) {
    return guard([&] {
        e->grads.clear();
        e->ex->upload_inputs_raw(inputs, n);
        e->ex->forward_uploaded();
    });
}
int sb_executor_num_outputs(sb_executor* e, int rank, int* n) {
    return guard([&] { *n = (int)e->ex->outputs_of_rank(rank).size(); });
}
int sb_executor_output(sb_executor* e, int rank, int idx, double* out, size_t cap, size_t* n, int64_t* dims, int* ndims) {
    return guard([&] {
        auto outs = e->ex->outputs_of_rank(rank);
        auto& t = outs.at((size_t)idx);
        if (dims && ndims) {
            if (*ndims < (int)t.spec.shape.size()) throw Error("dims buffer too small");
            for (size_t i = 0; i < t.spec.shape.size(); ++i) dims[i] = t.spec.shape[i];
            *ndims = (int)t.spec.shape.size();
        }
        copy_out(t.data, out, cap, n);
    });
}
int sb_executor_backward(sb_executor* e) {
    return guard([&] { e->grads = e->ex->backward_all_ranks(); });
}
int sb_executor_num_grads(sb_executor* e, int rank, int* n) {
    return guard([&] { *n = (int)gmap(e, rank).params.size(); });
}
int sb_executor_grad_name(sb_executor* e, int rank, int idx, char* buf, size_t cap) {
    return guard([&] {
        auto& g = gmap(e, rank);
        if (idx < 0 || idx >= (int)g.params.size()) throw Error("grad index out of range");
        auto it = g.params.begin();
        std::advance(it, idx);
        if (cap < it->first.size() + 1) throw Error("name buffer too small");
        std::memcpy(buf, it->first.c_str(), it->first.size() + 1);
    });
}
int sb_executor_grad(sb_executor* e, int rank, const char* dotted, double* out, size_t cap, size_t* n) {
    return guard([&] {
        auto& g = gmap(e, rank);
        auto it = g.params.find(dotted);
        if (it == g.params.end()) throw Error(std::string("no gradient for '") + dotted + "'");
        copy_out(it->second.data, out, cap, n);
    });
}
int sb_executor_input_grad(sb_executor* e, int rank, int idx, double* out, size_t cap, size_t* n) {
    return guard([&] { copy_out(gmap(e, rank).inputs.at((size_t)idx).data, out, cap, n); });
}
int sb_executor_ledger(sb_executor* e, int64_t* bytes) {
    return guard([&] { *bytes = e->ex->ledger_bytes(); });
}
int sb_executor_collectives(sb_executor* e, int64_t* c) {
    return guard([&] { *c = e->ex->collective_invocations(); });
}
int sb_executor_upload_inputs(sb_executor* e, const double* const* inputs, int n) {
    return guard([&] { e->ex->upload_inputs_raw(inputs, n); });
}
int sb_executor_step(sb_executor* e, int use_graph) {
    return guard([&] {
        if (use_graph) {
            e->ex->launch_graph();
        } else {
            e->ex->run_forward();
            e->ex->run_backward();
        }
    });
}
int sb_executor_step_loss(sb_executor* e, int use_graph, float* loss_host) {
    return guard([&] {
        if (!e->dloss && cudaMalloc(&e->dloss, 4) != cudaSuccess) throw Error("cudaMalloc failed");
        if (use_graph) {
            e->ex->launch_graph();
        } else {
            e->ex->run_forward();
            e->ex->run_backward();
        }
        e->ex->enqueue_loss(e->dloss);
        if (cudaMemcpyAsync(loss_host, e->dloss, 4, cudaMemcpyDeviceToHost, (cudaStream_t)e->ex->stream()) != cudaSuccess)
            throw Error("loss copy failed");
        e->ex->synchronize();
    });
}
int sb_executor_time_steps(sb_executor* e, int steps, int use_graph, float* ms) {
    return guard([&] { *ms = e->ex->time_steps(steps, use_graph != 0); });
}
int sb_executor_time_e2e(sb_executor* e, int steps, const double* const* inputs, int n_inputs, int use_graph,
                         float* ms, float* loss) {
    return guard([&] { *ms = e->ex->time_e2e(steps, inputs, n_inputs, use_graph != 0, loss); });
}
int sb_executor_kernels_per_step(sb_executor* e, int* n) {
    return guard([&] { *n = e->ex->kernel_launches_per_step(); });
}
int sb_executor_synchronize(sb_executor* e) {
    return guard([&] { e->ex->synchronize(); });
}
int sb_executor_stream(sb_executor* e, void** s) {
    return guard([&] { *s = e->ex->stream(); });
}
int sb_executor_describe(sb_executor* e, char* buf, size_t cap) {
    return guard([&] {
        std::string s = e->ex->describe();
        if (cap < s.size() + 1) throw Error("buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}
int sb_executor_profile(sb_executor* e, char* buf, size_t cap) {
    return guard([&] {
        auto p = e->ex->profile_step();
        std::ostringstream o;
        o << "{";
        for (size_t i = 0; i < p.size(); ++i) o << (i ? ", " : "") << "\"" << p[i].first << "\": " << p[i].second;
        o << "}";
        std::string s = o.str();
        if (cap < s.size() + 1) throw Error("buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}
int sb_executor_device_bytes(sb_executor* e, int64_t* b) {
    return guard([&] { *b = (int64_t)e->ex->device_bytes(); });
}

// ------------------------------------------------------------------ kernels
static void* g_gemm_ws = nullptr;
static size_t g_gemm_ws_bytes = 0;
static sbk::DT kdt(int d) {
    if (d < 0 || d > 2) throw Error("dtype code must be 0, 1 or 2");
    return (sbk::DT)d;
}
int sb_gemm(const void* A, int ta, int64_t sAb, int64_t sAm, int64_t sAk, const void* B, int tb, int64_t sBb, int64_t sBk,
            int64_t sBn, void* C, int tc, int64_t sCb, int64_t sCm, int64_t sCn, int64_t batch, int64_t M, int64_t N,
            int64_t K, float alpha, int accumulate, const void* bias, int epilogue, void* aux, void* stream) {
    return guard([&] {
        sbk::Gemm g;
        g.A = A;
        g.ta = kdt(ta);
        g.sAb = sAb;
        g.sAm = sAm;
        g.sAk = sAk;
        g.B = B;
        g.tb = kdt(tb);
        g.sBb = sBb;
        g.sBk = sBk;
        g.sBn = sBn;
        g.C = C;
        g.tc = kdt(tc);
        g.sCb = sCb;
        g.sCm = sCm;
        g.sCn = sCn;
        g.batch = batch;
        g.M = M;
        g.N = N;
        g.K = K;
        g.alpha = alpha;
        g.accumulate = accumulate != 0;
        g.bias = bias;
        g.tbias = g.tc == sbk::F32 ? g.ta : g.tc;
        g.epilogue = epilogue;
        g.aux = aux;
        g.ws = g_gemm_ws;
        g.ws_bytes = g_gemm_ws_bytes;
        sbk::gemm(g, (cudaStream_t)stream);
    });
}
int sb_gemm_engine(void) { return sbk::gemm_last_engine(); }
int sb_gemm_set_workspace(void* ws, size_t bytes) {
    g_gemm_ws = ws;
    g_gemm_ws_bytes = bytes;
    return 0;
}
int sb_gemm_force_simt(int on) {
    sbk::gemm_force_simt(on != 0);
    return 0;
}
int sb_set_mask_blocks(int n) {
    sbk::set_mask_blocks(n);
    return 0;
}
int sb_gemm_set_tile_n(int bn) {
    sbk::gemm2_set_tile_n(bn);
    return 0;
}
int sb_gemm_set_engine(int max_engine) {
    sbk::gemm_set_engine(max_engine);
    return 0;
}
int sb_attn_set_engine(int max_engine) {
    sbk::attn_set_engine(max_engine);
    return 0;
}
int sb_attn_engine(int bwd) { return sbk::attn_last_engine(bwd); }
int sb_attn_dropout_mask(uint32_t* bits, int64_t B, int64_t S, int64_t nh, uint64_t exec_seed, uint64_t node_seed,
                         double p, void* stream) {
    return guard([&] {
        u64 s1 = hash_combine(hash_combine(exec_seed, node_seed), 0xd0);
        sbk::dropout_mask_dual(bits, B * nh, S, s1, dropout_threshold(p), (cudaStream_t)stream);
    });
}
size_t sb_attn_bwd_workspace(int64_t B, int64_t S, int64_t nh, int64_t hd) { return sbk::attn_bwd_workspace(B, S, nh, hd); }
int sb_dropout_mask(uint32_t* bits, int64_t n, uint64_t exec_seed, uint64_t node_seed, double p, void* stream) {
    return guard([&] {
        u64 s1 = hash_combine(hash_combine(exec_seed, node_seed), 0xd0);
        sbk::dropout_mask(bits, n, s1, dropout_threshold(p), (cudaStream_t)stream);
    });
}
int sb_layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd, int dtype,
                     int64_t rows, int64_t n, float eps, void* stream) {
    return guard([&] {
        sbk::layernorm_fwd(x, gamma, beta, kdt(dtype), y, mean, rstd, kdt(dtype), rows, n, eps, (cudaStream_t)stream);
    });
}
int sb_bias_dropout_residual_ln_fwd(const void* partial, const void* bias, const void* residual, const void* gamma,
                                    const void* beta, void* sum, void* y, float* mean, float* rstd, int dtype, int64_t rows,
                                    int64_t n, float eps, uint64_t exec_seed, uint64_t node_seed, double p, void* stream) {
    return guard([&] {
        u64 s1 = hash_combine(hash_combine(exec_seed, node_seed), 0xd0);
        u64 thr = p > 0 ? dropout_threshold(p) : 0;
        sbk::bias_dropout_residual_ln_fwd(partial, bias, residual, gamma, beta, kdt(dtype), sum, y, mean, rstd, kdt(dtype),
                                          rows, n, eps, s1, thr, (float)(1.0 / (1.0 - p)), (cudaStream_t)stream);
    });
}
int sb_layernorm_bwd(const void* x, const float* mean, const float* rstd, const void* gamma, const void* g, void* gx,
                     float* dgamma, float* dbeta, int dtype, int64_t rows, int64_t n, int gx_accumulate, void* workspace,
                     void* stream) {
    return guard([&] {
        sbk::layernorm_bwd(x, mean, rstd, gamma, kdt(dtype), g, kdt(dtype), gx, dgamma, dbeta, kdt(dtype), rows, n,
                           (float*)workspace, (cudaStream_t)stream, gx_accumulate != 0, false);
    });
}
size_t sb_layernorm_bwd_workspace(int64_t rows, int64_t n) {
    return std::max(sbk::layernorm_bwd_workspace(rows, n), (size_t)296 * 3 * (size_t)n * 4);
}
int sb_bias_dropout_residual_ln_bwd(const void* sum, const float* mean, const float* rstd, const void* gamma,
                                    const void* g, void* g_res, void* g_partial, float* dbias, float* dgamma,
                                    float* dbeta, int dtype, int64_t rows, int64_t n, uint64_t exec_seed,
                                    uint64_t node_seed, double p, void* workspace, void* stream) {
    return guard([&] {
        u64 s1 = hash_combine(hash_combine(exec_seed, node_seed), 0xd0);
        u64 thr = p > 0 ? dropout_threshold(p) : 0;
        sbk::bias_dropout_residual_ln_bwd(sum, mean, rstd, gamma, kdt(dtype), g, g_res, g_partial, false, dbias, dgamma,
                                          dbeta, kdt(dtype), rows, n, s1, thr, (float)(1.0 / (1.0 - p)),
                                          (float*)workspace, (cudaStream_t)stream, false, false);
    });
}
size_t sb_bias_dropout_residual_ln_bwd_workspace(int64_t rows, int64_t n) {
    return std::max(sbk::bdrln_bwd_workspace(rows, n), (size_t)296 * 3 * (size_t)n * 4);
}
int sb_bias_gelu_fwd(const void* x, const void* bias, void* y, void* pre, int dtype, int64_t rows, int64_t n,
                     void* stream) {
    return guard([&] { sbk::bias_gelu_fwd(x, bias, y, pre, kdt(dtype), rows, n, (cudaStream_t)stream); });
}
int sb_bias_gelu_bwd(const void* pre, const void* g, void* gx, float* dbias, int dtype, int64_t rows, int64_t n,
                     void* workspace, void* stream) {
    return guard([&] {
        sbk::bias_gelu_bwd(pre, g, gx, dbias, kdt(dtype), rows, n, (float*)workspace, (cudaStream_t)stream);
    });
}
size_t sb_bias_gelu_bwd_workspace(int64_t rows, int64_t n) { return sbk::bias_grad_workspace(rows, n); }
int sb_embedding_fwd(const double* ids, int64_t n_ids, const void* table, int dtype, int64_t dim, int64_t vocab,
                     int64_t row0, int64_t local_rows, void* out, void* stream) {
    return guard([&] {
        sbk::embedding_fwd(ids, n_ids, table, kdt(dtype), dim, vocab, row0, local_rows, out, (cudaStream_t)stream);
    });
}
int sb_embedding_bwd(const double* ids, int64_t n_ids, const void* g, int dtype, int64_t dim, int64_t vocab,
                     int64_t row0, int64_t local_rows, float* gtable, void* workspace, void* stream) {
    return guard([&] {
        sbk::embedding_bwd(ids, n_ids, g, kdt(dtype), dim, vocab, row0, local_rows, gtable, workspace,
                           (cudaStream_t)stream);
    });
}
size_t sb_embedding_bwd_workspace(int64_t n_ids, int64_t dim) { return sbk::embedding_bwd_workspace(n_ids, dim); }
int sb_allreduce_local(const void* const* srcs, void* const* dsts, int ranks, int dtype, int64_t n, int accumulate,
                       void* stream) {
    return guard([&] {
        if (ranks < 1 || ranks > 16) throw Error("sb_allreduce_local: 1..16 ranks");
        sbk::sum_ranks(srcs, dsts, ranks, kdt(dtype), n, accumulate != 0, (cudaStream_t)stream);
    });
}
static sbk::Attn mk_attn(const void* q, const void* k, const void* v, void* o, int64_t ld_qkv, int64_t ld_o, float* lse,
                         int64_t B, int64_t S, int64_t nh, int64_t hd, float scale, uint64_t es, uint64_t ns, double p,
                         int dtype) {
    sbk::Attn a;
    a.q = q;
    a.k = k;
    a.v = v;
    a.o = o;
    a.ld_q = a.ld_k = a.ld_v = ld_qkv;
    a.ld_o = ld_o;
    a.lse = lse;
    a.B = B;
    a.S = S;
    a.nh = nh;
    a.hd = hd;
    a.scale = scale;
    a.s1 = p > 0 ? hash_combine(hash_combine(es, ns), 0xd0) : 0;
    a.thr = p > 0 ? dropout_threshold(p) : 0;
    a.dscale = (float)(1.0 / (1.0 - p));
    a.t = kdt(dtype);
    return a;
}
int sb_attn_fwd_ex(const void* q, const void* k, const void* v, void* o, int64_t ld_qkv, int64_t ld_o, float* lse,
                   int64_t B, int64_t S, int64_t nh, int64_t hd, float scale, uint64_t es, uint64_t ns, double p, int dtype,
                   const uint32_t* keep_bits, int flags, void* stream) {
    return guard([&] {
        if (flags & ~SB_ATTN_CAUSAL) throw Error("sb_attn_fwd_ex: unknown flags");
        sbk::Attn a = mk_attn(q, k, v, o, ld_qkv, ld_o, lse, B, S, nh, hd, scale, es, ns, p, dtype);
        a.mask = keep_bits;
        a.causal = flags & SB_ATTN_CAUSAL;
        sbk::attn_fwd(a, (cudaStream_t)stream);
    });
}
int sb_attn_fwd(const void* q, const void* k, const void* v, void* o, int64_t ld_qkv, int64_t ld_o, float* lse, int64_t B,
                int64_t S, int64_t nh, int64_t hd, float scale, uint64_t es, uint64_t ns, double p, int dtype,
                const uint32_t* keep_bits, void* stream) {
    return sb_attn_fwd_ex(q, k, v, o, ld_qkv, ld_o, lse, B, S, nh, hd, scale, es, ns, p, dtype, keep_bits, 0, stream);
}
int sb_attn_bwd_ex(const void* q, const void* k, const void* v, const void* o, int64_t ld_qkv, int64_t ld_o,
                   const float* lse, const void* dout, void* dq, void* dk, void* dv, void* workspace, int64_t B, int64_t S,
                   int64_t nh, int64_t hd, float scale, uint64_t es, uint64_t ns, double p, int dtype,
                   const uint32_t* keep_bits, int acc_mask, int flags, void* stream) {
    return guard([&] {
        if (flags & ~SB_ATTN_CAUSAL) throw Error("sb_attn_bwd_ex: unknown flags");
        sbk::Attn a = mk_attn(q, k, v, (void*)o, ld_qkv, ld_o, (float*)lse, B, S, nh, hd, scale, es, ns, p, dtype);
        a.acc_mask = acc_mask;
        a.mask = keep_bits;
        a.mask_t = keep_bits && S % 128 == 0 ? keep_bits + (B * nh * S * S) / 32 : nullptr;
        a.causal = flags & SB_ATTN_CAUSAL;
        sbk::attn_bwd(a, dout, ld_o, dq, dk, dv, ld_qkv, ld_qkv, ld_qkv, workspace, (cudaStream_t)stream);
    });
}
int sb_attn_bwd(const void* q, const void* k, const void* v, const void* o, int64_t ld_qkv, int64_t ld_o, const float* lse,
                const void* dout, void* dq, void* dk, void* dv, void* workspace, int64_t B, int64_t S, int64_t nh, int64_t hd,
                float scale, uint64_t es, uint64_t ns, double p, int dtype, const uint32_t* keep_bits, int acc_mask,
                void* stream) {
    return sb_attn_bwd_ex(q, k, v, o, ld_qkv, ld_o, lse, dout, dq, dk, dv, workspace, B, S, nh, hd, scale, es, ns, p, dtype,
                          keep_bits, acc_mask, 0, stream);
}

}  // extern "C"

// ------------------------------------------------------- pipeline executor (f1)
extern "C" {
int sb_pipeline_executor_create_tp(const sb_pipeline* p, int micro_batches, int tp, int train, uint64_t seed,
                                   int dtype, const int* devices, int fused, sb_pipeline_executor** out) {
    return guard([&] {
        std::vector<int> devs;
        if (devices) devs.assign(devices, devices + p->p.stages.size());
        auto* e = new sb_pipeline_executor;
        e->ex = std::make_unique<PipelineExecutor>(p->p, micro_batches, train != 0, seed, dtype ? sbk::BF16 : sbk::F32,
                                                   devs, fused != 0, tp);
        *out = e;
    });
}
int sb_pipeline_executor_create_dist(const sb_pipeline* p, int micro_batches, int tp, int train, uint64_t seed,
                                     int dtype, int fused, int rank, int world, const void* pp_uid128,
                                     const void* tp_uid128, sb_pipeline_executor** out) {
    return guard([&] {
        PipeDist d;
        d.rank = rank;
        d.world = world;
        d.pp_uid.assign((const char*)pp_uid128, (const char*)pp_uid128 + 128);
        if (tp > 1) {
            if (!tp_uid128) throw Error("tp > 1 needs the stage's tensor-parallel unique id");
            d.tp_uid.assign((const char*)tp_uid128, (const char*)tp_uid128 + 128);
        }
        auto* e = new sb_pipeline_executor;
        e->ex = std::make_unique<PipelineExecutor>(p->p, micro_batches, train != 0, seed, dtype ? sbk::BF16 : sbk::F32,
                                                   std::vector<int>{}, fused != 0, tp, &d);
        *out = e;
    });
}
int sb_pipeline_program(const sb_pipeline* p, int micro_batches, int tp, int rank, char* buf, size_t cap,
                        size_t* needed) {
    return guard([&] {
        // element count of every stage-boundary value per micro-batch, from a consumer's declared input shape
        std::map<std::string, long long> numel;
        for (auto& st : p->p.stages)
            for (size_t i = 0; i < st.consumes.size(); ++i) {
                const auto& at = st.module.forward->at(st.module.forward->inputs[i]).attrs;
                auto it = at.find("shape");
                if (it == at.end()) continue;
                long long n = 1;
                for (auto d : std::get<std::vector<i64>>(it->second)) n *= d;
                numel[st.consumes[i]] = n / micro_batches;
            }
        static const char* kinds[] = {"fwd_recv", "fwd_run", "fwd_send", "bwd_recv", "bwd_run", "bwd_send"};
        std::ostringstream o;
        for (auto& st : pipe_program(p->p, micro_batches, tp, rank))
            o << kinds[(int)st.kind] << " " << st.m << " " << st.idx << " " << st.peer << " "
              << (st.value.empty() ? "-" : st.value) << " " << (st.value.empty() ? 0 : numel[st.value]) << "\n";
        const std::string t = o.str();
        *needed = t.size() + 1;
        if (buf && cap >= t.size() + 1) std::memcpy(buf, t.c_str(), t.size() + 1);
    });
}
int sb_pipeline_executor_create(const sb_pipeline* p, int micro_batches, int train, uint64_t seed, int dtype,
                                const int* devices, int fused, sb_pipeline_executor** out) {
    return sb_pipeline_executor_create_tp(p, micro_batches, 1, train, seed, dtype, devices, fused, out);
}
int sb_pipeline_executor_forward(sb_pipeline_executor* e, const double* const* inputs, int n) {
    return guard([&] {
        e->grads.clear();
        e->outs = e->ex->forward_raw(inputs, n);
    });
}
int sb_pipeline_executor_num_outputs(sb_pipeline_executor* e, int* n) {
    return guard([&] { *n = (int)e->outs.size(); });
}
int sb_pipeline_executor_output(sb_pipeline_executor* e, int idx, double* out, size_t cap, size_t* n, int64_t* dims,
                                int* ndims) {
    return guard([&] {
        auto& t = e->outs.at((size_t)idx);
        if (dims && ndims) {
            if (*ndims < (int)t.spec.shape.size()) throw Error("dims buffer too small");
            for (size_t i = 0; i < t.spec.shape.size(); ++i) dims[i] = t.spec.shape[i];
            *ndims = (int)t.spec.shape.size();
        }
        copy_out(t.data, out, cap, n);
    });
}
int sb_pipeline_executor_backward(sb_pipeline_executor* e) {
    return guard([&] { e->grads = e->ex->backward(); });
}
static GradMap& pgmap(sb_pipeline_executor* e, int stage) {
    if (e->grads.empty()) throw Error("no gradients: call backward first");
    if (stage < 0 || stage >= (int)e->grads.size()) throw Error("stage slot out of range (stage * tp + rank)");
    return e->grads[(size_t)stage];
}
int sb_pipeline_executor_num_grads(sb_pipeline_executor* e, int stage, int* n) {
    return guard([&] { *n = (int)pgmap(e, stage).params.size(); });
}
int sb_pipeline_executor_grad_name(sb_pipeline_executor* e, int stage, int idx, char* buf, size_t cap) {
    return guard([&] {
        auto& g = pgmap(e, stage);
        if (idx < 0 || idx >= (int)g.params.size()) throw Error("grad index out of range");
        auto it = g.params.begin();
        std::advance(it, idx);
        if (cap < it->first.size() + 1) throw Error("name buffer too small");
        std::memcpy(buf, it->first.c_str(), it->first.size() + 1);
    });
}
int sb_pipeline_executor_grad(sb_pipeline_executor* e, int stage, const char* dotted, double* out, size_t cap, size_t* n) {
    return guard([&] {
        auto& g = pgmap(e, stage);
        auto it = g.params.find(dotted);
        if (it == g.params.end()) throw Error(std::string("no gradient for '") + dotted + "'");
        copy_out(it->second.data, out, cap, n);
    });
}
int sb_pipeline_executor_num_input_grads(sb_pipeline_executor* e, int stage, int* n) {
    return guard([&] { *n = (int)pgmap(e, stage).inputs.size(); });
}
int sb_pipeline_executor_input_grad(sb_pipeline_executor* e, int stage, int idx, double* out, size_t cap, size_t* n) {
    return guard([&] { copy_out(pgmap(e, stage).inputs.at((size_t)idx).data, out, cap, n); });
}
int sb_pipeline_executor_time_steps(sb_pipeline_executor* e, int steps, float* ms) {
    return guard([&] { *ms = e->ex->time_steps(steps); });
}
int sb_pipeline_executor_time_steps_ex(sb_pipeline_executor* e, int steps, int use_graph, float* ms) {
    return guard([&] { *ms = e->ex->time_steps(steps, use_graph != 0); });
}
int sb_executor_allreduce(sb_executor* e, void* buf, int64_t n, int dtype, void* stream) {
    return guard([&] { e->ex->all_reduce_device(buf, n, kdt(dtype), stream); });
}
int sb_pipeline_executor_free(sb_pipeline_executor* e) {
    delete e;
    return 0;
}
}  // extern "C"
