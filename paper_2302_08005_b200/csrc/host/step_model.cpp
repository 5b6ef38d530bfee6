// The reference's analytical cost model (proj/src/costmodel.cpp) restated over
// this library's IR: a walk of the scheduled module that counts forward flops
// (per-op forms of costmodel.cpp:40-56 and the module forms of :100-150),
// kernel launches (fused composites and EfficientAttention count once),
// ring-collective wire bytes (:25-33, :58-70, sync_backward :81-84) and
// activation bytes under the executor's ledger rule (checkpointed regions keep
// only their boundary tensors, :85-95), then the step-time / memory formulas of
// finish() (:229-255).
#include "step_model.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <sstream>

#include "schedule.hpp"

namespace sb {

namespace {

i64 vbytes(const ValueSpec& v) {
    i64 b = 0;
    for (auto& p : v.parts) b += p.numel() * dtype_bytes(p.dtype);
    return b;
}
i64 tbytes(const TensorSpec& t) { return t.numel() * dtype_bytes(t.dtype); }

i64 ring_allreduce_wire(i64 payload, int world) { return world <= 1 ? 0 : 2 * (world - 1) * payload / world; }
i64 ring_allgather_wire(i64 gathered, int world) { return world <= 1 ? 0 : (world - 1) * gathered / world; }

struct Walker {
    const EstimateOptions& opts;
    i64 flops = 0, recompute = 0, launches = 0, act = 0, fwd_wire = 0, bwd_wire = 0, params = 0;
    bool counting = true;  // off inside checkpointed regions

    static i64 op_flops(const Node& n, const std::vector<const ValueSpec*>& args, const ValueSpec& out) {
        const std::string& op = n.op;
        if (op == "matmul") {
            const TensorSpec& a = args[0]->one();
            return 2 * out.one().numel() * a.shape[(size_t)a.rank() - 1];
        }
        if (op == "add" || op == "mul" || op == "scale" || op == "relu" || op == "gelu" || op == "dropout")
            return out.one().numel();
        if (op == "softmax") return 5 * out.one().numel();
        if (op == "layernorm") return 8 * out.one().numel();
        if (op == "reduce_sum") return args[0]->one().numel();
        return 0;  // data movement and collectives
    }

    void collective(const Node& n, const std::vector<const ValueSpec*>& args, const ValueSpec& out) {
        i64 w = 0;
        if (n.op == "all_reduce") w = ring_allreduce_wire(vbytes(*args[0]), opts.world_size);
        else if (n.op == "all_gather") w = ring_allgather_wire(vbytes(out), opts.world_size);
        fwd_wire += w;
        bwd_wire += w;  // the gradient collective mirrors it
    }

    void add_params(const Module& m) {
        for (auto& p : m.params) params += tbytes(p.spec);
        for (auto& c : m.children) add_params(*c.mod);
    }

    ValueSpec module(const Module& m, const std::vector<TensorSpec>& ins) {
        const bool ckpt = get_flag(m.attrs, "checkpoint") || m.kind == "EfficientAttention";
        if (get_flag(m.attrs, "sync_backward") && opts.world_size > 1 && !ins.empty())
            bwd_wire += ring_allreduce_wire(tbytes(ins[0]), opts.world_size);
        if (ckpt && counting) {  // region rule: boundary inputs and outputs retained, internals recomputed
            counting = false;
            const i64 before = flops;
            ValueSpec out = body(m, ins);
            counting = true;
            recompute += flops - before;
            for (auto& t : ins) act += tbytes(t);
            act += vbytes(out);
            return out;
        }
        return body(m, ins);
    }

    ValueSpec body(const Module& m, const std::vector<TensorSpec>& ins) {
        const std::string& k = m.kind;
        if (k == "Linear" || k == "FusedQKV") {
            ValueSpec out = module_out_spec(m, ins);
            const Param* w = m.param("weight");
            const i64 rows = ins[0].numel() / w->spec.shape[1];
            flops += 2 * rows * w->spec.shape[0] * w->spec.shape[1];
            if (m.param("bias")) flops += rows * w->spec.shape[0];
            launches += 1;
            if (counting) act += vbytes(out);
            return out;
        }
        if (k == "LayerNorm" || k == "Dropout" || k == "Embedding") {
            ValueSpec out = module_out_spec(m, ins);
            if (k == "LayerNorm") flops += 8 * out.one().numel();
            if (k == "Dropout") flops += out.one().numel();
            launches += 1;
            if (counting) act += vbytes(out);
            return out;
        }
        if (k == "EfficientAttention") {  // one fused kernel; flops follow its reference graph
            Module ref = make_attention_core(get_int(m.attrs, "head_dim").value_or(1), get_double(m.attrs, "p").value_or(0.0),
                                             (u64)get_int(m.attrs, "seed").value_or(0));
            const bool saved = counting;
            counting = false;
            const i64 l0 = launches;
            ValueSpec out = graph(*ref.forward, ref, ins);
            launches = l0 + 1;
            counting = saved;
            return out;
        }
        const i64 l0 = launches;  // composite; a fused composite is one launch
        ValueSpec out = graph(*m.forward, m, ins);
        if (get_flag(m.attrs, "fused")) launches = l0 + 1;
        return out;
    }

    ValueSpec graph(const Graph& g, const Module& ctx, const std::vector<TensorSpec>& ins) {
        std::map<int, ValueSpec> env;
        size_t next = 0;
        ValueSpec result;
        for (auto& n : g.nodes) {
            switch (n.kind) {
                case NK::Input: env[n.id] = ValueSpec(ins[next++]); break;
                case NK::ParamRef: {
                    const Param* p = ctx.resolve_param(n.target);
                    if (!p) throw Error("unknown param '" + n.target + "'");
                    env[n.id] = ValueSpec(p->spec);
                    break;
                }
                case NK::CallOp: {
                    std::vector<const ValueSpec*> a;
                    for (int x : n.args) a.push_back(&env.at(x));
                    ValueSpec out = infer_op(n.op, a, n.attrs, n.id);
                    flops += op_flops(n, a, out);
                    launches += 1;
                    collective(n, a, out);
                    if (counting) act += vbytes(out);
                    env[n.id] = std::move(out);
                    break;
                }
                case NK::CallModule: {
                    const Module* s = ctx.resolve(n.target);
                    if (!s) throw Error("unknown submodule '" + n.target + "'");
                    std::vector<TensorSpec> si;
                    for (int x : n.args) si.push_back(env.at(x).one());
                    env[n.id] = module(*s, si);
                    break;
                }
                case NK::GetItem: {
                    const ValueSpec& v = env.at(n.args[0]);
                    env[n.id] = ValueSpec(v.parts.at((size_t)get_int(n.attrs, "index").value_or(0)));
                    break;
                }
                case NK::Output: {
                    std::vector<TensorSpec> parts;
                    bool any_tuple = false;
                    for (int x : n.args) {
                        const ValueSpec& v = env.at(x);
                        any_tuple |= v.tuple;
                        parts.insert(parts.end(), v.parts.begin(), v.parts.end());
                    }
                    result = (n.args.size() == 1 && !any_tuple) ? ValueSpec(parts[0]) : ValueSpec::of_tuple(parts);
                    break;
                }
            }
        }
        return result;
    }
};

}  // namespace

CostReport estimate(const Module& model, const EstimateOptions& opts) {
    if (!model.forward) throw Error("estimate needs a composite root");
    Walker w{opts};
    w.add_params(model);
    std::vector<TensorSpec> ins = declared_inputs(*model.forward);
    if (opts.batch > 0)
        for (auto& s : ins) {
            if (s.rank() < 1) throw Error("cannot apply batch override to scalar input");
            s.shape[0] = opts.batch;
        }
    w.graph(*model.forward, model, ins);
    const i64 rows = ins.empty() || ins[0].rank() < 1 ? 1 : ins[0].shape[0];

    CostReport r;  // finish() (costmodel.cpp:229-255)
    r.flops = w.flops;
    r.recompute_flops = w.recompute;
    r.launches = w.launches;
    r.collective_bytes = w.fwd_wire + w.bwd_wire;
    r.param_bytes = w.params;
    r.activation_bytes = w.act;
    const CostConstants& c = opts.constants;
    const double fwd = (double)w.flops / c.device_flops_per_s + (double)w.launches * c.kernel_launch_overhead_s;
    const double bwd = (double)(2 * w.flops + w.recompute) / c.device_flops_per_s +
                       (double)(2 * w.launches) * c.kernel_launch_overhead_s;
    const double comm = (double)r.collective_bytes / c.link_bytes_per_s;
    r.step_time_s = fwd + bwd + comm;
    const double grads = (double)w.params;
    r.peak_memory_bytes = w.params + (i64)(c.optimizer_state_multiplier * grads) + (i64)grads + w.act;
    r.oom = r.peak_memory_bytes > opts.device_memory_bytes;
    r.throughput_samples_per_s = r.oom ? 0.0 : (double)rows / std::max(r.step_time_s, 1e-30);
    return r;
}

int apply_checkpoint_ratio(Module& model, const std::string& container, double ratio) {  // costmodel.cpp:310-324
    Module* c = model.resolve(container);
    if (!c) throw Error("unknown module path '" + container + "'");
    const int layers = (int)c->children.size();
    const int count = std::clamp((int)std::floor(ratio * layers), 0, layers);
    for (int i = 0; i < layers; ++i) {
        if (i < count) c->children[(size_t)i].mod->attrs["checkpoint"] = (i64)1;
        else c->children[(size_t)i].mod->attrs.erase("checkpoint");
    }
    return count;
}

std::string CostReport::to_text() const {  // costmodel.cpp:326-338
    std::ostringstream o;
    o << "step_time_s           " << step_time_s << "\n";
    o << "flops                 " << flops << "\n";
    o << "recompute_flops       " << recompute_flops << "\n";
    o << "launches              " << launches << "\n";
    o << "collective_bytes      " << collective_bytes << "\n";
    o << "param_bytes           " << param_bytes << "\n";
    o << "activation_bytes      " << activation_bytes << "\n";
    o << "peak_memory_bytes     " << peak_memory_bytes << "\n";
    o << "oom                   " << (oom ? "true" : "false") << "\n";
    o << "throughput_samples_s  " << throughput_samples_per_s << "\n";
    return o.str();
}

}  // namespace sb
