// GPipe training step over pipeline_split stages (see pipeline_exec.hpp).
#include "pipeline_exec.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <tuple>
#include <stdexcept>

#include "../kernels/kernels.hpp"

namespace sb {

namespace {
void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(std::string("pipeline: ") + what + ": " + cudaGetErrorString(e));
}
#define PCK(x) ck((x), #x)

// the executor plans from declared input shapes: a stage runs on 1/M of the batch
Module micro_module(const Module& m, int micro) {
    Module out = m;
    if (micro == 1) return out;
    for (auto& n : out.forward->nodes) {
        if (n.kind != NK::Input) continue;
        auto it = n.attrs.find("shape");
        if (it == n.attrs.end()) throw Error("pipeline: stage input without a declared shape");
        auto shape = std::get<std::vector<i64>>(it->second);
        if (shape.empty() || shape[0] % micro)
            throw Error("pipeline: batch dimension not divisible into " + std::to_string(micro) + " micro-batches");
        shape[0] /= micro;
        it->second = shape;
    }
    return out;
}

struct Value {
    std::string name;
    int producer = -1;  // stage, or -1: a model input
    int out_idx = -1;   // output index of the producer / model input index
    int dev = 0;
    DT dt = sbk::F64;
    i64 numel = 0;
    std::vector<i64> shape;  // per micro-batch
    int model_out = -1;      // index among the model outputs, or -1
    std::vector<std::pair<int, int>> consumers;  // (stage, input idx)
    std::vector<void*> buf;   // [m] the value (producer dtype), on dev
    std::vector<void*> gbuf;  // [m] d loss / d value, fp32, on dev (produced values only)
    cudaEvent_t ginit = nullptr;
};

struct StageRt {
    std::unique_ptr<Executor> ex;
    int dev = 0;
    cudaStream_t st = nullptr;
    std::vector<int> in_val;            // consumed value per input
    std::vector<int> out_val;           // produced value per output
    std::vector<void*> tmp_in;          // per input: peer staging on this device (or null)
    std::vector<void*> tmp_grad;        // per input: peer staging of the input gradient on the producer's device
    std::vector<cudaEvent_t> ev_fwd, ev_bwd;  // [m]
    std::vector<std::vector<void*>> gin;      // [m][input]: model-input gradients (fp32, on dev)
};

size_t bytes_of(DT dt, i64 n) { return (size_t)n * (size_t)sbk::dt_bytes(dt); }

// Producer of every stage input and consumers of every stage output of a plan. A name
// may be produced by several stages (the partitioner threads a value through the stages
// in between, pipeline.cpp:343-420): a stage consumes the latest producer before it, as
// run_pipeline's environment does (executor.cpp:1541-1560).
struct Topo {
    std::vector<std::vector<std::pair<int, int>>> in_prod;               // [stage][input] -> (stage, output) or (-1, k)
    std::map<std::pair<int, int>, std::vector<std::pair<int, int>>> cons;  // (stage, output) -> [(stage, input)]
    explicit Topo(const StagePlan& plan) {
        std::map<std::string, std::pair<int, int>> cur;
        for (size_t k = 0; k < plan.model_inputs.size(); ++k) cur[plan.model_inputs[k]] = {-1, (int)k};
        for (size_t s = 0; s < plan.stages.size(); ++s) {
            const Stage& st = plan.stages[s];
            in_prod.emplace_back();
            for (size_t i = 0; i < st.consumes.size(); ++i) {
                auto it = cur.find(st.consumes[i]);
                if (it == cur.end()) throw Error("pipeline stage consumes unknown value '" + st.consumes[i] + "'");
                in_prod.back().push_back(it->second);
                if (it->second.first >= 0) cons[it->second].push_back({(int)s, (int)i});
            }
            for (size_t o = 0; o < st.produces.size(); ++o) cur[st.produces[o]] = {(int)s, (int)o};
        }
    }
};

void* dev_alloc(int dev, size_t bytes) {
    PCK(cudaSetDevice(dev));
    void* p = nullptr;
    PCK(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
    return p;
}
}  // namespace

void* p2p_comm_create(int world, int rank, const std::vector<char>& uid);  // executor.cpp (NCCL)
void p2p_comm_destroy(void* c);
void p2p_send(void* c, const void* buf, i64 n, DT dt, int peer, cudaStream_t st);
void p2p_recv(void* c, void* buf, i64 n, DT dt, int peer, cudaStream_t st);

std::vector<PipeStep> pipe_program(const StagePlan& plan, int micro, int tp, int rank) {
    const int S = (int)plan.stages.size();
    if (tp < 1 || micro < 1 || rank < 0 || rank >= S * tp) throw Error("pipe_program: bad rank / tp / micro");
    const int s = rank / tp, r = rank % tp;
    const Stage& st = plan.stages[(size_t)s];
    Topo topo(plan);
    // remote inputs sorted by (producer stage, output index)
    std::vector<std::tuple<int, int, int>> rin;  // (producer stage, output index, input index)
    for (size_t i = 0; i < st.consumes.size(); ++i) {
        const auto& pr = topo.in_prod[(size_t)s][i];
        if (pr.first >= 0 && pr.first != s) rin.push_back({pr.first, pr.second, (int)i});
    }
    std::sort(rin.begin(), rin.end());
    std::vector<PipeStep> prog;
    auto remote_consumers = [&](int o) {  // consumer stages in ascending order
        std::vector<int> t;
        for (auto& [cs, ci] : topo.cons[{s, o}])
            if (cs != s) t.push_back(cs);
        std::sort(t.begin(), t.end());
        return t;
    };
    for (int m = 0; m < micro; ++m) {
        for (auto& [ps, po, i] : rin) prog.push_back({PipeStep::FwdRecv, m, i, ps * tp + r, st.consumes[(size_t)i]});
        prog.push_back({PipeStep::FwdRun, m, -1, -1, ""});
        for (int o = 0; o < (int)st.produces.size(); ++o)
            for (int t : remote_consumers(o)) prog.push_back({PipeStep::FwdSend, m, o, t * tp + r, st.produces[(size_t)o]});
    }
    for (int m = micro - 1; m >= 0; --m) {
        for (int o = 0; o < (int)st.produces.size(); ++o)
            for (int t : remote_consumers(o)) prog.push_back({PipeStep::BwdRecv, m, o, t * tp + r, st.produces[(size_t)o]});
        prog.push_back({PipeStep::BwdRun, m, -1, -1, ""});
        for (auto& [ps, po, i] : rin) prog.push_back({PipeStep::BwdSend, m, i, ps * tp + r, st.consumes[(size_t)i]});
    }
    return prog;
}

struct PipelineExecutor::Impl {
    int M = 1, tp = 1;
    // distributed placement (one process per stage x tp rank)
    bool dist = false;
    int lstage = -1;
    void* pcomm = nullptr;
    std::vector<PipeStep> prog;
    std::map<int, void*> rtmp;  // produced value -> fp32 receive buffer of a consumer's input gradient
    std::map<int, void*> stmp;  // local input index -> fp32 send buffer of its gradient
    std::vector<StageRt> stages;
    std::vector<Value> values;  // model inputs first, then produced values
    std::vector<int> model_out_val;
    std::vector<std::vector<void*>> in_host_dev;  // [m][model input]: uploaded f64 slices (value buffers)
    bool ran_forward = false;
    int dev0 = 0;
    // the whole step (every micro-batch's forward and backward over all stage streams)
    // captured once into a CUDA graph when every local stage shares one device
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;

    ~Impl() {
        if (gexec) cudaGraphExecDestroy(gexec);
        if (graph) cudaGraphDestroy(graph);
        for (auto& [k, p] : rtmp) cudaFree(p);
        for (auto& [k, p] : stmp) cudaFree(p);
        if (pcomm) p2p_comm_destroy(pcomm);
        for (auto& v : values) {
            for (void* p : v.buf) cudaFree(p);
            for (void* p : v.gbuf) cudaFree(p);
            if (v.ginit) cudaEventDestroy(v.ginit);
        }
        for (auto& s : stages) {
            for (void* p : s.tmp_in) cudaFree(p);
            for (void* p : s.tmp_grad) cudaFree(p);
            for (auto e : s.ev_fwd) cudaEventDestroy(e);
            for (auto e : s.ev_bwd) cudaEventDestroy(e);
            for (auto& g : s.gin)
                for (void* p : g) cudaFree(p);
        }
    }

    // copy `bytes` from src (on sdev) to dst (on ddev), enqueued on `st` (a stream of ddev or sdev)
    static void move(void* dst, int ddev, const void* src, int sdev, size_t bytes, cudaStream_t st) {
        if (ddev == sdev) PCK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
        else PCK(cudaMemcpyPeerAsync(dst, ddev, src, sdev, bytes, st));
    }

    void set_inputs(StageRt& s, int m) {
        for (size_t i = 0; i < s.in_val.size(); ++i) {
            Value& v = values[(size_t)s.in_val[i]];
            const void* src = v.buf[(size_t)m];
            if (v.dev != s.dev) {
                move(s.tmp_in[i], s.dev, src, v.dev, bytes_of(v.dt, v.numel), s.st);
                src = s.tmp_in[i];
            }
            s.ex->set_input_from_device((int)i, src, v.dt);
        }
    }

    void wait_inputs(StageRt& s, int m) {
        for (int vi : s.in_val) {
            const Value& v = values[(size_t)vi];
            if (v.producer >= 0) PCK(cudaStreamWaitEvent(s.st, stages[(size_t)v.producer].ev_fwd[(size_t)m], 0));
        }
    }

    void stash_outputs(StageRt& s, int m) {
        for (size_t o = 0; o < s.out_val.size(); ++o) {
            Value& v = values[(size_t)s.out_val[o]];
            DeviceTensor t = s.ex->output_device((int)o);
            PCK(cudaMemcpyAsync(v.buf[(size_t)m], t.ptr, bytes_of(t.dt, t.numel), cudaMemcpyDeviceToDevice, s.st));
        }
    }

    // the backward of micro-batch m of stage s, its output gradients seeded from gbuf
    void stage_backward(StageRt& s, int m) {
        set_inputs(s, m);
        s.ex->run_forward();  // re-materialisation (GPipe): activations of micro-batch m
        for (size_t o = 0; o < s.out_val.size(); ++o)
            s.ex->set_output_grad_seed((int)o, values[(size_t)s.out_val[o]].gbuf[(size_t)m], sbk::F32);
        s.ex->run_backward();
    }

    void init_seeds(Value& v, cudaStream_t st) {
        for (int m = 0; m < M; ++m) {
            if (v.model_out >= 0) sbk::fill(v.gbuf[(size_t)m], sbk::F32, v.numel, 1.f, st);
            else PCK(cudaMemsetAsync(v.gbuf[(size_t)m], 0, bytes_of(sbk::F32, v.numel), st));
        }
    }

    // distributed placement: this rank's stage follows its transfer program
    void run_program(bool fwd) {
        StageRt& s = stages[(size_t)lstage];
        PCK(cudaSetDevice(s.dev));
        if (!fwd) {
            for (int vo : s.out_val) init_seeds(values[(size_t)vo], s.st);
            s.ex->zero_param_grads();
        }
        const i64 one = 1;
        for (const PipeStep& p : prog) {
            const bool f = p.kind <= PipeStep::FwdSend;
            if (f != fwd) continue;
            switch (p.kind) {
                case PipeStep::FwdRecv: {
                    Value& v = values[(size_t)s.in_val[(size_t)p.idx]];
                    p2p_recv(pcomm, v.buf[(size_t)p.m], v.numel, v.dt, p.peer, s.st);
                    break;
                }
                case PipeStep::FwdRun:
                    set_inputs(s, p.m);
                    s.ex->run_forward();
                    stash_outputs(s, p.m);
                    break;
                case PipeStep::FwdSend: {
                    Value& v = values[(size_t)s.out_val[(size_t)p.idx]];
                    p2p_send(pcomm, v.buf[(size_t)p.m], v.numel, v.dt, p.peer, s.st);
                    break;
                }
                case PipeStep::BwdRecv: {
                    const int vi = s.out_val[(size_t)p.idx];
                    Value& v = values[(size_t)vi];
                    p2p_recv(pcomm, rtmp.at(vi), v.numel, sbk::F32, p.peer, s.st);
                    sbk::strided_copy(rtmp.at(vi), sbk::F32, &one, v.gbuf[(size_t)p.m], sbk::F32, &one, &v.numel, 1, true,
                                      s.st);
                    break;
                }
                case PipeStep::BwdRun: {
                    stage_backward(s, p.m);
                    for (size_t i = 0; i < s.in_val.size(); ++i) {  // model inputs: keep their gradients
                        const Value& v = values[(size_t)s.in_val[i]];
                        if (v.producer >= 0) continue;
                        DeviceTensor g = s.ex->input_grad_device((int)i);
                        sbk::strided_copy(g.ptr, g.dt, &one, s.gin[(size_t)p.m][i], sbk::F32, &one, &g.numel, 1, false, s.st);
                    }
                    break;
                }
                case PipeStep::BwdSend: {
                    DeviceTensor g = s.ex->input_grad_device(p.idx);
                    void* t = stmp.at(p.idx);
                    sbk::strided_copy(g.ptr, g.dt, &one, t, sbk::F32, &one, &g.numel, 1, false, s.st);
                    p2p_send(pcomm, t, g.numel, sbk::F32, p.peer, s.st);
                    break;
                }
            }
        }
        if (fwd) ran_forward = true;
    }

    void forward_all() {
        if (dist) return run_program(true);
        for (int m = 0; m < M; ++m) {
            for (size_t si = 0; si < stages.size(); ++si) {
                StageRt& s = stages[si];
                PCK(cudaSetDevice(s.dev));
                wait_inputs(s, m);
                set_inputs(s, m);
                s.ex->run_forward();
                for (size_t o = 0; o < s.out_val.size(); ++o) {
                    Value& v = values[(size_t)s.out_val[o]];
                    DeviceTensor t = s.ex->output_device((int)o);
                    PCK(cudaMemcpyAsync(v.buf[(size_t)m], t.ptr, bytes_of(t.dt, t.numel), cudaMemcpyDeviceToDevice, s.st));
                }
                PCK(cudaEventRecord(s.ev_fwd[(size_t)m], s.st));
            }
        }
        ran_forward = true;
    }

    void backward_all() {
        if (!ran_forward) throw Error("pipeline backward requires a completed forward run");
        if (dist) return run_program(false);
        // gradient seeds of every produced value: ones for model outputs (loss = sum of
        // the outputs), zero otherwise; consumers add their input gradients on top
        for (auto& v : values) {
            if (v.producer < 0) continue;
            StageRt& p = stages[(size_t)v.producer];
            PCK(cudaSetDevice(p.dev));
            for (int m = 0; m < M; ++m) {
                if (v.model_out >= 0) sbk::fill(v.gbuf[(size_t)m], sbk::F32, v.numel, 1.f, p.st);
                else PCK(cudaMemsetAsync(v.gbuf[(size_t)m], 0, bytes_of(sbk::F32, v.numel), p.st));
            }
            PCK(cudaEventRecord(v.ginit, p.st));
        }
        for (auto& s : stages) {
            PCK(cudaSetDevice(s.dev));
            s.ex->zero_param_grads();
        }
        for (int m = M - 1; m >= 0; --m) {
            for (int si = (int)stages.size() - 1; si >= 0; --si) {
                StageRt& s = stages[(size_t)si];
                PCK(cudaSetDevice(s.dev));
                // the gradients of this stage's outputs are complete once every consumer's
                // backward of this micro-batch has added its input gradient
                for (int vo : s.out_val) {
                    PCK(cudaStreamWaitEvent(s.st, values[(size_t)vo].ginit, 0));
                    for (auto& [t, ti] : values[(size_t)vo].consumers)
                        PCK(cudaStreamWaitEvent(s.st, stages[(size_t)t].ev_bwd[(size_t)m], 0));
                }
                wait_inputs(s, m);
                set_inputs(s, m);
                s.ex->run_forward();  // re-materialisation (GPipe): activations of micro-batch m
                for (size_t o = 0; o < s.out_val.size(); ++o)
                    s.ex->set_output_grad_seed((int)o, values[(size_t)s.out_val[o]].gbuf[(size_t)m], sbk::F32);
                s.ex->run_backward();
                for (size_t i = 0; i < s.in_val.size(); ++i) {
                    Value& v = values[(size_t)s.in_val[i]];
                    DeviceTensor g = s.ex->input_grad_device((int)i);
                    const i64 n = g.numel, one = 1;
                    if (v.producer < 0) {  // a model input: keep its gradient for the caller
                        sbk::strided_copy(g.ptr, g.dt, &one, s.gin[(size_t)m][i], sbk::F32, &one, &n, 1, false, s.st);
                        continue;
                    }
                    PCK(cudaStreamWaitEvent(s.st, v.ginit, 0));
                    const void* src = g.ptr;
                    DT sdt = g.dt;
                    if (v.dev != s.dev) {
                        move(s.tmp_grad[i], v.dev, g.ptr, s.dev, bytes_of(g.dt, n), s.st);
                        src = s.tmp_grad[i];
                        PCK(cudaSetDevice(v.dev));  // the add runs on the producer's device
                    }
                    sbk::strided_copy(src, sdt, &one, v.gbuf[(size_t)m], sbk::F32, &one, &n, 1, true, s.st);
                    PCK(cudaSetDevice(s.dev));
                }
                PCK(cudaEventRecord(s.ev_bwd[(size_t)m], s.st));
            }
        }
    }

    void sync_all() {
        for (auto& s : stages) {
            if (!s.ex) continue;
            PCK(cudaSetDevice(s.dev));
            PCK(cudaStreamSynchronize(s.st));
        }
    }
};

PipelineExecutor::PipelineExecutor(const StagePlan& plan, int micro, bool train, u64 seed, DT compute,
                                   std::vector<int> devices, bool fused, int tp, const PipeDist* dist)
    : impl_(std::make_unique<Impl>()) {
    auto& I = *impl_;
    if (micro < 1) throw Error("micro_batches must be >= 1");
    if (tp < 1) throw Error("pipeline: tp must be >= 1");
    I.tp = tp;
    if (plan.stages.empty()) throw Error("pipeline: empty stage plan");
    int trank = 0;
    if (dist && dist->rank >= 0) {
        I.dist = true;
        if (dist->world != (int)plan.stages.size() * tp)
            throw Error("pipeline: the distributed world must be stages x tp processes");
        I.lstage = dist->rank / tp;
        trank = dist->rank % tp;
        devices.clear();
    }
    auto local = [&](size_t si) { return !I.dist || (int)si == I.lstage; };
    if (devices.empty()) {
        int d = 0;
        PCK(cudaGetDevice(&d));
        devices.assign(plan.stages.size(), d);
    }
    if (devices.size() != plan.stages.size()) throw Error("pipeline: one device per stage");
    I.M = micro;
    I.dev0 = devices[0];
    std::map<std::string, int> by_name;
    for (size_t k = 0; k < plan.model_inputs.size(); ++k) {
        Value v;
        v.name = plan.model_inputs[k];
        v.out_idx = (int)k;
        by_name[v.name] = (int)I.values.size();
        I.values.push_back(v);
    }
    for (size_t si = 0; si < plan.stages.size(); ++si) {
        const Stage& st = plan.stages[si];
        StageRt s;
        s.dev = devices[si];
        PCK(cudaSetDevice(s.dev));
        if (local(si)) {
            CommConfig cc;
            if (I.dist && tp > 1) {  // the stage's tensor parallelism over its own NCCL communicator
                cc.nccl = true;
                cc.rank = trank;
                cc.unique_id = dist->tp_uid;
            }
            s.ex = std::make_unique<Executor>(micro_module(st.module, micro), train, seed, tp, compute, cc, fused);
            s.ex->set_accumulate_param_grads(true);
            s.st = (cudaStream_t)s.ex->stream();
        }
        for (size_t i = 0; i < st.consumes.size(); ++i) {
            auto it = by_name.find(st.consumes[i]);
            if (it == by_name.end()) throw Error("pipeline stage consumes unknown value '" + st.consumes[i] + "'");
            s.in_val.push_back(it->second);
            I.values[(size_t)it->second].consumers.push_back({(int)si, (int)i});
        }
        for (size_t o = 0; o < st.produces.size(); ++o) {
            Value v;
            v.name = st.produces[o];
            v.producer = (int)si;
            v.out_idx = (int)o;
            v.dev = s.dev;
            v.dt = compute;  // (a remote stage's output: an activation in the compute dtype)
            if (s.ex) {
                DeviceTensor t = s.ex->output_device((int)o);
                v.dt = t.dt;
                v.numel = t.numel;
                v.shape = t.shape;
            }
            by_name[v.name] = (int)I.values.size();
            I.values.push_back(v);
            s.out_val.push_back(by_name[st.produces[o]]);
        }
        I.stages.push_back(std::move(s));
    }
    for (size_t k = 0; k < plan.model_outputs.size(); ++k) {
        auto it = by_name.find(plan.model_outputs[k]);
        if (it == by_name.end() || I.values[(size_t)it->second].producer < 0)
            throw Error("pipeline missing model output '" + plan.model_outputs[k] + "'");
        I.values[(size_t)it->second].model_out = (int)k;
        I.model_out_val.push_back(it->second);
    }
    // model inputs live (f64, per micro-batch) on their first consumer's device
    for (auto& v : I.values) {
        if (v.producer >= 0) continue;
        if (v.consumers.empty()) throw Error("pipeline: model input '" + v.name + "' is consumed by no stage");
        StageRt& c = I.stages[(size_t)v.consumers[0].first];
        v.dev = c.dev;
        v.dt = sbk::F64;
    }
    for (size_t si = 0; si < I.stages.size(); ++si) {
        StageRt& s = I.stages[si];
        if (!local(si)) continue;
        PCK(cudaSetDevice(s.dev));
        const Module mm = micro_module(plan.stages[si].module, micro);
        size_t i = 0;
        for (int id : mm.forward->inputs) {  // declared input shapes (one per consumed value, in order)
            Value& v = I.values[(size_t)s.in_val[i++]];
            if (v.numel) continue;
            const auto& at = mm.forward->at(id).attrs;
            auto it = at.find("shape");
            if (it == at.end()) throw Error("pipeline: stage input without a declared shape");
            v.shape = std::get<std::vector<i64>>(it->second);
            v.numel = 1;
            for (i64 d : v.shape) v.numel *= d;
        }
    }
    auto touched = [&](const Value& v) {  // produced or consumed by a stage of this process
        if (v.producer >= 0 && local((size_t)v.producer)) return true;
        for (auto& [cs, ci] : v.consumers)
            if (local((size_t)cs)) return true;
        return false;
    };
    for (auto& v : I.values) {
        if (!touched(v)) continue;
        for (int m = 0; m < micro; ++m) v.buf.push_back(dev_alloc(v.dev, bytes_of(v.dt, v.numel)));
        if (v.producer >= 0 && local((size_t)v.producer)) {
            for (int m = 0; m < micro; ++m) v.gbuf.push_back(dev_alloc(v.dev, bytes_of(sbk::F32, v.numel)));
            PCK(cudaSetDevice(v.dev));
            PCK(cudaEventCreateWithFlags(&v.ginit, cudaEventDisableTiming));
        }
    }
    for (auto& s : I.stages) {
        if (!s.ex) continue;
        PCK(cudaSetDevice(s.dev));
        s.ev_fwd.resize((size_t)micro);
        s.ev_bwd.resize((size_t)micro);
        for (int m = 0; m < micro; ++m) {
            PCK(cudaEventCreateWithFlags(&s.ev_fwd[(size_t)m], cudaEventDisableTiming));
            PCK(cudaEventCreateWithFlags(&s.ev_bwd[(size_t)m], cudaEventDisableTiming));
        }
        s.gin.assign((size_t)micro, std::vector<void*>(s.in_val.size(), nullptr));
        for (size_t i = 0; i < s.in_val.size(); ++i) {
            Value& v = I.values[(size_t)s.in_val[i]];
            s.tmp_in.push_back(v.dev != s.dev ? dev_alloc(s.dev, bytes_of(v.dt, v.numel)) : nullptr);
            s.tmp_grad.push_back(v.dev != s.dev && v.producer >= 0 ? dev_alloc(v.dev, bytes_of(sbk::F32, v.numel)) : nullptr);
            if (v.producer < 0)
                for (int m = 0; m < micro; ++m) s.gin[(size_t)m][i] = dev_alloc(s.dev, bytes_of(sbk::F32, v.numel));
        }
    }
    if (I.dist) {
        StageRt& s = I.stages[(size_t)I.lstage];
        for (int vo : s.out_val) {  // receive buffers for the consumers' input gradients
            bool remote = false;
            for (auto& [cs, ci] : I.values[(size_t)vo].consumers) remote |= cs != I.lstage;
            if (remote) I.rtmp[vo] = dev_alloc(s.dev, bytes_of(sbk::F32, I.values[(size_t)vo].numel));
        }
        for (size_t i = 0; i < s.in_val.size(); ++i) {
            const Value& v = I.values[(size_t)s.in_val[i]];
            if (v.producer >= 0 && v.producer != I.lstage) I.stmp[(int)i] = dev_alloc(s.dev, bytes_of(sbk::F32, v.numel));
        }
        I.prog = pipe_program(plan, micro, tp, dist->rank);
        PCK(cudaSetDevice(s.dev));
        I.pcomm = p2p_comm_create(dist->world, dist->rank, dist->pp_uid);
    }
}

PipelineExecutor::~PipelineExecutor() = default;
int PipelineExecutor::num_stages() const { return (int)impl_->stages.size(); }
int PipelineExecutor::micro_batches() const { return impl_->M; }

std::vector<HostTensor> PipelineExecutor::forward(const std::vector<HostTensor>& inputs) {
    auto& I = *impl_;
    std::vector<const double*> p;
    for (auto& v : I.values) {
        if (v.producer >= 0) continue;
        if (v.out_idx < (int)inputs.size() && (i64)inputs[(size_t)v.out_idx].data.size() != v.numel * I.M)
            throw Error("pipeline input '" + v.name + "': expected " + std::to_string(v.numel * I.M) + " elements");
    }
    for (auto& x : inputs) p.push_back(x.data.data());
    return forward_raw(p.data(), (int)p.size());
}

std::vector<HostTensor> PipelineExecutor::forward_raw(const double* const* inputs, int n) {
    auto& I = *impl_;
    int nin = 0;
    for (auto& v : I.values) nin += v.producer < 0;
    if (n != nin) throw Error("pipeline expects " + std::to_string(nin) + " inputs");
    for (auto& v : I.values) {
        if (v.producer >= 0 || v.buf.empty()) continue;  // (distributed: inputs of other ranks' stages)
        const double* x = inputs[v.out_idx];
        PCK(cudaSetDevice(v.dev));
        for (int m = 0; m < I.M; ++m)  // micro-batch m = rows [m*B/M, (m+1)*B/M) of dim 0: a contiguous slice
            PCK(cudaMemcpy(v.buf[(size_t)m], x + (size_t)m * (size_t)v.numel, bytes_of(sbk::F64, v.numel),
                           cudaMemcpyHostToDevice));
    }
    I.forward_all();
    I.sync_all();
    std::vector<HostTensor> outs;
    for (int vi : I.model_out_val) {
        const Value& v = I.values[(size_t)vi];
        if (v.buf.empty() || (I.dist && v.producer != I.lstage)) {  // produced by another rank's stage
            outs.push_back(HostTensor(TensorSpec{{0}, Dtype::F64}));
            continue;
        }
        TensorSpec sp;
        sp.shape = v.shape;
        sp.shape[0] *= I.M;
        HostTensor t(sp);
        PCK(cudaSetDevice(v.dev));
        double* d = (double*)dev_alloc(v.dev, bytes_of(sbk::F64, v.numel));
        for (int m = 0; m < I.M; ++m) {
            sbk::cast(v.buf[(size_t)m], v.dt, d, sbk::F64, v.numel, nullptr);
            PCK(cudaMemcpy(t.data.data() + (size_t)m * (size_t)v.numel, d, bytes_of(sbk::F64, v.numel),
                           cudaMemcpyDeviceToHost));
        }
        cudaFree(d);
        outs.push_back(std::move(t));
    }
    return outs;
}

std::vector<GradMap> PipelineExecutor::backward() {
    auto& I = *impl_;
    I.backward_all();
    I.sync_all();
    std::vector<GradMap> res;
    for (auto& s : I.stages) {
        if (!s.ex) continue;  // (distributed: only this rank's stage)
        PCK(cudaSetDevice(s.dev));
        std::vector<GradMap> per_rank = s.ex->grads_all_ranks();
        // model-input gradients concatenated over micro-batches; produced-value inputs: none
        std::vector<HostTensor> ins;
        for (size_t i = 0; i < s.in_val.size(); ++i) {
            const Value& v = I.values[(size_t)s.in_val[i]];
            if (v.producer >= 0) continue;
            TensorSpec sp;
            sp.shape = v.shape;
            sp.shape[0] *= I.M;
            HostTensor t(sp);
            std::vector<float> f((size_t)v.numel);
            for (int m = 0; m < I.M; ++m) {
                PCK(cudaMemcpy(f.data(), s.gin[(size_t)m][i], bytes_of(sbk::F32, v.numel), cudaMemcpyDeviceToHost));
                for (i64 e = 0; e < v.numel; ++e) t.data[(size_t)(m * v.numel + e)] = f[(size_t)e];
            }
            ins.push_back(std::move(t));
        }
        for (auto& g : per_rank) {
            g.inputs = ins;  // (replicated across the stage's ranks)
            res.push_back(std::move(g));
        }
    }
    return res;
}
int PipelineExecutor::tp() const { return impl_->tp; }

float PipelineExecutor::time_steps(int steps, bool use_graph) {
    auto& I = *impl_;
    if (!I.ran_forward) throw Error("time_steps: run forward() once first (uploads the inputs)");
    PCK(cudaSetDevice(I.dev0));
    cudaEvent_t a, b;
    PCK(cudaEventCreate(&a));
    PCK(cudaEventCreate(&b));
    I.sync_all();
    PCK(cudaSetDevice(I.dev0));
    cudaStream_t s0 = I.stages[I.dist ? (size_t)I.lstage : 0].st;
    bool one_dev = true;
    for (auto& s : I.stages)
        if (s.ex) one_dev &= s.dev == I.dev0;
    // one step on the stage streams, forked from and joined into s0
    cudaEvent_t fork;
    PCK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    auto enqueue_step = [&]() {
        PCK(cudaEventRecord(fork, s0));
        for (auto& s : I.stages)
            if (s.ex && s.st != s0) PCK(cudaStreamWaitEvent(s.st, fork, 0));
        I.forward_all();
        I.backward_all();
        PCK(cudaSetDevice(I.dev0));
        for (auto& s : I.stages)
            if (s.ex && s.st != s0) PCK(cudaStreamWaitEvent(s0, s.ev_bwd[0], 0));
    };
    if (use_graph && one_dev && !I.gexec) {
        PCK(cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal));
        enqueue_step();
        PCK(cudaStreamEndCapture(s0, &I.graph));
        PCK(cudaGraphInstantiate(&I.gexec, I.graph, 0));
    }
    const bool graph = use_graph && I.gexec;
    PCK(cudaEventRecord(a, s0));
    for (int k = 0; k < steps; ++k) {
        if (graph) PCK(cudaGraphLaunch(I.gexec, s0));
        else enqueue_step();
    }
    PCK(cudaEventRecord(b, s0));
    PCK(cudaEventSynchronize(b));
    float ms = 0;
    PCK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaEventDestroy(fork);
    I.sync_all();
    return ms;
}

}  // namespace sb
