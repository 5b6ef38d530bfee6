// B200 executor runtime: arena allocation, forward/backward launch lists,
// checkpoint recompute, collectives (device-local lockstep or NCCL), CUDA
// graph capture. Semantics per op mirror proj/src/executor.cpp (cited inline).
#include "executor.hpp"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <set>
#include <sstream>

#include "rng.hpp"
#include <nvtx3/nvToolsExt.h>

namespace sb {

#define CK(x)                                                                                       \
    do {                                                                                            \
        cudaError_t e_ = (x);                                                                       \
        if (e_ != cudaSuccess) throw Error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #x); \
    } while (0)

// ------------------------------------------------------------------ NCCL (dlopen)
// One NCCL per process: $SB_NCCL_LIB when set (the Python layer points it at the
// NCCL torch.distributed already loaded), else whatever libnccl.so.2 is already
// mapped (RTLD_NOLOAD), else the loader's libnccl.so.2.
void* nccl_handle() {
    static void* h = [] {
        void* p = nullptr;
        if (const char* e = getenv("SB_NCCL_LIB"); e && *e) p = dlopen(e, RTLD_NOW | RTLD_GLOBAL);
        if (!p) p = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!p) p = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!p) p = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        return p;
    }();
    return h;
}
namespace {
struct Nccl {
    void* h = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    void load() {
        if (h) return;
        h = nccl_handle();
        if (!h) throw Error("NCCL not available: dlopen(libnccl.so.2) failed");
        CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
        AllReduce = (decltype(AllReduce))dlsym(h, "ncclAllReduce");
        AllGather = (decltype(AllGather))dlsym(h, "ncclAllGather");
        CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
        Send = (decltype(Send))dlsym(h, "ncclSend");
        Recv = (decltype(Recv))dlsym(h, "ncclRecv");
        GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
        if (!CommInitRank || !AllReduce || !AllGather) throw Error("NCCL symbols missing");
    }
    void check(ncclResult_t r, const char* what) {
        if (r != ncclSuccess) throw Error(std::string("NCCL error in ") + what + ": " + GetErrorString(r));
    }
};
Nccl& nccl() {
    static Nccl n;
    return n;
}
ncclDataType_t nccl_dt(DT t) { return t == sbk::F32 ? ncclFloat32 : t == sbk::BF16 ? ncclBfloat16 : ncclFloat64; }

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// NVTX ranges per plan op (SB_NVTX=1; header-only NVTX v3, no-ops without a tool attached):
// "<op kind>[ (bwd)| (re)] <module path>" around each op's launches — eager steps only (a
// captured CUDA graph replays kernels, not host ranges)
struct NvtxRange {
    bool on;
    NvtxRange(const char* kind, const char* tag, const std::string& path) : on(enabled()) {
        if (!on) return;
        std::string n = std::string(kind) + tag + " " + path;
        nvtxRangePushA(n.c_str());
    }
    ~NvtxRange() {
        if (on) nvtxRangePop();
    }
    static bool enabled() {
        static const bool e = getenv("SB_NVTX") && atoi(getenv("SB_NVTX"));
        return e;
    }
};
}  // namespace

// ---- point-to-point transport of the pipeline executor (pipeline_exec.cpp) ----
void* p2p_comm_create(int world, int rank, const std::vector<char>& uid) {
    nccl().load();
    if (!nccl().Send || !nccl().Recv) throw Error("NCCL without ncclSend/ncclRecv");
    ncclUniqueId id;
    if (uid.size() != sizeof(id)) throw Error("nccl unique id must be 128 bytes");
    std::memcpy(&id, uid.data(), sizeof(id));
    ncclComm_t c = nullptr;
    nccl().check(nccl().CommInitRank(&c, world, id, rank), "ncclCommInitRank (pipeline)");
    return c;
}
void p2p_comm_destroy(void* c) {
    if (c && nccl().CommDestroy) nccl().CommDestroy((ncclComm_t)c);
}
void p2p_send(void* c, const void* buf, i64 n, DT dt, int peer, cudaStream_t st) {
    nccl().check(nccl().Send(buf, (size_t)n, nccl_dt(dt), peer, (ncclComm_t)c, st), "ncclSend");
}
void p2p_recv(void* c, void* buf, i64 n, DT dt, int peer, cudaStream_t st) {
    nccl().check(nccl().Recv(buf, (size_t)n, nccl_dt(dt), peer, (ncclComm_t)c, st), "ncclRecv");
}

// ------------------------------------------------------------------ per rank
struct RankCtx {
    Plan P;
    char* base = nullptr;
    size_t total = 0;
    std::vector<char*> fptr, gptr;  // per storage
    char* ws = nullptr;             // workspace
    size_t ws_bytes = 0;
    char* ws2 = nullptr;            // workspace of the side-stream weight gradients (ws_bytes)
    char* tmp = nullptr;            // grad-conversion temp
    size_t tmp_bytes = 0;
    size_t scratch_grad_bytes = 0;
    char* scratch_grad = nullptr;
    std::vector<std::pair<size_t, size_t>> region_grad_span;  // per region: offset,bytes in grad scratch
    // FusedLinearGelu op -> its bias gradient's column partials ([rows/32][out] fp32), written
    // by the consuming Linear's dGeLU dgrad epilogue (2-SM GEMM) instead of re-reading the
    // pre-activation gradient; colsum_ready: written during this backward
    std::map<int, float*> colsum;
    std::set<int> colsum_ready;
};

struct Step {
    int kind;  // 0 backward of op, 1 recompute forward op, 2 zero grad scratch of region
    int idx;
};

class ExecutorImpl {
public:
    bool train;
    u64 seed;
    int world;
    DT cdt;
    CommConfig comm;
    bool nan_guard = false;
    std::vector<RankCtx> ranks;  // Local: world contexts; Nccl: 1
    std::vector<Step> bsteps;
    cudaStream_t stream = nullptr;
    ncclComm_t ncomm = nullptr;
    i64 collectives = 0;
    bool ran_forward = false;
    // pipeline stages (f1): parameter gradients accumulate across backward calls
    // (micro-batches) instead of being overwritten, and output gradients can be
    // seeded from device buffers (the next stage's input gradients) instead of ones
    bool accum_params = false;
    std::vector<std::pair<const void*, DT>> out_seed;
    cudaGraphExec_t gexec = nullptr;
    cudaGraph_t graph = nullptr;
    int launches = 0;
    int* nan_flag = nullptr;
    // profiling
    bool profiling = false;
    std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> prof;

    int my_rank(int idx) const { return comm.nccl ? comm.rank : idx; }

    // ------------------------------------------ weight gradients on a side stream
    // The weight / bias gradients of a Linear (dW = g^T x, db = colsum g) feed nothing
    // else in the backward, so they are enqueued on a low-priority stream that forks
    // right before the layer's dgrad: the dgrad (critical path) keeps its SMs and the
    // weight-gradient CTAs fill the SMs its last wave, the attention backward's last
    // wave and the small reduction kernels leave idle. Joined before any checkpoint
    // region is recomputed (its scratch is reused) and at the end of the backward.
    // Only parameters whose gradient storage has a single backward writer move, so the
    // first-writer overwrite/accumulate order is unchanged.
    cudaStream_t wstream = nullptr;
    bool wside = false, wside_pending = false;
    std::set<int> wside_ok;  // gradient storages (weights / biases) with one backward writer
    std::vector<cudaEvent_t> wfork;
    size_t wfork_next = 0;
    cudaEvent_t wjoin_ev = nullptr;
    void init_wside() {
        // opt-in (SB_WGRAD_SIDE=1): measured neutral at C3 on one power-capped B200
        // (648.6-653.2 vs 648.6-650.7 samples/s, profiles/r2/summary.md §3)
        const char* e = getenv("SB_WGRAD_SIDE");
        wside = e && atoi(e) != 0 && !comm.nccl && world == 1;
        if (!wside) return;
        const Plan& P = ranks[0].P;
        std::map<int, int> writers;
        for (auto& st : bsteps)
            if (st.kind == 0)
                for (int g : grad_writes(P, P.fwd[(size_t)st.idx])) ++writers[g];
        for (auto& pv : P.params) {
            const int g = P.views[(size_t)pv.second].gst;
            if (writers[g] == 1 && P.st[(size_t)g].region < 0) wside_ok.insert(g);
        }
        int lo, hi;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&wstream, cudaStreamNonBlocking, lo));
        CK(cudaEventCreateWithFlags(&wjoin_ev, cudaEventDisableTiming));
    }
    bool wside_eligible(RankCtx& r, const Op& op) const {
        if (!wside) return false;
        if (!wside_ok.count(r.P.views[(size_t)op.in[1]].gst)) return false;
        if (op.has_bias && op.bias_grad && !wside_ok.count(r.P.views[(size_t)op.in[2]].gst)) return false;
        return true;
    }
    cudaEvent_t next_fork() {
        if (wfork_next == wfork.size()) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            wfork.push_back(e);
        }
        return wfork[wfork_next++];
    }
    void wside_join() {
        if (!wside_pending) return;
        CK(cudaEventRecord(wjoin_ev, wstream));
        CK(cudaStreamWaitEvent(stream, wjoin_ev, 0));
        wside_pending = false;
    }

    ExecutorImpl(const Module& root, bool tr, u64 sd, int w, DT c, const CommConfig& cc, bool fused)
        : train(tr), seed(sd), world(w), cdt(c), comm(cc) {
        if (world < 1) throw Error("world_size must be >= 1");
        {
            // SB_MAIN_PRIO=1: the executor stream above the side streams (keep bits, weight
            // gradients), below the communication stream (measured neutral, default off)
            int lo, hi;
            CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            static const int raise = getenv("SB_MAIN_PRIO") ? atoi(getenv("SB_MAIN_PRIO")) : 0;
            CK(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, raise && hi < lo ? std::min(lo, hi + 1) : lo));
        }
        int nr = comm.nccl ? 1 : world;
        ranks.resize((size_t)nr);
        for (int i = 0; i < nr; ++i) {
            LowerOptions lo;
            lo.rank = my_rank(i);
            lo.world = world;
            lo.train = train;
            lo.seed = seed;
            lo.cdt = cdt;
            lo.fused_kernels = fused;
            lo.keep_collectives = comm.nccl;
            ranks[(size_t)i].P = lower(root, lo);
            if (i > 0 && ranks[(size_t)i].P.structure() != ranks[0].P.structure())
                throw Error("per-rank plans differ structurally; lockstep execution impossible");
        }
        build_backward_steps();
        analyze_writes();
        for (auto& r : ranks) allocate(r);
        init_mask_stream();
        init_early_allreduce();
        init_wside();
        if (wside)
            for (auto& r : ranks) {
                CK(cudaMalloc(&r.ws2, r.ws_bytes));
            }
        if (comm.nccl) {
            nccl().load();
            ncclUniqueId id;
            if (comm.unique_id.size() != sizeof(id)) throw Error("nccl unique id must be 128 bytes");
            std::memcpy(&id, comm.unique_id.data(), sizeof(id));
            nccl().check(nccl().CommInitRank(&ncomm, world, id, comm.rank), "ncclCommInitRank");
        }
        CK(cudaMalloc(&nan_flag, sizeof(int)));
        sbk::init_workspace();
    }

    ~ExecutorImpl() {
        if (gexec) cudaGraphExecDestroy(gexec);
        if (graph) cudaGraphDestroy(graph);
        for (auto& r : ranks) {
            if (r.base) cudaFree(r.base);
            if (r.ws2) cudaFree(r.ws2);
        }
        for (auto e : wfork) cudaEventDestroy(e);
        if (wjoin_ev) cudaEventDestroy(wjoin_ev);
        if (wstream) cudaStreamDestroy(wstream);
        if (nan_flag) cudaFree(nan_flag);
        if (nan_counts) cudaFree(nan_counts);
        if (ncomm && nccl().CommDestroy) nccl().CommDestroy(ncomm);
        for (auto e : mask_ev)
            if (e) cudaEventDestroy(e);
        for (auto e : bwd_ev)
            if (e) cudaEventDestroy(e);
        for (auto e : ar_ev)
            if (e) cudaEventDestroy(e);
        for (auto e : dgrad_ev)
            if (e) cudaEventDestroy(e);
        for (auto e : far_gemm) cudaEventDestroy(e);
        for (auto e : far_done) cudaEventDestroy(e);
        if (cstream) cudaStreamDestroy(cstream);
        if (fork_ev) cudaEventDestroy(fork_ev);
        if (mstream) cudaStreamDestroy(mstream);
        if (stream) cudaStreamDestroy(stream);
    }

    // -------------------------------------------------------------- plan
    static std::set<int> grad_writes(const Plan& P, const Op& op) {
        // storages whose gradients this op's backward writes
        std::set<int> s;
        auto add = [&](int v) { s.insert(P.views[(size_t)v].gst); };
        switch (op.k) {
            case K::Embedding:
                // the id input receives a (zero) gradient too (executor.cpp:1216-1217),
                // which is what lets a SyncGrad on it run (and count) in backward
                add(op.in[0]);
                add(op.in[1]);
                break;
            case K::AllReduce:
                if (op.allreduce) add(op.in[0]);
                break;
            case K::Cast:
                if (P.st[(size_t)P.views[(size_t)op.out[0]].st].dt != sbk::F64) add(op.in[0]);
                break;
            default:
                for (int v : op.in) add(v);
        }
        if (op.dgelu_pre >= 0) add(op.dgelu_pre);
        return s;
    }

    void build_backward_steps() {
        const Plan& P = ranks[0].P;
        std::vector<bool> has(P.st.size(), false);
        for (int v : P.outputs) has[(size_t)P.views[(size_t)v].gst] = true;
        auto any_out = [&](const Op& op) {
            for (int v : op.out)
                if (has[(size_t)P.views[(size_t)v].gst]) return true;
            return false;
        };
        auto mark = [&](const Op& op) {
            for (int s : grad_writes(P, op)) has[(size_t)s] = true;
        };
        int i = (int)P.fwd.size() - 1;
        while (i >= 0) {
            const Op& op = P.fwd[(size_t)i];
            if (op.region >= 0) {
                const Region& R = P.regions[(size_t)op.region];
                // reference: backward_checkpoint re-runs the region with a tape,
                // then reverses the sub-tape (executor.cpp:1093-1120)
                bool flows = false;
                for (int j = R.first_op; j <= R.last_op; ++j) flows |= any_out(P.fwd[(size_t)j]);
                if (flows) {
                    bsteps.push_back({2, op.region});
                    for (int j = R.first_op; j <= R.last_op; ++j) bsteps.push_back({1, j});
                    for (int j = R.last_op; j >= R.first_op; --j) {
                        if (!any_out(P.fwd[(size_t)j])) continue;
                        bsteps.push_back({0, j});
                        mark(P.fwd[(size_t)j]);
                    }
                }
                i = R.first_op - 1;
                continue;
            }
            if (any_out(op)) {
                bsteps.push_back({0, i});
                mark(op);
            }
            --i;
        }
    }

    // ------------------------------------------------ first-writer analysis
    // Instead of zeroing every gradient and accumulating, each gradient write of
    // the (static) backward order is classified: the first write to a region
    // overwrites, later ones accumulate. Only storages that are read or
    // accumulated before being fully written are zeroed, once, at backward start.
    std::vector<std::map<int, bool>> step_ow;  // per backward step: view -> overwrite
    std::map<int, bool> seed_ow;               // output-gradient seeds
    std::vector<int> zero_gst;                 // persistent grad storages to zero
    std::vector<char> region_zero;             // region scratch needs zeroing
    const std::map<int, bool>* cur_ow = nullptr;
    bool OW(int v) const {
        if (!cur_ow) return false;
        auto it = cur_ow->find(v);
        return it != cur_ow->end() && it->second;
    }

    // (view, kernel can overwrite) in the order the backward writes them
    std::vector<std::pair<int, bool>> grad_slots(const Plan& P, const Op& op) const {
        std::vector<std::pair<int, bool>> s;
        auto direct = [&](int v) { return P.st[(size_t)P.views[(size_t)v].gst].gdt == P.cdt; };
        auto linear = [&](bool bias) {
            if (op.dgelu_pre >= 0) s.push_back({op.dgelu_pre, true});
            else s.push_back({op.in[0], direct(op.in[0])});
            s.push_back({op.in[1], true});
            if (bias && op.has_bias && op.bias_grad) s.push_back({op.in[2], true});
        };
        switch (op.k) {
            case K::Linear: linear(true); break;
            case K::FusedLinearGelu:
                if (!op.dgelu_fused) s.push_back({op.out[1], false});
                linear(true);
                break;
            case K::FusedLinearResLN:
                s.push_back({op.in[2], direct(op.in[2])});
                s.push_back({op.out[1], true});
                if (op.has_bias && op.bias_grad) s.push_back({op.in[5], true});
                s.push_back({op.in[3], true});
                s.push_back({op.in[4], true});
                linear(false);
                break;
            case K::LayerNorm:
                s.push_back({op.in[0], direct(op.in[0])});
                if (op.affine) {
                    s.push_back({op.in[1], true});
                    s.push_back({op.in[2], true});
                }
                break;
            case K::FlashAttn:
                for (int k = 0; k < 3; ++k) s.push_back({op.in[(size_t)k], true});
                break;
            case K::Embedding: s.push_back({op.in[1], false}); break;  // scatter-add: partial rows
            case K::SyncGrad:
                if (!op.ids_input) s.push_back({op.in[0], true});
                break;
            case K::Cast:
                if (P.st[(size_t)P.views[(size_t)op.out[0]].st].dt != sbk::F64) s.push_back({op.in[0], true});
                break;
            case K::Dropout: s.push_back({op.in[0], direct(op.in[0])}); break;
            case K::AllReduce:
                if (op.allreduce) s.push_back({op.in[0], true});
                break;
            case K::Add:
                s.push_back({op.in[0], direct(op.in[0])});
                s.push_back({op.in[1], direct(op.in[1])});
                break;
            default:
                for (int v : op.in) s.push_back({v, false});
        }
        return s;
    }
    std::vector<int> grad_reads(const Op& op) const {
        if (op.k == K::FusedLinearGelu && op.dgelu_fused) return {op.out[1]};
        if (op.k == K::FusedLinearResLN && op.sum_ext) return {op.out[0], op.out[2]};
        if (op.k == K::SyncGrad && op.ids_input) return {};
        return {op.out[0]};
    }

    struct Span {
        i64 lo, hi, ld, c0, c1;
        bool rowwise;
        i64 n;
    };
    static Span span_of(const View& v) {
        Span s{};
        s.lo = v.goff;
        s.hi = v.goff + 1;
        for (size_t d = 0; d < v.shape.size(); ++d) s.hi += (v.shape[d] - 1) * v.gstrides[d];
        i64 rows, cols, ld;
        s.rowwise = v.rowwise(rows, cols, ld, true);
        s.ld = s.rowwise ? ld : 0;
        s.c0 = s.rowwise && ld ? v.goff % ld : 0;
        s.c1 = s.c0 + (s.rowwise ? cols : 0);
        s.n = v.numel();
        return s;
    }
    static bool overlap(const Span& a, const Span& b) {
        if (a.hi <= b.lo || b.hi <= a.lo) return false;
        if (a.rowwise && b.rowwise && a.ld == b.ld && a.ld > 0 && (a.c1 <= b.c0 || b.c1 <= a.c0)) return false;
        return true;
    }
    static bool same(const Span& a, const Span& b) {
        return a.lo == b.lo && a.hi == b.hi && a.n == b.n && a.c0 == b.c0 && a.c1 == b.c1;
    }

    void analyze_writes() {
        const Plan& P = ranks[0].P;
        std::map<int, std::vector<Span>> written;
        std::vector<char> need(P.st.size(), 0);
        std::set<int> param_gst;
        for (auto& pv : P.params) param_gst.insert(P.views[(size_t)pv.second].gst);
        if (accum_params)  // every parameter-gradient write accumulates onto the previous micro-batches'
            for (int g : param_gst) {
                Span full{};
                full.hi = P.st[(size_t)g].numel;
                full.n = P.st[(size_t)g].numel;
                written[g].push_back(full);
            }
        auto covered = [&](int gst, const Span& r) {
            auto& w = written[gst];
            for (auto& s : w)
                if (same(s, r)) return true;
            i64 tot = 0;
            for (size_t i = 0; i < w.size(); ++i) {
                for (size_t j = i + 1; j < w.size(); ++j)
                    if (overlap(w[i], w[j])) return false;
                tot += w[i].n;
            }
            return r.lo == 0 && r.n == P.st[(size_t)gst].numel && tot >= r.n;
        };
        auto write = [&](std::map<int, bool>& modes, int v, bool ok) {
            int gst = P.views[(size_t)v].gst;
            Span sp = span_of(P.views[(size_t)v]);
            bool fresh = true;
            for (auto& s : written[gst]) fresh = fresh && !overlap(s, sp);
            if (modes.count(v)) {  // the same view twice in one op: both writes accumulate
                if (modes[v]) need[(size_t)gst] = 1;
                modes[v] = false;
            } else {
                bool ow = fresh && ok;
                if (!ow && fresh) need[(size_t)gst] = 1;  // accumulating onto never-written memory
                modes[v] = ow;
            }
            written[gst].push_back(sp);
        };
        for (int v : P.outputs) write(seed_ow, v, true);
        step_ow.assign(bsteps.size(), {});
        for (size_t si = 0; si < bsteps.size(); ++si) {
            if (bsteps[si].kind != 0) continue;
            const Op& op = P.fwd[(size_t)bsteps[si].idx];
            for (int v : grad_reads(op)) {
                int gst = P.views[(size_t)v].gst;
                if (!covered(gst, span_of(P.views[(size_t)v]))) need[(size_t)gst] = 1;
            }
            for (auto& [v, ok] : grad_slots(P, op)) write(step_ow[si], v, ok);
        }
        auto final_read = [&](int v) {
            int gst = P.views[(size_t)v].gst;
            if (!covered(gst, span_of(P.views[(size_t)v]))) need[(size_t)gst] = 1;
        };
        for (auto& pv : P.params) final_read(pv.second);
        for (int v : P.inputs) final_read(v);
        zero_gst.clear();
        region_zero.assign(P.regions.size(), 0);
        for (size_t g = 0; g < P.st.size(); ++g) {
            if (!need[g] || (accum_params && param_gst.count((int)g))) continue;  // (zeroed by zero_param_grads)
            if (P.st[g].region >= 0) region_zero[(size_t)P.st[g].region] = 1;
            else zero_gst.push_back((int)g);
        }
    }

    size_t workspace_need(const Plan& P) {
        size_t ws = 1 << 20;
        auto rows_of = [&](int v) { return P.views[(size_t)v].numel() / std::max<i64>(1, P.views[(size_t)v].shape.empty() ? 1 : P.views[(size_t)v].shape.back()); };
        for (auto& op : P.fwd) {
            switch (op.k) {
                case K::LayerNorm:
                    ws = std::max(ws, sbk::layernorm_bwd_workspace(rows_of(op.in[0]), P.views[(size_t)op.in[0]].shape.back()));
                    break;
                case K::Linear:
                case K::FusedLinearGelu:
                case K::FusedLinearResLN: {
                    const View& w = P.views[(size_t)op.in[1]];
                    ws = std::max(ws, sbk::bias_grad_workspace(rows_of(op.out[0]), P.views[(size_t)op.out[0]].shape.back()));
                    ws = std::max(ws, sbk::gemm_splitk_workspace(w.shape[0], w.shape[1]));
                    if (op.k == K::FusedLinearResLN)
                        ws = std::max(ws, sbk::bdrln_bwd_workspace(rows_of(op.out[0]), P.views[(size_t)op.out[0]].shape.back()));
                    break;
                }
                case K::FlashAttn: {
                    const auto& q = P.views[(size_t)op.in[0]];
                    ws = std::max(ws, sbk::attn_bwd_workspace(q.shape[0], q.shape[1], op.nh, op.hd));
                    break;
                }
                case K::Embedding:
                    ws = std::max(ws, sbk::embedding_bwd_workspace(P.views[(size_t)op.in[0]].numel(),
                                                                   P.views[(size_t)op.in[1]].shape[1]));
                    break;
                case K::AllGather:
                    ws = std::max(ws, (size_t)P.views[(size_t)op.out[0]].numel() * (size_t)sbk::dt_bytes(cdt));
                    break;
                default: break;
            }
        }
        return align_up(ws);
    }

    void allocate(RankCtx& r) {
        Plan& P = r.P;
        size_t off = 0;
        std::vector<size_t> foff(P.st.size(), SIZE_MAX), goff(P.st.size(), SIZE_MAX);
        // persistent forward
        for (size_t i = 0; i < P.st.size(); ++i) {
            auto& s = P.st[i];
            if (!s.has_fwd || s.region >= 0) continue;
            foff[i] = off;
            off = align_up(off + (size_t)s.numel * (size_t)sbk::dt_bytes(s.dt));
        }
        // persistent grads
        auto wants_grad = [&](const Storage& s) {
            if (s.kind == SKind::Aux) return false;
            if (s.kind == SKind::Act && s.dt == sbk::F64) return false;
            return true;
        };
        size_t gstart = off;
        for (size_t i = 0; i < P.st.size(); ++i) {
            auto& s = P.st[i];
            if (!wants_grad(s) || s.region >= 0) continue;
            goff[i] = off;
            off = align_up(off + (size_t)s.numel * (size_t)sbk::dt_bytes(s.gdt));
        }
        size_t gend = off;
        // checkpoint scratch: every region starts at the same base
        size_t sf = 0, sg = 0;
        std::vector<size_t> rf(P.regions.size(), 0), rg(P.regions.size(), 0);
        std::vector<size_t> lf(P.st.size(), 0), lg(P.st.size(), 0);
        for (size_t i = 0; i < P.st.size(); ++i) {
            auto& s = P.st[i];
            if (s.region < 0) continue;
            if (s.has_fwd) {
                lf[i] = rf[(size_t)s.region];
                rf[(size_t)s.region] = align_up(rf[(size_t)s.region] + (size_t)s.numel * (size_t)sbk::dt_bytes(s.dt));
            }
            if (wants_grad(s)) {
                lg[i] = rg[(size_t)s.region];
                rg[(size_t)s.region] = align_up(rg[(size_t)s.region] + (size_t)s.numel * (size_t)sbk::dt_bytes(s.gdt));
            }
        }
        for (size_t x : rf) sf = std::max(sf, x);
        for (size_t x : rg) sg = std::max(sg, x);
        size_t sf_off = off;
        off += sf;
        size_t sg_off = off;
        off += sg;
        r.ws_bytes = workspace_need(P);
        size_t ws_off = off;
        off += r.ws_bytes;
        // grad-conversion temp: largest activation view
        size_t tmp = 256;
        for (auto& v : P.views) tmp = std::max(tmp, (size_t)v.numel() * (size_t)sbk::dt_bytes(cdt));
        r.tmp_bytes = align_up(tmp);
        size_t tmp_off = off;
        off += r.tmp_bytes;
        std::vector<std::pair<int, size_t>> cs_off;
        const char* bias_epi = getenv("SB_BIAS_EPI");  // 0: bias gradients by the separate column-sum pass (A/B)
        if (cdt == sbk::BF16 && !(bias_epi && atoi(bias_epi) == 0))
            for (size_t i = 0; i < P.fwd.size(); ++i) {
                const Op& op = P.fwd[i];
                if (op.k != K::FusedLinearGelu || !op.dgelu_fused || !op.has_bias || !op.bias_grad) continue;
                const View& y = P.views[(size_t)op.out[0]];
                if (rows_of(y) % 32) continue;
                cs_off.push_back({(int)i, off});
                off += align_up((size_t)(rows_of(y) / 32) * (size_t)cols_of(y) * 4);
            }
        r.total = off;
        CK(cudaMalloc(&r.base, r.total));
        // on our (non-blocking) stream: a legacy-stream memset would race the
        // parameter uploads enqueued below
        CK(cudaMemsetAsync(r.base, 0, r.total, stream));
        CK(cudaStreamSynchronize(stream));
        r.fptr.assign(P.st.size(), nullptr);
        r.gptr.assign(P.st.size(), nullptr);
        for (size_t i = 0; i < P.st.size(); ++i) {
            auto& s = P.st[i];
            if (s.region >= 0) {
                if (s.has_fwd) r.fptr[i] = r.base + sf_off + lf[i];
                if (wants_grad(s)) r.gptr[i] = r.base + sg_off + lg[i];
            } else {
                if (foff[i] != SIZE_MAX) r.fptr[i] = r.base + foff[i];
                if (goff[i] != SIZE_MAX) r.gptr[i] = r.base + goff[i];
            }
        }
        r.ws = r.base + ws_off;
        r.tmp = r.base + tmp_off;
        r.colsum.clear();
        for (auto& [i, o] : cs_off) r.colsum[i] = (float*)(r.base + o);
        r.scratch_grad = r.base + sg_off;
        r.region_grad_span.clear();
        for (size_t k = 0; k < P.regions.size(); ++k) r.region_grad_span.push_back({sg_off, rg[k]});
        persistent_grad_span = {gstart, gend - gstart};
        // parameters: host init (bit-exact with the reference) -> compute dtype
        for (auto& [name, t] : P.param_init) {
            int v = -1;
            for (auto& pv : P.params)
                if (pv.first == name) v = pv.second;
            upload_f64(r, P.views[(size_t)v].st, t.data);
        }
        P.param_init.clear();
        P.param_init.shrink_to_fit();
    }
    std::pair<size_t, size_t> persistent_grad_span{0, 0};

    void upload_f64(RankCtx& r, int st, const std::vector<double>& data) {
        auto& s = r.P.st[(size_t)st];
        double* d = nullptr;
        CK(cudaMalloc(&d, data.size() * sizeof(double)));
        // same stream as the cast: a legacy-stream pageable cudaMemcpy may return
        // before its DMA lands, which a non-blocking stream would not wait for
        CK(cudaMemcpyAsync(d, data.data(), data.size() * sizeof(double), cudaMemcpyHostToDevice, stream));
        sbk::cast(d, sbk::F64, r.fptr[(size_t)st], s.dt, (i64)data.size(), stream);
        CK(cudaStreamSynchronize(stream));
        CK(cudaFree(d));
    }

    // ----------------------------------------------------------- helpers
    char* fp(RankCtx& r, int v) {
        auto& vw = r.P.views[(size_t)v];
        auto& s = r.P.st[(size_t)vw.st];
        return r.fptr[(size_t)vw.st] + vw.off * sbk::dt_bytes(s.dt);
    }
    char* gp(RankCtx& r, int v) {
        auto& vw = r.P.views[(size_t)v];
        auto& s = r.P.st[(size_t)vw.gst];
        if (!r.gptr[(size_t)vw.gst]) throw Error("internal: gradient storage not allocated");
        return r.gptr[(size_t)vw.gst] + vw.goff * sbk::dt_bytes(s.gdt);
    }
    DT gdt(RankCtx& r, int v) { return r.P.st[(size_t)r.P.views[(size_t)v].gst].gdt; }
    DT fdt(RankCtx& r, int v) { return r.P.st[(size_t)r.P.views[(size_t)v].st].dt; }
    const View& V(RankCtx& r, int v) { return r.P.views[(size_t)v]; }
    static i64 rows_of(const View& v) { return v.shape.empty() ? 1 : v.numel() / v.shape.back(); }
    static i64 cols_of(const View& v) { return v.shape.empty() ? 1 : v.shape.back(); }

    // A grad target in the compute dtype: direct pointer, or the temp buffer
    // (zeroed) which `flush` accumulates into an fp32 param/input gradient.
    struct GT {
        char* p;
        bool temp;
        int view;
    };
    GT gtarget(RankCtx& r, int v) {
        if (gdt(r, v) == cdt) return {gp(r, v), false, v};
        CK(cudaMemsetAsync(r.tmp, 0, (size_t)V(r, v).numel() * (size_t)sbk::dt_bytes(cdt), stream));
        if (!V(r, v).g_contiguous()) throw Error("internal: strided fp32 gradient target");
        return {r.tmp, true, v};
    }
    void flush(RankCtx& r, const GT& t) {
        if (!t.temp) return;
        sbk::accumulate(t.p, cdt, gp(r, t.view), gdt(r, t.view), V(r, t.view).numel(), 1.f, stream);
    }

    // every GEMM of the step goes through here: profiling tags them "gemm" and
    // counts their flops (the roofline of the dominant kernel in bench.py)
    double gemm_flops = 0;
    void run_gemm(const sbk::Gemm& g, cudaStream_t st = nullptr) {
        if (!st) st = stream;
        const bool prof = profiling;
        if (prof) {
            prof_begin("gemm");
            gemm_flops += 2.0 * (double)g.M * (double)g.N * (double)g.K * (double)g.batch;
        }
        sbk::gemm(g, st);
        if (prof) prof_end();
        ++launches;
    }

    void gemm_rowwise(RankCtx& r, const void* A, i64 lda, bool a_t, const void* B, i64 ldb, bool b_t, void* C, i64 ldc,
                      DT tc, i64 M, i64 N, i64 K, bool acc, const void* bias, int epi = 0, void* aux = nullptr,
                      cudaStream_t st = nullptr, float* colsum = nullptr) {
        // A(m,k): a_t ? A[k*lda + m] : A[m*lda + k];  B(k,n): b_t ? B[n*ldb + k] : B[k*ldb + n]
        sbk::Gemm g;
        g.A = A;
        g.ta = cdt;
        g.sAm = a_t ? 1 : lda;
        g.sAk = a_t ? lda : 1;
        g.B = B;
        g.tb = cdt;
        g.sBk = b_t ? 1 : ldb;
        g.sBn = b_t ? ldb : 1;
        g.C = C;
        g.tc = tc;
        g.sCm = ldc;
        g.sCn = 1;
        g.M = M;
        g.N = N;
        g.K = K;
        g.accumulate = acc;
        g.bias = bias;
        g.tbias = cdt;
        g.epilogue = epi;
        g.aux = aux;
        g.ws = st && st == wstream ? r.ws2 : r.ws;
        g.ws_bytes = r.ws_bytes;
        g.colsum = colsum;
        run_gemm(g, st);
    }

    // ------------------------------------------------------- collectives
    void all_reduce(std::vector<char*> bufs_in, std::vector<char*> bufs_out, DT t, i64 n, cudaStream_t st = nullptr) {
        if (!st) st = stream;
        if (comm.nccl) {
            nccl().check(nccl().AllReduce(bufs_in[0], bufs_out[0], (size_t)n, nccl_dt(t), ncclSum, ncomm, st),
                         "ncclAllReduce");
            return;
        }
        sbk::sum_ranks((const void* const*)bufs_in.data(), (void* const*)bufs_out.data(), (int)bufs_in.size(), t, n, false,
                       st);
        ++launches;
    }

    // ---------------------------------------- backward all-reduce overlap
    // A Linear whose input is a SyncGrad output (Megatron column-parallel layer,
    // sync_backward): its dgrad completes that gradient, so the SyncGrad's
    // all-reduce is issued on a communication stream right after the dgrad and
    // runs while the weight gradient GEMM runs on the executor stream; the
    // SyncGrad backward step then only waits for it (semantics unchanged:
    // executor.cpp:1071-1083).
    cudaStream_t cstream = nullptr;
    std::vector<int> early_ar;           // per forward op: SyncGrad op whose all-reduce follows its dgrad, or -1
    std::vector<cudaEvent_t> ar_ev;      // per SyncGrad op: its all-reduce completed (on cstream)
    std::vector<cudaEvent_t> dgrad_ev;   // per Linear op with early_ar: its dgrads are enqueued
    std::vector<char> ar_pending;

    void init_early_allreduce() {
        const Plan& P = ranks[0].P;
        early_ar.assign(P.fwd.size(), -1);
        if (world <= 1 && !comm.nccl) return;
        std::vector<int> pos(P.fwd.size(), -1);
        for (size_t k = 0; k < bsteps.size(); ++k)
            if (bsteps[k].kind == 0) pos[(size_t)bsteps[k].idx] = (int)k;
        for (size_t sidx = 0; sidx < P.fwd.size(); ++sidx) {
            const Op& sg = P.fwd[sidx];
            if (sg.k != K::SyncGrad || sg.ids_input || pos[sidx] < 0) continue;
            const int gst = P.views[(size_t)sg.out[0]].gst;
            // the last backward writer of the SyncGrad output's gradient before the SyncGrad step
            int last = -1;
            bool clean = true;
            for (int k = pos[sidx] - 1; k >= 0; --k) {
                const Step& st = bsteps[(size_t)k];
                if (st.kind == 2) {
                    clean = false;
                    break;
                }
                if (st.kind != 0) continue;
                if (grad_writes(P, P.fwd[(size_t)st.idx]).count(gst)) {
                    last = st.idx;
                    break;
                }
            }
            if (!clean || last < 0) continue;
            const Op& l = P.fwd[(size_t)last];
            if (l.k != K::Linear && l.k != K::FusedLinearGelu) continue;
            if (l.dgelu_pre >= 0 || P.views[(size_t)l.in[0]].gst != gst) continue;
            if (gdt(ranks[0], l.in[0]) != cdt) continue;  // dgrad through an fp32 temp: keep the plain order
            early_ar[(size_t)last] = (int)sidx;
        }
        bool any = false;
        ar_ev.assign(P.fwd.size(), nullptr);
        dgrad_ev.assign(P.fwd.size(), nullptr);
        ar_pending.assign(P.fwd.size(), 0);
        for (size_t k = 0; k < P.fwd.size(); ++k)
            if (early_ar[k] >= 0) {
                CK(cudaEventCreateWithFlags(&dgrad_ev[k], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&ar_ev[(size_t)early_ar[k]], cudaEventDisableTiming));
                any = true;
            }
        if (any || world > 1 || comm.nccl) {
            int lo, hi;
            CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CK(cudaStreamCreateWithPriority(&cstream, cudaStreamNonBlocking, hi));  // communication first
        }
    }

    // backward of a Linear / FusedLinearGelu whose dgrad feeds an early all-reduce
    void linear_bwd_overlapped(int i) {
        const int sidx = early_ar[(size_t)i];
        auto gin = [&](RankCtx& r, const Op& op) {
            if (op.k == K::FusedLinearGelu) {
                const View& y = V(r, op.out[0]);
                if (!op.dgelu_fused)
                    sbk::unary_bwd(2, fp(r, op.out[1]), gp(r, op.out[0]), gp(r, op.out[1]), cdt, cdt, y.numel(), 1.f,
                                   stream);
                return std::make_pair((const void*)gp(r, op.out[1]), cols_of(y));
            }
            const View& y = V(r, op.out[0]);
            return std::make_pair((const void*)gp(r, op.out[0]), cols_of(y));
        };
        std::vector<std::pair<const void*, i64>> g(ranks.size());
        for (size_t k = 0; k < ranks.size(); ++k) {
            const Op& op = ranks[k].P.fwd[(size_t)i];
            g[k] = gin(ranks[k], op);
            linear_bwd(ranks[k], op, g[k].first, g[k].second, 1);
        }
        // all-reduce of the SyncGrad output gradient on the communication stream
        CK(cudaEventRecord(dgrad_ev[(size_t)i], stream));
        CK(cudaStreamWaitEvent(cstream, dgrad_ev[(size_t)i], 0));
        std::vector<char*> b;
        for (auto& r : ranks) b.push_back(gp(r, r.P.fwd[(size_t)sidx].out[0]));
        all_reduce(b, b, cdt, V(ranks[0], ranks[0].P.fwd[(size_t)sidx].out[0]).numel(), cstream);
        CK(cudaEventRecord(ar_ev[(size_t)sidx], cstream));
        ar_pending[(size_t)sidx] = 1;
        CommSmReserve keep_sms(*this);
        for (size_t k = 0; k < ranks.size(); ++k) linear_bwd(ranks[k], ranks[k].P.fwd[(size_t)i], g[k].first, g[k].second, 2);
    }

    // ------------------------------------------------------- forward op
    void fwd_op(int i, bool recompute = false) {
        const Op& op0 = ranks[0].P.fwd[(size_t)i];
        NvtxRange trace(k_str(op0.k), recompute ? " (re)" : "", op0.path);
        if (profiling) prof_begin(std::string(k_str(op0.k)) + (recompute ? "(re)" : ""));
        switch (op0.k) {
            case K::AllReduce: {
                ++collectives;
                if (!op0.allreduce) break;
                std::vector<char*> in, out;
                for (auto& r : ranks) {
                    in.push_back(fp(r, r.P.fwd[(size_t)i].in[0]));
                    out.push_back(fp(r, r.P.fwd[(size_t)i].out[0]));
                }
                all_reduce(in, out, cdt, V(ranks[0], op0.in[0]).numel());
                break;
            }
            case K::AllGather: {
                ++collectives;
                const View& xv = V(ranks[0], op0.in[0]);
                i64 n = xv.numel(), inner = 1, outer = 1;
                for (size_t d = (size_t)op0.axis; d < xv.shape.size(); ++d) inner *= xv.shape[d];
                outer = n / inner;
                if (comm.nccl) {
                    RankCtx& r = ranks[0];
                    if (world > 1)
                        nccl().check(nccl().AllGather(fp(r, op0.in[0]), r.ws, (size_t)n, nccl_dt(cdt), ncomm, stream),
                                     "ncclAllGather");
                    else
                        CK(cudaMemcpyAsync(r.ws, fp(r, op0.in[0]), (size_t)n * sbk::dt_bytes(cdt), cudaMemcpyDeviceToDevice, stream));
                    // ws is (world, outer, inner) -> out (outer, world, inner)
                    i64 shape[3] = {outer, world, inner}, ss[3] = {inner, n, 1}, ds[3] = {world * inner, inner, 1};
                    sbk::strided_copy(r.ws, cdt, ss, fp(r, r.P.fwd[(size_t)i].out[0]), cdt, ds, shape, 3, false, stream);
                } else {
                    for (auto& dst : ranks)
                        for (int src = 0; src < world; ++src) {
                            i64 shape[2] = {outer, inner}, ss[2] = {inner, 1}, ds[2] = {world * inner, 1};
                            sbk::strided_copy(fp(ranks[(size_t)src], op0.in[0]), cdt, ss,
                                              fp(dst, dst.P.fwd[(size_t)i].out[0]) + (size_t)src * inner * sbk::dt_bytes(cdt),
                                              cdt, ds, shape, 2, false, stream);
                        }
                }
                break;
            }
            case K::FusedLinearResLN:
                if (op0.allreduce && fwd_ar_chunks(ranks[0], op0) > 1) {
                    fused_res_ln_overlapped(i, fwd_ar_chunks(ranks[0], op0));
                    break;
                }
                for (auto& r : ranks) fused_res_ln_gemm(r, r.P.fwd[(size_t)i]);
                if (op0.allreduce) {
                    ++collectives;
                    std::vector<char*> b;
                    for (auto& r : ranks) b.push_back(fp(r, r.P.fwd[(size_t)i].out[1]));
                    all_reduce(b, b, cdt, V(ranks[0], op0.out[1]).numel());
                }
                for (auto& r : ranks) fused_res_ln_tail(r, r.P.fwd[(size_t)i]);
                break;
            default:
                for (auto& r : ranks) fwd_local(r, r.P.fwd[(size_t)i]);
        }
        if (profiling) prof_end();
        if (nan_guard) check_nan(i);
    }

    // NaN guard (Executor::set_nan_guard, reference executor.cpp:308-316,845: the NaN check after
    // every forward op): each op's outputs are counted into a per-op device counter
    // (no host sync, so it also runs inside a captured graph); the counters are read
    // once after the forward (eager) or after the graph replay, and the first op that
    // produced a NaN is reported.
    int* nan_counts = nullptr;
    size_t nan_n = 0;
    void nan_alloc() {  // (not inside a graph capture: set_nan_guard)
        const size_t n = ranks[0].P.fwd.size() * ranks.size();
        if (nan_n < n) {
            if (nan_counts) cudaFree(nan_counts);
            CK(cudaMalloc(&nan_counts, n * sizeof(int)));
            nan_n = n;
        }
    }
    void nan_reset() { CK(cudaMemsetAsync(nan_counts, 0, nan_n * sizeof(int), stream)); }
    void check_nan(int i) {
        for (size_t k = 0; k < ranks.size(); ++k) {
            RankCtx& r = ranks[k];
            const Op& op = r.P.fwd[(size_t)i];
            if (op.k == K::Cast) continue;  // input / dtype conversions are not reference ops
            for (int v : op.out) {
                if (fdt(r, v) == sbk::F64 || r.P.st[(size_t)V(r, v).st].kind == SKind::Aux) continue;
                sbk::count_nan(fp(r, v), fdt(r, v), V(r, v).numel(), nan_counts + k * ranks[0].P.fwd.size() + (size_t)i,
                               stream);
            }
        }
    }
    void nan_report() {
        const size_t nf = ranks[0].P.fwd.size();
        std::vector<int> h(nf * ranks.size());
        CK(cudaMemcpyAsync(h.data(), nan_counts, h.size() * sizeof(int), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        for (size_t i = 0; i < nf; ++i)
            for (size_t k = 0; k < ranks.size(); ++k)
                if (h[k * nf + i])
                    throw Error(std::string("NaN produced by op '") + k_str(ranks[k].P.fwd[i].k) + "' on rank " +
                                std::to_string(ranks[k].P.rank));
    }

    // ---------------------------------------- forward all-reduce overlap
    // Row-parallel Linear (Megatron out.dense / dense2, sync forward) -> all_reduce ->
    // bias+dropout+residual+LayerNorm: the rows are cut into chunks; the GEMM of chunk
    // c+1 runs on the executor stream while chunk c is all-reduced on the
    // communication stream, and each chunk's LayerNorm tail waits only for its own
    // all-reduce. Every row's values are the unchunked ones (a row's GEMM, sum over
    // ranks and LayerNorm do not depend on other rows; the keep bits are indexed by
    // the global element index), so the semantics are the reference's
    // (executor.cpp:812-820 all_reduce, schedule.cpp:205-309 sync forward).
    std::vector<cudaEvent_t> far_gemm, far_done;  // per chunk (reused across ops)
    // NCCL kernels need SMs of their own to run beside a persistent GEMM: while a
    // collective is in flight on cstream, the 2-SM GEMM leaves $SB_COMM_SMS (16) SMs free
    struct CommSmReserve {
        explicit CommSmReserve(ExecutorImpl& e) {
            if (!(e.comm.nccl && e.world > 1)) return;
            static const int n = getenv("SB_COMM_SMS") ? atoi(getenv("SB_COMM_SMS")) : 16;
            sbk::gemm_set_sm_reserve(n);
            on = true;
        }
        ~CommSmReserve() {
            if (on) sbk::gemm_set_sm_reserve(0);
        }
        bool on = false;
    };
    int fwd_ar_chunk_cap = -1;
    int fwd_ar_chunks(RankCtx& r, const Op& op) {
        if (fwd_ar_chunk_cap < 0) {
            const char* e = getenv("SB_FWD_AR_CHUNKS");
            fwd_ar_chunk_cap = e ? std::max(1, atoi(e)) : 4;
        }
        if (!cstream) return 1;
        const View& y = V(r, op.out[0]);
        const i64 rows = rows_of(y), n = cols_of(y);
        if (op.dropout && !op.s1) return 1;
        // chunks of >= 256 rows (whole 2-SM GEMM tiles) whose keep bits start on a word
        int c = fwd_ar_chunk_cap;
        while (c > 1 && (rows % c || (rows / c) % 256 || ((rows / c) * n) % 32)) --c;
        return c;
    }
    void fused_res_ln_overlapped(int i, int nch) {
        ++collectives;
        while ((int)far_gemm.size() < nch) {
            cudaEvent_t a, b;
            CK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
            far_gemm.push_back(a);
            far_done.push_back(b);
        }
        const Op& op0 = ranks[0].P.fwd[(size_t)i];
        const i64 rows = rows_of(V(ranks[0], op0.out[0])), cr = rows / nch;
        const size_t eb = sbk::dt_bytes(cdt);
        CommSmReserve keep_sms(*this);
        for (int c = 0; c < nch; ++c) {
            std::vector<char*> part;
            for (auto& r : ranks) {
                const Op& op = r.P.fwd[(size_t)i];
                const View& x = V(r, op.in[0]);
                const View& w = V(r, op.in[1]);
                i64 xr, cols, ldx;
                x.rowwise(xr, cols, ldx);
                const i64 out_f = w.shape[0];
                char* pc = fp(r, op.out[1]) + (size_t)(c * cr * out_f) * eb;
                gemm_rowwise(r, fp(r, op.in[0]) + (size_t)(c * cr * ldx) * eb, ldx, false, fp(r, op.in[1]), cols, true,
                             pc, out_f, cdt, cr, out_f, cols, false, nullptr);
                ++launches;
                part.push_back(pc);
            }
            CK(cudaEventRecord(far_gemm[(size_t)c], stream));
            CK(cudaStreamWaitEvent(cstream, far_gemm[(size_t)c], 0));
            all_reduce(part, part, cdt, cr * V(ranks[0], op0.out[1]).shape.back(), cstream);
            CK(cudaEventRecord(far_done[(size_t)c], cstream));
        }
        for (int c = 0; c < nch; ++c) {
            CK(cudaStreamWaitEvent(stream, far_done[(size_t)c], 0));
            for (auto& r : ranks) fused_res_ln_tail(r, r.P.fwd[(size_t)i], c * cr, cr);
        }
    }

    void fused_res_ln_gemm(RankCtx& r, const Op& op) {
        const View& x = V(r, op.in[0]);
        const View& w = V(r, op.in[1]);
        i64 rows, cols, ldx;
        x.rowwise(rows, cols, ldx);
        i64 out_f = w.shape[0];
        gemm_rowwise(r, fp(r, op.in[0]), ldx, false, fp(r, op.in[1]), cols, true, fp(r, op.out[1]), out_f, cdt, rows,
                     out_f, cols, false, nullptr);
        ++launches;
    }
    // rows [row0, row0 + nrows) (all rows when nrows < 0)
    void fused_res_ln_tail(RankCtx& r, const Op& op, i64 row0 = 0, i64 nrows = -1) {
        const View& y = V(r, op.out[0]);
        i64 rows = rows_of(y), n = cols_of(y);
        if (nrows >= 0) rows = nrows;
        const size_t eo = (size_t)(row0 * n) * sbk::dt_bytes(cdt);
        const void* bias = op.has_bias && op.bias_on ? fp(r, op.in[5]) : nullptr;
        sbk::bias_dropout_residual_ln_fwd(fp(r, op.out[1]) + eo, bias, fp(r, op.in[2]) + eo, fp(r, op.in[3]), fp(r, op.in[4]),
                                          cdt, fp(r, op.out[2]) + eo, fp(r, op.out[0]) + eo,
                                          (float*)fp(r, op.out[3]) + row0, (float*)fp(r, op.out[4]) + row0, cdt, rows, n,
                                          (float)op.eps, op.s1, op.dropout ? op.thr : 0, (float)(1.0 / (1.0 - op.p)),
                                          stream,
                                          op.dropout ? (const uint32_t*)fp(r, op.out[5]) + (row0 * n) / 32 : nullptr);
        ++launches;
    }

    void fwd_local(RankCtx& r, const Op& op) {
        ++launches;
        switch (op.k) {
            case K::Cast:
                sbk::cast(fp(r, op.in[0]), fdt(r, op.in[0]), fp(r, op.out[0]), fdt(r, op.out[0]), V(r, op.out[0]).numel(), stream);
                break;
            case K::Linear: {
                const View& x = V(r, op.in[0]);
                const View& w = V(r, op.in[1]);
                i64 rows, cols, ldx;
                x.rowwise(rows, cols, ldx);
                i64 out_f = w.shape[0];
                gemm_rowwise(r, fp(r, op.in[0]), ldx, false, fp(r, op.in[1]), cols, true, fp(r, op.out[0]), out_f, cdt, rows,
                             out_f, cols, false, op.bias_on ? fp(r, op.in[2]) : nullptr, op.act ? 3 : 0);
                break;
            }
            case K::FusedLinearGelu: {
                const View& x = V(r, op.in[0]);
                const View& w = V(r, op.in[1]);
                i64 rows, cols, ldx;
                x.rowwise(rows, cols, ldx);
                i64 out_f = w.shape[0];
                gemm_rowwise(r, fp(r, op.in[0]), ldx, false, fp(r, op.in[1]), cols, true, fp(r, op.out[0]), out_f, cdt, rows,
                             out_f, cols, false, op.bias_on ? fp(r, op.in[2]) : nullptr, 1, fp(r, op.out[1]));
                break;
            }
            case K::LayerNorm: {
                const View& x = V(r, op.in[0]);
                sbk::layernorm_fwd(fp(r, op.in[0]), op.affine ? fp(r, op.in[1]) : nullptr,
                                   op.affine ? fp(r, op.in[2]) : nullptr, cdt, fp(r, op.out[0]), (float*)fp(r, op.out[1]),
                                   (float*)fp(r, op.out[2]), cdt, rows_of(x), cols_of(x), (float)op.eps, stream);
                break;
            }
            case K::Dropout:
                sbk::dropout(fp(r, op.in[0]), fp(r, op.out[0]), cdt, V(r, op.out[0]).numel(), op.s1, op.thr,
                             (float)(1.0 / (1.0 - op.p)), false, stream);
                break;
            case K::Add:
            case K::Mul:
                sbk::binary(op.k == K::Add ? 0 : 1, fp(r, op.in[0]), V(r, op.in[0]).numel(), fp(r, op.in[1]),
                            V(r, op.in[1]).numel(), fp(r, op.out[0]), cdt, V(r, op.out[0]).numel(), stream);
                break;
            case K::Scale:
            case K::Relu:
            case K::Gelu:
                sbk::unary(op.k == K::Scale ? 0 : op.k == K::Relu ? 1 : 2, fp(r, op.in[0]), fp(r, op.out[0]), cdt,
                           V(r, op.out[0]).numel(), (float)op.scale, stream);
                break;
            case K::Softmax: {
                i64 outer, n, inner;
                axis_split(V(r, op.in[0]), op.axis, outer, n, inner);
                sbk::softmax_fwd(fp(r, op.in[0]), fp(r, op.out[0]), cdt, outer, n, inner, stream,
                                 op.causal ? V(r, op.in[0]).shape[V(r, op.in[0]).shape.size() - 2] : 0);
                break;
            }
            case K::Matmul: {
                const View& a = V(r, op.in[0]);
                const View& b = V(r, op.in[1]);
                int ra = (int)a.shape.size();
                i64 m = a.shape[(size_t)ra - 2], k = a.shape[(size_t)ra - 1], n = b.shape.back();
                sbk::Gemm g;
                g.A = fp(r, op.in[0]);
                g.ta = cdt;
                g.sAb = m * k;
                g.sAm = k;
                g.sAk = 1;
                g.B = fp(r, op.in[1]);
                g.tb = cdt;
                g.sBb = k * n;
                g.sBk = n;
                g.sBn = 1;
                g.C = fp(r, op.out[0]);
                g.tc = cdt;
                g.sCb = m * n;
                g.sCm = n;
                g.sCn = 1;
                g.batch = a.numel() / (m * k);
                g.M = m;
                g.N = n;
                g.K = k;
                run_gemm(g);
                break;
            }
            case K::Permute: {
                const View& x = V(r, op.in[0]);
                const View& y = V(r, op.out[0]);
                std::vector<i64> ss(op.perm.size());
                for (size_t d = 0; d < op.perm.size(); ++d) ss[d] = x.strides[(size_t)op.perm[d]];
                sbk::strided_copy(fp(r, op.in[0]), cdt, ss.data(), fp(r, op.out[0]), cdt, y.strides.data(), y.shape.data(),
                                  (int)y.shape.size(), false, stream);
                break;
            }
            case K::Copy: {
                const View& x = V(r, op.in[0]);
                const View& y = V(r, op.out[0]);
                sbk::strided_copy(fp(r, op.in[0]), cdt, x.strides.data(), fp(r, op.out[0]), cdt, y.strides.data(),
                                  y.shape.data(), (int)y.shape.size(), false, stream);
                break;
            }
            case K::Concat: {
                const View& y = V(r, op.out[0]);
                i64 offset = 0;
                for (int v : op.in) {
                    const View& x = V(r, v);
                    char* dst = fp(r, op.out[0]) + (size_t)(offset * y.strides[(size_t)op.axis]) * sbk::dt_bytes(cdt);
                    sbk::strided_copy(fp(r, v), cdt, x.strides.data(), dst, cdt, y.strides.data(), x.shape.data(),
                                      (int)x.shape.size(), false, stream);
                    offset += x.shape[(size_t)op.axis];
                }
                break;
            }
            case K::ReduceSum: {
                const View& x = V(r, op.in[0]);
                if (op.reduce_all) {
                    sbk::reduce_all(fp(r, op.in[0]), cdt, x.numel(), fp(r, op.out[0]), cdt, false, stream);
                } else {
                    i64 outer, n, inner;
                    axis_split(x, op.axis, outer, n, inner);
                    sbk::reduce_axis(fp(r, op.in[0]), fp(r, op.out[0]), cdt, outer, n, inner, false, stream);
                }
                break;
            }
            case K::SyncGrad: --launches; break;  // identity forward (executor.cpp:450-461)
            case K::Embedding: {
                const View& ids = V(r, op.in[0]);
                const View& w = V(r, op.in[1]);
                sbk::embedding_fwd((const double*)fp(r, op.in[0]), ids.numel(), fp(r, op.in[1]), cdt, w.shape[1],
                                   op.full_rows, op.row0, w.shape[0], fp(r, op.out[0]), stream);
                break;
            }
            case K::FlashAttn: sbk::attn_fwd(attn_args(r, op), stream); break;  // keep bits: launch_masks()
            default: throw Error(std::string("internal: no forward launcher for ") + k_str(op.k));
        }
    }

    sbk::Attn attn_args(RankCtx& r, const Op& op) {
        sbk::Attn a;
        const View& q = V(r, op.in[0]);
        i64 rows, cols;
        a.q = fp(r, op.in[0]);
        a.k = fp(r, op.in[1]);
        a.v = fp(r, op.in[2]);
        a.o = fp(r, op.out[0]);
        q.rowwise(rows, cols, a.ld_q);
        V(r, op.in[1]).rowwise(rows, cols, a.ld_k);
        V(r, op.in[2]).rowwise(rows, cols, a.ld_v);
        a.ld_o = cols;
        a.lse = (float*)fp(r, op.out[1]);
        a.B = q.shape[0];
        a.S = q.shape[1];
        a.Sk = V(r, op.in[1]).shape[1] != a.S ? V(r, op.in[1]).shape[1] : 0;  // cross-attention keys
        a.nh = op.nh;
        a.hd = op.hd;
        a.scale = (float)op.scale;
        a.s1 = op.dropout ? op.s1 : 0;
        a.thr = op.dropout ? op.thr : 0;
        a.dscale = (float)(1.0 / (1.0 - op.p));
        a.t = cdt;
        a.mask = op.dropout ? (const uint32_t*)fp(r, op.out[2]) : nullptr;
        if (a.mask && a.S % 128 == 0 && a.keys() % 128 == 0) a.mask_t = a.mask + (a.B * a.nh * a.S * a.keys()) / 32;
        a.causal = op.causal;
        return a;
    }

    static void axis_split(const View& v, int axis, i64& outer, i64& n, i64& inner) {
        outer = 1;
        inner = 1;
        for (int d = 0; d < axis; ++d) outer *= v.shape[(size_t)d];
        n = v.shape.empty() ? 1 : v.shape[(size_t)axis];
        for (size_t d = (size_t)axis + 1; d < v.shape.size(); ++d) inner *= v.shape[d];
    }

    // ------------------------------------------------------ backward op
    // part: 1 dgrad only, 2 weight/bias gradients only, 3 both
    void linear_bwd(RankCtx& r, const Op& op, const void* g, i64 ldg, int part = 3) {
        // dx += g W (executor.cpp:101-118); dW += g^T x (:121-133); db += colsum g (:1146-1154)
        const View& x = V(r, op.in[0]);
        const View& w = V(r, op.in[1]);
        i64 rows, cols, ldx, gr, gc, ldgx;
        x.rowwise(rows, cols, ldx);
        i64 out_f = w.shape[0];
        const bool side = part == 3 && wside_eligible(r, op);
        if (side) {  // fork before the dgrad: everything g and x depend on is enqueued
            cudaEvent_t f = next_fork();
            CK(cudaEventRecord(f, stream));
            CK(cudaStreamWaitEvent(wstream, f, 0));
            wside_pending = true;
        }
        if (!(part & 1)) {
        } else if (op.dgelu_pre >= 0) {
            // dx lands directly as the producing GeLU's input gradient: gelu'(pre) * (g W);
            // the epilogue also leaves the column partials of the producer's bias gradient
            int fi = -1;
            for (size_t k = 0; k < r.P.fwd.size(); ++k)
                if (r.P.fwd[k].k == K::FusedLinearGelu && r.P.fwd[k].out[1] == op.dgelu_pre) fi = (int)k;
            auto cs = r.colsum.find(fi);
            float* csp = cs != r.colsum.end() && OW(op.dgelu_pre) ? cs->second : nullptr;
            gemm_rowwise(r, g, ldg, false, fp(r, op.in[1]), cols, false, gp(r, op.dgelu_pre), cols, cdt, rows, cols,
                         out_f, !OW(op.dgelu_pre), nullptr, 2, fp(r, op.dgelu_pre), nullptr, csp);
            if (csp && sbk::gemm_last_colsum()) r.colsum_ready.insert(fi);
        } else if (op.drelu) {
            // dx lands as the gradient at the folded ReLU's input: (g W) * (x > 0), x this op's input
            gemm_rowwise(r, g, ldg, false, fp(r, op.in[1]), cols, false, gp(r, op.in[0]), cols, cdt, rows, cols, out_f,
                         !OW(op.in[0]), nullptr, 4, fp(r, op.in[0]));
        } else {
            GT gx = gtarget(r, op.in[0]);
            if (gx.temp) ldgx = cols;
            else x.rowwise(gr, gc, ldgx, true);
            gemm_rowwise(r, g, ldg, false, fp(r, op.in[1]), cols, false, gx.p, ldgx, cdt, rows, cols, out_f,
                         gx.temp || !OW(op.in[0]), nullptr);
            flush(r, gx);
        }
        if (!(part & 2)) {
            ++launches;
            return;
        }
        cudaStream_t ws = side ? wstream : stream;
        gemm_rowwise(r, g, ldg, true, fp(r, op.in[0]), ldx, false, gp(r, op.in[1]), cols, gdt(r, op.in[1]), out_f, cols,
                     rows, !OW(op.in[1]), nullptr, 0, nullptr, ws);
        launches += (part & 1) ? 2 : 1;
        if (op.has_bias && op.bias_grad) {
            const int oi = (int)(&op - r.P.fwd.data());
            if (r.colsum_ready.erase(oi))  // partials from the consumer's dgrad epilogue
                sbk::bias_grad_partials(r.colsum.at(oi), rows / 32, out_f, (float*)gp(r, op.in[2]), ws, !OW(op.in[2]));
            else
                sbk::bias_grad(g, cdt, ldg, rows, out_f, (float*)gp(r, op.in[2]), (float*)(side ? r.ws2 : r.ws), ws,
                               !OW(op.in[2]));
            ++launches;
        }
    }

    void bwd_op(int i) {
        const Op& op0 = ranks[0].P.fwd[(size_t)i];
        NvtxRange trace(k_str(op0.k), " (bwd)", op0.path);
        if (profiling) prof_begin(std::string(k_str(op0.k)) + "(bwd)");
        if (early_ar.size() > (size_t)i && early_ar[(size_t)i] >= 0) {
            linear_bwd_overlapped(i);
            if (profiling) prof_end();
            return;
        }
        switch (op0.k) {
            case K::SyncGrad: {
                // Σ_r of the module input's gradient, accumulated on every rank (executor.cpp:1071-1083)
                ++collectives;
                if (op0.ids_input) break;  // id inputs are not differentiable: the sum is of zeros
                std::vector<char*> b;
                for (auto& r : ranks) b.push_back(gp(r, r.P.fwd[(size_t)i].out[0]));
                i64 n = V(ranks[0], op0.out[0]).numel();
                if (ar_pending.size() > (size_t)i && ar_pending[(size_t)i]) {
                    CK(cudaStreamWaitEvent(stream, ar_ev[(size_t)i], 0));  // issued right after the dgrad
                    ar_pending[(size_t)i] = 0;
                } else if (world > 1 || comm.nccl) {
                    all_reduce(b, b, cdt, n);
                }
                for (auto& r : ranks) {
                    const Op& op = r.P.fwd[(size_t)i];
                    accumulate_view(r, op.out[0], op.in[0], !OW(op.in[0]));
                }
                break;
            }
            case K::FusedLinearResLN: {
                for (auto& r : ranks) {
                    const Op& op = r.P.fwd[(size_t)i];
                    const View& y = V(r, op.out[0]);
                    i64 rows = rows_of(y), n = cols_of(y);
                    GT gres = gtarget(r, op.in[2]);
                    sbk::bias_dropout_residual_ln_bwd(
                        fp(r, op.out[2]), (float*)fp(r, op.out[3]), (float*)fp(r, op.out[4]), fp(r, op.in[3]), cdt,
                        gp(r, op.out[0]), gres.p, gp(r, op.out[1]), false,
                        op.has_bias && op.bias_grad ? (float*)gp(r, op.in[5]) : nullptr, (float*)gp(r, op.in[3]),
                        (float*)gp(r, op.in[4]), cdt, rows, n, op.s1, op.dropout ? op.thr : 0,
                        (float)(1.0 / (1.0 - op.p)), (float*)r.ws, stream, gres.temp || !OW(op.in[2]), !OW(op.in[3]),
                        op.dropout ? (const uint32_t*)fp(r, op.out[5]) : nullptr,
                        op.sum_ext ? gp(r, op.out[2]) : nullptr);  // (pre-LN: the residual stream's gradient)
                    flush(r, gres);
                    ++launches;
                    // the in-region all_reduce backpropagates as identity (executor.cpp:1227-1233)
                    Op lin = op;
                    lin.has_bias = false;
                    linear_bwd(r, lin, gp(r, op.out[1]), n);
                }
                break;
            }
            default:
                for (auto& r : ranks) bwd_local(r, r.P.fwd[(size_t)i]);
        }
        if (profiling) prof_end();
    }

    void accumulate_view(RankCtx& r, int from, int to, bool acc = true) {
        // grad(to) (+)= grad(from); equal shapes
        const View& a = V(r, from);
        const View& b = V(r, to);
        if (a.g_contiguous() && b.g_contiguous()) {
            if (acc) sbk::accumulate(gp(r, from), gdt(r, from), gp(r, to), gdt(r, to), a.numel(), 1.f, stream);
            else sbk::cast(gp(r, from), gdt(r, from), gp(r, to), gdt(r, to), a.numel(), stream);
        } else {
            if (gdt(r, from) != gdt(r, to)) throw Error("internal: strided dtype-converting accumulate");
            sbk::strided_copy(gp(r, from), gdt(r, from), a.gstrides.data(), gp(r, to), gdt(r, to), b.gstrides.data(),
                              a.shape.data(), (int)a.shape.size(), acc, stream);
        }
        ++launches;
    }

    void bwd_local(RankCtx& r, const Op& op) {
        ++launches;
        switch (op.k) {
            case K::Cast:
                if (fdt(r, op.out[0]) == sbk::F64) break;  // ids: not differentiable
                if (OW(op.in[0]))
                    sbk::cast(gp(r, op.out[0]), cdt, gp(r, op.in[0]), gdt(r, op.in[0]), V(r, op.out[0]).numel(), stream);
                else
                    sbk::accumulate(gp(r, op.out[0]), cdt, gp(r, op.in[0]), gdt(r, op.in[0]), V(r, op.out[0]).numel(), 1.f,
                                    stream);
                break;
            case K::Linear: {
                const View& y = V(r, op.out[0]);
                --launches;
                linear_bwd(r, op, gp(r, op.out[0]), cols_of(y));
                break;
            }
            case K::FusedLinearGelu: {
                const View& y = V(r, op.out[0]);
                if (!op.dgelu_fused)  // else the consumer's dgrad already wrote gelu'(pre) * g
                    sbk::unary_bwd(2, fp(r, op.out[1]), gp(r, op.out[0]), gp(r, op.out[1]), cdt, cdt, y.numel(), 1.f,
                                   stream);
                linear_bwd(r, op, gp(r, op.out[1]), cols_of(y));
                break;
            }
            case K::LayerNorm: {
                const View& x = V(r, op.in[0]);
                GT gx = gtarget(r, op.in[0]);
                sbk::layernorm_bwd(fp(r, op.in[0]), (float*)fp(r, op.out[1]), (float*)fp(r, op.out[2]),
                                   op.affine ? fp(r, op.in[1]) : nullptr, cdt, gp(r, op.out[0]), cdt, gx.p,
                                   op.affine ? (float*)gp(r, op.in[1]) : nullptr,
                                   op.affine ? (float*)gp(r, op.in[2]) : nullptr, cdt, rows_of(x), cols_of(x),
                                   (float*)r.ws, stream, gx.temp || !OW(op.in[0]), !op.affine || !OW(op.in[1]));
                flush(r, gx);
                break;
            }
            case K::Dropout: {
                GT gx = gtarget(r, op.in[0]);
                sbk::dropout(gp(r, op.out[0]), gx.p, cdt, V(r, op.out[0]).numel(), op.s1, op.thr,
                             (float)(1.0 / (1.0 - op.p)), gx.temp || !OW(op.in[0]), stream);
                flush(r, gx);
                break;
            }
            case K::Add: {
                i64 n = V(r, op.out[0]).numel();
                for (int k = 0; k < 2; ++k) {
                    GT gx = gtarget(r, op.in[(size_t)k]);
                    bool acc = gx.temp || !OW(op.in[(size_t)k]);
                    if (V(r, op.in[(size_t)k]).numel() == 1 && n != 1)
                        sbk::reduce_all(gp(r, op.out[0]), cdt, n, gx.p, cdt, acc, stream);
                    else if (acc)
                        sbk::accumulate(gp(r, op.out[0]), cdt, gx.p, cdt, n, 1.f, stream);
                    else
                        sbk::cast(gp(r, op.out[0]), cdt, gx.p, cdt, n, stream);
                    flush(r, gx);
                }
                break;
            }
            case K::Mul: {
                i64 n = V(r, op.out[0]).numel();
                for (int k = 0; k < 2; ++k) {
                    GT gx = gtarget(r, op.in[(size_t)k]);
                    int other = op.in[(size_t)(1 - k)];
                    sbk::mul_bwd(gp(r, op.out[0]), cdt, fp(r, other), V(r, other).numel(), gx.p, cdt,
                                 V(r, op.in[(size_t)k]).numel(), n, stream);
                    flush(r, gx);
                }
                break;
            }
            case K::Scale:
            case K::Relu:
            case K::Gelu: {
                GT gx = gtarget(r, op.in[0]);
                sbk::unary_bwd(op.k == K::Scale ? 0 : op.k == K::Relu ? 1 : 2, fp(r, op.in[0]), gp(r, op.out[0]), gx.p, cdt,
                               cdt, V(r, op.out[0]).numel(), (float)op.scale, stream);
                flush(r, gx);
                break;
            }
            case K::Softmax: {
                i64 outer, n, inner;
                axis_split(V(r, op.in[0]), op.axis, outer, n, inner);
                GT gx = gtarget(r, op.in[0]);
                sbk::softmax_bwd(fp(r, op.out[0]), gp(r, op.out[0]), gx.p, cdt, cdt, outer, n, inner, stream);
                flush(r, gx);
                break;
            }
            case K::Matmul: {
                // ga += g b^T ; gb += a^T g  (executor.cpp:1257-1264)
                const View& a = V(r, op.in[0]);
                const View& b = V(r, op.in[1]);
                int ra = (int)a.shape.size();
                i64 m = a.shape[(size_t)ra - 2], k = a.shape[(size_t)ra - 1], n = b.shape.back();
                i64 batch = a.numel() / (m * k);
                GT ga = gtarget(r, op.in[0]);
                sbk::Gemm g;
                g.ta = g.tb = cdt;
                g.A = gp(r, op.out[0]);
                g.sAb = m * n;
                g.sAm = n;
                g.sAk = 1;
                g.B = fp(r, op.in[1]);
                g.sBb = k * n;
                g.sBk = 1;
                g.sBn = n;
                g.C = ga.p;
                g.tc = cdt;
                g.sCb = m * k;
                g.sCm = k;
                g.sCn = 1;
                g.batch = batch;
                g.M = m;
                g.N = k;
                g.K = n;
                g.accumulate = true;
                run_gemm(g);
                flush(r, ga);
                GT gb = gtarget(r, op.in[1]);
                sbk::Gemm h;
                h.ta = h.tb = cdt;
                h.A = fp(r, op.in[0]);
                h.sAb = m * k;
                h.sAm = 1;
                h.sAk = k;
                h.B = gp(r, op.out[0]);
                h.sBb = m * n;
                h.sBk = n;
                h.sBn = 1;
                h.C = gb.p;
                h.tc = cdt;
                h.sCb = k * n;
                h.sCm = n;
                h.sCn = 1;
                h.batch = batch;
                h.M = k;
                h.N = n;
                h.K = m;
                h.accumulate = true;
                run_gemm(h);
                flush(r, gb);
                ++launches;
                break;
            }
            case K::Permute: {
                const View& x = V(r, op.in[0]);
                const View& y = V(r, op.out[0]);
                std::vector<i64> ds(op.perm.size());
                for (size_t d = 0; d < op.perm.size(); ++d) ds[d] = x.gstrides[(size_t)op.perm[d]];
                GT gx = gtarget(r, op.in[0]);
                if (gx.temp) {
                    std::vector<i64> cs(x.shape.size(), 1);
                    for (int d = (int)cs.size() - 2; d >= 0; --d) cs[(size_t)d] = cs[(size_t)d + 1] * x.shape[(size_t)d + 1];
                    for (size_t d = 0; d < op.perm.size(); ++d) ds[d] = cs[(size_t)op.perm[d]];
                }
                sbk::strided_copy(gp(r, op.out[0]), cdt, y.gstrides.data(), gx.p, cdt, ds.data(), y.shape.data(),
                                  (int)y.shape.size(), true, stream);
                flush(r, gx);
                break;
            }
            case K::Copy: {
                const View& x = V(r, op.in[0]);
                const View& y = V(r, op.out[0]);
                GT gx = gtarget(r, op.in[0]);
                std::vector<i64> ds = x.gstrides;
                if (gx.temp) ds = y.gstrides;
                sbk::strided_copy(gp(r, op.out[0]), cdt, y.gstrides.data(), gx.p, cdt, ds.data(), y.shape.data(),
                                  (int)y.shape.size(), true, stream);
                flush(r, gx);
                break;
            }
            case K::Concat: {
                const View& y = V(r, op.out[0]);
                i64 offset = 0;
                for (int v : op.in) {
                    const View& x = V(r, v);
                    const char* src = gp(r, op.out[0]) + (size_t)(offset * y.gstrides[(size_t)op.axis]) * sbk::dt_bytes(cdt);
                    GT gx = gtarget(r, v);
                    std::vector<i64> ds = x.gstrides;
                    if (gx.temp) {
                        ds.assign(x.shape.size(), 1);
                        for (int d = (int)ds.size() - 2; d >= 0; --d) ds[(size_t)d] = ds[(size_t)d + 1] * x.shape[(size_t)d + 1];
                    }
                    sbk::strided_copy(src, cdt, y.gstrides.data(), gx.p, cdt, ds.data(), x.shape.data(), (int)x.shape.size(),
                                      true, stream);
                    flush(r, gx);
                    offset += x.shape[(size_t)op.axis];
                }
                break;
            }
            case K::ReduceSum: {
                const View& x = V(r, op.in[0]);
                GT gx = gtarget(r, op.in[0]);
                if (op.reduce_all) {
                    sbk::add_scalar(gx.p, cdt, x.numel(), 0.f, gp(r, op.out[0]), stream);
                } else {
                    i64 outer, n, inner;
                    axis_split(x, op.axis, outer, n, inner);
                    sbk::broadcast_axis_acc(gp(r, op.out[0]), gx.p, cdt, outer, n, inner, stream);
                }
                flush(r, gx);
                break;
            }
            case K::AllReduce:
                if (op.allreduce) accumulate_view(r, op.out[0], op.in[0], !OW(op.in[0]));
                --launches;
                break;
            case K::AllGather: {
                // each rank keeps its own slice of its gradient (executor.cpp:1234-1244)
                const View& x = V(r, op.in[0]);
                i64 n = x.numel(), inner = 1;
                for (size_t d = (size_t)op.axis; d < x.shape.size(); ++d) inner *= x.shape[d];
                i64 outer = n / inner;
                GT gx = gtarget(r, op.in[0]);
                i64 shape[2] = {outer, inner}, ss[2] = {world * inner, 1}, ds[2] = {inner, 1};
                sbk::strided_copy(gp(r, op.out[0]) + (size_t)(r.P.rank * inner) * sbk::dt_bytes(cdt), cdt, ss, gx.p, cdt, ds,
                                  shape, 2, true, stream);
                flush(r, gx);
                break;
            }
            case K::Embedding: {
                const View& ids = V(r, op.in[0]);
                const View& w = V(r, op.in[1]);
                sbk::embedding_bwd((const double*)fp(r, op.in[0]), ids.numel(), gp(r, op.out[0]), cdt, w.shape[1],
                                   op.full_rows, op.row0, w.shape[0], (float*)gp(r, op.in[1]), r.ws, stream);
                break;
            }
            case K::FlashAttn: {
                sbk::Attn a = attn_args(r, op);
                a.acc_mask = (OW(op.in[0]) ? 0 : 1) | (OW(op.in[1]) ? 0 : 2) | (OW(op.in[2]) ? 0 : 4);
                i64 rows, cols, lq, lk, lv;
                V(r, op.in[0]).rowwise(rows, cols, lq, true);
                V(r, op.in[1]).rowwise(rows, cols, lk, true);
                V(r, op.in[2]).rowwise(rows, cols, lv, true);
                sbk::attn_bwd(a, gp(r, op.out[0]), a.ld_o, gp(r, op.in[0]), gp(r, op.in[1]), gp(r, op.in[2]), lq, lk, lv,
                              r.ws, stream);
                break;
            }
            default: throw Error(std::string("internal: no backward launcher for ") + k_str(op.k));
        }
    }

    // ----------------------------------------------------------- steps
    // Dropout keep bits of every attention op are a pure function of (seed,
    // node seed, index): they are generated on a low-priority side stream at the
    // start of the forward, overlapping the GEMMs (whose integer pipes idle),
    // and each attention op waits only for its own mask.
    cudaStream_t mstream = nullptr;
    cudaEvent_t fork_ev = nullptr;
    std::vector<cudaEvent_t> mask_ev;  // per forward op index (null when none)

    void init_mask_stream() {
        const Plan& P = ranks[0].P;
        mask_ev.assign(P.fwd.size(), nullptr);
        bool any = false;
        for (size_t i = 0; i < P.fwd.size(); ++i)
            if ((P.fwd[i].k == K::FlashAttn || P.fwd[i].k == K::FusedLinearResLN) && P.fwd[i].dropout) {
                CK(cudaEventCreateWithFlags(&mask_ev[i], cudaEventDisableTiming));
                any = true;
            }
        if (!any) return;
        bwd_ev.assign(P.fwd.size(), nullptr);
        for (size_t i = 0; i < P.fwd.size(); ++i)
            if (mask_ev[i]) CK(cudaEventCreateWithFlags(&bwd_ev[i], cudaEventDisableTiming));
        if (const char* e = getenv("SB_MASK_PHASE")) {
            regen_bwd = std::string(e) == "bwd";  // anything else: "fwd" or "inline"
            mask_inline = std::string(e) == "inline";
        }
        int lo, hi;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&mstream, cudaStreamNonBlocking, lo));  // lo = least priority
        CK(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
    }

    // Keep bits depend only on (executor seed, node seed, index) (rng.hpp,
    // executor.cpp:788-806), so every forward of this executor reads the same bits.
    // They are regenerated every step on a low-priority side stream (small
    // co-residing blocks, kernels/elementwise.cu). Placement (SB_MASK_PHASE):
    //   "fwd" (default): at the start of every forward, layer by layer ahead of
    //     the readers (each reader waits on mask_ev[i] only);
    //   "bwd": all masks before the first forward, then each step regenerates
    //     mask i right after its last reader (op i's backward);
    //   "inline": on the executor stream right before each reader.
    // The three measure within 2% of each other at C3: the hashing is integer-ALU
    // bound and costs its full duration wherever it runs.
    bool masks_valid = false;
    bool regen_bwd = false;  // default "fwd" placement (measured best of fwd / bwd / inline)
    bool mask_inline = false;  // "inline": on the executor stream right before each reader (no overlap)
    std::vector<cudaEvent_t> bwd_ev;  // per forward op index: its backward was enqueued
    std::vector<char> ev_real;        // mask_ev[i] last recorded outside a graph capture (waitable)

    bool capturing() {
        cudaStreamCaptureStatus st;
        CK(cudaStreamIsCapturing(stream, &st));
        return st != cudaStreamCaptureStatusNone;
    }

    void gen_mask(size_t i, cudaStream_t ms = nullptr) {
        const bool side = ms == nullptr;
        if (side) ms = mstream;
        for (auto& r : ranks) {
            const Op& op = r.P.fwd[i];
            if (op.k == K::FusedLinearResLN) {
                const View& y = V(r, op.out[0]);
                sbk::dropout_mask((uint32_t*)fp(r, op.out[5]), rows_of(y) * cols_of(y), op.s1, op.thr, ms);
                continue;
            }
            sbk::Attn a = attn_args(r, op);
            if (a.S % 128 == 0 && a.keys() % 128 == 0)
                sbk::dropout_mask_dual((uint32_t*)fp(r, op.out[2]), a.B * a.nh, a.S, op.s1, op.thr, ms, a.keys());
            else
                sbk::dropout_mask((uint32_t*)fp(r, op.out[2]), a.B * a.nh * a.S * a.keys(), op.s1, op.thr, ms);
        }
        if (!side) return;
        CK(cudaEventRecord(mask_ev[i], mstream));
        if (ev_real.size() != mask_ev.size()) ev_real.assign(mask_ev.size(), 0);
        ev_real[i] = !capturing();
    }

    void launch_masks() {
        if (!mstream) return;
        CK(cudaEventRecord(fork_ev, stream));
        CK(cudaStreamWaitEvent(mstream, fork_ev, 0));
        for (size_t i = 0; i < mask_ev.size(); ++i)
            if (mask_ev[i]) gen_mask(i);
        masks_valid = true;
    }

    void run_forward() {
        if (nan_guard) nan_reset();
        run_forward_ops();
        if (nan_guard && !capturing()) nan_report();
    }
    void run_forward_ops() {
        if (mask_inline) {
            for (size_t i = 0; i < ranks[0].P.fwd.size(); ++i) {
                if (mask_ev.size() > i && mask_ev[i]) gen_mask(i, stream);
                fwd_op((int)i);
            }
            ran_forward = true;
            return;
        }
        if (!regen_bwd || !masks_valid) launch_masks();
        const bool cap = capturing();
        cudaEvent_t last = nullptr;
        for (size_t i = 0; i < ranks[0].P.fwd.size(); ++i) {
            // (in bwd placement inside a graph capture the masks were made before the
            // capture or by the previous replay's backward, which the stream order covers)
            const bool has = mask_ev.size() > i && mask_ev[i];
            const bool wait = has && (regen_bwd ? (!cap && ev_real.size() > i && ev_real[i]) : true);
            if (wait) {
                CK(cudaStreamWaitEvent(stream, mask_ev[i], 0));
                last = mask_ev[i];
            }
            fwd_op((int)i);
        }
        if (last && !regen_bwd) CK(cudaStreamWaitEvent(stream, last, 0));  // join (graph capture needs it)
        ran_forward = true;
    }

    void run_backward() {
        for (auto& r : ranks) {
            // zero only what is read/accumulated before being fully written (analyze_writes)
            for (auto& [off, bytes] : zero_ranges(r)) CK(cudaMemsetAsync(r.base + off, 0, bytes, stream));
            // loss = sum of outputs: seed ones (executor.cpp:355-362)
            for (size_t k = 0; k < r.P.outputs.size(); ++k) {
                const int v = r.P.outputs[k];
                if (!V(r, v).g_contiguous()) throw Error("internal: strided model output gradient");
                const bool ow = seed_ow.count(v) && seed_ow[v];
                if (k < out_seed.size() && out_seed[k].first) {  // seeded by the caller (pipeline stage)
                    const i64 n = V(r, v).numel(), one = 1;
                    sbk::strided_copy(out_seed[k].first, out_seed[k].second, &one, gp(r, v), gdt(r, v), &one, &n, 1, !ow,
                                      stream);
                } else if (ow) sbk::fill(gp(r, v), gdt(r, v), V(r, v).numel(), 1.f, stream);
                else sbk::add_scalar(gp(r, v), gdt(r, v), V(r, v).numel(), 1.f, nullptr, stream);
                ++launches;
            }
        }
        const bool cap = capturing();
        cudaEvent_t last = nullptr;
        for (size_t si = 0; si < bsteps.size(); ++si) {
            const Step& s = bsteps[si];
            if (s.kind != 0) wside_join();  // a region's recompute / gradient scratch reuses memory
            if (s.kind == 2) {
                if (region_zero[(size_t)s.idx])
                    for (auto& r : ranks)
                        CK(cudaMemsetAsync(r.scratch_grad, 0, r.region_grad_span[(size_t)s.idx].second, stream));
            } else if (s.kind == 1) {
                fwd_op(s.idx, true);
            } else {
                cur_ow = &step_ow[si];
                bwd_op(s.idx);
                cur_ow = nullptr;
                const size_t i = (size_t)s.idx;
                if (regen_bwd && !mask_inline && masks_valid && mstream && mask_ev.size() > i && mask_ev[i]) {
                    // last reader of mask i done: regenerate it for the next step
                    CK(cudaEventRecord(bwd_ev[i], stream));
                    CK(cudaStreamWaitEvent(mstream, bwd_ev[i], 0));
                    gen_mask(i);
                    last = mask_ev[i];
                }
            }
        }
        wside_join();
        wfork_next = 0;
        if (cap && last) CK(cudaStreamWaitEvent(stream, last, 0));  // join the side stream into the graph
    }

    // merged [offset, bytes) ranges of the persistent gradient storages to zero
    std::vector<std::pair<size_t, size_t>> zero_ranges(RankCtx& r) {
        std::vector<std::pair<size_t, size_t>> v;
        for (int g : zero_gst) {
            if (!r.gptr[(size_t)g]) continue;
            size_t off = (size_t)(r.gptr[(size_t)g] - r.base);
            size_t bytes = (size_t)r.P.st[(size_t)g].numel * (size_t)sbk::dt_bytes(r.P.st[(size_t)g].gdt);
            v.push_back({off, (bytes + 255) / 256 * 256});
        }
        std::sort(v.begin(), v.end());
        std::vector<std::pair<size_t, size_t>> m;
        for (auto& x : v) {
            if (!m.empty() && m.back().first + m.back().second >= x.first)
                m.back().second = std::max(m.back().second, x.first + x.second - m.back().first);
            else
                m.push_back(x);
        }
        return m;
    }

    // ---------------------------------------------------------- profile
    std::vector<size_t> prof_open;
    void prof_begin(const std::string& name) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, stream);
        prof_open.push_back(prof.size());
        prof.push_back({name, {a, b}});
    }
    void prof_end() {
        cudaEventRecord(prof[prof_open.back()].second.second, stream);
        prof_open.pop_back();
    }
};

// ====================================================================== API
Executor::Executor(const Module& root, bool train, u64 seed, int world, DT compute, const CommConfig& comm, bool fused)
    : impl_(std::make_unique<ExecutorImpl>(root, train, seed, world, compute, comm, fused)) {}
Executor::~Executor() = default;
void Executor::set_nan_guard(bool on) {
    if (on) impl_->nan_alloc();
    impl_->nan_guard = on;
}

void Executor::upload_inputs(const std::vector<HostTensor>& inputs) {
    auto& I = *impl_;
    for (auto& r : I.ranks) {
        if (inputs.size() != r.P.inputs.size())
            throw Error("model expects " + std::to_string(r.P.inputs.size()) + " inputs, got " + std::to_string(inputs.size()));
        for (size_t k = 0; k < inputs.size(); ++k) {
            const View& v = r.P.views[(size_t)r.P.inputs[k]];
            if ((i64)inputs[k].data.size() != v.numel())
                throw Error("input " + std::to_string(k) + " has " + std::to_string(inputs[k].data.size()) +
                            " elements, expected " + std::to_string(v.numel()));
            CK(cudaMemcpyAsync(I.fp(r, r.P.inputs[k]), inputs[k].data.data(), inputs[k].data.size() * 8,
                               cudaMemcpyHostToDevice, I.stream));
        }
    }
}
void Executor::upload_inputs_raw(const double* const* inputs, int n) {
    auto& I = *impl_;
    for (auto& r : I.ranks) {
        if (n != (int)r.P.inputs.size())
            throw Error("model expects " + std::to_string(r.P.inputs.size()) + " inputs, got " + std::to_string(n));
        for (int k = 0; k < n; ++k) {
            const View& v = r.P.views[(size_t)r.P.inputs[(size_t)k]];
            CK(cudaMemcpyAsync(I.fp(r, r.P.inputs[(size_t)k]), inputs[k], (size_t)v.numel() * 8, cudaMemcpyHostToDevice,
                               I.stream));
        }
    }
}
void Executor::forward_uploaded() {
    impl_->collectives = 0;
    run_forward();
    synchronize();
}
void Executor::set_inputs_device(int idx, const void* dptr) {
    auto& I = *impl_;
    for (auto& r : I.ranks) {
        const View& v = r.P.views[(size_t)r.P.inputs[(size_t)idx]];
        CK(cudaMemcpyAsync(I.fp(r, r.P.inputs[(size_t)idx]), dptr, (size_t)v.numel() * 8, cudaMemcpyDeviceToDevice, I.stream));
    }
}
void* Executor::input_device_ptr(int idx) const {
    auto& I = *impl_;
    return I.fp(I.ranks[0], I.ranks[0].P.inputs[(size_t)idx]);
}

std::vector<HostTensor> Executor::forward(const std::vector<HostTensor>& inputs) {
    upload_inputs(inputs);
    impl_->collectives = 0;
    run_forward();
    synchronize();
    return outputs_of_rank(impl_->comm.nccl ? impl_->comm.rank : 0);
}
void Executor::run_forward() { impl_->run_forward(); }
void Executor::run_backward() {
    if (!impl_->ran_forward) throw Error("backward requires a completed forward run");
    impl_->run_backward();
}
void Executor::synchronize() { CK(cudaStreamSynchronize(impl_->stream)); }
void* Executor::stream() const { return impl_->stream; }

static HostTensor download(ExecutorImpl& I, RankCtx& r, int v, bool grad) {
    const View& vw = r.P.views[(size_t)v];
    TensorSpec s;
    s.shape = vw.shape;
    s.dtype = vw.rdt;
    HostTensor t(s);
    i64 n = vw.numel();
    DT dt = grad ? I.gdt(r, v) : I.fdt(r, v);
    const auto& strides = grad ? vw.gstrides : vw.strides;
    char* src = grad ? I.gp(r, v) : I.fp(r, v);
    double* d = nullptr;
    CK(cudaMalloc(&d, (size_t)std::max<i64>(n, 1) * 8));
    std::vector<i64> cs(vw.shape.size(), 1);
    for (int k = (int)cs.size() - 2; k >= 0; --k) cs[(size_t)k] = cs[(size_t)k + 1] * vw.shape[(size_t)k + 1];
    if (vw.shape.empty())
        sbk::cast(src, dt, d, sbk::F64, 1, I.stream);
    else
        sbk::strided_copy(src, dt, strides.data(), d, sbk::F64, cs.data(), vw.shape.data(), (int)vw.shape.size(), false,
                          I.stream);
    CK(cudaMemcpyAsync(t.data.data(), d, (size_t)n * 8, cudaMemcpyDeviceToHost, I.stream));
    CK(cudaStreamSynchronize(I.stream));
    CK(cudaFree(d));
    return t;
}

static RankCtx& rank_ctx(ExecutorImpl& I, int rank) {
    if (I.comm.nccl) {
        if (rank != I.comm.rank) throw Error("rank " + std::to_string(rank) + " lives in another process");
        return I.ranks[0];
    }
    if (rank < 0 || rank >= I.world) throw Error("rank out of range");
    return I.ranks[(size_t)rank];
}

std::vector<HostTensor> Executor::outputs_of_rank(int rank) const {
    auto& I = *impl_;
    RankCtx& r = rank_ctx(I, rank);
    std::vector<HostTensor> out;
    for (int v : r.P.outputs) out.push_back(download(I, r, v, false));
    return out;
}

std::vector<GradMap> Executor::backward_all_ranks() {
    auto& I = *impl_;
    run_backward();
    synchronize();
    std::vector<GradMap> maps;
    for (auto& r : I.ranks) {
        GradMap m;
        for (auto& [name, v] : r.P.params) m.params[name] = download(I, r, v, true);
        for (int v : r.P.inputs) m.inputs.push_back(download(I, r, v, true));
        maps.push_back(std::move(m));
    }
    return maps;
}
GradMap Executor::backward() { return backward_all_ranks()[0]; }
i64 Executor::ledger_bytes() const { return impl_->ranks[0].P.ledger_bytes; }
i64 Executor::collective_invocations() const { return impl_->collectives; }

// ---- pipeline-stage hooks (csrc/host/pipeline_exec.cpp) ----
void Executor::set_accumulate_param_grads(bool on) {
    auto& I = *impl_;
    if (I.accum_params == on) return;
    if (I.gexec) throw Error("set_accumulate_param_grads: the step graph is already captured");
    I.accum_params = on;
    I.analyze_writes();
}
void Executor::zero_param_grads() {
    auto& I = *impl_;
    for (auto& r : I.ranks) {
        std::set<int> done;
        for (auto& pv : r.P.params) {
            const int g = r.P.views[(size_t)pv.second].gst;
            if (!done.insert(g).second || !r.gptr[(size_t)g]) continue;
            CK(cudaMemsetAsync(r.gptr[(size_t)g], 0, (size_t)r.P.st[(size_t)g].numel * sbk::dt_bytes(r.P.st[(size_t)g].gdt),
                               I.stream));
        }
    }
}
void Executor::set_output_grad_seed(int idx, const void* dptr, DT dt) {
    auto& I = *impl_;
    if (idx < 0 || idx >= (int)I.ranks[0].P.outputs.size()) throw Error("set_output_grad_seed: output index out of range");
    // (lockstep ranks: every rank's output is seeded from the same buffer — stage-boundary
    // values are replicated across tensor-parallel ranks)
    if (I.out_seed.size() < I.ranks[0].P.outputs.size()) I.out_seed.resize(I.ranks[0].P.outputs.size(), {nullptr, sbk::F32});
    I.out_seed[(size_t)idx] = {dptr, dt};
}
DeviceTensor Executor::output_device(int idx) const {
    auto& I = *impl_;
    RankCtx& r = I.ranks[0];
    if (idx < 0 || idx >= (int)r.P.outputs.size()) throw Error("output index out of range");
    const int v = r.P.outputs[(size_t)idx];
    if (!I.V(r, v).contiguous()) throw Error("internal: strided output");
    return {I.fp(r, v), I.fdt(r, v), I.V(r, v).numel(), I.V(r, v).shape};
}
DeviceTensor Executor::input_grad_device(int idx) const {
    auto& I = *impl_;
    RankCtx& r = I.ranks[0];
    if (idx < 0 || idx >= (int)r.P.inputs.size()) throw Error("input index out of range");
    const int v = r.P.inputs[(size_t)idx];
    if (!I.V(r, v).g_contiguous()) throw Error("internal: strided input gradient");
    return {I.gp(r, v), I.gdt(r, v), I.V(r, v).numel(), I.V(r, v).shape};
}
void Executor::set_input_from_device(int idx, const void* src, DT dt) {
    auto& I = *impl_;
    for (auto& r : I.ranks) {
        const int v = r.P.inputs[(size_t)idx];
        const i64 n = I.V(r, v).numel(), one = 1;
        sbk::strided_copy(src, dt, &one, I.fp(r, v), I.fdt(r, v), &one, &n, 1, false, I.stream);
    }
}
std::vector<GradMap> Executor::grads_all_ranks() {
    auto& I = *impl_;
    synchronize();
    std::vector<GradMap> maps;
    for (auto& r : I.ranks) {
        GradMap m;
        for (auto& [name, v] : r.P.params) m.params[name] = download(I, r, v, true);
        for (int v : r.P.inputs) m.inputs.push_back(download(I, r, v, true));
        maps.push_back(std::move(m));
    }
    return maps;
}

void Executor::all_reduce_device(void* buf, i64 n, DT dt, void* st) {
    auto& I = *impl_;
    if (I.comm.nccl) {
        nccl().check(nccl().AllReduce(buf, buf, (size_t)n, nccl_dt(dt), ncclSum, I.ncomm,
                                          st ? (cudaStream_t)st : I.stream),
                       "ncclAllReduce");
        return;
    }
    if (I.world != 1) throw Error("all_reduce_device: a lockstep multi-rank executor has no communicator");
}

void Executor::enqueue_loss(float* dloss) {
    auto& I = *impl_;
    RankCtx& r = I.ranks[0];
    CK(cudaMemsetAsync(dloss, 0, 4, I.stream));
    for (int v : r.P.outputs) {
        const View& vw = r.P.views[(size_t)v];
        if (!vw.contiguous()) throw Error("internal: strided output");
        sbk::reduce_all(I.fp(r, v), I.fdt(r, v), vw.numel(), dloss, sbk::F32, true, I.stream);
    }
}

void Executor::capture_graph() {
    auto& I = *impl_;
    if (I.gexec) return;
    if (I.comm.nccl && I.world > 1) {
        // NCCL kernels are capturable; nothing special beyond using our stream.
    }
    if (I.regen_bwd && !I.mask_inline && !I.masks_valid && I.mstream) {  // the graph regenerates masks in its backward; prime once
        I.launch_masks();
        CK(cudaStreamSynchronize(I.mstream));
    }
    CK(cudaStreamBeginCapture(I.stream, cudaStreamCaptureModeThreadLocal));
    I.run_forward();
    I.run_backward();
    CK(cudaStreamEndCapture(I.stream, &I.graph));
    CK(cudaGraphInstantiate(&I.gexec, I.graph, 0));
}
void Executor::launch_graph() {
    auto& I = *impl_;
    if (!I.gexec) capture_graph();
    CK(cudaGraphLaunch(I.gexec, I.stream));
    if (I.nan_guard) I.nan_report();
}
int Executor::kernel_launches_per_step() const {
    // exact: the kernel nodes of the captured fwd+bwd graph
    auto& I = *impl_;
    if (!I.graph) return -1;
    size_t n = 0;
    CK(cudaGraphGetNodes(I.graph, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    CK(cudaGraphGetNodes(I.graph, nodes.data(), &n));
    int k = 0;
    for (auto nd : nodes) {
        cudaGraphNodeType t;
        CK(cudaGraphNodeGetType(nd, &t));
        k += t == cudaGraphNodeTypeKernel;
    }
    return k;
}
// End-to-end steps through the public API: every step copies its inputs from
// host memory (pinned by the caller for async DMA), runs fwd+bwd and reads the
// loss (sum of outputs) back to the host.
float Executor::time_e2e(int steps, const double* const* inputs, int n, bool use_graph, float* last_loss) {
    auto& I = *impl_;
    float* dloss = nullptr;
    float* hloss = nullptr;
    CK(cudaMalloc(&dloss, 4));
    CK(cudaMallocHost(&hloss, 4));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaStreamSynchronize(I.stream));
    CK(cudaEventRecord(a, I.stream));
    for (int i = 0; i < steps; ++i) {
        upload_inputs_raw(inputs, n);
        if (use_graph) {
            launch_graph();
        } else {
            I.run_forward();
            I.run_backward();
        }
        enqueue_loss(dloss);
        CK(cudaMemcpyAsync(hloss, dloss, 4, cudaMemcpyDeviceToHost, I.stream));
        CK(cudaStreamSynchronize(I.stream));
    }
    CK(cudaEventRecord(b, I.stream));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (last_loss) *last_loss = *hloss;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(dloss);
    cudaFreeHost(hloss);
    return ms;
}

float Executor::time_steps(int steps, bool use_graph) {
    auto& I = *impl_;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaStreamSynchronize(I.stream));
    CK(cudaEventRecord(a, I.stream));
    for (int i = 0; i < steps; ++i) {
        if (use_graph) {
            launch_graph();
        } else {
            I.run_forward();
            I.run_backward();
        }
    }
    CK(cudaEventRecord(b, I.stream));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms;
}
size_t Executor::device_bytes() const {
    size_t t = 0;
    for (auto& r : impl_->ranks) t += r.total;
    return t;
}
std::string Executor::describe() const {
    auto& I = *impl_;
    std::ostringstream o;
    const Plan& P = I.ranks[0].P;
    std::map<std::string, int> cnt;
    for (auto& op : P.fwd) cnt[k_str(op.k)]++;
    int early = 0;
    for (int e : I.early_ar) early += e >= 0;
    o << "{\"ops\": " << P.fwd.size() << ", \"regions\": " << P.regions.size() << ", \"backward_steps\": " << I.bsteps.size()
      << ", \"device_bytes\": " << device_bytes() << ", \"overlapped_backward_allreduces\": " << early
      << ", \"kinds\": {";
    bool first = true;
    for (auto& [k, c] : cnt) {
        o << (first ? "" : ", ") << "\"" << k << "\": " << c;
        first = false;
    }
    o << "}}";
    return o.str();
}

std::vector<std::pair<std::string, float>> Executor::profile_step() {
    auto& I = *impl_;
    I.profiling = true;
    I.prof.clear();
    I.gemm_flops = 0;
    // per-kind times need one stream: the side-stream weight gradients run inline here
    const bool wside = I.wside;
    I.wside = false;
    cudaEvent_t s0, s1;
    cudaEventCreate(&s0);
    cudaEventCreate(&s1);
    cudaEventRecord(s0, I.stream);
    I.run_forward();
    I.run_backward();
    cudaEventRecord(s1, I.stream);
    I.profiling = false;
    I.wside = wside;
    synchronize();
    std::map<std::string, float> acc;
    float total = 0;
    cudaEventElapsedTime(&total, s0, s1);
    cudaEventDestroy(s0);
    cudaEventDestroy(s1);
    acc["@step_ms"] = total;
    acc["@gemm_gflop"] = (float)(I.gemm_flops * 1e-9);
    for (auto& [name, ev] : I.prof) {
        float ms = 0;
        cudaEventElapsedTime(&ms, ev.first, ev.second);
        acc[name] += ms;
        cudaEventDestroy(ev.first);
        cudaEventDestroy(ev.second);
    }
    I.prof.clear();
    return {acc.begin(), acc.end()};
}

}  // namespace sb
