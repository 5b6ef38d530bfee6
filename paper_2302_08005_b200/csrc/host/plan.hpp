// Static device plan: a post-apply Module lowered once into typed device ops
// over storages/views, per rank. Replaces the reference's per-call graph
// interpreter + tape (proj/src/executor.cpp:285-1462): the tape becomes the
// forward op list, backward_record becomes the reverse list, checkpoint
// recompute becomes re-launching a region's forward ops inside backward.
#pragma once

#include <string>
#include <vector>

#include "../kernels/kernels.hpp"
#include "ir.hpp"

namespace sb {

using sbk::DT;

enum class SKind : int { Act, Param, Input, Aux };

struct Storage {
    i64 numel = 0;
    DT dt = sbk::F32;    // forward payload
    DT gdt = sbk::F32;   // gradient payload
    SKind kind = SKind::Act;
    bool has_fwd = true;   // false: grad-only storage (SyncGrad)
    bool needs_grad = false;
    int region = -1;       // checkpoint region whose scratch holds it (-1 persistent)
    std::string name;      // param path / debug
    size_t off = 0, goff = 0;  // byte offsets inside the arena (set at allocation)
    bool fwd_in_scratch = false, grad_in_scratch = false;
};

struct View {
    int st = -1;
    i64 off = 0;
    std::vector<i64> shape, strides;
    int gst = -1;
    i64 goff = 0;
    std::vector<i64> gstrides;
    Dtype rdt = Dtype::F64;  // the reference dtype (ledger accounting)
    i64 numel() const {
        i64 n = 1;
        for (i64 d : shape) n *= d;
        return n;
    }
    bool contiguous() const;
    bool g_contiguous() const;
    // rows x cols with uniform row stride `ld` (all leading dims collapsible).
    bool rowwise(i64& rows, i64& cols, i64& ld, bool grad = false) const;
};

enum class K : int {
    Cast,
    Linear,
    LayerNorm,
    Dropout,
    Add,
    Mul,
    Scale,
    Relu,
    Gelu,
    Softmax,
    Matmul,
    Permute,
    Copy,
    Concat,
    ReduceSum,
    AllReduce,
    AllGather,
    SyncGrad,
    Embedding,
    FusedLinearGelu,
    FusedLinearResLN,
    FlashAttn,
    FillOnes,
};
const char* k_str(K k);

struct Op {
    K k;
    std::vector<int> in, out;  // view ids
    int region = -1;
    std::string path;
    // attributes
    double p = 0, scale = 1, eps = 1e-5;
    u64 s1 = 0, thr = 0;  // dropout: s1 = hash_combine(hash_combine(seed, node_seed), 0xd0)
    bool dropout = false, bias_on = true, bias_grad = true, has_bias = false, qkv = false, allreduce = false;
    bool causal = false;  // FlashAttn / Softmax: attr "causal" (f2; the oracle extension oracle/causal_ext.py)
    bool affine = true;
    int axis = -1;
    std::vector<int> perm;
    i64 hd = 0, nh = 0;
    i64 full_rows = 0, row0 = 0;
    bool reduce_all = false;
    bool ids_input = false;  // SyncGrad over a non-differentiable id input (zero grad)
    // dgrad of this Linear-like op writes gelu'(pre) * (g W) straight into the
    // gradient of view `dgelu_pre` (the producing FusedLinearGelu's pre-activation)
    int dgelu_pre = -1;
    bool dgelu_fused = false;  // FusedLinearGelu whose GeLU backward was folded into its consumer
    // Linear -> ReLU folded (lower.cpp fuse_linear_relu): act = 1 on the Linear (its out[0] is
    // the ReLU's output, applied in the GEMM epilogue); drelu on the sole consumer of that
    // output, whose dgrad epilogue multiplies by (x > 0) — x its own input — so the gradient
    // it leaves is the one at the Linear's pre-activation
    int act = 0;
    bool drelu = false;
    // FusedLinearResLN whose pre-LN sum (out[2]) is also read by other ops (the residual
    // stream of a pre-LN block): its backward adds that sum's gradient (lower.cpp
    // fuse_residual_stream)
    bool sum_ext = false;
};

struct Region {
    int first_op = -1, last_op = -1;  // [first, last] inclusive in fwd
};

struct Plan {
    int rank = 0, world = 1;
    DT cdt = sbk::F32;
    bool train = true;
    std::vector<Storage> st;
    std::vector<View> views;
    std::vector<Op> fwd;
    std::vector<Region> regions;
    std::vector<int> inputs;                        // input views (f64)
    std::vector<int> outputs;                       // output views
    std::vector<std::pair<std::string, int>> params;  // dotted path -> view
    std::vector<std::pair<std::string, HostTensor>> param_init;  // host values (rank-local)
    i64 ledger_bytes = 0;
    i64 collectives_fwd = 0;  // forward all_reduce/all_gather count
    std::string structure() const;  // op kinds, for cross-rank lockstep check
};

struct LowerOptions {
    int rank = 0, world = 1;
    bool train = true;
    u64 seed = 0;
    DT cdt = sbk::F32;
    bool fused_kernels = true;  // lower recognised fused regions / EfficientAttention to fused kernels
    // NCCL executor at world 1: keep the one-rank collectives (all_reduce, SyncGrad) as real
    // NCCL calls so the communicator, the comm stream and graph capture of NCCL run
    bool keep_collectives = false;
    bool collect() const { return world > 1 || keep_collectives; }
};

Plan lower(const Module& root, const LowerOptions& o);

}  // namespace sb
