// Host-side launchers for the sm_100a kernels. Plain pointers, sizes, and an
// explicit stream; enqueue only (no implicit synchronisation). These are what
// the C-ABI (include/slapo_b200.h) exports one level below the executor.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace sbk {

using i64 = std::int64_t;
using u64 = std::uint64_t;

enum DT : int { F32 = 0, BF16 = 1, F64 = 2 };
inline int dt_bytes(DT d) { return d == F32 ? 4 : d == BF16 ? 2 : 8; }

// ------------------------------------------------------------------ GEMM
// C[b](m,n) = alpha * sum_k A[b](m,k) B[b](k,n)  (+ bias[n]) (+ C if accumulate)
// with arbitrary element strides; fp32 accumulation. epilogue: 0 none,
// 1 gelu (then `aux`, if set, receives the pre-activation in C's dtype),
// 2 dgelu: C (+)= gelu'(aux) * (A B) — a dgrad written as the gradient of a GeLU's input.
struct Gemm {
    const void* A = nullptr;
    DT ta = F32;
    i64 sAb = 0, sAm = 0, sAk = 0;
    const void* B = nullptr;
    DT tb = F32;
    i64 sBb = 0, sBk = 0, sBn = 0;
    void* C = nullptr;
    DT tc = F32;
    i64 sCb = 0, sCm = 0, sCn = 0;
    i64 batch = 1, M = 0, N = 0, K = 0;
    float alpha = 1.f;
    bool accumulate = false;
    const void* bias = nullptr;
    DT tbias = F32;
    int epilogue = 0;
    void* aux = nullptr;  // pre-activation (same layout as C) when epilogue == gelu
    void* ws = nullptr;   // scratch for deterministic split-K partials (optional)
    size_t ws_bytes = 0;
    // optional: fp32 column sums of the output, one row per 32 output rows ([M/32][N]) —
    // produced by the 2-SM kernel's epilogue when it can (gemm_last_colsum() reports it)
    float* colsum = nullptr;
};
void gemm(const Gemm& g, cudaStream_t s);
// whether the last gemm() call wrote g.colsum
bool gemm_last_colsum();
// Which engine the last gemm() call used: 0 SIMT, 1 tcgen05 1-SM, 2 tcgen05 2-SM (tests/bench).
int gemm_last_engine();
// engine cap: 0 best available, 1 at most the 1-SM tcgen05 kernel, 2 SIMT only
void gemm_set_engine(int e);
// 2-SM kernel cluster tile N: 0 default (256), 128 or 256 forced
void gemm2_set_tile_n(int bn);
// SMs the persistent 2-SM GEMM leaves free (for an NCCL collective running
// concurrently on another stream); 0 = use every SM.
void gemm_set_sm_reserve(int n);
// Force the SIMT engine (tests compare the tcgen05 kernel against it).
void gemm_force_simt(bool on);
// workspace the tcgen05 split-K path may use for an (M x N) fp32 output
inline size_t gemm_splitk_workspace(i64 M, i64 N) {
    size_t w = (size_t)16 * M * N * 4, cap = (size_t)48 << 20;
    return w < cap ? w : cap;
}

// ----------------------------------------------------------- elementwise
void fill(void* x, DT t, i64 n, float v, cudaStream_t s);
void cast(const void* x, DT tx, void* y, DT ty, i64 n, cudaStream_t s);
// y (+)= a ⊙/+ b with scalar broadcast flags (a_n / b_n == 1 -> scalar)
void binary(int op /*0 add 1 mul*/, const void* a, i64 a_n, const void* b, i64 b_n, void* y, DT t, i64 n,
            cudaStream_t s);
// y = f(x): 0 scale(c), 1 relu, 2 gelu
void unary(int op, const void* x, void* y, DT t, i64 n, float c, cudaStream_t s);
// gx += f'(x) * g  (relu: g*(x>0); gelu: g*gelu'(x); scale: c*g)
void unary_bwd(int op, const void* x, const void* g, void* gx, DT t, DT tg, i64 n, float c, cudaStream_t s);
// y += alpha * x (dtype-converting accumulate); if `scalar_out`, y[0] += alpha*sum(x)
void accumulate(const void* x, DT tx, void* y, DT ty, i64 n, float alpha, cudaStream_t s);
void reduce_all(const void* x, DT tx, i64 n, void* y, DT ty, bool accumulate, cudaStream_t s);
// y[o,i] (+)= sum_a x[o,a,i]   and its backward gx[o,a,i] += g[o,i]
void reduce_axis(const void* x, void* y, DT t, i64 outer, i64 adim, i64 inner, bool accumulate, cudaStream_t s);
void broadcast_axis_acc(const void* g, void* gx, DT t, i64 outer, i64 adim, i64 inner, cudaStream_t s);
// flag[0] += number of NaNs in x (the executor's NaN guard, executor.cpp:308-318)
void count_nan(const void* x, DT t, i64 n, int* flag, cudaStream_t s);
// one-time device workspace for deterministic reductions (call outside graph capture)
void init_workspace();
// x[i] += v (x[i] += g[0] when g != null)
void add_scalar(void* x, DT t, i64 n, float v, const void* g, cudaStream_t s);
// mul backward: ga += g * b (b scalar if b_n==1), reduced to scalar when a is scalar
void mul_bwd(const void* g, DT tg, const void* other, i64 other_n, void* ga, DT tga, i64 ga_n, i64 n, cudaStream_t s);

// --------------------------------------------------- counter-RNG dropout
// keep_i = (splitmix64(hash_combine(s1, base + i)) >> 11) >= thr, where
// s1 = hash_combine(stream_seed, 0xd0) (host-precomputed);
// y = keep ? x*scale : 0;  also used for backward (g -> gx, accumulate).
void dropout(const void* x, void* y, DT t, i64 n, u64 s1, u64 thr, float scale, bool accumulate, cudaStream_t s);
// Packed keep mask (bit i of word i/32) for tests / the attention kernels.
void dropout_mask(uint32_t* bits, i64 n, u64 s1, u64 thr, cudaStream_t s);
// attention keep bits, both layouts: bits[0, W) natural (element ((bh*S+i)*S+j)
// at bit e%32 of word e/32), bits[W, 2W) transposed (element ((bh*S+j)*S+i)),
// W = BH*S*S/32; S % 128 == 0
// natural (B*nh, S, Sk) + transposed (B*nh, Sk, S) keep bits; Sk = 0: S
void dropout_mask_dual(uint32_t* bits, i64 BH, i64 S, u64 s1, u64 thr, cudaStream_t s, i64 Sk = 0);
void set_mask_blocks(int n);  // experiments: persistent grid size of the keep-bit kernel (0 = full grid)

// --------------------------------------------------------- strided copy
// dst[idx] (+)= src[idx] over a rank<=8 index space with per-tensor strides.
void strided_copy(const void* src, DT ts, const i64* src_strides, void* dst, DT td, const i64* dst_strides,
                  const i64* shape, int rank, bool accumulate, cudaStream_t s);

// ------------------------------------------------------ norms / softmax
// Row-wise over (outer, n, inner) layout: element (o, j, i) at o*n*inner + j*inner + i.
// causal_nq > 0 (rows layout only): row r is query q = r % causal_nq and covers keys
// [0, min(n, q + 1 + n - causal_nq)); the rest are written as 0 (oracle/causal_ext.py)
void softmax_fwd(const void* x, void* y, DT t, i64 outer, i64 n, i64 inner, cudaStream_t s, i64 causal_nq = 0);
void softmax_bwd(const void* y, const void* g, void* gx, DT t, DT tg, i64 outer, i64 n, i64 inner, cudaStream_t s);
// LayerNorm over the last dim: y = gamma*(x-mu)*rstd + beta; gamma/beta may be null.
void layernorm_fwd(const void* x, const void* gamma, const void* beta, DT tp, void* y, float* mean, float* rstd,
                   DT t, i64 rows, i64 n, float eps, cudaStream_t s);
// gx += ...; dgamma/dbeta (+)= column sums (fp32) when non-null.
void layernorm_bwd(const void* x, const float* mean, const float* rstd, const void* gamma, DT tp, const void* g,
                   DT tg, void* gx, float* dgamma, float* dbeta, DT t, i64 rows, i64 n, float* workspace,
                   cudaStream_t s, bool gx_acc = true, bool col_acc = true);
size_t layernorm_bwd_workspace(i64 rows, i64 n);

// Fused bias + dropout + residual + LayerNorm (the .fuse'd BERT output block):
//   sum = dropout(partial + bias) + residual ; y = LN(sum)
// `sum` is saved for backward. dropout disabled when thr == 0. `keep`: the
// precomputed keep bits (dropout_mask of the same stream, bit row*n+col) or null
// to hash in place.
void bias_dropout_residual_ln_fwd(const void* partial, const void* bias, const void* residual, const void* gamma,
                                  const void* beta, DT tp, void* sum, void* y, float* mean, float* rstd, DT t,
                                  i64 rows, i64 n, float eps, u64 s1, u64 thr, float dscale, cudaStream_t s,
                                  const uint32_t* keep = nullptr);
// g_sum = LNbwd(g) (+ g_sum_extra: the sum's gradient from other consumers); g_res += g_sum;
// g_partial (+)= dropout_bwd(g_sum); dbias/dgamma/dbeta (+)=
void bias_dropout_residual_ln_bwd(const void* sum, const float* mean, const float* rstd, const void* gamma, DT tp,
                                  const void* g, void* g_res, void* g_partial, bool g_partial_accumulate,
                                  float* dbias, float* dgamma, float* dbeta, DT t, i64 rows, i64 n, u64 s1,
                                  u64 thr, float dscale, float* workspace, cudaStream_t s, bool gres_acc = true,
                                  bool col_acc = true, const uint32_t* keep = nullptr, const void* g_sum_extra = nullptr);
size_t bdrln_bwd_workspace(i64 rows, i64 n);

// column sums of g (rows x cols) into fp32 db (+=)
// db (+)= the fixed-order sum of `chunks` rows of fp32 column partials ([chunks][cols])
void bias_grad_partials(const float* partials, i64 chunks, i64 cols, float* db, cudaStream_t s, bool accum);
void bias_grad(const void* g, DT tg, i64 ld, i64 rows, i64 cols, float* db, float* workspace, cudaStream_t s,
               bool acc = true);
size_t bias_grad_workspace(i64 rows, i64 cols);
// standalone bias + GeLU (the product folds it into the GEMM epilogue): pre = x + b, y = gelu(pre);
// backward gx = g * gelu'(pre), db = column sums of gx (overwritten; workspace bias_grad_workspace)
void bias_gelu_fwd(const void* x, const void* b, void* y, void* pre, DT t, i64 rows, i64 n, cudaStream_t s);
void bias_gelu_bwd(const void* pre, const void* g, void* gx, float* db, DT t, i64 rows, i64 n, float* ws, cudaStream_t s);

// ---------------------------------------------------------- embedding
void embedding_fwd(const double* ids, i64 n_ids, const void* table, DT t, i64 dim, i64 full_rows, i64 row0,
                   i64 local_rows, void* out, cudaStream_t s);
// Deterministic scatter-add: sort (row, position) pairs, then each row's
// positions are summed in ascending order by one owner (no float atomics).
void embedding_bwd(const double* ids, i64 n_ids, const void* g, DT tg, i64 dim, i64 full_rows, i64 row0,
                   i64 local_rows, float* gtable, void* workspace, cudaStream_t s);
size_t embedding_bwd_workspace(i64 n_ids, i64 dim);

// ---------------------------------------------- simulated collectives
// dst_r = sum_{r'} src_{r'} in rank-ascending order (fp32 accumulation), for
// ranks that live on one device (the reference's lockstep simulator).
void sum_ranks(const void* const* srcs, void* const* dsts, int R, DT t, i64 n, bool accumulate, cudaStream_t s);

// --------------------------------------------------- flash attention
// q/k/v/o addressed as [b, s, h*hd + d] with row strides ld_q/ld_k/ld_v/ld_o
// (so a FusedQKV output is consumed in place). lse: (B, nh, S) fp32.
// Dropout on probabilities with the reference's flat index
// ((b*nh + h)*S + i)*S + j when thr != 0.
struct Attn {
    const void* q;
    const void* k;
    const void* v;
    void* o;
    i64 ld_q, ld_k, ld_v, ld_o;
    float* lse;
    i64 B, S, nh, hd;  // S: queries per sequence
    i64 Sk = 0;        // keys per sequence (cross-attention); 0: S
#ifdef __CUDACC__
    __host__ __device__
#endif
    i64 keys() const { return Sk ? Sk : S; }
    float scale;
    u64 s1 = 0, thr = 0;
    float dscale = 1.f;
    DT t;
    const uint32_t* mask = nullptr;    // precomputed keep bits (dropout_mask); required by the tensor-core paths
    const uint32_t* mask_t = nullptr;  // transposed keep bits (dropout_mask_dual); required by the tcgen05 backward
    int acc_mask = 7;                // backward: bit0/1/2 = dq/dk/dv accumulate (else overwrite)
    int causal = 0;                  // key j > query i masked out before the softmax (
                                     // not in the reference's op set): SIMT and mma.sync engines only
};
void attn_fwd(const Attn& a, cudaStream_t s);
// 0 = best available (tcgen05 > mma.sync > SIMT), 1 = at most mma.sync, 2 = SIMT only
void attn_set_engine(int e);
int attn_last_engine(int bwd);  // engine of the last fwd/bwd call: 3 tcgen05, 2 mma.sync, 1 SIMT
// dq/dk/dv accumulate (+=) or overwrite per acc_mask, with their own row
// strides; `ws` scratch of attn_bwd_workspace() bytes.
void attn_bwd(const Attn& a, const void* dout, i64 ld_do, void* dq, void* dk, void* dv, i64 ld_dq, i64 ld_dk,
              i64 ld_dv, void* ws, cudaStream_t s);
size_t attn_bwd_workspace(i64 B, i64 S, i64 nh, i64 hd);

}  // namespace sbk
