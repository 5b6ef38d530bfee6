// LayerNorm / softmax / fused bias+dropout+residual+LayerNorm kernels.
// One warp per row, fp32 statistics, two-pass mean/variance (biased, eps
// inside the sqrt) exactly as eval_layernorm_mod / backward_layernorm_mod
// (proj/src/executor.cpp:699-740, 1158-1197) and the layernorm op (:917-937,
// 1333-1364). Column reductions (dgamma/dbeta/dbias) go through fixed per-block
// partials so results are bitwise deterministic.
#include "common.cuh"

namespace sbk {

namespace {
constexpr int kWarps = 8;           // rows in flight per block
constexpr int kRowBlocks = 296;     // fixed grid for the backward column partials
}  // namespace

// vectorised register-resident variants (norm_vec.cu); false = shape not covered
bool ln_fwd_vec(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd, DT t, i64 rows,
                i64 n, float eps, cudaStream_t s);
bool bdrln_fwd_vec(const void* partial, const void* bias, const void* res, const void* gamma, const void* beta, void* sum,
                   void* y, float* mean, float* rstd, DT t, i64 rows, i64 n, float eps, u64 s1, u64 thr, float dscale,
                   const uint32_t* keep, cudaStream_t s);
bool ln_bwd_vec(int mode, const void* x, const float* mean, const float* rstd, const void* gamma, const void* g, void* gx,
                void* gres, bool gx_acc, bool gres_acc, DT t, i64 rows, i64 n, u64 s1, u64 thr, float dscale,
                const uint32_t* keep, float* ws, int ncol, int& nblocks, cudaStream_t s, const void* gext = nullptr);
static int vec_blocks(i64 rows) { return (int)std::min<i64>(296, std::max<i64>(1, (rows + kWarps - 1) / kWarps)); }

// ------------------------------------------------------------------ softmax
template <class T>
__global__ void k_softmax_rows(const T* x, T* y, i64 rows, i64 n, i64 nq) {
    i64 row = blockIdx.x * (i64)kWarps + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const T* px = x + row * n;
    T* py = y + row * n;
    i64 lim = n;
    if (nq > 0) lim = max((i64)1, min(n, row % nq + 1 + n - nq));  // causal (oracle/causal_ext.py)
    float mx = -INFINITY;
    for (i64 i = lane; i < lim; i += 32) mx = fmaxf(mx, to_f(px[i]));
    mx = warp_max(mx);
    float s = 0.f;
    for (i64 i = lane; i < lim; i += 32) s += __expf(to_f(px[i]) - mx);
    s = warp_sum(s);
    float inv = 1.f / s;
    for (i64 i = lane; i < n; i += 32) py[i] = i < lim ? from_f<T>(__expf(to_f(px[i]) - mx) * inv) : from_f<T>(0.f);
}
template <class T>
__global__ void k_softmax_cols(const T* x, T* y, i64 outer, i64 n, i64 inner) {
    i64 total = outer * inner;
    for (i64 c = blockIdx.x * (i64)blockDim.x + threadIdx.x; c < total; c += (i64)gridDim.x * blockDim.x) {
        i64 o = c / inner, in = c % inner;
        const T* px = x + o * n * inner + in;
        T* py = y + o * n * inner + in;
        float mx = -INFINITY, s = 0.f;
        for (i64 j = 0; j < n; ++j) mx = fmaxf(mx, to_f(px[j * inner]));
        for (i64 j = 0; j < n; ++j) s += __expf(to_f(px[j * inner]) - mx);
        for (i64 j = 0; j < n; ++j) py[j * inner] = from_f<T>(__expf(to_f(px[j * inner]) - mx) / s);
    }
}
void softmax_fwd(const void* x, void* y, DT t, i64 outer, i64 n, i64 inner, cudaStream_t s, i64 causal_nq) {
    if (causal_nq > 0 && inner != 1) throw std::runtime_error("softmax_fwd: causal needs the last axis");
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        if (inner == 1)
            k_softmax_rows<T><<<(unsigned)((outer + kWarps - 1) / kWarps), 32 * kWarps, 0, s>>>((const T*)x, (T*)y, outer, n,
                                                                                               causal_nq);
        else
            k_softmax_cols<T><<<grid_for(outer * inner, 256), 256, 0, s>>>((const T*)x, (T*)y, outer, n, inner);
    });
    SBK_CHECK_LAUNCH();
}
// gx += y * (g - sum(g*y))   (executor.cpp:1313-1332)
template <class T>
__global__ void k_softmax_bwd(const T* y, const T* g, T* gx, i64 outer, i64 n, i64 inner) {
    i64 total = outer * inner;
    i64 w = blockIdx.x * (i64)kWarps + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (w >= total) return;
    i64 o = w / inner, in = w % inner;
    i64 base = o * n * inner + in;
    float dot = 0.f;
    for (i64 j = lane; j < n; j += 32) dot += to_f(g[base + j * inner]) * to_f(y[base + j * inner]);
    dot = warp_sum(dot);
    for (i64 j = lane; j < n; j += 32) {
        i64 k = base + j * inner;
        gx[k] = from_f<T>(to_f(gx[k]) + to_f(y[k]) * (to_f(g[k]) - dot));
    }
}
void softmax_bwd(const void* y, const void* g, void* gx, DT t, DT tg, i64 outer, i64 n, i64 inner, cudaStream_t s) {
    (void)tg;
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        k_softmax_bwd<T><<<(unsigned)((outer * inner + kWarps - 1) / kWarps), 32 * kWarps, 0, s>>>(
            (const T*)y, (const T*)g, (T*)gx, outer, n, inner);
    });
    SBK_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- layernorm
// Row statistics from a row that is already materialised (x or `sum`).
template <class T>
__device__ __forceinline__ void row_stats(const T* px, i64 n, int lane, float eps, float& mean, float& rstd) {
    float s = 0.f;
    for (i64 i = lane; i < n; i += 32) s += to_f(px[i]);
    mean = warp_sum(s) / (float)n;
    float v = 0.f;
    for (i64 i = lane; i < n; i += 32) {
        float d = to_f(px[i]) - mean;
        v += d * d;
    }
    rstd = rsqrtf(warp_sum(v) / (float)n + eps);
}

template <class T, class P>
__global__ void k_ln_fwd(const T* x, const P* gamma, const P* beta, T* y, float* mean, float* rstd, i64 rows, i64 n,
                         float eps) {
    i64 row = blockIdx.x * (i64)kWarps + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const T* px = x + row * n;
    float mu, rs;
    row_stats(px, n, lane, eps, mu, rs);
    for (i64 i = lane; i < n; i += 32) {
        float h = (to_f(px[i]) - mu) * rs;
        if (gamma) h = to_f(gamma[i]) * h + to_f(beta[i]);
        y[row * n + i] = from_f<T>(h);
    }
    if (lane == 0) {
        mean[row] = mu;
        rstd[row] = rs;
    }
}
void layernorm_fwd(const void* x, const void* gamma, const void* beta, DT tp, void* y, float* mean, float* rstd, DT t,
                   i64 rows, i64 n, float eps, cudaStream_t s) {
    (void)tp;
    if (ln_fwd_vec(x, gamma, beta, y, mean, rstd, t, rows, n, eps, s)) {
        SBK_CHECK_LAUNCH();
        return;
    }
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        k_ln_fwd<T, T><<<(unsigned)((rows + kWarps - 1) / kWarps), 32 * kWarps, 0, s>>>(
            (const T*)x, (const T*)gamma, (const T*)beta, (T*)y, mean, rstd, rows, n, eps);
    });
    SBK_CHECK_LAUNCH();
}

// Backward of y = gamma*xhat + beta over rows in a fixed block-strided order.
// NCOL partial column sums per block go to ws[block][k*n + col] (k = 0 dgamma,
// 1 dbeta, 2 dbias) and are summed in block order by k_col_final.
template <class T, class P, int MODE>  // MODE 0: LayerNorm, 1: bias+dropout+residual+LN
__global__ void k_ln_bwd(const T* x, const float* mean, const float* rstd, const P* gamma, const T* g, T* gx, T* gres,
                         bool gx_acc, i64 rows, i64 n, uint64_t s1, uint64_t thr, float dscale, float* ws, int ncol,
                         bool gres_acc, const T* gext) {
    extern __shared__ float sh[];  // [kWarps][ncol][n]
    int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    float* mine = sh + (size_t)warp * ncol * n;
    for (i64 i = lane; i < (i64)ncol * n; i += 32) mine[i] = 0.f;
    for (i64 row = (i64)blockIdx.x * kWarps + warp; row < rows; row += (i64)gridDim.x * kWarps) {
        const T* px = x + row * n;
        const T* pg = g + row * n;
        float mu = mean[row], rs = rstd[row];
        float a = 0.f, b = 0.f;  // sums of gh and gh*xhat
        for (i64 i = lane; i < n; i += 32) {
            float xh = (to_f(px[i]) - mu) * rs;
            float gv = to_f(pg[i]);
            float gh = gamma ? gv * to_f(gamma[i]) : gv;
            a += gh;
            b += gh * xh;
            if (ncol >= 2) {
                mine[i] += gv * xh;  // dgamma
                mine[n + i] += gv;   // dbeta
            }
        }
        a = warp_sum(a) / (float)n;
        b = warp_sum(b) / (float)n;
        for (i64 i = lane; i < n; i += 32) {
            float xh = (to_f(px[i]) - mu) * rs;
            float gv = to_f(pg[i]);
            float gh = gamma ? gv * to_f(gamma[i]) : gv;
            float d = rs * (gh - a - xh * b);
            i64 k = row * n + i;
            if (MODE == 1 && gext) d += to_f(gext[k]);  // the sum's gradient from its other consumers
            if (MODE == 0) {
                gx[k] = from_f<T>(gx_acc ? to_f(gx[k]) + d : d);
            } else {
                // residual branch gets g_sum; the dense branch gets dropout_bwd(g_sum)
                gres[k] = from_f<T>(gres_acc ? to_f(gres[k]) + d : d);
                float gp = thr == 0 ? d : (d_keep(s1, (uint64_t)k, thr) ? d * dscale : 0.f);
                gx[k] = from_f<T>(gx_acc ? to_f(gx[k]) + gp : gp);
                if (ncol == 3) mine[2 * n + i] += gp;  // dbias
            }
        }
    }
    __syncthreads();
    // fixed-order reduction of the warps' partials -> this block's partial
    for (i64 i = threadIdx.x; i < (i64)ncol * n; i += blockDim.x) {
        float acc = 0.f;
        for (int w = 0; w < kWarps; ++w) acc += sh[(size_t)w * ncol * n + i];
        ws[(i64)blockIdx.x * ncol * n + i] = acc;
    }
}
// block = 32 columns x 32 warps: warp w sums partial rows w, w+32, ... of its lane's
// column with 8 loads in flight (the partials are L2-resident; a serial walk over the
// ~300 block partials was latency-bound at ~9 us), then warp 0 adds the 32 sums in
// warp order (fixed order: deterministic)
__global__ void __launch_bounds__(1024) k_col_final(const float* ws, int blocks, i64 ncoln, float* o0, float* o1, float* o2,
                                                    i64 n, bool accum) {
    __shared__ float part[32][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const i64 i = blockIdx.x * 32ll + lane;
    float acc = 0.f;
    if (i < ncoln) {
        int b = warp;
        for (; b + 7 * 32 < blocks; b += 8 * 32) {
            float a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = __ldcg(ws + (i64)(b + u * 32) * ncoln + i);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += a[u];
        }
        for (; b < blocks; b += 32) acc += __ldcg(ws + (i64)b * ncoln + i);
    }
    part[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && i < ncoln) {
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < 32; ++w) t += part[w][lane];
        int k = (int)(i / n);
        float* o = k == 0 ? o0 : k == 1 ? o1 : o2;
        if (o) o[i % n] = accum ? o[i % n] + t : t;
    }
}
static unsigned col_final_grid(i64 ncoln) { return (unsigned)((ncoln + 31) / 32); }
static int row_blocks(i64 rows) { return (int)std::min<i64>(kRowBlocks, std::max<i64>(1, (rows + kWarps - 1) / kWarps)); }
size_t layernorm_bwd_workspace(i64 rows, i64 n) { return (size_t)row_blocks(rows) * 2 * n * 4; }
size_t bdrln_bwd_workspace(i64 rows, i64 n) { return (size_t)row_blocks(rows) * 3 * n * 4; }

template <class K>
static void set_smem(K k, size_t bytes) {
    if (bytes > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

void layernorm_bwd(const void* x, const float* mean, const float* rstd, const void* gamma, DT tp, const void* g, DT tg,
                   void* gx, float* dgamma, float* dbeta, DT t, i64 rows, i64 n, float* ws, cudaStream_t s, bool gx_acc,
                   bool col_acc) {
    (void)tp;
    (void)tg;
    int ncol = (dgamma || dbeta) ? 2 : 0;
    int vb = vec_blocks(rows);
    if (ln_bwd_vec(0, x, mean, rstd, gamma, g, gx, nullptr, gx_acc, true, t, rows, n, 0, 0, 1.f, nullptr, ws, ncol, vb, s)) {
        if (ncol) k_col_final<<<col_final_grid(2 * n), 1024, 0, s>>>(ws, vb, 2 * n, dgamma, dbeta, nullptr, n, col_acc);
        SBK_CHECK_LAUNCH();
        return;
    }
    int nb = row_blocks(rows);
    size_t smem = (size_t)kWarps * ncol * n * 4;
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        auto k = k_ln_bwd<T, T, 0>;
        set_smem(k, smem);
        k<<<nb, 32 * kWarps, smem, s>>>((const T*)x, mean, rstd, (const T*)gamma, (const T*)g, (T*)gx, nullptr, gx_acc,
                                        rows, n, 0, 0, 1.f, ws, ncol, true, nullptr);
    });
    if (ncol) k_col_final<<<col_final_grid(2 * n), 1024, 0, s>>>(ws, nb, 2 * n, dgamma, dbeta, nullptr, n, col_acc);
    SBK_CHECK_LAUNCH();
}

// ------------------------------------------- fused bias+dropout+residual+LN
template <class T>
__global__ void k_bdrln_fwd(const T* partial, const T* bias, const T* res, const T* gamma, const T* beta, T* sum, T* y,
                            float* mean, float* rstd, i64 rows, i64 n, float eps, uint64_t s1, uint64_t thr,
                            float dscale) {
    i64 row = blockIdx.x * (i64)kWarps + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (row >= rows) return;
    // pass 1: sum = dropout(partial + bias) + residual (dropout index = flat (row, col))
    for (i64 i = lane; i < n; i += 32) {
        i64 k = row * n + i;
        float v = to_f(partial[k]) + (bias ? to_f(bias[i]) : 0.f);
        if (thr) v = d_keep(s1, (uint64_t)k, thr) ? v * dscale : 0.f;
        sum[k] = from_f<T>(v + to_f(res[k]));
    }
    __syncwarp();
    float mu, rs;
    row_stats(sum + row * n, n, lane, eps, mu, rs);
    for (i64 i = lane; i < n; i += 32) {
        i64 k = row * n + i;
        y[k] = from_f<T>(to_f(gamma[i]) * ((to_f(sum[k]) - mu) * rs) + to_f(beta[i]));
    }
    if (lane == 0) {
        mean[row] = mu;
        rstd[row] = rs;
    }
}
void bias_dropout_residual_ln_fwd(const void* partial, const void* bias, const void* residual, const void* gamma,
                                  const void* beta, DT tp, void* sum, void* y, float* mean, float* rstd, DT t, i64 rows,
                                  i64 n, float eps, u64 s1, u64 thr, float dscale, cudaStream_t s, const uint32_t* keep) {
    (void)tp;
    if (bdrln_fwd_vec(partial, bias, residual, gamma, beta, sum, y, mean, rstd, t, rows, n, eps, s1, thr, dscale, keep, s)) {
        SBK_CHECK_LAUNCH();
        return;
    }
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        k_bdrln_fwd<T><<<(unsigned)((rows + kWarps - 1) / kWarps), 32 * kWarps, 0, s>>>(
            (const T*)partial, (const T*)bias, (const T*)residual, (const T*)gamma, (const T*)beta, (T*)sum, (T*)y, mean,
            rstd, rows, n, eps, s1, thr, dscale);
    });
    SBK_CHECK_LAUNCH();
}
void bias_dropout_residual_ln_bwd(const void* sum, const float* mean, const float* rstd, const void* gamma, DT tp,
                                  const void* g, void* g_res, void* g_partial, bool g_partial_acc, float* dbias,
                                  float* dgamma, float* dbeta, DT t, i64 rows, i64 n, u64 s1, u64 thr, float dscale,
                                  float* ws, cudaStream_t s, bool gres_acc, bool col_acc, const uint32_t* keep,
                                  const void* gext) {
    (void)tp;
    int ncol = 3;
    int vb = vec_blocks(rows);
    if (ln_bwd_vec(1, sum, mean, rstd, gamma, g, g_partial, g_res, g_partial_acc, gres_acc, t, rows, n, s1, thr, dscale,
                   keep, ws, ncol, vb, s, gext)) {
        k_col_final<<<col_final_grid(3 * n), 1024, 0, s>>>(ws, vb, 3 * n, dgamma, dbeta, dbias, n, col_acc);
        SBK_CHECK_LAUNCH();
        return;
    }
    int nb = row_blocks(rows);
    size_t smem = (size_t)kWarps * ncol * n * 4;
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        auto k = k_ln_bwd<T, T, 1>;
        set_smem(k, smem);
        k<<<nb, 32 * kWarps, smem, s>>>((const T*)sum, mean, rstd, (const T*)gamma, (const T*)g, (T*)g_partial, (T*)g_res,
                                        g_partial_acc, rows, n, s1, thr, dscale, ws, ncol, gres_acc, (const T*)gext);
    });
    k_col_final<<<col_final_grid(3 * n), 1024, 0, s>>>(ws, nb, 3 * n, dgamma, dbeta, dbias, n, col_acc);
    SBK_CHECK_LAUNCH();
}

}  // namespace sbk
