#include <cstdlib>
// Vectorised LayerNorm family for rows of n = 32 * VEC * CPL elements: one
// warp per row, 16-byte loads/stores, the whole row in registers (single HBM
// read of every input), fp32 statistics. Backward keeps the per-column
// dgamma/dbeta/dbias partial sums in registers across the rows a warp visits
// and reduces them across warps/blocks in a fixed order (deterministic).
// Math as norm.cu (proj/src/executor.cpp:699-740, 1158-1197).
#include "common.cuh"

namespace sbk {

namespace {

template <class T>
struct Vec;
template <>
struct Vec<bf16> {
    static constexpr int N = 8;
    using R = uint4;
    __device__ static void unpack(const R& r, float* f) {
        const __nv_bfloat162* h = (const __nv_bfloat162*)&r;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float2 v = __bfloat1622float2(h[i]);
            f[2 * i] = v.x;
            f[2 * i + 1] = v.y;
        }
    }
    __device__ static R pack(const float* f) {
        R r;
        __nv_bfloat162* h = (__nv_bfloat162*)&r;
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
        return r;
    }
};
template <>
struct Vec<float> {
    static constexpr int N = 4;
    using R = float4;
    __device__ static void unpack(const R& r, float* f) {
        f[0] = r.x;
        f[1] = r.y;
        f[2] = r.z;
        f[3] = r.w;
    }
    __device__ static R pack(const float* f) { return make_float4(f[0], f[1], f[2], f[3]); }
};

constexpr int kW = 8;  // warps per block

template <class T, int CPL>
__device__ __forceinline__ void load_row(const T* p, int lane, float (&v)[CPL][Vec<T>::N]) {
    using V = Vec<T>;
#pragma unroll
    for (int c = 0; c < CPL; ++c) V::unpack(((const typename V::R*)p)[c * 32 + lane], v[c]);
}
template <class T, int CPL>
__device__ __forceinline__ void store_row(T* p, int lane, const float (&v)[CPL][Vec<T>::N]) {
    using V = Vec<T>;
#pragma unroll
    for (int c = 0; c < CPL; ++c) ((typename V::R*)p)[c * 32 + lane] = V::pack(v[c]);
}
template <int CPL, int VN>
__device__ __forceinline__ void stats(const float (&v)[CPL][VN], float n, float eps, float& mu, float& rs) {
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c)
#pragma unroll
        for (int e = 0; e < VN; ++e) s += v[c][e];
    mu = warp_sum(s) / n;
    float q = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c)
#pragma unroll
        for (int e = 0; e < VN; ++e) {
            float d = v[c][e] - mu;
            q += d * d;
        }
    rs = rsqrtf(warp_sum(q) / n + eps);
}
__device__ __forceinline__ int col_of(int c, int lane, int e, int VN) { return (c * 32 + lane) * VN + e; }
// the VN keep bits of elements idx0 .. idx0+VN-1 (idx0 % VN == 0, VN <= 8) from a
// dropout_mask bit array (bit i of word w = element 32w + i, i.e. byte idx/8, bit idx%8)
// keep bits of VN consecutive elements hashed in place (no precomputed bits);
// out of line so the hash does not inflate the register budget of the caller
template <int VN>
__device__ __noinline__ uint32_t hash_keep_bits(uint64_t s1, uint64_t thr, i64 idx0) {
    uint32_t m = 0;
    for (int e = 0; e < VN; ++e)
        if (d_keep(s1, (uint64_t)(idx0 + e), thr)) m |= 1u << e;
    return m;
}
template <int VN>
__device__ __forceinline__ uint32_t keep_bits(const uint32_t* keep, i64 idx0) {
    const uint32_t byte = ((const uint8_t*)keep)[idx0 >> 3];
    return VN == 8 ? byte : (byte >> (idx0 & 7)) & ((1u << VN) - 1);
}

template <class T, int CPL>
__global__ void __launch_bounds__(32 * kW) k_ln_fwd_v(const T* x, const T* gamma, const T* beta, T* y, float* mean,
                                                      float* rstd, i64 rows, int n, float eps) {
    constexpr int VN = Vec<T>::N;
    i64 row = blockIdx.x * (i64)kW + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (row >= rows) return;
    float v[CPL][VN];
    load_row<T, CPL>(x + row * n, lane, v);
    float mu, rs;
    stats<CPL, VN>(v, (float)n, eps, mu, rs);
    float g[CPL][VN], b[CPL][VN];
    if (gamma) {
        load_row<T, CPL>(gamma, lane, g);
        load_row<T, CPL>(beta, lane, b);
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c)
#pragma unroll
        for (int e = 0; e < VN; ++e) {
            float h = (v[c][e] - mu) * rs;
            v[c][e] = gamma ? g[c][e] * h + b[c][e] : h;
        }
    store_row<T, CPL>(y + row * n, lane, v);
    if (lane == 0) {
        mean[row] = mu;
        rstd[row] = rs;
    }
}

template <class T, int CPL>
__global__ void __launch_bounds__(32 * kW) k_bdrln_fwd_v(const T* partial, const T* bias, const T* res, const T* gamma,
                                                         const T* beta, T* sum, T* y, float* mean, float* rstd, i64 rows,
                                                         int n, float eps, uint64_t s1, uint64_t thr, float dscale,
                                                         const uint32_t* keep) {
    constexpr int VN = Vec<T>::N;
    i64 row = blockIdx.x * (i64)kW + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (row >= rows) return;
    float v[CPL][VN], r[CPL][VN];
    load_row<T, CPL>(partial + row * n, lane, v);
    load_row<T, CPL>(res + row * n, lane, r);
    float bb[CPL][VN];
    if (bias) load_row<T, CPL>(bias, lane, bb);
    uint32_t kb[CPL];
    if (thr && keep) {
#pragma unroll
        for (int c = 0; c < CPL; ++c) kb[c] = keep_bits<VN>(keep, row * n + col_of(c, lane, 0, VN));
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c)
#pragma unroll
        for (int e = 0; e < VN; ++e) {
            float t = v[c][e] + (bias ? bb[c][e] : 0.f);
            if (thr) {
                const bool kept = keep ? ((kb[c] >> e) & 1) : d_keep(s1, (uint64_t)(row * n + col_of(c, lane, e, VN)), thr);
                t = kept ? t * dscale : 0.f;
            }
            v[c][e] = t + r[c][e];
        }
    // `sum` is rounded to the storage dtype before the statistics, exactly as
    // the backward will re-read it
    store_row<T, CPL>(sum + row * n, lane, v);
#pragma unroll
    for (int c = 0; c < CPL; ++c)
#pragma unroll
        for (int e = 0; e < VN; ++e) v[c][e] = to_f(from_f<T>(v[c][e]));
    float mu, rs;
    stats<CPL, VN>(v, (float)n, eps, mu, rs);
    load_row<T, CPL>(gamma, lane, r);
    load_row<T, CPL>(beta, lane, bb);
#pragma unroll
    for (int c = 0; c < CPL; ++c)
#pragma unroll
        for (int e = 0; e < VN; ++e) v[c][e] = r[c][e] * ((v[c][e] - mu) * rs) + bb[c][e];
    store_row<T, CPL>(y + row * n, lane, v);
    if (lane == 0) {
        mean[row] = mu;
        rstd[row] = rs;
    }
}

// bias+dropout+residual+LayerNorm forward with WPR warps per row (each warp owns
// CPL/WPR 16-byte column chunks) and NR rows per warp group in flight (all their
// loads issued before any math: bytes in flight for HBM): few registers, 16-warp
// blocks; the row mean and variance are combined across the WPR warps through
// shared memory in a fixed order.
template <class T, int CPL, int WPR, int NR, int MINB = 2>
__global__ void __launch_bounds__(512, MINB) k_bdrln_fwd_w(const T* partial, const T* bias, const T* res, const T* gamma,
                                                     const T* beta, T* sum, T* y, float* mean, float* rstd, i64 rows,
                                                     int n, float eps, uint64_t s1, uint64_t thr, float dscale,
                                                     const uint32_t* keep) {
    using V = Vec<T>;
    constexpr int VN = V::N, CW = CPL / WPR, RPB = 16 / WPR;
    __shared__ float red[2][2][16][NR];
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31, slot = warp / WPR, part = warp % WPR;
    // row groups of NR consecutive rows, grid-strided; the next group's inputs are loaded
    // while the current one is processed (rows % (RPB * NR) == 0)
    const i64 gstep = (i64)gridDim.x * RPB;
    i64 grp = (i64)blockIdx.x * RPB + slot;
    const i64 ngrp = rows / NR;
    typename V::R pn[NR][CW], rn[NR][CW];
    auto prefetch = [&](i64 gi) {
        if (gi >= ngrp) return;
#pragma unroll
        for (int k = 0; k < NR; ++k)
#pragma unroll
            for (int c = 0; c < CW; ++c) {
                const int ch = (part * CW + c) * 32 + lane;
                pn[k][c] = __ldcs((const typename V::R*)(partial + (gi * NR + k) * n) + ch);
                rn[k][c] = __ldcs((const typename V::R*)(res + (gi * NR + k) * n) + ch);
            }
    };
    // per-column parameters: this thread always owns the same columns
    // (kept packed: unpacked at each use, one ALU op per element)
    typename V::R bbp[CW], gmp[CW], btp[CW];
#pragma unroll
    for (int c = 0; c < CW; ++c) {
        const int ch = (part * CW + c) * 32 + lane;
        if (bias) bbp[c] = ((const typename V::R*)bias)[ch];
        else bbp[c] = typename V::R{};
        gmp[c] = ((const typename V::R*)gamma)[ch];
        btp[c] = ((const typename V::R*)beta)[ch];
    }
    const float inv_n = 1.f / (float)n;
    prefetch(grp);
    for (int it = 0; grp < ngrp; grp += gstep, ++it) {
        const i64 row0 = grp * NR;
        float v[NR][CW][VN];
        float sm[NR];
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            sm[k] = 0.f;
#pragma unroll
            for (int c = 0; c < CW; ++c) V::unpack(pn[k][c], v[k][c]);
        }
        float rv[NR][CW][VN];
#pragma unroll
        for (int k = 0; k < NR; ++k)
#pragma unroll
            for (int c = 0; c < CW; ++c) V::unpack(rn[k][c], rv[k][c]);
        prefetch(grp + gstep);
#pragma unroll
        for (int k = 0; k < NR; ++k) {
#pragma unroll
            for (int c = 0; c < CW; ++c) {
                const int ch = (part * CW + c) * 32 + lane;
                uint32_t kb = 0;
                if (thr) kb = keep_bits<VN>(keep, (row0 + k) * n + (i64)ch * VN);  // keep != null (host)
                float bbv[VN];
                V::unpack(bbp[c], bbv);
#pragma unroll
                for (int e = 0; e < VN; ++e) {
                    float t = v[k][c][e] + bbv[e];
                    if (thr) t = ((kb >> e) & 1) ? t * dscale : 0.f;
                    v[k][c][e] = t + rv[k][c][e];
                }
                // `sum` rounded to the storage dtype first: pack once, and the statistics
                // read the rounded values back from the packed vector
                const typename V::R packed = V::pack(v[k][c]);
                ((typename V::R*)(sum + (row0 + k) * n))[ch] = packed;
                V::unpack(packed, v[k][c]);
#pragma unroll
                for (int e = 0; e < VN; ++e) sm[k] += v[k][c][e];
            }
        }
        auto row_sums = [&](float (&xx)[NR], int which) {
#pragma unroll
            for (int k = 0; k < NR; ++k) xx[k] = warp_sum(xx[k]);
            if (WPR > 1) {
                if (lane == 0)
#pragma unroll
                    for (int k = 0; k < NR; ++k) red[it & 1][which][warp][k] = xx[k];
                asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(32 * WPR) : "memory");
#pragma unroll
                for (int k = 0; k < NR; ++k) {
                    xx[k] = 0.f;
#pragma unroll
                    for (int w = 0; w < WPR; ++w) xx[k] += red[it & 1][which][slot * WPR + w][k];
                }
            }
        };
        row_sums(sm, 0);
        float mu[NR], q[NR];
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            mu[k] = sm[k] * inv_n;  // (n a power of two: the same bits as / n)
            q[k] = 0.f;
#pragma unroll
            for (int c = 0; c < CW; ++c)
#pragma unroll
                for (int e = 0; e < VN; ++e) {
                    const float d = v[k][c][e] - mu[k];
                    q[k] += d * d;
                }
        }
        row_sums(q, 1);
#pragma unroll
        for (int c = 0; c < CW; ++c) {
            const int ch = (part * CW + c) * 32 + lane;
            float gmv[VN], btv[VN];
            V::unpack(gmp[c], gmv);
            V::unpack(btp[c], btv);
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                const float rs = rsqrtf(q[k] * inv_n + eps);
                float o[VN];
#pragma unroll
                for (int e = 0; e < VN; ++e) o[e] = gmv[e] * ((v[k][c][e] - mu[k]) * rs) + btv[e];
                ((typename V::R*)(y + (row0 + k) * n))[ch] = V::pack(o);
            }
        }
        if (lane == 0 && part == 0)
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                mean[row0 + k] = mu[k];
                rstd[row0 + k] = rsqrtf(q[k] / (float)n + eps);
            }
    }
}

// MODE 0: LayerNorm backward (gx += ...). MODE 1: fused bias+dropout+residual+LN
// backward: g_sum = LNbwd(g); gres += g_sum; gx (=g_partial) (+)= dropout_bwd(g_sum);
// NCOL column partials (dgamma, dbeta[, dbias]) -> ws[block][k*n + col].
template <class T, int CPL, int MODE>
__global__ void __launch_bounds__(32 * kW, 1)
    k_ln_bwd_v(const T* x, const float* mean, const float* rstd, const T* gamma, const T* g, T* gx, T* gres, bool gx_acc,
               i64 rows, int n, uint64_t s1, uint64_t thr, float dscale, const uint32_t* keep, float* ws, int ncol,
               bool gres_acc, const T* gext) {
    constexpr int VN = Vec<T>::N;
    extern __shared__ float sh[];  // [kW][ncol][n]
    int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    float gm[CPL][VN];
    if (gamma) load_row<T, CPL>(gamma, lane, gm);
    float pg[CPL][VN] = {}, pb[CPL][VN] = {}, pd[CPL][VN] = {};
    for (i64 row = (i64)blockIdx.x * kW + warp; row < rows; row += (i64)gridDim.x * kW) {
        float xv[CPL][VN], gv[CPL][VN];
        load_row<T, CPL>(x + row * n, lane, xv);
        load_row<T, CPL>(g + row * n, lane, gv);
        float mu = mean[row], rs = rstd[row];
        float a = 0.f, b = 0.f;
#pragma unroll
        for (int c = 0; c < CPL; ++c)
#pragma unroll
            for (int e = 0; e < VN; ++e) {
                float xh = (xv[c][e] - mu) * rs;
                float gh = gamma ? gv[c][e] * gm[c][e] : gv[c][e];
                a += gh;
                b += gh * xh;
                pg[c][e] += gv[c][e] * xh;
                pb[c][e] += gv[c][e];
                xv[c][e] = xh;
            }
        a = warp_sum(a) / (float)n;
        b = warp_sum(b) / (float)n;
#pragma unroll
        for (int c = 0; c < CPL; ++c)
#pragma unroll
            for (int e = 0; e < VN; ++e) {
                float gh = gamma ? gv[c][e] * gm[c][e] : gv[c][e];
                gv[c][e] = rs * (gh - a - xv[c][e] * b);  // d(sum) / dx
            }
        if (MODE == 1 && gext) {  // + the sum's gradient from its other consumers (pre-LN residual stream)
            float ex[CPL][VN];
            load_row<T, CPL>(gext + row * n, lane, ex);
#pragma unroll
            for (int c = 0; c < CPL; ++c)
#pragma unroll
                for (int e = 0; e < VN; ++e) gv[c][e] += ex[c][e];
        }
        if (MODE == 0) {
            float o[CPL][VN] = {};
            if (gx_acc) load_row<T, CPL>(gx + row * n, lane, o);
#pragma unroll
            for (int c = 0; c < CPL; ++c)
#pragma unroll
                for (int e = 0; e < VN; ++e) o[c][e] += gv[c][e];
            store_row<T, CPL>(gx + row * n, lane, o);
        } else {
            float o[CPL][VN] = {};
            if (gres_acc) load_row<T, CPL>(gres + row * n, lane, o);
#pragma unroll
            for (int c = 0; c < CPL; ++c)
#pragma unroll
                for (int e = 0; e < VN; ++e) o[c][e] += gv[c][e];
            store_row<T, CPL>(gres + row * n, lane, o);
            uint32_t kb[CPL];
            if (thr && keep) {
#pragma unroll
                for (int c = 0; c < CPL; ++c) kb[c] = keep_bits<VN>(keep, row * n + col_of(c, lane, 0, VN));
            }
#pragma unroll
            for (int c = 0; c < CPL; ++c)
#pragma unroll
                for (int e = 0; e < VN; ++e) {
                    float d = gv[c][e];
                    if (thr) {
                        const bool kept =
                            keep ? ((kb[c] >> e) & 1) : d_keep(s1, (uint64_t)(row * n + col_of(c, lane, e, VN)), thr);
                        d = kept ? d * dscale : 0.f;
                    }
                    gv[c][e] = d;
                    pd[c][e] += d;
                }
            if (gx_acc) {
                load_row<T, CPL>(gx + row * n, lane, o);
#pragma unroll
                for (int c = 0; c < CPL; ++c)
#pragma unroll
                    for (int e = 0; e < VN; ++e) gv[c][e] += o[c][e];
            }
            store_row<T, CPL>(gx + row * n, lane, gv);
        }
    }
    if (ncol == 0) return;
    float* mine = sh + (size_t)warp * ncol * n;
#pragma unroll
    for (int c = 0; c < CPL; ++c)
#pragma unroll
        for (int e = 0; e < VN; ++e) {
            int col = col_of(c, lane, e, VN);
            mine[col] = pg[c][e];
            mine[n + col] = pb[c][e];
            if (ncol == 3) mine[2 * n + col] = pd[c][e];
        }
    __syncthreads();
    for (int i = threadIdx.x; i < ncol * n; i += blockDim.x) {
        float acc = 0.f;
        for (int w = 0; w < kW; ++w) acc += sh[(size_t)w * ncol * n + i];
        ws[(i64)blockIdx.x * ncol * n + i] = acc;
    }
}

// The same backward with WPR warps per row (each warp owns CPL/WPR 16-byte
// column chunks): a quarter of the registers of the warp-per-row kernel (the
// per-column dgamma/dbeta/dbias partials dominate), so 16-warp blocks fit and
// co-reside with other work. The two row sums are combined across the WPR warps
// through shared memory in a fixed order (deterministic).
template <class T, int CPL, int MODE, int WPR, int MINB = 1, bool PF2 = (CPL >= 8 && CPL / WPR == 1)>
__global__ void __launch_bounds__(512, MINB)
    k_ln_bwd_w(const T* x, const float* mean, const float* rstd, const T* gamma, const T* g, T* gx, T* gres, bool gx_acc,
               i64 rows, int n, uint64_t s1, uint64_t thr, float dscale, const uint32_t* keep, float* ws, int ncol,
               bool gres_acc, const T* gext) {
    constexpr int VN = Vec<T>::N, CW = CPL / WPR, RPB = 16 / WPR;  // chunks per warp, rows per block pass
    extern __shared__ float sh[];  // [16 warps][ncol][CW*32*VN] column partials | red[2][16][2]
    float* red = sh + (size_t)16 * ncol * (CW * 32 * VN);
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31, slot = warp / WPR, part = warp % WPR;
    using V = Vec<T>;
    typename V::R gmp[CW];  // packed; unpacked at each use
#pragma unroll
    for (int c = 0; c < CW; ++c)
        gmp[c] = gamma ? ((const typename V::R*)gamma)[(part * CW + c) * 32 + lane] : typename V::R{};
    float pg[CW][VN] = {}, pb[CW][VN] = {}, pd[CW][VN] = {};
    int it = 0;
    // software pipeline: the next row's x / g / statistics are loaded while this row is processed
    const i64 rstep = (i64)gridDim.x * RPB;
    i64 row = (i64)blockIdx.x * RPB + slot;
    // rows in flight: the next one (PF2: the next two — 2048-wide rows at one chunk per warp,
    // 37.2 -> 35.3 us; no gain at 1024 / 768 — profiles/r2/ln_bwd_pf2_ab.log) loaded while this
    // one is processed
    typename V::R xn[CW], gn[CW], xn2[CW], gn2[CW];
    float mun = 0.f, rsn = 0.f, mun2 = 0.f, rsn2 = 0.f;
    auto load = [&](i64 r, typename V::R(&xd)[CW], typename V::R(&gd)[CW], float& mu_d, float& rs_d) {
        if (r >= rows) return;
#pragma unroll
        for (int c = 0; c < CW; ++c) {
            xd[c] = __ldcs((const typename V::R*)(x + r * n) + (part * CW + c) * 32 + lane);
            gd[c] = __ldcs((const typename V::R*)(g + r * n) + (part * CW + c) * 32 + lane);
        }
        mu_d = mean[r];
        rs_d = rstd[r];
    };
    load(row, xn, gn, mun, rsn);
    if (PF2) load(row + rstep, xn2, gn2, mun2, rsn2);
    for (; row < rows; row += rstep, ++it) {
        float xv[CW][VN], gv[CW][VN];
#pragma unroll
        for (int c = 0; c < CW; ++c) {
            V::unpack(xn[c], xv[c]);
            V::unpack(gn[c], gv[c]);
        }
        const float mu = mun, rs = rsn;
        if (PF2) {
#pragma unroll
            for (int c = 0; c < CW; ++c) {
                xn[c] = xn2[c];
                gn[c] = gn2[c];
            }
            mun = mun2;
            rsn = rsn2;
            load(row + 2 * rstep, xn2, gn2, mun2, rsn2);
        } else {
            load(row + rstep, xn, gn, mun, rsn);
        }
        float a = 0.f, b = 0.f;
#pragma unroll
        for (int c = 0; c < CW; ++c) {
            float gm[VN];
            V::unpack(gmp[c], gm);
#pragma unroll
            for (int e = 0; e < VN; ++e) {
                const float xh = (xv[c][e] - mu) * rs;
                const float gh = gamma ? gv[c][e] * gm[e] : gv[c][e];
                a += gh;
                b += gh * xh;
                pg[c][e] += gv[c][e] * xh;
                pb[c][e] += gv[c][e];
                xv[c][e] = xh;
            }
        }
        a = warp_sum(a);
        b = warp_sum(b);
        if (WPR > 1) {
            float* rr = red + ((it & 1) * 16 + warp) * 2;
            if (lane == 0) {
                rr[0] = a;
                rr[1] = b;
            }
            asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(32 * WPR) : "memory");
            const float* r0 = red + ((it & 1) * 16 + slot * WPR) * 2;
            a = 0.f;
            b = 0.f;
#pragma unroll
            for (int w = 0; w < WPR; ++w) {
                a += r0[2 * w];
                b += r0[2 * w + 1];
            }
        }
        a /= (float)n;
        b /= (float)n;
#pragma unroll
        for (int c = 0; c < CW; ++c) {
            float gm[VN];
            V::unpack(gmp[c], gm);
#pragma unroll
            for (int e = 0; e < VN; ++e) {
                const float gh = gamma ? gv[c][e] * gm[e] : gv[c][e];
                gv[c][e] = rs * (gh - a - xv[c][e] * b);  // d(sum) / dx
            }
        }
        typename V::R* gxr = (typename V::R*)(gx + row * n);
        if (MODE == 0) {
#pragma unroll
            for (int c = 0; c < CW; ++c) {
                float o[VN];
                if (gx_acc) V::unpack(gxr[(part * CW + c) * 32 + lane], o);
#pragma unroll
                for (int e = 0; e < VN; ++e) o[e] = (gx_acc ? o[e] : 0.f) + gv[c][e];
                gxr[(part * CW + c) * 32 + lane] = V::pack(o);
            }
        } else {
            typename V::R* grr = (typename V::R*)(gres + row * n);
#pragma unroll
            for (int c = 0; c < CW; ++c) {
                const int ch = (part * CW + c) * 32 + lane;
                float o[VN];
                if (gext) {  // + the sum's gradient from its other consumers (pre-LN residual stream)
                    V::unpack(((const typename V::R*)(gext + row * n))[ch], o);
#pragma unroll
                    for (int e = 0; e < VN; ++e) gv[c][e] += o[e];
                }
                if (gres_acc) V::unpack(grr[ch], o);
#pragma unroll
                for (int e = 0; e < VN; ++e) o[e] = (gres_acc ? o[e] : 0.f) + gv[c][e];
                grr[ch] = V::pack(o);
                uint32_t kb = 0;
                if (thr) kb = keep_bits<VN>(keep, row * n + (i64)ch * VN);  // keep != null (host)
#pragma unroll
                for (int e = 0; e < VN; ++e) {
                    float d = gv[c][e];
                    if (thr) d = ((kb >> e) & 1) ? d * dscale : 0.f;
                    gv[c][e] = d;
                    pd[c][e] += d;
                }
                if (gx_acc) {
                    V::unpack(gxr[ch], o);
#pragma unroll
                    for (int e = 0; e < VN; ++e) gv[c][e] += o[e];
                }
                gxr[ch] = V::pack(gv[c]);
            }
        }
    }
    if (ncol == 0) return;
    // column partials: warp's own segment, then a fixed-order sum over the row slots
    constexpr int SEG = CW * 32 * VN;
    float* mine = sh + (size_t)warp * ncol * SEG;
#pragma unroll
    for (int c = 0; c < CW; ++c)
#pragma unroll
        for (int e = 0; e < VN; ++e) {
            const int lc = (c * 32 + lane) * VN + e;
            mine[lc] = pg[c][e];
            mine[SEG + lc] = pb[c][e];
            if (ncol == 3) mine[2 * SEG + lc] = pd[c][e];
        }
    __syncthreads();
    for (int i = threadIdx.x; i < ncol * n; i += blockDim.x) {
        const int k = i / n, col = i % n;
        // column col: chunk col / VN -> owning part = (chunk / 32) / CW, local = col - part * SEG
        const int prt = (col / VN / 32) / CW, lc = col - prt * SEG;
        float acc = 0.f;
        for (int sl = 0; sl < RPB; ++sl) acc += sh[(size_t)(sl * WPR + prt) * ncol * SEG + (size_t)k * SEG + lc];
        ws[(i64)blockIdx.x * ncol * n + i] = acc;
    }
}

template <class T, class F>
bool with_cpl(int n, F&& f) {
    constexpr int VN = Vec<T>::N;
    if (n % (32 * VN)) return false;
    switch (n / (32 * VN)) {
        case 1: f(std::integral_constant<int, 1>{}); return true;
        case 2: f(std::integral_constant<int, 2>{}); return true;
        case 3: f(std::integral_constant<int, 3>{}); return true;
        case 4: f(std::integral_constant<int, 4>{}); return true;
        case 6: f(std::integral_constant<int, 6>{}); return true;
        case 8: f(std::integral_constant<int, 8>{}); return true;
        default: return false;
    }
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }
// SB_LN_NARROW=1: one warp per row everywhere (A/B and diagnostics)
bool ln_narrow() {
    static const bool on = getenv("SB_LN_NARROW") && atoi(getenv("SB_LN_NARROW"));
    return on;
}

}  // namespace

int ln_bwd_blocks(i64 rows);  // norm.cu

bool ln_fwd_vec(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd, DT t, i64 rows,
                i64 n, float eps, cudaStream_t s) {
    if (t == F64 || !aligned16(x) || !aligned16(y) || (gamma && (!aligned16(gamma) || !aligned16(beta)))) return false;
    bool ok = false;
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        if constexpr (!std::is_same_v<T, double>) {
            ok = with_cpl<T>((int)n, [&](auto cc) {
                k_ln_fwd_v<T, decltype(cc)::value><<<(unsigned)((rows + kW - 1) / kW), 32 * kW, 0, s>>>(
                    (const T*)x, (const T*)gamma, (const T*)beta, (T*)y, mean, rstd, rows, (int)n, eps);
            });
        }
    });
    return ok;
}

bool bdrln_fwd_vec(const void* partial, const void* bias, const void* res, const void* gamma, const void* beta, void* sum,
                   void* y, float* mean, float* rstd, DT t, i64 rows, i64 n, float eps, u64 s1, u64 thr, float dscale,
                   const uint32_t* keep, cudaStream_t s) {
    for (const void* p : {partial, res, gamma, beta, (const void*)sum, (const void*)y})
        if (!aligned16(p)) return false;
    if (t == F64 || (bias && !aligned16(bias))) return false;
    bool ok = false;
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        if constexpr (!std::is_same_v<T, double>) {
            ok = with_cpl<T>((int)n, [&](auto cc) {
                constexpr int CPL = decltype(cc)::value;
                if constexpr (CPL % 4 == 0) {
                    // 4 warps per row, 16-warp blocks (4 rows per block)
                    if ((thr == 0 || keep) && !ln_narrow()) {
                        // 4 warps per row, persistent grid of two 16-warp blocks per SM (<= 64 registers);
                        // 2048-wide bf16 rows (CPL 8): one block per SM (<= 128 registers: 292 B of
                        // spills at 64)
                        static int sms = 0;
                        if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
                        if constexpr (CPL >= 8) {
                            const unsigned blocks = (unsigned)std::min<i64>(sms, (rows + 3) / 4);
                            k_bdrln_fwd_w<T, CPL, 4, 1, 1><<<blocks, 512, 0, s>>>(
                                (const T*)partial, (const T*)bias, (const T*)res, (const T*)gamma, (const T*)beta, (T*)sum,
                                (T*)y, mean, rstd, rows, (int)n, eps, s1, thr, dscale, keep);
                        } else {
                            const unsigned blocks = (unsigned)std::min<i64>(2 * sms, (rows + 3) / 4);
                            k_bdrln_fwd_w<T, CPL, 4, 1><<<blocks, 512, 0, s>>>(
                                (const T*)partial, (const T*)bias, (const T*)res, (const T*)gamma, (const T*)beta, (T*)sum,
                                (T*)y, mean, rstd, rows, (int)n, eps, s1, thr, dscale, keep);
                        }
                        return;
                    }
                }
                if constexpr (CPL == 3) {
                    // 768-wide bf16 rows (T5-base): 3 warps per row, 15-warp blocks (5 rows), two per SM
                    if ((thr == 0 || keep) && !ln_narrow()) {
                        static int sms3 = 0;
                        if (!sms3) cudaDeviceGetAttribute(&sms3, cudaDevAttrMultiProcessorCount, 0);
                        const unsigned blocks = (unsigned)std::min<i64>(2 * sms3, (rows + 4) / 5);
                        k_bdrln_fwd_w<T, 3, 3, 1><<<blocks, 480, 0, s>>>(
                            (const T*)partial, (const T*)bias, (const T*)res, (const T*)gamma, (const T*)beta, (T*)sum,
                            (T*)y, mean, rstd, rows, (int)n, eps, s1, thr, dscale, keep);
                        return;
                    }
                }
                k_bdrln_fwd_v<T, CPL><<<(unsigned)((rows + kW - 1) / kW), 32 * kW, 0, s>>>(
                    (const T*)partial, (const T*)bias, (const T*)res, (const T*)gamma, (const T*)beta, (T*)sum, (T*)y,
                    mean, rstd, rows, (int)n, eps, s1, thr, dscale, keep);
            });
        }
    });
    return ok;
}

// mode 0: LN backward into gx (+=); mode 1: bdrln backward. Writes ncol column
// partials per block to ws (the caller finishes with the fixed-order column sum).
bool ln_bwd_vec(int mode, const void* x, const float* mean, const float* rstd, const void* gamma, const void* g, void* gx,
                void* gres, bool gx_acc, bool gres_acc, DT t, i64 rows, i64 n, u64 s1, u64 thr, float dscale,
                const uint32_t* keep, float* ws, int ncol, int& nblocks, cudaStream_t s, const void* gext) {
    if (gext && !aligned16(gext)) return false;
    for (const void* p : {x, g, (const void*)gx})
        if (!aligned16(p)) return false;
    if (t == F64 || (gamma && !aligned16(gamma)) || (gres && !aligned16(gres))) return false;
    size_t smem = (size_t)kW * ncol * n * 4;
    if (smem > 200 * 1024) return false;
    bool ok = false;
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        if constexpr (!std::is_same_v<T, double>) {
            ok = with_cpl<T>((int)n, [&](auto cc) {
                constexpr int CPL = decltype(cc)::value;
                auto launch = [&](auto k) {
                    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    k<<<nblocks, 32 * kW, smem, s>>>((const T*)x, mean, rstd, (const T*)gamma, (const T*)g, (T*)gx,
                                                     (T*)gres, gx_acc, rows, (int)n, s1, thr, dscale, keep, ws,
                                                     ncol, gres_acc, (const T*)gext);
                };
                if constexpr (CPL % 4 == 0) {
                  if ((thr == 0 || keep) && !ln_narrow()) {
                    // 2, 4 or 8 warps per row, one 16-warp block per SM (<= 128 registers); SB_LN_WPR=2 / 4
                    // forces 2 / 4 warps per row at CPL 4, SB_LN_WPR=4 / 8 forces 4 / 8 at CPL 8
                    static const int wpr_env = getenv("SB_LN_WPR") ? atoi(getenv("SB_LN_WPR")) : 0;
                    auto go = [&](auto wc) {
                        constexpr int WPR = decltype(wc)::value;
                        const size_t sm2 = (size_t)16 * ncol * (n / WPR) * 4 + 2 * 16 * 2 * 4;
                        auto k = mode == 0 ? k_ln_bwd_w<T, CPL, 0, WPR> : k_ln_bwd_w<T, CPL, 1, WPR>;
                        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
                        // one persistent block per SM (the column finish then sums one partial row per SM)
                        static int sms_w = 0;
                        if (!sms_w) cudaDeviceGetAttribute(&sms_w, cudaDevAttrMultiProcessorCount, 0);
                        if (!getenv("SB_LN_TWO_WAVES")) nblocks = std::min(nblocks, sms_w);
                        const int nb = nblocks;
                        k<<<nb, 512, sm2, s>>>((const T*)x, mean, rstd, (const T*)gamma, (const T*)g, (T*)gx, (T*)gres,
                                               gx_acc, rows, (int)n, s1, thr, dscale, keep, ws, ncol, gres_acc,
                                               (const T*)gext);
                        return nb;
                    };
                    if constexpr (CPL >= 8) {
                        // 2048-wide bf16 rows, one block per SM: the plain backward with 4 warps per
                        // row (35.0 us at 8192 rows), the fused one with 8 (41.3 us; 45.0 with 4,
                        // which spills) — ln_minb2.log, ln_wpr8.log
                        if (wpr_env == 8 || (wpr_env == 0 && mode == 1)) go(std::integral_constant<int, 8>{});
                        else go(std::integral_constant<int, 4>{});
                    } else {
                        // one 16-warp block per SM (<= 128 registers, no spills): the plain LayerNorm
                        // backward with 2 warps per row (41.2 -> 33.0 us at 16384 x 1024), the fused
                        // one with 4 (41.4 -> 37.1 us; at 2 it keeps more live state and spills) —
                        // profiles/r2/ln_wpr.log, ln_minb.log
                        if (wpr_env == 2 || (wpr_env == 0 && mode == 0)) go(std::integral_constant<int, 2>{});
                        else go(std::integral_constant<int, 4>{});
                    }
                    return;
                  }
                }
                if constexpr (CPL == 3) {
                    // 768-wide bf16 rows (T5-base): 3 warps per row (one chunk each), 15-warp
                    // blocks (5 rows), one per SM
                    if ((thr == 0 || keep) && !ln_narrow()) {
                        const size_t sm2 = (size_t)16 * ncol * (n / 3) * 4 + 2 * 16 * 2 * 4;
                        auto k = mode == 0 ? k_ln_bwd_w<T, 3, 0, 3> : k_ln_bwd_w<T, 3, 1, 3>;
                        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
                        static int sms_3 = 0;
                        if (!sms_3) cudaDeviceGetAttribute(&sms_3, cudaDevAttrMultiProcessorCount, 0);
                        if (!getenv("SB_LN_TWO_WAVES")) nblocks = std::min(nblocks, sms_3);
                        k<<<nblocks, 480, sm2, s>>>((const T*)x, mean, rstd, (const T*)gamma, (const T*)g, (T*)gx,
                                                    (T*)gres, gx_acc, rows, (int)n, s1, thr, dscale, keep, ws, ncol,
                                                    gres_acc, (const T*)gext);
                        return;
                    }
                }
                if (mode == 0) launch(k_ln_bwd_v<T, CPL, 0>);
                else launch(k_ln_bwd_v<T, CPL, 1>);
            });
        }
    });
    return ok;
}

}  // namespace sbk
