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

// MODE 0: LayerNorm backward (gx += ...). MODE 1: fused bias+dropout+residual+LN
// backward: g_sum = LNbwd(g); gres += g_sum; gx (=g_partial) (+)= dropout_bwd(g_sum);
// NCOL column partials (dgamma, dbeta[, dbias]) -> ws[block][k*n + col].
template <class T, int CPL, int MODE>
__global__ void __launch_bounds__(32 * kW, 1)
    k_ln_bwd_v(const T* x, const float* mean, const float* rstd, const T* gamma, const T* g, T* gx, T* gres, bool gx_acc,
               i64 rows, int n, uint64_t s1, uint64_t thr, float dscale, const uint32_t* keep, float* ws, int ncol,
               bool gres_acc) {
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
                k_bdrln_fwd_v<T, decltype(cc)::value><<<(unsigned)((rows + kW - 1) / kW), 32 * kW, 0, s>>>(
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
                const uint32_t* keep, float* ws, int ncol, int nblocks, cudaStream_t s) {
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
                                                     ncol, gres_acc);
                };
                if (mode == 0) launch(k_ln_bwd_v<T, CPL, 0>);
                else launch(k_ln_bwd_v<T, CPL, 1>);
            });
        }
    });
    return ok;
}

}  // namespace sbk
