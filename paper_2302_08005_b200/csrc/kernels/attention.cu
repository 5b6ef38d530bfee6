// Fused attention for .replace(EfficientAttention): S = scale*Q K^T, online
// softmax, counter-RNG dropout on the probabilities, O = P V — never
// materialising the (B, nh, S, S) scores. Same math as the reference graph
// (proj/src/library.cpp:9-34 evaluated by executor.cpp:494-528):
//   O_i = sum_j keep_ij/(1-p) * softmax(s_i)_j * v_j,
// dropout index ((b*nh + h)*S + i)*S + j (rank-local, executor.cpp:800-802).
// Backward recomputes P from the saved log-sum-exp:
//   D_i = dO_i . O_i ; dS_ij = P_ij (keep_ij/(1-p) dO_i.v_j - D_i)
//   dQ = scale dS K ; dK = scale dS^T Q ; dV = (P∘keep/(1-p))^T dO.
//
// This file holds the portable SIMT version (any head_dim <= 128, fp32 math),
// used for the parity path and as the GPU oracle of the tensor-core kernel.
#include "common.cuh"

namespace sbk {

bool attn_fwd_tc_try(const Attn& a, cudaStream_t s);  // attention_tc.cu (mma.sync)
bool attn_fwd_sm100_try(const Attn& a, cudaStream_t s);  // attention_sm100.cu (tcgen05)
bool attn_bwd_sm100_try(const Attn& a, const void* dout, i64 ld_do, void* dq, void* dk, void* dv, i64 ld_dq, i64 ld_dk,
                        i64 ld_dv, void* ws, cudaStream_t s);
size_t attn_bwd_sm100_workspace(i64 B, i64 S, i64 nh, i64 hd);
bool attn_bwd_tc_try(const Attn& a, const void* dout, i64 ld_do, void* dq, void* dk, void* dv, i64 ld_dq, i64 ld_dk,
                     i64 ld_dv, float* delta, cudaStream_t s);

namespace {
constexpr int kT = 64;  // rows per block / keys per tile

// the reference's flat index of probability (b, h, query i, key j) in a (B, nh, Sq, Sk) tensor
__device__ __forceinline__ uint64_t drop_index(i64 b, i64 h, i64 nh, i64 Sq, i64 Sk, i64 i, i64 j) {
    return (uint64_t)(((b * nh + h) * Sq + i) * Sk + j);
}

template <class T, int HD>
__global__ void __launch_bounds__(kT) k_attn_fwd(Attn a) {
    extern __shared__ float sm[];
    float* Ks = sm;                 // [kT][HD]
    float* Vs = Ks + kT * HD;       // [kT][HD]
    float* Ss = Vs + kT * HD;       // [kT threads][kT]
    const int hd = (int)a.hd;
    i64 b = blockIdx.z, h = blockIdx.y, i = (i64)blockIdx.x * kT + threadIdx.x;
    const i64 Sk = a.keys();
    const T* Q = (const T*)a.q;
    const T* Kg = (const T*)a.k;
    const T* Vg = (const T*)a.v;
    float q[HD], o[HD];
    bool valid = i < a.S;
#pragma unroll
    for (int d = 0; d < HD; ++d) {
        q[d] = (valid && d < hd) ? to_f(Q[(b * a.S + i) * a.ld_q + h * hd + d]) : 0.f;
        o[d] = 0.f;
    }
    float m = -INFINITY, l = 0.f;
    float* srow = Ss + threadIdx.x * kT;
    // causal: key tiles past this block's last query are fully masked
    const i64 jend = a.causal ? min(Sk, (i64)(blockIdx.x + 1) * kT) : Sk;
    for (i64 j0 = 0; j0 < jend; j0 += kT) {
        __syncthreads();
        for (int e = threadIdx.x; e < kT * HD; e += kT) {
            int jj = e / HD, d = e % HD;
            i64 j = j0 + jj;
            bool ok = j < Sk && d < hd;
            Ks[e] = ok ? to_f(Kg[(b * Sk + j) * a.ld_k + h * hd + d]) : 0.f;
            Vs[e] = ok ? to_f(Vg[(b * Sk + j) * a.ld_v + h * hd + d]) : 0.f;
        }
        __syncthreads();
        int nj = (int)min((i64)kT, Sk - j0);
        float tmax = -INFINITY;
        for (int jj = 0; jj < nj; ++jj) {
            float s = 0.f;
#pragma unroll
            for (int d = 0; d < HD; ++d) s = fmaf(q[d], Ks[jj * HD + d], s);
            s = (a.causal && j0 + jj > i) ? -INFINITY : s * a.scale;
            srow[jj] = s;
            tmax = fmaxf(tmax, s);
        }
        float mn = fmaxf(m, tmax);
        float corr = __expf(m - mn);
        l *= corr;
#pragma unroll
        for (int d = 0; d < HD; ++d) o[d] *= corr;
        for (int jj = 0; jj < nj; ++jj) {
            float p = __expf(srow[jj] - mn);
            l += p;
            if (a.thr && !d_keep(a.s1, drop_index(b, h, a.nh, a.S, Sk, i, j0 + jj), a.thr)) continue;
            float w = a.thr ? p * a.dscale : p;
#pragma unroll
            for (int d = 0; d < HD; ++d) o[d] = fmaf(w, Vs[jj * HD + d], o[d]);
        }
        m = mn;
    }
    if (!valid) return;
    T* O = (T*)a.o;
    float inv = 1.f / l;
    for (int d = 0; d < hd; ++d) O[(b * a.S + i) * a.ld_o + h * hd + d] = from_f<T>(o[d] * inv);
    a.lse[(b * a.nh + h) * a.S + i] = m + __logf(l);
}

template <class T>
__global__ void k_attn_delta(const T* dout, i64 ld_do, const T* o, i64 ld_o, float* delta, i64 B, i64 S, i64 nh, i64 hd) {
    i64 w = blockIdx.x * 8 + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (w >= B * nh * S) return;
    i64 i = w % S, h = (w / S) % nh, b = w / (S * nh);
    float acc = 0.f;
    for (i64 d = lane; d < hd; d += 32)
        acc += to_f(dout[(b * S + i) * ld_do + h * hd + d]) * to_f(o[(b * S + i) * ld_o + h * hd + d]);
    acc = warp_sum(acc);
    if (lane == 0) delta[(b * nh + h) * S + i] = acc;
}

// one thread per key j: dK_j, dV_j over all queries
template <class T, int HD>
__global__ void __launch_bounds__(kT) k_attn_dkdv(Attn a, const T* dout, i64 ld_do, T* dk, T* dv, i64 ld_dk, i64 ld_dv,
                                                  const float* delta) {
    extern __shared__ float sm[];
    float* Qs = sm;              // [kT][HD]
    float* Ds = Qs + kT * HD;    // dO tile
    float* Ls = Ds + kT * HD;    // lse
    float* Es = Ls + kT;         // delta
    const int hd = (int)a.hd;
    i64 b = blockIdx.z, h = blockIdx.y, j = (i64)blockIdx.x * kT + threadIdx.x;
    const i64 Sk = a.keys();
    bool valid = j < Sk;
    float k[HD], v[HD], gk[HD], gv[HD];
#pragma unroll
    for (int d = 0; d < HD; ++d) {
        k[d] = (valid && d < hd) ? to_f(((const T*)a.k)[(b * Sk + j) * a.ld_k + h * hd + d]) : 0.f;
        v[d] = (valid && d < hd) ? to_f(((const T*)a.v)[(b * Sk + j) * a.ld_v + h * hd + d]) : 0.f;
        gk[d] = gv[d] = 0.f;
    }
    // causal: query tiles before this key block see none of its keys
    for (i64 i0 = a.causal ? (i64)blockIdx.x * kT : 0; i0 < a.S; i0 += kT) {
        __syncthreads();
        for (int e = threadIdx.x; e < kT * HD; e += kT) {
            int ii = e / HD, d = e % HD;
            i64 i = i0 + ii;
            bool ok = i < a.S && d < hd;
            Qs[e] = ok ? to_f(((const T*)a.q)[(b * a.S + i) * a.ld_q + h * hd + d]) : 0.f;
            Ds[e] = ok ? to_f(dout[(b * a.S + i) * ld_do + h * hd + d]) : 0.f;
        }
        if (threadIdx.x < kT) {
            i64 i = i0 + threadIdx.x;
            Ls[threadIdx.x] = i < a.S ? a.lse[(b * a.nh + h) * a.S + i] : 0.f;
            Es[threadIdx.x] = i < a.S ? delta[(b * a.nh + h) * a.S + i] : 0.f;
        }
        __syncthreads();
        if (!valid) continue;
        int ni = (int)min((i64)kT, a.S - i0);
        for (int ii = 0; ii < ni; ++ii) {
            float s = 0.f, dpd = 0.f;
#pragma unroll
            for (int d = 0; d < HD; ++d) {
                s = fmaf(Qs[ii * HD + d], k[d], s);
                dpd = fmaf(Ds[ii * HD + d], v[d], dpd);
            }
            float p = (a.causal && j > i0 + ii) ? 0.f : __expf(s * a.scale - Ls[ii]);
            bool keep = !a.thr || d_keep(a.s1, drop_index(b, h, a.nh, a.S, Sk, i0 + ii, j), a.thr);
            float c = a.thr ? (keep ? a.dscale : 0.f) : 1.f;
            float pd = p * c;
            float ds = p * (c * dpd - Es[ii]);
#pragma unroll
            for (int d = 0; d < HD; ++d) {
                gv[d] = fmaf(pd, Ds[ii * HD + d], gv[d]);
                gk[d] = fmaf(ds, Qs[ii * HD + d], gk[d]);
            }
        }
    }
    if (!valid) return;
    for (int d = 0; d < hd; ++d) {
        i64 ik = (b * Sk + j) * ld_dk + h * hd + d, iv = (b * Sk + j) * ld_dv + h * hd + d;
        dk[ik] = from_f<T>(((a.acc_mask & 2) ? to_f(dk[ik]) : 0.f) + a.scale * gk[d]);
        dv[iv] = from_f<T>(((a.acc_mask & 4) ? to_f(dv[iv]) : 0.f) + gv[d]);
    }
}

// one thread per query i: dQ_i over all keys
template <class T, int HD>
__global__ void __launch_bounds__(kT) k_attn_dq(Attn a, const T* dout, i64 ld_do, T* dq, i64 ld_dq, const float* delta) {
    extern __shared__ float sm[];
    float* Ks = sm;
    float* Vs = Ks + kT * HD;
    const int hd = (int)a.hd;
    i64 b = blockIdx.z, h = blockIdx.y, i = (i64)blockIdx.x * kT + threadIdx.x;
    const i64 Sk = a.keys();
    bool valid = i < a.S;
    float q[HD], g[HD], gq[HD];
#pragma unroll
    for (int d = 0; d < HD; ++d) {
        q[d] = (valid && d < hd) ? to_f(((const T*)a.q)[(b * a.S + i) * a.ld_q + h * hd + d]) : 0.f;
        g[d] = (valid && d < hd) ? to_f(dout[(b * a.S + i) * ld_do + h * hd + d]) : 0.f;
        gq[d] = 0.f;
    }
    float L = valid ? a.lse[(b * a.nh + h) * a.S + i] : 0.f, E = valid ? delta[(b * a.nh + h) * a.S + i] : 0.f;
    const i64 jend = a.causal ? min(Sk, (i64)(blockIdx.x + 1) * kT) : Sk;
    for (i64 j0 = 0; j0 < jend; j0 += kT) {
        __syncthreads();
        for (int e = threadIdx.x; e < kT * HD; e += kT) {
            int jj = e / HD, d = e % HD;
            i64 j = j0 + jj;
            bool ok = j < Sk && d < hd;
            Ks[e] = ok ? to_f(((const T*)a.k)[(b * Sk + j) * a.ld_k + h * hd + d]) : 0.f;
            Vs[e] = ok ? to_f(((const T*)a.v)[(b * Sk + j) * a.ld_v + h * hd + d]) : 0.f;
        }
        __syncthreads();
        if (!valid) continue;
        int nj = (int)min((i64)kT, Sk - j0);
        for (int jj = 0; jj < nj; ++jj) {
            float s = 0.f, dpd = 0.f;
#pragma unroll
            for (int d = 0; d < HD; ++d) {
                s = fmaf(q[d], Ks[jj * HD + d], s);
                dpd = fmaf(g[d], Vs[jj * HD + d], dpd);
            }
            float p = (a.causal && j0 + jj > i) ? 0.f : __expf(s * a.scale - L);
            bool keep = !a.thr || d_keep(a.s1, drop_index(b, h, a.nh, a.S, Sk, i, j0 + jj), a.thr);
            float c = a.thr ? (keep ? a.dscale : 0.f) : 1.f;
            float ds = p * (c * dpd - E);
#pragma unroll
            for (int d = 0; d < HD; ++d) gq[d] = fmaf(ds, Ks[jj * HD + d], gq[d]);
        }
    }
    if (!valid) return;
    for (int d = 0; d < hd; ++d) {
        i64 k = (b * a.S + i) * ld_dq + h * hd + d;
        dq[k] = from_f<T>(((a.acc_mask & 1) ? to_f(dq[k]) : 0.f) + a.scale * gq[d]);
    }
}

template <int HD, class F>
void with_hd(i64 hd, F&& f) {
    if (hd <= 16) f(std::integral_constant<int, 16>{});
    else if (hd <= 32) f(std::integral_constant<int, 32>{});
    else if (hd <= 64) f(std::integral_constant<int, 64>{});
    else if (hd <= 128) f(std::integral_constant<int, 128>{});
    else throw std::runtime_error("attention: head_dim > 128 unsupported");
}

template <class K>
void smem_attr(K k, size_t bytes) {
    if (bytes > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}
}  // namespace

// engine selection: 0 = best available, 1 = at most mma.sync, 2 = SIMT only
int g_attn_max_engine = 0;
int g_attn_last_fwd = -1, g_attn_last_bwd = -1;  // 3 tcgen05, 2 mma.sync, 1 SIMT

void attn_set_engine(int e) { g_attn_max_engine = e; }

size_t attn_bwd_workspace(i64 B, i64 S, i64 nh, i64 hd) {
    return std::max((size_t)(B * nh * S) * 4, attn_bwd_sm100_workspace(B, S, nh, hd));
}
int attn_last_engine(int bwd) { return bwd ? g_attn_last_bwd : g_attn_last_fwd; }

void attn_fwd(const Attn& a, cudaStream_t s) {
    if (a.causal && a.keys() != a.S) throw std::runtime_error("attention: causal needs as many keys as queries");
    if (g_attn_max_engine == 0 && attn_fwd_sm100_try(a, s)) {
        g_attn_last_fwd = 3;
        return;
    }
    if (g_attn_max_engine <= 1 && attn_fwd_tc_try(a, s)) {
        g_attn_last_fwd = 2;
        return;
    }
    g_attn_last_fwd = 1;
    dim3 grid((unsigned)((a.S + kT - 1) / kT), (unsigned)a.nh, (unsigned)a.B);
    dispatch(a.t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        if constexpr (!std::is_same_v<T, double>) {
            with_hd<0>(a.hd, [&](auto hdc) {
                constexpr int HD = decltype(hdc)::value;
                size_t smem = (size_t)(2 * kT * HD + kT * kT) * 4;
                auto k = k_attn_fwd<T, HD>;
                smem_attr(k, smem);
                k<<<grid, kT, smem, s>>>(a);
            });
        } else {
            throw std::runtime_error("attention: f64 unsupported");
        }
    });
    SBK_CHECK_LAUNCH();
}

void attn_bwd(const Attn& a, const void* dout, i64 ld_do, void* dq, void* dk, void* dv, i64 ld_dq, i64 ld_dk, i64 ld_dv,
              void* ws, cudaStream_t s) {
    if (a.causal && a.keys() != a.S) throw std::runtime_error("attention: causal needs as many keys as queries");
    float* delta = (float*)ws;
    if (g_attn_max_engine == 0 && attn_bwd_sm100_try(a, dout, ld_do, dq, dk, dv, ld_dq, ld_dk, ld_dv, ws, s)) {
        g_attn_last_bwd = 3;
        return;
    }
    if (g_attn_max_engine <= 1 && attn_bwd_tc_try(a, dout, ld_do, dq, dk, dv, ld_dq, ld_dk, ld_dv, delta, s)) {
        g_attn_last_bwd = 2;
        return;
    }
    g_attn_last_bwd = 1;
    dim3 grid((unsigned)((a.S + kT - 1) / kT), (unsigned)a.nh, (unsigned)a.B);
    dispatch(a.t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        if constexpr (!std::is_same_v<T, double>) {
            i64 rows = a.B * a.nh * a.S;
            k_attn_delta<T><<<(unsigned)((rows + 7) / 8), 256, 0, s>>>((const T*)dout, ld_do, (const T*)a.o, a.ld_o, delta,
                                                                       a.B, a.S, a.nh, a.hd);
            with_hd<0>(a.hd, [&](auto hdc) {
                constexpr int HD = decltype(hdc)::value;
                size_t s1 = (size_t)(2 * kT * HD + 2 * kT) * 4, s2 = (size_t)(2 * kT * HD) * 4;
                auto k1 = k_attn_dkdv<T, HD>;
                auto k2 = k_attn_dq<T, HD>;
                smem_attr(k1, s1);
                smem_attr(k2, s2);
                const dim3 gk((unsigned)((a.keys() + kT - 1) / kT), (unsigned)a.nh, (unsigned)a.B);  // one thread per key
                k1<<<gk, kT, s1, s>>>(a, (const T*)dout, ld_do, (T*)dk, (T*)dv, ld_dk, ld_dv, delta);
                k2<<<grid, kT, s2, s>>>(a, (const T*)dout, ld_do, (T*)dq, ld_dq, delta);
            });
        } else {
            throw std::runtime_error("attention: f64 unsupported");
        }
    });
    SBK_CHECK_LAUNCH();
}

}  // namespace sbk
