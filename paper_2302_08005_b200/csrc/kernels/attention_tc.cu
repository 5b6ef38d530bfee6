// Tensor-core flash attention (bf16 in, fp32 accumulate) for
// .replace(EfficientAttention), head_dim 64/128, S % 64 == 0.
//
// Forward: per (64-query block, head, batch) 4 warps x 16 query rows; K/V
// tiles of 64 keys double-buffered in swizzled shared memory via cp.async;
// S = Q K^T and O += P V on mma.sync m16n8k16 with P re-used from the S
// accumulator registers; online softmax in fp32; dropout from a precomputed
// 1-bit keep mask (same bits as the reference's counter RNG, kernels in
// elementwise.cu) so forward, backward and checkpoint recompute agree exactly.
// Backward (deterministic, no atomics): one kernel owns a 64-key block and
// sweeps all query blocks for dK/dV (computing S^T, dP^T directly), one owns a
// 64-query block and sweeps all key blocks for dQ.
#include "common.cuh"

namespace sbk {

namespace {

constexpr int TB = 64;  // rows per tile (queries or keys)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// tile [TB rows][D cols] bf16, 16-byte chunks XOR-swizzled by row so ldmatrix
// of 8 rows at one column hits 8 distinct bank groups.
template <int D>
__device__ __forceinline__ int swz(int row, int chunk) {
    return row * D + ((chunk ^ (row & 7)) << 3);
}

template <int D>
__device__ __forceinline__ void load_tile(bf16* sm, const bf16* g, long long ld, int tid, int nthreads) {
    constexpr int CH = D / 8;  // 16B chunks per row
    for (int e = tid; e < TB * CH; e += nthreads) {
        int r = e / CH, c = e % CH;
        cp_async16(sm + swz<D>(r, c), g + (long long)r * ld + c * 8);
    }
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const bf16* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(su32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const bf16* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(su32(p)));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *(uint32_t*)&v;
}

// A fragments (16 rows x D) of a swizzled row-major tile, rows r0..r0+15
template <int D>
__device__ __forceinline__ void load_a_frags(uint32_t (&a)[D / 16][4], const bf16* sm, int r0, int lane) {
#pragma unroll
    for (int k = 0; k < D / 16; ++k) {
        int row = r0 + (lane & 15), chunk = 2 * k + (lane >> 4);
        ldsm_x4(a[k], sm + swz<D>(row, chunk));
    }
}

// acc[n-tile][4] += A(16 x D, frags) * B where B(k=d, n=row of tile) = tile[n][d]
// (non-transposed: tile rows are the N dimension) — for S = Q K^T style products.
template <int D, int NT>
__device__ __forceinline__ void mma_abt(float (&acc)[NT][4], const uint32_t (&a)[D / 16][4], const bf16* tile, int lane) {
#pragma unroll
    for (int n2 = 0; n2 < NT / 2; ++n2) {  // two 8-wide n tiles per ldmatrix.x4
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
            uint32_t b[4];
            int row = n2 * 16 + (lane & 7) + ((lane >> 4) << 3), chunk = 2 * k + ((lane >> 3) & 1);
            ldsm_x4(b, tile + swz<D>(row, chunk));
            mma16816(acc[2 * n2], a[k], b[0], b[1]);
            mma16816(acc[2 * n2 + 1], a[k], b[2], b[3]);
        }
    }
}

// acc[d-tile][4] += P(16 x TB, as A frags from C layout) * tile where
// B(k=row of tile, n=d) = tile[k][d] (transposed ldmatrix) — for O += P V.
template <int D>
__device__ __forceinline__ void mma_pv(float (&acc)[D / 8][4], const float (&p)[TB / 8][4], const bf16* tile, int lane) {
#pragma unroll
    for (int ks = 0; ks < TB / 16; ++ks) {
        uint32_t a[4] = {pack2(p[2 * ks][0], p[2 * ks][1]), pack2(p[2 * ks][2], p[2 * ks][3]),
                         pack2(p[2 * ks + 1][0], p[2 * ks + 1][1]), pack2(p[2 * ks + 1][2], p[2 * ks + 1][3])};
#pragma unroll
        for (int n2 = 0; n2 < D / 16; ++n2) {
            uint32_t b[4];
            int row = ks * 16 + (lane & 7) + (((lane >> 3) & 1) << 3), chunk = 2 * n2 + (lane >> 4);
            ldsm_x4_t(b, tile + swz<D>(row, chunk));
            mma16816(acc[2 * n2], a, b[0], b[1]);
            mma16816(acc[2 * n2 + 1], a, b[2], b[3]);
        }
    }
}

struct MaskRef {
    const uint32_t* bits;  // keep bit of element ((bh*S + i)*S + j)
    long long S;
    float scale;  // 1/(1-p)
};
// keep bits of keys [j0, j0+64) for query row i (j0 % 64 == 0, S % 64 == 0: one aligned 64-bit word)
__device__ __forceinline__ uint64_t row_bits(const MaskRef& m, long long bh, long long i, long long j0) {
    long long e = (bh * m.S + i) * m.S + j0;
    return __ldg((const unsigned long long*)(m.bits + (e >> 5)));
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ------------------------------------------------------------------- forward
template <int D>
__global__ void __launch_bounds__(128, 4) k_fa_fwd(Attn a, MaskRef mk) {
    extern __shared__ __align__(128) bf16 fsm[];
    bf16* Qs = fsm;
    bf16* Ks = Qs + TB * D;     // 2 stages
    bf16* Vs = Ks + 2 * TB * D;  // 2 stages
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const long long b = blockIdx.z, h = blockIdx.y, q0 = (long long)blockIdx.x * TB;
    const long long bh = b * a.nh + h;
    const bf16* Q = (const bf16*)a.q + (b * a.S + q0) * a.ld_q + h * D;
    const bf16* Kg = (const bf16*)a.k + b * a.S * a.ld_k + h * D;
    const bf16* Vg = (const bf16*)a.v + b * a.S * a.ld_v + h * D;
    load_tile<D>(Qs, Q, a.ld_q, tid, 128);
    load_tile<D>(Ks, Kg, a.ld_k, tid, 128);
    load_tile<D>(Vs, Vg, a.ld_v, tid, 128);
    cp_commit();
    const float sl2 = a.scale * 1.4426950408889634f;  // exp(x) = exp2(x*log2e)
    float o[D / 8][4] = {};
    float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
    uint32_t qa[D / 16][4];
    const int nblk = a.causal ? (int)blockIdx.x + 1 : (int)(a.S / TB);  // causal: stop at the diagonal block
    const int g = lane >> 2, t = lane & 3;
    for (int jb = 0; jb < nblk; ++jb) {
        int st = jb & 1;
        if (jb + 1 < nblk) {
            load_tile<D>(Ks + (st ^ 1) * TB * D, Kg + (long long)(jb + 1) * TB * a.ld_k, a.ld_k, tid, 128);
            load_tile<D>(Vs + (st ^ 1) * TB * D, Vg + (long long)(jb + 1) * TB * a.ld_v, a.ld_v, tid, 128);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        if (jb == 0) load_a_frags<D>(qa, Qs, warp * 16, lane);
        float s[TB / 8][4] = {};
        mma_abt<D, TB / 8>(s, qa, Ks + st * TB * D, lane);
        if (a.causal && jb == (int)blockIdx.x) {  // diagonal block: key > query -> -inf (the diagonal stays)
#pragma unroll
            for (int n = 0; n < TB / 8; ++n)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (n * 8 + 2 * t + (e & 1) > warp * 16 + g + 8 * (e >> 1)) s[n][e] = -INFINITY;
        }
        // online softmax (rows g and g+8 of this warp's 16)
        float mx[2] = {m[0], m[1]};
#pragma unroll
        for (int n = 0; n < TB / 8; ++n) {
            mx[0] = fmaxf(mx[0], fmaxf(s[n][0], s[n][1]) * sl2);
            mx[1] = fmaxf(mx[1], fmaxf(s[n][2], s[n][3]) * sl2);
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
            mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
        }
        float corr[2] = {ex2(m[0] - mx[0]), ex2(m[1] - mx[1])};
        m[0] = mx[0];
        m[1] = mx[1];
        float rs[2] = {0.f, 0.f};
        const long long i0 = q0 + warp * 16 + g;
        uint64_t mb[2] = {~0ull, ~0ull};
        if (mk.bits) {
            mb[0] = row_bits(mk, bh, i0, (long long)jb * TB);
            mb[1] = row_bits(mk, bh, i0 + 8, (long long)jb * TB);
        }
#pragma unroll
        for (int n = 0; n < TB / 8; ++n) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                int r = e >> 1;
                float pv = ex2(s[n][e] * sl2 - m[r]);
                rs[r] += pv;  // the normaliser counts every probability (dropout acts after softmax)
                if (mk.bits) pv = ((mb[r] >> (n * 8 + 2 * t + (e & 1))) & 1) ? pv * mk.scale : 0.f;
                s[n][e] = pv;
            }
        }
        l[0] = l[0] * corr[0] + rs[0];
        l[1] = l[1] * corr[1] + rs[1];
#pragma unroll
        for (int n = 0; n < D / 8; ++n) {
            o[n][0] *= corr[0];
            o[n][1] *= corr[0];
            o[n][2] *= corr[1];
            o[n][3] *= corr[1];
        }
        mma_pv<D>(o, s, Vs + st * TB * D, lane);
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        l[r] += __shfl_xor_sync(0xffffffffu, l[r], 1);
        l[r] += __shfl_xor_sync(0xffffffffu, l[r], 2);
    }
    bf16* O = (bf16*)a.o + (b * a.S + q0 + warp * 16) * a.ld_o + h * D;
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            float inv = 1.f / l[r];
            *(uint32_t*)(O + (long long)(g + 8 * r) * a.ld_o + n * 8 + 2 * t) = pack2(o[n][2 * r] * inv, o[n][2 * r + 1] * inv);
        }
    }
    if (t == 0) {
#pragma unroll
        for (int r = 0; r < 2; ++r)
            a.lse[bh * a.S + q0 + warp * 16 + g + 8 * r] = (m[r] + log2f(l[r])) * 0.6931471805599453f;  // natural log
    }
}

// --------------------------------------------------------------- dK / dV
// Block owns 64 keys (4 warps x 16); sweeps query blocks. Per warp:
//   S^T = K Q^T, P^T = exp(S^T*scale - lse), dP^T = V dO^T,
//   dS^T = P^T (c dP^T - D), dV += (c P^T) dO, dK += dS^T Q  (c = keep/(1-p))
template <int D>
__global__ void __launch_bounds__(128) k_fa_dkdv(Attn a, MaskRef mk, const bf16* dO, long long ld_do, bf16* dk,
                                                 bf16* dv, long long ld_dk, long long ld_dv, const float* delta) {
    extern __shared__ __align__(128) bf16 bsm[];
    bf16* Ks = bsm;
    bf16* Vs = Ks + TB * D;
    bf16* Qs = Vs + TB * D;       // 2 stages
    bf16* Ds = Qs + 2 * TB * D;   // dO, 2 stages
    float* Ls = (float*)(Ds + 2 * TB * D);  // lse, 2 stages
    float* Es = Ls + 2 * TB;                // delta, 2 stages
    uint64_t* Ms = (uint64_t*)(Es + 2 * TB);  // keep bits of (query, this key block), 2 stages
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int g = lane >> 2, t = lane & 3;
    const long long b = blockIdx.z, h = blockIdx.y, k0 = (long long)blockIdx.x * TB;
    const long long bh = b * a.nh + h;
    const bf16* Kg = (const bf16*)a.k + (b * a.S + k0) * a.ld_k + h * D;
    const bf16* Vg = (const bf16*)a.v + (b * a.S + k0) * a.ld_v + h * D;
    const bf16* Qg = (const bf16*)a.q + b * a.S * a.ld_q + h * D;
    const bf16* Og = dO + b * a.S * ld_do + h * D;
    load_tile<D>(Ks, Kg, a.ld_k, tid, 128);
    load_tile<D>(Vs, Vg, a.ld_v, tid, 128);
    auto load_q = [&](int ib, int st) {
        load_tile<D>(Qs + st * TB * D, Qg + (long long)ib * TB * a.ld_q, a.ld_q, tid, 128);
        load_tile<D>(Ds + st * TB * D, Og + (long long)ib * TB * ld_do, ld_do, tid, 128);
        if (tid < TB) {
            Ls[st * TB + tid] = a.lse[bh * a.S + ib * TB + tid] * 1.4426950408889634f;
            Es[st * TB + tid] = delta[bh * a.S + ib * TB + tid];
            Ms[st * TB + tid] = mk.bits ? row_bits(mk, bh, (long long)ib * TB + tid, k0) : ~0ull;
        }
    };
    const int ib0 = a.causal ? (int)blockIdx.x : 0;  // causal: earlier query blocks see none of these keys
    load_q(ib0, ib0 & 1);
    cp_commit();
    cp_wait<0>();
    __syncthreads();
    uint32_t ka[D / 16][4], va[D / 16][4];
    load_a_frags<D>(ka, Ks, warp * 16, lane);
    load_a_frags<D>(va, Vs, warp * 16, lane);
    float gk[D / 8][4] = {}, gv[D / 8][4] = {};
    const float sl2 = a.scale * 1.4426950408889634f;
    const int nblk = (int)(a.S / TB);
    const long long j0 = k0 + warp * 16 + g;  // this thread's key rows: j0, j0+8
    for (int ib = ib0; ib < nblk; ++ib) {
        int st = ib & 1;
        if (ib + 1 < nblk) {
            __syncthreads();  // stage st^1 is free (consumed two iterations ago)
            load_q(ib + 1, st ^ 1);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const bf16* q = Qs + st * TB * D;
        const bf16* d = Ds + st * TB * D;
        float s[TB / 8][4] = {}, dp[TB / 8][4] = {};
        mma_abt<D, TB / 8>(s, ka, q, lane);   // S^T (keys x queries)
        mma_abt<D, TB / 8>(dp, va, d, lane);  // dP^T = V dO^T
#pragma unroll
        for (int n = 0; n < TB / 8; ++n) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                int qi = n * 8 + 2 * t + (e & 1);  // query within the block
                float p = ex2(s[n][e] * sl2 - Ls[st * TB + qi]);
                if (a.causal && ib == (int)blockIdx.x && warp * 16 + g + 8 * (e >> 1) > qi) p = 0.f;
                float c = mk.bits ? (((Ms[st * TB + qi] >> (warp * 16 + g + 8 * (e >> 1))) & 1) ? mk.scale : 0.f) : 1.f;
                float dsv = p * (c * dp[n][e] - Es[st * TB + qi]);
                s[n][e] = p * c;   // dropped probabilities for dV
                dp[n][e] = dsv;    // dS^T
            }
        }
        mma_pv<D>(gv, s, d, lane);   // dV += P^T dO
        mma_pv<D>(gk, dp, q, lane);  // dK += dS^T Q
    }
    // accumulate into the (strided) gradient views
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            long long row = b * a.S + j0 + 8 * r;
            __nv_bfloat162* pk = (__nv_bfloat162*)(dk + row * ld_dk + h * D + n * 8 + 2 * t);
            __nv_bfloat162* pv = (__nv_bfloat162*)(dv + row * ld_dv + h * D + n * 8 + 2 * t);
            float2 ok = (a.acc_mask & 2) ? __bfloat1622float2(*pk) : make_float2(0.f, 0.f);
            float2 ov = (a.acc_mask & 4) ? __bfloat1622float2(*pv) : make_float2(0.f, 0.f);
            *pk = __floats2bfloat162_rn(ok.x + a.scale * gk[n][2 * r], ok.y + a.scale * gk[n][2 * r + 1]);
            *pv = __floats2bfloat162_rn(ov.x + gv[n][2 * r], ov.y + gv[n][2 * r + 1]);
        }
    }
}

// -------------------------------------------------------------------- dQ
template <int D>
__global__ void __launch_bounds__(128) k_fa_dq(Attn a, MaskRef mk, const bf16* dO, long long ld_do, bf16* dq,
                                               long long ld_dq, const float* delta) {
    extern __shared__ __align__(128) bf16 qsm[];
    bf16* Qs = qsm;
    bf16* Ds = Qs + TB * D;
    bf16* Ks = Ds + TB * D;        // 2 stages
    bf16* Vs = Ks + 2 * TB * D;    // 2 stages
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int g = lane >> 2, t = lane & 3;
    const long long b = blockIdx.z, h = blockIdx.y, q0 = (long long)blockIdx.x * TB;
    const long long bh = b * a.nh + h;
    load_tile<D>(Qs, (const bf16*)a.q + (b * a.S + q0) * a.ld_q + h * D, a.ld_q, tid, 128);
    load_tile<D>(Ds, dO + (b * a.S + q0) * ld_do + h * D, ld_do, tid, 128);
    const bf16* Kg = (const bf16*)a.k + b * a.S * a.ld_k + h * D;
    const bf16* Vg = (const bf16*)a.v + b * a.S * a.ld_v + h * D;
    load_tile<D>(Ks, Kg, a.ld_k, tid, 128);
    load_tile<D>(Vs, Vg, a.ld_v, tid, 128);
    cp_commit();
    const long long i0 = q0 + warp * 16 + g;
    const float L2[2] = {a.lse[bh * a.S + i0] * 1.4426950408889634f, a.lse[bh * a.S + i0 + 8] * 1.4426950408889634f};
    const float E[2] = {delta[bh * a.S + i0], delta[bh * a.S + i0 + 8]};
    const float sl2 = a.scale * 1.4426950408889634f;
    uint32_t qa[D / 16][4], da[D / 16][4];
    float gq[D / 8][4] = {};
    const int nblk = a.causal ? (int)blockIdx.x + 1 : (int)(a.S / TB);
    for (int jb = 0; jb < nblk; ++jb) {
        int st = jb & 1;
        if (jb + 1 < nblk) {
            load_tile<D>(Ks + (st ^ 1) * TB * D, Kg + (long long)(jb + 1) * TB * a.ld_k, a.ld_k, tid, 128);
            load_tile<D>(Vs + (st ^ 1) * TB * D, Vg + (long long)(jb + 1) * TB * a.ld_v, a.ld_v, tid, 128);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        if (jb == 0) {
            load_a_frags<D>(qa, Qs, warp * 16, lane);
            load_a_frags<D>(da, Ds, warp * 16, lane);
        }
        const bf16* k = Ks + st * TB * D;
        float s[TB / 8][4] = {}, dp[TB / 8][4] = {};
        mma_abt<D, TB / 8>(s, qa, k, lane);
        mma_abt<D, TB / 8>(dp, da, Vs + st * TB * D, lane);
        uint64_t mb[2] = {~0ull, ~0ull};
        if (mk.bits) {
            mb[0] = row_bits(mk, bh, i0, (long long)jb * TB);
            mb[1] = row_bits(mk, bh, i0 + 8, (long long)jb * TB);
        }
#pragma unroll
        for (int n = 0; n < TB / 8; ++n) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                int r = e >> 1;
                float p = ex2(s[n][e] * sl2 - L2[r]);
                if (a.causal && jb == (int)blockIdx.x && n * 8 + 2 * t + (e & 1) > warp * 16 + g + 8 * r) p = 0.f;
                float c = mk.bits ? (((mb[r] >> (n * 8 + 2 * t + (e & 1))) & 1) ? mk.scale : 0.f) : 1.f;
                s[n][e] = p * (c * dp[n][e] - E[r]);  // dS
            }
        }
        mma_pv<D>(gq, s, k, lane);  // dQ += dS K
        __syncthreads();
    }
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            __nv_bfloat162* p = (__nv_bfloat162*)(dq + (b * a.S + i0 + 8 * r) * ld_dq + h * D + n * 8 + 2 * t);
            float2 ov = (a.acc_mask & 1) ? __bfloat1622float2(*p) : make_float2(0.f, 0.f);
            *p = __floats2bfloat162_rn(ov.x + a.scale * gq[n][2 * r], ov.y + a.scale * gq[n][2 * r + 1]);
        }
    }
}

bool fits(const Attn& a) {
    if (a.keys() != a.S) return false;  // (cross-attention: the SIMT and tcgen05 engines)
    if (a.t != BF16 || (a.hd != 64 && a.hd != 128) || a.S % TB || a.S < TB) return false;
    auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    if (!al(a.q) || !al(a.k) || !al(a.v) || !al(a.o)) return false;
    if (a.ld_q % 8 || a.ld_k % 8 || a.ld_v % 8 || a.ld_o % 8) return false;
    if (a.thr && !a.mask) return false;
    return true;
}

template <class K>
void smem_attr(K k, int bytes) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

}  // namespace

__global__ void k_fa_delta(const bf16* dout, long long ld_do, const bf16* o, long long ld_o, float* delta, long long B,
                           long long S, long long nh, long long hd) {
    long long w = blockIdx.x * 8 + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (w >= B * nh * S) return;
    long long i = w % S, h = (w / S) % nh, b = w / (S * nh);
    float acc = 0.f;
    for (long long d = lane * 2; d < hd; d += 64) {
        float2 x = __bfloat1622float2(*(const __nv_bfloat162*)(dout + (b * S + i) * ld_do + h * hd + d));
        float2 y = __bfloat1622float2(*(const __nv_bfloat162*)(o + (b * S + i) * ld_o + h * hd + d));
        acc += x.x * y.x + x.y * y.y;
    }
    acc = warp_sum(acc);
    if (lane == 0) delta[(b * nh + h) * S + i] = acc;
}

bool attn_fwd_tc_try(const Attn& a, cudaStream_t s) {
    if (!fits(a)) return false;
    MaskRef mk{a.thr ? a.mask : nullptr, a.S, a.dscale};
    dim3 grid((unsigned)(a.S / TB), (unsigned)a.nh, (unsigned)a.B);
    if (a.hd == 64) {
        int smem = 5 * TB * 64 * 2;
        smem_attr(k_fa_fwd<64>, smem);
        k_fa_fwd<64><<<grid, 128, smem, s>>>(a, mk);
    } else {
        int smem = 5 * TB * 128 * 2;
        smem_attr(k_fa_fwd<128>, smem);
        k_fa_fwd<128><<<grid, 128, smem, s>>>(a, mk);
    }
    SBK_CHECK_LAUNCH();
    return true;
}

bool attn_bwd_tc_try(const Attn& a, const void* dout, i64 ld_do, void* dq, void* dk, void* dv, i64 ld_dq, i64 ld_dk,
                     i64 ld_dv, float* delta, cudaStream_t s) {
    if (!fits(a)) return false;
    auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    if (!al(dout) || ld_do % 8 || ld_dq % 2 || ld_dk % 2 || ld_dv % 2) return false;
    MaskRef mk{a.thr ? a.mask : nullptr, a.S, a.dscale};
    long long rows = a.B * a.nh * a.S;
    k_fa_delta<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>((const bf16*)dout, ld_do, (const bf16*)a.o, a.ld_o, delta, a.B,
                                                          a.S, a.nh, a.hd);
    dim3 grid((unsigned)(a.S / TB), (unsigned)a.nh, (unsigned)a.B);
    auto go = [&](auto dc) {
        constexpr int D = decltype(dc)::value;
        int s1 = 6 * TB * D * 2 + 4 * TB * 4 + 2 * TB * 8, s2 = 6 * TB * D * 2;
        smem_attr(k_fa_dkdv<D>, s1);
        smem_attr(k_fa_dq<D>, s2);
        k_fa_dkdv<D><<<grid, 128, s1, s>>>(a, mk, (const bf16*)dout, ld_do, (bf16*)dk, (bf16*)dv, ld_dk, ld_dv, delta);
        k_fa_dq<D><<<grid, 128, s2, s>>>(a, mk, (const bf16*)dout, ld_do, (bf16*)dq, ld_dq, delta);
    };
    if (a.hd == 64) go(std::integral_constant<int, 64>{});
    else go(std::integral_constant<int, 128>{});
    SBK_CHECK_LAUNCH();
    return true;
}

}  // namespace sbk
