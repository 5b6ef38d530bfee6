// tcgen05 flash attention for .replace(EfficientAttention) (head_dim 64,
// S % 128 == 0): the reference's attention core (proj/src/library.cpp:9-34,
// executed as EfficientAttention at proj/src/executor.cpp:494-528) with the
// reference's counter-RNG dropout on the probabilities (executor.cpp:793-806)
// supplied as precomputed keep bits.
//
// Forward, one CTA per (batch, head, pair of 128-query tiles):
//   warp 0      TMA producer: Q tiles once, then 128-key K/V chunks through a
//               ring of NS stages (128B swizzle; q/k/v are column blocks of the
//               FusedQKV output, consumed in place through 2D tensor maps)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 4-7   softmax of query tile A, warps 8-11 of tile B (one thread per
//               query row = one TMEM lane)
// TMEM per tile (256 columns): S (128 fp32 cols), P (bf16 pairs, 64 cols), O
// (64 fp32 cols). S = Q K^T (SS MMA) -> softmax threads read S, write
// P = exp2(S*c - m) * keep as bf16 into TMEM -> O += P V (TS MMA, A from TMEM).
// The two tiles alternate so the tensor pipe computes one tile's S/PV while the
// other tile's softmax runs. The running max is rescaled lazily (only when it
// grows by more than 2^8), and O is touched only then; S(j+1)'s completion
// implies PV(j)'s (tcgen05.commit tracks every earlier MMA), so no extra wait.
#include "tc5.cuh"

namespace sbk {

using namespace tc5;

namespace {

constexpr int FD = 64;    // head dim
constexpr int FT = 128;   // rows per tile (queries / keys)
constexpr int FNS = 3;    // K/V ring stages
constexpr int F_TILE_BYTES = FT * FD * 2;  // 16 KB
constexpr int F_SMEM = 1024 + 2 * F_TILE_BYTES + FNS * 2 * F_TILE_BYTES + 256;

struct FwdArgs {
    bf16* o;
    long long ld_o;
    float* lse;
    const uint32_t* mask;  // keep bits or null
    float dscale;          // 1/(1-p)
    float c;               // scale * log2(e)
    int S, nh;
};

__global__ void __launch_bounds__(384, 1)
    k_fa5_fwd(const __grid_constant__ CUtensorMap tQ, const __grid_constant__ CUtensorMap tK,
              const __grid_constant__ CUtensorMap tV, FwdArgs fa) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sQ = smem;                        // [2][FT][FD]
    uint8_t* sK = sQ + 2 * F_TILE_BYTES;       // [FNS][FT][FD]
    uint8_t* sV = sK + FNS * F_TILE_BYTES;     // [FNS][FT][FD]
    uint64_t* bars = (uint64_t*)(sV + FNS * F_TILE_BYTES);
    uint64_t* q_full = bars;
    uint64_t* kv_full = q_full + 1;
    uint64_t* kv_empty = kv_full + FNS;
    uint64_t* s_full = kv_empty + FNS;  // [2]
    uint64_t* p_full = s_full + 2;      // [2]
    uint64_t* o_done = p_full + 2;      // [2]
    uint32_t* tslot = (uint32_t*)(o_done + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int S = fa.S, nj = S / FT;
    const int b = blockIdx.z, h = blockIdx.y;
    const int tile0 = blockIdx.x * 2;
    const int ntile = (tile0 + 1 < nj) ? 2 : 1;  // query tiles in this CTA
    const int row_base = b * S;                  // first token row of this sequence

    if (threadIdx.x == 0) {
        tma_prefetch(&tQ);
        tma_prefetch(&tK);
        tma_prefetch(&tV);
        mbar_init(q_full, 1);
        for (int s = 0; s < FNS; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        for (int g = 0; g < 2; ++g) {
            mbar_init(&s_full[g], 1);
            mbar_init(&p_full[g], 4);  // one arrival per softmax warp
            mbar_init(&o_done[g], 1);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(tslot);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ TMA producer
            mbar_expect_tx(q_full, ntile * F_TILE_BYTES);
            for (int g = 0; g < ntile; ++g)
                tma_load_2d(sQ + g * F_TILE_BYTES, &tQ, q_full, h * FD, row_base + (tile0 + g) * FT);
            for (int j = 0; j < nj; ++j) {
                const int s = j % FNS;
                mbar_wait(&kv_empty[s], ((j / FNS) & 1) ^ 1);
                mbar_expect_tx(&kv_full[s], 2 * F_TILE_BYTES);
                tma_load_2d(sK + s * F_TILE_BYTES, &tK, &kv_full[s], h * FD, row_base + j * FT);
                tma_load_2d(sV + s * F_TILE_BYTES, &tV, &kv_full[s], h * FD, row_base + j * FT);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------------------------ MMA issuer
            constexpr uint32_t id_s = idesc_bf16(FT, FT, false, false);  // S = Q K^T
            constexpr uint32_t id_o = idesc_bf16(FT, FD, false, true);   // O += P V (V MN-major)
            auto issue_s = [&](int g, int j) {
                const uint32_t a = smem_u32(sQ + g * F_TILE_BYTES), bk = smem_u32(sK + (j % FNS) * F_TILE_BYTES);
#pragma unroll
                for (int kk = 0; kk < FD / 16; ++kk)
                    mma_ss(tmem + g * 256, desc_kmajor(a, kk), desc_kmajor(bk, kk), id_s, kk > 0);
                mma_commit(&s_full[g]);
            };
            auto issue_pv = [&](int g, int j) {
                const uint32_t bv = smem_u32(sV + (j % FNS) * F_TILE_BYTES);
#pragma unroll
                for (int kk = 0; kk < FT / 16; ++kk)
                    mma_ts(tmem + g * 256 + 192, tmem + g * 256 + 128 + kk * 8, desc_mnmajor(bv, kk), id_o,
                           (j | kk) != 0);
                mma_commit(&o_done[g]);
            };
            mbar_wait(q_full, 0);
            mbar_wait(&kv_full[0], 0);
            fence_after();
            for (int g = 0; g < ntile; ++g) issue_s(g, 0);
            for (int j = 0; j < nj; ++j) {
                for (int g = 0; g < ntile; ++g) {
                    mbar_wait(&p_full[g], j & 1);
                    fence_after();
                    issue_pv(g, j);
                    if (j + 1 < nj) {
                        if (g == 0) {
                            mbar_wait(&kv_full[(j + 1) % FNS], ((j + 1) / FNS) & 1);
                            fence_after();
                        }
                        issue_s(g, j + 1);
                    }
                }
                mma_commit(&kv_empty[j % FNS]);  // K_j, V_j no longer read once these complete
            }
        }
    } else if (warp >= 4) {
        // ---------------------------------------------------- softmax
        const int g = (warp - 4) / 4, q = warp & 3;
        if (g < ntile) {
            const int row = q * 32 + lane;  // TMEM lane = query row within the tile
            const long long qi = (long long)(tile0 + g) * FT + row;
            const long long bh = (long long)b * fa.nh + h;
            const uint32_t t_row = tmem + ((uint32_t)(q * 32) << 16) + g * 256;
            const uint4* mrow = fa.mask ? (const uint4*)(fa.mask + ((bh * S + qi) * S >> 5)) : nullptr;
            float m_used = 0.f, l = 0.f;
            for (int j = 0; j < nj; ++j) {
                uint4 mw = make_uint4(~0u, ~0u, ~0u, ~0u);
                if (mrow) mw = __ldg(mrow + j);
                mbar_wait(&s_full[g], j & 1);
                fence_after();
                if (j == 0) {  // first chunk: exact row max (one extra TMEM read of S)
                    float mx = -INFINITY;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t s[32];
                        tmem_ld32_nowait(t_row + c * 32, s);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 32; ++e) mx = fmaxf(mx, __uint_as_float(s[e]));
                    }
                    m_used = mx * fa.c;
                }
                // P = exp2(S*c - m_used) * keep -> TMEM (bf16 pairs); returns this chunk's max of S
                auto pass = [&](float& lc) {
                    float mx = -INFINITY;
                    lc = 0.f;
#pragma unroll 1
                    for (int c = 0; c < 4; ++c) {
                        uint32_t s[32];
                        tmem_ld32_nowait(t_row + c * 32, s);
                        tmem_ld_wait();
                        const uint32_t mword = c == 0 ? mw.x : c == 1 ? mw.y : c == 2 ? mw.z : mw.w;
                        uint32_t pk[16];
#pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            const float s0 = __uint_as_float(s[2 * e]), s1 = __uint_as_float(s[2 * e + 1]);
                            mx = fmaxf(mx, fmaxf(s0, s1));
                            float p0 = ex2f(fmaf(s0, fa.c, -m_used));
                            float p1 = ex2f(fmaf(s1, fa.c, -m_used));
                            lc += p0 + p1;  // the normaliser counts every probability (dropout acts after softmax)
                            p0 = ((mword >> (2 * e)) & 1) ? p0 : 0.f;
                            p1 = ((mword >> (2 * e + 1)) & 1) ? p1 : 0.f;
                            pk[e] = pack_bf16(p0, p1);
                        }
                        tmem_st16(t_row + 128 + c * 16, pk);
                    }
                    return mx * fa.c;
                };
                float lc;
                const float mx = pass(lc);
                if (__any_sync(0xffffffffu, mx > m_used + 8.f)) {
                    // rare: the running max grew by > 2^8 -> rescale O (PV(j-1) is complete) and l, redo
                    const float m_new = fmaxf(m_used, mx);
                    const float f = ex2f(m_used - m_new);
                    l *= f;
                    m_used = m_new;
                    if (j > 0) {
#pragma unroll
                        for (int c = 0; c < 2; ++c) {
                            uint32_t o[32];
                            tmem_ld32_nowait(t_row + 192 + c * 32, o);
                            tmem_ld_wait();
#pragma unroll
                            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * f);
                            tmem_st32(t_row + 192 + c * 32, o);
                        }
                    }
                    tmem_st_wait();
                    pass(lc);
                }
                l += lc;
                tmem_st_wait();
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[g]);
            }
            // ------------------------------------------------ epilogue
            mbar_wait(&o_done[g], (nj - 1) & 1);
            fence_after();
            const float inv = fa.dscale / l;
            bf16* orow = fa.o + (long long)(row_base + qi) * fa.ld_o + (long long)h * FD;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                uint32_t o[32];
                tmem_ld32_nowait(t_row + 192 + c * 32, o);
                tmem_ld_wait();
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    uint4 w;
                    w.x = pack_bf16(__uint_as_float(o[8 * v + 0]) * inv, __uint_as_float(o[8 * v + 1]) * inv);
                    w.y = pack_bf16(__uint_as_float(o[8 * v + 2]) * inv, __uint_as_float(o[8 * v + 3]) * inv);
                    w.z = pack_bf16(__uint_as_float(o[8 * v + 4]) * inv, __uint_as_float(o[8 * v + 5]) * inv);
                    w.w = pack_bf16(__uint_as_float(o[8 * v + 6]) * inv, __uint_as_float(o[8 * v + 7]) * inv);
                    *(uint4*)(orow + c * 32 + v * 8) = w;
                }
            }
            fa.lse[bh * S + qi] = (m_used + __log2f(l)) * 0.6931471805599453f;  // natural log
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        tmem_dealloc<512>(tmem);
    }
}

bool fwd_fits(const Attn& a) {
    if (a.t != BF16 || a.hd != FD || a.S % FT || a.S < FT) return false;
    if (a.thr && !a.mask) return false;
    auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    if (!al(a.q) || !al(a.k) || !al(a.v) || !al(a.o) || a.ld_o % 8) return false;
    if (a.ld_q % 8 || a.ld_k % 8 || a.ld_v % 8) return false;
    if (a.B * a.S > (1ll << 31) || a.nh * FD > a.ld_q) return false;
    return true;
}

}  // namespace

bool attn_fwd_sm100_try(const Attn& a, cudaStream_t s) {
    if (!fwd_fits(a)) return false;
    CUtensorMap tq, tk, tv;
    const long long rows = a.B * a.S, cols = a.nh * FD;
    if (!make_map_bf16(&tq, a.q, cols, rows, a.ld_q, FT) || !make_map_bf16(&tk, a.k, cols, rows, a.ld_k, FT) ||
        !make_map_bf16(&tv, a.v, cols, rows, a.ld_v, FT))
        return false;
    FwdArgs fa{(bf16*)a.o, a.ld_o, a.lse, a.thr ? a.mask : nullptr, a.thr ? a.dscale : 1.f,
               a.scale * 1.4426950408889634f, (int)a.S, (int)a.nh};
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_fa5_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, F_SMEM);
        attr = true;
    }
    dim3 grid((unsigned)((a.S / FT + 1) / 2), (unsigned)a.nh, (unsigned)a.B);
    k_fa5_fwd<<<grid, 384, F_SMEM, s>>>(tq, tk, tv, fa);
    SBK_CHECK_LAUNCH();
    return true;
}

}  // namespace sbk
