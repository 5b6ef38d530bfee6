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
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <type_traits>

#include "tc5.cuh"

namespace sbk {

using namespace tc5;

namespace {

constexpr int FD = 64;    // head dim
constexpr int FT = 128;   // rows per tile (queries / keys)
constexpr int F_TILE_BYTES = FT * FD * 2;  // 16 KB
// NT query tiles per CTA: 2 (one CTA per SM, the tiles ping-pong) or 1 (two CTAs
// per SM, each with half the TMEM, overlapping each other's prologue/epilogue)
template <int NT>
struct FCfg {
    static constexpr int NS = NT == 2 ? 3 : 2;  // K/V ring stages
    static constexpr int THREADS = (4 + 4 * NT) * 32;
    static constexpr uint32_t TCOLS = NT == 2 ? 512 : 256;
    static constexpr int SMEM = 1024 + NT * F_TILE_BYTES + NS * 2 * F_TILE_BYTES + NS * NT * 2048 + 256;
};

struct FwdArgs {
    bf16* o;
    long long ld_o;
    float* lse;
    const uint32_t* mask;  // keep bits or null
    float dscale;          // 1/(1-p)
    float c;               // scale * log2(e)
    int S, nh;
    int dbg;               // debugging switches (SB_ATTN_DBG): 1 skip softmax math, 4 skip MMAs
    int Sk = 0;            // keys per sequence (cross-attention, k_fa6_fwd<false, D> only); 0: S
};

template <int NT>
__global__ void __launch_bounds__(FCfg<NT>::THREADS, NT == 1 ? 2 : 1)
    k_fa5_fwd(const __grid_constant__ CUtensorMap tQ, const __grid_constant__ CUtensorMap tK,
              const __grid_constant__ CUtensorMap tV, const __grid_constant__ CUtensorMap tM, FwdArgs fa) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-aligned, derived from smem_raw by pointer arithmetic so accesses stay ld/st.shared
    uint8_t* smem = smem_raw + ((1024 - (tc5::smem_u32(smem_raw) & 1023)) & 1023);
    constexpr int FNS = FCfg<NT>::NS;
    uint8_t* sQ = smem;                        // [NT][FT][FD]
    uint8_t* sK = sQ + NT * F_TILE_BYTES;      // [FNS][FT][FD]
    uint8_t* sV = sK + FNS * F_TILE_BYTES;     // [FNS][FT][FD]
    uint8_t* sM = sV + FNS * F_TILE_BYTES;     // [FNS][NT tiles][128 rows][4 words] keep bits
    uint64_t* bars = (uint64_t*)(sM + FNS * NT * 2048);
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
    const int tile0 = blockIdx.x * NT;
    const int ntile = (NT == 2 && tile0 + 1 < nj) ? 2 : 1;  // query tiles in this CTA
    const int row_base = b * S;                  // first token row of this sequence

    if (threadIdx.x == 0) {
        tma_prefetch(&tQ);
        tma_prefetch(&tK);
        tma_prefetch(&tV);
        if (fa.mask) tma_prefetch(&tM);
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
    if (warp == 1) tmem_alloc<FCfg<NT>::TCOLS>(tslot);
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
                mbar_expect_tx(&kv_full[s], 2 * F_TILE_BYTES + (fa.mask ? ntile * 2048 : 0));
                tma_load_2d(sK + s * F_TILE_BYTES, &tK, &kv_full[s], h * FD, row_base + j * FT);
                tma_load_2d(sV + s * F_TILE_BYTES, &tV, &kv_full[s], h * FD, row_base + j * FT);
                if (fa.mask)  // keep bits of (query rows of each tile, key chunk j)
                    for (int g = 0; g < ntile; ++g)
                        tma_load_2d(sM + (s * NT + g) * 2048, &tM, &kv_full[s], j * (FT / 32),
                                    (b * fa.nh + h) * S + (tile0 + g) * FT);
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
            float m_used = 0.f, l = 0.f;
            for (int j = 0; j < nj; ++j) {
                mbar_wait(&kv_full[j % FNS], (j / FNS) & 1);  // keep bits of chunk j landed
                mbar_wait(&s_full[g], j & 1);
                fence_after();
                const uint4 mw = fa.mask ? *(const uint4*)(sM + ((j % FNS) * NT + g) * 2048 + row * 16)
                                         : make_uint4(~0u, ~0u, ~0u, ~0u);
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
        tmem_dealloc<FCfg<NT>::TCOLS>(tmem);
    }
}

// Forward with 64-key chunks, four persistent CTAs per SM, each walking 128-query
// tiles (tile t = (b*nh + h)*S/128 + q-tile, grid-strided):
//   warps 0-3   softmax (thread = query row = TMEM lane) + the tile epilogue
//   warp 4      TMA producer: Q per tile (Q buffer released by the tile's last
//               S MMA), K/V chunks of 64 keys through a 2-stage ring
//   warp 5      TMEM allocator (128 columns) + tcgen05.mma issuer
// TMEM: S [0,64) fp32, overwritten in place by P (bf16 pairs, [0,32)) as the
// softmax consumes it; O [64,128). Per chunk: S = Q K^T -> softmax -> O += P V.
// S(j+1) is issued right after PV(j), which reads P(j) from the same columns
// (in-order tcgen05.mma execution); the next tile's first S overlaps this
// tile's epilogue, and its first PV waits until the epilogue has read O.
// Keep bits are read per row from the natural-layout mask one chunk ahead.
// Head dim D = 64 or 128 (template): a D = 128 row is two 64-column (128-byte)
// swizzle panels, each its own TMA box; S = Q K^T takes its 8 K16 steps across
// both panels, O += P V is one M128 N128 MMA per K16 step (the two V panels are
// the two MN atoms of the B descriptor, LBO = one panel). TMEM S [0,64) + O
// [64, 64 + D): 128 columns (four CTAs per SM) at D = 64, 256 (two) at D = 128 —
// at D = 128 the chunk's MMA time (512 cycles) matches its exp2 time.
constexpr int KC6 = 64;                      // keys per chunk
constexpr int F6_NS = 2;                     // K/V stages
constexpr int F6_THREADS = 192;
constexpr int F6_MASK_BYTES = 2048;         // keep bits of 128 query rows x 128 keys (two chunks)
#ifndef F6_CTAS
#define F6_CTAS 4  // resident CTAs per SM (head dim 64)
#endif
#ifndef F6_QBUF
#define F6_QBUF 1  // Q tile buffers (2: the next tile's Q loads while this tile runs)
#endif
#ifndef F6_ONEPASS
// S read from TMEM once (64 registers per row: max, then exp2 from registers) instead of
// twice: 0 never, 1 always, 2 for causal tiles and head dim 128 (fa_ab.log: 67.9 -> 64.0 us
// causal hd 128, 57.7 -> 56.3 us causal hd 64; the non-causal hd-64 tile runs 68.1 -> 70.5)
#define F6_ONEPASS 2
#endif
template <int D>
struct F6 {
    static constexpr int PANELS = D / 64;
    static constexpr int Q_BYTES = FT * D * 2;      // 16 / 32 KB
    static constexpr int KV_BYTES = KC6 * D * 2;    // 8 / 16 KB
    static constexpr int Q_PANEL = FT * 128, KV_PANEL = KC6 * 128;
    static constexpr int CTAS = D == 64 ? F6_CTAS : 2;
    static constexpr uint32_t TCOLS = D == 64 ? 128 : 256;
    static constexpr int SMEM = 1024 + F6_QBUF * Q_BYTES + F6_NS * 2 * KV_BYTES + 2 * F6_MASK_BYTES + 160;
};
constexpr int F6_KV_BYTES = F6<64>::KV_BYTES;
constexpr int F6_SMEM = F6<64>::SMEM;
constexpr float kLazy6 = 8.f;                // lazy rescale threshold (log2 units)

template <bool CAUSAL, int D = 64>
__global__ void __launch_bounds__(F6_THREADS, F6<D>::CTAS)
    k_fa6_fwd(const __grid_constant__ CUtensorMap tQ, const __grid_constant__ CUtensorMap tK,
              const __grid_constant__ CUtensorMap tV, const __grid_constant__ CUtensorMap tM, FwdArgs fa,
              int ntiles) {
    using C = F6<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (tc5::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* sQ = smem;                          // [F6_QBUF][panel][FT][64]
    uint8_t* sK = sQ + F6_QBUF * C::Q_BYTES;     // [F6_NS][panel][KC6][64]
    uint8_t* sV = sK + F6_NS * C::KV_BYTES;      // [F6_NS][panel][KC6][64]
    uint8_t* sMk = sV + F6_NS * C::KV_BYTES;     // [2][128 rows][4 words]: keep bits of a chunk pair
    uint64_t* bars = (uint64_t*)(sMk + 2 * F6_MASK_BYTES);
    uint64_t* q_full = bars;                // [F6_QBUF]
    uint64_t* q_empty = q_full + F6_QBUF;   // [F6_QBUF]
    uint64_t* kv_full = q_empty + F6_QBUF;  // [F6_NS]
    uint64_t* kv_empty = kv_full + F6_NS;   // [F6_NS]
    uint64_t* s_full = kv_empty + F6_NS;
    uint64_t* p_full = s_full + 1;
    uint64_t* o_done = p_full + 1;
    uint64_t* o_free = o_done + 1;          // epilogue has read O (4 softmax warps)
    uint64_t* m_full = o_free + 1;          // [2] keep bits of a chunk pair landed
    uint64_t* m_empty = m_full + 2;         // [2] the 4 softmax warps have read them
    uint32_t* tslot = (uint32_t*)(m_empty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int S = fa.S, Sk = fa.Sk ? fa.Sk : S, nj = Sk / KC6, nq = S / FT, nbh = ntiles / nq;
    // causal tiles differ in length (q-tile i has i+1 128-key spans), so they are walked
    // heaviest q-tile first — the grid-stride walk then balances instead of handing every
    // CTA the same q-tile (gridDim % nq == 0)
    auto tile_qt = [&](int t) { return CAUSAL ? nq - 1 - t / nbh : t % nq; };
    auto tile_bh = [&](int t) { return CAUSAL ? t % nbh : t / nq; };

    if (threadIdx.x == 0) {
        for (int x = 0; x < F6_QBUF; ++x) {
            mbar_init(&q_full[x], 1);
            mbar_init(&q_empty[x], 1);
        }
        for (int s = 0; s < F6_NS; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(p_full, 4);
        mbar_init(o_done, 1);
        mbar_init(o_free, 4);
        for (int x = 0; x < 2; ++x) {
            mbar_init(&m_full[x], 1);
            mbar_init(&m_empty[x], 4);
        }
        fence_barrier_init();
    }
    if (warp == 5) tmem_alloc<C::TCOLS>(tslot);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tslot;

    if (warp == 4) {
        if (lane == 0) {
            // ------------------------------------------------ TMA producer
            int u = 0, n = 0, pp = 0;  // chunks / tiles / keep-bit chunk pairs loaded by this CTA
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++n) {
                const int bh = tile_bh(t), b = bh / fa.nh, h = bh % fa.nh;
                const int row_base = b * S, kv_base = b * Sk;  // (query rows / key rows)
                const int qb = n % F6_QBUF;
                mbar_wait(&q_empty[qb], ((n / F6_QBUF) & 1) ^ 1);
                mbar_expect_tx(&q_full[qb], C::Q_BYTES);
#pragma unroll
                for (int pn = 0; pn < C::PANELS; ++pn)
                    tma_load_2d(sQ + qb * C::Q_BYTES + pn * C::Q_PANEL, &tQ, &q_full[qb], h * D + 64 * pn,
                                row_base + tile_qt(t) * FT);
                const int njt = CAUSAL ? (tile_qt(t) + 1) * (FT / KC6) : nj;  // causal: up to the diagonal
                for (int j = 0; j < njt; ++j, ++u) {
                    const int s = u % F6_NS;
                    if (fa.mask && (j & 1) == 0) {  // keep bits of chunks j, j+1 for the tile's 128 rows
                        const int ms = pp & 1;
                        mbar_wait(&m_empty[ms], ((pp >> 1) & 1) ^ 1);
                        mbar_expect_tx(&m_full[ms], F6_MASK_BYTES);
                        tma_load_2d(sMk + ms * F6_MASK_BYTES, &tM, &m_full[ms], j * (KC6 / 32),
                                    (b * fa.nh + h) * S + tile_qt(t) * FT);
                        ++pp;
                    }
                    mbar_wait(&kv_empty[s], ((u / F6_NS) & 1) ^ 1);
                    if (fa.dbg & 8) {  // debugging: no K/V traffic
                        mbar_arrive(&kv_full[s]);
                        continue;
                    }
                    mbar_expect_tx(&kv_full[s], 2 * C::KV_BYTES);
#pragma unroll
                    for (int pn = 0; pn < C::PANELS; ++pn) {
                        tma_load_2d(sK + s * C::KV_BYTES + pn * C::KV_PANEL, &tK, &kv_full[s], h * D + 64 * pn,
                                    kv_base + j * KC6);
                        tma_load_2d(sV + s * C::KV_BYTES + pn * C::KV_PANEL, &tV, &kv_full[s], h * D + 64 * pn,
                                    kv_base + j * KC6);
                    }
                }
            }
        }
    } else if (warp == 5) {
        // ------------------------------------------------ MMA issuer (whole warp, one elected
        // lane issues: descriptors in uniform registers, no per-MMA divergence loop)
        constexpr uint32_t id_s = idesc_bf16(FT, KC6, false, false);  // S = Q K^T
        constexpr uint32_t id_o = idesc_bf16(FT, D, false, true);     // O += P V (V MN-major)
        const uint32_t a0 = smem_u32(sQ), k0 = smem_u32(sK), v0 = smem_u32(sV);
        int u = 0, n = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++n) {
            const int qb = n % F6_QBUF;
            const uint32_t aq = a0 + qb * C::Q_BYTES;
            mbar_wait(&q_full[qb], (n / F6_QBUF) & 1);
            const int njt = CAUSAL ? (tile_qt(t) + 1) * (FT / KC6) : nj;
            for (int j = 0; j < njt; ++j, ++u) {
                const int s = u % F6_NS;
                mbar_wait(&kv_full[s], (u / F6_NS) & 1);
                fence_after();
                // S(j) overwrites P(j-1) in TMEM: tcgen05.mma executes in issue order, so
                // PV(j-1) (issued first) has read it (the CUTLASS Blackwell FMHA relies on the same)
                if (!(fa.dbg & 4)) {
                    const uint32_t ak = k0 + s * C::KV_BYTES;
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk)  // K16 step kk: panel kk / 4, 32-byte column kk % 4
                        mma_ss_w(tmem, desc_kmajor(aq + (kk >> 2) * C::Q_PANEL, kk & 3),
                                 desc_kmajor(ak + (kk >> 2) * C::KV_PANEL, kk & 3), id_s, kk);
                }
                mma_commit_w(s_full);
                if (j == njt - 1) mma_commit_w(&q_empty[qb]);  // last read of this tile's Q
                if (j == 0 && n > 0) mbar_wait(o_free, (n - 1) & 1);  // previous epilogue read O
                mbar_wait(p_full, u & 1);
                fence_after();
                if (!(fa.dbg & 4)) {
                    // (desc_mnmajor's LBO is 8 KB = one V panel: the second 64 columns of N)
                    static_assert(C::KV_PANEL == 8192, "V panel must match desc_mnmajor's LBO");
                    const uint64_t dv = desc_mnmajor(v0 + s * C::KV_BYTES, 0);
#pragma unroll
                    for (int kk = 0; kk < KC6 / 16; ++kk) mma_ts_w(tmem + 64, tmem + kk * 8, dv + 128 * kk, id_o, j | kk);
                }
                mma_commit_w(o_done);
                mma_commit_w(&kv_empty[s]);
            }
        }
    } else {
        // ---------------------------------------------------- softmax (warps 0-3)
        const int row = warp * 32 + lane;
        const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);
        int u = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const long long bh = tile_bh(t);
            const long long qi = (long long)tile_qt(t) * FT + row;
            const int b = (int)(bh / fa.nh), h = (int)(bh % fa.nh);
            float m_used = 0.f, l = 0.f;
            const int njt = CAUSAL ? (tile_qt(t) + 1) * (FT / KC6) : nj;
            for (int j = 0; j < njt; ++j, ++u) {
                // causal: in the diagonal chunks, keys past this row's query are masked (-inf);
                // key 0 <= every query, so chunk 0 always sets a finite running max
                const int kmax = CAUSAL ? (int)(qi - (long long)j * KC6) : KC6;  // keys [0, kmax] of the chunk kept
                // keep bits of chunk j (chunk pair u / 2 of this CTA's walk, staged by TMA)
                uint2 mw = make_uint2(~0u, ~0u);
                if (fa.mask) {
                    const int pr = u >> 1, ms = pr & 1;
                    mbar_wait(&m_full[ms], (pr >> 1) & 1);
                    mw = *(const uint2*)(sMk + ms * F6_MASK_BYTES + row * 16 + (j & 1) * 8);
                }
                mbar_wait(s_full, u & 1);
                fence_after();
                if (fa.dbg & 1) {
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive(p_full);
                        if (fa.mask && (j & 1)) mbar_arrive(&m_empty[(u >> 1) & 1]);
                    }
                    l = 1.f;
                    continue;
                }
                // pass 1: row max of S (P overwrites S in place, so the max comes first)
                float mx = -INFINITY;
                constexpr bool ONEPASS = F6_ONEPASS == 1 || (F6_ONEPASS == 2 && (CAUSAL || D == 128));
                uint32_t s0[32], s1[32];
                if constexpr (ONEPASS) {
                    tmem_ld32_nowait(t_row, s0);
                    tmem_ld32_nowait(t_row + 32, s1);
                    tmem_ld_wait();
                    if (kmax < KC6 - 1) {
#pragma unroll
                        for (int e = 0; e < 32; ++e) {
                            if (e > kmax) s0[e] = __float_as_uint(-INFINITY);
                            if (32 + e > kmax) s1[e] = __float_as_uint(-INFINITY);
                        }
                    }
#pragma unroll
                    for (int e = 0; e < 32; e += 2) {
                        mx = fmax3(mx, __uint_as_float(s0[e]), __uint_as_float(s0[e + 1]));
                        mx = fmax3(mx, __uint_as_float(s1[e]), __uint_as_float(s1[e + 1]));
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        uint32_t sv[32];
                        tmem_ld32_nowait(t_row + c * 32, sv);
                        tmem_ld_wait();
                        if (kmax < KC6 - 1) {
#pragma unroll
                            for (int e = 0; e < 32; ++e)
                                if (c * 32 + e > kmax) sv[e] = __float_as_uint(-INFINITY);
                        }
#pragma unroll
                        for (int e = 0; e < 32; e += 2) mx = fmax3(mx, __uint_as_float(sv[e]), __uint_as_float(sv[e + 1]));
                    }
                }
                mx *= fa.c;
                if (j == 0) m_used = mx;
                // rare: the running max grew by > 2^kLazy6 -> rescale l now and O once P is out
                // (S(j) completing implies PV(j-1) did: in-order MMAs, so O is final until PV(j))
                float f_res = 0.f;
                const bool rescale = __any_sync(0xffffffffu, mx > m_used + kLazy6);
                if (rescale) {
                    const float m_new = fmaxf(m_used, mx);
                    f_res = ex2f(m_used - m_new);
                    l *= f_res;
                    m_used = m_new;
                }
                // pass 2: P = exp2(S*c - m_used) * keep -> TMEM (bf16 pairs over S's first 32 columns)
                float2 lc2 = make_float2(0.f, 0.f);
                const float2 c2 = make_float2(fa.c, fa.c), nm2 = make_float2(-m_used, -m_used);
                // 32 columns of S (registers) -> P bf16 pairs -> TMEM columns [c * 16, c * 16 + 16)
                auto p_half = [&](const uint32_t(&sv)[32], uint32_t mword, int c) {
                    uint32_t pk[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) {  // element pairs on the packed-fp32 pipe
                        const float2 a =
                            ffma2(make_float2(__uint_as_float(sv[2 * e]), __uint_as_float(sv[2 * e + 1])), c2, nm2);
                        float2 p = make_float2(ex2f(a.x), ex2f(a.y));
                        lc2 = fadd2(lc2, p);  // the normaliser counts every probability (dropout acts after softmax)
                        p.x = ((mword >> (2 * e)) & 1) ? p.x : 0.f;
                        p.y = ((mword >> (2 * e + 1)) & 1) ? p.y : 0.f;
                        pk[e] = pack_bf16(p.x, p.y);
                    }
                    tmem_st16(t_row + c * 16, pk);
                };
                if constexpr (ONEPASS) {
                    p_half(s0, mw.x, 0);
                    p_half(s1, mw.y, 1);
                } else {
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        uint32_t sv[32];
                        tmem_ld32_nowait(t_row + c * 32, sv);
                        tmem_ld_wait();
                        if (kmax < KC6 - 1) {
#pragma unroll
                            for (int e = 0; e < 32; ++e)
                                if (c * 32 + e > kmax) sv[e] = __float_as_uint(-INFINITY);
                        }
                        p_half(sv, c == 0 ? mw.x : mw.y, c);
                    }
                }
                l += lc2.x + lc2.y;
                if (rescale) {
                    mbar_wait(o_done, (u - 1) & 1);
                    fence_after();
#pragma unroll
                    for (int c = 0; c < D / 32; ++c) {
                        uint32_t o[32];
                        tmem_ld32_nowait(t_row + 64 + c * 32, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * f_res);
                        tmem_st32(t_row + 64 + c * 32, o);
                    }
                }
                tmem_st_wait();
                fence_before();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(p_full);
                    if (fa.mask && (j & 1)) {  // this warp is done with the chunk pair's keep bits
                        fence_proxy_async();
                        mbar_arrive(&m_empty[(u >> 1) & 1]);
                    }
                }
            }
            // ------------------------------------------------ epilogue
            mbar_wait(o_done, (u - 1) & 1);
            fence_after();
            const float inv = fa.dscale / l;
            bf16* orow = fa.o + (long long)(b * S + qi) * fa.ld_o + (long long)h * D;
#pragma unroll
            for (int half = 0; half < D / 64; ++half) {  // 64 columns of O at a time (registers)
                uint32_t o[2][32];
                tmem_ld32_nowait(t_row + 64 + half * 64, o[0]);
                tmem_ld32_nowait(t_row + 96 + half * 64, o[1]);
                tmem_ld_wait();
                if (half == D / 64 - 1) {
                    fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(o_free);  // O may be overwritten by the next tile's PV
                }
#pragma unroll
                for (int c = 0; c < 2; ++c)
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        uint4 w;
                        w.x = pack_bf16(__uint_as_float(o[c][8 * v + 0]) * inv, __uint_as_float(o[c][8 * v + 1]) * inv);
                        w.y = pack_bf16(__uint_as_float(o[c][8 * v + 2]) * inv, __uint_as_float(o[c][8 * v + 3]) * inv);
                        w.z = pack_bf16(__uint_as_float(o[c][8 * v + 4]) * inv, __uint_as_float(o[c][8 * v + 5]) * inv);
                        w.w = pack_bf16(__uint_as_float(o[c][8 * v + 6]) * inv, __uint_as_float(o[c][8 * v + 7]) * inv);
                        *(uint4*)(orow + half * 64 + c * 32 + v * 8) = w;
                    }
            }
            fa.lse[bh * S + qi] = (m_used + __log2f(l)) * 0.6931471805599453f;  // natural log
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 5) {
        fence_after();
        tmem_dealloc<C::TCOLS>(tmem);
    }
}

bool fwd_fits(const Attn& a, int hd = FD) {
    // cross-attention (keys != queries): non-causal, whole 128-key blocks
    if (a.keys() != a.S && (a.causal || a.keys() % FT || a.keys() < FT)) return false;
    if (a.t != BF16 || a.hd != hd || a.S % FT || a.S < FT) return false;
    if (a.thr && !a.mask) return false;
    auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    if (!al(a.q) || !al(a.k) || !al(a.v) || !al(a.o) || a.ld_o % 8) return false;
    if (a.ld_q % 8 || a.ld_k % 8 || a.ld_v % 8) return false;
    if (a.B * a.S > (1ll << 31) || a.nh * hd > a.ld_q) return false;
    return true;
}

// ------------------------------------------------------------------ backward
// One CTA per (batch, head), sweeping key blocks j (outer) and query blocks i
// (inner) — the reference's attention backward (executor.cpp:1257-1378) as the
// flash-attention recurrence. Per (j, i):
//   S^T  = K_j Q_i^T            (SS MMA, TMEM [0,128))
//   dP^T = V_j dO_i^T           (SS MMA, TMEM [128,256))
//   8 softmax warps (thread = key row, half the query columns each):
//     P^T = exp2(S^T c - lse2_q), Z^T = keep/(1-p) P^T -> TMEM [448,512) (bf16 pairs),
//     dS^T = P^T (keep/(1-p) dP^T - delta_q) -> shared memory (bf16, 128B swizzle, 2 buffers)
//   dV_j += Z^T dO_i            (TS MMA, A from TMEM, TMEM [256,320))
//   dK_j += dS^T Q_i            (SS MMA, dS^T read K-major, TMEM [320,384))
//   dQ_ij = dS K_j              (SS MMA, the same dS^T bytes read MN-major, TMEM [384,448))
// The MMA issue order per step is dV, dK, S/dP of the next step, dQ, so the
// next softmax starts while dQ is computed. 4 dQ warps (thread = query row)
// drain dQ_ij from TMEM and add it into this CTA's private fp32 accumulator
// (j = 0 stores, the last j writes bf16): dQ needs no cross-CTA reduction, so
// the backward is deterministic without atomics or inter-CTA waits. dK_j / dV_j
// are drained by the softmax warps while block j+1 starts.
// delta_q = dO_q . O_q and lse2 = lse * log2(e) come from k_fa5_prep.
constexpr int B_STAGE = 2 * F_TILE_BYTES + 1024 + 2048;  // Q, dO, lse2[128], delta[128], keep bits [128][4]
constexpr int B_NST = 3;  // Q / dO / lse / delta / keep-bit stages
constexpr int B_SMEM = 1024 + 2 * F_TILE_BYTES + B_NST * B_STAGE + 4 * F_TILE_BYTES + 12 * 2048 + 256;

struct BwdArgs {
    const float* lse2;
    const float* delta;
    float* dqacc;
    const uint32_t* mask_t;
    float dscale, c, scale;
    bf16* dq;
    bf16* dk;
    bf16* dv;
    long long ld_dq, ld_dk, ld_dv;
    int S, nh, acc;
    int dbg;  // debugging switches (SB_ATTN_DBG): 1 skip softmax math, 2 skip dQ accumulation, 4 skip MMAs
    unsigned long long* ts;  // debugging timeline (SB_ATTN_TS): [role][event], CTA (0,0) only
    int Sk = 0;  // keys per sequence (cross-attention, non-causal k_fa7_bwd / k_fa8_bwd); 0: S
};
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// delta = rowsum(dO * O) and lse2 = lse * log2(e); D/8 threads per (b, h, query) row
template <int D = FD>
__global__ void k_fa5_prep(const bf16* dout, long long ld_do, const bf16* o, long long ld_o, const float* lse,
                           float* lse2, float* delta, long long BH, int S, int nh, float sgn) {
    constexpr int TPR = D / 8;
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long idx = tid / TPR;
    const int part = (int)(tid % TPR);
    const bool ok = idx < BH * S;
    float acc = 0.f;
    if (ok) {
        const long long bh = idx / S, q = idx % S, b = bh / nh, h = bh % nh;
        const uint4 a = *((const uint4*)(dout + (b * S + q) * ld_do + h * D) + part);
        const uint4 c = *((const uint4*)(o + (b * S + q) * ld_o + h * D) + part);
        const __nv_bfloat162* pa = (const __nv_bfloat162*)&a;
        const __nv_bfloat162* pc = (const __nv_bfloat162*)&c;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            float2 fa = __bfloat1622float2(pa[t]), fc = __bfloat1622float2(pc[t]);
            acc = fmaf(fa.x, fc.x, fmaf(fa.y, fc.y, acc));
        }
    }
#pragma unroll
    for (int m = 1; m < TPR; m <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if (ok && part == 0) {
        delta[idx] = sgn * acc;
        lse2[idx] = sgn * lse[idx] * 1.4426950408889634f;
    }
}

__device__ __forceinline__ uint64_t desc_kmajor_2blk(uint32_t base, int kk) {
    // K-major tile of 128 rows x 128 bf16 stored as two 64-column blocks of 16 KB
    return sdesc(base + (kk >> 2) * 16384 + (kk & 3) * 32, 1, 1024 >> 4);
}

__device__ __forceinline__ void store_bf16x8(bf16* dst, const float (&f)[8], bool acc) {
    float g[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) g[t] = f[t];
    uint4* d = (uint4*)dst;
    if (acc) {
        uint4 old = *d;
        const __nv_bfloat162* po = (const __nv_bfloat162*)&old;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            float2 x = __bfloat1622float2(po[t]);
            g[2 * t] += x.x;
            g[2 * t + 1] += x.y;
        }
    }
    *d = make_uint4(pack_bf16(g[0], g[1]), pack_bf16(g[2], g[3]), pack_bf16(g[4], g[5]), pack_bf16(g[6], g[7]));
}

// A warp writes 32 rows (thread = row, 64 fp32 values each) as bf16 (x scale,
// += the existing values when acc) with coalesced 128-byte rows: 8 rows at a
// time go through a 2 KB fp32 staging buffer (16-byte units XOR-swizzled by
// row), then each store instruction covers 4 full rows.
__device__ __forceinline__ void warp_rows_out(float* stage, bf16* dst0, long long ld, const float (&f)[64], float sc,
                                              bool acc, int lane) {
    uint4* st4 = (uint4*)stage;
    const int c = lane & 7;
    // accumulate mode: the 8 old 16-byte chunks this lane will update, loaded up front (one latency)
    uint4 old[8];
    if (acc) {
#pragma unroll
        for (int q = 0; q < 8; ++q) old[q] = *(const uint4*)(dst0 + (long long)(q * 4 + (lane >> 3)) * ld + c * 8);
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        if ((lane >> 3) == p) {
            const int rr = lane & 7;
#pragma unroll
            for (int u = 0; u < 16; ++u)
                st4[rr * 16 + (u ^ rr)] = make_uint4(__float_as_uint(f[4 * u]), __float_as_uint(f[4 * u + 1]),
                                                     __float_as_uint(f[4 * u + 2]), __float_as_uint(f[4 * u + 3]));
        }
        __syncwarp();
#pragma unroll
        for (int it = 0; it < 2; ++it) {
            const int rr = it * 4 + (lane >> 3);
            const uint4 a = st4[rr * 16 + ((2 * c) ^ rr)], b = st4[rr * 16 + ((2 * c + 1) ^ rr)];
            float g[8] = {__uint_as_float(a.x) * sc, __uint_as_float(a.y) * sc, __uint_as_float(a.z) * sc,
                          __uint_as_float(a.w) * sc, __uint_as_float(b.x) * sc, __uint_as_float(b.y) * sc,
                          __uint_as_float(b.z) * sc, __uint_as_float(b.w) * sc};
            if (acc) {
                const __nv_bfloat162* po = (const __nv_bfloat162*)&old[p * 2 + it];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    float2 x = __bfloat1622float2(po[t]);
                    g[2 * t] += x.x;
                    g[2 * t + 1] += x.y;
                }
            }
            *(uint4*)(dst0 + (long long)(p * 8 + rr) * ld + c * 8) =
                make_uint4(pack_bf16(g[0], g[1]), pack_bf16(g[2], g[3]), pack_bf16(g[4], g[5]), pack_bf16(g[6], g[7]));
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(512, 1)
    k_fa5_bwd(const __grid_constant__ CUtensorMap tK, const __grid_constant__ CUtensorMap tV,
              const __grid_constant__ CUtensorMap tQ, const __grid_constant__ CUtensorMap tdO,
              const __grid_constant__ CUtensorMap tM, BwdArgs ba) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-aligned, derived from smem_raw by pointer arithmetic so accesses stay ld/st.shared
    uint8_t* smem = smem_raw + ((1024 - (tc5::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* sKV = smem;                        // {K, V} of the current key block
    uint8_t* sStage = sKV + 2 * F_TILE_BYTES;   // [B_NST][B_STAGE]
    uint8_t* sDS = sStage + B_NST * B_STAGE;    // [2] x dS^T [2 q-blocks][128 keys][64 q] bf16, swizzled
    float* sOut = (float*)(sDS + 4 * F_TILE_BYTES);  // [12 warps][2 KB] output staging
    uint64_t* bars = (uint64_t*)(sDS + 4 * F_TILE_BYTES + 12 * 2048);
    uint64_t* kv_full = bars;
    uint64_t* kv_empty = bars + 1;
    uint64_t* st_full = bars + 2;              // [B_NST]
    uint64_t* st_empty = st_full + B_NST;      // [B_NST]
    uint64_t* sdp_full = st_empty + B_NST;     // [2 query halves]
    uint64_t* sm_done = sdp_full + 2;          // [2 query halves]
    uint64_t* dq_full = sm_done + 2;
    uint64_t* dq_free = dq_full + 1;
    uint64_t* acc_full = dq_free + 1;  // dK_j / dV_j complete
    uint64_t* acc_free = acc_full + 1;  // dK_j / dV_j read out of TMEM
    uint32_t* tslot = (uint32_t*)(acc_free + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int S = ba.S, nj = S / FT, nsteps = nj * nj;
    const int h = blockIdx.x, b = blockIdx.y;
    const long long bh = (long long)b * ba.nh + h;
    const int row_base = b * S;

    if (threadIdx.x == 0) {
        tma_prefetch(&tK);
        tma_prefetch(&tV);
        tma_prefetch(&tQ);
        tma_prefetch(&tdO);
        if (ba.mask_t) tma_prefetch(&tM);
        mbar_init(kv_full, 1);
        mbar_init(kv_empty, 1);
        for (int s = 0; s < B_NST; ++s) {
            mbar_init(&st_full[s], 1);
            mbar_init(&st_empty[s], 1);
        }
        for (int hh = 0; hh < 2; ++hh) {
            mbar_init(&sdp_full[hh], 1);
            mbar_init(&sm_done[hh], 8);
        }
        mbar_init(dq_full, 1);
        mbar_init(dq_free, 4);
        mbar_init(acc_full, 1);
        mbar_init(acc_free, 8);
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
            for (int u = 0; u < nsteps; ++u) {
                const int j = u / nj, i = u % nj;
                if (i == 0) {  // single K/V buffer: block j after the last reader of block j-1
                    mbar_wait(kv_empty, (j & 1) ^ 1);
                    mbar_expect_tx(kv_full, 2 * F_TILE_BYTES);
                    tma_load_2d(sKV, &tK, kv_full, h * FD, row_base + j * FT);
                    tma_load_2d(sKV + F_TILE_BYTES, &tV, kv_full, h * FD, row_base + j * FT);
                }
                const int s = u % B_NST;
                uint8_t* st = sStage + s * B_STAGE;
                mbar_wait(&st_empty[s], ((u / B_NST) & 1) ^ 1);
                if (ba.ts && blockIdx.x == 0 && blockIdx.y == 0) ba.ts[0 * 64 + u] = gtime();
                mbar_expect_tx(&st_full[s], 2 * F_TILE_BYTES + 1024 + (ba.mask_t ? 2048 : 0));
                tma_load_2d(st, &tQ, &st_full[s], h * FD, row_base + i * FT);
                tma_load_2d(st + F_TILE_BYTES, &tdO, &st_full[s], h * FD, row_base + i * FT);
                bulk_load(st + 2 * F_TILE_BYTES, ba.lse2 + bh * S + i * FT, 512, &st_full[s]);
                bulk_load(st + 2 * F_TILE_BYTES + 512, ba.delta + bh * S + i * FT, 512, &st_full[s]);
                // transposed keep bits of (key rows of block j, query block i): [128 keys][4 words]
                if (ba.mask_t)
                    tma_load_2d(st + 2 * F_TILE_BYTES + 1024, &tM, &st_full[s], i * (FT / 32), (int)(bh * S) + j * FT);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------------------------ MMA issuer
            // Each step's 128 query columns are two halves: while the softmax
            // warps work on half b of step u, the tensor pipe runs dV/dK of half
            // a and S/dP of half a of step u+1, and vice versa.
            constexpr uint32_t id_s = idesc_bf16(FT, FT / 2, false, false);
            constexpr uint32_t id_kv = idesc_bf16(FT, FD, false, true);
            constexpr uint32_t id_q = idesc_bf16(FT, FD, true, true);
            const bool mm = !(ba.dbg & 4);
            auto issue_sdp = [&](int u, int hh) {
                const int j = u / nj, i = u % nj, s = u % B_NST;
                const uint32_t aK = smem_u32(sKV), aV = aK + F_TILE_BYTES;
                const uint32_t aQ = smem_u32(sStage + s * B_STAGE) + hh * (F_TILE_BYTES / 2), adO = aQ + F_TILE_BYTES;
                if (hh == 0) {
                    if (i == 0) mbar_wait(kv_full, j & 1);
                    mbar_wait(&st_full[s], (u / B_NST) & 1);
                    fence_after();
                }
                if (mm) {
#pragma unroll
                    for (int kk = 0; kk < FD / 16; ++kk)  // S^T half = K Q_half^T
                        mma_ss(tmem + hh * 64, desc_kmajor(aK, kk), desc_kmajor(aQ, kk), id_s, kk > 0);
#pragma unroll
                    for (int kk = 0; kk < FD / 16; ++kk)  // dP^T half = V dO_half^T
                        mma_ss(tmem + 128 + hh * 64, desc_kmajor(aV, kk), desc_kmajor(adO, kk), id_s, kk > 0);
                }
                mma_commit(&sdp_full[hh]);
            };
            issue_sdp(0, 0);
            issue_sdp(0, 1);
            for (int u = 0; u < nsteps; ++u) {
                const int j = u / nj, i = u % nj, s = u % B_NST;
                const uint32_t aK = smem_u32(sKV);
                const uint32_t aQ = smem_u32(sStage + s * B_STAGE), adO = aQ + F_TILE_BYTES;
                const uint32_t aDS = smem_u32(sDS + (u & 1) * 2 * F_TILE_BYTES);
#pragma unroll 1
                for (int hh = 0; hh < 2; ++hh) {
                    mbar_wait(&sm_done[hh], u & 1);
                    if (hh == 0 && i == 0 && j > 0) mbar_wait(acc_free, (j - 1) & 1);  // dK/dV of block j-1 drained
                    if (ba.ts && blockIdx.x == 0 && blockIdx.y == 0 && hh == 1) ba.ts[1 * 64 + u] = gtime();
                    fence_after();
                    if (mm) {
#pragma unroll
                        for (int k4 = 0; k4 < 4; ++k4) {  // dV += Z^T_half dO_half
                            const int kk = hh * 4 + k4;
                            mma_ts(tmem + 256, tmem + 448 + kk * 8, desc_mnmajor(adO, kk), id_kv, (i | kk) != 0);
                        }
#pragma unroll
                        for (int k4 = 0; k4 < 4; ++k4) {  // dK += dS^T_half Q_half
                            const int kk = hh * 4 + k4;
                            mma_ss(tmem + 320, desc_kmajor_2blk(aDS, kk), desc_mnmajor(aQ, kk), id_kv, (i | kk) != 0);
                        }
                    }
                    if (hh == 1) {
                        mma_commit(&st_empty[s]);  // Q, dO, lse, delta, keep bits of this step are no longer read
                        if (i == nj - 1) mma_commit(acc_full);
                    }
                    // (at the last query block of key block j, S/dP of block j+1 need its
                    // K/V, loaded into the single K/V buffer only after dQ below releases K_j)
                    if (u + 1 < nsteps && i != nj - 1) issue_sdp(u + 1, hh);
                }
                if (ba.ts && blockIdx.x == 0 && blockIdx.y == 0) ba.ts[2 * 64 + u] = gtime();
                if (u > 0) {
                    mbar_wait(dq_free, (u - 1) & 1);  // dQ of the previous step has left TMEM
                    fence_after();
                }
                if (ba.ts && blockIdx.x == 0 && blockIdx.y == 0) ba.ts[3 * 64 + u] = gtime();
                if (mm) {
#pragma unroll
                    for (int kk = 0; kk < FT / 16; ++kk)  // dQ_ij = dS K
                        mma_ss(tmem + 384, sdesc(aDS + kk * 2048, 16384 >> 4, 1024 >> 4), desc_mnmajor(aK, kk), id_q,
                               kk > 0);
                }
                mma_commit(dq_full);
                if (i == nj - 1) {
                    mma_commit(kv_empty);  // K_j, V_j no longer read
                    if (u + 1 < nsteps) {
                        issue_sdp(u + 1, 0);
                        issue_sdp(u + 1, 1);
                    }
                }
            }
        }
    } else if (warp >= 4 && warp < 12) {
        // ------------------------------------------------------------------
        // 8 softmax warps: quarter q4 = TMEM lanes (key rows), half hf = 64 of
        // the 128 query columns
        const int q4 = warp & 3, hf = (warp - 4) >> 2, k = q4 * 32 + lane;
        const uint32_t t_lane = tmem + ((uint32_t)(q4 * 32) << 16);
        // dK_j (hf 1) / dV_j (hf 0) -> global
        float* my_stage = sOut + (warp - 4) * 512;
        auto drain_kv = [&](int j) {
            mbar_wait(acc_full, j & 1);
            fence_after();
            float f[64];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                uint32_t r[32];
                tmem_ld32_nowait(t_lane + 256 + hf * 64 + hh * 32, r);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; ++e) f[hh * 32 + e] = __uint_as_float(r[e]);
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_free);
            const long long kg0 = (long long)j * FT + q4 * 32;  // first key row of this warp
            if (hf)
                warp_rows_out(my_stage, ba.dk + (row_base + kg0) * ba.ld_dk + (long long)h * FD, ba.ld_dk, f, ba.scale,
                              ba.acc & 2, lane);
            else
                warp_rows_out(my_stage, ba.dv + (row_base + kg0) * ba.ld_dv + (long long)h * FD, ba.ld_dv, f, 1.f,
                              ba.acc & 4, lane);
        };
        const int g = hf;  // 32-column group of each query half
        for (int u = 0; u < nsteps; ++u) {
            const int j = u / nj, i = u % nj, s = u % B_NST;
            if (i == 0 && j > 0) drain_kv(j - 1);  // TMEM dK/dV free before dV/dK of block j start
            const float* lse_s = (const float*)(sStage + s * B_STAGE + 2 * F_TILE_BYTES);
            const float* dl_s = lse_s + FT;
            uint8_t* ds_buf = sDS + (u & 1) * 2 * F_TILE_BYTES;
            mbar_wait(&st_full[s], (u / B_NST) & 1);
            const uint4 mw = ba.mask_t ? *(const uint4*)(sStage + s * B_STAGE + 2 * F_TILE_BYTES + 1024 + k * 16)
                                       : make_uint4(~0u, ~0u, ~0u, ~0u);
#pragma unroll 1
            for (int hh = 0; hh < 2; ++hh) {
                const int c = hh * 2 + g;  // 32-query chunk
                mbar_wait(&sdp_full[hh], u & 1);
                fence_after();
                if (ba.ts && blockIdx.x == 0 && blockIdx.y == 0 && warp == 4 && lane == 0 && hh == 0)
                    ba.ts[4 * 64 + u] = gtime();
                if (!(ba.dbg & 1)) {
                    uint32_t sv[32], dp[32];
                    tmem_ld32_nowait(t_lane + c * 32, sv);
                    tmem_ld32_nowait(t_lane + 128 + c * 32, dp);
                    tmem_ld_wait();
                    const uint32_t mword = c == 0 ? mw.x : c == 1 ? mw.y : c == 2 ? mw.z : mw.w;
                    uint32_t zk[16], dk[16];
#pragma unroll
                    for (int e4 = 0; e4 < 8; ++e4) {
                        const float4 l4 = *(const float4*)(lse_s + c * 32 + e4 * 4);
                        const float4 d4 = *(const float4*)(dl_s + c * 32 + e4 * 4);
                        const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dv[4] = {d4.x, d4.y, d4.z, d4.w};
                        float z[4], ds[4];
#pragma unroll
                        for (int e1 = 0; e1 < 4; ++e1) {
                            const int e = e4 * 4 + e1;
                            const float p = ex2f(fmaf(__uint_as_float(sv[e]), ba.c, -lv[e1]));
                            const float kd = ((mword >> e) & 1) ? ba.dscale : 0.f;
                            z[e1] = p * kd;
                            ds[e1] = p * fmaf(kd, __uint_as_float(dp[e]), -dv[e1]);
                        }
                        zk[2 * e4] = pack_bf16(z[0], z[1]);
                        zk[2 * e4 + 1] = pack_bf16(z[2], z[3]);
                        dk[2 * e4] = pack_bf16(ds[0], ds[1]);
                        dk[2 * e4 + 1] = pack_bf16(ds[2], ds[3]);
                    }
                    tmem_st16(t_lane + 448 + c * 16, zk);
                    // dS^T row k, queries c*32..c*32+31: q-block c/2 (= hh), 16-byte chunks (c%2)*4 + v
                    uint8_t* rowp = ds_buf + hh * 16384 + k * 128;
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const int ch = ((c & 1) * 4 + v) ^ (k & 7);
                        *(uint4*)(rowp + ch * 16) = make_uint4(dk[4 * v], dk[4 * v + 1], dk[4 * v + 2], dk[4 * v + 3]);
                    }
                    tmem_st_wait();
                }
                fence_proxy_async();
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm_done[hh]);
            }
            if (ba.ts && blockIdx.x == 0 && blockIdx.y == 0 && warp == 4 && lane == 0) ba.ts[5 * 64 + u] = gtime();
        }
        drain_kv(nj - 1);
    } else if (warp >= 12) {
        // ---------------------------------------------------- dQ warps (thread = query row)
        const int q4 = warp & 3, r = q4 * 32 + lane;
        const uint32_t t_row = tmem + ((uint32_t)(q4 * 32) << 16) + 384;
        for (int u = 0; u < nsteps; ++u) {
            const int j = u / nj, i = u % nj;
            // private fp32 accumulator, thread-major: float4 v of query row r of
            // block i at ((bh*nj + i)*16 + v)*128 + r, so a warp's accesses coalesce
            float4* acc = (float4*)ba.dqacc + ((bh * nj + i) * 16) * FT + r;
            float f[64];
            if (j > 0 && !(ba.dbg & 2)) {  // this thread's own partial sum (written by it at step u - nj)
#pragma unroll
                for (int v = 0; v < 16; ++v) {
                    const float4 a4 = __ldcg(acc + v * FT);
                    f[4 * v] = a4.x;
                    f[4 * v + 1] = a4.y;
                    f[4 * v + 2] = a4.z;
                    f[4 * v + 3] = a4.w;
                }
            } else {
#pragma unroll
                for (int e = 0; e < 64; ++e) f[e] = 0.f;
            }
            mbar_wait(dq_full, u & 1);
            fence_after();
            if (ba.ts && blockIdx.x == 0 && blockIdx.y == 0 && warp == 12 && lane == 0) ba.ts[6 * 64 + u] = gtime();
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                uint32_t d[32];
                tmem_ld32_nowait(t_row + hh * 32, d);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; ++e) f[hh * 32 + e] += __uint_as_float(d[e]);
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(dq_free);
            if (ba.dbg & 2) continue;
            if (j == nj - 1) {
                const long long q0 = (long long)i * FT + q4 * 32;  // first query row of this warp
                warp_rows_out(sOut + (8 + q4) * 512, ba.dq + (row_base + q0) * ba.ld_dq + (long long)h * FD, ba.ld_dq,
                              f, ba.scale, ba.acc & 1, lane);
            } else {
#pragma unroll
                for (int v = 0; v < 16; ++v)
                    __stcg(acc + v * FT, make_float4(f[4 * v], f[4 * v + 1], f[4 * v + 2], f[4 * v + 3]));
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        tmem_dealloc<512>(tmem);
    }
}


// ---------------------------------------------------------------- backward v7
// Same recurrence and CTA = (batch, head) sweep as k_fa5_bwd, re-laid-out so the
// tensor pipe reads most operands from TMEM and twice as many warps run the
// softmax (the round-2 timeline showed the fa5 step bound by 8 softmax warps and
// by a pipeline drain at every key block):
//   * K_j and V_j live in TMEM (cols [448,480) / [480,512), bf16 pairs, lane = key)
//     as the A operand of S^T = K Q^T and dP^T = V dO^T (TS MMAs: only the 2 KB
//     B slice per K16 step comes from shared memory); the softmax warps copy
//     block j+1 into TMEM from shared memory as soon as block j's last S/dP MMAs
//     completed, so the next block starts without a drain;
//   * Z^T = keep/(1-p) P^T and dS^T overwrite the S^T columns they came from
//     (bf16 pairs) and feed dV += Z^T dO and dK += dS^T Q as TS MMAs; dS^T also
//     goes to shared memory (128B swizzle) for dQ = dS K (SS, MN-major A);
//   * K is double-buffered in shared memory (dQ of block j reads K_j while K_{j+1}
//     lands), V has one staging buffer (it only feeds the TMEM copy);
//   * 16 softmax warps (lane quarter x 16-query column group), 4 dQ warps.
// TMEM: S^T/Z^T/dS^T [0,128), dP^T [128,256), dV [256,320), dK [320,384),
// dQ [384,448), K [448,480), V [480,512).
constexpr int B7_NST = 2;
constexpr int B7_STAGE = 2 * F_TILE_BYTES + 1024 + 2048;  // Q, dO, lse2[128], delta[128], keep bits [128][4]
constexpr int B7_WARPS = 23;                              // 16 softmax, 4 dQ, producer, MMA, dQ-MMA
// The single-thread roles get the highest warp ids: the warp schedulers favour
// higher ids, and a starved MMA issuer stalls every other role.
constexpr int W_PROD = 20, W_MMA = 21, W_DQMMA = 22;
constexpr int B7_OUT = 2048;  // per-warp output staging: 32 rows x 32 bf16, row-major (TMA store box)
constexpr int B7_SMEM = 1024 + 3 * F_TILE_BYTES + B7_NST * B7_STAGE + 4 * F_TILE_BYTES + 20 * B7_OUT + 256;

__device__ __forceinline__ void store_row_bf16(bf16* dst, const float* f, int n16, float sc, bool acc) {
    // n16 x 8 values of one row -> bf16 (x sc, += the existing values when acc), 16-byte stores
    for (int c = 0; c < n16; ++c) {
        float g[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) g[t] = f[c * 8 + t] * sc;
        uint4* d = (uint4*)dst + c;
        if (acc) {
            const uint4 old = *d;
            const __nv_bfloat162* po = (const __nv_bfloat162*)&old;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const float2 x = __bfloat1622float2(po[t]);
                g[2 * t] += x.x;
                g[2 * t + 1] += x.y;
            }
        }
        *d = make_uint4(pack_bf16(g[0], g[1]), pack_bf16(g[2], g[3]), pack_bf16(g[4], g[5]), pack_bf16(g[6], g[7]));
    }
}

// A warp's 32 rows (thread = row) x 32 fp32 -> bf16 (x sc) -> its staging slot (64B swizzle) ->
// one TMA bulk-tensor store of the 32x32 box at (c0, r0): the global write is
// coalesced by the TMA engine instead of 32 scattered 16-byte stores per instruction.
__device__ __forceinline__ void warp_tile_tma(uint8_t* stage, const CUtensorMap* map, int c0, int r0, const float* f,
                                              float sc, int lane) {
    if (lane == 0) bulk_wait_read0();  // the previous store from this slot has read it
    __syncwarp();
    // 64-byte TMA swizzle: 16-byte chunk c of row r sits at chunk c ^ ((r >> 1) & 3)
    // (conflict-free: the 8 lanes of a store phase hit 8 distinct bank groups)
    uint4* row = (uint4*)(stage + lane * 64);
#pragma unroll
    for (int c = 0; c < 4; ++c)
        row[c ^ ((lane >> 1) & 3)] = make_uint4(pack_bf16(f[8 * c] * sc, f[8 * c + 1] * sc), pack_bf16(f[8 * c + 2] * sc, f[8 * c + 3] * sc),
                                                pack_bf16(f[8 * c + 4] * sc, f[8 * c + 5] * sc), pack_bf16(f[8 * c + 6] * sc, f[8 * c + 7] * sc));
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
        tma_store_2d_cta(map, stage, c0, r0);
        bulk_commit_group();
    }
}

// step u -> (key block j, query block i): all nj x nj pairs, or for causal attention only
// the i >= j ones (queries at or after the keys; the rest is masked out entirely)
template <bool CAUSAL>
__device__ __forceinline__ void step_ji(int u, int nj, int& j, int& i, int nq = 0) {
    if (!CAUSAL) {  // nq query blocks per key block (cross-attention: nq != nj)
        if (!nq) nq = nj;
        j = u / nq;
        i = u % nq;
        return;
    }
    j = 0;
    int cnt = nj;
    while (u >= cnt) {
        u -= cnt;
        ++j;
        --cnt;
    }
    i = j + u;
}

template <bool CAUSAL>
__global__ void __launch_bounds__(B7_WARPS * 32, 1)
    k_fa7_bwd(const __grid_constant__ CUtensorMap tK, const __grid_constant__ CUtensorMap tV,
              const __grid_constant__ CUtensorMap tQ, const __grid_constant__ CUtensorMap tdO,
              const __grid_constant__ CUtensorMap tM, const __grid_constant__ CUtensorMap tdQ,
              const __grid_constant__ CUtensorMap tdK, const __grid_constant__ CUtensorMap tdV, BwdArgs ba) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (tc5::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* sK = smem;                              // [2] K_j (dQ's B operand; TMEM copy source)
    uint8_t* sV = sK + 2 * F_TILE_BYTES;             // V_j staging (TMEM copy source)
    uint8_t* sStage = sV + F_TILE_BYTES;             // [B7_NST][B7_STAGE]
    uint8_t* sDS = sStage + B7_NST * B7_STAGE;       // [2] x dS^T [2 q-halves][128 keys][64 q] bf16, swizzled
    uint8_t* sOut = sDS + 4 * F_TILE_BYTES;         // [20 warps][B7_OUT]
    uint64_t* bars = (uint64_t*)(sOut + 20 * B7_OUT);
    uint64_t* kv_full = bars;               // [2] K_j -> sK[j&1], V_j -> sV landed
    uint64_t* k_empty = bars + 2;           // [2] sK[b] no longer read (dQ of its block done)
    uint64_t* v_empty = bars + 4;           // sV copied into TMEM
    uint64_t* kv_tmem = bars + 5;           // K_j / V_j in TMEM
    uint64_t* st_full = bars + 6;           // [B7_NST]
    uint64_t* st_empty = st_full + B7_NST;  // [B7_NST]
    uint64_t* sdp_full = st_empty + B7_NST; // [2 halves]
    uint64_t* sm_done = sdp_full + 2;       // [2 halves]
    uint64_t* dq_full = sm_done + 2;
    uint64_t* dq_free = dq_full + 1;
    uint64_t* acc_full = dq_free + 1;
    uint64_t* acc_free = acc_full + 1;
    uint64_t* ds_free = acc_free + 1;       // [2] dS^T buffer b no longer read (its dQ MMAs done)
    uint64_t* ds_full = ds_free + 2;        // [2] dS^T buffer b written (both halves)
    uint32_t* tslot = (uint32_t*)(ds_full + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    // nj key blocks (outer) x nq query blocks (inner); cross-attention (Sk != S) is non-causal
    const int S = ba.S, Sk = ba.Sk ? ba.Sk : S, nj = Sk / FT, nq = S / FT;
    const int nsteps = CAUSAL ? nj * (nj + 1) / 2 : nj * nq;
    auto first_i = [&](int j) { return CAUSAL ? j : 0; };  // first query block of key block j
    const int h = blockIdx.x, b = blockIdx.y;
    const long long bh = (long long)b * ba.nh + h;
    const int row_base = b * S, kv_base = b * Sk;  // (query rows / key rows)
    const bool TS7 = ba.ts && blockIdx.x == 0 && blockIdx.y == 0;
    if (TS7 && threadIdx.x == 0) ba.ts[14 * 64 + 63] = gtime();

    if (threadIdx.x == 0) {
        tma_prefetch(&tK);
        tma_prefetch(&tV);
        tma_prefetch(&tQ);
        tma_prefetch(&tdO);
        if (ba.mask_t) tma_prefetch(&tM);
        for (int x = 0; x < 2; ++x) {
            mbar_init(&kv_full[x], 1);
            mbar_init(&k_empty[x], 1);
            mbar_init(&sdp_full[x], 1);
            mbar_init(&sm_done[x], 16);
        }
        mbar_init(v_empty, 8);
        mbar_init(kv_tmem, 16);
        for (int s = 0; s < B7_NST; ++s) {
            mbar_init(&st_full[s], 1);
            mbar_init(&st_empty[s], 1);
        }
        mbar_init(dq_full, 1);
        mbar_init(dq_free, 4);
        mbar_init(acc_full, 1);
        mbar_init(acc_free, 16);
        for (int x = 0; x < 2; ++x) {
            mbar_init(&ds_free[x], 1);
            mbar_init(&ds_full[x], 16);
        }
        fence_barrier_init();
    }
    if (warp == W_MMA) tmem_alloc<512>(tslot);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tslot;

    if (warp == W_PROD) {
        if (lane == 0) {
            // ------------------------------------------------ TMA producer
            auto load_kv = [&](int j) {
                const int kb = j & 1;
                if (j >= 2) mbar_wait(&k_empty[kb], ((j >> 1) & 1) ^ 1);
                if (j >= 1) mbar_wait(v_empty, (j - 1) & 1);
                mbar_expect_tx(&kv_full[kb], 2 * F_TILE_BYTES);
                tma_load_2d(sK + kb * F_TILE_BYTES, &tK, &kv_full[kb], h * FD, kv_base + j * FT);
                tma_load_2d(sV, &tV, &kv_full[kb], h * FD, kv_base + j * FT);
            };
            load_kv(0);
            // K/V of block j+1 go out before the stage of step (j, min(2, nj-1)): late
            // enough that V_j has been copied into TMEM (so the wait is short), early
            // enough that block j+1 never waits for them
            for (int u = 0; u < nsteps; ++u) {
                int j, i;
                step_ji<CAUSAL>(u, nj, j, i, nq);
                const int bl = (CAUSAL ? nj : nq) - first_i(j);  // steps of key block j
                if (i - first_i(j) == (bl > 2 ? 2 : bl - 1) && j + 1 < nj) load_kv(j + 1);
                const int s = u % B7_NST;
                uint8_t* st = sStage + s * B7_STAGE;
                if (TS7) ba.ts[14 * 64 + u] = gtime();
                mbar_wait(&st_empty[s], ((u / B7_NST) & 1) ^ 1);
                if (TS7) ba.ts[15 * 64 + u] = gtime();
                if (ba.dbg & 128) {  // debugging: no per-step loads
                    mbar_arrive(&st_full[s]);
                    continue;
                }
                mbar_expect_tx(&st_full[s], 2 * F_TILE_BYTES + 1024 + (ba.mask_t ? 2048 : 0));
                tma_load_2d(st, &tQ, &st_full[s], h * FD, row_base + i * FT);
                tma_load_2d(st + F_TILE_BYTES, &tdO, &st_full[s], h * FD, row_base + i * FT);
                bulk_load(st + 2 * F_TILE_BYTES, ba.lse2 + bh * S + i * FT, 512, &st_full[s]);
                bulk_load(st + 2 * F_TILE_BYTES + 512, ba.delta + bh * S + i * FT, 512, &st_full[s]);
                if (ba.mask_t)
                    tma_load_2d(st + 2 * F_TILE_BYTES + 1024, &tM, &st_full[s], i * (FT / 32), (int)(bh * Sk) + j * FT);
            }
        }
    } else if (warp == W_MMA) {
        // ------------------------------------------------ MMA issuer (whole warp, one
        // elected lane issues: descriptors stay in uniform registers, each MMA is a
        // couple of instructions; the 32-cycle M128 N64 K16 MMAs are issue-bound otherwise)
        constexpr uint32_t id_s = idesc_bf16(FT, FT / 2, false, false);  // S^T / dP^T half: M128 N64
        constexpr uint32_t id_kv = idesc_bf16(FT, FD, false, true);      // dV / dK: M128 N64, B MN-major
        constexpr uint32_t id_q = idesc_bf16(FT, FD, true, true);        // dQ: A and B MN-major
        const bool mm = !(ba.dbg & 4);
        const uint32_t stage0 = smem_u32(sStage);
        auto issue_sdp = [&](int u, int hh) {
            int j, i;
            step_ji<CAUSAL>(u, nj, j, i, nq);
            const int s = u % B7_NST;
            const uint32_t aQ = stage0 + s * B7_STAGE + hh * (F_TILE_BYTES / 2);
            if (hh == 0) {
                if (i == first_i(j)) mbar_wait(kv_tmem, j & 1);  // K_j / V_j in TMEM
                mbar_wait(&st_full[s], (u / B7_NST) & 1);
                fence_after();
            }
            if (mm) {
                const uint64_t dq = desc_kmajor(aQ, 0), ddo = desc_kmajor(aQ + F_TILE_BYTES, 0);
#pragma unroll
                for (int kk = 0; kk < FD / 16; ++kk)  // S^T half = K Q_half^T
                    mma_ts_w(tmem + hh * 64, tmem + 448 + kk * 8, dq + 2 * kk, id_s, kk);
#pragma unroll
                for (int kk = 0; kk < FD / 16; ++kk)  // dP^T half = V dO_half^T
                    mma_ts_w(tmem + 128 + hh * 64, tmem + 480 + kk * 8, ddo + 2 * kk, id_s, kk);
            }
            mma_commit_w(&sdp_full[hh]);
        };
        issue_sdp(0, 0);
        issue_sdp(0, 1);
        for (int u = 0; u < nsteps; ++u) {
            int j, i;
            step_ji<CAUSAL>(u, nj, j, i, nq);
            const int s = u % B7_NST;
            const int acc0 = i != first_i(j);  // dK / dV accumulate after the block's first step
            const uint32_t aQ = stage0 + s * B7_STAGE, adO = aQ + F_TILE_BYTES;
#pragma unroll 1
            for (int hh = 0; hh < 2; ++hh) {
                mbar_wait(&sm_done[hh], u & 1);
                if (hh == 0 && i == first_i(j) && j > 0) mbar_wait(acc_free, (j - 1) & 1);  // dK/dV of block j-1 drained
                if (TS7 && lane == 0) ba.ts[hh * 64 + u] = gtime();
                fence_after();
                if (mm) {
                    const uint64_t bdo = desc_mnmajor(adO, hh * 4), bq = desc_mnmajor(aQ, hh * 4);
#pragma unroll
                    for (int k4 = 0; k4 < 4; ++k4)  // dV += Z^T_half dO_half (Z^T: 8 cols per 16 queries)
                        mma_ts_w(tmem + 256, tmem + hh * 64 + k4 * 16, bdo + 128 * k4, id_kv, acc0 | hh | k4);
#pragma unroll
                    for (int k4 = 0; k4 < 4; ++k4)  // dK += dS^T_half Q_half
                        mma_ts_w(tmem + 320, tmem + hh * 64 + k4 * 16 + 8, bq + 128 * k4, id_kv, acc0 | hh | k4);
                }
                if (hh == 1) {
                    mma_commit_w(&st_empty[s]);  // Q, dO, lse, delta, keep bits of this step are no longer read
                    if (i == nq - 1) mma_commit_w(acc_full);
                }
                if (u + 1 < nsteps) issue_sdp(u + 1, hh);
            }
        }
    } else if (warp == W_DQMMA) {
        // ------------------------------------------------ dQ MMA issuer (a warp of its own:
        // tcgen05.mma issue blocks while the tensor pipe drains, so these would otherwise
        // delay the S/dP issue the softmax warps wait for)
        constexpr uint32_t id_q = idesc_bf16(FT, FD, true, true);  // dQ: A and B MN-major
        const bool mm = !(ba.dbg & 4);
        const uint32_t ds0 = smem_u32(sDS), k0 = smem_u32(sK);
        for (int u = 0; u < nsteps; ++u) {
            int j, i;
            step_ji<CAUSAL>(u, nj, j, i, nq);
            mbar_wait(&ds_full[u & 1], (u >> 1) & 1);  // dS^T(u) written (both halves)
            if (u > 0) mbar_wait(dq_free, (u - 1) & 1);  // dQ of the previous step has left TMEM
            if (TS7 && lane == 0) ba.ts[2 * 64 + u] = gtime();
            fence_after();
            if (mm) {
                const uint64_t da = sdesc(ds0 + (u & 1) * 2 * F_TILE_BYTES, 16384 >> 4, 1024 >> 4),
                               db = desc_mnmajor(k0 + (j & 1) * F_TILE_BYTES, 0);
#pragma unroll
                for (int kk = 0; kk < FT / 16; ++kk)  // dQ_ij = dS K
                    mma_ss_w(tmem + 384, da + 128 * kk, db + 128 * kk, id_q, kk);
            }
            mma_commit_w(dq_full);
            mma_commit_w(&ds_free[u & 1]);
            if (i == nq - 1) mma_commit_w(&k_empty[j & 1]);  // K_j no longer read
        }
    } else if (warp < 16) {
        // ------------------------------------------------------------------
        // 16 softmax warps: lane quarter q4 (key rows), column group cg = 16 of
        // the 64 queries of each half
        const int q4 = warp & 3, cg = warp >> 2, k = q4 * 32 + lane;
        const uint32_t t_lane = tmem + ((uint32_t)(q4 * 32) << 16);
        // K_j (cg 0, 1) / V_j (cg 2, 3) rows -> TMEM (16 of their 32 bf16-pair columns each)
        auto kv_to_tmem = [&](int j) {
            mbar_wait(&kv_full[j & 1], (j >> 1) & 1);
            const uint8_t* src = (cg < 2 ? sK + (j & 1) * F_TILE_BYTES : sV) + k * 128;
            uint32_t r[16];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint4 x = *(const uint4*)(src + ((((cg & 1) * 4 + c) ^ (k & 7)) * 16));
                r[4 * c] = x.x;
                r[4 * c + 1] = x.y;
                r[4 * c + 2] = x.z;
                r[4 * c + 3] = x.w;
            }
            uint32_t r0[8], r1[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                r0[t] = r[t];
                r1[t] = r[8 + t];
            }
            const uint32_t col = (cg < 2 ? 448 : 480) + (cg & 1) * 16;
            tmem_st8(t_lane + col, r0);
            tmem_st8(t_lane + col + 8, r1);
            tmem_st_wait();
            fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(kv_tmem);
                if (cg >= 2) mbar_arrive(v_empty);
            }
        };
        // dV_j (cg 0, 1) / dK_j (cg 2, 3): 32 of the 64 columns of this thread's key row
        auto drain_kv = [&](int j) {
            mbar_wait(acc_full, j & 1);
            fence_after();
            uint32_t r[32];
            tmem_ld32_nowait(t_lane + 256 + cg * 32, r);
            tmem_ld_wait();
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_free);
            float f[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) f[e] = __uint_as_float(r[e]);
            const long long row = kv_base + (long long)j * FT + k;
            if (ba.dbg & 32) return;
            const bool acc = cg >= 2 ? (ba.acc & 2) : (ba.acc & 4);
            if (!acc)  // coalesced: staged tile + TMA store
                warp_tile_tma(sOut + warp * B7_OUT, cg >= 2 ? &tdK : &tdV, h * FD + (cg & 1) * 32,
                              kv_base + j * FT + q4 * 32, f, cg >= 2 ? ba.scale : 1.f, lane);
            else if (cg >= 2)
                store_row_bf16(ba.dk + row * ba.ld_dk + (long long)h * FD + (cg & 1) * 32, f, 4, ba.scale, true);
            else
                store_row_bf16(ba.dv + row * ba.ld_dv + (long long)h * FD + (cg & 1) * 32, f, 4, 1.f, true);
        };
        kv_to_tmem(0);
        for (int u = 0; u < nsteps; ++u) {
            int j, i;
            step_ji<CAUSAL>(u, nj, j, i, nq);
            const int s = u % B7_NST;
            const float* lse_s = (const float*)(sStage + s * B7_STAGE + 2 * F_TILE_BYTES);
            const float* dl_s = lse_s + FT;
            uint8_t* ds_buf = sDS + (u & 1) * 2 * F_TILE_BYTES;
            mbar_wait(&st_full[s], (u / B7_NST) & 1);
#pragma unroll 1
            for (int hh = 0; hh < 2; ++hh) {
                const int q0 = hh * 64 + cg * 16;  // first query (of the 128-query block) of this thread's columns
                mbar_wait(&sdp_full[hh], u & 1);
                if (TS7 && warp == 0 && lane == 0) ba.ts[(3 + 2 * hh) * 64 + u] = gtime();
                if (TS7 && lane == 0 && u == 5) ba.ts[(12 + hh) * 64 + warp] = gtime();
                fence_after();
                if (hh == 1 && i == nq - 1 && j + 1 < nj) kv_to_tmem(j + 1);  // block j's S/dP all complete
                uint32_t sv[16], dp[16];
                if (!(ba.dbg & 8)) {
                    tmem_ld16_nowait(t_lane + q0, sv);
                    tmem_ld16_nowait(t_lane + 128 + q0, dp);
                } else {
#pragma unroll
                    for (int e = 0; e < 16; ++e) sv[e] = dp[e] = e;
                }
                const uint32_t mword =
                    ba.mask_t ? *(const uint32_t*)(sStage + s * B7_STAGE + 2 * F_TILE_BYTES + 1024 + k * 16 + (q0 >> 5) * 4) >>
                                    (q0 & 16)
                              : 0xFFFFu;
                tmem_ld_wait();
                if (CAUSAL && i == j) {  // diagonal block: key k sees queries q >= k only
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        if (q0 + e < k) sv[e] = __float_as_uint(-INFINITY);
                }
                uint32_t zk[8], dk[8];
#pragma unroll
                for (int e4 = 0; e4 < 4; ++e4) {
                    if (ba.dbg & 1) {
                        zk[2 * e4] = zk[2 * e4 + 1] = dk[2 * e4] = dk[2 * e4 + 1] = sv[e4] ^ dp[e4];
                        continue;
                    }
                    // (lse2 and delta are stored negated by the prep kernel)
                    const float4 l4 = *(const float4*)(lse_s + q0 + e4 * 4);
                    const float4 d4 = *(const float4*)(dl_s + q0 + e4 * 4);
                    const float2 lv[2] = {make_float2(l4.x, l4.y), make_float2(l4.z, l4.w)};
                    const float2 dv[2] = {make_float2(d4.x, d4.y), make_float2(d4.z, d4.w)};
                    const float2 c2 = make_float2(ba.c, ba.c);
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) {  // element pairs on the packed-fp32 pipe
                        const int e = e4 * 4 + e2 * 2;
                        const float2 a = ffma2(make_float2(__uint_as_float(sv[e]), __uint_as_float(sv[e + 1])), c2, lv[e2]);
                        const float2 p = make_float2(ex2f(a.x), ex2f(a.y));
                        const float2 kd = make_float2(((mword >> e) & 1) ? ba.dscale : 0.f,
                                                      ((mword >> (e + 1)) & 1) ? ba.dscale : 0.f);
                        const float2 z = fmul2(p, kd);
                        const float2 ds =
                            fmul2(p, ffma2(kd, make_float2(__uint_as_float(dp[e]), __uint_as_float(dp[e + 1])), dv[e2]));
                        zk[2 * e4 + e2] = pack_bf16(z.x, z.y);
                        dk[2 * e4 + e2] = pack_bf16(ds.x, ds.y);
                    }
                }
                if (!(ba.dbg & 64)) {
                    tmem_st8(t_lane + q0, zk);      // Z^T over this group's S^T columns
                    tmem_st8(t_lane + q0 + 8, dk);  // dS^T next to it
                }
                // dS^T row k, queries q0..q0+15 of half hh: 16-byte chunks cg*2, cg*2+1 of the 128 B row
                if (hh == 0 && u >= 2) mbar_wait(&ds_free[u & 1], ((u >> 1) - 1) & 1);  // dQ(u-2) read this buffer
                uint8_t* rowp = ds_buf + hh * 16384 + k * 128;
                if (!(ba.dbg & 16)) {
                    *(uint4*)(rowp + (((cg * 2) ^ (k & 7)) * 16)) = make_uint4(dk[0], dk[1], dk[2], dk[3]);
                    *(uint4*)(rowp + (((cg * 2 + 1) ^ (k & 7)) * 16)) = make_uint4(dk[4], dk[5], dk[6], dk[7]);
                }
                tmem_st_wait();
                fence_proxy_async();
                fence_before();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&sm_done[hh]);
                    if (hh == 1) mbar_arrive(&ds_full[u & 1]);
                }
                if (TS7 && warp == 0 && lane == 0) ba.ts[(4 + 2 * hh) * 64 + u] = gtime();
                if (TS7 && lane == 0 && u == 5) ba.ts[(8 + hh) * 64 + warp] = gtime();
                if (TS7 && lane == 0 && u == 6) ba.ts[(10 + hh) * 64 + warp] = gtime();
                if (hh == 0 && i == first_i(j) && j > 0) drain_kv(j - 1);  // TMEM dK/dV free before dV/dK of block j start
            }
        }
        drain_kv(nj - 1);
    } else {
        // ---------------------------------------------------- 4 dQ warps (thread = query row)
        // dQ_ij leaves TMEM right away (dQ(u+1) waits for dq_free); the row's fp32
        // partial sum over key blocks lives in this CTA's private L2-resident buffer:
        // written at j = 0, then red.global.add (performed at L2, no read round trip;
        // every address is only ever updated by this one thread, in program order, so
        // the summation order — and the result — is fixed), read back at the last j.
        const int q4 = warp & 3, r = q4 * 32 + lane;
        const uint32_t t_row = tmem + ((uint32_t)(q4 * 32) << 16) + 384;
        for (int u = 0; u < nsteps; ++u) {
            int j, i;
            step_ji<CAUSAL>(u, nj, j, i, nq);
            // thread-major: float4 v of query row r of block i at ((bh*nq + i)*16 + v)*128 + r
            float4* acc = (float4*)ba.dqacc + ((bh * nq + i) * 16) * FT + r;
            const bool last = j == (CAUSAL ? i : nj - 1), dbg = ba.dbg & 2;  // query block i's last key block
            float f[32];
            if (last && j > 0 && !dbg) {  // the final partial sum's first half, before dQ(u) lands
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                    const float4 a4 = __ldcg(acc + v * FT);
                    f[4 * v] = a4.x;
                    f[4 * v + 1] = a4.y;
                    f[4 * v + 2] = a4.z;
                    f[4 * v + 3] = a4.w;
                }
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) f[e] = 0.f;
            }
            mbar_wait(dq_full, u & 1);
            if (TS7 && warp == 16 && lane == 0) ba.ts[7 * 64 + u] = gtime();
            fence_after();
            uint32_t d[32];
#pragma unroll 1
            for (int pss = 0; pss < 2; ++pss) {
                tmem_ld32_nowait(t_row + pss * 32, d);
                tmem_ld_wait();
                if (pss == 1) {
                    fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(dq_free);
                }
                if (dbg) continue;
                if (!last) {
#pragma unroll
                    for (int v = 0; v < 8; ++v) {
                        const float4 x = make_float4(__uint_as_float(d[4 * v]), __uint_as_float(d[4 * v + 1]),
                                                     __uint_as_float(d[4 * v + 2]), __uint_as_float(d[4 * v + 3]));
                        if (j == 0) __stcg(acc + (pss * 8 + v) * FT, x);
                        else red_add_v4((float*)(acc + (pss * 8 + v) * FT), x);
                    }
                    continue;
                }
                if (pss == 1 && j > 0) {
#pragma unroll
                    for (int v = 0; v < 8; ++v) {
                        const float4 a4 = __ldcg(acc + (8 + v) * FT);
                        f[4 * v] = a4.x;
                        f[4 * v + 1] = a4.y;
                        f[4 * v + 2] = a4.z;
                        f[4 * v + 3] = a4.w;
                    }
                } else if (pss == 1) {
#pragma unroll
                    for (int e = 0; e < 32; ++e) f[e] = 0.f;
                }
#pragma unroll
                for (int e = 0; e < 32; ++e) f[e] += __uint_as_float(d[e]);
                if (!(ba.acc & 1))
                    warp_tile_tma(sOut + warp * B7_OUT, &tdQ, h * FD + pss * 32, row_base + i * FT + q4 * 32, f, ba.scale,
                                  lane);
                else {
                    const long long row = row_base + (long long)i * FT + r;
                    store_row_bf16(ba.dq + row * ba.ld_dq + (long long)h * FD + pss * 32, f, 4, ba.scale, true);
                }
            }
        }
    }
    if (lane == 0) bulk_wait0();  // this warp's TMA stores have completed
    fence_before();
    __syncthreads();
    if (TS7 && threadIdx.x == 0) ba.ts[15 * 64 + 63] = gtime();
    if (warp == W_MMA) {
        fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// ------------------------------------------------------- backward, head_dim 128
// The v7 recurrence re-laid-out for head_dim 128 (GPT-Neo, BASELINE.json C4),
// where dV, dK (128 keys x 128 fp32 each) and dQ leave no TMEM for K/V operands:
//   * CTA = (batch, head); key blocks j of 128 (outer), query blocks i of 64
//     (inner), each in two halves of 32 queries (one half's softmax overlaps the
//     other half's MMAs);
//   * S^T = K Q^T and dP^T = V dO^T are SS MMAs (M128 N32, K = 128 over the two
//     64-column panels of K / V and of the Q / dO stage);
//   * Z^T and dS^T overwrite the S^T columns they came from (bf16 pairs) and feed
//     dV += Z^T dO and dK += dS^T Q as TS MMAs (M128 N128, B MN-major over both
//     panels: LBO = one panel);
//   * dQ^T = K^T dS^T (M128 = head dims, N64 = queries, SS: K read MN-major,
//     LBO = one K panel; dS^T from shared memory) by its own issuer warp; 4 dQ
//     warps (thread = head dim) add it into the CTA's private fp32 accumulator
//     (stored at a query block's first key block, red.global.add after, read back
//     at the last: every address has one writer in program order — deterministic);
//   * K double-buffered, V single-buffered (the next V loads after the block's
//     last dP^T MMA), dK / dV drained by the softmax warps while the next key
//     block starts.
// TMEM: S^T [0,64), dP^T [64,128), dV [128,256), dK [256,384), dQ^T [384,448).
constexpr int B8_D = 128, B8_QT = 64;                          // head dim, queries per step
constexpr int B8_KV = FT * B8_D * 2;                           // 32 KB: K or V tile (2 panels of 16 KB)
constexpr int B8_QP = B8_QT * 128;                             // 8 KB: one 64-column panel of a Q / dO stage
// Q, dO, lse2[64], delta[64], keep bits [128 keys][4 words]: the 128-query word span holding this
// block's 64 (a TMA box row must be a multiple of 16 bytes)
constexpr int B8_STAGE_RAW = 4 * B8_QP + 2 * B8_QT * 4 + FT * 16;
constexpr int B8_STAGE = (B8_STAGE_RAW + 1023) & ~1023;
constexpr int B8_NST = 2;
constexpr int B8_DS = FT * B8_QT * 2;                          // 16 KB: dS^T [128 keys][64 queries] bf16
constexpr int B8_SMEM = 1024 + 2 * B8_KV + B8_KV + B8_NST * B8_STAGE + 2 * B8_DS + 256;
constexpr int B8_WARPS = 15;                                   // 8 softmax, 4 dQ, producer, MMA, dQ-MMA
constexpr int W8_PROD = 12, W8_MMA = 13, W8_DQMMA = 14;

// step u -> (key block j of 128, query block i of 64): all pairs, or for causal
// attention the i >= 2j ones (the block's last query is at or after its first key)
template <bool CAUSAL>
__device__ __forceinline__ void step_ji8(int u, int nj, int nq, int& j, int& i) {
    if (!CAUSAL) {
        j = u / nq;
        i = u % nq;
        return;
    }
    j = 0;
    int cnt = nq;
    while (u >= cnt) {
        u -= cnt;
        ++j;
        cnt -= 2;
    }
    i = 2 * j + u;
}

template <bool CAUSAL>
__global__ void __launch_bounds__(B8_WARPS * 32, 1)
    k_fa8_bwd(const __grid_constant__ CUtensorMap tK, const __grid_constant__ CUtensorMap tV,
              const __grid_constant__ CUtensorMap tQ, const __grid_constant__ CUtensorMap tdO,
              const __grid_constant__ CUtensorMap tM, BwdArgs ba) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (tc5::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* sK = smem;                      // [2] K_j: 2 panels [128 keys][64 dims]
    uint8_t* sV = sK + 2 * B8_KV;            // V_j
    uint8_t* sStage = sV + B8_KV;            // [B8_NST][B8_STAGE]
    uint8_t* sDS = sStage + B8_NST * B8_STAGE;  // [2] dS^T
    uint64_t* bars = (uint64_t*)(sDS + 2 * B8_DS);
    uint64_t* k_full = bars;                 // [2]
    uint64_t* k_empty = bars + 2;            // [2] (dQ of its block done)
    uint64_t* v_full = bars + 4;
    uint64_t* v_empty = bars + 5;            // the block's last dP^T MMA done
    uint64_t* st_full = bars + 6;            // [B8_NST]
    uint64_t* st_empty = st_full + B8_NST;   // [B8_NST]
    uint64_t* sdp_full = st_empty + B8_NST;  // [2 halves]
    uint64_t* sm_done = sdp_full + 2;        // [2 halves]
    uint64_t* dq_full = sm_done + 2;
    uint64_t* dq_free = dq_full + 1;
    uint64_t* acc_full = dq_free + 1;
    uint64_t* acc_free = acc_full + 1;
    uint64_t* ds_free = acc_free + 1;        // [2]
    uint64_t* ds_full = ds_free + 2;         // [2]
    uint32_t* tslot = (uint32_t*)(ds_full + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int S = ba.S, Sk = ba.Sk ? ba.Sk : S, nj = Sk / FT, nq = S / B8_QT;  // (cross-attention: Sk != S)
    int nsteps = nj * nq;
    if (CAUSAL) {
        nsteps = 0;
        for (int j = 0; j < nj; ++j) nsteps += nq - 2 * j;
    }
    auto first_i = [&](int j) { return CAUSAL ? 2 * j : 0; };
    const int h = blockIdx.x, b = blockIdx.y;
    const long long bh = (long long)b * ba.nh + h;
    const int row_base = b * S, kv_base = b * Sk;  // (query rows / key rows)

    if (threadIdx.x == 0) {
        for (int x = 0; x < 2; ++x) {
            mbar_init(&k_full[x], 1);
            mbar_init(&k_empty[x], 1);
            mbar_init(&sdp_full[x], 1);
            mbar_init(&sm_done[x], 8);
            mbar_init(&ds_free[x], 1);
            mbar_init(&ds_full[x], 8);
        }
        mbar_init(v_full, 1);
        mbar_init(v_empty, 1);
        for (int s = 0; s < B8_NST; ++s) {
            mbar_init(&st_full[s], 1);
            mbar_init(&st_empty[s], 1);
        }
        mbar_init(dq_full, 1);
        mbar_init(dq_free, 4);
        mbar_init(acc_full, 1);
        mbar_init(acc_free, 8);
        fence_barrier_init();
    }
    if (warp == W8_MMA) tmem_alloc<512>(tslot);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tslot;

    if (warp == W8_PROD) {
        if (lane == 0) {
            // ------------------------------------------------ TMA producer
            auto load_k = [&](int j) {
                const int kb = j & 1;
                if (j >= 2) mbar_wait(&k_empty[kb], ((j >> 1) - 1) & 1);
                mbar_expect_tx(&k_full[kb], B8_KV);
                for (int p = 0; p < 2; ++p)
                    tma_load_2d(sK + kb * B8_KV + p * (B8_KV / 2), &tK, &k_full[kb], h * B8_D + 64 * p, kv_base + j * FT);
            };
            auto load_v = [&](int j) {
                if (j >= 1) mbar_wait(v_empty, (j - 1) & 1);
                mbar_expect_tx(v_full, B8_KV);
                for (int p = 0; p < 2; ++p)
                    tma_load_2d(sV + p * (B8_KV / 2), &tV, v_full, h * B8_D + 64 * p, kv_base + j * FT);
            };
            load_k(0);
            load_v(0);
            for (int u = 0; u < nsteps; ++u) {
                int j, i;
                step_ji8<CAUSAL>(u, nj, nq, j, i);
                const int s = u % B8_NST;
                uint8_t* st = sStage + s * B8_STAGE;
                mbar_wait(&st_empty[s], ((u / B8_NST) & 1) ^ 1);
                mbar_expect_tx(&st_full[s], 4 * B8_QP + 2 * B8_QT * 4 + (ba.mask_t ? FT * 16 : 0));
                for (int p = 0; p < 2; ++p) {
                    tma_load_2d(st + p * B8_QP, &tQ, &st_full[s], h * B8_D + 64 * p, row_base + i * B8_QT);
                    tma_load_2d(st + (2 + p) * B8_QP, &tdO, &st_full[s], h * B8_D + 64 * p, row_base + i * B8_QT);
                }
                bulk_load(st + 4 * B8_QP, ba.lse2 + bh * S + i * B8_QT, B8_QT * 4, &st_full[s]);
                bulk_load(st + 4 * B8_QP + B8_QT * 4, ba.delta + bh * S + i * B8_QT, B8_QT * 4, &st_full[s]);
                if (ba.mask_t)
                    tma_load_2d(st + 4 * B8_QP + 2 * B8_QT * 4, &tM, &st_full[s], (i >> 1) * 4, (int)(bh * Sk) + j * FT);
                // K_{j+1} into the other buffer once block j is under way (its previous user,
                // block j-1, releases it with its last dQ); V_{j+1} after block j's last stage
                if (j + 1 < nj && i == first_i(j) + (nq - first_i(j) > 1 ? 1 : 0)) load_k(j + 1);
                if (i == nq - 1 && j + 1 < nj) load_v(j + 1);
            }
        }
    } else if (warp == W8_MMA) {
        // ------------------------------------------------ MMA issuer (elected lane)
        constexpr uint32_t id_s = idesc_bf16(FT, 32, false, false);   // S^T / dP^T half: M128 N32
        constexpr uint32_t id_kv = idesc_bf16(FT, B8_D, false, true);  // dV / dK: M128 N128, B MN-major
        const bool mm = !(ba.dbg & 4);
        const uint32_t stage0 = smem_u32(sStage), k0 = smem_u32(sK), v0 = smem_u32(sV);
        auto issue_sdp = [&](int u, int hh) {
            int j, i;
            step_ji8<CAUSAL>(u, nj, nq, j, i);
            const int s = u % B8_NST;
            const uint32_t aQ = stage0 + s * B8_STAGE, adO = aQ + 2 * B8_QP;
            if (hh == 0) {
                if (i == first_i(j)) {
                    mbar_wait(&k_full[j & 1], (j >> 1) & 1);
                    mbar_wait(v_full, j & 1);
                }
                mbar_wait(&st_full[s], (u / B8_NST) & 1);
                fence_after();
            }
            if (mm) {
                const uint32_t ak = k0 + (j & 1) * B8_KV;
#pragma unroll
                for (int kk = 0; kk < B8_D / 16; ++kk)  // S^T half = K Q_half^T
                    mma_ss_w(tmem + hh * 32, desc_kmajor(ak + (kk >> 2) * (B8_KV / 2), kk & 3),
                             desc_kmajor(aQ + (kk >> 2) * B8_QP + hh * 4096, kk & 3), id_s, kk);
#pragma unroll
                for (int kk = 0; kk < B8_D / 16; ++kk)  // dP^T half = V dO_half^T
                    mma_ss_w(tmem + 64 + hh * 32, desc_kmajor(v0 + (kk >> 2) * (B8_KV / 2), kk & 3),
                             desc_kmajor(adO + (kk >> 2) * B8_QP + hh * 4096, kk & 3), id_s, kk);
            }
            mma_commit_w(&sdp_full[hh]);
            if (hh == 1 && i == nq - 1) mma_commit_w(v_empty);  // V_j read for the last time
        };
        issue_sdp(0, 0);
        issue_sdp(0, 1);
        for (int u = 0; u < nsteps; ++u) {
            int j, i;
            step_ji8<CAUSAL>(u, nj, nq, j, i);
            const int s = u % B8_NST;
            const int acc0 = i != first_i(j);
            const uint32_t aQ = stage0 + s * B8_STAGE, adO = aQ + 2 * B8_QP;
#pragma unroll 1
            for (int hh = 0; hh < 2; ++hh) {
                mbar_wait(&sm_done[hh], u & 1);
                if (hh == 0 && i == first_i(j) && j > 0) mbar_wait(acc_free, (j - 1) & 1);
                fence_after();
                if (mm) {
#pragma unroll
                    for (int k2 = 0; k2 < 2; ++k2)  // dV += Z^T_half dO_half (Z^T: 8 cols per 16 queries)
                        mma_ts_w(tmem + 128, tmem + hh * 32 + k2 * 16, desc_mnmajor(adO, 2 * hh + k2), id_kv,
                                 acc0 | hh | k2);
#pragma unroll
                    for (int k2 = 0; k2 < 2; ++k2)  // dK += dS^T_half Q_half
                        mma_ts_w(tmem + 256, tmem + hh * 32 + k2 * 16 + 8, desc_mnmajor(aQ, 2 * hh + k2), id_kv,
                                 acc0 | hh | k2);
                }
                if (hh == 1) {
                    mma_commit_w(&st_empty[s]);
                    if (i == nq - 1) mma_commit_w(acc_full);
                }
                if (u + 1 < nsteps) issue_sdp(u + 1, hh);
            }
        }
    } else if (warp == W8_DQMMA) {
        // ------------------------------------------------ dQ^T = K^T dS^T issuer
        constexpr uint32_t id_q = idesc_bf16(FT, B8_QT, true, true);  // M128 (dims) N64 (queries), both MN-major
        const bool mm = !(ba.dbg & 4);
        const uint32_t ds0 = smem_u32(sDS), k0 = smem_u32(sK);
        for (int u = 0; u < nsteps; ++u) {
            int j, i;
            step_ji8<CAUSAL>(u, nj, nq, j, i);
            mbar_wait(&ds_full[u & 1], (u >> 1) & 1);
            if (u > 0) mbar_wait(dq_free, (u - 1) & 1);
            fence_after();
            if (mm) {
                const uint32_t ak = k0 + (j & 1) * B8_KV, ad = ds0 + (u & 1) * B8_DS;
#pragma unroll
                for (int kk = 0; kk < FT / 16; ++kk)  // 16 keys per step: 16 rows of 128 B
                    mma_ss_w(tmem + 384, sdesc(ak + kk * 2048, (B8_KV / 2) >> 4, 1024 >> 4), desc_mnmajor(ad, kk), id_q,
                             kk);
            }
            mma_commit_w(dq_full);
            mma_commit_w(&ds_free[u & 1]);
            if (i == nq - 1) mma_commit_w(&k_empty[j & 1]);
        }
    } else if (warp < 8) {
        // ------------------------------------------------ 8 softmax warps: lane quarter q4
        // (key rows), column group cg = 16 of the 32 queries of each half
        const int q4 = warp & 3, cg = warp >> 2, k = q4 * 32 + lane;
        const uint32_t t_lane = tmem + ((uint32_t)(q4 * 32) << 16);
        // dV_j (cg 0) / dK_j (cg 1): this thread's key row, 128 columns in four chunks
        auto drain_kv = [&](int j) {
            mbar_wait(acc_full, j & 1);
            fence_after();
            const long long row = kv_base + (long long)j * FT + k;
            const bool acc = cg == 1 ? (ba.acc & 2) : (ba.acc & 4);
            bf16* dst = cg == 1 ? ba.dk + row * ba.ld_dk + (long long)h * B8_D : ba.dv + row * ba.ld_dv + (long long)h * B8_D;
            const float sc = cg == 1 ? ba.scale : 1.f;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                uint32_t r[32];
                tmem_ld32_nowait(t_lane + 128 + cg * 128 + c * 32, r);
                tmem_ld_wait();
                if (c == 3) {
                    fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(acc_free);
                }
                float f[32];
#pragma unroll
                for (int e = 0; e < 32; ++e) f[e] = __uint_as_float(r[e]);
                if (!(ba.dbg & 32)) store_row_bf16(dst + c * 32, f, 4, sc, acc);
            }
        };
        for (int u = 0; u < nsteps; ++u) {
            int j, i;
            step_ji8<CAUSAL>(u, nj, nq, j, i);
            const int s = u % B8_NST;
            const uint8_t* st = sStage + s * B8_STAGE;
            const float* lse_s = (const float*)(st + 4 * B8_QP);
            const float* dl_s = lse_s + B8_QT;
            uint8_t* ds_buf = sDS + (u & 1) * B8_DS;
            mbar_wait(&st_full[s], (u / B8_NST) & 1);
#pragma unroll 1
            for (int hh = 0; hh < 2; ++hh) {
                const int q0 = hh * 32 + cg * 16;  // first query (of the 64) of this thread's columns
                mbar_wait(&sdp_full[hh], u & 1);
                fence_after();
                uint32_t sv[16], dp[16];
                tmem_ld16_nowait(t_lane + q0, sv);
                tmem_ld16_nowait(t_lane + 64 + q0, dp);
                const uint32_t mword =
                    ba.mask_t ? *(const uint32_t*)(st + 4 * B8_QP + 2 * B8_QT * 4 + k * 16 + ((i & 1) * 2 + hh) * 4) >> (cg * 16)
                              : 0xFFFFu;
                tmem_ld_wait();
                if (CAUSAL && i <= 2 * j + 1) {  // diagonal blocks: key k sees queries at or after it
                    const int qd = i * B8_QT + q0 - j * FT - k;  // (query - key) of element 0
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        if (qd + e < 0) sv[e] = __float_as_uint(-INFINITY);
                }
                uint32_t zk[8], dk[8];
#pragma unroll
                for (int e4 = 0; e4 < 4; ++e4) {
                    const float4 l4 = *(const float4*)(lse_s + q0 + e4 * 4);  // (negated by the prep kernel)
                    const float4 d4 = *(const float4*)(dl_s + q0 + e4 * 4);
                    const float2 lv[2] = {make_float2(l4.x, l4.y), make_float2(l4.z, l4.w)};
                    const float2 dv[2] = {make_float2(d4.x, d4.y), make_float2(d4.z, d4.w)};
                    const float2 c2 = make_float2(ba.c, ba.c);
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) {
                        const int e = e4 * 4 + e2 * 2;
                        const float2 a = ffma2(make_float2(__uint_as_float(sv[e]), __uint_as_float(sv[e + 1])), c2, lv[e2]);
                        const float2 p = make_float2(ex2f(a.x), ex2f(a.y));
                        const float2 kd = make_float2(((mword >> e) & 1) ? ba.dscale : 0.f,
                                                      ((mword >> (e + 1)) & 1) ? ba.dscale : 0.f);
                        const float2 z = fmul2(p, kd);
                        const float2 ds =
                            fmul2(p, ffma2(kd, make_float2(__uint_as_float(dp[e]), __uint_as_float(dp[e + 1])), dv[e2]));
                        zk[2 * e4 + e2] = pack_bf16(z.x, z.y);
                        dk[2 * e4 + e2] = pack_bf16(ds.x, ds.y);
                    }
                }
                tmem_st8(t_lane + q0, zk);      // Z^T over this group's S^T columns
                tmem_st8(t_lane + q0 + 8, dk);  // dS^T next to it
                // dS^T row k, queries q0..q0+15: 16-byte chunks q0/8, q0/8+1 of the 128 B row (128B swizzle)
                if (hh == 0 && u >= 2) mbar_wait(&ds_free[u & 1], ((u >> 1) - 1) & 1);
                uint8_t* rowp = ds_buf + k * 128;
                const int c0 = q0 >> 3;
                *(uint4*)(rowp + ((c0 ^ (k & 7)) * 16)) = make_uint4(dk[0], dk[1], dk[2], dk[3]);
                *(uint4*)(rowp + (((c0 + 1) ^ (k & 7)) * 16)) = make_uint4(dk[4], dk[5], dk[6], dk[7]);
                tmem_st_wait();
                fence_proxy_async();
                fence_before();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&sm_done[hh]);
                    if (hh == 1) mbar_arrive(&ds_full[u & 1]);
                }
                if (hh == 0 && i == first_i(j) && j > 0) drain_kv(j - 1);
            }
        }
        drain_kv(nj - 1);
    } else {
        // ------------------------------------------------ 4 dQ warps (thread = head dim d)
        const int d = (warp - 8) * 32 + lane;
        const uint32_t t_row = tmem + ((uint32_t)((warp - 8) * 32) << 16) + 384;
        for (int u = 0; u < nsteps; ++u) {
            int j, i;
            step_ji8<CAUSAL>(u, nj, nq, j, i);
            const bool last = j == (CAUSAL ? i / 2 : nj - 1), dbg = ba.dbg & 2;
            float* acc = ba.dqacc + ((bh * S) + (long long)i * B8_QT) * B8_D + d;  // [query][dim] of this block
            mbar_wait(dq_full, u & 1);
            fence_after();
#pragma unroll 1
            for (int pss = 0; pss < 2; ++pss) {
                uint32_t r[32];
                tmem_ld32_nowait(t_row + pss * 32, r);
                tmem_ld_wait();
                if (pss == 1) {
                    fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(dq_free);
                }
                if (dbg) continue;
                if (!last) {
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        float* p = acc + (long long)(pss * 32 + c) * B8_D;
                        if (j == 0) __stcg(p, __uint_as_float(r[c]));
                        else atomicAdd(p, __uint_as_float(r[c]));  // (one writer per address: ordered)
                    }
                    continue;
                }
                float f[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) f[c] = j > 0 ? __ldcg(acc + (long long)(pss * 32 + c) * B8_D) : 0.f;
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const long long q = row_base + (long long)i * B8_QT + pss * 32 + c;
                    bf16* o = ba.dq + q * ba.ld_dq + (long long)h * B8_D + d;
                    float v = (f[c] + __uint_as_float(r[c])) * ba.scale;
                    if (ba.acc & 1) v += __bfloat162float(*o);
                    *o = __float2bfloat16_rn(v);
                }
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == W8_MMA) {
        fence_after();
        tmem_dealloc<512>(tmem);
    }
}

bool bwd_fits(const Attn& a, const void* dout, i64 ld_do, i64 ld_dq, i64 ld_dk, i64 ld_dv) {
    if (!fwd_fits(a)) return false;
    if (a.thr && !a.mask_t) return false;
    auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    if (!al(dout) || ld_do % 8 || ld_dq % 8 || ld_dk % 8 || ld_dv % 8) return false;
    return true;
}

struct BwdWs {
    float* lse2;
    float* delta;
    float* dqacc;
};
size_t carve(const Attn& a, void* base, BwdWs* w) {
    const size_t rows = (size_t)(a.B * a.nh * a.S);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~(size_t)255;
        return o;
    };
    size_t o_l = take(rows * 4), o_d = take(rows * 4), o_q = take(rows * (size_t)std::max<i64>(a.hd, FD) * 4);
    if (w) {
        char* c = (char*)base;
        *w = BwdWs{(float*)(c + o_l), (float*)(c + o_d), (float*)(c + o_q)};
    }
    return off;
}

}  // namespace

bool attn_fwd_sm100_try(const Attn& a, cudaStream_t s) {
    static int nt_env = getenv("SB_ATTN_FWD_NT") ? atoi(getenv("SB_ATTN_FWD_NT")) : 6;
    if (a.hd == 128) {  // head dim 128 (GPT-Neo, C4): the 64-key-chunk kernel, two CTAs per SM
        if (!fwd_fits(a, 128)) return false;
        CUtensorMap tq, tk6, tv6, tm6;
        const long long rows = a.B * a.S, krows = a.B * a.keys(), cols = a.nh * 128;
        if (!make_map_bf16(&tq, a.q, cols, rows, a.ld_q, FT) || !make_map_bf16(&tk6, a.k, cols, krows, a.ld_k, KC6) ||
            !make_map_bf16(&tv6, a.v, cols, krows, a.ld_v, KC6))
            return false;
        memset(&tm6, 0, sizeof(tm6));
        if (a.thr && !make_map_u32(&tm6, a.mask, a.keys() / 32, a.B * a.nh * a.S, a.keys() / 32, 2 * KC6 / 32, FT))
            return false;
        FwdArgs fa{(bf16*)a.o, a.ld_o, a.lse, a.thr ? a.mask : nullptr, a.thr ? a.dscale : 1.f,
                   a.scale * 1.4426950408889634f, (int)a.S, (int)a.nh, 0};
        fa.Sk = (int)a.keys();
        if (const char* e = getenv("SB_ATTN_DBG")) fa.dbg = atoi(e);
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_fa6_fwd<false, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, F6<128>::SMEM);
            cudaFuncSetAttribute(k_fa6_fwd<true, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, F6<128>::SMEM);
            attr = true;
        }
        static int sms = 0;
        if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        const long long ntiles = a.B * a.nh * (a.S / FT);
        const int grid = (int)std::min<long long>(ntiles, (long long)F6<128>::CTAS * sms);
        if (a.causal) k_fa6_fwd<true, 128><<<grid, F6_THREADS, F6<128>::SMEM, s>>>(tq, tk6, tv6, tm6, fa, (int)ntiles);
        else k_fa6_fwd<false, 128><<<grid, F6_THREADS, F6<128>::SMEM, s>>>(tq, tk6, tv6, tm6, fa, (int)ntiles);
        SBK_CHECK_LAUNCH();
        return true;
    }
    if ((a.causal && nt_env != 6) || !fwd_fits(a)) return false;  // causal: the 64-key-chunk kernel only
    if (a.keys() != a.S && nt_env != 6) return false;               // cross-attention likewise
    CUtensorMap tq, tk, tv, tm;
    const long long rows = a.B * a.S, cols = a.nh * FD;
    if (!make_map_bf16(&tq, a.q, cols, rows, a.ld_q, FT) || !make_map_bf16(&tk, a.k, cols, rows, a.ld_k, FT) ||
        !make_map_bf16(&tv, a.v, cols, rows, a.ld_v, FT))
        return false;
    memset(&tm, 0, sizeof(tm));
    if (a.thr && !make_map_u32(&tm, a.mask, a.S / 32, a.B * a.nh * a.S, a.S / 32, FT / 32, FT)) return false;
    FwdArgs fa{(bf16*)a.o, a.ld_o, a.lse, a.thr ? a.mask : nullptr, a.thr ? a.dscale : 1.f,
               a.scale * 1.4426950408889634f, (int)a.S, (int)a.nh, 0};
    if (const char* e = getenv("SB_ATTN_DBG")) fa.dbg = atoi(e);
    auto go = [&](auto ntc) {
        constexpr int NT = decltype(ntc)::value;
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_fa5_fwd<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, FCfg<NT>::SMEM);
            attr = true;
        }
        dim3 grid((unsigned)((a.S / FT + NT - 1) / NT), (unsigned)a.nh, (unsigned)a.B);
        k_fa5_fwd<NT><<<grid, FCfg<NT>::THREADS, FCfg<NT>::SMEM, s>>>(tq, tk, tv, tm, fa);
    };
    if (nt_env == 6) {
        CUtensorMap tk6, tv6, tm6;
        const long long krows = a.B * a.keys();
        if (!make_map_bf16(&tk6, a.k, cols, krows, a.ld_k, KC6) || !make_map_bf16(&tv6, a.v, cols, krows, a.ld_v, KC6))
            return false;
        memset(&tm6, 0, sizeof(tm6));
        if (a.thr && !make_map_u32(&tm6, a.mask, a.keys() / 32, a.B * a.nh * a.S, a.keys() / 32, 2 * KC6 / 32, FT))
            return false;
        fa.Sk = (int)a.keys();
        static bool attr6 = false;
        if (!attr6) {
            cudaFuncSetAttribute(k_fa6_fwd<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, F6_SMEM);
            cudaFuncSetAttribute(k_fa6_fwd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, F6_SMEM);
            attr6 = true;
        }
        static int sms = 0;
        if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        const long long ntiles = a.B * a.nh * (a.S / FT);
        const int grid = (int)std::min<long long>(ntiles, (long long)F6_CTAS * sms);
        if (a.causal) k_fa6_fwd<true><<<grid, F6_THREADS, F6_SMEM, s>>>(tq, tk6, tv6, tm6, fa, (int)ntiles);
        else k_fa6_fwd<false><<<grid, F6_THREADS, F6_SMEM, s>>>(tq, tk6, tv6, tm6, fa, (int)ntiles);
    } else if (nt_env == 2) go(std::integral_constant<int, 2>{});
    else go(std::integral_constant<int, 1>{});
    SBK_CHECK_LAUNCH();
    return true;
}

}  // namespace sbk

namespace sbk {

size_t attn_bwd_sm100_workspace(i64 B, i64 S, i64 nh, i64 hd) {
    Attn a;
    a.B = B;
    a.S = S;
    a.nh = nh;
    a.hd = hd;
    return carve(a, nullptr, nullptr);
}

static bool attn_bwd_hd128(const Attn& a, const void* dout, i64 ld_do, void* dq, void* dk, void* dv, i64 ld_dq,
                           i64 ld_dk, i64 ld_dv, void* ws, cudaStream_t s) {
    if (!fwd_fits(a, 128) || (a.thr && !a.mask_t)) return false;
    auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    if (!al(dout) || ld_do % 8 || ((uintptr_t)dq & 1) || ((uintptr_t)dk & 15) || ((uintptr_t)dv & 15) || ld_dk % 8 ||
        ld_dv % 8)
        return false;
    CUtensorMap tq, tk, tv, tdo, tm;
    const long long rows = a.B * a.S, krows = a.B * a.keys(), cols = a.nh * 128;
    if (!make_map_bf16(&tq, a.q, cols, rows, a.ld_q, B8_QT) || !make_map_bf16(&tk, a.k, cols, krows, a.ld_k, FT) ||
        !make_map_bf16(&tv, a.v, cols, krows, a.ld_v, FT) || !make_map_bf16(&tdo, dout, cols, rows, ld_do, B8_QT))
        return false;
    memset(&tm, 0, sizeof(tm));
    // transposed keep bits: a row per key, words over the queries
    if (a.thr && !make_map_u32(&tm, a.mask_t, a.S / 32, a.B * a.nh * a.keys(), a.S / 32, 4, FT)) return false;
    BwdWs w;
    carve(a, ws, &w);
    const long long BH = a.B * a.nh, n = BH * a.S;
    k_fa5_prep<128><<<(unsigned)((n * 16 + 255) / 256), 256, 0, s>>>((const bf16*)dout, ld_do, (const bf16*)a.o, a.ld_o,
                                                                    a.lse, w.lse2, w.delta, BH, (int)a.S, (int)a.nh, -1.f);
    SBK_CHECK_LAUNCH();
    BwdArgs ba{w.lse2, w.delta, w.dqacc, a.thr ? a.mask_t : nullptr, a.thr ? a.dscale : 1.f,
               a.scale * 1.4426950408889634f, a.scale, (bf16*)dq, (bf16*)dk, (bf16*)dv, ld_dq, ld_dk, ld_dv,
               (int)a.S, (int)a.nh, a.acc_mask, 0};
    ba.Sk = (int)a.keys();
    if (const char* e = getenv("SB_ATTN_DBG")) ba.dbg = atoi(e);
    ba.ts = nullptr;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_fa8_bwd<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, B8_SMEM);
        cudaFuncSetAttribute(k_fa8_bwd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, B8_SMEM);
        attr = true;
    }
    dim3 grid((unsigned)a.nh, (unsigned)a.B);
    if (a.causal) k_fa8_bwd<true><<<grid, B8_WARPS * 32, B8_SMEM, s>>>(tk, tv, tq, tdo, tm, ba);
    else k_fa8_bwd<false><<<grid, B8_WARPS * 32, B8_SMEM, s>>>(tk, tv, tq, tdo, tm, ba);
    SBK_CHECK_LAUNCH();
    return true;
}

bool attn_bwd_sm100_try(const Attn& a, const void* dout, i64 ld_do, void* dq, void* dk, void* dv, i64 ld_dq, i64 ld_dk,
                        i64 ld_dv, void* ws, cudaStream_t s) {
    if (a.hd == 128) return attn_bwd_hd128(a, dout, ld_do, dq, dk, dv, ld_dq, ld_dk, ld_dv, ws, s);
    if (!bwd_fits(a, dout, ld_do, ld_dq, ld_dk, ld_dv)) return false;
    // fa5 (A/B only): neither causal nor cross-attention
    if ((a.causal || a.keys() != a.S) && getenv("SB_ATTN_BWD") && atoi(getenv("SB_ATTN_BWD")) == 5) return false;
    CUtensorMap tq, tk, tv, tdo, tm;
    const long long rows = a.B * a.S, krows = a.B * a.keys(), cols = a.nh * FD;
    if (!make_map_bf16(&tq, a.q, cols, rows, a.ld_q, FT) || !make_map_bf16(&tk, a.k, cols, krows, a.ld_k, FT) ||
        !make_map_bf16(&tv, a.v, cols, krows, a.ld_v, FT) || !make_map_bf16(&tdo, dout, cols, rows, ld_do, FT))
        return false;
    memset(&tm, 0, sizeof(tm));
    // transposed keep bits: a row per key, words over the queries
    if (a.thr && !make_map_u32(&tm, a.mask_t, a.S / 32, a.B * a.nh * a.keys(), a.S / 32, FT / 32, FT)) return false;
    BwdWs w;
    carve(a, ws, &w);
    const long long BH = a.B * a.nh;
    const long long n = BH * a.S;
    // SB_ATTN_BWD=5 selects the round-1 kernel (A/B runs); v7 reads lse2 and delta negated
    static const int ver = getenv("SB_ATTN_BWD") ? atoi(getenv("SB_ATTN_BWD")) : 7;
    k_fa5_prep<FD><<<(unsigned)((n * 8 + 255) / 256), 256, 0, s>>>((const bf16*)dout, ld_do, (const bf16*)a.o, a.ld_o, a.lse,
                                                              w.lse2, w.delta, BH, (int)a.S, (int)a.nh,
                                                              ver == 5 ? 1.f : -1.f);
    SBK_CHECK_LAUNCH();
    BwdArgs ba{w.lse2, w.delta, w.dqacc, a.thr ? a.mask_t : nullptr, a.thr ? a.dscale : 1.f,
               a.scale * 1.4426950408889634f, a.scale, (bf16*)dq, (bf16*)dk, (bf16*)dv, ld_dq, ld_dk, ld_dv,
               (int)a.S, (int)a.nh, a.acc_mask, 0};
    ba.Sk = (int)a.keys();
    if (const char* e = getenv("SB_ATTN_DBG")) ba.dbg = atoi(e);
    ba.ts = nullptr;
    static unsigned long long* ts_buf = nullptr;
    if (getenv("SB_ATTN_TS")) {
        if (!ts_buf) cudaMalloc(&ts_buf, 16 * 64 * 8);
        cudaMemsetAsync(ts_buf, 0, 16 * 64 * 8, s);
        ba.ts = ts_buf;
    }
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_fa5_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, B_SMEM);
        cudaFuncSetAttribute(k_fa7_bwd<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, B7_SMEM);
        cudaFuncSetAttribute(k_fa7_bwd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, B7_SMEM);
        attr = true;
    }
    dim3 grid((unsigned)a.nh, (unsigned)a.B);
    if (ver == 5) k_fa5_bwd<<<grid, 512, B_SMEM, s>>>(tk, tv, tq, tdo, tm, ba);
    else {
        CUtensorMap tdq, tdk, tdv;
        if (!make_map_bf16_plain(&tdq, dq, cols, rows, ld_dq, 32, 32) || !make_map_bf16_plain(&tdk, dk, cols, krows, ld_dk, 32, 32) ||
            !make_map_bf16_plain(&tdv, dv, cols, krows, ld_dv, 32, 32))
            throw std::runtime_error("attention backward: output tensor maps rejected");
        if (a.causal) k_fa7_bwd<true><<<grid, B7_WARPS * 32, B7_SMEM, s>>>(tk, tv, tq, tdo, tm, tdq, tdk, tdv, ba);
        else k_fa7_bwd<false><<<grid, B7_WARPS * 32, B7_SMEM, s>>>(tk, tv, tq, tdo, tm, tdq, tdk, tdv, ba);
    }
    SBK_CHECK_LAUNCH();
    if (ba.ts) {
        unsigned long long h_ts[16 * 64];
        cudaMemcpyAsync(h_ts, ba.ts, sizeof(h_ts), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        unsigned long long t0 = ~0ull;
        for (auto x : h_ts)
            if (x && x < t0) t0 = x;
        const char* names5[8] = {"prod st_empty ok", "mma sm_done_b ok", "mma sdp(u+1) issued", "mma dq_free ok",
                                 "smax sdp ok", "smax done", "dq dq_full ok", ""};
        const char* names7[8] = {"mma sm_done0 ok", "mma sm_done1 ok", "mma dq issue", "smax sdp0 ok",
                                 "smax h0 done", "smax sdp1 ok", "smax h1 done", "dq dq_full ok"};
        const char** names = ver == 5 ? names5 : names7;
        if (ver != 5) {
            const char* wn[6] = {"u5 h0 done by warp", "u5 h1 done by warp", "u6 h0 done by warp", "u6 h1 done by warp",
                                 "u5 sdp0 ok by warp", "u5 sdp1 ok by warp"};
            for (int r = 8; r < 14; ++r) {
                fprintf(stderr, "%-22s", wn[r - 8]);
                for (int w = 0; w < 16; ++w) fprintf(stderr, " %6lld", h_ts[r * 64 + w] ? (long long)(h_ts[r * 64 + w] - t0) : -1);
                fprintf(stderr, "\n");
            }
        }
        if (ver != 5) {
            const char* pn[2] = {"prod wait st_empty", "prod st_empty ok"};
            for (int r = 14; r < 16; ++r) {
                fprintf(stderr, "%-22s", pn[r - 14]);
                for (int u = 0; u < 16; ++u) fprintf(stderr, " %6lld", h_ts[r * 64 + u] ? (long long)(h_ts[r * 64 + u] - t0) : -1);
                fprintf(stderr, "  cta %s %lld", r == 14 ? "start" : "end", (long long)(h_ts[r * 64 + 63] - t0));
                fprintf(stderr, "\n");
            }
        }
        for (int r = 0; r < (ver == 5 ? 7 : 8); ++r) {
            fprintf(stderr, "%-22s", names[r]);
            for (int u = 0; u < 16; ++u) fprintf(stderr, " %6lld", h_ts[r * 64 + u] ? (long long)(h_ts[r * 64 + u] - t0) : -1);
            fprintf(stderr, "\n");
        }
    }
    return true;
}

}  // namespace sbk
