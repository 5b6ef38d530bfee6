// 2-SM tcgen05 GEMM (cta_group::2) for the Linear layers of the hot path
// (proj/src/executor.cpp:80-133: y = x W^T + b, dx = g W, dW = g^T x).
//
// A cluster of two CTAs (one TPC) computes a 256 x 256 output tile: each CTA
// loads its own 128 rows of A and its own 128-row half of B with TMA
// (128B swizzle), and the leader CTA issues tcgen05.mma.cta_group::2 with
// M = 256, N = 256 that reads both CTAs' shared memory — half the per-SM
// operand traffic of the 1-SM kernel (gemm_tc.cu) for the same MMA rate. Each
// CTA's TMEM holds its 128 accumulator rows, double-buffered (2 x 256 columns)
// so the epilogue of tile i overlaps the MMAs of tile i+1.
//
// Warp roles per CTA (320 threads): warp 0 TMA producer, warp 1 TMEM
// allocator + (leader only) the single MMA-issuing thread, warps 2-9 epilogue
// (TMEM lane quarter = warp % 4, two warps per quarter). The epilogue applies
// alpha / bias / GeLU (+ pre-activation side output) / dGeLU in registers,
// stages 32 x 32 chunks in shared memory and writes them with TMA bulk tensor
// stores (coalesced, asynchronous); an accumulating epilogue (C += ...) reads
// and writes C directly.
//
// Barriers: full[s] lives in the leader (count 2: the leader's expect_tx and
// the follower's remote arrive; both CTAs' TMA loads complete_tx on it),
// empty[s] / tfull[a] in both CTAs (the MMA commit multicasts to the pair),
// tempty[a] in the leader (16 arrivals: 8 epilogue warps x 2 CTAs).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "tc5.cuh"

namespace sbk {

using namespace tc5;

namespace {

constexpr int G_BM = 128;  // rows of A per CTA (cluster tile M = 256)
constexpr int G_BK = 64;
constexpr int G_A = G_BM * G_BK * 2;  // 16 KB
constexpr int G_EPI_BUF = 4096;       // one staging slot per epilogue warp: 32 rows x 128 B
// cluster tile N = BN (256 or 128: the narrower tile evens out the last wave of
// N = 1024 problems); each CTA loads BN/2 rows of B per stage
template <int BN>
struct Cfg {
    static constexpr int B_BYTES = (BN / 2) * G_BK * 2;
    static constexpr int STAGE = G_A + B_BYTES;
#ifndef G2_ST256
#define G2_ST256 6
#endif
#ifndef G2_ST128
#define G2_ST128 8
#endif
    static constexpr int ST = BN == 256 ? G2_ST256 : G2_ST128;
    static constexpr int SMEM = 1024 + ST * STAGE + 8 * G_EPI_BUF + 256;
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on a peer CTA's mbarrier (default .release.cta semantics, as CUTLASS's ClusterBarrier::arrive(cta))
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_u32(uint32_t addr, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(addr), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_u32(uint32_t addr, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr),
        "r"(parity)
        : "memory");
}
// TMA load multicast to the CTAs in `mask` (same smem offset in each), completion
// signalled on each destination pair's leader mbarrier
__device__ __forceinline__ void tma_load_2sm_mc(uint32_t dst, const CUtensorMap* map, uint32_t bar_cluster, int c0, int c1,
                                                uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
        "[%0], [%1, {%4, %5}], [%2], %3;" ::"r"(dst),
        "l"((uint64_t)map), "r"(bar_cluster), "h"(mask), "r"(c0), "r"(c1)
        : "memory");
}
// TMA load whose completion is signalled on the leader CTA's mbarrier
__device__ __forceinline__ void tma_load_2sm(uint32_t dst, const CUtensorMap* map, uint32_t bar_cluster, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];" ::"r"(dst),
        "l"((uint64_t)map), "r"(bar_cluster), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"((uint64_t)map),
                 "r"(src), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void mma_cta2(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_mc(uint32_t bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     bar),
                 "h"(mask)
                 : "memory");
}

__device__ __forceinline__ float tanh_fast(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// tanh-GeLU and its derivative with the polynomial folded (5 FP ops + one MUFU):
//   u = x (c + c a x^2);  gelu = 0.5 x (1 + tanh u)
//   gelu' = 0.5 (1 + t) + 0.5 x (1 - t^2) (c + 3 c a x^2)
__device__ __forceinline__ float gelu_fast(float x) {
    const float c = 0.7978845608028654f, ca = 0.7978845608028654f * 0.044715f;
    const float x2 = x * x;
    const float t = tanh_fast(x * fmaf(ca, x2, c));
    const float hx = 0.5f * x;
    return fmaf(hx, t, hx);
}
__device__ __forceinline__ float gelu_grad_fast(float x) {
    const float c = 0.7978845608028654f, ca = 0.7978845608028654f * 0.044715f;
    const float x2 = x * x;
    const float t = tanh_fast(x * fmaf(ca, x2, c));
    const float hx = 0.5f * x;
    return fmaf(0.5f, t, 0.5f) + hx * fmaf(-t, t, 1.f) * fmaf(3.f * ca, x2, c);
}

struct Epi2 {
    void* C;
    long long ldc;
    int c_f32;
    const bf16* bias;
    int gelu;  // 1: C = gelu(v), aux = v;  2: C = gelu'(aux) * v
    bf16* aux;
    int accumulate;  // C += v (direct stores; no TMA store)
    float alpha;
    int partial;  // split-K: fp32 partials through tC at row z*M + m
    long long M, N;
    unsigned long long* ts;  // debugging timeline (SB_GEMM_TS): cluster 0, [role][k-block]
    float* colsum;           // column sums of the output per 32 rows ([M/32][N]) or null
};
__device__ __forceinline__ unsigned long long gtime2() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
struct Sched2 {
    int m_blks, n_blks, splits, kblocks;  // pair tiles of 256 x BN, k-blocks per split
    int pairs;                            // CTA pairs per cluster (N-adjacent tiles)
    __host__ __device__ int tiles() const { return m_blks * (n_blks / pairs) * splits; }  // cluster tiles
};

// PAIRS = 2: a cluster of two CTA pairs computes two N-adjacent 256 x BN tiles that
// share their A rows; each pair loads half of the A block and multicasts it to both
// pairs (a quarter less L2->SM traffic per stage), so every stage is freed only
// when both pairs' MMAs have consumed it.
template <int G_BN, bool A_MN, bool B_MN, int PAIRS>
__global__ void __cluster_dims__(2 * PAIRS, 1, 1) __launch_bounds__(320, 1)
    k_gemm2(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
            const __grid_constant__ CUtensorMap tC, const __grid_constant__ CUtensorMap tX, Epi2 ep, Sched2 sc) {
    constexpr int G_ST = Cfg<G_BN>::ST, G_STAGE = Cfg<G_BN>::STAGE;
    extern __shared__ uint8_t smem_raw[];
    // 1024-aligned, derived from smem_raw by pointer arithmetic so accesses stay ld/st.shared
    uint8_t* smem = smem_raw + ((1024 - (tc5::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* epi = smem + G_ST * G_STAGE;  // [8 warps][4 KB staging]
    uint64_t* full = (uint64_t*)(epi + 8 * G_EPI_BUF);
    uint64_t* empty = full + G_ST;
    uint64_t* tfull = empty + G_ST;   // [2]
    uint64_t* tempty = tfull + 2;     // [2]
    uint32_t* tslot = (uint32_t*)(tempty + 2);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t crank = cluster_rank();
    const uint32_t rank = crank & 1u, pair = crank >> 1, lead_rank = crank & ~1u;  // rank in the pair
    const bool leader = rank == 0;
    const int cluster = blockIdx.x / (2 * PAIRS), nclusters = gridDim.x / (2 * PAIRS);
    const int ntiles = sc.tiles();

    if (threadIdx.x == 0) {
        tma_prefetch(&tA);
        tma_prefetch(&tB);
        if (!ep.accumulate) tma_prefetch(&tC);
        if (ep.gelu == 1) tma_prefetch(&tX);
        for (int s = 0; s < G_ST; ++s) {
            mbar_init(&full[s], 2);
            mbar_init(&empty[s], PAIRS);  // freed by every pair's MMA commit
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 16);
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_before();
    cluster_sync_all();  // barriers of both CTAs initialised, TMEM allocated
    fence_after();
    const uint32_t tmem = *tslot;

    auto tile_coords = [&](int tile, int& m0, int& n0, int& z) {  // this pair's tile of the cluster tile
        const int ncl = sc.n_blks / PAIRS, per = sc.m_blks * ncl;
        z = tile / per;
        const int r = tile % per;
        m0 = (r / ncl) * 256;  // consecutive tiles share the A row block (L2 reuse)
        n0 = ((r % ncl) * PAIRS + (int)pair) * G_BN;
    };

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer (both CTAs): this CTA's halves of A and B
            const uint32_t sbase = smem_u32(smem);
            int it = 0;
            for (int tile = cluster; tile < ntiles; tile += nclusters) {
                int m0, n0, z;
                tile_coords(tile, m0, n0, z);
                const int ma = m0 + (int)rank * G_BM, nb = n0 + (int)rank * (G_BN / 2);
                for (int kb = 0; kb < sc.kblocks; ++kb, ++it) {
                    const int s = it % G_ST;
                    mbar_wait(&empty[s], ((it / G_ST) & 1) ^ 1);
                    if (ep.ts && cluster == 0 && it < 128) ep.ts[rank * 128 + it] = gtime2();
                    const uint32_t fb_local = smem_u32(&full[s]);
                    const uint32_t fb = mapa_shared(fb_local, lead_rank);
                    if (leader) mbar_expect_tx_u32(fb_local, 2 * G_STAGE);
                    else mbar_arrive_cluster(fb);
                    const uint32_t sa = sbase + s * G_STAGE, sb = sa + G_A;
                    const int kc = (z * sc.kblocks + kb) * G_BK;
                    if (PAIRS == 2) {  // this pair's 64-row share of the A block, to both pairs
                        const uint16_t mc = (uint16_t)((1u << rank) | (1u << (rank + 2)));
                        if (A_MN) tma_load_2sm_mc(sa + pair * 8192, &tA, fb, ma + (int)pair * 64, kc, mc);
                        else tma_load_2sm_mc(sa + pair * 8192, &tA, fb, kc, ma + (int)pair * 64, mc);
                    } else if (A_MN) {
                        tma_load_2sm(sa, &tA, fb, ma, kc);
                        tma_load_2sm(sa + 8192, &tA, fb, ma + 64, kc);
                    } else {
                        tma_load_2sm(sa, &tA, fb, kc, ma);
                    }
                    if (B_MN) {
                        tma_load_2sm(sb, &tB, fb, nb, kc);
                        if (G_BN == 256) tma_load_2sm(sb + 8192, &tB, fb, nb + 64, kc);
                    } else {
                        tma_load_2sm(sb, &tB, fb, kc, nb);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            // ---------------- MMA issuer (leader CTA, one thread for the pair)
            constexpr uint32_t idesc = idesc_bf16(256, G_BN, A_MN, B_MN);
            const uint32_t sbase = smem_u32(smem);
            int it = 0, lt = 0;
            for (int tile = cluster; tile < ntiles; tile += nclusters, ++lt) {
                const int acc = lt & 1;
                mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);  // both CTAs drained this accumulator
                fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * G_BN);
                for (int kb = 0; kb < sc.kblocks; ++kb, ++it) {
                    const int s = it % G_ST;
                    mbar_wait(&full[s], (it / G_ST) & 1);
                    fence_after();
                    if (ep.ts && cluster == 0 && it < 128) ep.ts[2 * 128 + it] = gtime2();
                    const uint32_t a_base = sbase + s * G_STAGE, b_base = a_base + G_A;
#pragma unroll
                    for (int k = 0; k < G_BK / 16; ++k) {
                        const uint64_t da = A_MN ? sdesc(a_base + k * 2048, 8192 >> 4, 1024 >> 4)
                                                 : sdesc(a_base + k * 32, 1, 1024 >> 4);
                        const uint64_t db = B_MN ? sdesc(b_base + k * 2048, 8192 >> 4, 1024 >> 4)
                                                 : sdesc(b_base + k * 32, 1, 1024 >> 4);
                        mma_cta2(d, da, db, idesc, (kb | k) != 0);
                    }
                    commit_mc(smem_u32(&empty[s]), PAIRS == 2 ? 0xF : 0x3);  // frees this stage in every CTA
                }
                commit_mc(smem_u32(&tfull[acc]), (uint16_t)(0x3u << (2 * pair)));  // accumulator complete in the pair
            }
        }
    } else {
        // ---------------- epilogue: TMEM -> registers -> smem -> TMA store
        const int q = warp & 3, half = (warp - 2) / 4;
        uint8_t* mybuf = epi + (warp - 2) * G_EPI_BUF;
        const uint32_t tempty0 = mapa_shared(smem_u32(&tempty[0]), lead_rank);
        int lt = 0, nst = 0;
        // dGeLU epilogue: each lane's 64 B of the pre-activation (its row, the chunk's 32
        // columns) loaded straight into registers two chunks ahead — the first two of a
        // tile are issued before the accumulator wait, so their latency hides behind it.
        // Ragged edges (M, N multiples of 32, not of the tile): the TMA loads zero-fill
        // beyond M / N and the TMA stores clip, so only the direct global accesses (bias,
        // pre-activation, accumulate, split-K rows) skip a warp's chunks past the edge.
        uint4 axa[4], axb[4];
        auto aux_ld = [&](uint4(&w)[4], long long row, long long col) {
            const uint4* src = (const uint4*)(ep.aux + row * ep.ldc + col);
#pragma unroll
            for (int j = 0; j < 4; ++j) w[j] = __ldg(src + j);
        };
        for (int tile = cluster; tile < ntiles; tile += nclusters, ++lt) {
            const int acc = lt & 1;
            int m0, n0, z;
            tile_coords(tile, m0, n0, z);
            const long long row0 = m0 + (long long)rank * G_BM + q * 32;  // first row of this warp
            const bool row_ok = row0 < ep.M;
            if ((ep.gelu == 2 || ep.gelu == 4) && row_ok) {
                if (n0 + half * 32 < ep.N) aux_ld(axa, row0 + lane, n0 + half * 32);
                if (half + 2 < G_BN / 32 && n0 + (half + 2) * 32 < ep.N) aux_ld(axb, row0 + lane, n0 + (half + 2) * 32);
            }
            mbar_wait(&tfull[acc], (lt >> 1) & 1);
            fence_after();
#pragma unroll 1
            for (int c = half; c < G_BN / 32; c += 2) {
                uint32_t r[32];
                tmem_ld32_nowait(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * G_BN + c * 32), r);
                tmem_ld_wait();
                if (c + 2 >= G_BN / 32) {  // last TMEM read of this tile by this warp
                    fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(tempty0 + acc * 8);
                }
                const long long col = n0 + c * 32;
                if (!row_ok || col >= ep.N) continue;  // past the ragged edge (later chunks too)
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * ep.alpha;
                const long long row = row0 + lane;
                if (ep.partial) {
                    // fp32 split-K partial: staging [32 rows][128 B], 128B swizzle
                    uint8_t* buf = mybuf;
                    if (nst >= 1 && lane == 0) bulk_wait_read<0>();
                    __syncwarp();
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        *(float4*)(buf + lane * 128 + ((u ^ (lane & 7)) << 4)) =
                            make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_2d(&tC, smem_u32(buf), (int)col, (int)(z * ep.M + row0));
                        bulk_commit();
                    }
                    ++nst;
                    continue;
                }
                if (ep.bias) {
                    const uint4* bp = (const uint4*)(ep.bias + col);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        uint4 w = __ldg(bp + j);
                        const bf16* e = (const bf16*)&w;
#pragma unroll
                        for (int t = 0; t < 8; ++t) v[8 * j + t] += __bfloat162float(e[t]);
                    }
                }
                uint32_t pre[16];
                if (ep.gelu == 1) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) pre[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = gelu_fast(v[j]);
                } else if (ep.gelu == 3) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
                } else if (ep.gelu == 2 || ep.gelu == 4) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const bf16* e = (const bf16*)&axa[j];
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            const float a = __bfloat162float(e[t]);
                            v[8 * j + t] = ep.gelu == 2 ? v[8 * j + t] * gelu_grad_fast(a) : (a > 0.f ? v[8 * j + t] : 0.f);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) axa[j] = axb[j];
                    if (c + 4 < G_BN / 32 && col + 128 < ep.N) aux_ld(axb, row, col + 128);  // this warp's chunk after next
                }
                if (ep.accumulate) {
                    // C += v, direct read-modify-write of this thread's row
                    if (ep.c_f32) {
                        float4* dst = (float4*)((float*)ep.C + row * ep.ldc + col);
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            float4 p = dst[j];
                            dst[j] = make_float4(v[4 * j] + p.x, v[4 * j + 1] + p.y, v[4 * j + 2] + p.z,
                                                 v[4 * j + 3] + p.w);
                        }
                    } else {
                        uint4* dst = (uint4*)((bf16*)ep.C + row * ep.ldc + col);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            uint4 p = dst[j];
                            const bf16* pe = (const bf16*)&p;
                            uint4 w;
                            uint32_t* wp = (uint32_t*)&w;
#pragma unroll
                            for (int t = 0; t < 4; ++t)
                                wp[t] = pack_bf16(v[8 * j + 2 * t] + __bfloat162float(pe[2 * t]),
                                                  v[8 * j + 2 * t + 1] + __bfloat162float(pe[2 * t + 1]));
                            dst[j] = w;
                        }
                    }
                    continue;
                }
                if (ep.colsum) {
                    // this warp's 32 rows summed per column (a bias gradient's partial): a
                    // reduce-scatter across the lanes, halving the columns each level, ends
                    // with lane L holding column L (fixed order: deterministic)
                    float t16[16], t8[8], t4[4], t2[2];
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const bool up = lane & 16;
                        t16[c] = (up ? v[c + 16] : v[c]) + __shfl_xor_sync(0xffffffffu, up ? v[c] : v[c + 16], 16);
                    }
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const bool up = lane & 8;
                        t8[c] = (up ? t16[c + 8] : t16[c]) + __shfl_xor_sync(0xffffffffu, up ? t16[c] : t16[c + 8], 8);
                    }
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const bool up = lane & 4;
                        t4[c] = (up ? t8[c + 4] : t8[c]) + __shfl_xor_sync(0xffffffffu, up ? t8[c] : t8[c + 4], 4);
                    }
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const bool up = lane & 2;
                        t2[c] = (up ? t4[c + 2] : t4[c]) + __shfl_xor_sync(0xffffffffu, up ? t4[c] : t4[c + 2], 2);
                    }
                    const bool up = lane & 1;
                    const float t1 = (up ? t2[1] : t2[0]) + __shfl_xor_sync(0xffffffffu, up ? t2[0] : t2[1], 1);
                    ep.colsum[(row0 >> 5) * ep.N + col + lane] = t1;
                }
                uint8_t* buf = mybuf;
                if (nst >= 1 && lane == 0) bulk_wait_read<0>();
                __syncwarp();
                if (ep.c_f32) {
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        *(float4*)(buf + lane * 128 + ((u ^ (lane & 7)) << 4)) =
                            make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
                } else {
                    // bf16: [32 rows][64 B], 64B swizzle (16-byte unit ^ (row >> 1) & 3); aux in the upper 2 KB
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int pu = (u ^ ((lane >> 1) & 3)) << 4;
                        *(uint4*)(buf + lane * 64 + pu) =
                            make_uint4(pack_bf16(v[8 * u], v[8 * u + 1]), pack_bf16(v[8 * u + 2], v[8 * u + 3]),
                                       pack_bf16(v[8 * u + 4], v[8 * u + 5]), pack_bf16(v[8 * u + 6], v[8 * u + 7]));
                        if (ep.gelu == 1)
                            *(uint4*)(buf + 2048 + lane * 64 + pu) =
                                make_uint4(pre[4 * u], pre[4 * u + 1], pre[4 * u + 2], pre[4 * u + 3]);
                    }
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    tma_store_2d(&tC, smem_u32(buf), (int)col, (int)row0);
                    if (ep.gelu == 1) tma_store_2d(&tX, smem_u32(buf + 2048), (int)col, (int)row0);
                    bulk_commit();
                }
                ++nst;
            }
        }
        if (lane == 0) bulk_wait_all();
    }
    __syncwarp();
    fence_before();
    cluster_sync_all();  // no remote arrive or multicast commit targets an exited CTA
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn2() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    });
    return fn;
}

// C / aux / partial store map: box {32 elements, 32 rows}; bf16 rows are 64 B
// (64B swizzle), fp32 rows 128 B (128B swizzle) — matching the staging layout
bool make_store_map(CUtensorMap* m, const void* base, bool f32, long long cols, long long rows, long long ld) {
    auto fn = encode_fn2();
    if (!fn) return false;
    const int es = f32 ? 4 : 2;
    if ((ld * es) % 16 || ((uintptr_t)base & 15)) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t el[2] = {1, 1};
    return fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
              dims, strides, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
              f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int g_sms2 = 0;
int g_sm_reserve = 0;

// co-resident clusters of the persistent kernel (GPCs need not split into whole 4-CTA clusters)
template <int BN, bool A_MN, bool B_MN, int PAIRS>
int max_clusters2() {
    static int mc = 0;
    if (!mc) {
        if (!g_sms2) cudaDeviceGetAttribute(&g_sms2, cudaDevAttrMultiProcessorCount, 0);
        auto k = k_gemm2<BN, A_MN, B_MN, PAIRS>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2 * PAIRS;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(2 * PAIRS * (g_sms2 / (2 * PAIRS)));
        cfg.blockDim = dim3(320);
        cfg.dynamicSmemBytes = Cfg<BN>::SMEM;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&mc, k, &cfg) != cudaSuccess || mc <= 0) mc = g_sms2 / (2 * PAIRS);
        mc = std::min(mc, g_sms2 / (2 * PAIRS));
    }
    return mc;
}

template <int BN, bool A_MN, bool B_MN, int PAIRS>
void launch2(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const CUtensorMap& tx, const Epi2& ep,
             const Sched2& sc, cudaStream_t s) {
    auto k = k_gemm2<BN, A_MN, B_MN, PAIRS>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM);
        attr = true;
    }
    if (!g_sms2) cudaDeviceGetAttribute(&g_sms2, cudaDevAttrMultiProcessorCount, 0);
    int max_clusters = max_clusters2<BN, A_MN, B_MN, PAIRS>();
    // SMs left to a concurrent collective (gemm_set_sm_reserve)
    if (g_sm_reserve > 0) max_clusters = std::max(1, std::min(max_clusters, (g_sms2 - g_sm_reserve) / (2 * PAIRS)));
    const int clusters = std::min(sc.tiles(), max_clusters);
    k<<<clusters * 2 * PAIRS, 320, Cfg<BN>::SMEM, s>>>(ta, tb, tc, tx, ep, sc);
}

}  // namespace

void gemm_set_sm_reserve(int n) { g_sm_reserve = std::max(0, n); }

bool g_tc2_disabled = false;
bool g_tc2_colsum_done = false;
int g_tc2_bn = 0;  // cluster tile N: 0 default (256), 128 or 256 forced (tests)
void gemm2_set_tile_n(int bn) { g_tc2_bn = bn; }

// splitk reduce kernel of gemm_tc.cu
void splitk_reduce_launch(const float* partial, int splits, i64 M, i64 N, void* C, DT tc, i64 ldc, const void* bias,
                          bool accumulate, cudaStream_t s);

bool gemm_tc2_try(const Gemm& g, cudaStream_t s) {
    if (g_tc2_disabled) return false;
    if (g.ta != BF16 || g.tb != BF16 || g.batch != 1 || g.sCn != 1) return false;
    if (g.tc != BF16 && g.tc != F32) return false;
    if (g.epilogue && (g.tc != BF16 || (g.epilogue != 3 && !g.aux))) return false;
    if (g.bias && g.tbias != BF16) return false;
    const bool a_mn = g.sAm == 1 && g.sAk != 1, b_mn = g.sBn == 1 && g.sBk != 1;
    const bool a_k = g.sAk == 1 && !a_mn, b_k = g.sBk == 1 && !b_mn;
    if (!(a_mn || a_k) || !(b_mn || b_k)) return false;
    const long long M = g.M, N = g.N, K = g.K;
    // M, N multiples of 32 (a warp's epilogue chunk): ragged last tiles (TMA zero-fill / clip)
    if (M % 32 || N % 32 || K % G_BK || M <= 0 || N <= 0 || K <= 0) return false;
    const long long lda = a_mn ? g.sAk : g.sAm, ldb = b_mn ? g.sBk : g.sBn, ldc = g.sCm;
    auto al16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    if (lda % 8 || ldb % 8 || ldc % 8 || !al16(g.A) || !al16(g.B) || !al16(g.C)) return false;
    if (g.aux && !al16(g.aux)) return false;
    CUtensorMap ta, tb, tc, tx;
    memset(&tc, 0, sizeof(tc));
    memset(&tx, 0, sizeof(tx));
    if (!g_sms2) cudaDeviceGetAttribute(&g_sms2, cudaDevAttrMultiProcessorCount, 0);
    // tile N 256 (measured: the 256x128 tile, though it evens out the last wave of
    // N = 1024 problems, runs 30-40% slower on the BERT-large shapes)
    const int G_BN = g_tc2_bn ? g_tc2_bn : 256;
    // two CTA pairs per cluster sharing A (multicast) for mainloop-dominated problems
    // (K >= 4096) when N holds an even number of tiles: a quarter less L2->SM traffic per
    // stage, but 4-CTA clusters fit only 33 per chip (132 SMs): measured +2-3% on
    // K = 4096 / 16384, -3-6% on the K = 1024 GEMMs with GeLU / dGeLU / bias epilogues
    static const int pairs_env = getenv("SB_GEMM_PAIRS") ? atoi(getenv("SB_GEMM_PAIRS")) : 0;
    const long long m_blks = (M + 255) / 256, n_blks = (N + G_BN - 1) / G_BN;
    const int pairs = n_blks % 2 ? 1 : pairs_env ? pairs_env : (K >= 4096 ? 2 : 1);
    // pair slots of the persistent grid (the split-K model below counts waves in them)
    const int clusters = pairs == 2 ? 2 * (G_BN == 256 ? max_clusters2<256, false, false, 2>()
                                                       : max_clusters2<128, false, false, 2>())
                                    : g_sms2 / 2;
    if (!(a_mn ? make_map_bf16(&ta, g.A, M, K, lda, 64) : make_map_bf16(&ta, g.A, K, M, lda, pairs == 2 ? 64 : G_BM)))
        return false;
    if (!(b_mn ? make_map_bf16(&tb, g.B, N, K, ldb, 64) : make_map_bf16(&tb, g.B, K, N, ldb, G_BN / 2))) return false;
    const int kblocks = (int)(K / G_BK);
    const long long tiles = m_blks * n_blks;  // pair tiles
    int splits = 1;
    // long-K, few-tile problems (the weight gradients) -> deterministic split-K, with the
    // split count from a wave model: ceil(tiles * s / clusters) waves of kblocks / s
    // k-blocks each (~0.33 us per k-block per tile, measured), plus the fp32 partials'
    // reduce ((s + 1) * M * N * 4 bytes at ~5 TB/s) and its launch (~3 us)
    static const int force = getenv("SB_GEMM_SPLITS") ? atoi(getenv("SB_GEMM_SPLITS")) : 0;
    if (tiles < clusters && kblocks >= 32 && g.ws && !g.epilogue) {
        auto cost = [&](int sp) {
            const double waves = (double)((tiles * sp + clusters - 1) / clusters);
            const double t = waves * (double)kblocks / sp * 0.33e-6;
            return sp == 1 ? t : t + (double)(sp + 1) * M * N * 4 / 5e12 + 3e-6;
        };
        double best = cost(1);
        for (int sp = 2; sp <= 16; ++sp)
            if (kblocks % sp == 0 && kblocks / sp >= 8 && (size_t)sp * M * N * 4 <= g.ws_bytes &&
                (force ? sp == force : cost(sp) < best)) {
                best = cost(sp);
                splits = sp;
            }
        if (force == 1) splits = 1;
    }
    Epi2 ep{};
    ep.C = g.C;
    ep.ldc = ldc;
    ep.c_f32 = g.tc == F32;
    ep.bias = (const bf16*)g.bias;
    ep.gelu = g.epilogue;
    ep.aux = (bf16*)g.aux;
    ep.accumulate = g.accumulate && splits == 1;
    ep.alpha = g.alpha;
    ep.partial = splits > 1;
    ep.M = M;
    ep.N = N;
    ep.colsum = splits == 1 && !ep.accumulate ? g.colsum : nullptr;
    if (splits > 1) {
        if (!make_store_map(&tc, g.ws, true, N, (long long)splits * M, N)) return false;
    } else if (!ep.accumulate) {
        if (!make_store_map(&tc, g.C, ep.c_f32, N, M, ldc)) return false;
    }
    if (g.epilogue == 1 && splits == 1) {  // GeLU: pre-activation store map
        if (!make_store_map(&tx, g.aux, false, N, M, ldc)) return false;
    }
    Sched2 sc{(int)m_blks, (int)n_blks, splits, kblocks / splits, pairs};
    static unsigned long long* ts_buf = nullptr;
    ep.ts = nullptr;
    if (getenv("SB_GEMM_TS")) {
        if (!ts_buf) cudaMalloc(&ts_buf, 3 * 128 * 8);
        cudaMemsetAsync(ts_buf, 0, 3 * 128 * 8, s);
        ep.ts = ts_buf;
    }
    auto go = [&](auto bn) {
        constexpr int BN = decltype(bn)::value;
        auto go2 = [&](auto pc) {
            constexpr int PR = decltype(pc)::value;
            if (!a_mn && !b_mn) launch2<BN, false, false, PR>(ta, tb, tc, tx, ep, sc, s);
            else if (!a_mn && b_mn) launch2<BN, false, true, PR>(ta, tb, tc, tx, ep, sc, s);
            else if (a_mn && b_mn) launch2<BN, true, true, PR>(ta, tb, tc, tx, ep, sc, s);
            else launch2<BN, true, false, PR>(ta, tb, tc, tx, ep, sc, s);
        };
        if (pairs == 2) go2(std::integral_constant<int, 2>{});
        else go2(std::integral_constant<int, 1>{});
    };
    if (G_BN == 256) go(std::integral_constant<int, 256>{});
    else go(std::integral_constant<int, 128>{});
    SBK_CHECK_LAUNCH();
    if (ep.ts) {
        unsigned long long h[3 * 128];
        cudaMemcpyAsync(h, ep.ts, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        const char* nm[3] = {"prod0 empty ok", "prod1 empty ok", "mma full ok"};
        for (int r = 0; r < 3; ++r) {
            fprintf(stderr, "%-16s", nm[r]);
            for (int i = 0; i < 40; ++i) fprintf(stderr, " %5lld", h[r * 128 + i] ? (long long)(h[r * 128 + i] - h[0]) : -1);
            fprintf(stderr, "\n");
        }
    }
    g_tc2_colsum_done = ep.colsum != nullptr;
    if (splits > 1)
        splitk_reduce_launch((const float*)g.ws, splits, M, N, g.C, g.tc, ldc, g.bias, g.accumulate, s);
    return true;
}

}  // namespace sbk
