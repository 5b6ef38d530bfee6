// tcgen05 GEMM for sm_100a: TMA -> shared memory (128B swizzle) -> tcgen05.mma
// with the fp32 accumulator in TMEM -> tcgen05.ld epilogue (alpha, bias, GeLU
// with pre-activation side output, accumulate, bf16/fp32 store).
//
// One kernel covers the three Linear GEMMs of the hot path
// (proj/src/executor.cpp:80-133):
//   forward  y  = x W^T : A K-major, B K-major
//   dgrad    dx = g W   : A K-major, B MN-major
//   wgrad    dW = g^T x : A MN-major, B MN-major, long K -> deterministic split-K
// Persistent: one CTA per SM walks a static tile schedule. Warp roles (320
// threads): warp 0 TMA producer, warp 1 TMEM allocator + single-thread MMA
// issuer, warps 2-9 epilogue (TMEM lane quarter = warp % 4, two warps per
// quarter splitting the columns). Two TMEM
// accumulators (2 x BN columns) let the epilogue of tile i overlap the MMAs of
// tile i+1. mbarrier rings: STAGES {full, empty} between TMA and MMA, and
// {tmem_full, tmem_empty} x 2 between MMA and epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "tc5.cuh"

namespace sbk {

namespace {

constexpr int BM = 128, BK = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    // tcgen05 shared-memory matrix descriptor, 128B swizzle, version 1
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(lbo & 0x3FFF) << 16) | ((uint64_t)(sbo & 0x3FFF) << 32) |
           (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// tanh.approx (one MUFU op): the bf16 epilogues do not need tanhf's accuracy
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

struct Epi {
    void* C;
    long long ldc;
    int c_f32;
    const bf16* bias;
    int gelu;        // 1: C = gelu(v), aux = v (forward);  2: C = gelu'(aux) * v (dgrad of a GeLU input)
    bf16* aux;
    int accumulate;
    float alpha;
    float* partial;  // split-K: fp32 partials [split][M][N]
    long long M, N;
};

struct Sched {
    int m_blks, n_blks, splits, kblocks;  // kblocks per split
    __host__ __device__ int tiles() const { return m_blks * n_blks * splits; }
};

__device__ __forceinline__ void tile_coords(const Sched& sc, int tile, int BN, int& m0, int& n0, int& z) {
    int per = sc.m_blks * sc.n_blks;
    z = tile / per;
    int r = tile % per;
    m0 = (r / sc.n_blks) * BM;  // consecutive tiles share the A row block (L2 reuse)
    n0 = (r % sc.n_blks) * BN;
}

template <int BN>
__device__ __forceinline__ void epilogue_chunk(const Epi& ep, int z, long long row, long long col, const uint32_t (&r)[32]) {
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * ep.alpha;
    if (ep.partial) {
        float4* dst = (float4*)(ep.partial + ((long long)z * ep.M + row) * ep.N + col);
#pragma unroll
        for (int j = 0; j < 8; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        return;
    }
    if (ep.bias) {
        const uint4* bp = (const uint4*)(ep.bias + col);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint4 w = bp[j];
            const bf16* e = (const bf16*)&w;
#pragma unroll
            for (int t = 0; t < 8; ++t) v[8 * j + t] += __bfloat162float(e[t]);
        }
    }
    if (ep.gelu == 1) {
        uint4* ax = (uint4*)(ep.aux + row * ep.ldc + col);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint4 w;
            bf16* e = (bf16*)&w;
#pragma unroll
            for (int t = 0; t < 8; ++t) e[t] = __float2bfloat16_rn(v[8 * j + t]);
            ax[j] = w;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = gelu_fast(v[j]);
    } else if (ep.gelu == 2 || ep.gelu == 4) {
        const uint4* ax = (const uint4*)(ep.aux + row * ep.ldc + col);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint4 w = ax[j];
            const bf16* e = (const bf16*)&w;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const float a = __bfloat162float(e[t]);
                v[8 * j + t] = ep.gelu == 2 ? v[8 * j + t] * gelu_grad_fast(a) : (a > 0.f ? v[8 * j + t] : 0.f);
            }
        }
    } else if (ep.gelu == 3) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
    }
    if (ep.c_f32) {
        float4* dst = (float4*)((float*)ep.C + row * ep.ldc + col);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float4 o = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            if (ep.accumulate) {
                float4 p = dst[j];
                o.x += p.x;
                o.y += p.y;
                o.z += p.z;
                o.w += p.w;
            }
            dst[j] = o;
        }
    } else {
        uint4* dst = (uint4*)((bf16*)ep.C + row * ep.ldc + col);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint4 w;
            bf16* e = (bf16*)&w;
            if (ep.accumulate) {
                uint4 p = dst[j];
                const bf16* pe = (const bf16*)&p;
#pragma unroll
                for (int t = 0; t < 8; ++t) e[t] = __float2bfloat16_rn(v[8 * j + t] + __bfloat162float(pe[t]));
            } else {
#pragma unroll
                for (int t = 0; t < 8; ++t) e[t] = __float2bfloat16_rn(v[8 * j + t]);
            }
            dst[j] = w;
        }
    }
}

template <int BN, int STAGES, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(320, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, Epi ep, Sched sc) {
    constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE = A_BYTES + B_BYTES;
    constexpr uint32_t TCOLS = 2 * BN;  // two accumulators
    extern __shared__ uint8_t smem_raw[];
    // 1024-aligned, derived from smem_raw by pointer arithmetic so accesses stay ld/st.shared
    uint8_t* smem = smem_raw + ((1024 - (tc5::smem_u32(smem_raw) & 1023)) & 1023);
    uint64_t* full = (uint64_t*)(smem + STAGES * STAGE);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;  // [2]
    uint64_t* tempty = tfull + 2;      // [2]
    uint32_t* tslot = (uint32_t*)(tempty + 2);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int ntiles = sc.tiles();

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tB) : "memory");
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 8);  // one arrival per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer: all k-blocks of all this CTA's tiles
            int it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                int m0, n0, z;
                tile_coords(sc, tile, BN, m0, n0, z);
                for (int kb = 0; kb < sc.kblocks; ++kb, ++it) {
                    int s = it % STAGES;
                    mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
                    uint8_t* sa = smem + s * STAGE;
                    uint8_t* sbp = sa + A_BYTES;
                    mbar_expect_tx(&full[s], STAGE);
                    int kc = (z * sc.kblocks + kb) * BK;
                    if (A_MN) {
#pragma unroll
                        for (int c = 0; c < BM / 64; ++c) tma_load_2d(sa + c * 8192, &tA, &full[s], m0 + 64 * c, kc);
                    } else {
                        tma_load_2d(sa, &tA, &full[s], kc, m0);
                    }
                    if (B_MN) {
#pragma unroll
                        for (int c = 0; c < BN / 64; ++c) tma_load_2d(sbp + c * 8192, &tB, &full[s], n0 + 64 * c, kc);
                    } else {
                        tma_load_2d(sbp, &tB, &full[s], kc, n0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer (one thread for the whole CTA)
            constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) |
                                       ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
            int it = 0, lt = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {
                const int acc = lt & 1;
                mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);  // epilogue drained this accumulator
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t d = tmem + (uint32_t)(acc * BN);
                for (int kb = 0; kb < sc.kblocks; ++kb, ++it) {
                    int s = it % STAGES;
                    mbar_wait(&full[s], (it / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    uint32_t a_base = smem_u32(smem + s * STAGE), b_base = a_base + A_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        uint64_t da = A_MN ? sdesc(a_base + k * 2048, 8192 >> 4, 1024 >> 4)
                                           : sdesc(a_base + k * 32, 1, 1024 >> 4);
                        uint64_t db = B_MN ? sdesc(b_base + k * 2048, 8192 >> 4, 1024 >> 4)
                                           : sdesc(b_base + k * 32, 1, 1024 >> 4);
                        mma_bf16(d, da, db, idesc, (kb | k) != 0);
                    }
                    mma_commit(&empty[s]);  // frees the smem slot once these MMAs have read it
                }
                mma_commit(&tfull[acc]);  // accumulator complete
            }
        }
    } else {
        // ---------------- epilogue: TMEM -> registers -> global. 8 warps: two per
        // TMEM lane quarter (= warp % 4), splitting the 32-column chunks
        const int q = warp & 3;
        const int half = (warp - 2) / 4;
        int lt = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {
            const int acc = lt & 1;
            int m0, n0, z;
            tile_coords(sc, tile, BN, m0, n0, z);
            const long long row = m0 + q * 32 + lane;
            mbar_wait(&tfull[acc], (lt >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
            for (int c = half; c < BN / 32; c += 2) {
                uint32_t r[32];
                tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c * 32), r);
                epilogue_chunk<BN>(ep, z, row, n0 + c * 32, r);
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
    }
}

// split-K reduction in fixed split order (deterministic), then the epilogue
template <class TC>
__global__ void k_splitk_reduce(const float* partial, int splits, long long M, long long N, TC* C, long long ldc,
                                const bf16* bias, int accumulate) {
    long long total = M * N / 4;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        long long e = i * 4, m = e / N, n = e % N;
        float4 acc = ((const float4*)partial)[i];
        for (int s = 1; s < splits; ++s) {
            float4 p = ((const float4*)(partial + (long long)s * M * N))[i];
            acc.x += p.x;
            acc.y += p.y;
            acc.z += p.z;
            acc.w += p.w;
        }
        float v[4] = {acc.x, acc.y, acc.z, acc.w};
        for (int t = 0; t < 4; ++t) {
            if (bias) v[t] += __bfloat162float(bias[n + t]);
            TC* d = C + m * ldc + n + t;
            if (accumulate) v[t] += to_f(*d);
            *d = from_f<TC>(v[t]);
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// 2D bf16 tensor map: inner dim `inner` (contiguous), `outer` rows with row
// stride `ld` elements, box {64, box_outer}, 128B swizzle.
bool make_map(CUtensorMap* m, const void* base, long long inner, long long outer, long long ld, int box_outer) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
    cuuint32_t box[2] = {64, (cuuint32_t)box_outer};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int g_num_sms = 0;

template <int BN, int STAGES, bool A_MN, bool B_MN>
void launch(const CUtensorMap& ta, const CUtensorMap& tb, const Epi& ep, const Sched& sc, cudaStream_t s) {
    constexpr int smem = STAGES * (BM * BK * 2 + BN * BK * 2) + 1024 + 256;
    auto k = k_gemm_tc<BN, STAGES, A_MN, B_MN>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    if (!g_num_sms) cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, 0);
    int grid = std::min(sc.tiles(), g_num_sms);
    k<<<grid, 320, smem, s>>>(ta, tb, ep, sc);
}

bool g_tc_disabled = false;

}  // namespace

void gemm_tc_disable(bool off) { g_tc_disabled = off; }

void splitk_reduce_launch(const float* partial, int splits, i64 M, i64 N, void* C, DT tc, i64 ldc, const void* bias,
                          bool accumulate, cudaStream_t s) {
    unsigned blocks = grid_for(M * N / 4, 256);
    if (tc == F32)
        k_splitk_reduce<float><<<blocks, 256, 0, s>>>(partial, splits, M, N, (float*)C, ldc, (const bf16*)bias,
                                                      accumulate);
    else
        k_splitk_reduce<bf16><<<blocks, 256, 0, s>>>(partial, splits, M, N, (bf16*)C, ldc, (const bf16*)bias, accumulate);
    SBK_CHECK_LAUNCH();
}

bool tc5::make_map_bf16(CUtensorMap* m, const void* base, long long inner, long long outer, long long ld, int box_outer) {
    return make_map(m, base, inner, outer, ld, box_outer);
}

bool tc5::make_map_bf16_plain(CUtensorMap* m, const void* base, long long inner, long long outer, long long ld,
                              int box_inner, int box_outer) {
    auto fn = encode_fn();
    if (!fn || (ld * 2) % 16 || ((uintptr_t)base & 15)) return false;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
    cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, box_inner * 2 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool tc5::make_map_u32(CUtensorMap* m, const void* base, long long inner, long long outer, long long ld, int box_inner,
                       int box_outer) {
    auto fn = encode_fn();
    if (!fn || (ld * 4) % 16 || ((uintptr_t)base & 15)) return false;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
    cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool gemm_tc_try(const Gemm& g, cudaStream_t s) {
    if (g_tc_disabled) return false;
    if (g.ta != BF16 || g.tb != BF16 || g.batch != 1 || g.sCn != 1) return false;
    if (g.tc != BF16 && g.tc != F32) return false;
    if (g.epilogue && (g.tc != BF16 || (g.epilogue != 3 && !g.aux))) return false;
    if (g.bias && g.tbias != BF16) return false;
    const bool a_mn = g.sAm == 1 && g.sAk != 1, b_mn = g.sBn == 1 && g.sBk != 1;
    const bool a_k = g.sAk == 1 && !a_mn, b_k = g.sBk == 1 && !b_mn;
    if (!(a_mn || a_k) || !(b_mn || b_k)) return false;
    const long long M = g.M, N = g.N, K = g.K;
    if (M % BM || N % 128 || K % BK || M <= 0 || N <= 0 || K <= 0) return false;
    const long long lda = a_mn ? g.sAk : g.sAm, ldb = b_mn ? g.sBk : g.sBn, ldc = g.sCm;
    auto al16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    if (lda % 8 || ldb % 8 || ldc % 8 || !al16(g.A) || !al16(g.B) || !al16(g.C)) return false;
    if (g.aux && !al16(g.aux)) return false;
    const int BNs = (N % 256 == 0) ? 256 : 128;
    CUtensorMap ta, tb;
    // A: K-major (rows M, inner K) or MN-major (rows K, inner M)
    if (!(a_mn ? make_map(&ta, g.A, M, K, lda, 64) : make_map(&ta, g.A, K, M, lda, BM))) return false;
    if (!(b_mn ? make_map(&tb, g.B, N, K, ldb, 64) : make_map(&tb, g.B, K, N, ldb, BNs))) return false;
    int kblocks = (int)(K / BK);
    long long tiles = (M / BM) * (N / BNs);
    int splits = 1;
    // long-K, few-tile problems (the weight gradients) -> deterministic split-K
    if (tiles < 148 && kblocks >= 32 && g.ws && !g.epilogue) {
        int want = (int)((296 + tiles - 1) / tiles);
        for (int sp = std::min(want, 16); sp > 1; --sp)
            if (kblocks % sp == 0 && kblocks / sp >= 8 && (size_t)sp * M * N * 4 <= g.ws_bytes) {
                splits = sp;
                break;
            }
    }
    Epi ep{};
    ep.C = g.C;
    ep.ldc = ldc;
    ep.c_f32 = g.tc == F32;
    ep.bias = (const bf16*)g.bias;
    ep.gelu = g.epilogue;
    ep.aux = (bf16*)g.aux;
    ep.accumulate = g.accumulate;
    ep.alpha = g.alpha;
    ep.partial = splits > 1 ? (float*)g.ws : nullptr;
    ep.M = M;
    ep.N = N;
    Sched sc{(int)(M / BM), (int)(N / BNs), splits, kblocks / splits};
    if (BNs == 256) {
        if (!a_mn && !b_mn) launch<256, 4, false, false>(ta, tb, ep, sc, s);
        else if (!a_mn && b_mn) launch<256, 4, false, true>(ta, tb, ep, sc, s);
        else if (a_mn && b_mn) launch<256, 4, true, true>(ta, tb, ep, sc, s);
        else launch<256, 4, true, false>(ta, tb, ep, sc, s);
    } else {
        if (!a_mn && !b_mn) launch<128, 6, false, false>(ta, tb, ep, sc, s);
        else if (!a_mn && b_mn) launch<128, 6, false, true>(ta, tb, ep, sc, s);
        else if (a_mn && b_mn) launch<128, 6, true, true>(ta, tb, ep, sc, s);
        else launch<128, 6, true, false>(ta, tb, ep, sc, s);
    }
    SBK_CHECK_LAUNCH();
    if (splits > 1) {
        unsigned blocks = grid_for(M * N / 4, 256);
        if (g.tc == F32)
            k_splitk_reduce<float><<<blocks, 256, 0, s>>>((const float*)g.ws, splits, M, N, (float*)g.C, ldc,
                                                           (const bf16*)g.bias, g.accumulate);
        else
            k_splitk_reduce<bf16><<<blocks, 256, 0, s>>>((const float*)g.ws, splits, M, N, (bf16*)g.C, ldc,
                                                          (const bf16*)g.bias, g.accumulate);
        SBK_CHECK_LAUNCH();
    }
    return true;
}

}  // namespace sbk
