// Elementwise / reduction / copy / RNG-dropout / embedding / simulated
// collective kernels. HBM-bound: grid-stride loops, 16-byte vector accesses on
// the hot contiguous paths, deterministic fixed-order reductions (no float
// atomics), so identical runs give identical bits (the reference's
// determinism contract, proj/tests/executor_test.cpp:273-283).
#include <algorithm>

#include "common.cuh"

namespace sbk {

namespace {
float* g_red_ws = nullptr;  // deterministic reduction partials
constexpr int kRedBlocks = 296;
}  // namespace

void init_workspace() {
    if (!g_red_ws) cudaMalloc(&g_red_ws, sizeof(float) * kRedBlocks * 2);
}

// --------------------------------------------------- 16-byte bf16 elementwise
// contiguous bf16 with n % 8 == 0 and 16-byte aligned operands: 8 elements per
// thread and access (same per-element math as the scalar kernels: same bits)
__device__ __forceinline__ void bf8_unpack(const uint4& r, float* f) {
    const __nv_bfloat162* h = (const __nv_bfloat162*)&r;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 v = __bfloat1622float2(h[i]);
        f[2 * i] = v.x;
        f[2 * i + 1] = v.y;
    }
}
__device__ __forceinline__ uint4 bf8_pack(const float* f) {
    uint4 r;
    __nv_bfloat162* h = (__nv_bfloat162*)&r;
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    return r;
}
static bool vec8_ok(i64 n, std::initializer_list<const void*> ps) {
    if (n % 8 || n / 8 >= (1ll << 31)) return false;
    for (const void* p : ps)
        if (((uintptr_t)p & 15) != 0) return false;
    return true;
}
static unsigned vec8_grid(i64 n) { return (unsigned)std::min<i64>((n / 8 + 255) / 256, 148 * 16); }
// kind: 0 fill(c) | 1 unary(op, c) | 2 unary_bwd(op, c) | 3 binary add / mul (op) | 4 y += c x
__global__ void k_vec8(int kind, int op, const uint4* x, const uint4* g, uint4* y, int n8, float c) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += gridDim.x * blockDim.x) {
        float a[8], b[8], o[8];
        if (kind == 0) {
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = c;
        } else if (kind == 1) {
            bf8_unpack(x[i], a);
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = op == 0 ? a[e] * c : op == 1 ? (a[e] > 0.f ? a[e] : 0.f) : gelu_f(a[e]);
        } else if (kind == 2) {  // gx += d(x, g)
            bf8_unpack(g[i], b);
            bf8_unpack(y[i], o);
            if (op != 0) bf8_unpack(x[i], a);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float d = op == 0 ? c * b[e] : op == 1 ? (a[e] > 0.f ? b[e] : 0.f) : b[e] * gelu_grad_f(a[e]);
                o[e] = o[e] + d;
            }
        } else if (kind == 3) {
            bf8_unpack(x[i], a);
            bf8_unpack(g[i], b);
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = op == 0 ? a[e] + b[e] : a[e] * b[e];
        } else {
            bf8_unpack(x[i], a);
            bf8_unpack(y[i], o);
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = o[e] + c * a[e];
        }
        y[i] = bf8_pack(o);
    }
}

// ------------------------------------------------------------------- fill/cast
template <class T>
__global__ void k_fill(T* x, i64 n, float v) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) x[i] = from_f<T>(v);
}
void fill(void* x, DT t, i64 n, float v, cudaStream_t s) {
    if (t == BF16 && vec8_ok(n, {x})) {
        k_vec8<<<vec8_grid(n), 256, 0, s>>>(0, 0, nullptr, nullptr, (uint4*)x, (int)(n / 8), v);
        SBK_CHECK_LAUNCH();
        return;
    }
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        k_fill<T><<<grid_for(n, 256), 256, 0, s>>>((T*)x, n, v);
    });
    SBK_CHECK_LAUNCH();
}

template <class A, class B>
__device__ __forceinline__ B conv(A a) {
    if constexpr (std::is_same_v<A, B>) return a;
    else if constexpr (std::is_same_v<A, double> && std::is_same_v<B, bf16>) return __double2bfloat16(a);
    else if constexpr (std::is_same_v<A, double>) return (B)a;
    else if constexpr (std::is_same_v<B, double>) return (double)to_f<A>(a);
    else return from_f<B>(to_f<A>(a));
}

template <class A, class B>
__global__ void k_cast(const A* x, B* y, i64 n) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) y[i] = conv<A, B>(x[i]);
}
void cast(const void* x, DT tx, void* y, DT ty, i64 n, cudaStream_t s) {
    if (tx == ty) {  // same type: a device copy
        if (n > 0 && cudaMemcpyAsync(y, x, (size_t)n * dt_bytes(tx), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            throw std::runtime_error("cast: device copy failed");
        return;
    }
    dispatch(tx, [&](auto* pa) {
        using A = std::remove_pointer_t<decltype(pa)>;
        dispatch(ty, [&](auto* pb) {
            using B = std::remove_pointer_t<decltype(pb)>;
            k_cast<A, B><<<grid_for(n, 256), 256, 0, s>>>((const A*)x, (B*)y, n);
        });
    });
    SBK_CHECK_LAUNCH();
}

// ------------------------------------------------------------------- binary
template <class T>
__global__ void k_binary(int op, const T* a, i64 an, const T* b, i64 bn, T* y, i64 n) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        float av = to_f(a[an == 1 ? 0 : i]), bv = to_f(b[bn == 1 ? 0 : i]);
        y[i] = from_f<T>(op == 0 ? av + bv : av * bv);
    }
}
void binary(int op, const void* a, i64 a_n, const void* b, i64 b_n, void* y, DT t, i64 n, cudaStream_t s) {
    if (t == BF16 && a_n == n && b_n == n && vec8_ok(n, {a, b, y})) {
        k_vec8<<<vec8_grid(n), 256, 0, s>>>(3, op, (const uint4*)a, (const uint4*)b, (uint4*)y, (int)(n / 8), 0.f);
        SBK_CHECK_LAUNCH();
        return;
    }
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        k_binary<T><<<grid_for(n, 256), 256, 0, s>>>(op, (const T*)a, a_n, (const T*)b, b_n, (T*)y, n);
    });
    SBK_CHECK_LAUNCH();
}

template <class T>
__global__ void k_unary(int op, const T* x, T* y, i64 n, float c) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        float v = to_f(x[i]);
        y[i] = from_f<T>(op == 0 ? v * c : op == 1 ? (v > 0.f ? v : 0.f) : gelu_f(v));
    }
}
void unary(int op, const void* x, void* y, DT t, i64 n, float c, cudaStream_t s) {
    if (t == BF16 && vec8_ok(n, {x, y})) {
        k_vec8<<<vec8_grid(n), 256, 0, s>>>(1, op, (const uint4*)x, nullptr, (uint4*)y, (int)(n / 8), c);
        SBK_CHECK_LAUNCH();
        return;
    }
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        k_unary<T><<<grid_for(n, 256), 256, 0, s>>>(op, (const T*)x, (T*)y, n, c);
    });
    SBK_CHECK_LAUNCH();
}

template <class T>
__global__ void k_unary_bwd(int op, const T* x, const T* g, T* gx, i64 n, float c) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        float gv = to_f(g[i]), d;
        if (op == 0) d = c * gv;
        else if (op == 1) d = to_f(x[i]) > 0.f ? gv : 0.f;  // executor.cpp:1298-1305
        else d = gv * gelu_grad_f(to_f(x[i]));
        gx[i] = from_f<T>(to_f(gx[i]) + d);
    }
}
void unary_bwd(int op, const void* x, const void* g, void* gx, DT t, DT tg, i64 n, float c, cudaStream_t s) {
    (void)tg;
    if (t == BF16 && vec8_ok(n, {x, g, gx})) {
        k_vec8<<<vec8_grid(n), 256, 0, s>>>(2, op, (const uint4*)x, (const uint4*)g, (uint4*)gx, (int)(n / 8), c);
        SBK_CHECK_LAUNCH();
        return;
    }
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        k_unary_bwd<T><<<grid_for(n, 256), 256, 0, s>>>(op, (const T*)x, (const T*)g, (T*)gx, n, c);
    });
    SBK_CHECK_LAUNCH();
}

template <class A, class B>
__global__ void k_acc(const A* x, B* y, i64 n, float alpha) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        y[i] = from_f<B>(to_f(y[i]) + alpha * to_f(x[i]));
}
void accumulate(const void* x, DT tx, void* y, DT ty, i64 n, float alpha, cudaStream_t s) {
    dispatch(tx, [&](auto* pa) {
        using A = std::remove_pointer_t<decltype(pa)>;
        dispatch(ty, [&](auto* pb) {
            using B = std::remove_pointer_t<decltype(pb)>;
            k_acc<A, B><<<grid_for(n, 256), 256, 0, s>>>((const A*)x, (B*)y, n, alpha);
        });
    });
    SBK_CHECK_LAUNCH();
}

template <class T>
__global__ void k_add_scalar(T* x, i64 n, float v, const T* g) {
    float add = g ? to_f(g[0]) : v;
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        x[i] = from_f<T>(to_f(x[i]) + add);
}
void add_scalar(void* x, DT t, i64 n, float v, const void* g, cudaStream_t s) {
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        k_add_scalar<T><<<grid_for(n, 256), 256, 0, s>>>((T*)x, n, v, (const T*)g);
    });
    SBK_CHECK_LAUNCH();
}

// deterministic sum: fixed grid partials, then one block in fixed order
template <class A>
__global__ void k_red_partial(const A* x, i64 n, float* part) {
    __shared__ float sh[32];
    float acc = 0.f;
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) acc += to_f(x[i]);
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : 0.f;
        v = warp_sum(v);
        if (threadIdx.x == 0) part[blockIdx.x] = v;
    }
}
template <class B>
__global__ void k_red_final(const float* part, int np, B* y, bool acc) {
    __shared__ float sh[32];
    float v = 0.f;
    for (int i = threadIdx.x; i < np; i += blockDim.x) v += part[i];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        float w = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : 0.f;
        w = warp_sum(w);
        if (threadIdx.x == 0) y[0] = from_f<B>(acc ? to_f(y[0]) + w : w);
    }
}
void reduce_all(const void* x, DT tx, i64 n, void* y, DT ty, bool acc, cudaStream_t s) {
    init_workspace();
    int nb = (int)std::min<i64>(kRedBlocks, std::max<i64>(1, (n + 255) / 256));
    dispatch(tx, [&](auto* pa) {
        using A = std::remove_pointer_t<decltype(pa)>;
        k_red_partial<A><<<nb, 256, 0, s>>>((const A*)x, n, g_red_ws);
    });
    dispatch(ty, [&](auto* pb) {
        using B = std::remove_pointer_t<decltype(pb)>;
        k_red_final<B><<<1, 256, 0, s>>>(g_red_ws, nb, (B*)y, acc);
    });
    SBK_CHECK_LAUNCH();
}

template <class T>
__global__ void k_reduce_axis(const T* x, T* y, i64 outer, i64 adim, i64 inner, bool acc) {
    i64 n = outer * inner;
    for (i64 idx = blockIdx.x * (i64)blockDim.x + threadIdx.x; idx < n; idx += (i64)gridDim.x * blockDim.x) {
        i64 o = idx / inner, i = idx % inner;
        float s = 0.f;
        for (i64 a = 0; a < adim; ++a) s += to_f(x[(o * adim + a) * inner + i]);
        y[idx] = from_f<T>(acc ? to_f(y[idx]) + s : s);
    }
}
void reduce_axis(const void* x, void* y, DT t, i64 outer, i64 adim, i64 inner, bool acc, cudaStream_t s) {
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        k_reduce_axis<T><<<grid_for(outer * inner, 256), 256, 0, s>>>((const T*)x, (T*)y, outer, adim, inner, acc);
    });
    SBK_CHECK_LAUNCH();
}
template <class T>
__global__ void k_bcast_axis(const T* g, T* gx, i64 outer, i64 adim, i64 inner) {
    i64 n = outer * adim * inner;
    for (i64 idx = blockIdx.x * (i64)blockDim.x + threadIdx.x; idx < n; idx += (i64)gridDim.x * blockDim.x) {
        i64 o = idx / (adim * inner), i = idx % inner;
        gx[idx] = from_f<T>(to_f(gx[idx]) + to_f(g[o * inner + i]));
    }
}
void broadcast_axis_acc(const void* g, void* gx, DT t, i64 outer, i64 adim, i64 inner, cudaStream_t s) {
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        k_bcast_axis<T><<<grid_for(outer * adim * inner, 256), 256, 0, s>>>((const T*)g, (T*)gx, outer, adim, inner);
    });
    SBK_CHECK_LAUNCH();
}

// ga += g * other, reduced to a scalar when ga_n == 1 and n > 1
template <class T>
__global__ void k_mul_bwd(const T* g, const T* other, i64 on, T* ga, i64 n) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        ga[i] = from_f<T>(to_f(ga[i]) + to_f(g[i]) * to_f(other[on == 1 ? 0 : i]));
}
template <class T>
__global__ void k_mul_bwd_scalar(const T* g, const T* other, i64 on, T* ga, i64 n) {
    __shared__ float sh[32];
    float acc = 0.f;
    for (i64 i = threadIdx.x; i < n; i += blockDim.x) acc += to_f(g[i]) * to_f(other[on == 1 ? 0 : i]);
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : 0.f;
        v = warp_sum(v);
        if (threadIdx.x == 0) ga[0] = from_f<T>(to_f(ga[0]) + v);
    }
}
void mul_bwd(const void* g, DT tg, const void* other, i64 other_n, void* ga, DT tga, i64 ga_n, i64 n, cudaStream_t s) {
    (void)tga;
    dispatch(tg, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        if (ga_n == 1 && n > 1)
            k_mul_bwd_scalar<T><<<1, 1024, 0, s>>>((const T*)g, (const T*)other, other_n, (T*)ga, n);
        else
            k_mul_bwd<T><<<grid_for(n, 256), 256, 0, s>>>((const T*)g, (const T*)other, other_n, (T*)ga, n);
    });
    SBK_CHECK_LAUNCH();
}

// -------------------------------------------------------------------- dropout
template <class T>
__global__ void k_dropout(const T* x, T* y, i64 n, uint64_t s1, uint64_t thr, float scale, bool acc) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        float v = d_keep(s1, (uint64_t)i, thr) ? to_f(x[i]) * scale : 0.f;
        y[i] = from_f<T>(acc ? to_f(y[i]) + v : v);
    }
}
void dropout(const void* x, void* y, DT t, i64 n, u64 s1, u64 thr, float scale, bool acc, cudaStream_t s) {
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        k_dropout<T><<<grid_for(n, 256), 256, 0, s>>>((const T*)x, (T*)y, n, s1, thr, scale, acc);
    });
    SBK_CHECK_LAUNCH();
}
__global__ void k_dropout_mask(uint32_t* bits, i64 n, uint64_t s1, uint64_t thr, uint32_t one) {
    const i64 nw = (n + 31) / 32;
    const uint64_t key = d_keep_key(s1), T = thr << 11;
    for (i64 w = blockIdx.x * (i64)blockDim.x + threadIdx.x; w < nw; w += (i64)gridDim.x * blockDim.x) {
        // 32 independent hash chains per thread: fully unrolled so they interleave
        uint32_t m = d_keep_word_fast(s1, (uint64_t)w * 32 + key, T, one);
        if (w == nw - 1 && (n & 31)) m &= (1u << (n & 31)) - 1;
        bits[w] = m;
    }
}


// Attention keep bits in two layouts from one set of hashes: natural (bit j of
// query row i: element ((bh*S + i)*S + j), read by the forward, one row per
// thread) and transposed (bit i of key row j, read by the backward, one key per
// thread). A warp owns a 32x32 (query, key) block: lane = query row computes
// its 32 keep bits, and 32 ballots transpose the block.
__global__ void k_dropout_mask_dual(uint32_t* bits, uint32_t* bits_t, int S, int Sk, long long BH, uint64_t s1,
                                    uint64_t thr, uint32_t one) {
    // grid-stride over 32x32 (query, key) blocks, one per warp: a small persistent grid
    // (g_mask_blocks blocks of 4 warps) co-resides with the GEMM / attention CTAs and
    // uses their idle issue slots without crowding out their producer / MMA warps
    const int lane = threadIdx.x & 31;
    const int nb = S / 32, nbk = Sk / 32;  // query / key blocks of 32 (Sk != S: cross-attention)
    const long long nblk = BH * nb * nbk;
    for (long long w = (long long)blockIdx.x * 4 + (threadIdx.x >> 5); w < nblk; w += (long long)gridDim.x * 4) {
        const int kb = (int)(w % nbk), qb = (int)((w / nbk) % nb);
        const long long bh = w / ((long long)nb * nbk);
        const long long e0 = (bh * S + qb * 32 + lane) * Sk + kb * 32;  // flat index of (query qb*32+lane, key kb*32)
        const uint32_t m = d_keep_word_fast(s1, (uint64_t)e0 + d_keep_key(s1), thr << 11, one);
        bits[e0 >> 5] = m;
        // 32x32 bit-matrix transpose across the warp (lane = row -> lane = column):
        // swap the off-diagonal blocks of width 16, 8, 4, 2, 1
        uint32_t t = m;
#pragma unroll
        for (int j = 16; j > 0; j >>= 1) {
            const uint32_t msk = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu
                                 : j == 2 ? 0x33333333u : 0x55555555u;
            const uint32_t y = __shfl_xor_sync(0xffffffffu, t, j);
            t = (lane & j) ? (t & ~msk) | ((y >> j) & msk) : (t & msk) | ((y & msk) << j);
        }
        bits_t[((bh * Sk + kb * 32 + lane) * S + qb * 32) >> 5] = t;
    }
}
int g_mask_blocks = 0;  // grid of the keep-bit kernels: 0 full grid (measured best), -1 one block per SM, n > 0 n blocks
void set_mask_blocks(int n) { g_mask_blocks = n; }
static unsigned mask_grid(long long work_blocks) {
    if (g_mask_blocks == 0) return (unsigned)std::max(1ll, work_blocks);
    if (g_mask_blocks > 0) return (unsigned)g_mask_blocks;
    static int sms = 0;
    if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    return (unsigned)sms;
}
void dropout_mask_dual(uint32_t* bits, i64 BH, i64 S, u64 s1, u64 thr, cudaStream_t s, i64 Sk) {
    if (!Sk) Sk = S;
    if (S % 32 || Sk % 32) throw std::runtime_error("dropout_mask_dual: S % 32 != 0");
    const i64 words = BH * S * Sk / 32;
    const i64 nblk = BH * (S / 32) * (Sk / 32);
    const unsigned grid = mask_grid((nblk + 3) / 4);
    static bool attr = false;
    if (!attr) {
        // same shared-memory carveout as the GEMM / attention kernels, so an SM never has to
        // drain to reconfigure between them and the side-stream hashing can co-reside
        cudaFuncSetAttribute(k_dropout_mask_dual, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        attr = true;
    }
    k_dropout_mask_dual<<<grid, 128, 0, s>>>(bits, bits + words, (int)S, (int)Sk, BH, s1, thr, 1u);
    SBK_CHECK_LAUNCH();
}
void dropout_mask(uint32_t* bits, i64 n, u64 s1, u64 thr, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_dropout_mask, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        attr = true;
    }
    k_dropout_mask<<<mask_grid(((n + 31) / 32 + 127) / 128), 128, 0, s>>>(bits, n, s1, thr, 1u);
    SBK_CHECK_LAUNCH();
}

// --------------------------------------------------------------- strided copy
struct Idx8 {
    i64 shape[8], ss[8], ds[8];
    int rank;
};
template <class A, class B>
__global__ void k_strided(const A* src, B* dst, Idx8 ix, i64 n, bool acc) {
    for (i64 lin = blockIdx.x * (i64)blockDim.x + threadIdx.x; lin < n; lin += (i64)gridDim.x * blockDim.x) {
        i64 rem = lin, so = 0, dof = 0;
        for (int d = ix.rank - 1; d >= 0; --d) {
            i64 c = rem % ix.shape[d];
            rem /= ix.shape[d];
            so += c * ix.ss[d];
            dof += c * ix.ds[d];
        }
        if constexpr (std::is_same_v<B, double>) {
            dst[dof] = acc ? dst[dof] + conv<A, double>(src[so]) : conv<A, double>(src[so]);
        } else {
            B v = conv<A, B>(src[so]);
            dst[dof] = acc ? from_f<B>(to_f(dst[dof]) + to_f(v)) : v;
        }
    }
}
void strided_copy(const void* src, DT ts, const i64* sst, void* dst, DT td, const i64* dstr, const i64* shape, int rank,
                  bool acc, cudaStream_t s) {
    if (rank > 8) throw std::runtime_error("strided_copy: rank > 8");
    Idx8 ix{};
    ix.rank = rank;
    i64 n = 1;
    for (int d = 0; d < rank; ++d) {
        ix.shape[d] = shape[d];
        ix.ss[d] = sst[d];
        ix.ds[d] = dstr[d];
        n *= shape[d];
    }
    if (n == 0) return;
    dispatch(ts, [&](auto* pa) {
        using A = std::remove_pointer_t<decltype(pa)>;
        dispatch(td, [&](auto* pb) {
            using B = std::remove_pointer_t<decltype(pb)>;
            k_strided<A, B><<<grid_for(n, 256), 256, 0, s>>>((const A*)src, (B*)dst, ix, n, acc);
        });
    });
    SBK_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ nan guard
template <class T>
__global__ void k_nan(const T* x, i64 n, int* flag) {
    int c = 0;
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) c += isnan(to_f(x[i]));
    if (c) atomicAdd(flag, c);
}
void count_nan(const void* x, DT t, i64 n, int* flag, cudaStream_t s) {
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        k_nan<T><<<grid_for(n, 256), 256, 0, s>>>((const T*)x, n, flag);
    });
    SBK_CHECK_LAUNCH();
}

// ---------------------------------------------------------- rank-local sums
struct Ptrs16 {
    const void* src[16];
    void* dst[16];
};
template <class T>
__global__ void k_sum_ranks(Ptrs16 p, int R, i64 n, bool acc) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        float s = 0.f;
        for (int r = 0; r < R; ++r) s += to_f(((const T*)p.src[r])[i]);  // rank-ascending fold (executor.cpp:813-817)
        for (int r = 0; r < R; ++r) {
            T* d = (T*)p.dst[r];
            d[i] = from_f<T>(acc ? to_f(d[i]) + s : s);
        }
    }
}
void sum_ranks(const void* const* srcs, void* const* dsts, int R, DT t, i64 n, bool acc, cudaStream_t s) {
    if (R > 16) throw std::runtime_error("sum_ranks: more than 16 ranks");
    Ptrs16 p{};
    for (int r = 0; r < R; ++r) {
        p.src[r] = srcs[r];
        p.dst[r] = dsts[r];
    }
    dispatch(t, [&](auto* q) {
        using T = std::remove_pointer_t<decltype(q)>;
        k_sum_ranks<T><<<grid_for(n, 256), 256, 0, s>>>(p, R, n, acc);
    });
    SBK_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ embedding
// row = llround(raw) mod V, vocab-parallel rows [row0, row0+local) (executor.cpp:14-17,749-784)
__device__ __forceinline__ i64 d_row(double raw, i64 V) {
    i64 i = (i64)llround(raw) % V;
    return i < 0 ? i + V : i;
}
template <class T>
__global__ void k_emb_fwd(const double* ids, i64 n, const T* table, i64 dim, i64 V, i64 row0, i64 local, T* out) {
    i64 total = n * dim;
    for (i64 idx = blockIdx.x * (i64)blockDim.x + threadIdx.x; idx < total; idx += (i64)gridDim.x * blockDim.x) {
        i64 i = idx / dim, d = idx % dim;
        i64 r = d_row(ids[i], V) - row0;
        out[idx] = (r >= 0 && r < local) ? table[r * dim + d] : from_f<T>(0.f);
    }
}
// 16-byte vectors (bf16, dim % 8 == 0): one row-slice per thread, the id read once per vector
__global__ void k_emb_fwd_v(const double* ids, int n, const uint4* table, int vdim, i64 V, i64 row0, i64 local,
                            uint4* out) {
    const int total = n * vdim;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int i = idx / vdim, d = idx - i * vdim;
        const i64 r = d_row(ids[i], V) - row0;
        out[idx] = (r >= 0 && r < local) ? __ldg(table + r * vdim + d) : make_uint4(0, 0, 0, 0);
    }
}
void embedding_fwd(const double* ids, i64 n, const void* table, DT t, i64 dim, i64 V, i64 row0, i64 local, void* out,
                   cudaStream_t s) {
    if (t == BF16 && dim % 8 == 0 && n * (dim / 8) < (1ll << 31) && ((uintptr_t)table & 15) == 0 &&
        ((uintptr_t)out & 15) == 0) {
        const i64 total = n * (dim / 8);
        k_emb_fwd_v<<<(unsigned)std::min<i64>((total + 255) / 256, 148 * 16), 256, 0, s>>>(
            ids, (int)n, (const uint4*)table, (int)(dim / 8), V, row0, local, (uint4*)out);
        SBK_CHECK_LAUNCH();
        return;
    }
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        k_emb_fwd<T><<<grid_for(n * dim, 256), 256, 0, s>>>(ids, n, (const T*)table, dim, V, row0, local, (T*)out);
    });
    SBK_CHECK_LAUNCH();
}
// ------------------------------------------------------------------ bias grad
// db[c] += sum_r g[r*ld + c]: fixed row chunks -> partials -> ordered sum.
constexpr int kBiasChunk = 256;
template <class T>
__global__ void k_bias_partial(const T* g, i64 ld, i64 rows, i64 cols, float* part) {
    i64 c = blockIdx.x * (i64)blockDim.x + threadIdx.x;
    i64 r0 = (i64)blockIdx.y * kBiasChunk;
    if (c >= cols) return;
    float acc = 0.f;
    i64 r1 = r0 + kBiasChunk < rows ? r0 + kBiasChunk : rows;
    for (i64 r = r0; r < r1; ++r) acc += to_f(g[r * ld + c]);
    part[(i64)blockIdx.y * cols + c] = acc;
}
// bf16, cols % 8 == 0, 16-byte aligned rows: thread = 8 columns (one 16-byte load per
// row), 16 rows of loads in flight; row chunks of kBiasChunkV summed in row order
constexpr int kBiasChunkV = 32;
__global__ void k_bias_partial_v(const bf16* g, i64 ld, i64 rows, i64 cols, float* part) {
    const i64 c8 = blockIdx.x * (i64)blockDim.x + threadIdx.x;  // 8-column group
    if (c8 * 8 >= cols) return;
    const i64 r0 = (i64)blockIdx.y * kBiasChunkV;
    const i64 r1 = r0 + kBiasChunkV < rows ? r0 + kBiasChunkV : rows;
    float acc[8] = {};
    i64 r = r0;
    for (; r + 16 <= r1; r += 16) {
        uint4 v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldcs((const uint4*)(g + (r + u) * ld) + c8);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const __nv_bfloat162* h = (const __nv_bfloat162*)&v[u];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                float2 f = __bfloat1622float2(h[t]);
                acc[2 * t] += f.x;
                acc[2 * t + 1] += f.y;
            }
        }
    }
    for (; r < r1; ++r) {
        uint4 v = *((const uint4*)(g + r * ld) + c8);
        const __nv_bfloat162* h = (const __nv_bfloat162*)&v;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            float2 f = __bfloat1622float2(h[t]);
            acc[2 * t] += f.x;
            acc[2 * t + 1] += f.y;
        }
    }
    float4* o = (float4*)(part + (i64)blockIdx.y * cols + c8 * 8);
    o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
}
// block = 32 columns x 32 warps: warp w sums chunks w, w+32, ... (8 loads in flight);
// then the 32 sums in warp order (fixed order: deterministic)
__global__ void __launch_bounds__(1024) k_bias_final(const float* part, i64 chunks, i64 cols, float* db, bool accum) {
    __shared__ float s[32][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const i64 c = blockIdx.x * 32ll + lane;
    float acc = 0.f;
    if (c < cols) {
        i64 k = warp;
        for (; k + 7 * 32 < chunks; k += 8 * 32) {  // 8 loads in flight, summed in chunk order
            float a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = part[(k + u * 32) * cols + c];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += a[u];
        }
        for (; k < chunks; k += 32) acc += part[k * cols + c];
    }
    s[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && c < cols) {
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < 32; ++w) t += s[w][lane];
        db[c] = accum ? db[c] + t : t;
    }
}
void bias_grad_partials(const float* partials, i64 chunks, i64 cols, float* db, cudaStream_t s, bool accum) {
    k_bias_final<<<(unsigned)((cols + 31) / 32), 1024, 0, s>>>(partials, chunks, cols, db, accum);
    SBK_CHECK_LAUNCH();
}
size_t bias_grad_workspace(i64 rows, i64 cols) { return (size_t)((rows + kBiasChunkV - 1) / kBiasChunkV) * cols * 4; }
void bias_grad(const void* g, DT tg, i64 ld, i64 rows, i64 cols, float* db, float* ws, cudaStream_t s, bool accum) {
    i64 chunks = (rows + kBiasChunk - 1) / kBiasChunk;
    if (tg == BF16 && cols % 8 == 0 && ld % 8 == 0 && ((uintptr_t)g & 15) == 0) {
        chunks = (rows + kBiasChunkV - 1) / kBiasChunkV;
        dim3 grid((unsigned)((cols / 8 + 127) / 128), (unsigned)chunks);
        k_bias_partial_v<<<grid, 128, 0, s>>>((const bf16*)g, ld, rows, cols, ws);
    } else {
        dim3 grid((unsigned)((cols + 127) / 128), (unsigned)chunks);
        dispatch(tg, [&](auto* p) {
            using T = std::remove_pointer_t<decltype(p)>;
            k_bias_partial<T><<<grid, 128, 0, s>>>((const T*)g, ld, rows, cols, ws);
        });
    }
    k_bias_final<<<(unsigned)((cols + 31) / 32), 1024, 0, s>>>(ws, chunks, cols, db, accum);
    SBK_CHECK_LAUNCH();
}

// ------------------------------------------------- bias + GeLU (standalone)
// The .fuse'd Linear->gelu region outside a GEMM (the product path folds it into
// the tcgen05 GEMM epilogue): pre = x + b[col], y = gelu(pre); backward
// gx = g * gelu'(pre) (db = column sums of gx via bias_grad).
template <class T>
__global__ void k_bias_gelu_fwd(const T* x, const T* b, T* y, T* pre, i64 rows, i64 n) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < rows * n; i += (i64)gridDim.x * blockDim.x) {
        const float v = to_f(x[i]) + (b ? to_f(b[i % n]) : 0.f);
        if (pre) pre[i] = from_f<T>(v);
        y[i] = from_f<T>(gelu_f(v));
    }
}
template <class T>
__global__ void k_bias_gelu_bwd(const T* pre, const T* g, T* gx, i64 total) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < total; i += (i64)gridDim.x * blockDim.x)
        gx[i] = from_f<T>(to_f(g[i]) * gelu_grad_f(to_f(pre[i])));
}
void bias_gelu_fwd(const void* x, const void* b, void* y, void* pre, DT t, i64 rows, i64 n, cudaStream_t s) {
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        if constexpr (!std::is_same_v<T, double>)
            k_bias_gelu_fwd<T><<<grid_for(rows * n, 256), 256, 0, s>>>((const T*)x, (const T*)b, (T*)y, (T*)pre, rows, n);
        else
            throw std::runtime_error("bias_gelu: f64 unsupported");
    });
    SBK_CHECK_LAUNCH();
}
void bias_gelu_bwd(const void* pre, const void* g, void* gx, float* db, DT t, i64 rows, i64 n, float* ws, cudaStream_t s) {
    dispatch(t, [&](auto* p) {
        using T = std::remove_pointer_t<decltype(p)>;
        if constexpr (!std::is_same_v<T, double>)
            k_bias_gelu_bwd<T><<<grid_for(rows * n, 256), 256, 0, s>>>((const T*)pre, (const T*)g, (T*)gx, rows * n);
        else
            throw std::runtime_error("bias_gelu: f64 unsupported");
    });
    SBK_CHECK_LAUNCH();
    if (db) bias_grad(gx, t, n, rows, n, db, ws, s, false);
}

}  // namespace sbk
