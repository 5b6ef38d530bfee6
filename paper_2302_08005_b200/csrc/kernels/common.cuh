// Shared device helpers for the sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "kernels.hpp"

namespace sbk {

using bf16 = __nv_bfloat16;

#define SBK_CHECK_LAUNCH()                                                                                \
    do {                                                                                                  \
        cudaError_t e_ = cudaGetLastError();                                                              \
        if (e_ != cudaSuccess) throw std::runtime_error(std::string("kernel launch failed: ") +           \
                                                        cudaGetErrorString(e_) + " in " + __func__);      \
    } while (0)

template <class T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<bf16>(bf16 x) { return __bfloat162float(x); }
template <>
__device__ __forceinline__ float to_f<double>(double x) { return (float)x; }

template <class T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }
template <>
__device__ __forceinline__ double from_f<double>(float x) { return (double)x; }

// Counter RNG core (proj/include/slapo/rng.hpp:16-24), 64-bit integer math.
__device__ __forceinline__ uint64_t d_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
// splitmix64 on 32-bit halves (the 64-bit C expression compiles to ~1.6x more
// SASS): x += golden; x = (x ^ x>>30) * M1; x = (x ^ x>>27) * M2; x ^= x>>31.
__device__ __forceinline__ void sm64_xs(uint32_t& lo, uint32_t& hi, int k) {
    lo ^= __funnelshift_r(lo, hi, k);
    hi ^= hi >> k;
}
__device__ __forceinline__ void sm64_mul(uint32_t& lo, uint32_t& hi, uint32_t mlo, uint32_t mhi) {
    const unsigned long long p = (unsigned long long)lo * mlo;
    hi = (uint32_t)(p >> 32) + lo * mhi + hi * mlo;
    lo = (uint32_t)p;
}
__device__ __forceinline__ void sm64_add(uint32_t& lo, uint32_t& hi, uint32_t clo, uint32_t chi) {
    asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(lo), "+r"(hi) : "r"(clo), "r"(chi));
}
// all but the final xor-shift of splitmix64
__device__ __forceinline__ void sm64_body(uint32_t& lo, uint32_t& hi) {
    sm64_add(lo, hi, 0x7f4a7c15u, 0x9e3779b9u);
    sm64_xs(lo, hi, 30);
    sm64_mul(lo, hi, 0x1ce4e5b9u, 0xbf58476du);
    sm64_xs(lo, hi, 27);
    sm64_mul(lo, hi, 0x133111ebu, 0x94d049bbu);
}

// keep test of element i for a stream with s1 = hash_combine(stream_seed, 0xd0):
//   uniform01(stream_seed, 0xd0, i) >= p   <=>   (h >> 11) >= thr   <=>   h >= thr << 11
// with h = splitmix64(splitmix64(s1 ^ (i + golden + (s1 << 6) + (s1 >> 2)))).
// `k` = golden + (s1 << 6) + (s1 >> 2) is per stream (d_keep_key).
__device__ __forceinline__ uint64_t d_keep_key(uint64_t s1) { return 0x9e3779b97f4a7c15ULL + (s1 << 6) + (s1 >> 2); }
__device__ __forceinline__ bool d_keep_k(uint64_t s1, uint64_t key, uint64_t i, uint64_t thr) {
    const uint64_t x = s1 ^ (i + key);
    uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
    sm64_body(lo, hi);
    sm64_xs(lo, hi, 31);  // end of the inner splitmix64
    sm64_body(lo, hi);
    const uint64_t T = thr << 11;  // thr < 2^53
    const uint32_t thi = (uint32_t)(T >> 32), tlo = (uint32_t)T;
    const uint32_t hhi = hi ^ (hi >> 31);
    if (hhi != thi) return hhi > thi;
    return (lo ^ __funnelshift_r(lo, hi, 31)) >= tlo;  // rare (2^-32): compare the low word
}
__device__ __forceinline__ bool d_keep(uint64_t s1, uint64_t i, uint64_t thr) {
    return d_keep_k(s1, d_keep_key(s1), i, thr);
}
// keep bits of the 32 elements e0 .. e0+31 (bit b = element e0 + b); bk = e0 + d_keep_key(s1),
// T = thr << 11. The index add is one 64-bit mad and the >= T test a borrow chain, so the
// hash (integer-ALU bound) carries no extra compare/select work per element.
__device__ __forceinline__ uint32_t d_keep_word(uint64_t s1, uint64_t bk, uint64_t T) {
    const uint32_t tlo = (uint32_t)T, thi = (uint32_t)(T >> 32);
    uint32_t m = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
        unsigned long long d;
        asm("mad.wide.u32 %0, %1, 1, %2;" : "=l"(d) : "r"((uint32_t)b), "l"(bk));
        d ^= s1;
        uint32_t lo = (uint32_t)d, hi = (uint32_t)(d >> 32);
        sm64_body(lo, hi);
        sm64_xs(lo, hi, 31);
        sm64_body(lo, hi);
        sm64_xs(lo, hi, 31);
        uint32_t bit;
        asm("{\n\t.reg .u32 t;\n\tsub.cc.u32 t, %1, %3;\n\tsubc.cc.u32 t, %2, %4;\n\taddc.u32 %0, 0, 0;\n\t}"
            : "=r"(bit)
            : "r"(lo), "r"(hi), "r"(tlo), "r"(thi));
        m |= bit << b;
    }
    return m;
}

static __device__ __noinline__ uint32_t d_keep_word_slow(uint64_t s1, uint64_t bk, uint64_t T) { return d_keep_word(s1, bk, T); }
// 64-bit multiply by a constant in three IMADs (the generic form compiles to four)
__device__ __forceinline__ void sm64_mul3(uint32_t& lo, uint32_t& hi, uint32_t mlo, uint32_t mhi) {
    asm("{\n\t.reg .u32 pl, ph, t;\n\t"
        "mul.lo.u32 pl, %0, %2;\n\tmul.hi.u32 ph, %0, %2;\n\t"
        "mad.lo.u32 t, %0, %3, ph;\n\tmad.lo.u32 %1, %1, %2, t;\n\tmov.u32 %0, pl;\n\t}"
        : "+r"(lo), "+r"(hi)
        : "r"(mlo), "r"(mhi));
}
// d_keep_word with fewer integer ops per element (same bits; 250 vs 307 us per
// 134M elements on B200, ALU-pipe bound):
//  * the 32 indices bk .. bk+31 share their high word (checked), so the first
//    `+ golden` and `x ^= x >> 30` on the high word take one of two precomputed
//    values, selected by the carry with FMA-pipe mads (`one` = 1 from a kernel
//    argument, so ptxas keeps them off the ALU pipe);
//  * 64-bit products in three IMADs, and only the high word of the final one;
//  * the final `h ^= h >> 31` is skipped: for T's high word t < 2^31,
//    f(v) = v ^ (v >> 31) satisfies f(v) > t <=> v > t and f(v) == t <=> v == t,
//    so h >= T is v > t, or v == t and a low-word compare; a tie (p ~ 2^-32 per
//    element) reruns the exact d_keep_word for the word.
// Falls back to d_keep_word when t >= 2^31 (p >= 0.5) or the indices cross a 2^32 boundary.
__device__ __forceinline__ uint32_t d_keep_word_fast(uint64_t s1, uint64_t bk, uint64_t T, uint32_t one) {
    const uint32_t thi = (uint32_t)(T >> 32), bklo = (uint32_t)bk, s1lo = (uint32_t)s1;
    if ((thi >> 31) | (bklo > 0xFFFFFFFFu - 31u)) return d_keep_word_slow(s1, bk, T);
    const uint32_t h0 = ((uint32_t)(bk >> 32) ^ (uint32_t)(s1 >> 32)) + 0x9e3779b9u;
    const uint32_t H0 = h0 ^ (h0 >> 30), dH = ((h0 + 1u) ^ ((h0 + 1u) >> 30)) - H0;
    uint32_t m = 0;
    bool tie = false;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
        const uint32_t x = (bklo + (uint32_t)b) ^ s1lo;
        uint32_t lo, cy, h, hi;
        asm("add.cc.u32 %0, %2, 0x7f4a7c15;\n\taddc.u32 %1, 0, 0;" : "=r"(lo), "=r"(cy) : "r"(x));
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h) : "r"(cy), "r"(one), "r"(h0));
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(hi) : "r"(cy), "r"(dH), "r"(H0));
        lo ^= __funnelshift_r(lo, h, 30);
        sm64_mul3(lo, hi, 0x1ce4e5b9u, 0xbf58476du);
        sm64_xs(lo, hi, 27);
        sm64_mul3(lo, hi, 0x133111ebu, 0x94d049bbu);
        sm64_xs(lo, hi, 31);
        sm64_add(lo, hi, 0x7f4a7c15u, 0x9e3779b9u);
        sm64_xs(lo, hi, 30);
        sm64_mul3(lo, hi, 0x1ce4e5b9u, 0xbf58476du);
        sm64_xs(lo, hi, 27);
        uint32_t v;  // high word of (lo, hi) * M2
        asm("{\n\t.reg .u32 t;\n\tmul.lo.u32 t, %1, %4;\n\tmad.lo.u32 t, %2, %3, t;\n\tmad.hi.u32 %0, %1, %3, t;\n\t}"
            : "=r"(v)
            : "r"(lo), "r"(hi), "r"(0x133111ebu), "r"(0x94d049bbu));
        m |= (uint32_t)(v >= thi) << b;
        tie |= v == thi;
    }
    if (tie) return d_keep_word_slow(s1, bk, T);
    return m;
}

__device__ __forceinline__ float gelu_f(float x) {
    const float c = 0.7978845608028654f, a = 0.044715f;
    float u = c * (x + a * x * x * x);
    return 0.5f * x * (1.f + tanhf(u));
}
__device__ __forceinline__ float gelu_grad_f(float x) {
    const float c = 0.7978845608028654f, a = 0.044715f;
    float u = c * (x + a * x * x * x);
    float t = tanhf(u);
    return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * c * (1.f + 3.f * a * x * x);
}

template <class F>
void dispatch(DT t, F&& f) {
    switch (t) {
        case F32: f((float*)nullptr); break;
        case BF16: f((bf16*)nullptr); break;
        case F64: f((double*)nullptr); break;
    }
}

inline unsigned grid_for(i64 n, int threads, int per_thread = 1) {
    i64 b = (n + (i64)threads * per_thread - 1) / ((i64)threads * per_thread);
    if (b < 1) b = 1;
    if (b > 148 * 64) b = 148 * 64;
    return (unsigned)b;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

}  // namespace sbk
