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
// keep test of element i for a stream with s1 = hash_combine(stream_seed, 0xd0):
//   uniform01(stream_seed, 0xd0, i) >= p   <=>   (h >> 11) >= thr
__device__ __forceinline__ bool d_keep(uint64_t s1, uint64_t i, uint64_t thr) {
    uint64_t h = d_splitmix64(d_splitmix64(s1 ^ (i + 0x9e3779b97f4a7c15ULL + (s1 << 6) + (s1 >> 2))));
    return (h >> 11) >= thr;
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
