// TMEM load throughput microbenchmark: W warps per CTA, each repeatedly tcgen05.ld 32x32b.xN
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int N> __device__ __forceinline__ void ld(uint32_t a, uint32_t* r);
template <> __device__ __forceinline__ void ld<32>(uint32_t a, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) : "r"(a));
}
template <int W, int ITERS>
__global__ void __launch_bounds__(W * 32, 1) ktm(unsigned long long* out, float* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp / 4) * 32;
    float acc = 0.f;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) {
        uint32_t r[32];
        ld<32>(t + ((i * 32) & 511 & ~31) * 0, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 1.2345f) sink[threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}
template <int W> void run() {
    unsigned long long* d; float* sink; cudaMalloc(&d, 8 * 148); cudaMalloc(&sink, 4096);
    constexpr int IT = 2000;
    ktm<W, IT><<<148, W * 32>>>(d, sink);
    ktm<W, IT><<<148, W * 32>>>(d, sink);
    cudaDeviceSynchronize();
    unsigned long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double bytes = (double)W * IT * 32 * 32 * 4;  // per CTA (SM)
    printf("warps %2d: %llu cycles -> %.1f B/clk per SM (%s)\n", W, h[0], bytes / h[0], cudaGetErrorString(cudaGetLastError()));
}
int main() { run<1>(); run<2>(); run<4>(); run<8>(); run<16>(); return 0; }
