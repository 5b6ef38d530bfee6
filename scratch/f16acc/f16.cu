// layout of an f16 accumulator (tcgen05.mma kind::f16, D format f16) in TMEM
#include "../../paper_2302_08005_b200/csrc/kernels/tc5.cuh"
#include <cuda_bf16.h>
#include <cstdio>
using namespace sbk::tc5;
__global__ void k(uint32_t* out, int dfmt) {
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    __shared__ __align__(1024) __nv_bfloat16 A[128 * 64], B[64 * 64];
    for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) A[i] = __float2bfloat16(1.f);
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) B[i] = __float2bfloat16((i / 64) * 0.25f);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (threadIdx.x < 32) tmem_alloc<128>(&slot);
    fence_proxy_async();
    fence_before(); __syncthreads(); fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x < 32) {
        uint32_t id = idesc_bf16(128, 64, false, false);
        id = (id & ~(3u << 4)) | ((uint32_t)dfmt << 4);
        mma_ss_w(tmem, desc_kmajor(smem_u32(A), 0), desc_kmajor(smem_u32(B), 0), id, 0);
        mma_commit_w(&bar);
    }
    mbar_wait(&bar, 0);
    fence_after();
    if (threadIdx.x < 32) {
        uint32_t r[32];
        tmem_ld32_nowait(tmem, r); tmem_ld_wait();
        if (threadIdx.x == 0) for (int c = 0; c < 32; ++c) out[c] = r[c];
        tmem_ld32_nowait(tmem + 32, r); tmem_ld_wait();
        if (threadIdx.x == 0) for (int c = 0; c < 32; ++c) out[32 + c] = r[c];
    }
    fence_before(); __syncthreads();
    if (threadIdx.x < 32) { fence_after(); tmem_dealloc<128>(tmem); }
}
int main() {
    uint32_t* d; cudaMalloc(&d, 64 * 4);
    for (int fmt : {1, 0}) {
        cudaMemset(d, 0, 256);
        k<<<1, 128>>>(d, fmt);
        cudaError_t e = cudaDeviceSynchronize();
        uint32_t h[64]; cudaMemcpy(h, d, 256, cudaMemcpyDeviceToHost);
        printf("D format %d (%s): ", fmt, cudaGetErrorString(e));
        for (int c = 0; c < 40; ++c) printf("%08x ", h[c]);
        printf("\n");
    }
}
