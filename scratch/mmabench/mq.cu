// (1) tcgen05.mma issue-queue depth: cycles to issue n back-to-back SS M128 N64 K16
//     MMAs vs cycles until they complete;
// (2) does an MMA-issuing warp blocked on a full queue slow the other warps of its
//     SM sub-partition? A compute warp on the same SMSP (warp 4 = SMSP 0, MMA warp 0)
//     vs on another SMSP (warp 5) counts FMA iterations while the MMA warp issues.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2302_08005_b200/csrc/kernels/tc5.cuh"
using namespace sbk::tc5;
__global__ void __launch_bounds__(256, 1) kq(unsigned long long* out, int n, int spin) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    __shared__ volatile int stop;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); stop = 0; }
    if (warp == 0) tmem_alloc<512>(&slot);
    fence_before(); __syncthreads(); fence_after();
    const uint32_t tmem = slot;
    if (warp == 0) {
        constexpr uint32_t id = idesc_bf16(128, 64, false, false);
        const uint32_t a0 = smem_u32(sm), b0 = a0 + 32768;
        const uint64_t da = desc_kmajor(a0, 0), db = desc_kmajor(b0, 0);
        unsigned long long t0 = clock64();
        for (int r = 0; r < n; ++r) mma_ss_w(tmem, da + 2 * (r & 3), db + 2 * (r & 3), id, 1);
        unsigned long long t1 = clock64();
        mma_commit_w(&bar);
        mbar_wait(&bar, 0);
        unsigned long long t2 = clock64();
        if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; stop = 1; }
    } else if (spin && (warp == 4 || warp == 5)) {
        float x = threadIdx.x, y = 1.0001f;
        unsigned long long it = 0;
        unsigned long long t0 = clock64();
        while (!stop) {
#pragma unroll
            for (int k = 0; k < 64; ++k) x = fmaf(x, y, 0.5f);
            ++it;
        }
        unsigned long long t1 = clock64();
        if ((threadIdx.x & 31) == 0) { out[2 + (warp - 4) * 2] = it; out[3 + (warp - 4) * 2] = t1 - t0; }
        if (x == 0.123f) out[10] = 1;
    }
    fence_before(); __syncthreads();
    if (warp == 0) { fence_after(); tmem_dealloc<512>(tmem); }
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 128);
    cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    for (int n : {1, 2, 4, 8, 16, 32, 64, 256}) {
        unsigned long long h[8] = {};
        kq<<<1, 256, 65536 + 1024>>>(d, n, 0); cudaDeviceSynchronize();
        kq<<<1, 256, 65536 + 1024>>>(d, n, 0); cudaDeviceSynchronize();
        cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
        printf("n %3d: issue %6llu cyc, complete %6llu cyc\n", n, h[0], h[1]);
    }
    for (int n : {1024, 8192}) {
        unsigned long long h[8] = {};
        kq<<<1, 256, 65536 + 1024>>>(d, n, 1); cudaDeviceSynchronize();
        cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
        printf("n %d with FMA warps: issue %llu complete %llu; same-SMSP warp %.1f cyc/iter, other-SMSP warp %.1f cyc/iter (%s)\n",
               n, h[0], h[1], (double)h[3] / h[2], (double)h[5] / h[4], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
