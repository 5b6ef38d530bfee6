// tcgen05.mma issue/throughput microbenchmark: one CTA per SM, one elected thread
// issues NMMA MMAs of M128 x N x K16 (SS or TS) into one accumulator, then commits
// and waits; cycles per MMA vs the 128*N/256 floor.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2302_08005_b200/csrc/kernels/tc5.cuh"
using namespace sbk::tc5;
template <int N, bool TS, int NMMA>
__global__ void __launch_bounds__(128, 1) kmb(unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&slot);
    fence_before(); __syncthreads(); fence_after();
    const uint32_t tmem = slot;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0;
    fence_proxy_async();
    __syncthreads();
    if (warp == 0) {
        constexpr uint32_t id = idesc_bf16(128, N, false, false);
        const uint32_t a0 = smem_u32(sm), b0 = a0 + 32768;
        const uint64_t da = desc_kmajor(a0, 0), db = desc_kmajor(b0, 0);
        unsigned long long t0 = clock64();
        for (int r = 0; r < NMMA / 4; ++r) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (TS) mma_ts_w(tmem, tmem + 256 + kk * 8, db + 2 * kk, id, 1);
                else mma_ss_w(tmem, da + 2 * kk, db + 2 * kk, id, 1);
            }
        }
        unsigned long long t1 = clock64();
        mma_commit_w(&bar);
        mbar_wait(&bar, 0);
        unsigned long long t2 = clock64();
        if (threadIdx.x == 0) { out[2 * blockIdx.x] = t1 - t0; out[2 * blockIdx.x + 1] = t2 - t0; }
    }
    fence_before(); __syncthreads();
    if (warp == 0) { fence_after(); tmem_dealloc<512>(tmem); }
}
template <int N, bool TS> void run() {
    constexpr int NM = 4096;
    unsigned long long* d; cudaMalloc(&d, 16 * 148);
    auto k = kmb<N, TS, NM>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    k<<<148, 128, 65536 + 1024>>>(d); k<<<148, 128, 65536 + 1024>>>(d);
    cudaDeviceSynchronize();
    unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%s M128 N%3d K16: issue %.1f cyc/mma, complete %.1f cyc/mma (floor %d) %s\n", TS ? "TS" : "SS", N,
           (double)h[0] / NM, (double)h[1] / NM, 128 * N / 256, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    run<64, false>(); run<64, true>(); run<128, false>(); run<128, true>(); run<256, false>(); run<256, true>();
    run<32, true>(); run<32, false>();
    return 0;
}
