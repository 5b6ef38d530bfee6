// mbarrier handshake latency: ping-pong between warp 1 lane 0 and warp 0 (all lanes)
#include "../../paper_2302_08005_b200/csrc/kernels/tc5.cuh"
#include <cstdio>
using namespace sbk;
using namespace sbk::tc5;
template <int MODE>  // 0: plain arrive, 1: tcgen05.commit (no MMA in flight), 2: commit after one small MMA
__global__ void __launch_bounds__(128) k_hs(int iters, long long* out) {
    __shared__ uint64_t bars[2];
    __shared__ uint32_t slot;
    __shared__ __align__(1024) uint8_t buf[2 * 8192];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<128>(&slot);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = slot;
    long long t0 = clock64();
    if (warp == 1) {
        if (lane == 0) {
            for (int i = 0; i < iters; ++i) {
                if (MODE == 0) mbar_arrive(&bars[0]);
                else {
                    if (MODE == 2) {
                        const uint32_t a = smem_u32(buf), b = smem_u32(buf + 8192);
                        mma_ss(tmem, desc_kmajor(a, 0), desc_kmajor(b, 0), idesc_bf16(128, 64, false, false), 0);
                    }
                    mma_commit(&bars[0]);
                }
                mbar_wait(&bars[1], i & 1);
            }
        }
    } else if (warp == 0) {
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&bars[0], i & 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars[1]);
        }
    }
    long long t1 = clock64();
    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        tmem_dealloc<128>(tmem);
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = (t1 - t0) / iters;
}
int main() {
    long long* d;
    cudaMalloc(&d, 8);
    for (int mode = 0; mode < 3; ++mode)
        for (int grid : {1, 148, 592}) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            const int iters = 20000;
            auto go = [&]() {
                if (mode == 0) k_hs<0><<<grid, 128>>>(iters, d);
                if (mode == 1) k_hs<1><<<grid, 128>>>(iters, d);
                if (mode == 2) k_hs<2><<<grid, 128>>>(iters, d);
            };
            go();
            cudaEventRecord(a);
            go();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            long long cyc;
            cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
            printf("mode %d grid %4d: %.1f ns per round trip, %lld cycles (block 0)  %s\n", mode, grid, ms * 1e6 / iters,
                   cyc, cudaGetErrorString(cudaGetLastError()));
        }
}
