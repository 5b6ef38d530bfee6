// round-trip latency of the synchronisation hops the attention kernels chain:
// mbarrier arrive -> try_wait between two warps, and tcgen05.commit -> mbarrier
#include "../../paper_2302_08005_b200/csrc/kernels/tc5.cuh"
#include <cstdio>
using namespace sbk::tc5;
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ unsigned long long clk() { unsigned long long t; asm volatile("mov.u64 %0, %clock64;" : "=l"(t)); return t; }
template <int MODE>
__global__ void __launch_bounds__(64, 1) k(int iters, unsigned long long* out) {
    __shared__ uint64_t b1, b2;
    __shared__ uint32_t slot;
    __shared__ __align__(1024) uint8_t sm[16384];
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) { mbar_init(&b1, 1); mbar_init(&b2, 1); fence_barrier_init(); }
    if (w == 0) { tmem_alloc<128>(&slot); }
    fence_before(); __syncthreads(); fence_after();
    const uint32_t tmem = slot;
    unsigned long long t0 = clk();
    if (w == 0) {
        for (int i = 0; i < iters; ++i) {
            if (MODE == 0) { if (lane == 0) mbar_arrive(&b1); }
            else {
                if (MODE == 2) {
                    const uint64_t da = sdesc(smem_u32(sm), 1, 64), db = sdesc(smem_u32(sm + 8192), 1, 64);
                    const uint32_t id = idesc_bf16(128, 64, false, false);
                    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;\n\t}" ::"r"(tmem), "l"(da), "l"(db), "r"(id));
                }
                mma_commit_w(&b1);
            }
            mbar_wait(&b2, i & 1);
        }
    } else {
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&b1, i & 1);
            if (MODE != 0) fence_after();
            if (lane == 0) mbar_arrive(&b2);
        }
    }
    unsigned long long t1 = clk();
    __syncthreads();
    if (threadIdx.x == 0) out[0] = (t1 - t0);
    if (w == 0) tmem_dealloc<128>(tmem);
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 8);
    const int iters = 2000;
    auto run = [&](const char* nm, auto kern) {
        kern<<<1, 64>>>(iters, d); cudaDeviceSynchronize();
        kern<<<1, 64>>>(iters, d); cudaDeviceSynchronize();
        unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("%-40s %8.1f cycles per round trip  (%s)\n", nm, (double)c / iters, cudaGetErrorString(cudaGetLastError()));
    };
    run("mbarrier arrive <-> wait (2 warps)", k<0>);
    run("tcgen05.commit (no MMA) -> wait, arrive back", k<1>);
    run("1 MMA M128N64K16 + commit -> wait, back", k<2>);
}
