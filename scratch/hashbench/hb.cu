// microbenchmark: splitmix64 keep-mask variants (pipe balance ALU vs FMA)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
struct K { uint32_t c4, c32, c2, one; };
__device__ __forceinline__ uint64_t ref_sm(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL; x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL; return x ^ (x >> 31);
}
__device__ __forceinline__ bool ref_keep(uint64_t s1, uint64_t i, uint64_t thr) {
    uint64_t h = ref_sm(ref_sm(s1 ^ (i + 0x9e3779b97f4a7c15ULL + (s1 << 6) + (s1 >> 2))));
    return (h >> 11) >= thr;
}
// xorshift right by k: ALU form or FMA form (mul.hi by 2^(32-k) held in a register)
template <bool F, bool H = false> __device__ __forceinline__ void xs(uint32_t& lo, uint32_t& hi, int k, uint32_t m) {
    if (H) {  // lo on the ALU (funnel shift), hi >> k as mul.hi on the FMA pipe
        uint32_t c;
        asm("mul.hi.u32 %0, %1, %2;" : "=r"(c) : "r"(hi), "r"(m));
        lo ^= __funnelshift_r(lo, hi, k); hi ^= c;
    } else if (F) {
        uint32_t a, b, c;
        asm("mul.hi.u32 %0, %1, %2;" : "=r"(a) : "r"(lo), "r"(m));
        asm("mul.lo.u32 %0, %1, %2;" : "=r"(b) : "r"(hi), "r"(m));
        asm("mul.hi.u32 %0, %1, %2;" : "=r"(c) : "r"(hi), "r"(m));
        lo = lo ^ a ^ b; hi = hi ^ c;
    } else {
        lo ^= __funnelshift_r(lo, hi, k); hi ^= hi >> k;
    }
}
__device__ __forceinline__ void mul(uint32_t& lo, uint32_t& hi, uint32_t mlo, uint32_t mhi) {
    const unsigned long long p = (unsigned long long)lo * mlo;
    hi = (uint32_t)(p >> 32) + lo * mhi + hi * mlo; lo = (uint32_t)p;
}
template <bool F> __device__ __forceinline__ void addg(uint32_t& lo, uint32_t& hi, uint32_t one) {
    if (F) {  // (lo*1 + G) as a 64-bit mad, then + hi<<32
        unsigned long long d;
        asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(lo), "r"(one), "l"(0x9e3779b97f4a7c15ULL));
        lo = (uint32_t)d; hi = hi + (uint32_t)(d >> 32);
    } else {
        asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(lo), "+r"(hi) : "r"(0x7f4a7c15u), "r"(0x9e3779b9u));
    }
}
template <int V> __device__ __forceinline__ uint32_t keep_word(uint64_t s1, uint64_t bk, uint64_t T, const K& kc) {
    // V bits: 0..5 = xorshift i uses FMA form (order: sm1 xs30, xs27, xs31, sm2 xs30, xs27, xs31), bit 6/7 = add via mad
    uint32_t m = 0;
    const uint32_t tlo = (uint32_t)T, thi = (uint32_t)(T >> 32);
#pragma unroll
    for (int b = 0; b < 32; ++b) {
        unsigned long long d;
        asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"((uint32_t)b), "r"(kc.one), "l"(bk));
        d ^= s1;
        uint32_t lo = (uint32_t)d, hi = (uint32_t)(d >> 32);
        addg<(V >> 6) & 1>(lo, hi, kc.one);
        constexpr int HM = (V >> 8) & 63;
        xs<(V >> 0) & 1, (HM >> 0) & 1>(lo, hi, 30, kc.c4); mul(lo, hi, 0x1ce4e5b9u, 0xbf58476du);
        xs<(V >> 1) & 1, (HM >> 1) & 1>(lo, hi, 27, kc.c32); mul(lo, hi, 0x133111ebu, 0x94d049bbu);
        xs<(V >> 2) & 1, (HM >> 2) & 1>(lo, hi, 31, kc.c2);
        addg<(V >> 7) & 1>(lo, hi, kc.one);
        xs<(V >> 3) & 1, (HM >> 3) & 1>(lo, hi, 30, kc.c4); mul(lo, hi, 0x1ce4e5b9u, 0xbf58476du);
        xs<(V >> 4) & 1, (HM >> 4) & 1>(lo, hi, 27, kc.c32); mul(lo, hi, 0x133111ebu, 0x94d049bbu);
        xs<(V >> 5) & 1, (HM >> 5) & 1>(lo, hi, 31, kc.c2);
        uint32_t bit;
        asm("{\n\t.reg .u32 t;\n\tsub.cc.u32 t, %1, %3;\n\tsubc.cc.u32 t, %2, %4;\n\taddc.u32 %0, 0, 0;\n\t}"
            : "=r"(bit) : "r"(lo), "r"(hi), "r"(tlo), "r"(thi));
        m += bit << b;
    }
    return m;
}
template <int V> __global__ void kmask(uint32_t* bits, long long nw, uint64_t s1, uint64_t thr, K kc) {
    const uint64_t key = 0x9e3779b97f4a7c15ULL + (s1 << 6) + (s1 >> 2), T = thr << 11;
    for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < nw; w += (long long)gridDim.x * blockDim.x)
        bits[w] = keep_word<V>(s1, (uint64_t)w * 32 + key, T, kc);
}
__global__ void kref(uint32_t* bits, long long nw, uint64_t s1, uint64_t thr) {
    for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < nw; w += (long long)gridDim.x * blockDim.x) {
        uint32_t m = 0;
        for (int b = 0; b < 32; ++b) if (ref_keep(s1, w * 32 + b, thr)) m |= 1u << b;
        bits[w] = m;
    }
}
template <int V> float run(uint32_t* d, uint32_t* r, long long nw, uint64_t s1, uint64_t thr, K kc, int* bad) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    kmask<V><<<148 * 8, 256>>>(d, nw, s1, thr, kc);
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) kmask<V><<<148 * 8, 256>>>(d, nw, s1, thr, kc);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    // compare
    static uint32_t* h1 = nullptr; static uint32_t* h2 = nullptr;
    if (!h1) { h1 = new uint32_t[nw]; h2 = new uint32_t[nw]; cudaMemcpy(h2, r, nw * 4, cudaMemcpyDeviceToHost); }
    cudaMemcpy(h1, d, nw * 4, cudaMemcpyDeviceToHost);
    *bad = 0; for (long long i = 0; i < nw; ++i) if (h1[i] != h2[i]) ++*bad;
    return ms / 5;
}
int main() {
    const long long n = 32ll * 16 * 512 * 512, nw = n / 32;
    uint32_t *d, *r; cudaMalloc(&d, nw * 4); cudaMalloc(&r, nw * 4);
    uint64_t s1 = 0x123456789abcdefULL, thr = (uint64_t)(0.1 * 9007199254740992.0) + 1;
    K kc{4, 32, 2, 1};
    kref<<<148 * 8, 256>>>(r, nw, s1, thr);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); kref<<<148 * 8, 256>>>(r, nw, s1, thr); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); printf("ref 64-bit C: %.1f us\n", ms * 1000);
    int bad;
#define R(V) { float t = run<V>(d, r, nw, s1, thr, kc, &bad); printf("V=%3d (xsF=%d%d%d%d%d%d addF=%d%d): %.1f us bad=%d\n", V, V&1,(V>>1)&1,(V>>2)&1,(V>>3)&1,(V>>4)&1,(V>>5)&1,(V>>6)&1,(V>>7)&1, t*1000, bad); }
    R(0) R(63*256) R(9*256) R(27*256) R(18*256) R(45*256) R(7*256) R(56*256) R(21*256)
    return 0;
}
