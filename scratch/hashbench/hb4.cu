// keep-word hash variants: which xorshift / add steps run on the FMA pipe (IMAD / IMAD.HI /
// IMAD.WIDE) instead of the ALU pipe (SHF / LOP3 / IADD3). Validated against d_keep_word.
#include "../../paper_2302_08005_b200/csrc/kernels/common.cuh"
#include <cstdio>
#include <vector>
#include <algorithm>
using namespace sbk;
struct Mul { uint32_t one, m30, m27, m31; };
// x ^= x >> k on 64 bits; LO: low word via IMAD.HI + IMAD, HI: high word via IMAD.HI
template <bool LO, bool HI>
__device__ __forceinline__ void xs(uint32_t& lo, uint32_t& hi, int k, uint32_t m) {
    if (LO) {
        uint32_t t;
        asm("{\n\t.reg .u32 a;\n\tmul.hi.u32 a, %1, %3;\n\tmad.lo.u32 %0, %2, %3, a;\n\t}" : "=r"(t) : "r"(lo), "r"(hi), "r"(m));
        lo ^= t;
    } else {
        lo ^= __funnelshift_r(lo, hi, k);
    }
    if (HI) {
        uint32_t t;
        asm("mul.hi.u32 %0, %1, %2;" : "=r"(t) : "r"(hi), "r"(m));
        hi ^= t;
    } else {
        hi ^= hi >> k;
    }
}
template <int F>
__device__ __forceinline__ uint32_t keep_var(uint64_t s1, uint64_t bk, uint64_t T, Mul mu) {
    const uint32_t one = mu.one;
    const uint32_t thi = (uint32_t)(T >> 32), bklo = (uint32_t)bk, s1lo = (uint32_t)s1;
    if ((thi >> 31) | (bklo > 0xFFFFFFFFu - 31u)) return d_keep_word_slow(s1, bk, T);
    const uint32_t h0 = ((uint32_t)(bk >> 32) ^ (uint32_t)(s1 >> 32)) + 0x9e3779b9u;
    const uint32_t H0 = h0 ^ (h0 >> 30), dH = ((h0 + 1u) ^ ((h0 + 1u) >> 30)) - H0;
    const uint32_t K = H0 - h0 * dH;
    const unsigned long long C0 = ((unsigned long long)h0 << 32) | 0x7f4a7c15u;
    uint32_t m = 0;
    bool tie = false;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
        const uint32_t x = (bklo + (uint32_t)b) ^ s1lo;
        uint32_t lo, h, hi;
        if (F & 1) {
            unsigned long long d;
            asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(x), "r"(one), "l"(C0));
            lo = (uint32_t)d;
            h = (uint32_t)(d >> 32);
            asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(hi) : "r"(h), "r"(dH), "r"(K));
        } else {
            uint32_t cy;
            asm("add.cc.u32 %0, %2, 0x7f4a7c15;\n\taddc.u32 %1, 0, 0;" : "=r"(lo), "=r"(cy) : "r"(x));
            asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h) : "r"(cy), "r"(one), "r"(h0));
            asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(hi) : "r"(cy), "r"(dH), "r"(H0));
        }
        // first xorshift 30 (low word only; the high word came precomputed)
        if (F & 4) {
            uint32_t t;
            asm("{\n\t.reg .u32 a;\n\tmul.hi.u32 a, %1, %3;\n\tmad.lo.u32 %0, %2, %3, a;\n\t}" : "=r"(t) : "r"(lo), "r"(h), "r"(mu.m30));
            lo ^= t;
        } else {
            lo ^= __funnelshift_r(lo, h, 30);
        }
        sm64_mul3(lo, hi, 0x1ce4e5b9u, 0xbf58476du);
        xs<(F & 8) != 0, (F & 128) != 0>(lo, hi, 27, mu.m27);
        sm64_mul3(lo, hi, 0x133111ebu, 0x94d049bbu);
        xs<(F & 16) != 0, (F & 256) != 0>(lo, hi, 31, mu.m31);
        if (F & 2) {
            uint32_t hc;
            asm("mad.lo.u32 %0, %1, %2, 0x9e3779b9;" : "=r"(hc) : "r"(hi), "r"(one));
            unsigned long long d, c = ((unsigned long long)hc << 32) | 0x7f4a7c15u;
            asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(lo), "r"(one), "l"(c));
            lo = (uint32_t)d;
            hi = (uint32_t)(d >> 32);
        } else {
            sm64_add(lo, hi, 0x7f4a7c15u, 0x9e3779b9u);
        }
        xs<(F & 32) != 0, (F & 512) != 0>(lo, hi, 30, mu.m30);
        sm64_mul3(lo, hi, 0x1ce4e5b9u, 0xbf58476du);
        xs<(F & 64) != 0, (F & 1024) != 0>(lo, hi, 27, mu.m27);
        uint32_t v;
        asm("{\n\t.reg .u32 t;\n\tmul.lo.u32 t, %1, %4;\n\tmad.lo.u32 t, %2, %3, t;\n\tmad.hi.u32 %0, %1, %3, t;\n\t}"
            : "=r"(v) : "r"(lo), "r"(hi), "r"(0x133111ebu), "r"(0x94d049bbu));
        m |= (uint32_t)(v >= thi) << b;
        tie |= v == thi;
    }
    if (tie) return d_keep_word_slow(s1, bk, T);
    return m;
}
template <int F>
__global__ void kval(const uint64_t* s1s, const uint64_t* bks, const uint64_t* Ts, int n, uint32_t* out, Mul mu) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = F < 0 ? d_keep_word(s1s[i], bks[i], Ts[i]) : keep_var<F < 0 ? 0 : F>(s1s[i], bks[i], Ts[i], mu);
}
template <int F>
__global__ void kbench(uint32_t* out, long long words, uint64_t s1, uint64_t T, Mul mu) {
    const uint64_t key = d_keep_key(s1);
    for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < words; w += (long long)gridDim.x * blockDim.x)
        out[w] = F < 0 ? d_keep_word_fast(s1, (uint64_t)w * 32 + key, T, mu.one) : keep_var<F < 0 ? 0 : F>(s1, (uint64_t)w * 32 + key, T, mu);
}
static uint64_t rng = 88172645463325252ull;
static uint64_t r64() { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return rng; }
int main() {
    const int n = 1 << 20;
    std::vector<uint64_t> s1(n), bk(n), T(n);
    for (int i = 0; i < n; ++i) {
        s1[i] = r64(); bk[i] = r64();
        if (i % 7 == 0) bk[i] |= 0xFFFFFFF0ull;
        double p = (i % 3 == 0) ? 0.1 : (r64() % 1000) / 1000.0;
        T[i] = ((uint64_t)(p * 9007199254740992.0)) << 11;
    }
    uint64_t *ds1, *dbk, *dT; uint32_t* dout;
    cudaMalloc(&ds1, n * 8); cudaMalloc(&dbk, n * 8); cudaMalloc(&dT, n * 8); cudaMalloc(&dout, n * 4);
    cudaMemcpy(ds1, s1.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dbk, bk.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dT, T.data(), n * 8, cudaMemcpyHostToDevice);
    Mul mu{1u, 1u << 2, 1u << 5, 1u << 1};
    std::vector<uint32_t> want(n), got(n);
    kval<-1><<<n / 256, 256>>>(ds1, dbk, dT, n, dout, mu);
    cudaMemcpy(want.data(), dout, n * 4, cudaMemcpyDeviceToHost);
    const long long words = 134217728ll / 32;
    uint32_t* big; cudaMalloc(&big, words * 4);
    uint64_t s1b = 0x1234567890abcdefull, Tb = ((uint64_t)(0.1 * 9007199254740992.0)) << 11;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char* name, auto kern, auto vk) {
        vk<<<n / 256, 256>>>(ds1, dbk, dT, n, dout, mu);
        cudaMemcpy(got.data(), dout, n * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < n; ++i) bad += got[i] != want[i];
        float best = 1e9;
        for (int g : {148 * 16, 148 * 8, 148 * 4}) for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            kern<<<g, 128>>>(big, words, s1b, Tb, mu);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            best = std::min(best, ms);
        }
        printf("%-34s %7.1f us per 134M elements  mismatches=%d\n", name, best * 1000, bad);
    };
    run("current (d_keep_word_fast)", kbench<-1>, kval<0>);
#define V(F, nm) run(nm, kbench<F>, kval<F>);
    V(0, "F0 same as current")
    V(3, "F3 adds as mad.wide")
    V(3 | 4, "F7 + first lo funnel")
    V(3 | 8 | 32, "adds + lo xs27a, xs30b")
    V(3 | 8 | 16 | 32, "adds + lo 3 xs")
    V(3 | 8 | 16 | 32 | 64, "adds + lo 4 xs")
    V(3 | 4 | 8 | 16 | 32 | 64, "adds + all lo")
    V(3 | 128 | 256, "adds + hi xs27a, xs31")
    V(3 | 8 | 128, "adds + xs27a both halves")
    V(3 | 8 | 32 | 128 | 512, "adds + xs27a, xs30b both")
    V(8 | 32, "lo xs27a, xs30b only")
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
