// GEMM front end: dispatches bf16 Linear-shaped problems to the tcgen05
// kernel (gemm_tc.cu) and everything else — fp32 parity path, batched
// attention matmuls of the unscheduled model, odd strides — to a tiled SIMT
// kernel with fp32 accumulation and an arbitrary-stride operand model.
// Replaces linear_fwd / linear_dx / linear_dw / matmul_fwd
// (proj/src/executor.cpp:38-133).
#include "common.cuh"

namespace sbk {

bool gemm_tc_try(const Gemm& g, cudaStream_t s);   // gemm_tc.cu  (1-SM tcgen05)
bool gemm_tc2_try(const Gemm& g, cudaStream_t s);  // gemm_tc2.cu (2-SM tcgen05)

namespace {
int g_last_engine = 0;
bool g_force_simt = false;

constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;

template <class TA, class TB, class TC>
__global__ void __launch_bounds__(256) k_gemm_simt(Gemm g) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const TA* A = (const TA*)g.A + (i64)blockIdx.z * g.sAb;
    const TB* B = (const TB*)g.B + (i64)blockIdx.z * g.sBb;
    TC* C = (TC*)g.C + (i64)blockIdx.z * g.sCb;
    TC* X = g.aux ? (TC*)g.aux + (i64)blockIdx.z * g.sCb : nullptr;
    i64 m0 = (i64)blockIdx.y * BM, n0 = (i64)blockIdx.x * BN;
    int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    float acc[TM][TN] = {};
    for (i64 k0 = 0; k0 < g.K; k0 += BK) {
        for (int e = threadIdx.x; e < BM * BK; e += 256) {
            int mm = e / BK, kk = e % BK;
            i64 m = m0 + mm, k = k0 + kk;
            As[kk][mm] = (m < g.M && k < g.K) ? to_f(A[m * g.sAm + k * g.sAk]) : 0.f;
        }
        for (int e = threadIdx.x; e < BN * BK; e += 256) {
            int kk = e / BN, nn = e % BN;
            i64 n = n0 + nn, k = k0 + kk;
            Bs[kk][nn] = (n < g.N && k < g.K) ? to_f(B[k * g.sBk + n * g.sBn]) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float a[TM], b[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
            for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx * TN + j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
    const TC* bias = (const TC*)g.bias;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        i64 m = m0 + ty * TM + i;
        if (m >= g.M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            i64 n = n0 + tx * TN + j;
            if (n >= g.N) continue;
            float v = g.alpha * acc[i][j];
            if (bias) v += to_f(bias[n]);
            i64 ci = m * g.sCm + n * g.sCn;
            if (g.epilogue == 1) {
                if (X) X[ci] = from_f<TC>(v);
                v = gelu_f(v);
            } else if (g.epilogue == 2) {
                v *= gelu_grad_f(to_f(X[ci]));  // dgrad straight into a GeLU input's gradient
            } else if (g.epilogue == 3) {
                v = fmaxf(v, 0.f);  // ReLU
            } else if (g.epilogue == 4) {
                v = to_f(X[ci]) > 0.f ? v : 0.f;  // dgrad times the ReLU mask of the activation X
            }
            if (g.accumulate) v += to_f(C[ci]);
            C[ci] = from_f<TC>(v);
        }
    }
}
}  // namespace

int g_gemm_max_engine = 0;  // 0 best available, 1 at most the 1-SM tcgen05 kernel, 2 SIMT
int gemm_last_engine() { return g_last_engine; }
void gemm_force_simt(bool on) { g_force_simt = on; }
void gemm_set_engine(int e) { g_gemm_max_engine = e; }

extern bool g_tc2_colsum_done;
bool gemm_last_colsum() { return g_tc2_colsum_done; }
void gemm(const Gemm& g, cudaStream_t s) {
    g_tc2_colsum_done = false;
    if (g.M == 0 || g.N == 0) return;
    if (!g_force_simt && g_gemm_max_engine == 0 && gemm_tc2_try(g, s)) {
        g_last_engine = 2;
        return;
    }
    if (!g_force_simt && g_gemm_max_engine <= 1 && gemm_tc_try(g, s)) {
        g_last_engine = 1;
        return;
    }
    g_last_engine = 0;
    if (g.bias && g.tbias != g.tc && !(g.tbias == g.ta && g.tc == g.ta))
        throw std::runtime_error("gemm: bias dtype must match C");
    dim3 grid((unsigned)((g.N + BN - 1) / BN), (unsigned)((g.M + BM - 1) / BM), (unsigned)g.batch);
    auto launch = [&](auto* pa, auto* pc) {
        using TA = std::remove_pointer_t<decltype(pa)>;
        using TC = std::remove_pointer_t<decltype(pc)>;
        k_gemm_simt<TA, TA, TC><<<grid, 256, 0, s>>>(g);
    };
    if (g.ta != g.tb) throw std::runtime_error("gemm: A and B dtypes must match");
    if (g.ta == F32 && g.tc == F32) launch((float*)nullptr, (float*)nullptr);
    else if (g.ta == BF16 && g.tc == BF16) launch((bf16*)nullptr, (bf16*)nullptr);
    else if (g.ta == BF16 && g.tc == F32) launch((bf16*)nullptr, (float*)nullptr);
    else if (g.ta == F64 && g.tc == F64) launch((double*)nullptr, (double*)nullptr);
    else throw std::runtime_error("gemm: unsupported dtype combination");
    SBK_CHECK_LAUNCH();
}

}  // namespace sbk
