// tcgen05 GEMM (placeholder until the tensor-core kernel lands).
#include "common.cuh"
namespace sbk {
bool gemm_tc_try(const Gemm&, cudaStream_t) { return false; }
}  // namespace sbk
