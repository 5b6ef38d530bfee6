// Tensor-core attention (placeholder until the sm_100a kernel lands).
#include "common.cuh"
namespace sbk {
bool attn_fwd_tc_try(const Attn&, cudaStream_t) { return false; }
bool attn_bwd_tc_try(const Attn&, const void*, i64, void*, void*, void*, i64, i64, i64, float*, cudaStream_t) { return false; }
}  // namespace sbk
