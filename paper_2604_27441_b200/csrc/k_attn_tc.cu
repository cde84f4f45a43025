// k_attn_tc.cu -- tcgen05/TMEM spatial attention (bf16 operands, fp32
// softmax/accumulation) for head_dim 32.  (placeholder: not yet enabled)
#include "launch.cuh"

namespace nvrec {

bool tc_supported(const Dims& D) { return false; }

cudaError_t launch_attn_tc(const Act& A, const Dims& D, const int* count, cudaStream_t s) {
  return cudaErrorNotSupported;
}

}  // namespace nvrec
