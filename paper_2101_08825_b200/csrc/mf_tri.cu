// mf_tri.cu -- specialised 2D kernel (placeholder until written).
#include "mf_common.cuh"
bool mf_tri_supported(const AsmParams &) { return false; }
cudaError_t mf_launch_tri(const AsmParams &, cudaStream_t) {
  return cudaErrorNotSupported;
}
