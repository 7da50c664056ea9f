// mf_hex.cu -- specialised 3D hex Q1 kernel (placeholder until written).
#include "mf_common.cuh"
bool mf_hex_supported(const AsmParams &) { return false; }
cudaError_t mf_launch_hex(const AsmParams &, cudaStream_t) {
  return cudaErrorNotSupported;
}
