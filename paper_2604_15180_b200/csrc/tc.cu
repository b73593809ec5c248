// tc.cu -- bf16 tensor-core path (placeholder until the tcgen05 kernels land).
#include "tc.cuh"

namespace adattn_b200 {

bool tc_supported(const Geom&) { return false; }
std::string tc_envelope() { return "not built in this revision"; }
size_t tc_forward_workspace(const Geom&) { return 0; }
size_t tc_backward_workspace(const Geom&) { return 0; }
cudaError_t tc_forward(const Geom&, const void*, const void*, const void*, void*, double*,
                       double*, uint32_t*, int32_t*, void*, cudaStream_t) {
  return cudaErrorNotSupported;
}
cudaError_t tc_delta(const Geom&, const void*, const void*, const void*, const double*,
                     const double*, const uint32_t*, const void*, double*, void*, cudaStream_t) {
  return cudaErrorNotSupported;
}
cudaError_t tc_backward(const Geom&, const void*, const void*, const void*, const double*,
                        const double*, const uint32_t*, const void*, void*, void*, void*,
                        double*, void*, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace adattn_b200
