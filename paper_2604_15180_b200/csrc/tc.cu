// tc.cu -- dispatch for the bf16 tensor-core path and its TMA descriptor helper.
#include <cudaTypedefs.h>

#include <mutex>

#include "tc.cuh"
#include "tc_host.cuh"

namespace adattn_b200 {
namespace tc {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

cudaError_t make_tmap_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                         uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace tc

// Envelope of the tensor-core kernels: bf16 inputs, 64x64
// reference tiles, d == dv in {64, 128}, n a multiple of 256, m of 64.
bool tc_supported(const Geom& g) {
  return g.in_dtype == ADATTN_BF16 && g.block_r == 64 && g.block_c == 64 && g.d == g.dv &&
         (g.d == 64 || g.d == 128) && g.n % 256 == 0 && g.m % 128 == 0 && g.bins <= 32 &&
         g.bins >= 2;
}
std::string tc_envelope() {
  return "bf16 inputs, block_r=block_c=64, d=dv in {64,128}, n%256==0, m%128==0, 2<=bins<=32";
}
size_t tc_forward_workspace(const Geom&) { return 0; }
size_t tc_backward_workspace(const Geom& g) { return tc::backward_workspace(g); }

cudaError_t tc_forward(const Geom& g, const void* q, const void* k, const void* v, void* out,
                       double* tau, double* row_max, uint32_t* mask, int32_t* steps, void*,
                       cudaStream_t st) {
  return tc::forward(g, q, k, v, out, tau, row_max, mask, steps, st);
}
cudaError_t tc_delta(const Geom& g, const void* q, const void* k, const void* v,
                     const double* tau, const double* row_max, const uint32_t* mask,
                     const void* dout, double* delta, void* ws, cudaStream_t st) {
  return tc::backward(g, q, k, v, tau, row_max, mask, dout, nullptr, nullptr, nullptr, delta, ws,
                      true, st);
}
cudaError_t tc_backward(const Geom& g, const void* q, const void* k, const void* v,
                        const double* tau, const double* row_max, const uint32_t* mask,
                        const void* dout, void* dq, void* dk, void* dv, double* delta, void* ws,
                        cudaStream_t st) {
  return tc::backward(g, q, k, v, tau, row_max, mask, dout, dq, dk, dv, delta, ws, false, st);
}

}  // namespace adattn_b200
