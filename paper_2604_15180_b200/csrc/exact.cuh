// exact.cuh -- launchers of the fp64 EXACT path (exact.cu).
#pragma once
#include "common.cuh"

namespace adattn_b200 {

bool exact_supported(const Geom& g);

// exact_generic.cu: any block size and width (block_r or block_c > 64, d or dv > 128)
bool exact_generic_needed(const Geom& g);
cudaError_t exact_generic_forward(const Geom& g, const void* q, const void* k, const void* v,
                                  void* out, double* tau, double* row_max, uint32_t* mask,
                                  int32_t* steps, cudaStream_t st);
cudaError_t exact_generic_delta(const Geom& g, const void* q, const void* k, const void* v,
                                const double* tau, const double* row_max, const uint32_t* mask,
                                const void* dout, double* delta, cudaStream_t st);
cudaError_t exact_generic_backward(const Geom& g, const void* q, const void* k, const void* v,
                                   const double* tau, const double* row_max, const uint32_t* mask,
                                   const void* dout, void* dq, void* dk, void* dv, double* delta,
                                   unsigned long long* visited, cudaStream_t st);

cudaError_t exact_forward(const Geom& g, const void* q, const void* k, const void* v, void* out,
                          double* tau, double* row_max, uint32_t* mask, int32_t* steps,
                          cudaStream_t st);

cudaError_t exact_delta(const Geom& g, const void* q, const void* k, const void* v,
                        const double* tau, const double* row_max, const uint32_t* mask,
                        const void* dout, double* delta, cudaStream_t st);

cudaError_t exact_backward(const Geom& g, const void* q, const void* k, const void* v,
                           const double* tau, const double* row_max, const uint32_t* mask,
                           const void* dout, void* dq, void* dk, void* dv, double* delta,
                           unsigned long long* visited, cudaStream_t st);

}  // namespace adattn_b200
