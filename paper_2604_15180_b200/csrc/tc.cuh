// tc.cuh -- launchers of the bf16 tensor-core (tcgen05/TMEM/TMA) path.
#pragma once
#include <string>

#include "common.cuh"

namespace adattn_b200 {

bool tc_supported(const Geom& g);
std::string tc_envelope();
size_t tc_forward_workspace(const Geom& g);
size_t tc_backward_workspace(const Geom& g);
// the forward fills g.ubar_out (delta fold) for this (unpadded) geometry
bool tc_delta_fold(const Geom& g);
// bytes of the support-list buffer the forward fills for the backward's delta (0: off)
size_t tc_delta_supp_bytes(const Geom& g);

cudaError_t tc_forward(const Geom& g, const void* q, const void* k, const void* v, void* out,
                       double* tau, double* row_max, uint32_t* mask, int32_t* steps,
                       void* workspace, cudaStream_t st);
cudaError_t tc_delta(const Geom& g, const void* q, const void* k, const void* v,
                     const double* tau, const double* row_max, const uint32_t* mask,
                     const void* dout, double* delta, void* workspace, cudaStream_t st);
cudaError_t tc_backward(const Geom& g, const void* q, const void* k, const void* v,
                        const double* tau, const double* row_max, const uint32_t* mask,
                        const void* dout, void* dq, void* dk, void* dv, double* delta,
                        void* workspace, cudaStream_t st);

uint64_t flushes_of(const Geom& g);
uint64_t addressable_of(const Geom& g);

}  // namespace adattn_b200
