// tc_host.cuh -- host helpers for the tensor-core path: TMA tensor maps.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace adattn_b200 {

// ELL nonzero-block lists (lists.cu): per row block its active key blocks
// (ascending, capacity t_c), per key block its active query blocks (ascending,
// capacity t_r) -- the lists the backward kernels walk.
cudaError_t ell_row_lists(const Geom& g, const uint32_t* mask, int32_t* rcnt, uint16_t* rcol,
                          cudaStream_t st);
cudaError_t ell_col_lists(const Geom& g, const int32_t* rcnt, const uint16_t* rcol, int32_t* ccnt,
                          uint16_t* crow, cudaStream_t st);
inline size_t ell_bytes(const Geom& g) {
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  return al((size_t)g.bh * g.t_r * 4) + al((size_t)g.bh * g.t_r * g.t_c * 2) +
         al((size_t)g.bh * g.t_c * 4) + al((size_t)g.bh * g.t_c * g.t_r * 2);
}

namespace tc {

// 2-D bf16 tensor map over a row-major [rows][cols] matrix, box = 64 columns
// (128 B, SWIZZLE_128B) x box_rows rows.
cudaError_t make_tmap_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                         uint32_t box_rows);
cudaError_t make_tmap_3d_chunks(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                                uint32_t box_rows);

int alpha_kind(double alpha);

// Candidate-list plan of the forward: `cap` entries per epilogue thread (0 =
// refinement by sweeps only), `slots` resident-CTA slots (%nsmid).
struct CandPlan {
  int cap, slots;
};
CandPlan cand_plan(const Geom& g);
size_t forward_workspace(const Geom& g);
size_t forward_cand_bytes(const Geom& g);
size_t forward_wtm_offset(const Geom& g);
int forward_wtm_slots();
bool pv_f16_enabled();
// the forward fills g.ubar_out (delta fold) for this geometry
bool fwd_delta_fold(const Geom& g);
// delta from support lists: layout of the forward -> backward buffer (delta_aux) --
// per 256-row block (a forward CTA's rows, global row index / 256) a fallback flag and a
// pool of 256 * cap (key, u bits) entries; per row and key half (count, pool offset)
struct SuppLayout {
  uint32_t* flag;   // [nblk] 256-row blocks whose rows the tensor-core kernels handle
  uint32_t* hflag;  // [bh] heads with a flagged block (sparse backward: whole head)
  int2* cnt;        // [rows][2] (count, pool offset)
  uint2* ent;       // [nblk][256 cap] (key, t bits)
  int32_t* kcnt;    // [bh][m] support entries per key (forward atomics)
  int32_t* koff;    // [bh][m + 1] their exclusive prefix (backward)
  int32_t* kcur;    // [bh][m] scatter cursors (backward)
  int32_t* krow;    // [nblk 256 cap] key-major lists: query row ...
  float2* kpd;      // ... and (p, dS)
  int32_t* klong;   // [1 + bh m]: count, then the keys with long lists (keys kernel)
  int cap;
  size_t nblk;
};
bool delta_supp_possible(const Geom& g);  // list mode, ADATTN_DELTA_SUPP != 0
bool delta_supp_enabled(const Geom& g);   // ... and the forward does not fold delta
size_t supp_bytes(const Geom& g);
SuppLayout supp_layout(const Geom& g, void* base);

// Power-of-two-scaled fp16 copies of bf16 operands (tc_common.cuh f16_pow2_scale),
// per head (`heads` consecutive blocks of `elems` values, elems % 8 == 0), so a head's
// results never depend on the other heads of the call (chunked run_host, sharded
// multi-GPU runs).  f16_absmax: atomicMax of max |x| (float bits) into
// maxbits[h] (caller zeroes them); f16_convert_scaled: dst = fp16(src * s(maxbits[h])).
// need (optional): heads with need[h] == 0 get a non-finite maximum -- no copy, and a
// bf16 plan should a tensor-core kernel still take the head.
cudaError_t f16_absmax(const void* src, int heads, size_t elems, uint32_t* maxbits,
                       cudaStream_t st, const uint32_t* need = nullptr);
cudaError_t f16_convert_scaled(const void* src, void* dst, int heads, size_t elems,
                               const uint32_t* maxbits, cudaStream_t st);

cudaError_t forward(const Geom& g, const void* q, const void* k, const void* v, void* out,
                    double* tau, double* row_max, uint32_t* mask, int32_t* steps, void* ws,
                    cudaStream_t st);

size_t backward_workspace(const Geom& g);

cudaError_t backward(const Geom& g, const void* q, const void* k, const void* v, const double* tau,
                     const double* row_max, const uint32_t* mask, const void* dout, void* dq,
                     void* dk, void* dv, double* delta, void* workspace, bool delta_only,
                     cudaStream_t st);

}  // namespace tc
}  // namespace adattn_b200
