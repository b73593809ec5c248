// lists.cu -- per-row-block lists of the active key blocks (CSR) and the
// transposed per-key-block lists of the active query blocks, built from a
// device PackedBlockMask (all heads concatenated).
//
// Order follows the reference: a row block's key blocks in the order
// PackedBlockMask::for_each_set visits them (ascending j; bitpack.hpp:85-92),
// and a key block's query blocks in ascending i (the row order in which
// PackedBlockMask::transposed() sets them; bitpack.cpp:138-143) -- the lists the
// reference's output pass and key-major backward sweep walk
// (attention.cpp:334-352, 464-506).
#include <cuda_runtime.h>

#include <cstdint>

#include "adattn_b200.h"
#include "common.cuh"

namespace adattn_b200 {
namespace {

// counts: rowptr[r] = popcount of row block r; colptr[h * t_c + j] += 1 per set bit
__global__ void lists_count(const uint32_t* __restrict__ mask, int rows_total, int t_r, int t_c,
                            int wpr, int64_t* rowptr, unsigned long long* colcnt) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows_total) return;
  const uint32_t* row = mask + (size_t)r * wpr;
  const int h = r / t_r;
  int64_t n = 0;
  for (int w = 0; w < wpr; ++w) {
    uint32_t bits = row[w];
    n += __popc(bits);
    if (colcnt)
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        const int j = 32 * w + b;
        if (j < t_c) atomicAdd(&colcnt[(size_t)h * t_c + j], 1ull);
      }
  }
  if (rowptr) rowptr[r] = n;
}

// in-place exclusive scan of a[0..n) (n+1 entries, a[n] = total), one CTA
__global__ void lists_scan(int64_t* a, int n) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x, T = blockDim.x;
  const int per = (n + T - 1) / T;
  const int b0 = min(n, t * per), b1 = min(n, b0 + per);
  int64_t s = 0;
  for (int i = b0; i < b1; ++i) s += a[i];
  part[t] = s;
  __syncthreads();
  for (int o = 1; o < T; o <<= 1) {  // Hillis-Steele inclusive scan of the partials
    const int64_t v = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int64_t run = part[t] - s;  // exclusive prefix of this thread's range
  for (int i = b0; i < b1; ++i) {
    const int64_t v = a[i];
    a[i] = run;
    run += v;
  }
  if (t == T - 1) a[n] = part[T - 1];
}

__global__ void lists_fill_rows(const uint32_t* __restrict__ mask, int rows_total, int t_c,
                                int wpr, const int64_t* __restrict__ rowptr, int32_t* cols) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows_total) return;
  const uint32_t* row = mask + (size_t)r * wpr;
  int64_t o = rowptr[r];
  for (int w = 0; w < wpr; ++w) {
    uint32_t bits = row[w];
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int j = 32 * w + b;
      if (j < t_c) cols[o++] = j;
    }
  }
}

__global__ void lists_fill_cols(const uint32_t* __restrict__ mask, int cols_total, int t_r,
                                int t_c, int wpr, const int64_t* __restrict__ colptr,
                                int32_t* rows) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols_total) return;
  const int h = c / t_c, j = c - h * t_c;
  const uint32_t* m = mask + (size_t)h * t_r * wpr + (j >> 5);
  const uint32_t bit = 1u << (j & 31);
  int64_t o = colptr[c];
  for (int i = 0; i < t_r; ++i)
    if (m[(size_t)i * wpr] & bit) rows[o++] = i;
}

// ELL row lists: one thread per (head, row block) writes the ascending active
// key blocks of its mask row at rcol[row * t_c ..] and their count
__global__ void ell_rows_kernel(const uint32_t* __restrict__ mask, int rows_total, int t_c, int wpr,
                                int32_t* __restrict__ rcnt, uint16_t* __restrict__ rcol) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows_total) return;
  const uint32_t* row = mask + (size_t)r * wpr;
  uint16_t* out = rcol + (size_t)r * t_c;
  int n = 0;
  for (int w = 0; w < wpr; ++w)
    for (uint32_t bits = row[w]; bits; bits &= bits - 1) {
      const int j = 32 * w + __ffs(bits) - 1;
      if (j < t_c) out[n++] = (uint16_t)j;
    }
  rcnt[r] = n;
}

// ELL column lists from the row lists: one warp per (head, key block j); lane l
// looks j up (binary search) in the lists of row blocks l, l + 32, ..., and a
// ballot keeps the hits in ascending row order
__global__ void ell_cols_kernel(const int32_t* __restrict__ rcnt, const uint16_t* __restrict__ rcol,
                                int cols_total, int t_r, int t_c, int32_t* __restrict__ ccnt,
                                uint16_t* __restrict__ crow) {
  const int c = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= cols_total) return;
  const int h = c / t_c, j = c - h * t_c;
  uint16_t* out = crow + (size_t)c * t_r;
  int n = 0;
  for (int i0 = 0; i0 < t_r; i0 += 32) {
    const int i = i0 + lane;
    bool hit = false;
    if (i < t_r) {
      const size_t row = (size_t)h * t_r + i;
      const uint16_t* l = rcol + row * t_c;
      int lo = 0, hi = rcnt[row];  // first entry >= j
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (l[mid] < j) lo = mid + 1;
        else hi = mid;
      }
      hit = lo < rcnt[row] && l[lo] == j;
    }
    const uint32_t b = __ballot_sync(0xffffffffu, hit);
    if (hit) out[n + __popc(b & ((1u << lane) - 1u))] = (uint16_t)i;
    n += __popc(b);
  }
  if (lane == 0) ccnt[c] = n;
}

}  // namespace

cudaError_t ell_row_lists(const Geom& g, const uint32_t* mask, int32_t* rcnt, uint16_t* rcol,
                          cudaStream_t st) {
  const int R = g.bh * g.t_r, T = 128;
  ell_rows_kernel<<<(R + T - 1) / T, T, 0, st>>>(mask, R, g.t_c, g.wpr, rcnt, rcol);
  note_launch();
  return cudaGetLastError();
}

cudaError_t ell_col_lists(const Geom& g, const int32_t* rcnt, const uint16_t* rcol, int32_t* ccnt,
                          uint16_t* crow, cudaStream_t st) {
  const int Cn = g.bh * g.t_c, T = 256;
  const size_t threads = (size_t)Cn * 32;
  ell_cols_kernel<<<(unsigned)((threads + T - 1) / T), T, 0, st>>>(rcnt, rcol, Cn, g.t_r, g.t_c,
                                                                    ccnt, crow);
  note_launch();
  return cudaGetLastError();
}

cudaError_t block_lists(const Geom& g, const uint32_t* mask, int64_t* rowptr, int32_t* cols,
                        int64_t* colptr, int32_t* rows, cudaStream_t st) {
  const int R = g.bh * g.t_r, Cn = g.bh * g.t_c;
  const int T = 256;
  const bool want_rows = rowptr != nullptr, want_cols = colptr != nullptr;
  if (want_cols && cudaMemsetAsync(colptr, 0, sizeof(int64_t) * ((size_t)Cn + 1), st)) return cudaGetLastError();
  lists_count<<<(R + T - 1) / T, T, 0, st>>>(mask, R, g.t_r, g.t_c, g.wpr, rowptr,
                                              want_cols ? reinterpret_cast<unsigned long long*>(colptr) : nullptr);
  note_launch();
  if (want_rows) {
    lists_scan<<<1, 1024, 0, st>>>(rowptr, R);
    note_launch();
    if (cols) {
      lists_fill_rows<<<(R + T - 1) / T, T, 0, st>>>(mask, R, g.t_c, g.wpr, rowptr, cols);
      note_launch();
    }
  }
  if (want_cols) {
    lists_scan<<<1, 1024, 0, st>>>(colptr, Cn);
    note_launch();
    if (rows) {
      lists_fill_cols<<<(Cn + T - 1) / T, T, 0, st>>>(mask, Cn, g.t_r, g.t_c, g.wpr, colptr, rows);
      note_launch();
    }
  }
  return cudaGetLastError();
}

}  // namespace adattn_b200
