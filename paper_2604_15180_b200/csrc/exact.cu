// exact.cu -- EXACT path: fp64 SIMT kernels that keep the reference's
// operation order, so fp32/bf16-representable inputs give bit-identical
// tau / row_max / mask / out / delta / dq / dk / dv to the reference
// (/root/reference/proj/src/attention.cpp).  Compiled with -fmad=false: every
// a*b+c below is a separate multiply and add unless written as fma(), and
// fma() is only used where the product is exact (fp32/bf16 operands), where it
// equals the reference's `s += a[x] * b[x]` bit for bit.
//
// One CTA of 256 threads per 64-row query tile (forward, delta, dQ) or per
// 64-key tile (dK/dV), one writer per output element (the reference's
// determinism rule, README.md:30-33), fixed ascending accumulation order.
#include <cuda_bf16.h>
#include <math_constants.h>

#include "common.cuh"
#include "exact.cuh"

namespace adattn_b200 {
namespace {

constexpr int kThreads = 256;
constexpr int kTile = 64;   // max block_r / block_c on this path
constexpr int kChunk = 16;  // key/query chunk for the backward kernels
constexpr int kLdz = kTile + 1;
constexpr double kMaskSlack = 1e-9;       // attention.cpp:25
constexpr double kDerivBaseFloor = 1e-12; // attention.cpp:27

__host__ __device__ __forceinline__ int odd_ld(int w) { return w | 1; }

// s += a*b with the reference's rounding: fused when the product is exact.
template <bool kExactProd>
__device__ __forceinline__ double madd(double a, double b, double acc) {
  if constexpr (kExactProd) return fma(a, b, acc);
  else return acc + a * b;
}

// dst[r*ld + x] = src[row0 + r][x] for r < valid_rows, 0 for valid_rows <= r < rows.
__device__ __forceinline__ void load_rows(double* dst, int ld, const void* src, size_t base,
                                          int row0, int valid_rows, int rows, int width,
                                          int dtype) {
  for (int i = threadIdx.x; i < rows * width; i += kThreads) {
    const int r = i / width, x = i - r * width;
    double val = 0.0;
    if (r < valid_rows) val = load_elem(src, base + (size_t)(row0 + r) * width + x, dtype);
    dst[r * ld + x] = val;
  }
}

__device__ __forceinline__ double dmaxd(double a, double b) { return (a < b) ? b : a; }

// 64x64 score micro-tiles: thread (ty, tx) owns rows 4ty..4ty+3, cols tx+16j.
template <bool kExactProd>
__device__ __forceinline__ void score_tile(const double* __restrict__ sQ, int ldq,
                                           const double* __restrict__ sK, int ldk, int d,
                                           double acc[4][4]) {
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int x = 0; x < d; ++x) {
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = sQ[(ty * 4 + i) * ldq + x];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = sK[(tx + 16 * j) * ldk + x];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = madd<kExactProd>(a[i], b[j], acc[i][j]);
  }
}

// z of compute_z_block (attention.cpp:81)
__device__ __forceinline__ double centre(double s, double m, double am1) {
  return s == m ? 1.0 : am1 * (s - m) + 1.0;
}

// --------------------------------------------------------------- forward

template <bool kExactProd>
__global__ void __launch_bounds__(kThreads, 1)
    exact_forward_kernel(Geom g, const void* __restrict__ q, const void* __restrict__ k,
                         const void* __restrict__ v, void* __restrict__ out,
                         double* __restrict__ tau_out, double* __restrict__ rmax_out,
                         uint32_t* __restrict__ mask_out, int32_t* __restrict__ steps_out) {
  const int it = blockIdx.x, bh = blockIdx.y;
  const int r0 = it * g.block_r;
  const int nr = min(g.block_r, g.n - r0);
  const int jlim = g.causal ? (r0 + nr - 1) / g.block_c : g.t_c - 1;
  const int ldq = odd_ld(g.d), ldk = odd_ld(max(g.d, g.dv));
  extern __shared__ double smem[];
  double* sQ = smem;
  double* sK = sQ + kTile * ldq;
  double* sZ = sK + kTile * ldk;
  double* sRowMax = sZ + kTile * kLdz;
  double* sTau = sRowMax + kTile;
  uint32_t* sCnt = reinterpret_cast<uint32_t*>(sTau + kTile);
  uint32_t* sAct = sCnt + kTile * g.bins;

  const size_t qbase = (size_t)bh * g.n * g.d, kbase = (size_t)bh * g.m * g.d;
  const size_t vbase = (size_t)bh * g.m * g.dv;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const double am1 = g.alpha - 1.0;
  const double e0 = g.e0, e1 = e0 - 1.0, e2 = e0 - 2.0;

  unsigned long long* const pacc = tid == 0 ? g.phase_ns : nullptr;
  unsigned long long pt = pacc ? global_ns() : 0ull;
  load_rows(sQ, ldq, q, qbase, r0, nr, kTile, g.d, g.in_dtype);
  for (int i = tid; i < kTile; i += kThreads) sRowMax[i] = -CUDART_INF;
  for (int i = tid; i < kTile * g.bins; i += kThreads) sCnt[i] = 0u;

  // Phase 1: row maxima (attention.cpp:182-195)
  for (int jt = 0; jt <= jlim; ++jt) {
    const int c0 = jt * g.block_c, nc = min(g.block_c, g.m - c0);
    __syncthreads();
    load_rows(sK, ldk, k, kbase, c0, nc, kTile, g.d, g.in_dtype);
    __syncthreads();
    double acc[4][4];
    score_tile<kExactProd>(sQ, ldq, sK, ldk, g.d, acc);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = ty * 4 + i;
      double lm = -CUDART_INF;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = tx + 16 * j;
        const bool ok = r < nr && c < nc && !(g.causal && c0 + c > r0 + r);
        if (ok) lm = dmaxd(lm, g.scale * acc[i][j]);
      }
#pragma unroll
      for (int off = 8; off >= 1; off >>= 1) lm = dmaxd(lm, __shfl_xor_sync(0xffffffffu, lm, off));
      if (tx == 0 && r < nr) sRowMax[r] = dmaxd(sRowMax[r], lm);
    }
  }

  phase_tick(pacc, 0, pt);
  // Phase 2: histogram counts of z >= 0 (attention.cpp:110-155, 201-210)
  for (int jt = 0; jt <= jlim; ++jt) {
    const int c0 = jt * g.block_c, nc = min(g.block_c, g.m - c0);
    __syncthreads();
    load_rows(sK, ldk, k, kbase, c0, nc, kTile, g.d, g.in_dtype);
    __syncthreads();
    double acc[4][4];
    score_tile<kExactProd>(sQ, ldq, sK, ldk, g.d, acc);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = ty * 4 + i;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = tx + 16 * j;
        const bool ok = r < nr && c < nc && !(g.causal && c0 + c > r0 + r);
        if (!ok) continue;
        const double z = centre(g.scale * acc[i][j], sRowMax[r], am1);
        if (!(z >= 0.0)) continue;
        const int b = min((int)(g.bins * z), g.bins - 1);
        atomicAdd(&sCnt[r * g.bins + b], 1u);
      }
    }
  }
  __syncthreads();

  // Threshold init per row (attention.cpp:223-228)
  RowSolve rs;
  const bool own_row = tid < nr;
  if (own_row) {
    double th, lo, hi;
    solve_histogram_dev(&sCnt[tid * g.bins], g.bins, g.alpha, th, lo, hi);
    if (g.tau_h_out) g.tau_h_out[(size_t)bh * g.n + r0 + tid] = th;
    rs.tau = th;
    rs.lo = lo;
    rs.hi = hi;
    rs.f = rs.f1 = rs.f2 = rs.f_hi = 0.0;
    rs.sec_tau = rs.sec_f = rs.best_tau = 0.0;
    rs.best_af = CUDART_INF;
    rs.steps = 0;
    rs.sec_seeded = false;
    rs.done = false;
  }

  phase_tick(pacc, 1, pt);
  // Phase 3: refinement passes (attention.cpp:234-332)
  const bool need_sec = g.alpha > 2.0;
  bool first_pass = true;
  for (;;) {
    if (own_row) {
      rs.f = -1.0;
      rs.f1 = 0.0;
      rs.f2 = 0.0;
      if (first_pass) rs.f_hi = -1.0;
    }
    for (int w = tid; w < g.wpr; w += kThreads) sAct[w] = 0u;
    for (int jt = 0; jt <= jlim; ++jt) {
      const int c0 = jt * g.block_c, nc = min(g.block_c, g.m - c0);
      __syncthreads();
      load_rows(sK, ldk, k, kbase, c0, nc, kTile, g.d, g.in_dtype);
      __syncthreads();
      double acc[4][4];
      score_tile<kExactProd>(sQ, ldq, sK, ldk, g.d, acc);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = ty * 4 + i;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = tx + 16 * j;
          if (r < nr && c < nc)
            sZ[r * kLdz + c] = (g.causal && c0 + c > r0 + r)
                                   ? -CUDART_INF
                                   : centre(g.scale * acc[i][j], sRowMax[r], am1);
        }
      }
      __syncthreads();
      int any = 0;
      if (own_row) {
        const double* zr = sZ + tid * kLdz;
        if (rs.done) {
          for (int c = 0; c < nc; ++c) any |= (zr[c] > rs.tau - kMaskSlack);
        } else {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, shi = 0.0;
          for (int c = 0; c < nc; ++c) {
            const double t = zr[c] - rs.tau;
            any |= (t > -kMaskSlack);
            if (t > 0.0) {
              s0 += pow_e(t, e0);
              s1 += pow_e(e1 < 0.0 ? dmaxd(t, kDerivBaseFloor) : t, e1);
              s2 += pow_e(e2 < 0.0 ? dmaxd(t, kDerivBaseFloor) : t, e2);
            }
            if (first_pass && need_sec) {
              const double th = zr[c] - rs.hi;
              if (th > 0.0) shi += pow_e(th, e0);
            }
          }
          rs.f += s0;
          rs.f1 -= e0 * s1;
          rs.f2 += e0 * (e0 - 1.0) * s2;
          if (first_pass && need_sec) rs.f_hi += shi;
        }
      }
      if (__syncthreads_or(any) && tid == 0) sAct[jt >> 5] |= 1u << (jt & 31);
    }
    int stepped = 0;
    if (own_row) stepped = row_step(rs, g.alpha, g.refine_tol, g.refine_iters, need_sec);
    first_pass = false;
    if (!__syncthreads_or(stepped)) break;
  }

  const size_t rowbase = (size_t)bh * g.n + r0;
  if (own_row) {
    tau_out[rowbase + tid] = rs.tau;
    rmax_out[rowbase + tid] = sRowMax[tid];
    if (steps_out) steps_out[rowbase + tid] = rs.steps;
    sTau[tid] = rs.tau;
  }
  for (int w = tid; w < g.wpr; w += kThreads)
    mask_out[((size_t)bh * g.t_r + it) * g.wpr + w] = sAct[w];

  phase_tick(pacc, 2, pt);
  // Phase 4: O over the set mask bits, ascending (attention.cpp:334-352)
  const int xg = tid & 31, rg = tid >> 5;
  double oacc[8][4];
#pragma unroll
  for (int ii = 0; ii < 8; ++ii)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) oacc[ii][jj] = 0.0;
  for (int jt = 0; jt <= jlim; ++jt) {
    if (!((sAct[jt >> 5] >> (jt & 31)) & 1u)) continue;
    const int c0 = jt * g.block_c, nc = min(g.block_c, g.m - c0);
    __syncthreads();
    load_rows(sK, ldk, k, kbase, c0, nc, kTile, g.d, g.in_dtype);
    __syncthreads();
    double acc[4][4];
    score_tile<kExactProd>(sQ, ldq, sK, ldk, g.d, acc);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = ty * 4 + i;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = tx + 16 * j;
        double pv = 0.0;
        if (r < nr && c < nc && !(g.causal && c0 + c > r0 + r)) {
          const double t = centre(g.scale * acc[i][j], sRowMax[r], am1) - sTau[r];
          if (t > 0.0) pv = pow_e(t, e0);
        }
        sZ[r * kLdz + c] = pv;
      }
    }
    __syncthreads();
    load_rows(sK, ldk, v, vbase, c0, nc, kTile, g.dv, g.in_dtype);
    __syncthreads();
    for (int c = 0; c < nc; ++c) {
#pragma unroll
      for (int ii = 0; ii < 8; ++ii) {
        const double pv = sZ[(rg + 8 * ii) * kLdz + c];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int x = xg + 32 * jj;
          if (x < g.dv) oacc[ii][jj] = oacc[ii][jj] + pv * sK[c * ldk + x];
        }
      }
    }
  }
  const size_t obase = (size_t)bh * g.n * g.dv;
#pragma unroll
  for (int ii = 0; ii < 8; ++ii) {
    const int r = rg + 8 * ii;
    if (r >= nr) continue;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int x = xg + 32 * jj;
      if (x < g.dv) store_elem(out, obase + (size_t)(r0 + r) * g.dv + x, g.out_dtype, oacc[ii][jj]);
    }
  }
  phase_tick(pacc, 3, pt);
}

// ---------------------------------------------------------- compute_delta

__device__ __forceinline__ bool mask_bit(const uint32_t* mask, const Geom& g, int bh, int it,
                                         int jt) {
  return (mask[((size_t)bh * g.t_r + it) * g.wpr + (jt >> 5)] >> (jt & 31)) & 1u;
}

template <bool kExactProd>
__global__ void __launch_bounds__(kThreads, 1)
    exact_delta_kernel(Geom g, const void* __restrict__ q, const void* __restrict__ k,
                       const void* __restrict__ v, const double* __restrict__ tau,
                       const double* __restrict__ row_max, const uint32_t* __restrict__ mask,
                       const void* __restrict__ dout, double* __restrict__ delta) {
  const int it = blockIdx.x, bh = blockIdx.y;
  const int r0 = it * g.block_r, nr = min(g.block_r, g.n - r0);
  const int ldq = odd_ld(g.d), ldv = odd_ld(g.dv);
  extern __shared__ double smem[];
  double* sQ = smem;
  double* sDO = sQ + kTile * ldq;
  double* sKc = sDO + kTile * ldv;
  double* sVc = sKc + kChunk * ldq;
  double* sZ = sVc + kChunk * ldv;          // [64][17]
  double* sDP = sZ + kTile * (kChunk + 1);  // [64][17]
  double* sRm = sDP + kTile * (kChunk + 1);
  double* sTau = sRm + kTile;
  const int tid = threadIdx.x;
  const size_t qbase = (size_t)bh * g.n * g.d, kbase = (size_t)bh * g.m * g.d;
  const size_t vbase = (size_t)bh * g.m * g.dv, obase = (size_t)bh * g.n * g.dv;
  const size_t rowbase = (size_t)bh * g.n + r0;
  const double am1 = g.alpha - 1.0, e0 = g.e0, ue = 2.0 - g.alpha;

  load_rows(sQ, ldq, q, qbase, r0, nr, kTile, g.d, g.in_dtype);
  load_rows(sDO, ldv, dout, obase, r0, nr, kTile, g.dv, g.in_dtype);
  for (int i = tid; i < kTile; i += kThreads) {
    sRm[i] = i < nr ? row_max[rowbase + i] : 0.0;
    sTau[i] = i < nr ? tau[rowbase + i] : 0.0;
  }
  double num = 0.0, den = 0.0;
  const int r = tid >> 2, cq = tid & 3;
  for (int jt = 0; jt < g.t_c; ++jt) {
    if (!mask_bit(mask, g, bh, it, jt)) continue;
    const int c0 = jt * g.block_c, nc = min(g.block_c, g.m - c0);
    for (int cc = 0; cc < nc; cc += kChunk) {
      const int ncc = min(kChunk, nc - cc);
      __syncthreads();
      load_rows(sKc, ldq, k, kbase, c0 + cc, ncc, kChunk, g.d, g.in_dtype);
      load_rows(sVc, ldv, v, vbase, c0 + cc, ncc, kChunk, g.dv, g.in_dtype);
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = cq + 4 * j;
        double s = 0.0, dp = 0.0;
        for (int x = 0; x < g.d; ++x) s = madd<kExactProd>(sQ[r * ldq + x], sKc[c * ldq + x], s);
        for (int x = 0; x < g.dv; ++x)
          dp = madd<kExactProd>(sDO[r * ldv + x], sVc[c * ldv + x], dp);
        const int cg = c0 + cc + c;
        const bool ok = r < nr && c < ncc && !(g.causal && cg > r0 + r);
        sZ[r * (kChunk + 1) + c] = ok ? centre(g.scale * s, sRm[r], am1) : -CUDART_INF;
        sDP[r * (kChunk + 1) + c] = dp;
      }
      __syncthreads();
      if (tid < nr) {
        for (int c = 0; c < ncc; ++c) {
          const double t = sZ[tid * (kChunk + 1) + c] - sTau[tid];
          if (t <= 0.0) continue;
          const double pv = pow_e(t, e0);
          const double u = pow_e(pv, ue);
          num += u * sDP[tid * (kChunk + 1) + c];
          den += u;
        }
      }
    }
  }
  if (tid < nr) delta[rowbase + tid] = den > 0.0 ? num / den : 0.0;
}

// ------------------------------------------------- backward: key-major dK/dV

template <bool kExactProd>
__global__ void __launch_bounds__(kThreads, 1)
    exact_dkdv_kernel(Geom g, const void* __restrict__ q, const void* __restrict__ k,
                      const void* __restrict__ v, const double* __restrict__ tau,
                      const double* __restrict__ row_max, const uint32_t* __restrict__ mask,
                      const void* __restrict__ dout, const double* __restrict__ delta,
                      void* __restrict__ dk, void* __restrict__ dv,
                      unsigned long long* __restrict__ visited) {
  const int jt = blockIdx.x, bh = blockIdx.y;
  const int c0 = jt * g.block_c, nc = min(g.block_c, g.m - c0);
  const int ldq = odd_ld(g.d), ldv = odd_ld(g.dv);
  extern __shared__ double smem[];
  double* sK = smem;
  double* sV = sK + kTile * ldq;
  double* sQc = sV + kTile * ldv;
  double* sDOc = sQc + kChunk * ldq;
  double* sP = sDOc + kChunk * ldv;       // [16][65]
  double* sDS = sP + kChunk * kLdz;       // [16][65]
  double* sRm = sDS + kChunk * kLdz;
  double* sTau = sRm + kChunk;
  double* sDl = sTau + kChunk;
  const int tid = threadIdx.x;
  const size_t qbase = (size_t)bh * g.n * g.d, kbase = (size_t)bh * g.m * g.d;
  const size_t vbase = (size_t)bh * g.m * g.dv, obase = (size_t)bh * g.n * g.dv;
  const double am1 = g.alpha - 1.0, e0 = g.e0, ue = 2.0 - g.alpha;

  load_rows(sK, ldq, k, kbase, c0, nc, kTile, g.d, g.in_dtype);
  load_rows(sV, ldv, v, vbase, c0, nc, kTile, g.dv, g.in_dtype);
  // accumulator ownership: key row kc, columns xq + 4*jj
  const int kc = tid >> 2, xq = tid & 3;
  double accV[32], accK[32];
#pragma unroll
  for (int jj = 0; jj < 32; ++jj) accV[jj] = accK[jj] = 0.0;
  // score ownership inside a 16x64 chunk: row sr, columns sc + 16*j
  const int sr = tid >> 4, sc = tid & 15;
  unsigned long long nvis = 0;
  for (int it = 0; it < g.t_r; ++it) {
    if (!mask_bit(mask, g, bh, it, jt)) continue;
    ++nvis;
    const int r0 = it * g.block_r, nr = min(g.block_r, g.n - r0);
    for (int rc = 0; rc < nr; rc += kChunk) {
      const int nrc = min(kChunk, nr - rc);
      __syncthreads();
      load_rows(sQc, ldq, q, qbase, r0 + rc, nrc, kChunk, g.d, g.in_dtype);
      load_rows(sDOc, ldv, dout, obase, r0 + rc, nrc, kChunk, g.dv, g.in_dtype);
      for (int i = tid; i < kChunk; i += kThreads) {
        const size_t row = (size_t)bh * g.n + r0 + rc + i;
        sRm[i] = i < nrc ? row_max[row] : 0.0;
        sTau[i] = i < nrc ? tau[row] : 0.0;
        sDl[i] = i < nrc ? delta[row] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = sc + 16 * j;
        double s = 0.0, dp = 0.0;
        for (int x = 0; x < g.d; ++x) s = madd<kExactProd>(sQc[sr * ldq + x], sK[c * ldq + x], s);
        for (int x = 0; x < g.dv; ++x)
          dp = madd<kExactProd>(sDOc[sr * ldv + x], sV[c * ldv + x], dp);
        double pv = 0.0, ds = 0.0;
        const bool ok = sr < nrc && c < nc && !(g.causal && c0 + c > r0 + rc + sr);
        if (ok) {
          const double t = centre(g.scale * s, sRm[sr], am1) - sTau[sr];
          if (t > 0.0) {
            pv = pow_e(t, e0);
            const double u = pow_e(pv, ue);
            ds = u * (dp - sDl[sr]);
          }
        }
        sP[sr * kLdz + c] = pv;
        sDS[sr * kLdz + c] = ds;
      }
      __syncthreads();
      for (int rr = 0; rr < nrc; ++rr) {
        const double pv = sP[rr * kLdz + kc];
        const double ds = sDS[rr * kLdz + kc];
        if (pv != 0.0) {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const int x = xq + 4 * jj;
            if (x < g.dv) accV[jj] = accV[jj] + pv * sDOc[rr * ldv + x];
          }
        }
        if (ds != 0.0) {
          const double w = g.scale * ds;
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const int x = xq + 4 * jj;
            if (x < g.d) accK[jj] = accK[jj] + w * sQc[rr * ldq + x];
          }
        }
      }
    }
  }
  if (kc < nc) {
    const size_t kr = (size_t)bh * g.m + c0 + kc;
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
      const int x = xq + 4 * jj;
      if (x < g.dv) store_elem(dv, kr * g.dv + x, g.out_dtype, accV[jj]);
      if (x < g.d) store_elem(dk, kr * g.d + x, g.out_dtype, accK[jj]);
    }
  }
  if (tid == 0 && nvis) atomicAdd(visited, nvis);
}

// ----------------------------------------------- backward: query-major dQ

template <bool kExactProd>
__global__ void __launch_bounds__(kThreads, 1)
    exact_dq_kernel(Geom g, const void* __restrict__ q, const void* __restrict__ k,
                    const void* __restrict__ v, const double* __restrict__ tau,
                    const double* __restrict__ row_max, const uint32_t* __restrict__ mask,
                    const void* __restrict__ dout, const double* __restrict__ delta,
                    void* __restrict__ dq, unsigned long long* __restrict__ visited) {
  const int it = blockIdx.x, bh = blockIdx.y;
  const int r0 = it * g.block_r, nr = min(g.block_r, g.n - r0);
  const int ldq = odd_ld(g.d), ldv = odd_ld(g.dv);
  extern __shared__ double smem[];
  double* sQ = smem;
  double* sDO = sQ + kTile * ldq;
  double* sKc = sDO + kTile * ldv;
  double* sVc = sKc + kChunk * ldq;
  double* sW = sVc + kChunk * ldv;  // [64][17]
  double* sRm = sW + kTile * (kChunk + 1);
  double* sTau = sRm + kTile;
  double* sDl = sTau + kTile;
  const int tid = threadIdx.x;
  const size_t qbase = (size_t)bh * g.n * g.d, kbase = (size_t)bh * g.m * g.d;
  const size_t vbase = (size_t)bh * g.m * g.dv, obase = (size_t)bh * g.n * g.dv;
  const size_t rowbase = (size_t)bh * g.n + r0;
  const double am1 = g.alpha - 1.0, e0 = g.e0, ue = 2.0 - g.alpha;

  load_rows(sQ, ldq, q, qbase, r0, nr, kTile, g.d, g.in_dtype);
  load_rows(sDO, ldv, dout, obase, r0, nr, kTile, g.dv, g.in_dtype);
  for (int i = tid; i < kTile; i += kThreads) {
    sRm[i] = i < nr ? row_max[rowbase + i] : 0.0;
    sTau[i] = i < nr ? tau[rowbase + i] : 0.0;
    sDl[i] = i < nr ? delta[rowbase + i] : 0.0;
  }
  const int r = tid >> 2, xq = tid & 3;
  double accQ[32];
#pragma unroll
  for (int jj = 0; jj < 32; ++jj) accQ[jj] = 0.0;
  unsigned long long nvis = 0;
  for (int jt = 0; jt < g.t_c; ++jt) {
    if (!mask_bit(mask, g, bh, it, jt)) continue;
    ++nvis;
    const int c0 = jt * g.block_c, nc = min(g.block_c, g.m - c0);
    for (int cc = 0; cc < nc; cc += kChunk) {
      const int ncc = min(kChunk, nc - cc);
      __syncthreads();
      load_rows(sKc, ldq, k, kbase, c0 + cc, ncc, kChunk, g.d, g.in_dtype);
      load_rows(sVc, ldv, v, vbase, c0 + cc, ncc, kChunk, g.dv, g.in_dtype);
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = xq + 4 * j;
        double w = 0.0;
        const bool ok = r < nr && c < ncc && !(g.causal && c0 + cc + c > r0 + r);
        if (ok) {
          double s = 0.0;
          for (int x = 0; x < g.d; ++x) s = madd<kExactProd>(sQ[r * ldq + x], sKc[c * ldq + x], s);
          const double t = centre(g.scale * s, sRm[r], am1) - sTau[r];
          if (t > 0.0) {
            const double u = pow_e(pow_e(t, e0), ue);
            double dp = 0.0;
            for (int x = 0; x < g.dv; ++x)
              dp = madd<kExactProd>(sDO[r * ldv + x], sVc[c * ldv + x], dp);
            w = g.scale * u * (dp - sDl[r]);
          }
        }
        sW[r * (kChunk + 1) + c] = w;
      }
      __syncthreads();
      for (int c = 0; c < ncc; ++c) {
        const double w = sW[r * (kChunk + 1) + c];
        if (w == 0.0) continue;
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          const int x = xq + 4 * jj;
          if (x < g.d) accQ[jj] = accQ[jj] + w * sKc[c * ldq + x];
        }
      }
    }
  }
  if (r < nr) {
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
      const int x = xq + 4 * jj;
      if (x < g.d) store_elem(dq, (rowbase + r) * g.d + x, g.out_dtype, accQ[jj]);
    }
  }
  if (tid == 0 && nvis) atomicAdd(visited, nvis);
}

template <typename K>
cudaError_t prep(K kernel, size_t smem) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

}  // namespace

// (grid.y carries the head index: at most 65535 heads per call).  Blocks > 64 or
// widths > 128 run on the one-thread-per-row kernels of exact_generic.cu.
bool exact_supported(const Geom& g) { return g.bh <= 65535; }

static size_t fwd_smem(const Geom& g) {
  const int ldq = odd_ld(g.d), ldk = odd_ld(g.d > g.dv ? g.d : g.dv);
  return sizeof(double) * ((size_t)kTile * ldq + (size_t)kTile * ldk + (size_t)kTile * kLdz +
                           2 * kTile) +
         sizeof(uint32_t) * ((size_t)kTile * g.bins + g.wpr);
}
static size_t delta_smem(const Geom& g) {
  const int ldq = odd_ld(g.d), ldv = odd_ld(g.dv);
  return sizeof(double) * ((size_t)kTile * ldq + (size_t)kTile * ldv + (size_t)kChunk * ldq +
                           (size_t)kChunk * ldv + 2 * (size_t)kTile * (kChunk + 1) + 2 * kTile);
}
static size_t dkdv_smem(const Geom& g) {
  const int ldq = odd_ld(g.d), ldv = odd_ld(g.dv);
  return sizeof(double) * ((size_t)kTile * ldq + (size_t)kTile * ldv + (size_t)kChunk * ldq +
                           (size_t)kChunk * ldv + 2 * (size_t)kChunk * kLdz + 3 * kChunk);
}
static size_t dq_smem(const Geom& g) {
  const int ldq = odd_ld(g.d), ldv = odd_ld(g.dv);
  return sizeof(double) * ((size_t)kTile * ldq + (size_t)kTile * ldv + (size_t)kChunk * ldq +
                           (size_t)kChunk * ldv + (size_t)kTile * (kChunk + 1) + 3 * kTile);
}

cudaError_t exact_forward(const Geom& g, const void* q, const void* k, const void* v, void* out,
                          double* tau, double* row_max, uint32_t* mask, int32_t* steps,
                          cudaStream_t st) {
  if (exact_generic_needed(g))
    return exact_generic_forward(g, q, k, v, out, tau, row_max, mask, steps, st);
  const size_t smem = fwd_smem(g);
  const dim3 grid(g.t_r, g.bh);
  cudaError_t e;
  if (g.in_dtype == ADATTN_F64) {
    if ((e = prep(exact_forward_kernel<false>, smem))) return e;
    prof_begin("exact_fwd", st);
    exact_forward_kernel<false><<<grid, kThreads, smem, st>>>(g, q, k, v, out, tau, row_max,
                                                             mask, steps);
  } else {
    if ((e = prep(exact_forward_kernel<true>, smem))) return e;
    prof_begin("exact_fwd", st);
    exact_forward_kernel<true><<<grid, kThreads, smem, st>>>(g, q, k, v, out, tau, row_max,
                                                            mask, steps);
  }
  prof_end(st);
  note_launch();
  return cudaGetLastError();
}

cudaError_t exact_delta(const Geom& g, const void* q, const void* k, const void* v,
                        const double* tau, const double* row_max, const uint32_t* mask,
                        const void* dout, double* delta, cudaStream_t st) {
  if (exact_generic_needed(g))
    return exact_generic_delta(g, q, k, v, tau, row_max, mask, dout, delta, st);
  const size_t smem = delta_smem(g);
  const dim3 grid(g.t_r, g.bh);
  cudaError_t e;
  if (g.in_dtype == ADATTN_F64) {
    if ((e = prep(exact_delta_kernel<false>, smem))) return e;
    exact_delta_kernel<false><<<grid, kThreads, smem, st>>>(g, q, k, v, tau, row_max, mask,
                                                           dout, delta);
  } else {
    if ((e = prep(exact_delta_kernel<true>, smem))) return e;
    exact_delta_kernel<true><<<grid, kThreads, smem, st>>>(g, q, k, v, tau, row_max, mask,
                                                          dout, delta);
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t exact_backward(const Geom& g, const void* q, const void* k, const void* v,
                           const double* tau, const double* row_max, const uint32_t* mask,
                           const void* dout, void* dq, void* dk, void* dv, double* delta,
                           unsigned long long* visited, cudaStream_t st) {
  if (exact_generic_needed(g))
    return exact_generic_backward(g, q, k, v, tau, row_max, mask, dout, dq, dk, dv, delta,
                                  visited, st);
  cudaError_t e = exact_delta(g, q, k, v, tau, row_max, mask, dout, delta, st);
  if (e) return e;
  const size_t s1 = dkdv_smem(g), s2 = dq_smem(g);
  if (g.in_dtype == ADATTN_F64) {
    if ((e = prep(exact_dkdv_kernel<false>, s1))) return e;
    if ((e = prep(exact_dq_kernel<false>, s2))) return e;
    exact_dkdv_kernel<false><<<dim3(g.t_c, g.bh), kThreads, s1, st>>>(
        g, q, k, v, tau, row_max, mask, dout, delta, dk, dv, visited);
    exact_dq_kernel<false><<<dim3(g.t_r, g.bh), kThreads, s2, st>>>(g, q, k, v, tau, row_max,
                                                                    mask, dout, delta, dq, visited);
  } else {
    if ((e = prep(exact_dkdv_kernel<true>, s1))) return e;
    if ((e = prep(exact_dq_kernel<true>, s2))) return e;
    exact_dkdv_kernel<true><<<dim3(g.t_c, g.bh), kThreads, s1, st>>>(
        g, q, k, v, tau, row_max, mask, dout, delta, dk, dv, visited);
    exact_dq_kernel<true><<<dim3(g.t_r, g.bh), kThreads, s2, st>>>(g, q, k, v, tau, row_max,
                                                                   mask, dout, delta, dq, visited);
  }
  note_launch();
  note_launch();
  return cudaGetLastError();
}

}  // namespace adattn_b200
