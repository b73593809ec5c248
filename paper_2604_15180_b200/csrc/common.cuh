// common.cuh -- shared geometry, element loads and the per-row threshold
// solver (histogram init + safeguarded step) used by every kernel family.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "adattn_b200.h"

namespace adattn_b200 {

// Launch-time geometry shared by all kernels (one problem = B*H heads).
struct Geom {
  int bh;         // batch * heads
  int n, m, d, dv;
  // rows / keys that exist (the tensor-core path runs ragged problems padded to
  // n % 256 == 0, m % 128 == 0; rows >= n_valid and keys >= m_valid are padding)
  int n_valid, m_valid;
  int t_r, t_c;   // query / key tile counts
  int wpr;        // mask words per tile row = ceil(t_c / 32)
  int block_r, block_c;
  int bins;
  int causal;
  int refine_iters;
  int in_dtype, out_dtype;
  double alpha, scale, refine_tol;
  double e0;      // 1/(alpha-1)
  // PhaseTimings (attention.hpp:62-66): when set, one thread per forward CTA adds the
  // nanoseconds it spends in each reference phase (max, histogram, refinement,
  // output) to phase_ns[0..3]
  unsigned long long* phase_ns = nullptr;
  // when set, the forward writes each row's histogram solution tau_h
  // (solve_histogram, histogram.cpp:73-161) to tau_h_out[bh * n + row]
  double* tau_h_out = nullptr;
  // nonzero-block lists (ELL: per row block the count and the ascending key blocks,
  // [bh][t_r] / [bh][t_r][t_c] in the caller's geometry): emitted by the forward
  // when set, consumed by the backward when set (else built from the mask)
  int32_t* rl_cnt_out = nullptr;
  uint16_t* rl_col_out = nullptr;
  const int32_t* rl_cnt_in = nullptr;
  const uint16_t* rl_col_in = nullptr;
  // delta fold (tensor-core path): the forward writes Ubar_i = sum_j u_ij v_j
  // ([bh][n][dv] fp32) then sum_j u_ij ([bh][n] fp32) to ubar_out; the backward
  // reads them from ubar_in and forms delta_i = dO_i . Ubar_i / sum_j u_ij
  // (attention.cpp:411-446) instead of running the delta kernel
  float* ubar_out = nullptr;
  const float* ubar_in = nullptr;
  // delta from the support lists (tensor-core list mode, tc.cu supp_layout): the forward
  // writes each row's keys and u with t > 0 at the final tau to supp_out; the backward
  // forms delta_i = sum u_ij (dO_i . v_j) / sum u_ij from supp_in (the delta kernel takes
  // the heads flagged as overflowed)
  void* supp_out = nullptr;
  const void* supp_in = nullptr;
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// close phase `i` of this CTA: add the time since `t` and restart the clock
__device__ __forceinline__ void phase_tick(unsigned long long* acc, int i, unsigned long long& t) {
  if (acc) {
    const unsigned long long now = global_ns();
    atomicAdd(acc + i, now - t);
    t = now;
  }
}

__device__ __forceinline__ double load_elem(const void* base, size_t i, int dtype) {
  if (dtype == ADATTN_BF16)
    return (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[i]);
  if (dtype == ADATTN_F32) return (double)reinterpret_cast<const float*>(base)[i];
  return reinterpret_cast<const double*>(base)[i];
}

__device__ __forceinline__ void store_elem(void* base, size_t i, int dtype, double v) {
  if (dtype == ADATTN_F64)
    reinterpret_cast<double*>(base)[i] = v;
  else
    reinterpret_cast<float*>(base)[i] = (float)v;
}

// pow_e (reference internal.hpp:13-19): exponent fast paths.
template <typename T>
__device__ __forceinline__ T pow_e(T base, T e) {
  if (e == T(1)) return base;
  if (e == T(2)) return base * base;
  if (e == T(0)) return T(1);
  if (e == T(0.5)) return sqrt(base);
  return pow(base, e);
}

// f_h_eval, left-edge representatives (reference histogram.cpp:40-50).
__device__ inline double f_h_eval_dev(const uint32_t* counts, int bins, double width,
                                      double tau, double alpha) {
  const double e0 = 1.0 / (alpha - 1.0);
  double sum = 0.0;
  for (int k = 0; k < bins; ++k) {
    if (counts[k] == 0) continue;
    const double t = (k + 0.0) * width - tau;
    if (t > 0.0) sum += (double)counts[k] * pow_e(t, e0);
  }
  return sum - 1.0;
}

// solve_histogram (reference histogram.cpp:73-161) + refine_bracket (163-165).
// Writes tau_h and the refinement bracket [tau_h, tau_h + 1/B].
// floor_out (optional): the bracket floor edge index (-1: no edge with f_h >= 0).
__device__ inline void solve_histogram_dev(const uint32_t* counts, int bins, double alpha,
                                           double& tau_h, double& lo_out, double& hi_out,
                                           int* floor_out = nullptr) {
  const int B = bins;
  const double w = 1.0 / bins;
  const double e0 = 1.0 / (alpha - 1.0);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  int floor_k = -1;
  for (int k = B - 1; k >= 0; --k) {
    const double tau = k * w;
    double fh;
    if (e0 == 1.0)
      fh = s1 - tau * s0 - 1.0;
    else if (e0 == 2.0)
      fh = s2 - 2.0 * tau * s1 + tau * tau * s0 - 1.0;
    else
      fh = f_h_eval_dev(counts, bins, w, tau, alpha);
    if (fh >= 0.0) {
      floor_k = k;
      break;
    }
    const double v = k * w;
    s0 += counts[k];
    s1 += counts[k] * v;
    s2 += counts[k] * v * v;
  }
  if (floor_out) *floor_out = floor_k;
  double th = 0.0;
  if (floor_k >= 0) {
    const double lo = floor_k * w;
    const double hi = (floor_k + 1) * w;
    double tau;
    if (e0 == 1.0) {
      tau = (s1 - 1.0) / s0;
    } else if (e0 == 2.0) {
      double disc = s1 * s1 - s0 * (s2 - 1.0);
      disc = disc < 0.0 ? 0.0 : disc;
      tau = (s1 - sqrt(disc)) / s0;
    } else {
      // bisect_f_h (histogram.cpp:57-69)
      double blo = lo, bhi = hi;
      tau = -1.0;
      for (int it = 0; it < 200 && bhi - blo > 1e-10; ++it) {
        const double mid = 0.5 * (blo + bhi);
        const double val = f_h_eval_dev(counts, bins, w, mid, alpha);
        if (val == 0.0) {
          tau = mid;
          break;
        }
        if (val > 0.0)
          blo = mid;
        else
          bhi = mid;
      }
      if (tau < 0.0) tau = blo;
    }
    const double top = nextafter(hi, lo);
    th = tau < lo ? lo : (top < tau ? top : tau);
  }
  tau_h = th;
  lo_out = th;
  hi_out = th + w;
}

// propose_step (reference internal.hpp:32-55).
__device__ __forceinline__ double propose_step_dev(double alpha, double tau, double f,
                                                   double f1, double f2, double sec_tau,
                                                   double sec_f, double lo, double hi) {
  const double kStepDenomFloor = 1e-300;
  double prop;
  if (alpha <= 1.5) {
    const double denom = 2.0 * f1 * f1 - f * f2;
    prop = fabs(denom) < kStepDenomFloor ? __longlong_as_double(0x7ff8000000000000ll)
                                         : tau - 2.0 * f * f1 / denom;
  } else if (alpha <= 2.0) {
    prop = fabs(f1) < kStepDenomFloor ? __longlong_as_double(0x7ff8000000000000ll)
                                      : tau - f / f1;
  } else {
    const double denom = f - sec_f;
    prop = fabs(denom) < kStepDenomFloor ? __longlong_as_double(0x7ff8000000000000ll)
                                         : tau - f * (tau - sec_tau) / denom;
  }
  if (!isfinite(prop) || prop < lo || prop > hi) return 0.5 * (lo + hi);
  return prop;
}

// RowSolve (reference attention.cpp:212-222): per-row refinement state.
struct RowSolve {
  double tau, lo, hi, f, f1, f2, f_hi, sec_tau, sec_f, best_tau, best_af;
  int steps;
  bool sec_seeded, done;
};

// Post-pass update of one row (reference attention.cpp:284-321).
// Returns true when the row moved (another pass is needed).
__device__ __forceinline__ bool row_step(RowSolve& rs, double alpha, double refine_tol,
                                         int refine_iters, bool need_sec) {
  if (rs.done) return false;
  if (fabs(rs.f) < rs.best_af) {
    rs.best_af = fabs(rs.f);
    rs.best_tau = rs.tau;
  }
  if (rs.f > 0.0)
    rs.lo = rs.tau;
  else
    rs.hi = rs.tau;
  if (fabs(rs.f) <= refine_tol || rs.steps >= refine_iters) {
    rs.done = true;
    if (rs.tau != rs.best_tau) {
      rs.tau = rs.best_tau;
      return true;
    }
    return false;
  }
  if (need_sec && !rs.sec_seeded) {
    rs.sec_tau = rs.hi;
    rs.sec_f = rs.f_hi;
    rs.sec_seeded = true;
  }
  const double prop =
      propose_step_dev(alpha, rs.tau, rs.f, rs.f1, rs.f2, rs.sec_tau, rs.sec_f, rs.lo, rs.hi);
  rs.sec_tau = rs.tau;
  rs.sec_f = rs.f;
  rs.tau = prop;
  ++rs.steps;
  return true;
}

// Launch accounting (exported through adattn_b200_launch_count).
void note_launch();

// Per-row-block active key-block lists and their transpose (csrc/lists.cu).
cudaError_t block_lists(const Geom& g, const uint32_t* mask, int64_t* rowptr, int32_t* cols,
                        int64_t* colptr, int32_t* rows, cudaStream_t st);

// Optional per-kernel event timing (adattn_b200_profile_enable).
void prof_begin(const char* name, cudaStream_t st);
void prof_end(cudaStream_t st);

}  // namespace adattn_b200
