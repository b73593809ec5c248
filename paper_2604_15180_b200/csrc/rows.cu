// rows.cu -- batched row-wise threshold solver on materialised scores
// (the paper's inference variant).
//
// One CTA per row restates, in fp64 with the reference's formulas:
//   center_scores (entmax.cpp:22-57)      -> z, max, visible count
//   build_histogram (histogram.cpp:26-38) -> counts of min(floor(B z), B-1), z >= 0
//   solve_histogram + refine_bracket (histogram.cpp:73-165; common.cuh)
//   hybrid_solve (hybrid.cpp:35-106)      -> straddle check, best-of, tol stop,
//                                            propose_step (internal.hpp:32-55)
//   solve_bisection (entmax.cpp:128-164)  -> method 2
//   entmax_apply (entmax.cpp:166-180)     -> optional probabilities
// Every f evaluation is one pass over the row (z recomputed from the input);
// the three bracket/init evaluations of hybrid_solve share one pass.  Sums are
// fp64 block reductions, so results agree with the sequential reference to
// rounding (~1e-15), not bit for bit.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "adattn_b200.h"
#include "common.cuh"

namespace adattn_b200 {
namespace {

constexpr int kRowThreads = 256;
enum RowErr { RE_NONE = 0, RE_MASKED = 1, RE_NONFINITE = 2, RE_STRADDLE = 3 };


struct RowsArgs {
  adattn_rows_problem p;
  const void* scores;
  const uint8_t* mask;
  double* tau;
  double* residual;
  int32_t* iterations;
  int32_t* converged;
  float* probs;
  double* trace;
  int* err;  // per-call error word (RowsError)
};

__device__ __forceinline__ double load_s(const void* base, size_t i, int dt) {
  return load_elem(base, i, dt);
}

// Block-wide sum of K doubles (all threads get the result).
template <int K>
__device__ __forceinline__ void block_sum(double* v, double* red) {
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) red[warp * K + k] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = 0.0;
    for (int w = 0; w < kRowThreads / 32; ++w) s += red[w * K + k];
    v[k] = s;
  }
}

struct Deriv {
  double f, f1, f2;
};

__global__ void __launch_bounds__(kRowThreads) entmax_rows_kernel(const RowsArgs a) {
  __shared__ double red[kRowThreads / 32 * 9];
  __shared__ uint32_t hist[32];
  const adattn_rows_problem& p = a.p;
  const int64_t row = blockIdx.x;
  const int n = p.n, dt = p.in_dtype;
  const size_t base = (size_t)row * n;
  const double alpha = p.alpha, e0 = 1.0 / (alpha - 1.0), e1 = e0 - 1.0, e2 = e0 - 2.0;
  const double kFloor = 1e-12;  // kDerivBaseFloor (types.hpp)
  auto masked = [&](int j) { return a.mask && a.mask[base + j]; };

  // ---- center_scores: max and visible count; non-finite unmasked -> error
  double mx = -CUDART_INF, vis = 0.0, bad = 0.0;
  for (int j = threadIdx.x; j < n; j += kRowThreads) {
    if (masked(j)) continue;
    const double s = load_s(a.scores, base + j, dt);
    if (!isfinite(s)) bad = 1.0;
    mx = fmax(mx, s);
    vis += 1.0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  {
    __shared__ double smx[kRowThreads / 32];
    if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = -CUDART_INF;
    for (int w = 0; w < kRowThreads / 32; ++w) mx = fmax(mx, smx[w]);
  }
  double cv[2] = {vis, bad};
  block_sum<2>(cv, red);
  const int visible = (int)cv[0];
  if (cv[1] > 0.0 || visible == 0) {
    if (threadIdx.x == 0) atomicMax(a.err, visible == 0 ? RE_MASKED : RE_NONFINITE);
    return;
  }
  auto zval = [&](int j) -> double {  // centred score; masked -> -inf
    if (masked(j)) return -CUDART_INF;
    const double s = load_s(a.scores, base + j, dt);
    return s == mx ? 1.0 : (alpha - 1.0) * (s - mx) + 1.0;
  };
  // f, f', f'' at up to three thresholds in one pass (f_eval, entmax.cpp:59-78)
  auto f_eval3 = [&](int cnt, const double* taus, Deriv* out) {
    double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = threadIdx.x; j < n; j += kRowThreads) {
      const double z = zval(j);
      for (int q = 0; q < cnt; ++q) {
        const double t = z - taus[q];
        if (!(t > 0.0)) continue;
        acc[3 * q] += pow_e(t, e0);
        acc[3 * q + 1] += pow_e(e1 < 0.0 ? fmax(t, kFloor) : t, e1);
        acc[3 * q + 2] += pow_e(e2 < 0.0 ? fmax(t, kFloor) : t, e2);
      }
    }
    block_sum<9>(acc, red);
    for (int q = 0; q < cnt; ++q)
      out[q] = {acc[3 * q] - 1.0, -e0 * acc[3 * q + 1], e0 * (e0 - 1.0) * acc[3 * q + 2]};
  };
  const int tl = p.trace_len;
  double* tr = a.trace ? a.trace + (size_t)row * (tl > 0 ? tl : 0) : nullptr;
  int ntr = 0;
  auto record = [&](double t) {
    if (tr && threadIdx.x == 0 && ntr < tl) tr[ntr] = t;
    ++ntr;
  };

  double tau_final, res_final;
  int iters = 0;
  bool conv = false;
  if (p.method == ADATTN_ROWS_BISECTION) {
    // solve_bisection (entmax.cpp:128-164)
    double lo = 0.0, hi = 1.0 - pow((double)visible, 1.0 - alpha);
    if (hi <= lo) {
      Deriv d;
      const double z0 = 0.0;
      f_eval3(1, &z0, &d);
      tau_final = 0.0;
      res_final = d.f;
      record(0.0);
      iters = 1;
    } else {
      double tau = lo, res = 0.0;
      for (int it = 0; it < p.max_iters; ++it) {
        tau = 0.5 * (lo + hi);
        Deriv d;
        f_eval3(1, &tau, &d);
        res = d.f;
        record(tau);
        ++iters;
        if (fabs(res) <= p.tol) break;
        if (res > 0.0)
          lo = tau;
        else
          hi = tau;
      }
      tau_final = tau;
      res_final = res;
    }
    conv = fabs(res_final) <= p.tol;
  } else {
    double lo, hi, init;
    if (p.method == ADATTN_ROWS_HYBRID) {
      lo = 0.0;
      hi = 1.0 - pow((double)visible, 1.0 - alpha);
      init = 0.5 * (lo + hi);
    } else {
      // build_histogram + solve_histogram + refine_bracket
      if (threadIdx.x < 32) hist[threadIdx.x] = 0u;
      __syncthreads();
      const int B = p.bins;
      for (int j = threadIdx.x; j < n; j += kRowThreads) {
        const double z = zval(j);
        if (!(z >= 0.0)) continue;
        const int k = min((int)(B * z), B - 1);
        atomicAdd(&hist[k], 1u);
      }
      __syncthreads();
      uint32_t c[32];
      for (int k = 0; k < 32; ++k) c[k] = k < B ? hist[k] : 0u;
      solve_histogram_dev(c, B, alpha, init, lo, hi);
    }
    // hybrid_solve (hybrid.cpp:35-106)
    const double taus[3] = {lo, hi, init};
    Deriv d3[3];
    f_eval3(3, taus, d3);
    const double slack = 1e-9;  // kStraddleSlack
    if (d3[0].f < -slack || d3[1].f > slack) {
      if (threadIdx.x == 0) atomicMax(a.err, RE_STRADDLE);
      return;
    }
    double tau = init;
    Deriv d = d3[2];
    double sec_tau = d.f > 0.0 ? hi : lo, sec_f = d.f > 0.0 ? d3[1].f : d3[0].f;
    auto shrink = [&](double t, double fv) {
      if (fv > 0.0)
        lo = t;
      else
        hi = t;
    };
    shrink(tau, d.f);
    record(tau);
    double best_tau = tau, best_af = fabs(d.f), best_res = d.f;
    if (fabs(d.f) <= p.tol) {
      conv = true;
    } else {
      for (int it = 0; it < p.max_iters; ++it) {
        const double prop = propose_step_dev(alpha, tau, d.f, d.f1, d.f2, sec_tau, sec_f, lo, hi);
        sec_tau = tau;
        sec_f = d.f;
        tau = prop;
        f_eval3(1, &tau, &d);
        shrink(tau, d.f);
        record(tau);
        ++iters;
        if (fabs(d.f) < best_af) {
          best_tau = tau;
          best_af = fabs(d.f);
          best_res = d.f;
        }
        if (fabs(d.f) <= p.tol) {
          conv = true;
          break;
        }
      }
    }
    tau_final = best_tau;
    res_final = best_res;
  }
  // carry the last iterate forward (solver_bench's tally, hybrid.cpp:124-130)
  if (tr && threadIdx.x == 0)
    for (int k = ntr; k < tl; ++k) tr[k] = ntr > 0 ? tr[ntr - 1] : tau_final;
  if (threadIdx.x == 0) {
    a.tau[row] = tau_final;
    if (a.residual) a.residual[row] = res_final;
    if (a.iterations) a.iterations[row] = iters;
    if (a.converged) a.converged[row] = conv ? 1 : 0;
  }
  if (a.probs)
    for (int j = threadIdx.x; j < n; j += kRowThreads) {
      const double t = zval(j) - tau_final;
      a.probs[base + j] = t > 0.0 ? (float)pow_e(t, e0) : 0.f;
    }
}

}  // namespace

const char* rows_error_message(int code) {
  switch (code) {
    case RE_MASKED: return "center_scores: every entry is masked";
    case RE_NONFINITE: return "center_scores: non-finite unmasked score";
    case RE_STRADDLE: return "hybrid_solve: bracket does not straddle the root";
    default: return "";
  }
}

cudaError_t entmax_rows(const adattn_rows_problem& p, const void* scores, const uint8_t* mask,
                        double* tau, double* residual, int32_t* iterations, int32_t* converged,
                        float* probs, double* trace, cudaStream_t st, int* row_err) {
  // per-call error word (concurrent calls on different streams do not share it)
  int* err = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&err), sizeof(int), st);
  if (e) return e;
  if ((e = cudaMemsetAsync(err, 0, sizeof(int), st))) return e;
  RowsArgs a{p, scores, mask, tau, residual, iterations, converged, probs, trace, err};
  entmax_rows_kernel<<<(unsigned)p.rows, kRowThreads, 0, st>>>(a);
  note_launch();
  if ((e = cudaGetLastError())) return e;
  if ((e = cudaMemcpyAsync(row_err, err, sizeof(int), cudaMemcpyDeviceToHost, st))) return e;
  if ((e = cudaFreeAsync(err, st))) return e;
  return cudaStreamSynchronize(st);
}

}  // namespace adattn_b200
