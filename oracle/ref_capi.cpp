// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// C entry points over the reference library itself, compiled by
// oracle/Makefile from the reference's own sources under /root/reference
// (nothing copied).  Same signatures as adattn_oracle.h with prefix ref_
// instead of orc_, so tests can run the restatement and the reference on
// identical inputs and compare bit-for-bit.  Output: oracle/_ref/ only.
#include <cstring>
#include <stdexcept>
#include <string>

#include "adattn/attention.hpp"
#include "adattn/entmax.hpp"
#include "adattn/histogram.hpp"
#include "adattn/hybrid.hpp"
#include "adattn/rng.hpp"
#include "adattn/tensor_io.hpp"
#include "adattn_oracle.h"

namespace {

thread_local std::string g_err;

adattn::Matrix to_matrix(const double* src, int rows, int cols) {
  adattn::Matrix m(rows, cols);
  std::memcpy(m.data.data(), src, sizeof(double) * size_t(rows) * cols);
  return m;
}

adattn::AttentionProblem to_problem(const orc_params* p, const double* q, const double* k,
                                    const double* v) {
  adattn::AttentionProblem ap;
  ap.q = to_matrix(q, p->n, p->d);
  ap.k = to_matrix(k, p->m, p->d);
  ap.v = to_matrix(v, p->m, p->dv);
  ap.alpha = p->alpha;
  ap.scale = p->scale;
  ap.causal = p->causal != 0;
  ap.block_r = p->block_r;
  ap.block_c = p->block_c;
  ap.bins = p->bins;
  ap.refine_iters = p->refine_iters;
  ap.refine_tol = p->refine_tol;
  return ap;
}

// Rebuild an AttentionResult (tau, row_max, mask) for backward/compute_delta.
adattn::AttentionResult to_result(const orc_params* p, const double* tau,
                                  const double* row_max, const uint32_t* mask) {
  const int t_r = (p->n + p->block_r - 1) / p->block_r;
  const int t_c = (p->m + p->block_c - 1) / p->block_c;
  const int wpr = (t_c + 31) / 32;
  adattn::AttentionResult res{adattn::Matrix(p->n, p->dv), std::vector<double>(tau, tau + p->n),
                              std::vector<double>(row_max, row_max + p->n),
                              adattn::PackedBlockMask(t_r, t_c), adattn::AttentionStats{}};
  for (int i = 0; i < t_r; ++i)
    for (int j = 0; j < t_c; ++j)
      if ((mask[size_t(i) * wpr + j / 32] >> (j % 32)) & 1u) res.mask.set(i, j);
  return res;
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::overflow_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

void export_result(const adattn::AttentionResult& res, double* out, double* tau,
                   double* row_max, uint32_t* mask, orc_stats* stats) {
  std::memcpy(out, res.out.data.data(), sizeof(double) * res.out.data.size());
  std::memcpy(tau, res.tau.data(), sizeof(double) * res.tau.size());
  std::memcpy(row_max, res.row_max.data(), sizeof(double) * res.row_max.size());
  const auto& w = res.mask.words();
  std::memcpy(mask, w.data(), sizeof(uint32_t) * w.size());
  if (stats) {
    stats->block_sparsity = res.stats.block_sparsity;
    stats->blocks_visited_fwd = res.stats.blocks_visited_fwd;
    stats->blocks_visited_bwd = res.stats.blocks_visited_bwd;
    stats->flushes = res.stats.flushes;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_forward(const orc_params* p, const double* q, const double* k, const double* v,
                int threads, double* out, double* tau, double* row_max, uint32_t* mask,
                int32_t* row_steps, orc_stats* stats) {
  return guarded([&] {
    const adattn::AttentionProblem ap = to_problem(p, q, k, v);
    const adattn::AttentionResult res = adattn::forward(ap, threads);
    export_result(res, out, tau, row_max, mask, stats);
    if (row_steps)
      for (int i = 0; i < p->n; ++i) row_steps[i] = -1;  // not exported by the reference
  });
}

// forward with PhaseTimings (threads<=1 only fills them, attention.cpp:170)
int ref_forward_timed(const orc_params* p, const double* q, const double* k, const double* v,
                      int threads, double* out, double* tau, double* row_max, uint32_t* mask,
                      orc_stats* stats, double* phase_ms) {
  return guarded([&] {
    const adattn::AttentionProblem ap = to_problem(p, q, k, v);
    adattn::PhaseTimings t;
    const adattn::AttentionResult res = adattn::forward(ap, threads, &t);
    export_result(res, out, tau, row_max, mask, stats);
    if (phase_ms)
      for (int i = 0; i < 4; ++i) phase_ms[i] = t.ms[i];
  });
}

int ref_dense_reference(const orc_params* p, const double* q, const double* k,
                        const double* v, double* out, double* tau, double* row_max,
                        uint32_t* mask, orc_stats* stats) {
  return guarded([&] {
    const adattn::AttentionProblem ap = to_problem(p, q, k, v);
    const adattn::AttentionResult res = adattn::dense_reference(ap);
    export_result(res, out, tau, row_max, mask, stats);
  });
}

int ref_compute_delta(const orc_params* p, const double* q, const double* k, const double* v,
                      const double* tau, const double* row_max, const uint32_t* mask,
                      const double* dout, int threads, double* delta) {
  return guarded([&] {
    const adattn::AttentionProblem ap = to_problem(p, q, k, v);
    const adattn::AttentionResult res = to_result(p, tau, row_max, mask);
    const adattn::Matrix dO = to_matrix(dout, p->n, p->dv);
    const std::vector<double> dl = adattn::compute_delta(ap, res, dO, threads);
    std::memcpy(delta, dl.data(), sizeof(double) * dl.size());
  });
}

int ref_backward(const orc_params* p, const double* q, const double* k, const double* v,
                 const double* tau, const double* row_max, const uint32_t* mask,
                 const double* dout, int threads, double* dq, double* dk, double* dv,
                 double* delta, uint64_t* visited_bwd) {
  return guarded([&] {
    const adattn::AttentionProblem ap = to_problem(p, q, k, v);
    adattn::AttentionResult res = to_result(p, tau, row_max, mask);
    const adattn::Matrix dO = to_matrix(dout, p->n, p->dv);
    const adattn::AttentionGradients g = adattn::backward(ap, res, dO, threads);
    std::memcpy(dq, g.dq.data.data(), sizeof(double) * g.dq.data.size());
    std::memcpy(dk, g.dk.data.data(), sizeof(double) * g.dk.data.size());
    std::memcpy(dv, g.dv.data.data(), sizeof(double) * g.dv.data.size());
    std::memcpy(delta, g.delta.data(), sizeof(double) * g.delta.size());
    if (visited_bwd) *visited_bwd = res.stats.blocks_visited_bwd;
  });
}

double ref_block_sparsity(const uint32_t* mask, int t_r, int t_c, int causal) {
  adattn::PackedBlockMask m(t_r, t_c);
  const int wpr = (t_c + 31) / 32;
  for (int i = 0; i < t_r; ++i)
    for (int j = 0; j < t_c; ++j)
      if ((mask[size_t(i) * wpr + j / 32] >> (j % 32)) & 1u) m.set(i, j);
  return adattn::block_sparsity(m, causal != 0);
}

int ref_solve_histogram(const uint32_t* counts, int bins, double alpha, double* tau_h,
                        int* bracket_floor, double* lo, double* hi) {
  return guarded([&] {
    adattn::Histogram h;
    h.bins = bins;
    h.width = 1.0 / bins;
    h.counts.assign(counts, counts + bins);
    const adattn::HistogramSolution s = adattn::solve_histogram(h, alpha);
    const auto [l, u] = adattn::refine_bracket(s);
    if (tau_h) *tau_h = s.tau_h;
    if (bracket_floor) *bracket_floor = s.bracket_floor;
    if (lo) *lo = l;
    if (hi) *hi = u;
  });
}

void ref_f_eval(const double* z, int n, double alpha, double tau, double* f, double* f1,
                double* f2) {
  adattn::CenteredScores cs;
  cs.z.assign(z, z + n);
  cs.alpha = alpha;
  cs.visible_n = n;
  const adattn::FDerivatives d = adattn::f_eval(cs, tau);
  *f = d.f;
  *f1 = d.f1;
  *f2 = d.f2;
}

void ref_gaussian_fill(uint64_t seed, double scale, double* out, size_t count) {
  adattn::Xoshiro256pp rng(seed);
  for (size_t i = 0; i < count; ++i) out[i] = scale * rng.gaussian();
}

void ref_xoshiro_next(uint64_t seed, uint64_t* out, size_t count) {
  adattn::Xoshiro256pp rng(seed);
  for (size_t i = 0; i < count; ++i) out[i] = rng.next();
}

// hybrid_solve replay (hybrid.cpp:35-106) for the per-row step count the
// reference keeps private (RowSolve.steps, attention.cpp:219).
int ref_hybrid_steps(const double* z, int n, double alpha, double init, double lo, double hi,
                     double tol, int max_iters, double* final_tau) {
  int steps = -1;
  guarded([&] {
    adattn::CenteredScores cs;
    cs.z.assign(z, z + n);
    cs.alpha = alpha;
    cs.visible_n = n;
    const adattn::SolverTrace t = adattn::hybrid_solve(cs, init, lo, hi, {alpha, tol, max_iters});
    steps = int(t.iterations.size()) - 1;
    if (final_tau) *final_tau = t.final_tau;
  });
  return steps;
}

// The reference's ATN1 tensor I/O (tensor_io.cpp:39-112), for byte-level
// comparison with the product's csrc/io.cu.  Returns 0, or 1 with the
// exception message in ref_last_error().
int ref_save_tensor(const char* path, int dtype, int rank, const uint32_t* dims,
                    const double* values) {
  return guarded([&] {
    adattn::Tensor t;
    t.dtype = adattn::Dtype(dtype);
    t.dims.assign(dims, dims + rank);
    t.values.assign(values, values + t.count());
    adattn::save_tensor(t, path);
  });
}

int ref_load_tensor(const char* path, int* dtype, int* rank, uint32_t* dims, double* values,
                    size_t capacity, size_t* count) {
  return guarded([&] {
    const adattn::Tensor t = adattn::load_tensor(path);
    *dtype = int(t.dtype);
    *rank = int(t.dims.size());
    for (size_t i = 0; i < t.dims.size(); ++i) dims[i] = t.dims[i];
    *count = t.values.size();
    if (values && capacity >= t.values.size())
      std::memcpy(values, t.values.data(), t.values.size() * sizeof(double));
  });
}

}  // extern "C"
