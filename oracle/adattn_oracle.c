/*
 * adattn_oracle.c -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the
 * reference's tiled alpha-entmax attention, written in plain C from the
 * reference's behaviour (file:line cited per function).  Every floating-point
 * expression keeps the reference's operation order so that, compiled with
 * -ffp-contract=off like oracle/_ref, results are bit-identical to the
 * reference; tests/test_oracle.py asserts exactly that.
 *
 * Not linked into, loaded by, or called from the product path.
 */
#include "adattn_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_INVALID 1
#define ORC_OVERFLOW 2
#define ORC_OTHER 3

static _Thread_local char g_err[256];

const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* kMaskSlack, kDerivBaseFloor (attention.cpp:25-27), kStepDenomFloor (internal.hpp:21) */
static const double kMaskSlack = 1e-9;
static const double kDerivBaseFloor = 1e-12;
static const double kStepDenomFloor = 1e-300;

/* pow_e (internal.hpp:13-19) */
static inline double pow_e(double base, double e) {
  if (e == 1.0) return base;
  if (e == 2.0) return base * base;
  if (e == 0.0) return 1.0;
  if (e == 0.5) return sqrt(base);
  return pow(base, e);
}

static inline double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */
static inline double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */

/* dot (attention.cpp:29-33): sequential, x ascending */
static inline double dot(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int x = 0; x < d; ++x) s += a[x] * b[x];
  return s;
}

/* ---------------------------------------------------------------- geometry */

typedef struct {
  int n, m, d, dv, t_r, t_c, wpr;
  double scale;
} geom_t;

/* validate (attention.cpp:42-63), same checks and messages. */
static int validate(const orc_params* p, geom_t* g) {
  g->n = p->n;
  g->m = p->m;
  g->d = p->d;
  g->dv = p->dv;
  if (g->n < 1 || g->m < 1 || g->d < 1 || g->dv < 1)
    return fail(ORC_INVALID, "attention: empty operand");
  if (p->causal && g->m != g->n)
    return fail(ORC_INVALID, "attention: causal needs square score matrix");
  if (!(p->alpha > 1.0)) return fail(ORC_INVALID, "attention: alpha must exceed 1");
  if (p->block_r < 1 || p->block_c < 1) return fail(ORC_INVALID, "attention: bad tile size");
  if (p->refine_iters < 0 || !(p->refine_tol > 0.0))
    return fail(ORC_INVALID, "attention: bad refinement config");
  g->t_r = (g->n + p->block_r - 1) / p->block_r;
  g->t_c = (g->m + p->block_c - 1) / p->block_c;
  g->wpr = (g->t_c + 31) / 32;
  g->scale = p->scale != 0.0 ? p->scale : 1.0 / sqrt((double)g->d);
  return 0;
}

/* PackedHistogramAcc ctor checks (bitpack.cpp:55-65) with word_bits_for
 * (attention.cpp:35).  Returns bits per bin or 0 on error. */
static int bits_per_bin_for(int bins) {
  const int word_bits = bins <= 16 ? 64 : 128;
  if (bins <= 0 || word_bits % bins != 0) {
    fail(ORC_INVALID, "PackedHistogramAcc: bins must divide word_bits");
    return 0;
  }
  const int b = word_bits / bins;
  if (b < 4) {
    fail(ORC_INVALID, "PackedHistogramAcc: needs at least 4 bits per bin");
    return 0;
  }
  return b;
}

/* compute_z_block (attention.cpp:68-84) */
static void compute_z_block(const orc_params* p, const geom_t* g, const double* q,
                            const double* k, const double* row_max, int r0, int nr, int c0,
                            int nc, double* buf) {
  for (int r = 0; r < nr; ++r) {
    const double* qrow = q + (size_t)(r0 + r) * g->d;
    const double m = row_max[r0 + r];
    double* dst = buf + (size_t)r * nc;
    for (int c = 0; c < nc; ++c) {
      if (p->causal && c0 + c > r0 + r) {
        dst[c] = -INFINITY;
        continue;
      }
      const double s = g->scale * dot(qrow, k + (size_t)(c0 + c) * g->d, g->d);
      dst[c] = s == m ? 1.0 : (p->alpha - 1.0) * (s - m) + 1.0;
    }
  }
}

/* ------------------------------------------------------------ parallel_for */
/* parallel_for (attention.cpp:86-100): atomic work counter over `count` tasks. */
typedef void (*task_fn)(void* ctx, int i);
typedef struct {
  task_fn fn;
  void* ctx;
  int count;
  atomic_int next;
} pool_t;

static void* pool_worker(void* arg) {
  pool_t* pl = (pool_t*)arg;
  for (int i; (i = atomic_fetch_add(&pl->next, 1)) < pl->count;) pl->fn(pl->ctx, i);
  return NULL;
}

static void parallel_for(int count, int threads, task_fn fn, void* ctx) {
  if (threads > count) threads = count;
  if (threads <= 1) {
    for (int i = 0; i < count; ++i) fn(ctx, i);
    return;
  }
  pool_t pl;
  pl.fn = fn;
  pl.ctx = ctx;
  pl.count = count;
  atomic_init(&pl.next, 0);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, pool_worker, &pl);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
}

/* -------------------------------------------------------------- histogram */

/* f_h_eval, left edge (histogram.cpp:40-50) */
static double f_h_eval(const uint32_t* counts, int bins, double width, double tau,
                       double alpha) {
  const double e0 = 1.0 / (alpha - 1.0);
  double sum = 0.0;
  for (int k = 0; k < bins; ++k) {
    if (counts[k] == 0) continue;
    const double t = (k + 0.0) * width - tau;
    if (t > 0.0) sum += (double)counts[k] * pow_e(t, e0);
  }
  return sum - 1.0;
}

/* bisect_f_h (histogram.cpp:57-69) */
static double bisect_f_h(const uint32_t* counts, int bins, double width, double alpha,
                         double lo, double hi) {
  for (int it = 0; it < 200 && hi - lo > 1e-10; ++it) {
    const double mid = 0.5 * (lo + hi);
    const double v = f_h_eval(counts, bins, width, mid, alpha);
    if (v == 0.0) return mid;
    if (v > 0.0)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

/* solve_histogram, kLeftEdge (histogram.cpp:73-161) + refine_bracket (163-165) */
int orc_solve_histogram(const uint32_t* counts, int bins, double alpha, double* tau_h,
                        int* bracket_floor, double* lo_out, double* hi_out) {
  if (!(alpha > 1.0)) return fail(ORC_INVALID, "solve_histogram: alpha must exceed 1");
  uint64_t total = 0;
  for (int k = 0; k < bins; ++k) total += counts[k];
  if (total == 0) return fail(ORC_INVALID, "solve_histogram: empty histogram");
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
      fh = f_h_eval(counts, bins, w, tau, alpha);
    if (fh >= 0.0) {
      floor_k = k;
      break;
    }
    const double v = k * w;
    s0 += counts[k];
    s1 += counts[k] * v;
    s2 += counts[k] * v * v;
  }
  double th;
  int fk;
  if (floor_k < 0) {
    th = 0.0;
    fk = 0;
  } else {
    fk = floor_k;
    const double lo = floor_k * w;
    const double hi = (floor_k + 1) * w;
    double tau;
    if (e0 == 1.0) {
      tau = (s1 - 1.0) / s0;
    } else if (e0 == 2.0) {
      const double disc = dmax(s1 * s1 - s0 * (s2 - 1.0), 0.0);
      tau = (s1 - sqrt(disc)) / s0;
    } else {
      tau = bisect_f_h(counts, bins, w, alpha, lo, hi);
    }
    /* std::clamp(tau, lo, nextafter(hi, lo)) */
    const double top = nextafter(hi, lo);
    th = tau < lo ? lo : (top < tau ? top : tau);
  }
  if (tau_h) *tau_h = th;
  if (bracket_floor) *bracket_floor = fk;
  if (lo_out) *lo_out = th;
  if (hi_out) *hi_out = th + w;
  return 0;
}

/* propose_step (internal.hpp:32-55) */
double orc_propose_step(double alpha, double tau, double f, double f1, double f2,
                        double sec_tau, double sec_f, double lo, double hi, int* kind) {
  double prop;
  int k;
  if (alpha <= 1.5) {
    k = 1;
    const double denom = 2.0 * f1 * f1 - f * f2;
    prop = fabs(denom) < kStepDenomFloor ? NAN : tau - 2.0 * f * f1 / denom;
  } else if (alpha <= 2.0) {
    k = 2;
    prop = fabs(f1) < kStepDenomFloor ? NAN : tau - f / f1;
  } else {
    k = 3;
    const double denom = f - sec_f;
    prop = fabs(denom) < kStepDenomFloor ? NAN : tau - f * (tau - sec_tau) / denom;
  }
  if (!isfinite(prop) || prop < lo || prop > hi) {
    if (kind) *kind = 4;
    return 0.5 * (lo + hi);
  }
  if (kind) *kind = k;
  return prop;
}

/* f_eval (entmax.cpp:59-78) */
void orc_f_eval(const double* z, int n, double alpha, double tau, double* f, double* f1,
                double* f2) {
  const double e0 = 1.0 / (alpha - 1.0);
  const double e1 = e0 - 1.0;
  const double e2 = e0 - 2.0;
  double sum0 = 0.0, sum1 = 0.0, sum2 = 0.0;
  for (int i = 0; i < n; ++i) {
    const double t = z[i] - tau;
    if (!(t > 0.0)) continue;
    sum0 += pow_e(t, e0);
    const double t1 = e1 < 0.0 ? dmax(t, kDerivBaseFloor) : t;
    sum1 += pow_e(t1, e1);
    const double t2 = e2 < 0.0 ? dmax(t, kDerivBaseFloor) : t;
    sum2 += pow_e(t2, e2);
  }
  *f = sum0 - 1.0;
  *f1 = -e0 * sum1;
  *f2 = e0 * (e0 - 1.0) * sum2;
}

/* ------------------------------------------------------------------ masks */

static inline void mask_set(uint32_t* mask, int wpr, int i, int j) {
  mask[(size_t)i * wpr + j / 32] |= (uint32_t)1 << (j % 32);
}
static inline int mask_test(const uint32_t* mask, int wpr, int i, int j) {
  return (int)((mask[(size_t)i * wpr + j / 32] >> (j % 32)) & 1u);
}

/* block_sparsity (attention.cpp:541-551) */
double orc_block_sparsity(const uint32_t* mask, int t_r, int t_c, int causal) {
  const int wpr = (t_c + 31) / 32;
  int64_t addressable = 0, active = 0;
  for (int i = 0; i < t_r; ++i)
    for (int j = 0; j < t_c; ++j) {
      if (causal && (int64_t)j * t_r >= (int64_t)(i + 1) * t_c) continue;
      ++addressable;
      if (mask_test(mask, wpr, i, j)) ++active;
    }
  return addressable == 0 ? 0.0 : (double)(addressable - active) / (double)addressable;
}

static uint64_t mask_popcount(const uint32_t* mask, size_t words) {
  uint64_t pc = 0;
  for (size_t i = 0; i < words; ++i) pc += (uint64_t)__builtin_popcount(mask[i]);
  return pc;
}

/* ---------------------------------------------------------------- forward */

typedef struct {
  double tau, lo, hi, f, f1, f2, f_hi, sec_tau, sec_f, best_tau, best_af;
  int sec_seeded, steps, done;
} row_solve_t; /* RowSolve (attention.cpp:212-222) */

typedef struct {
  const orc_params* p;
  const geom_t* g;
  const double *q, *k, *v;
  double *out, *tau, *row_max;
  uint32_t* mask;
  int32_t* row_steps;
  double* tau_h;        /* nullable: per-row solve_histogram result */
  uint32_t* counts_out; /* nullable: per-row histogram counts [n][bins] */
  int flush_limit_log2; /* bits per bin */
  atomic_ullong flushes;
} fwd_ctx;

static void forward_tile(void* vctx, int it) {
  fwd_ctx* C = (fwd_ctx*)vctx;
  const orc_params* p = C->p;
  const geom_t* g = C->g;
  const int r0 = it * p->block_r;
  const int r1 = (g->n < r0 + p->block_r) ? g->n : r0 + p->block_r;
  const int nr = r1 - r0;
  const int jlim = p->causal ? (r1 - 1) / p->block_c : g->t_c - 1;
  const int bins = p->bins;
  const double e0 = 1.0 / (p->alpha - 1.0);
  const double e1 = e0 - 1.0;
  const double e2 = e0 - 2.0;
  double* zbuf = (double*)malloc(sizeof(double) * (size_t)nr * p->block_c);

  /* Phase 1: row maxima (attention.cpp:182-195) */
  for (int r = 0; r < nr; ++r) C->row_max[r0 + r] = -INFINITY;
  for (int jt = 0; jt <= jlim; ++jt) {
    const int c0 = jt * p->block_c;
    const int c1 = (g->m < c0 + p->block_c) ? g->m : c0 + p->block_c;
    for (int r = 0; r < nr; ++r) {
      const double* qrow = C->q + (size_t)(r0 + r) * g->d;
      const int cend = p->causal ? ((c1 < r0 + r + 1) ? c1 : r0 + r + 1) : c1;
      double m = C->row_max[r0 + r];
      for (int c = c0; c < cend; ++c)
        m = dmax(m, g->scale * dot(qrow, C->k + (size_t)c * g->d, g->d));
      C->row_max[r0 + r] = m;
    }
  }

  /* Phase 2: histogram counts (TileHistogramStream, attention.cpp:110-155,
   * 201-210).  The packed per-position accumulators receive at most one count
   * per tile and drain every 2^b-1 tiles, so their totals equal plain counts;
   * only the flush events are bookkeeping. */
  uint32_t* counts = (uint32_t*)calloc((size_t)nr * bins, sizeof(uint32_t));
  for (int jt = 0; jt <= jlim; ++jt) {
    const int c0 = jt * p->block_c;
    const int nc = ((g->m < c0 + p->block_c) ? g->m : c0 + p->block_c) - c0;
    compute_z_block(p, g, C->q, C->k, C->row_max, r0, nr, c0, nc, zbuf);
    for (int r = 0; r < nr; ++r)
      for (int c = 0; c < nc; ++c) {
        const double z = zbuf[(size_t)r * nc + c];
        if (!(z >= 0.0)) continue;
        const int b = (int)(bins * z);
        counts[(size_t)r * bins + (b < bins - 1 ? b : bins - 1)]++;
      }
  }
  {
    const int J = jlim + 1;
    const unsigned long long L =
        C->flush_limit_log2 >= 64 ? ~0ull : ((1ull << C->flush_limit_log2) - 1ull);
    atomic_fetch_add(&C->flushes, (unsigned long long)((J + L - 1) / L));
  }

  if (C->counts_out)
    memcpy(C->counts_out + (size_t)r0 * bins, counts, sizeof(uint32_t) * (size_t)nr * bins);
  row_solve_t* rows = (row_solve_t*)calloc((size_t)nr, sizeof(row_solve_t));
  for (int r = 0; r < nr; ++r) {
    double lo, hi, th;
    orc_solve_histogram(counts + (size_t)r * bins, bins, p->alpha, &th, NULL, &lo, &hi);
    if (C->tau_h) C->tau_h[r0 + r] = th;
    rows[r].tau = th;
    rows[r].lo = lo;
    rows[r].hi = hi;
    rows[r].best_af = INFINITY;
  }
  free(counts);

  /* Phase 3: streaming refinement (attention.cpp:234-332) */
  const int need_sec = p->alpha > 2.0;
  uint8_t* blk_active = (uint8_t*)calloc((size_t)jlim + 1, 1);
  int first_pass = 1;
  for (;;) {
    for (int r = 0; r < nr; ++r) {
      rows[r].f = -1.0;
      rows[r].f1 = 0.0;
      rows[r].f2 = 0.0;
      if (first_pass) rows[r].f_hi = -1.0;
    }
    memset(blk_active, 0, (size_t)jlim + 1);
    for (int jt = 0; jt <= jlim; ++jt) {
      const int c0 = jt * p->block_c;
      const int nc = ((g->m < c0 + p->block_c) ? g->m : c0 + p->block_c) - c0;
      compute_z_block(p, g, C->q, C->k, C->row_max, r0, nr, c0, nc, zbuf);
      uint8_t any = 0;
      for (int r = 0; r < nr; ++r) {
        row_solve_t* rs = &rows[r];
        const double* zr = zbuf + (size_t)r * nc;
        if (rs->done) {
          for (int c = 0; c < nc; ++c) any |= (uint8_t)(zr[c] > rs->tau - kMaskSlack);
          continue;
        }
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, shi = 0.0;
        for (int c = 0; c < nc; ++c) {
          const double t = zr[c] - rs->tau;
          any |= (uint8_t)(t > -kMaskSlack);
          if (t > 0.0) {
            s0 += pow_e(t, e0);
            s1 += pow_e(e1 < 0.0 ? dmax(t, kDerivBaseFloor) : t, e1);
            s2 += pow_e(e2 < 0.0 ? dmax(t, kDerivBaseFloor) : t, e2);
          }
          if (first_pass && need_sec) {
            const double th = zr[c] - rs->hi;
            if (th > 0.0) shi += pow_e(th, e0);
          }
        }
        rs->f += s0;
        rs->f1 -= e0 * s1;
        rs->f2 += e0 * (e0 - 1.0) * s2;
        if (first_pass && need_sec) rs->f_hi += shi;
      }
      blk_active[jt] = any;
    }

    int stepped = 0;
    for (int r = 0; r < nr; ++r) {
      row_solve_t* rs = &rows[r];
      if (rs->done) continue;
      if (fabs(rs->f) < rs->best_af) {
        rs->best_af = fabs(rs->f);
        rs->best_tau = rs->tau;
      }
      if (rs->f > 0.0)
        rs->lo = rs->tau;
      else
        rs->hi = rs->tau;
      if (fabs(rs->f) <= p->refine_tol || rs->steps >= p->refine_iters) {
        rs->done = 1;
        if (rs->tau != rs->best_tau) {
          rs->tau = rs->best_tau;
          stepped = 1;
        }
        continue;
      }
      if (need_sec && !rs->sec_seeded) {
        rs->sec_tau = rs->hi;
        rs->sec_f = rs->f_hi;
        rs->sec_seeded = 1;
      }
      const double prop = orc_propose_step(p->alpha, rs->tau, rs->f, rs->f1, rs->f2,
                                           rs->sec_tau, rs->sec_f, rs->lo, rs->hi, NULL);
      rs->sec_tau = rs->tau;
      rs->sec_f = rs->f;
      rs->tau = prop;
      ++rs->steps;
      stepped = 1;
    }
    first_pass = 0;
    if (!stepped) break;
  }
  for (int r = 0; r < nr; ++r) {
    C->tau[r0 + r] = rows[r].tau;
    if (C->row_steps) C->row_steps[r0 + r] = rows[r].steps;
  }
  for (int jt = 0; jt <= jlim; ++jt)
    if (blk_active[jt]) mask_set(C->mask, g->wpr, it, jt);

  /* Phase 4: output over the set mask bits, ascending (attention.cpp:334-352) */
  for (int jt = 0; jt < g->t_c; ++jt) {
    if (!mask_test(C->mask, g->wpr, it, jt)) continue;
    const int c0 = jt * p->block_c;
    const int nc = ((g->m < c0 + p->block_c) ? g->m : c0 + p->block_c) - c0;
    compute_z_block(p, g, C->q, C->k, C->row_max, r0, nr, c0, nc, zbuf);
    for (int r = 0; r < nr; ++r) {
      const double* zr = zbuf + (size_t)r * nc;
      double* orow = C->out + (size_t)(r0 + r) * g->dv;
      for (int c = 0; c < nc; ++c) {
        const double t = zr[c] - C->tau[r0 + r];
        if (t <= 0.0) continue;
        const double pv = pow_e(t, e0);
        const double* vrow = C->v + (size_t)(c0 + c) * g->dv;
        for (int x = 0; x < g->dv; ++x) orow[x] += pv * vrow[x];
      }
    }
  }
  free(blk_active);
  free(rows);
  free(zbuf);
}

int orc_forward(const orc_params* p, const double* q, const double* k, const double* v,
                int threads, double* out, double* tau, double* row_max, uint32_t* mask,
                int32_t* row_steps, orc_stats* stats) {
  return orc_forward_ex(p, q, k, v, threads, out, tau, row_max, mask, row_steps, stats, NULL,
                        NULL);
}

int orc_forward_ex(const orc_params* p, const double* q, const double* k, const double* v,
                   int threads, double* out, double* tau, double* row_max, uint32_t* mask,
                   int32_t* row_steps, orc_stats* stats, double* tau_h, uint32_t* counts) {
  geom_t g;
  int rc = validate(p, &g);
  if (rc) return rc;
  const int bpb = bits_per_bin_for(p->bins);
  if (!bpb) return ORC_INVALID;
  memset(out, 0, sizeof(double) * (size_t)g.n * g.dv);
  memset(mask, 0, sizeof(uint32_t) * (size_t)g.t_r * g.wpr);
  fwd_ctx C;
  C.p = p;
  C.g = &g;
  C.q = q;
  C.k = k;
  C.v = v;
  C.out = out;
  C.tau = tau;
  C.row_max = row_max;
  C.mask = mask;
  C.row_steps = row_steps;
  C.tau_h = tau_h;
  C.counts_out = counts;
  C.flush_limit_log2 = bpb;
  atomic_init(&C.flushes, 0);
  parallel_for(g.t_r, threads, forward_tile, &C);
  if (stats) {
    stats->blocks_visited_fwd = mask_popcount(mask, (size_t)g.t_r * g.wpr);
    stats->blocks_visited_bwd = 0;
    stats->flushes = atomic_load(&C.flushes);
    stats->block_sparsity = orc_block_sparsity(mask, g.t_r, g.t_c, p->causal);
  }
  return 0;
}

/* -------------------------------------------------------- dense reference */

/* solve_exact (entmax.cpp:80-126) on descending-sorted visible z */
static int cmp_desc(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) ? -1 : (x < y) ? 1 : 0;
}

static double solve_exact_sorted(const double* sorted, int n, double alpha) {
  double tau = 0.0;
  if (alpha == 2.0) {
    double cumsum = 0.0;
    for (int k = 1; k <= n; ++k) {
      cumsum += sorted[k - 1];
      const double cand = (cumsum - 1.0) / k;
      if (k == n || sorted[k] <= cand) {
        tau = cand;
        break;
      }
    }
  } else {
    double s1 = 0.0, s2 = 0.0;
    for (int k = 1; k <= n; ++k) {
      s1 += sorted[k - 1];
      s2 += sorted[k - 1] * sorted[k - 1];
      const double mean = s1 / k;
      const double disc = dmax(1.0 / k - (s2 / k - mean * mean), 0.0);
      const double cand = mean - sqrt(disc);
      if (k == n || sorted[k] <= cand) {
        tau = cand;
        break;
      }
    }
  }
  return tau;
}

/* solve_bisection (entmax.cpp:128-164), tol 1e-14, 200 iterations */
static double solve_bisection(const double* z, int n, int visible, double alpha) {
  double lo = 0.0;
  double hi = 1.0 - pow((double)visible, 1.0 - alpha);
  if (hi <= lo) return 0.0;
  double tau = lo;
  for (int it = 0; it < 200; ++it) {
    tau = 0.5 * (lo + hi);
    double f, f1, f2;
    orc_f_eval(z, n, alpha, tau, &f, &f1, &f2);
    if (fabs(f) <= 1e-14) break;
    if (f > 0.0)
      lo = tau;
    else
      hi = tau;
  }
  return tau;
}

int orc_dense_reference(const orc_params* p, const double* q, const double* k,
                        const double* v, double* out, double* tau, double* row_max,
                        uint32_t* mask, orc_stats* stats) {
  geom_t g;
  int rc = validate(p, &g);
  if (rc) return rc;
  if (g.n > 4096 || g.m > 4096)
    return fail(ORC_INVALID, "dense_reference: capped at 4096 rows");
  memset(out, 0, sizeof(double) * (size_t)g.n * g.dv);
  memset(mask, 0, sizeof(uint32_t) * (size_t)g.t_r * g.wpr);
  double* s = (double*)malloc(sizeof(double) * (size_t)g.m);
  double* z = (double*)malloc(sizeof(double) * (size_t)g.m);
  double* sorted = (double*)malloc(sizeof(double) * (size_t)g.m);
  const double e0 = 1.0 / (p->alpha - 1.0);
  for (int i = 0; i < g.n; ++i) {
    double m = -INFINITY;
    for (int j = 0; j < g.m; ++j) {
      s[j] = g.scale * dot(q + (size_t)i * g.d, k + (size_t)j * g.d, g.d);
      if (!p->causal || j <= i) m = dmax(m, s[j]);
    }
    row_max[i] = m;
    /* center_scores (entmax.cpp:22-57) */
    int visible = 0, ns = 0;
    for (int j = 0; j < g.m; ++j) {
      if (p->causal && j > i) {
        z[j] = -INFINITY;
        continue;
      }
      ++visible;
      z[j] = s[j] == m ? 1.0 : (p->alpha - 1.0) * (s[j] - m) + 1.0;
      sorted[ns++] = z[j];
    }
    double t;
    if (p->alpha == 1.5 || p->alpha == 2.0) {
      /* std::stable_sort descending; equal keys are interchangeable values */
      qsort(sorted, (size_t)ns, sizeof(double), cmp_desc);
      t = solve_exact_sorted(sorted, ns, p->alpha);
    } else {
      t = solve_bisection(z, g.m, visible, p->alpha);
    }
    tau[i] = t;
    /* entmax_apply (entmax.cpp:166-180) then O row over the support */
    double* orow = out + (size_t)i * g.dv;
    for (int j = 0; j < g.m; ++j) {
      const double tt = z[j] - t;
      if (!(tt > 0.0)) continue;
      const double pj = pow_e(tt, e0);
      const double* vrow = v + (size_t)j * g.dv;
      for (int x = 0; x < g.dv; ++x) orow[x] += pj * vrow[x];
      mask_set(mask, g.wpr, i / p->block_r, j / p->block_c);
    }
  }
  free(s);
  free(z);
  free(sorted);
  if (stats) {
    memset(stats, 0, sizeof *stats);
    stats->block_sparsity = orc_block_sparsity(mask, g.t_r, g.t_c, p->causal);
  }
  return 0;
}

/* ---------------------------------------------------------- compute_delta */

typedef struct {
  const orc_params* p;
  const geom_t* g;
  const double *q, *k, *v, *tau, *row_max, *dout;
  const uint32_t* mask;
  double* delta;
} delta_ctx;

static void delta_tile(void* vctx, int it) {
  delta_ctx* C = (delta_ctx*)vctx;
  const orc_params* p = C->p;
  const geom_t* g = C->g;
  const double e0 = 1.0 / (p->alpha - 1.0);
  const int r0 = it * p->block_r;
  const int nr = ((g->n < r0 + p->block_r) ? g->n : r0 + p->block_r) - r0;
  double* zbuf = (double*)malloc(sizeof(double) * (size_t)nr * p->block_c);
  double* num = (double*)calloc((size_t)nr, sizeof(double));
  double* den = (double*)calloc((size_t)nr, sizeof(double));
  for (int jt = 0; jt < g->t_c; ++jt) {
    if (!mask_test(C->mask, g->wpr, it, jt)) continue;
    const int c0 = jt * p->block_c;
    const int nc = ((g->m < c0 + p->block_c) ? g->m : c0 + p->block_c) - c0;
    compute_z_block(p, g, C->q, C->k, C->row_max, r0, nr, c0, nc, zbuf);
    for (int r = 0; r < nr; ++r) {
      const double* zr = zbuf + (size_t)r * nc;
      const double* dorow = C->dout + (size_t)(r0 + r) * g->dv;
      for (int c = 0; c < nc; ++c) {
        const double t = zr[c] - C->tau[r0 + r];
        if (t <= 0.0) continue;
        const double pv = pow_e(t, e0);
        const double u = pow_e(pv, 2.0 - p->alpha);
        num[r] += u * dot(dorow, C->v + (size_t)(c0 + c) * g->dv, g->dv);
        den[r] += u;
      }
    }
  }
  for (int r = 0; r < nr; ++r) C->delta[r0 + r] = den[r] > 0.0 ? num[r] / den[r] : 0.0;
  free(zbuf);
  free(num);
  free(den);
}

int orc_compute_delta(const orc_params* p, const double* q, const double* k,
                      const double* v, const double* tau, const double* row_max,
                      const uint32_t* mask, const double* dout, int threads,
                      double* delta) {
  geom_t g;
  int rc = validate(p, &g);
  if (rc) return rc;
  delta_ctx C = {p, &g, q, k, v, tau, row_max, dout, mask, delta};
  parallel_for(g.t_r, threads, delta_tile, &C);
  return 0;
}

/* --------------------------------------------------------------- backward */

typedef struct {
  const orc_params* p;
  const geom_t* g;
  const double *q, *k, *v, *tau, *row_max, *dout, *delta;
  const uint32_t *mask, *tmask;
  int twpr;
  double *dq, *dk, *dv;
  atomic_ullong visited;
} bwd_ctx;

/* key-major sweep (attention.cpp:464-506) */
static void bwd_key_tile(void* vctx, int jt) {
  bwd_ctx* C = (bwd_ctx*)vctx;
  const orc_params* p = C->p;
  const geom_t* g = C->g;
  const double e0 = 1.0 / (p->alpha - 1.0);
  const int c0 = jt * p->block_c;
  const int nc = ((g->m < c0 + p->block_c) ? g->m : c0 + p->block_c) - c0;
  double* zbuf = (double*)malloc(sizeof(double) * (size_t)p->block_r * nc);
  double* ds = (double*)malloc(sizeof(double) * (size_t)nc);
  double* pv = (double*)malloc(sizeof(double) * (size_t)nc);
  for (int it = 0; it < g->t_r; ++it) {
    if (!mask_test(C->tmask, C->twpr, jt, it)) continue;
    const int r0 = it * p->block_r;
    const int nr = ((g->n < r0 + p->block_r) ? g->n : r0 + p->block_r) - r0;
    compute_z_block(p, g, C->q, C->k, C->row_max, r0, nr, c0, nc, zbuf);
    for (int r = 0; r < nr; ++r) {
      const double* zr = zbuf + (size_t)r * nc;
      const double* dorow = C->dout + (size_t)(r0 + r) * g->dv;
      const double* qrow = C->q + (size_t)(r0 + r) * g->d;
      const double dl = C->delta[r0 + r];
      for (int c = 0; c < nc; ++c) {
        const double t = zr[c] - C->tau[r0 + r];
        if (t <= 0.0) {
          pv[c] = 0.0;
          ds[c] = 0.0;
          continue;
        }
        pv[c] = pow_e(t, e0);
        const double u = pow_e(pv[c], 2.0 - p->alpha);
        const double dp = dot(dorow, C->v + (size_t)(c0 + c) * g->dv, g->dv);
        ds[c] = u * (dp - dl);
      }
      for (int c = 0; c < nc; ++c) {
        if (pv[c] != 0.0) {
          double* dvrow = C->dv + (size_t)(c0 + c) * g->dv;
          for (int x = 0; x < g->dv; ++x) dvrow[x] += pv[c] * dorow[x];
        }
        if (ds[c] != 0.0) {
          double* dkrow = C->dk + (size_t)(c0 + c) * g->d;
          const double w = g->scale * ds[c];
          for (int x = 0; x < g->d; ++x) dkrow[x] += w * qrow[x];
        }
      }
    }
    atomic_fetch_add(&C->visited, 1ull);
  }
  free(zbuf);
  free(ds);
  free(pv);
}

/* query-major sweep (attention.cpp:508-535) */
static void bwd_query_tile(void* vctx, int it) {
  bwd_ctx* C = (bwd_ctx*)vctx;
  const orc_params* p = C->p;
  const geom_t* g = C->g;
  const double e0 = 1.0 / (p->alpha - 1.0);
  const int r0 = it * p->block_r;
  const int nr = ((g->n < r0 + p->block_r) ? g->n : r0 + p->block_r) - r0;
  double* zbuf = (double*)malloc(sizeof(double) * (size_t)nr * p->block_c);
  for (int jt = 0; jt < g->t_c; ++jt) {
    if (!mask_test(C->mask, g->wpr, it, jt)) continue;
    const int c0 = jt * p->block_c;
    const int nc = ((g->m < c0 + p->block_c) ? g->m : c0 + p->block_c) - c0;
    compute_z_block(p, g, C->q, C->k, C->row_max, r0, nr, c0, nc, zbuf);
    for (int r = 0; r < nr; ++r) {
      const double* zr = zbuf + (size_t)r * nc;
      const double* dorow = C->dout + (size_t)(r0 + r) * g->dv;
      double* dqrow = C->dq + (size_t)(r0 + r) * g->d;
      const double dl = C->delta[r0 + r];
      for (int c = 0; c < nc; ++c) {
        const double t = zr[c] - C->tau[r0 + r];
        if (t <= 0.0) continue;
        const double u = pow_e(pow_e(t, e0), 2.0 - p->alpha);
        const double dp = dot(dorow, C->v + (size_t)(c0 + c) * g->dv, g->dv);
        const double w = g->scale * u * (dp - dl);
        const double* krow = C->k + (size_t)(c0 + c) * g->d;
        for (int x = 0; x < g->d; ++x) dqrow[x] += w * krow[x];
      }
    }
    atomic_fetch_add(&C->visited, 1ull);
  }
  free(zbuf);
}

int orc_backward(const orc_params* p, const double* q, const double* k, const double* v,
                 const double* tau, const double* row_max, const uint32_t* mask,
                 const double* dout, int threads, double* dq, double* dk, double* dv,
                 double* delta, uint64_t* visited_bwd) {
  geom_t g;
  int rc = validate(p, &g);
  if (rc) return rc;
  memset(dq, 0, sizeof(double) * (size_t)g.n * g.d);
  memset(dk, 0, sizeof(double) * (size_t)g.m * g.d);
  memset(dv, 0, sizeof(double) * (size_t)g.m * g.dv);
  rc = orc_compute_delta(p, q, k, v, tau, row_max, mask, dout, threads, delta);
  if (rc) return rc;
  /* PackedBlockMask::transposed (bitpack.cpp:138-143) */
  const int twpr = (g.t_r + 31) / 32;
  uint32_t* tmask = (uint32_t*)calloc((size_t)g.t_c * twpr, sizeof(uint32_t));
  for (int i = 0; i < g.t_r; ++i)
    for (int j = 0; j < g.t_c; ++j)
      if (mask_test(mask, g.wpr, i, j)) mask_set(tmask, twpr, j, i);
  bwd_ctx C;
  C.p = p;
  C.g = &g;
  C.q = q;
  C.k = k;
  C.v = v;
  C.tau = tau;
  C.row_max = row_max;
  C.dout = dout;
  C.delta = delta;
  C.mask = mask;
  C.tmask = tmask;
  C.twpr = twpr;
  C.dq = dq;
  C.dk = dk;
  C.dv = dv;
  atomic_init(&C.visited, 0);
  parallel_for(g.t_c, threads, bwd_key_tile, &C);
  parallel_for(g.t_r, threads, bwd_query_tile, &C);
  if (visited_bwd) *visited_bwd = atomic_load(&C.visited);
  free(tmask);
  return 0;
}

/* -------------------------------------------------------------------- rng */
/* SplitMix64 + Xoshiro256pp with polar Gaussian (rng.hpp:10-72) */
typedef struct {
  uint64_t s[4];
  double spare;
  int spare_valid;
} xo_t;

static uint64_t splitmix_next(uint64_t* st) {
  uint64_t z = (*st += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static void xo_seed(xo_t* x, uint64_t seed) {
  uint64_t sm = seed;
  for (int i = 0; i < 4; ++i) x->s[i] = splitmix_next(&sm);
  x->spare_valid = 0;
  x->spare = 0.0;
}
static inline uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
static uint64_t xo_next(xo_t* x) {
  uint64_t* s = x->s;
  const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}
static double xo_uniform(xo_t* x) { return (double)(xo_next(x) >> 11) * 0x1.0p-53; }
static double xo_gauss(xo_t* x) {
  if (x->spare_valid) {
    x->spare_valid = 0;
    return x->spare;
  }
  double u, v, r2;
  do {
    u = 2.0 * xo_uniform(x) - 1.0;
    v = 2.0 * xo_uniform(x) - 1.0;
    r2 = u * u + v * v;
  } while (r2 >= 1.0 || r2 == 0.0);
  const double sc = sqrt(-2.0 * log(r2) / r2);
  x->spare = v * sc;
  x->spare_valid = 1;
  return u * sc;
}

void orc_gaussian_fill(uint64_t seed, double scale, double* out, size_t count) {
  xo_t x;
  xo_seed(&x, seed);
  for (size_t i = 0; i < count; ++i) out[i] = scale * xo_gauss(&x);
}

void orc_xoshiro_next(uint64_t seed, uint64_t* out, size_t count) {
  xo_t x;
  xo_seed(&x, seed);
  for (size_t i = 0; i < count; ++i) out[i] = xo_next(&x);
}

void orc_gen_attn_inputs(uint64_t seed, int n, int d, double qscale, double* q, double* k,
                         double* v, double* dout) {
  xo_t x;
  xo_seed(&x, seed);
  const size_t cnt = (size_t)n * d;
  for (size_t i = 0; i < cnt; ++i) q[i] = qscale * xo_gauss(&x);
  for (size_t i = 0; i < cnt; ++i) k[i] = 1.0 * xo_gauss(&x);
  for (size_t i = 0; i < cnt; ++i) v[i] = 1.0 * xo_gauss(&x);
  for (size_t i = 0; i < cnt; ++i) dout[i] = 1.0 * xo_gauss(&x);
}
