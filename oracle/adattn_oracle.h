/*
 * adattn_oracle.h -- TEST INFRASTRUCTURE ONLY (the CPU checker, never the product).
 *
 * Plain-C restatement of the reference's tiled alpha-entmax attention
 * (/root/reference/proj/src/attention.cpp, histogram.cpp, bitpack.cpp,
 * entmax.cpp, internal.hpp).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement bit-for-bit
 * against the reference itself, compiled from its own sources by
 * oracle/Makefile into oracle/_ref/libadattn_ref.so (same entry points,
 * prefix ref_ instead of orc_), and against the reference test-suite
 * known-answer vectors (tests/golden/).
 *
 * All matrices are row-major double.  Masks use the reference's
 * PackedBlockMask layout (bitpack.hpp:72-110): t_r rows of ceil(t_c/32)
 * little-endian u32 words, bit j%32 of word j/32 is key tile j.
 */
#ifndef ADATTN_ORACLE_H
#define ADATTN_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors AttentionProblem (attention.hpp:24-36) minus the matrices. */
typedef struct {
  int32_t n, m, d, dv;
  double alpha;
  double scale; /* 0 => 1/sqrt(d) (attention.cpp:61) */
  int32_t causal;
  int32_t block_r, block_c;
  int32_t bins;
  int32_t refine_iters;
  double refine_tol;
} orc_params;

/* Mirrors AttentionStats (attention.hpp:38-43). */
typedef struct {
  double block_sparsity;
  uint64_t blocks_visited_fwd;
  uint64_t blocks_visited_bwd;
  uint64_t flushes;
} orc_stats;

/* Error codes: 0 ok, 1 invalid_argument, 2 overflow_error, 3 other. */
const char* orc_last_error(void);

/* forward (attention.cpp:157-361).  row_steps (nullable) receives each row's
 * RowSolve.steps (attention.cpp:219), which the reference keeps private. */
int orc_forward(const orc_params* p, const double* q, const double* k, const double* v,
                int threads, double* out, double* tau, double* row_max, uint32_t* mask,
                int32_t* row_steps, orc_stats* stats);

/* forward plus the reference's private per-row histogram state (nullable):
 * tau_h[n] (solve_histogram, attention.cpp:223-228) and counts[n][bins]
 * (the streamed histogram, attention.cpp:201-210). */
int orc_forward_ex(const orc_params* p, const double* q, const double* k, const double* v,
                   int threads, double* out, double* tau, double* row_max, uint32_t* mask,
                   int32_t* row_steps, orc_stats* stats, double* tau_h, uint32_t* counts);

/* dense_reference (attention.cpp:363-409). */
int orc_dense_reference(const orc_params* p, const double* q, const double* k,
                        const double* v, double* out, double* tau, double* row_max,
                        uint32_t* mask, orc_stats* stats);

/* compute_delta (attention.cpp:411-446). */
int orc_compute_delta(const orc_params* p, const double* q, const double* k,
                      const double* v, const double* tau, const double* row_max,
                      const uint32_t* mask, const double* dout, int threads, double* delta);

/* backward (attention.cpp:448-539); visited_bwd (nullable) mirrors
 * res.stats.blocks_visited_bwd. */
int orc_backward(const orc_params* p, const double* q, const double* k, const double* v,
                 const double* tau, const double* row_max, const uint32_t* mask,
                 const double* dout, int threads, double* dq, double* dk, double* dv,
                 double* delta, uint64_t* visited_bwd);

/* block_sparsity (attention.cpp:541-551). */
double orc_block_sparsity(const uint32_t* mask, int t_r, int t_c, int causal);

/* solve_histogram, left-edge mode (histogram.cpp:73-161) + refine_bracket (163-165). */
int orc_solve_histogram(const uint32_t* counts, int bins, double alpha, double* tau_h,
                        int* bracket_floor, double* lo, double* hi);

/* propose_step (internal.hpp:32-55).  kind: 1 halley 2 newton 3 secant 4 bisection. */
double orc_propose_step(double alpha, double tau, double f, double f1, double f2,
                        double sec_tau, double sec_f, double lo, double hi, int* kind);

/* f_eval (entmax.cpp:59-78) on an explicit centred vector. */
void orc_f_eval(const double* z, int n, double alpha, double tau, double* f, double* f1,
                double* f2);

/* Xoshiro256pp(seed) (rng.hpp:25-72): `count` draws of scale*gaussian(), in order. */
void orc_gaussian_fill(uint64_t seed, double scale, double* out, size_t count);
/* Same generator state, raw next() outputs. */
void orc_xoshiro_next(uint64_t seed, uint64_t* out, size_t count);
/* cmd_attn input stream (atn_main.cpp:227-232): Q=qscale*N, K, V, dO ~ N(0,1)
 * drawn in that order from one generator.  Q,K,V,dO are n x d. */
void orc_gen_attn_inputs(uint64_t seed, int n, int d, double qscale, double* q, double* k,
                         double* v, double* dout);

#ifdef __cplusplus
}
#endif
#endif
