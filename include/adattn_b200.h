/*
 * adattn_b200.h -- C-ABI of the B200-native alpha-entmax attention library
 * (libadattn_b200.so).  Plain pointers and sizes only; no CUDA or torch types
 * cross this boundary (streams travel as void*).
 *
 * Each entry point replaces one reference interface (paths relative to
 * /root/reference/proj):
 *
 *   adattn_b200_forward        <- adattn::forward        include/adattn/attention.hpp:72-76
 *                                                         (src/attention.cpp:157-361)
 *   adattn_b200_forward_timed  <- adattn::forward with a PhaseTimings* (attention.hpp:62-76)
 *   adattn_b200_forward_ex     <- the same, plus the private per-row tau_h (attention.cpp:223)
 *   adattn_b200_compute_delta  <- adattn::compute_delta  attention.hpp:82-85 (attention.cpp:411-446)
 *   adattn_b200_backward       <- adattn::backward       attention.hpp:87-92 (attention.cpp:448-539)
 *   adattn_b200_backward_ex    <- the same, walking the forward's nonzero-block lists
 *   adattn_b200_stats          <- AttentionStats fill + adattn::block_sparsity
 *                                                         attention.hpp:38-43, 94-97 (attention.cpp:355-359, 541-551)
 *   adattn_b200_validate       <- validate() + PackedHistogramAcc ctor checks
 *                                                         attention.cpp:42-63, 160; bitpack.cpp:55-65
 *   adattn_b200_last_error     <- the what() string of the reference's std::invalid_argument
 *
 * The reference is single-head; this ABI batches B x H independent heads
 * ("harness loops over heads").  Tensors are dense row-major:
 *   q    [B][H][n][d]     k [B][H][m][d]     v [B][H][m][dv]     dout [B][H][n][dv]
 *   out  [B][H][n][dv]    dq [B][H][n][d]    dk [B][H][m][d]     dv   [B][H][m][dv]
 *   tau, row_max, delta [B][H][n] (double; tau on the centred z scale, attention.hpp:46-49)
 *   row_steps [B][H][n] (int32, nullable; the reference's private RowSolve.steps)
 *   mask [B][H][t_r][ceil(t_c/32)] u32 -- the reference PackedBlockMask word layout
 *        (bitpack.hpp:72-110), byte-identical to PackedBlockMask::serialize() payload.
 * All device pointers must be 16-byte aligned.
 *
 * Return codes replace exceptions: 0 ok; ADATTN_ERR_INVALID where the
 * reference throws std::invalid_argument (same message via last_error);
 * ADATTN_ERR_UNSUPPORTED for a valid problem outside this build's GPU
 * envelope; ADATTN_ERR_CUDA for a CUDA failure; ADATTN_ERR_WORKSPACE for a
 * short workspace.  There is no CPU fallback.
 */
#ifndef ADATTN_B200_H
#define ADATTN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADATTN_B200_ABI_VERSION 2

enum {
  ADATTN_OK = 0,
  ADATTN_ERR_INVALID = 1,
  ADATTN_ERR_UNSUPPORTED = 4,
  ADATTN_ERR_CUDA = 5,
  ADATTN_ERR_WORKSPACE = 6,
  ADATTN_ERR_IO = 7
};

/* element types */
enum { ADATTN_F32 = 0, ADATTN_BF16 = 1, ADATTN_F64 = 2 };

/* compute paths:
 *   EXACT -- fp64 SIMT kernels; reproduce the reference's operation order
 *            (bit-identical results for fp32/bf16-representable inputs).
 *            The "fp32 path" of the north star.
 *   TC    -- bf16 tcgen05/TMEM tensor-core kernels, fp32 epilogue math.
 *   AUTO  -- TC for bf16 inputs when the shape is in its envelope, else EXACT. */
enum { ADATTN_PATH_AUTO = 0, ADATTN_PATH_EXACT = 1, ADATTN_PATH_TC = 2 };

/* Mirrors AttentionProblem (attention.hpp:24-36) plus batching and dtypes. */
typedef struct {
  int32_t batch, heads;
  int32_t n, m, d, dv;
  double alpha;
  double scale; /* 0 => 1/sqrt(d) */
  int32_t causal;
  int32_t block_r, block_c;
  int32_t bins;
  int32_t refine_iters;
  double refine_tol;
  int32_t in_dtype;  /* q, k, v, dout: ADATTN_F32 | ADATTN_BF16 | ADATTN_F64 */
  int32_t out_dtype; /* out, dq, dk, dv: ADATTN_F32 | ADATTN_F64 */
  int32_t path;      /* ADATTN_PATH_* */
  int32_t reserved;
} adattn_problem;

/* Mirrors AttentionStats (attention.hpp:38-43), aggregated over heads. */
typedef struct {
  double block_sparsity;
  uint64_t blocks_visited_fwd;
  uint64_t blocks_visited_bwd;
  uint64_t flushes;
  uint64_t addressable_blocks;
  uint64_t active_blocks;
} adattn_stats;

int adattn_b200_abi_version(void);
const char* adattn_b200_last_error(void);

/* Same checks and messages as the reference's validate(); returns
 * ADATTN_ERR_INVALID or ADATTN_ERR_UNSUPPORTED accordingly. */
int adattn_b200_validate(const adattn_problem* p);

/* The path AUTO resolves to (ADATTN_PATH_EXACT or ADATTN_PATH_TC), or <0. */
int adattn_b200_resolved_path(const adattn_problem* p);

size_t adattn_b200_forward_workspace(const adattn_problem* p);
size_t adattn_b200_backward_workspace(const adattn_problem* p);

/* Device pointers; all work is enqueued on `stream` (cudaStream_t or NULL). */
int adattn_b200_forward(const adattn_problem* p, const void* q, const void* k, const void* v,
                        void* out, double* tau, double* row_max, uint32_t* mask,
                        int32_t* row_steps, void* workspace, size_t workspace_bytes,
                        void* stream);

/* forward + PhaseTimings (attention.hpp:62-66; filled by the reference at
 * attention.cpp:196-199, 229-232, 329-332, 352): phase_ms[0..3] = row max,
 * histogram (+ tau_h), refinement (+ mask), output.  The forward's duration
 * (CUDA events on `stream`) split by the share of CTA time each phase took
 * (one %globaltimer-stamped thread per CTA).  Synchronises `stream`. */
int adattn_b200_forward_timed(const adattn_problem* p, const void* q, const void* k,
                              const void* v, void* out, double* tau, double* row_max,
                              uint32_t* mask, int32_t* row_steps, void* workspace,
                              size_t workspace_bytes, void* stream, double* phase_ms);

/* Optional outputs of adattn_b200_forward_ex (every field nullable):
 *   phase_ms -- HOST double[4]: PhaseTimings as adattn_b200_forward_timed
 *               (synchronises `stream` when set);
 *   tau_h    -- DEVICE double[B][H][n]: each row's histogram solution tau_h
 *               (solve_histogram, histogram.cpp:73-161), the start of the
 *               refinement -- kept private by the reference (attention.cpp:223). */
typedef struct {
  double* phase_ms;
  double* tau_h;
  /* DEVICE nonzero-block lists emitted by the forward (both or neither):
   *   block_cnt  int32 [B][H][t_r]        active key blocks per row block;
   *   block_cols uint16 [B][H][t_r][t_c]  their indices, ascending (the first
   *              block_cnt entries of each row; PackedBlockMask::for_each_set
   *              order, bitpack.hpp:85-92).
   * Pass them to adattn_b200_backward_ex: its kernels walk these lists (and
   * their transpose) to skip zero tiles (attention.cpp:334-352, 462-535). */
  int32_t* block_cnt;
  uint16_t* block_cols;
  /* DEVICE buffer (optional; size from adattn_b200_delta_aux_bytes, NULL or 0
   * bytes: not filled) the forward leaves for the backward's delta
   * (attention.cpp:411-446), which it then forms without the delta pre-pass (two
   * products per active tile).  Default (candidate-list mode, alpha >= 1.4): the
   * support lists -- for every row the keys j and u_ij = p_ij^(2 - alpha) of its
   * scores with t > 0 at the final tau, pooled per 256-row block; the backward
   * sums delta_i = sum_j u_ij (dO_i . v_j) / sum_j u_ij (blocks whose pool
   * overflowed fall back to the pre-pass).  With the delta fold
   * (ADATTN_DELTA_FOLD=1): float Ubar_i = sum_j u_ij v_j [B][H][n][dv], then
   * sum_j u_ij [B][H][n], and delta_i = dO_i . Ubar_i / sum_j u_ij. */
  float* delta_aux;
} adattn_forward_extras;

/* Bytes of adattn_forward_extras.delta_aux the forward fills for this problem
 * (tensor-core path, no padded dimension; support lists in candidate-list mode,
 * else the fold where it applies), else 0. */
size_t adattn_b200_delta_aux_bytes(const adattn_problem* p);

int adattn_b200_forward_ex(const adattn_problem* p, const void* q, const void* k,
                           const void* v, void* out, double* tau, double* row_max,
                           uint32_t* mask, int32_t* row_steps, void* workspace,
                           size_t workspace_bytes, void* stream, const adattn_forward_extras* ex);

int adattn_b200_compute_delta(const adattn_problem* p, const void* q, const void* k,
                              const void* v, const double* tau, const double* row_max,
                              const uint32_t* mask, const void* dout, double* delta,
                              void* workspace, size_t workspace_bytes, void* stream);

int adattn_b200_backward(const adattn_problem* p, const void* q, const void* k,
                         const void* v, const double* tau, const double* row_max,
                         const uint32_t* mask, const void* dout, void* dq, void* dk,
                         void* dv, double* delta, void* workspace, size_t workspace_bytes,
                         void* stream);

/* backward with the forward's nonzero-block lists (adattn_forward_extras
 * block_cnt / block_cols; NULL extras or lists: built from `mask`, as
 * adattn_b200_backward does) and its delta_aux (NULL: the delta pre-pass). */
typedef struct {
  const int32_t* block_cnt;
  const uint16_t* block_cols;
  /* the forward's delta_aux (adattn_forward_extras), or NULL: delta pre-pass */
  const float* delta_aux;
} adattn_backward_extras;

int adattn_b200_backward_ex(const adattn_problem* p, const void* q, const void* k,
                            const void* v, const double* tau, const double* row_max,
                            const uint32_t* mask, const void* dout, void* dq, void* dk,
                            void* dv, double* delta, void* workspace, size_t workspace_bytes,
                            void* stream, const adattn_backward_extras* ex);

/* Mask statistics (synchronises `stream`): popcounts, block sparsity over the
 * addressable blocks, visits (fwd = nnz, bwd = 2 nnz) and the flush count of
 * the reference's packed histogram stream. */
int adattn_b200_stats(const adattn_problem* p, const uint32_t* mask, adattn_stats* out,
                      void* stream);

/* Nonzero-block lists of a forward's device mask (all B*H heads, head-major):
 *   rowptr[bh*t_r + 1], cols[nnz]: per row block, its active key blocks in the
 *     order PackedBlockMask::for_each_set visits them (ascending j;
 *     bitpack.hpp:85-92) -- the lists the output pass walks (attention.cpp:334-352);
 *   colptr[bh*t_c + 1], rows[nnz]: per key block, its active query blocks in
 *     ascending i (PackedBlockMask::transposed, bitpack.cpp:138-143) -- the
 *     key-major backward sweep (attention.cpp:464-506).
 * Pointer arrays are exclusive prefix sums (entry [count] = nnz, i.e.
 * adattn_stats.active_blocks); block indices are local to the head.  Any output
 * may be NULL (rowptr is required for cols, colptr for rows).  Enqueued on
 * `stream`; device pointers. */
int adattn_b200_block_lists(const adattn_problem* p, const uint32_t* mask, int64_t* rowptr,
                            int32_t* cols, int64_t* colptr, int32_t* rows, void* stream);

/* block_sparsity (attention.cpp:541-551) of a device mask of `heads` x t_r x
 * ceil(t_c/32) words, aggregated over heads; synchronises `stream`. */
int adattn_b200_mask_sparsity(const uint32_t* mask, int32_t heads, int32_t t_r, int32_t t_c,
                              int32_t causal, adattn_stats* out, void* stream);

/* End-to-end call on HOST buffers (the reference's value-semantics calling
 * convention): uploads inputs, runs forward (+ backward when dout != NULL),
 * downloads results.  Device buffers are cached between calls.  Heads are
 * independent, so the call runs as a pipeline over chunks of heads on three
 * streams (uploads / kernels / downloads): 2-head chunks at both ends, ~16
 * chunks of >= 4 heads in between; a chunk's forward starts once its q, k, v
 * are resident and its forward outputs go back while its backward runs.
 * ADATTN_HOST_CHUNKS=n forces n equal chunks.  Results are identical to the
 * device entry points. */
int adattn_b200_run_host(const adattn_problem* p, const void* q, const void* k, const void* v,
                         const void* dout, void* out, double* tau, double* row_max,
                         uint32_t* mask, void* dq, void* dk, void* dv, double* delta,
                         adattn_stats* stats);

/* Number of kernels this library has launched in this process (profiling aid). */
uint64_t adattn_b200_launch_count(void);

/* Per-kernel CUDA-event timing (off by default).  While enabled every kernel
 * launch is bracketed by events on its own stream.  profile_read synchronises,
 * writes up to `max` durations (ms) and '\n'-separated kernel names, returns
 * the number recorded and clears the log. */
void adattn_b200_profile_enable(int on);
int adattn_b200_profile_read(char* names, size_t names_len, double* ms, int max);

/* ---- Row-wise thresholds on materialised scores ----
 * The paper's inference variant and the reference's
 * per-vector solver (atn solve / bench-solver): for each of `rows` score rows
 * of length n (in_dtype F32 / BF16 / F64; mask[r*n+j] != 0 excludes an entry),
 * center_scores (entmax.cpp:22-57) then
 *   ADATTN_ROWS_HISTOGRAM_HYBRID: build_histogram + solve_histogram +
 *     refine_bracket, hybrid_solve from tau_h (histogram.cpp, hybrid.cpp:35-106);
 *   ADATTN_ROWS_HYBRID: hybrid_solve from the midpoint of [0, 1 - n^(1-alpha)];
 *   ADATTN_ROWS_BISECTION: solve_bisection (entmax.cpp:128-164).
 * Outputs (device pointers; all but tau nullable): tau on the centred scale
 * (best iterate), residual f(tau), iterations (trace length - 1, or the
 * bisection count), converged, probabilities [rows][n] fp32
 * (entmax_apply), trace [rows][trace_len] of iterates (iteration 0 = start;
 * the last iterate carried forward).  fp64 arithmetic; errors as the
 * reference's exceptions (ADATTN_ERR_INVALID + message). */
typedef enum {
  ADATTN_ROWS_HISTOGRAM_HYBRID = 0,
  ADATTN_ROWS_HYBRID = 1,
  ADATTN_ROWS_BISECTION = 2
} adattn_rows_method;

typedef struct {
  int64_t rows;
  int32_t n;
  int32_t in_dtype;
  double alpha;
  int32_t bins;      /* 2..32, histogram method */
  int32_t max_iters;
  double tol;
  int32_t method;    /* adattn_rows_method */
  int32_t trace_len; /* 0: no trace */
} adattn_rows_problem;

int adattn_b200_entmax_rows(const adattn_rows_problem* p, const void* scores,
                            const uint8_t* mask, double* tau, double* residual,
                            int32_t* iterations, int32_t* converged, float* probs,
                            double* trace, void* stream);

/* ---- I/O around the hot path ----------------------------
 * ATN1 tensor files, replacing adattn::save_tensor / load_tensor
 * (tensor_io.hpp:28-29, tensor_io.cpp:39-112): dtype 0 = f32, 1 = f64,
 * rank 1..3.  Errors: ADATTN_ERR_INVALID (bad arguments, the reference's
 * std::invalid_argument) or ADATTN_ERR_IO (parse / file errors, the
 * reference's std::runtime_error, message with the byte offset) and
 * adattn_b200_io_last_error().  tensor_load with values == NULL only fills
 * dtype, rank, dims and count. */
int adattn_b200_tensor_save(const char* path, int dtype, int rank, const uint32_t* dims,
                            const double* values);
int adattn_b200_tensor_load(const char* path, int* dtype, int* rank, uint32_t* dims,
                            double* values, size_t capacity, size_t* count);
const char* adattn_b200_io_last_error(void);

/* `atn attn`'s inputs (atn_main.cpp:227-232): Q = qscale N(0,1), then K, V and
 * dO ~ N(0,1), [n][d] row-major, drawn in that order from Xoshiro256pp(seed)
 * (rng.hpp:25-72; include/adattn_b200/rng.hpp). */
void adattn_b200_attn_inputs(uint64_t seed, int32_t n, int32_t d, double qscale, double* q,
                             double* k, double* v, double* dout);
/* The generator's raw stream (pinning): n_next next() values and n_gauss
 * gaussian() values, each from a fresh Xoshiro256pp(seed). */
void adattn_b200_xoshiro(uint64_t seed, uint64_t* next_out, size_t n_next, double* gauss_out,
                         size_t n_gauss);

#ifdef __cplusplus
}
#endif
#endif
