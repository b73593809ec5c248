// capi.cu -- the C-ABI (include/adattn_b200.h): validation with the
// reference's messages, path dispatch, mask statistics and the host-buffer
// end-to-end entry.  No CPU compute fallback: every numeric result comes from
// a CUDA kernel; a problem outside the GPU envelope is refused.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "adattn_b200.h"
#include "common.cuh"
#include "exact.cuh"
#include "tc.cuh"

namespace adattn_b200 {
cudaError_t entmax_rows(const adattn_rows_problem& p, const void* scores, const uint8_t* mask,
                        double* tau, double* residual, int32_t* iterations, int32_t* converged,
                        float* probs, double* trace, cudaStream_t st, int* row_err);
const char* rows_error_message(int code);
cudaError_t ell_row_lists(const Geom& g, const uint32_t* mask, int32_t* rcnt, uint16_t* rcol,
                          cudaStream_t st);
}  // namespace adattn_b200

namespace adattn_b200 {

static std::atomic<uint64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {
struct ProfRec {
  std::string name;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
}  // namespace

void prof_begin(const char* name, cudaStream_t st) {
  std::lock_guard<std::mutex> l(g_prof_mu);
  if (!g_prof_on) return;
  ProfRec r;
  r.name = name;
  cudaEventCreate(&r.a);
  cudaEventCreate(&r.b);
  cudaEventRecord(r.a, st);
  g_prof.push_back(r);
}
void prof_end(cudaStream_t st) {
  std::lock_guard<std::mutex> l(g_prof_mu);
  if (!g_prof_on || g_prof.empty()) return;
  cudaEventRecord(g_prof.back().b, st);
}

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(ADATTN_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// validate (attention.cpp:42-63) + PackedHistogramAcc ctor (bitpack.cpp:55-65,
// attention.cpp:35, 160), same order and messages; then this build's envelope.
int check(const adattn_problem* p, Geom* out) {
  if (!p) return fail(ADATTN_ERR_INVALID, "adattn_b200: null problem");
  if (p->batch < 1 || p->heads < 1)
    return fail(ADATTN_ERR_INVALID, "adattn_b200: batch and heads must be positive");
  if (p->n < 1 || p->m < 1 || p->d < 1 || p->dv < 1)
    return fail(ADATTN_ERR_INVALID, "attention: empty operand");
  if (p->causal && p->m != p->n)
    return fail(ADATTN_ERR_INVALID, "attention: causal needs square score matrix");
  if (!(p->alpha > 1.0)) return fail(ADATTN_ERR_INVALID, "attention: alpha must exceed 1");
  if (p->block_r < 1 || p->block_c < 1)
    return fail(ADATTN_ERR_INVALID, "attention: bad tile size");
  if (p->refine_iters < 0 || !(p->refine_tol > 0.0))
    return fail(ADATTN_ERR_INVALID, "attention: bad refinement config");
  const int word_bits = p->bins <= 16 ? 64 : 128;
  if (p->bins <= 0 || word_bits % p->bins != 0)
    return fail(ADATTN_ERR_INVALID, "PackedHistogramAcc: bins must divide word_bits");
  if (word_bits / p->bins < 4)
    return fail(ADATTN_ERR_INVALID, "PackedHistogramAcc: needs at least 4 bits per bin");
  if (p->in_dtype != ADATTN_F32 && p->in_dtype != ADATTN_BF16 && p->in_dtype != ADATTN_F64)
    return fail(ADATTN_ERR_INVALID, "adattn_b200: bad in_dtype");
  if (p->out_dtype != ADATTN_F32 && p->out_dtype != ADATTN_F64)
    return fail(ADATTN_ERR_INVALID, "adattn_b200: bad out_dtype");
  if (p->path < ADATTN_PATH_AUTO || p->path > ADATTN_PATH_TC)
    return fail(ADATTN_ERR_INVALID, "adattn_b200: bad path");
  Geom g;
  g.bh = p->batch * p->heads;
  g.n = p->n;
  g.m = p->m;
  g.n_valid = p->n;
  g.m_valid = p->m;
  g.d = p->d;
  g.dv = p->dv;
  g.block_r = p->block_r;
  g.block_c = p->block_c;
  g.t_r = (p->n + p->block_r - 1) / p->block_r;
  g.t_c = (p->m + p->block_c - 1) / p->block_c;
  g.wpr = (g.t_c + 31) / 32;
  g.bins = p->bins;
  g.causal = p->causal ? 1 : 0;
  g.refine_iters = p->refine_iters;
  g.in_dtype = p->in_dtype;
  g.out_dtype = p->out_dtype;
  g.alpha = p->alpha;
  g.scale = p->scale != 0.0 ? p->scale : 1.0 / std::sqrt((double)p->d);
  g.refine_tol = p->refine_tol;
  g.e0 = 1.0 / (p->alpha - 1.0);
  if (out) *out = g;
  return ADATTN_OK;
}

int resolve(const adattn_problem* p, const Geom& g) {
  const bool tc_ok = p->in_dtype == ADATTN_BF16 && tc_supported(g);
  if (p->path == ADATTN_PATH_TC) {
    if (!tc_ok)
      return -fail(ADATTN_ERR_UNSUPPORTED,
                   "adattn_b200: tensor-core path needs " + tc_envelope());
    return ADATTN_PATH_TC;
  }
  if (p->path == ADATTN_PATH_AUTO && tc_ok) return ADATTN_PATH_TC;
  if (!exact_supported(g))
    return -fail(ADATTN_ERR_UNSUPPORTED,
                 "adattn_b200: exact path supports batch*heads <= 65535");
  return ADATTN_PATH_EXACT;
}

// ------------------------------------------------------------- stats kernel
__global__ void mask_stats_kernel(Geom g, const uint32_t* __restrict__ mask,
                                  unsigned long long* __restrict__ acc) {
  unsigned long long nnz = 0, active = 0;
  const size_t words = (size_t)g.bh * g.t_r * g.wpr;
  for (size_t w = blockIdx.x * (size_t)blockDim.x + threadIdx.x; w < words;
       w += (size_t)gridDim.x * blockDim.x) {
    const uint32_t bits = mask[w];
    if (!bits) continue;
    const int wi = (int)(w % g.wpr);
    const int i = (int)((w / g.wpr) % g.t_r);
    nnz += __popc(bits);
    uint32_t addr = 0;
    for (int b = 0; b < 32; ++b) {
      const long long j = (long long)wi * 32 + b;
      if (j >= g.t_c) break;
      if (!g.causal || j * g.t_r < (long long)(i + 1) * g.t_c) addr |= 1u << b;
    }
    active += __popc(bits & addr);
  }
  for (int off = 16; off; off >>= 1) {
    nnz += __shfl_xor_sync(0xffffffffu, nnz, off);
    active += __shfl_xor_sync(0xffffffffu, active, off);
  }
  if ((threadIdx.x & 31) == 0) {
    if (nnz) atomicAdd(&acc[0], nnz);
    if (active) atomicAdd(&acc[1], active);
  }
}

// Host buffers for adattn_b200_run_host (kept across calls).
struct HostCtx {
  std::mutex mu;
  void* buf[16] = {};
  size_t cap[16] = {};
  cudaStream_t stream = nullptr;
  static constexpr int kMaxChunks = 64;
  cudaStream_t streams[3] = {};  // host->device, kernels, device->host
  cudaEvent_t in_ready[kMaxChunks] = {}, done[kMaxChunks] = {}, fwd_done[kMaxChunks] = {},
              do_ready[kMaxChunks] = {};
  void* get(int slot, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (cap[slot] < bytes) {
      if (buf[slot]) cudaFree(buf[slot]);
      buf[slot] = nullptr;
      if (cudaMalloc(&buf[slot], bytes) != cudaSuccess) {
        cap[slot] = 0;
        return nullptr;
      }
      cap[slot] = bytes;
    }
    return buf[slot];
  }
};
HostCtx& host_ctx() {
  static HostCtx* c = new HostCtx();
  return *c;
}

size_t elem_size(int dtype) { return dtype == ADATTN_BF16 ? 2 : dtype == ADATTN_F32 ? 4 : 8; }

// ---- ragged problems on the tensor-core path ---------------------------------
// The tensor-core kernels tile 256 query rows x 128 keys.  A problem with
// n % 256 != 0 or m % 128 != 0 runs on zero-padded copies (padding rows /
// keys appended to every head); the kernels mask keys >= m_valid like the
// causal diagonal and keep rows >= n_valid out of the mask, padding rows get
// zero dO and tau = row_max = 0, so they add exactly nothing to dK / dV, and
// the results are copied back row by row.  The reference's tiling of the
// real problem (t_r, t_c, ceil(t_c / 32) mask words) is unchanged: the
// padded geometry adds at most one key tile (t_c rounds up to even), which
// never changes the word count.
// Widths work the same way: d, dv <= 128 pad (zero columns) to one D in {64, 128};
// zero columns add exact zeros to every dot product, the scale stays 1/sqrt(d), and
// the extra output / gradient columns are dropped.
bool tc_ragged(const Geom& g) {
  return g.n % 256 != 0 || g.m % 128 != 0 || g.d != g.dv || (g.d != 64 && g.d != 128);
}

Geom padded_geom(const Geom& g) {
  Geom p = g;
  p.n = (g.n + 255) / 256 * 256;
  p.m = g.causal ? p.n : (g.m + 127) / 128 * 128;
  p.t_r = p.n / 64;
  p.t_c = p.m / 64;
  p.wpr = (p.t_c + 31) / 32;
  p.d = p.dv = (g.d > 64 || g.dv > 64) ? 128 : 64;
  return p;
}

// stream-ordered scratch, freed (stream-ordered) when the call returns
class Scratch {
 public:
  explicit Scratch(cudaStream_t st) : st_(st) {}
  ~Scratch() {
    for (void* p : ptrs_) cudaFreeAsync(p, st_);
  }
  // zero-filled device buffer of `bytes` (nullptr with err set on failure)
  void* zeros(size_t bytes) {
    void* p = nullptr;
    if (err_) return nullptr;
    if ((err_ = cudaMallocAsync(&p, bytes ? bytes : 16, st_))) return nullptr;
    ptrs_.push_back(p);
    if ((err_ = cudaMemsetAsync(p, 0, bytes ? bytes : 16, st_))) return nullptr;
    return p;
  }
  // the first `rows` rows x `width` bytes of every head: from a tensor of src_rows
  // rows of src_pitch bytes per head into one of dst_rows rows of dst_pitch bytes
  void copy(void* dst, size_t dst_rows, size_t dst_pitch, const void* src, size_t src_rows,
            size_t src_pitch, size_t rows, size_t width, int heads) {
    if (err_ || !dst || !src) return;
    cudaMemcpy3DParms c = {};
    c.srcPtr = make_cudaPitchedPtr(const_cast<void*>(src), src_pitch, width, src_rows);
    c.dstPtr = make_cudaPitchedPtr(dst, dst_pitch, width, dst_rows);
    c.extent = make_cudaExtent(width, rows, (size_t)heads);
    c.kind = cudaMemcpyDeviceToDevice;
    err_ = cudaMemcpy3DAsync(&c, st_);
  }
  // same row width on both sides
  void rows(void* dst, size_t dst_rows, const void* src, size_t src_rows, size_t rows,
            size_t row_bytes, int heads) {
    copy(dst, dst_rows, row_bytes, src, src_rows, row_bytes, rows, row_bytes, heads);
  }
  // a zero-padded copy of a per-head tensor (rows -> prow rows, row_bytes -> prow_bytes)
  void* pad(const void* src, size_t rows, size_t prow, size_t row_bytes, int heads,
            size_t prow_bytes = 0) {
    if (!src) return nullptr;
    if (!prow_bytes) prow_bytes = row_bytes;
    void* d = zeros(prow * prow_bytes * heads);
    copy(d, prow, prow_bytes, src, rows, row_bytes, rows, row_bytes, heads);
    return d;
  }
  cudaError_t error() const { return err_; }

 private:
  cudaStream_t st_;
  std::vector<void*> ptrs_;
  cudaError_t err_ = cudaSuccess;
};

}  // namespace

uint64_t flushes_of(const Geom& g) {
  const int word_bits = g.bins <= 16 ? 64 : 128;
  const int bits = word_bits / g.bins;
  const unsigned long long L = bits >= 64 ? ~0ull : ((1ull << bits) - 1ull);
  uint64_t per_head = 0;
  for (int it = 0; it < g.t_r; ++it) {
    const int r1 = std::min(g.n, (it + 1) * g.block_r);
    const int jlim = g.causal ? (r1 - 1) / g.block_c : g.t_c - 1;
    const unsigned long long J = (unsigned long long)jlim + 1;
    per_head += (J + L - 1) / L;
  }
  return per_head * (uint64_t)g.bh;
}

uint64_t addressable_of(const Geom& g) {
  uint64_t per_head = 0;
  for (int i = 0; i < g.t_r; ++i) {
    if (!g.causal) {
      per_head += (uint64_t)g.t_c;
      continue;
    }
    // count j in [0, t_c) with j * t_r < (i + 1) * t_c
    const long long lim = ((long long)(i + 1) * g.t_c + g.t_r - 1) / g.t_r;
    per_head += (uint64_t)std::min<long long>(lim, g.t_c);
  }
  return per_head * (uint64_t)g.bh;
}

}  // namespace adattn_b200

using namespace adattn_b200;

extern "C" {

int adattn_b200_abi_version(void) { return ADATTN_B200_ABI_VERSION; }

const char* adattn_b200_last_error(void) { return g_err.c_str(); }

uint64_t adattn_b200_launch_count(void) { return g_launches.load(); }

void adattn_b200_profile_enable(int on) {
  std::lock_guard<std::mutex> l(g_prof_mu);
  g_prof_on = on != 0;
}

int adattn_b200_profile_read(char* names, size_t names_len, double* ms, int max) {
  std::lock_guard<std::mutex> l(g_prof_mu);
  int n = 0;
  std::string all;
  for (auto& r : g_prof) {
    cudaEventSynchronize(r.b);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    if (n < max && ms) ms[n] = t;
    if (n < max) {
      all += r.name;
      all += '\n';
    }
    ++n;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.clear();
  if (names && names_len) {
    const size_t k = std::min(all.size(), names_len - 1);
    std::memcpy(names, all.data(), k);
    names[k] = 0;
  }
  return std::min(n, max);
}

int adattn_b200_validate(const adattn_problem* p) {
  Geom g;
  int rc = check(p, &g);
  if (rc) return rc;
  const int path = resolve(p, g);
  return path < 0 ? -path : ADATTN_OK;
}

int adattn_b200_resolved_path(const adattn_problem* p) {
  Geom g;
  int rc = check(p, &g);
  if (rc) return -rc;
  return resolve(p, g);
}

size_t adattn_b200_forward_workspace(const adattn_problem* p) {
  Geom g;
  if (check(p, &g)) return 0;
  return resolve(p, g) == ADATTN_PATH_TC ? tc_forward_workspace(padded_geom(g)) : 0;
}

size_t adattn_b200_backward_workspace(const adattn_problem* p) {
  Geom g;
  if (check(p, &g)) return 0;
  return resolve(p, g) == ADATTN_PATH_TC ? tc_backward_workspace(padded_geom(g)) : 16;
}

}  // extern "C"

namespace {
// padded copies of the backward inputs of a ragged problem (padding rows: zero
// dO, tau = row_max = 0; padding row blocks: empty mask rows)
struct BwdPadded {
  const void *q, *k, *v, *dout;
  const double *tau, *rm;
  const uint32_t* mask;
  BwdPadded(Scratch& sc, const Geom& g, const Geom& gp, const void* q0, const void* k0,
            const void* v0, const double* tau0, const double* rm0, const uint32_t* mask0,
            const void* dout0) {
    const size_t ei = elem_size(g.in_dtype);
    const int H = g.bh;
    q = sc.pad(q0, g.n, gp.n, g.d * ei, H, gp.d * ei);
    k = sc.pad(k0, g.m, gp.m, g.d * ei, H, gp.d * ei);
    v = sc.pad(v0, g.m, gp.m, g.dv * ei, H, gp.dv * ei);
    dout = sc.pad(dout0, g.n, gp.n, g.dv * ei, H, gp.dv * ei);
    tau = (const double*)sc.pad(tau0, g.n, gp.n, 8, H);
    rm = (const double*)sc.pad(rm0, g.n, gp.n, 8, H);
    mask = (const uint32_t*)sc.pad(mask0, g.t_r, gp.t_r, g.wpr * 4, H);
  }
};

int forward_impl(const adattn_problem* p, const void* q, const void* k, const void* v,
                 void* out, double* tau, double* row_max, uint32_t* mask, int32_t* row_steps,
                 void* workspace, size_t workspace_bytes, void* stream,
                 unsigned long long* phase_ns, double* tau_h, int32_t* lcnt, uint16_t* lcol,
                 float* ubar = nullptr) {
  Geom g;
  int rc = check(p, &g);
  if (rc) return rc;
  g.phase_ns = phase_ns;
  g.tau_h_out = tau_h;
  g.rl_cnt_out = lcnt && lcol ? lcnt : nullptr;
  g.rl_col_out = lcnt && lcol ? lcol : nullptr;
  const int path = resolve(p, g);
  if (path < 0) return -path;
  if (!q || !k || !v || !out || !tau || !row_max || !mask)
    return fail(ADATTN_ERR_INVALID, "adattn_b200_forward: null buffer");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  if (path == ADATTN_PATH_TC) {
    const Geom gp = padded_geom(g);
    if (workspace_bytes < tc_forward_workspace(gp))
      return fail(ADATTN_ERR_WORKSPACE, "adattn_b200_forward: workspace too small");
    if (!tc_ragged(g)) {
      g.ubar_out = ubar;  // (delta fold / support lists: unpadded problems only)
      g.supp_out = ubar;
      e = tc_forward(g, q, k, v, out, tau, row_max, mask, row_steps, workspace, st);
    } else {
      Scratch sc(st);
      const size_t ei = elem_size(g.in_dtype), eo = elem_size(g.out_dtype);
      const int H = g.bh;
      void* qp = sc.pad(q, g.n, gp.n, g.d * ei, H, gp.d * ei);
      void* kp = sc.pad(k, g.m, gp.m, g.d * ei, H, gp.d * ei);
      void* vp = sc.pad(v, g.m, gp.m, g.dv * ei, H, gp.dv * ei);
      void* op = sc.zeros((size_t)H * gp.n * gp.dv * eo);
      double* tp = (double*)sc.zeros((size_t)H * gp.n * 8);
      double* rp = (double*)sc.zeros((size_t)H * gp.n * 8);
      uint32_t* mp = (uint32_t*)sc.zeros((size_t)H * gp.t_r * gp.wpr * 4);
      int32_t* sp = row_steps ? (int32_t*)sc.zeros((size_t)H * gp.n * 4) : nullptr;
      Geom gr = gp;
      gr.tau_h_out = tau_h ? (double*)sc.zeros((size_t)H * gp.n * 8) : nullptr;
      if ((e = sc.error())) return cuda_fail(e, "adattn_b200_forward (padding)");
      if ((e = tc_forward(gr, qp, kp, vp, op, tp, rp, mp, sp, workspace, st)))
        return cuda_fail(e, "adattn_b200_forward");
      sc.copy(out, g.n, g.dv * eo, op, gp.n, gp.dv * eo, g.n, g.dv * eo, H);
      sc.rows(tau, g.n, tp, gp.n, g.n, 8, H);
      sc.rows(row_max, g.n, rp, gp.n, g.n, 8, H);
      sc.rows(mask, g.t_r, mp, gp.t_r, g.t_r, g.wpr * 4, H);
      sc.rows(row_steps, g.n, sp, gp.n, g.n, 4, H);
      sc.rows(tau_h, g.n, gr.tau_h_out, gp.n, g.n, 8, H);
      e = sc.error();
    }
  } else {
    e = exact_forward(g, q, k, v, out, tau, row_max, mask, row_steps, st);
    // the EXACT kernels keep no list state: the lists come from the finished mask
    if (!e && g.rl_cnt_out) e = ell_row_lists(g, mask, g.rl_cnt_out, g.rl_col_out, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "adattn_b200_forward");
  return ADATTN_OK;
}
}  // namespace

extern "C" {

int adattn_b200_forward(const adattn_problem* p, const void* q, const void* k, const void* v,
                        void* out, double* tau, double* row_max, uint32_t* mask,
                        int32_t* row_steps, void* workspace, size_t workspace_bytes,
                        void* stream) {
  return forward_impl(p, q, k, v, out, tau, row_max, mask, row_steps, workspace, workspace_bytes,
                      stream, nullptr, nullptr, nullptr, nullptr);
}

int adattn_b200_forward_timed(const adattn_problem* p, const void* q, const void* k,
                              const void* v, void* out, double* tau, double* row_max,
                              uint32_t* mask, int32_t* row_steps, void* workspace,
                              size_t workspace_bytes, void* stream, double* phase_ms) {
  adattn_forward_extras ex{phase_ms, nullptr, nullptr, nullptr, nullptr};
  if (!phase_ms) return fail(ADATTN_ERR_INVALID, "adattn_b200_forward_timed: null phase_ms");
  return adattn_b200_forward_ex(p, q, k, v, out, tau, row_max, mask, row_steps, workspace,
                                workspace_bytes, stream, &ex);
}

size_t adattn_b200_delta_aux_bytes(const adattn_problem* p) {
  Geom g;
  if (!p || check(p, &g)) return 0;
  if (resolve(p, g) != ADATTN_PATH_TC || tc_ragged(g)) return 0;
  float dummy = 0.f;
  g.ubar_out = &dummy;
  if (tc_delta_fold(g)) return (size_t)g.bh * g.n * (g.dv + 1) * sizeof(float);
  return tc_delta_supp_bytes(g);  // support lists (list mode), else 0
}

int adattn_b200_forward_ex(const adattn_problem* p, const void* q, const void* k,
                           const void* v, void* out, double* tau, double* row_max,
                           uint32_t* mask, int32_t* row_steps, void* workspace,
                           size_t workspace_bytes, void* stream, const adattn_forward_extras* ex) {
  double* const tau_h = ex ? ex->tau_h : nullptr;
  double* const phase_ms = ex ? ex->phase_ms : nullptr;
  int32_t* const lcnt = ex ? ex->block_cnt : nullptr;
  uint16_t* const lcol = ex ? ex->block_cols : nullptr;
  float* const ubar = ex && adattn_b200_delta_aux_bytes(p) ? ex->delta_aux : nullptr;
  if (!phase_ms)
    return forward_impl(p, q, k, v, out, tau, row_max, mask, row_steps, workspace,
                        workspace_bytes, stream, nullptr, tau_h, lcnt, lcol, ubar);
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* acc = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&acc), 4 * sizeof(unsigned long long), st);
  if (!e) e = cudaMemsetAsync(acc, 0, 4 * sizeof(unsigned long long), st);
  if (!e) e = cudaEventCreate(&e0);
  if (!e) e = cudaEventCreate(&e1);
  if (!e) e = cudaEventRecord(e0, st);
  if (e) return cuda_fail(e, "adattn_b200_forward_ex");
  int rc = forward_impl(p, q, k, v, out, tau, row_max, mask, row_steps, workspace,
                        workspace_bytes, stream, acc, tau_h, lcnt, lcol, ubar);
  unsigned long long ns[4] = {0, 0, 0, 0};
  float total = 0.f;
  e = cudaEventRecord(e1, st);
  if (!e) e = cudaMemcpyAsync(ns, acc, sizeof ns, cudaMemcpyDeviceToHost, st);
  if (!e) e = cudaStreamSynchronize(st);
  if (!e) e = cudaEventElapsedTime(&total, e0, e1);
  cudaFreeAsync(acc, st);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rc) return rc;
  if (e) return cuda_fail(e, "adattn_b200_forward_ex");
  // the forward's event-timed duration, split by the CTAs' per-phase time shares
  const double sum = double(ns[0]) + double(ns[1]) + double(ns[2]) + double(ns[3]);
  for (int i = 0; i < 4; ++i) phase_ms[i] = sum > 0.0 ? double(total) * double(ns[i]) / sum : 0.0;
  return ADATTN_OK;
}

int adattn_b200_compute_delta(const adattn_problem* p, const void* q, const void* k,
                              const void* v, const double* tau, const double* row_max,
                              const uint32_t* mask, const void* dout, double* delta,
                              void* workspace, size_t workspace_bytes, void* stream) {
  Geom g;
  int rc = check(p, &g);
  if (rc) return rc;
  const int path = resolve(p, g);
  if (path < 0) return -path;
  if (!q || !k || !v || !tau || !row_max || !mask || !dout || !delta)
    return fail(ADATTN_ERR_INVALID, "compute_delta: null buffer");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  if (path == ADATTN_PATH_TC) {
    const Geom gp = padded_geom(g);
    if (workspace_bytes < tc_backward_workspace(gp))
      return fail(ADATTN_ERR_WORKSPACE, "adattn_b200_compute_delta: workspace too small");
    if (!tc_ragged(g)) {
      e = tc_delta(g, q, k, v, tau, row_max, mask, dout, delta, workspace, st);
    } else {
      Scratch sc(st);
      BwdPadded b(sc, g, gp, q, k, v, tau, row_max, mask, dout);
      double* dlp = (double*)sc.zeros((size_t)g.bh * gp.n * 8);
      if ((e = sc.error())) return cuda_fail(e, "adattn_b200_compute_delta (padding)");
      if ((e = tc_delta(gp, b.q, b.k, b.v, b.tau, b.rm, b.mask, b.dout, dlp, workspace, st)))
        return cuda_fail(e, "adattn_b200_compute_delta");
      sc.rows(delta, g.n, dlp, gp.n, g.n, 8, g.bh);
      e = sc.error();
    }
  } else {
    e = exact_delta(g, q, k, v, tau, row_max, mask, dout, delta, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "adattn_b200_compute_delta");
  return ADATTN_OK;
}

int adattn_b200_backward(const adattn_problem* p, const void* q, const void* k,
                         const void* v, const double* tau, const double* row_max,
                         const uint32_t* mask, const void* dout, void* dq, void* dk,
                         void* dv, double* delta, void* workspace, size_t workspace_bytes,
                         void* stream) {
  return adattn_b200_backward_ex(p, q, k, v, tau, row_max, mask, dout, dq, dk, dv, delta,
                                 workspace, workspace_bytes, stream, nullptr);
}

int adattn_b200_backward_ex(const adattn_problem* p, const void* q, const void* k,
                            const void* v, const double* tau, const double* row_max,
                            const uint32_t* mask, const void* dout, void* dq, void* dk,
                            void* dv, double* delta, void* workspace, size_t workspace_bytes,
                            void* stream, const adattn_backward_extras* ex) {
  Geom g;
  int rc = check(p, &g);
  if (rc) return rc;
  if (ex && ex->block_cnt && ex->block_cols) {  // the forward's nonzero-block lists
    g.rl_cnt_in = ex->block_cnt;
    g.rl_col_in = ex->block_cols;
  }
  const int path = resolve(p, g);
  if (path < 0) return -path;
  if (!q || !k || !v || !tau || !row_max || !mask || !dout || !dq || !dk || !dv || !delta)
    return fail(ADATTN_ERR_INVALID, "backward: null buffer");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  if (path == ADATTN_PATH_TC) {
    const Geom gp = padded_geom(g);
    if (workspace_bytes < tc_backward_workspace(gp))
      return fail(ADATTN_ERR_WORKSPACE, "adattn_b200_backward: workspace too small");
    if (!tc_ragged(g)) {
      if (ex && ex->delta_aux && adattn_b200_delta_aux_bytes(p)) {
        Geom gf = g;
        float dummy = 0.f;
        gf.ubar_out = &dummy;
        if (tc_delta_fold(gf)) g.ubar_in = ex->delta_aux;
        else g.supp_in = ex->delta_aux;
      }
      e = tc_backward(g, q, k, v, tau, row_max, mask, dout, dq, dk, dv, delta, workspace, st);
    } else {
      Scratch sc(st);
      BwdPadded b(sc, g, gp, q, k, v, tau, row_max, mask, dout);
      Geom gq = gp;  // lists of the padded geometry come from the padded mask
      gq.rl_cnt_in = nullptr;
      gq.rl_col_in = nullptr;
      const size_t eo = elem_size(g.out_dtype);
      const int H = g.bh;
      void* dqp = sc.zeros((size_t)H * gp.n * gp.d * eo);
      void* dkp = sc.zeros((size_t)H * gp.m * gp.d * eo);
      void* dvp = sc.zeros((size_t)H * gp.m * gp.dv * eo);
      double* dlp = (double*)sc.zeros((size_t)H * gp.n * 8);
      if ((e = sc.error())) return cuda_fail(e, "adattn_b200_backward (padding)");
      if ((e = tc_backward(gq, b.q, b.k, b.v, b.tau, b.rm, b.mask, b.dout, dqp, dkp, dvp, dlp,
                           workspace, st)))
        return cuda_fail(e, "adattn_b200_backward");
      sc.copy(dq, g.n, g.d * eo, dqp, gp.n, gp.d * eo, g.n, g.d * eo, H);
      sc.copy(dk, g.m, g.d * eo, dkp, gp.m, gp.d * eo, g.m, g.d * eo, H);
      sc.copy(dv, g.m, g.dv * eo, dvp, gp.m, gp.dv * eo, g.m, g.dv * eo, H);
      sc.rows(delta, g.n, dlp, gp.n, g.n, 8, H);
      e = sc.error();
    }
  } else {
    if (workspace_bytes < 8 || !workspace)
      return fail(ADATTN_ERR_WORKSPACE, "adattn_b200_backward: workspace too small");
    unsigned long long* visited = reinterpret_cast<unsigned long long*>(workspace);
    cudaMemsetAsync(visited, 0, sizeof(unsigned long long), st);
    e = exact_backward(g, q, k, v, tau, row_max, mask, dout, dq, dk, dv, delta, visited, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "adattn_b200_backward");
  return ADATTN_OK;
}

static int stats_impl(const Geom& g, const uint32_t* mask, adattn_stats* out,
                      cudaStream_t st) {
  if (!mask || !out) return fail(ADATTN_ERR_INVALID, "adattn_b200_stats: null buffer");
  unsigned long long* acc = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&acc, 2 * sizeof(unsigned long long), st);
  if (e) return cuda_fail(e, "adattn_b200_stats");
  cudaMemsetAsync(acc, 0, 2 * sizeof(unsigned long long), st);
  const size_t words = (size_t)g.bh * g.t_r * g.wpr;
  const int blocks = (int)std::min<size_t>((words + 255) / 256, 4096);
  prof_begin("mask_stats", st);
  mask_stats_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(g, mask, acc);
  prof_end(st);
  note_launch();
  unsigned long long h[2] = {0, 0};
  cudaMemcpyAsync(h, acc, sizeof h, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(acc, st);
  e = cudaStreamSynchronize(st);
  if (e) return cuda_fail(e, "adattn_b200_stats");
  out->blocks_visited_fwd = h[0];
  out->blocks_visited_bwd = 2 * h[0];
  out->active_blocks = h[1];
  out->addressable_blocks = addressable_of(g);
  out->flushes = flushes_of(g);
  out->block_sparsity =
      out->addressable_blocks == 0
          ? 0.0
          : double(out->addressable_blocks - out->active_blocks) / double(out->addressable_blocks);
  return ADATTN_OK;
}

int adattn_b200_stats(const adattn_problem* p, const uint32_t* mask, adattn_stats* out,
                      void* stream) {
  Geom g;
  int rc = check(p, &g);
  if (rc) return rc;
  return stats_impl(g, mask, out, (cudaStream_t)stream);
}

int adattn_b200_entmax_rows(const adattn_rows_problem* p, const void* scores,
                            const uint8_t* mask, double* tau, double* residual,
                            int32_t* iterations, int32_t* converged, float* probs,
                            double* trace, void* stream) {
  if (!p || !scores || !tau) return fail(ADATTN_ERR_INVALID, "entmax_rows: null argument");
  if (!(p->alpha > 1.0)) return fail(ADATTN_ERR_INVALID, "center_scores: alpha must exceed 1");
  if (p->n < 1) return fail(ADATTN_ERR_INVALID, "center_scores: empty score vector");
  if (p->rows < 1 || p->rows > 0x7fffffffLL)
    return fail(ADATTN_ERR_INVALID, "entmax_rows: rows must be in [1, 2^31)");
  if (p->in_dtype != ADATTN_F32 && p->in_dtype != ADATTN_BF16 && p->in_dtype != ADATTN_F64)
    return fail(ADATTN_ERR_INVALID, "entmax_rows: unknown input dtype");
  if (p->trace_len < 0) return fail(ADATTN_ERR_INVALID, "entmax_rows: negative trace_len");
  if (p->method == ADATTN_ROWS_HISTOGRAM_HYBRID) {
    if (p->bins < 2) return fail(ADATTN_ERR_INVALID, "build_histogram: bins must be >= 2");
    if (p->bins > 32)
      return fail(ADATTN_ERR_UNSUPPORTED, "entmax_rows: bins > 32 is outside the GPU envelope");
  } else if (p->method == ADATTN_ROWS_BISECTION) {
    if (p->max_iters < 1)
      return fail(ADATTN_ERR_INVALID, "solve_bisection: max_iters must be positive");
  } else if (p->method != ADATTN_ROWS_HYBRID) {
    return fail(ADATTN_ERR_INVALID, "entmax_rows: unknown method");
  }
  int row_err = 0;
  const cudaError_t e = entmax_rows(*p, scores, mask, tau, residual, iterations, converged, probs,
                                    trace, (cudaStream_t)stream, &row_err);
  if (e) return fail(ADATTN_ERR_CUDA, std::string("entmax_rows: ") + cudaGetErrorString(e));
  if (row_err) return fail(ADATTN_ERR_INVALID, rows_error_message(row_err));
  return ADATTN_OK;
}

int adattn_b200_block_lists(const adattn_problem* p, const uint32_t* mask, int64_t* rowptr,
                            int32_t* cols, int64_t* colptr, int32_t* rows, void* stream) {
  Geom g;
  int rc = check(p, &g);
  if (rc) return rc;
  if (!mask) return fail(ADATTN_ERR_INVALID, "block_lists: null mask");
  if ((cols && !rowptr) || (rows && !colptr))
    return fail(ADATTN_ERR_INVALID, "block_lists: list without its pointer array");
  cudaError_t e = block_lists(g, mask, rowptr, cols, colptr, rows, (cudaStream_t)stream);
  if (e) return cuda_fail(e, "adattn_b200_block_lists");
  return ADATTN_OK;
}

int adattn_b200_mask_sparsity(const uint32_t* mask, int32_t heads, int32_t t_r, int32_t t_c,
                              int32_t causal, adattn_stats* out, void* stream) {
  if (heads < 1 || t_r < 1 || t_c < 1)
    return fail(ADATTN_ERR_INVALID, "PackedBlockMask: bad dimensions");
  Geom g{};
  g.bh = heads;
  g.n = t_r;
  g.m = t_c;
  g.block_r = g.block_c = 1;
  g.t_r = t_r;
  g.t_c = t_c;
  g.wpr = (t_c + 31) / 32;
  g.bins = 8;
  g.causal = causal ? 1 : 0;
  return stats_impl(g, mask, out, (cudaStream_t)stream);
}

int adattn_b200_run_host(const adattn_problem* p, const void* q, const void* k, const void* v,
                         const void* dout, void* out, double* tau, double* row_max,
                         uint32_t* mask, void* dq, void* dk, void* dv, double* delta,
                         adattn_stats* stats) {
  Geom g;
  int rc = check(p, &g);
  if (rc) return rc;
  const int path = resolve(p, g);
  if (path < 0) return -path;
  HostCtx& c = host_ctx();
  std::lock_guard<std::mutex> lock(c.mu);
  if (!c.stream) {
    for (int i = 0; i < 3; ++i)
      if (cudaStreamCreateWithFlags(&c.streams[i], cudaStreamNonBlocking) != cudaSuccess)
        return fail(ADATTN_ERR_CUDA, "adattn_b200_run_host: stream create failed");
    c.stream = c.streams[1];
    for (int i = 0; i < HostCtx::kMaxChunks; ++i)
      if (cudaEventCreateWithFlags(&c.in_ready[i], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&c.done[i], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&c.fwd_done[i], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&c.do_ready[i], cudaEventDisableTiming) != cudaSuccess)
        return fail(ADATTN_ERR_CUDA, "adattn_b200_run_host: event create failed");
  }
  const size_t ei = elem_size(p->in_dtype), eo = elem_size(p->out_dtype);
  const size_t BH = (size_t)g.bh;
  const size_t nq = BH * g.n * g.d, nk = BH * g.m * g.d, nv = BH * g.m * g.dv;
  const size_t no = BH * g.n * g.dv, nrow = BH * g.n;
  const size_t mwords = BH * g.t_r * g.wpr;
  void* dQ = c.get(0, nq * ei);
  void* dK = c.get(1, nk * ei);
  void* dV = c.get(2, nv * ei);
  void* dO = c.get(3, no * eo);
  double* dTau = (double*)c.get(4, nrow * 8);
  double* dRm = (double*)c.get(5, nrow * 8);
  uint32_t* dMask = (uint32_t*)c.get(6, mwords * 4);
  void *dDO = nullptr, *dDQ = nullptr, *dDK = nullptr, *dDV = nullptr;
  double* dDl = nullptr;
  if (dout) {
    dDO = c.get(8, no * ei);
    dDQ = c.get(9, nq * eo);
    dDK = c.get(10, nk * eo);
    dDV = c.get(11, nv * eo);
    dDl = (double*)c.get(12, nrow * 8);
    if (!dDO || !dDQ || !dDK || !dDV || !dDl)
      return fail(ADATTN_ERR_CUDA, "adattn_b200_run_host: device allocation failed");
  }
  // Heads are independent: the call runs as a pipeline over chunks of heads on
  // three streams -- host->device copies of chunk i+1 and device->host copies
  // of chunk i-1 overlap the kernels of chunk i.  Each chunk is a sub-problem
  // (batch 1, `hc` heads) over the same buffers at the chunk's offset.
  // Chunk schedule: two 2-head chunks at each end (short pipeline fill: the first
  // forward needs only its q, k, v; short drain: the last backward's gradients are the
  // only transfer left) and ~16 equal chunks of >= 4 heads in between (few kernel
  // tails).  A 2 / 15 x 4 / 2 taper measured slower (a big chunk's downloads outlast a
  // short final chunk).  ADATTN_HOST_CHUNKS=n forces n equal chunks.
  std::vector<std::pair<size_t, size_t>> chunks;  // (first head, heads)
  {
    const char* env = std::getenv("ADATTN_HOST_CHUNKS");
    if (env && *env) {
      int nch = std::max(1, std::min(HostCtx::kMaxChunks, std::atoi(env)));
      nch = (int)std::min<size_t>((size_t)nch, BH);
      while (nch > 1 && BH % (size_t)nch != 0) --nch;
      for (int i = 0; i < nch; ++i) chunks.push_back({i * (BH / nch), BH / nch});
    } else if (BH >= 24) {
      const size_t mid = BH - 8;
      const size_t nm = std::min<size_t>(16, mid / 4);
      size_t h0 = 0;
      for (int e = 0; e < 2; ++e, h0 += 2) chunks.push_back({h0, 2});
      for (size_t i = 0; i < nm; ++i) {
        const size_t n = mid / nm + (i < mid % nm ? 1 : 0);
        chunks.push_back({h0, n});
        h0 += n;
      }
      for (int e = 0; e < 2; ++e, h0 += 2) chunks.push_back({h0, 2});
    } else {
      int nch = (int)std::min<size_t>(16, BH);
      while (nch > 1 && (BH % (size_t)nch != 0 || BH / (size_t)nch < 4)) --nch;
      for (int i = 0; i < nch; ++i) chunks.push_back({i * (BH / nch), BH / nch});
    }
  }
  size_t hmax = 0;
  for (auto& ch : chunks) hmax = std::max(hmax, ch.second);
  adattn_problem sp = *p;
  sp.batch = 1;
  sp.heads = (int32_t)hmax;
  const size_t wsf = adattn_b200_forward_workspace(&sp);
  const size_t wsb = adattn_b200_backward_workspace(&sp);
  void* ws = c.get(7, std::max(wsf, wsb));
  // delta fold: the chunk's forward leaves sum u v and sum u for its backward
  const size_t aux_bytes = dout ? adattn_b200_delta_aux_bytes(&sp) : 0;
  float* aux = aux_bytes ? (float*)c.get(13, aux_bytes) : nullptr;
  if (aux_bytes && !aux)
    return fail(ADATTN_ERR_CUDA, "adattn_b200_run_host: device allocation failed");
  if (!dQ || !dK || !dV || !dO || !dTau || !dRm || !dMask || !ws)
    return fail(ADATTN_ERR_CUDA, "adattn_b200_run_host: device allocation failed");
  cudaStream_t sin = c.streams[0], sc = c.streams[1], sout = c.streams[2];
  auto cb = [](const void* base, size_t off) { return (const char*)base + off; };
  auto mb = [](void* base, size_t off) { return (char*)base + off; };
  // per-head sizes
  const size_t cq = (size_t)g.n * g.d * ei, ck = (size_t)g.m * g.d * ei, cv = (size_t)g.m * g.dv * ei;
  const size_t cdo = (size_t)g.n * g.dv * ei, co = (size_t)g.n * g.dv * eo;
  const size_t cgq = (size_t)g.n * g.d * eo, cgk = (size_t)g.m * g.d * eo, cgv = (size_t)g.m * g.dv * eo;
  const size_t crow = g.n, cmw = (size_t)g.t_r * g.wpr;
  for (size_t i = 0; i < chunks.size(); ++i) {
    const size_t h = chunks[i].first, hn = chunks[i].second;
    sp.heads = (int32_t)hn;
    cudaMemcpyAsync(mb(dQ, h * cq), cb(q, h * cq), hn * cq, cudaMemcpyHostToDevice, sin);
    cudaMemcpyAsync(mb(dK, h * ck), cb(k, h * ck), hn * ck, cudaMemcpyHostToDevice, sin);
    cudaMemcpyAsync(mb(dV, h * cv), cb(v, h * cv), hn * cv, cudaMemcpyHostToDevice, sin);
    cudaEventRecord(c.in_ready[i], sin);
    if (dout) {  // dO lands while the chunk's forward runs
      cudaMemcpyAsync(mb(dDO, h * cdo), cb(dout, h * cdo), hn * cdo, cudaMemcpyHostToDevice, sin);
      cudaEventRecord(c.do_ready[i], sin);
    }
    cudaStreamWaitEvent(sc, c.in_ready[i], 0);
    adattn_forward_extras fx{nullptr, nullptr, nullptr, nullptr, aux};
    rc = adattn_b200_forward_ex(&sp, mb(dQ, h * cq), mb(dK, h * ck), mb(dV, h * cv),
                                mb(dO, h * co), dTau + h * crow, dRm + h * crow, dMask + h * cmw,
                                nullptr, ws, std::max(wsf, wsb), sc, &fx);
    if (rc) return rc;
    // the forward's outputs go back while the chunk's backward runs
    cudaEventRecord(c.fwd_done[i], sc);
    cudaStreamWaitEvent(sout, c.fwd_done[i], 0);
    if (out) cudaMemcpyAsync(mb(out, h * co), mb(dO, h * co), hn * co, cudaMemcpyDeviceToHost, sout);
    if (tau)
      cudaMemcpyAsync(tau + h * crow, dTau + h * crow, hn * crow * 8, cudaMemcpyDeviceToHost, sout);
    if (row_max)
      cudaMemcpyAsync(row_max + h * crow, dRm + h * crow, hn * crow * 8, cudaMemcpyDeviceToHost, sout);
    if (mask)
      cudaMemcpyAsync(mask + h * cmw, dMask + h * cmw, hn * cmw * 4, cudaMemcpyDeviceToHost, sout);
    if (dout) {
      cudaStreamWaitEvent(sc, c.do_ready[i], 0);
      adattn_backward_extras bx{nullptr, nullptr, aux};
      rc = adattn_b200_backward_ex(&sp, mb(dQ, h * cq), mb(dK, h * ck), mb(dV, h * cv),
                                   dTau + h * crow, dRm + h * crow, dMask + h * cmw,
                                   mb(dDO, h * cdo), mb(dDQ, h * cgq), mb(dDK, h * cgk),
                                   mb(dDV, h * cgv), dDl + h * crow, ws, std::max(wsf, wsb), sc,
                                   &bx);
      if (rc) return rc;
    }
    cudaEventRecord(c.done[i], sc);
    cudaStreamWaitEvent(sout, c.done[i], 0);
    if (dout) {
      if (dq) cudaMemcpyAsync(mb(dq, h * cgq), mb(dDQ, h * cgq), hn * cgq, cudaMemcpyDeviceToHost, sout);
      if (dk) cudaMemcpyAsync(mb(dk, h * cgk), mb(dDK, h * cgk), hn * cgk, cudaMemcpyDeviceToHost, sout);
      if (dv) cudaMemcpyAsync(mb(dv, h * cgv), mb(dDV, h * cgv), hn * cgv, cudaMemcpyDeviceToHost, sout);
      if (delta)
        cudaMemcpyAsync(delta + h * crow, dDl + h * crow, hn * crow * 8, cudaMemcpyDeviceToHost, sout);
    }
  }
  if (stats) {
    rc = adattn_b200_stats(p, dMask, stats, sc);  // whole problem (synchronises sc)
    if (rc) return rc;
  }
  cudaError_t e = cudaStreamSynchronize(sout);
  if (!e) e = cudaStreamSynchronize(sc);
  if (!e) e = cudaStreamSynchronize(sin);
  if (e) return cuda_fail(e, "adattn_b200_run_host");
  return ADATTN_OK;
}

}  // extern "C"
