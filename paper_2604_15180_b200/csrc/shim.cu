// shim.cu -- the C++ drop-in (include/adattn_b200/attention.hpp) over the C-ABI:
// the reference's value-semantics API (attention.hpp:72-97) with the same
// exceptions, running every numeric step on the GPU (EXACT path, fp64).
#include <cuda_runtime.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "adattn_b200.h"
#include "adattn_b200/attention.hpp"

namespace adattn {

// ------------------------------------------------------------ PackedBlockMask
PackedBlockMask::PackedBlockMask(int t_r, int t_c)
    : t_r_(t_r), t_c_(t_c), words_per_row_((t_c + 31) / 32) {
  if (t_r < 1 || t_c < 1) throw std::invalid_argument("PackedBlockMask: bad dimensions");
  words_.assign(size_t(t_r) * words_per_row_, 0u);
}

void PackedBlockMask::set(int i, int j) {
  if (i < 0 || i >= t_r_ || j < 0 || j >= t_c_)
    throw std::invalid_argument("PackedBlockMask: index out of range");
  words_[size_t(i) * words_per_row_ + j / 32] |= 1u << (j % 32);
}

bool PackedBlockMask::test(int i, int j) const {
  if (i < 0 || i >= t_r_ || j < 0 || j >= t_c_)
    throw std::invalid_argument("PackedBlockMask: index out of range");
  return (words_[size_t(i) * words_per_row_ + j / 32] >> (j % 32)) & 1u;
}

int PackedBlockMask::row_popcount(int i) const {
  int pc = 0;
  for (int m = 0; m < words_per_row_; ++m)
    pc += __builtin_popcount(words_[size_t(i) * words_per_row_ + m]);
  return pc;
}

uint64_t PackedBlockMask::total_popcount() const {
  uint64_t pc = 0;
  for (uint32_t w : words_) pc += (uint64_t)__builtin_popcount(w);
  return pc;
}

PackedBlockMask PackedBlockMask::transposed() const {
  PackedBlockMask out(t_c_, t_r_);
  for (int i = 0; i < t_r_; ++i) for_each_set(i, [&](int j) { out.set(j, i); });
  return out;
}

std::vector<uint8_t> PackedBlockMask::serialize() const {
  std::vector<uint8_t> out(8 + words_.size() * 4);
  auto put = [&](size_t at, uint32_t v) {
    for (int b = 0; b < 4; ++b) out[at + b] = uint8_t(v >> (8 * b));
  };
  put(0, uint32_t(t_r_));
  put(4, uint32_t(t_c_));
  for (size_t m = 0; m < words_.size(); ++m) put(8 + 4 * m, words_[m]);
  return out;
}

PackedBlockMask PackedBlockMask::deserialize(const std::vector<uint8_t>& bytes) {
  auto get = [&](size_t at) {
    return uint32_t(bytes[at]) | uint32_t(bytes[at + 1]) << 8 | uint32_t(bytes[at + 2]) << 16 |
           uint32_t(bytes[at + 3]) << 24;
  };
  if (bytes.size() < 8) throw std::invalid_argument("PackedBlockMask: truncated header");
  const uint32_t t_r = get(0), t_c = get(4);
  if (t_r < 1 || t_c < 1 || t_r > (1u << 24) || t_c > (1u << 24))
    throw std::invalid_argument("PackedBlockMask: implausible dimensions");
  PackedBlockMask m{int(t_r), int(t_c)};
  if (bytes.size() != 8 + m.words_.size() * 4)
    throw std::invalid_argument("PackedBlockMask: payload size mismatch");
  for (size_t i = 0; i < m.words_.size(); ++i) m.words_[i] = get(8 + 4 * i);
  return m;
}

namespace {

void cuda_check(cudaError_t e, const char* where) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(where) + ": " + cudaGetErrorString(e));
}

void abi_check(int rc) {
  if (rc == ADATTN_OK) return;
  const std::string msg = adattn_b200_last_error();
  if (rc == ADATTN_ERR_INVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// Device copy of a host array, freed on scope exit.
template <typename T>
struct Dev {
  T* p = nullptr;
  size_t n = 0;
  explicit Dev(size_t count) : n(count) {
    cuda_check(cudaMalloc(&p, sizeof(T) * (count ? count : 1)), "cudaMalloc");
  }
  Dev(const T* host, size_t count) : Dev(count) {
    if (count) cuda_check(cudaMemcpy(p, host, sizeof(T) * count, cudaMemcpyHostToDevice), "upload");
  }
  void get(T* host) const {
    if (n) cuda_check(cudaMemcpy(host, p, sizeof(T) * n, cudaMemcpyDeviceToHost), "download");
  }
  ~Dev() { cudaFree(p); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};

// validate() order and messages (attention.cpp:42-63); the C-ABI checks the rest.
adattn_problem describe(const AttentionProblem& p) {
  const int n = p.q.rows, m = p.k.rows, d = p.q.cols, dv = p.v.cols;
  if (n < 1 || m < 1 || d < 1 || dv < 1) throw std::invalid_argument("attention: empty operand");
  if (p.k.cols != d) throw std::invalid_argument("attention: q/k width mismatch");
  if (p.v.rows != m) throw std::invalid_argument("attention: k/v length mismatch");
  adattn_problem a{};
  a.batch = 1;
  a.heads = 1;
  a.n = n;
  a.m = m;
  a.d = d;
  a.dv = dv;
  a.alpha = p.alpha;
  a.scale = p.scale;
  a.causal = p.causal ? 1 : 0;
  a.block_r = p.block_r;
  a.block_c = p.block_c;
  a.bins = p.bins;
  a.refine_iters = p.refine_iters;
  a.refine_tol = p.refine_tol;
  a.in_dtype = ADATTN_F64;
  a.out_dtype = ADATTN_F64;
  a.path = ADATTN_PATH_EXACT;
  abi_check(adattn_b200_validate(&a));
  return a;
}

int tiles(int len, int block) { return (len + block - 1) / block; }

}  // namespace

AttentionResult forward(const AttentionProblem& p, int threads, PhaseTimings* timings) {
  const adattn_problem a = describe(p);
  const int t_r = tiles(a.n, a.block_r), t_c = tiles(a.m, a.block_c);
  AttentionResult res{Matrix(a.n, a.dv), std::vector<double>(a.n), std::vector<double>(a.n),
                      PackedBlockMask(t_r, t_c), AttentionStats{}};
  Dev<double> q(p.q.data.data(), p.q.data.size()), k(p.k.data.data(), p.k.data.size()),
      v(p.v.data.data(), p.v.data.size());
  Dev<double> out(res.out.data.size()), tau(a.n), rmax(a.n);
  Dev<uint32_t> mask(res.mask.words().size());
  if (timings && threads <= 1) {  // filled like the reference (attention.cpp:170)
    double ph[4];
    abi_check(adattn_b200_forward_timed(&a, q.p, k.p, v.p, out.p, tau.p, rmax.p, mask.p, nullptr,
                                        nullptr, 0, nullptr, ph));
    for (int i = 0; i < 4; ++i) timings->ms[i] += ph[i];
  } else {
    abi_check(adattn_b200_forward(&a, q.p, k.p, v.p, out.p, tau.p, rmax.p, mask.p, nullptr,
                                  nullptr, 0, nullptr));
  }
  adattn_stats st{};
  abi_check(adattn_b200_stats(&a, mask.p, &st, nullptr));
  out.get(res.out.data.data());
  tau.get(res.tau.data());
  rmax.get(res.row_max.data());
  mask.get(res.mask.mutable_words().data());
  res.stats.block_sparsity = st.block_sparsity;
  res.stats.blocks_visited_fwd = st.blocks_visited_fwd;
  res.stats.flushes = st.flushes;
  return res;
}

namespace {

struct BwdInputs {
  Dev<double> q, k, v, tau, rmax, dout;
  Dev<uint32_t> mask;
  BwdInputs(const AttentionProblem& p, const AttentionResult& res, const Matrix& dout_)
      : q(p.q.data.data(), p.q.data.size()),
        k(p.k.data.data(), p.k.data.size()),
        v(p.v.data.data(), p.v.data.size()),
        tau(res.tau.data(), res.tau.size()),
        rmax(res.row_max.data(), res.row_max.size()),
        dout(dout_.data.data(), dout_.data.size()),
        mask(res.mask.words().data(), res.mask.words().size()) {}
};

}  // namespace

std::vector<double> compute_delta(const AttentionProblem& p, const AttentionResult& res,
                                  const Matrix& dout, int threads) {
  (void)threads;
  const adattn_problem a = describe(p);
  if (dout.rows != a.n || dout.cols != a.dv)
    throw std::invalid_argument("compute_delta: dout shape mismatch");
  BwdInputs in(p, res, dout);
  Dev<double> delta(a.n);
  abi_check(adattn_b200_compute_delta(&a, in.q.p, in.k.p, in.v.p, in.tau.p, in.rmax.p, in.mask.p,
                                      in.dout.p, delta.p, nullptr, 0, nullptr));
  std::vector<double> out(a.n);
  delta.get(out.data());
  return out;
}

AttentionGradients backward(const AttentionProblem& p, AttentionResult& res, const Matrix& dout,
                            int threads) {
  (void)threads;
  const adattn_problem a = describe(p);
  if (dout.rows != a.n || dout.cols != a.dv)
    throw std::invalid_argument("backward: dout shape mismatch");
  BwdInputs in(p, res, dout);
  AttentionGradients g{Matrix(a.n, a.d), Matrix(a.m, a.d), Matrix(a.m, a.dv),
                       std::vector<double>(a.n)};
  Dev<double> dq(g.dq.data.size()), dk(g.dk.data.size()), dv(g.dv.data.size()), delta(a.n);
  const size_t ws_bytes = adattn_b200_backward_workspace(&a);
  Dev<uint8_t> ws(ws_bytes);
  abi_check(adattn_b200_backward(&a, in.q.p, in.k.p, in.v.p, in.tau.p, in.rmax.p, in.mask.p,
                                 in.dout.p, dq.p, dk.p, dv.p, delta.p, ws.p, ws_bytes, nullptr));
  cuda_check(cudaDeviceSynchronize(), "backward");
  dq.get(g.dq.data.data());
  dk.get(g.dk.data.data());
  dv.get(g.dv.data.data());
  delta.get(g.delta.data());
  res.stats.blocks_visited_bwd = 2 * res.mask.total_popcount();  // attention.cpp:537
  return g;
}

double block_sparsity(const PackedBlockMask& mask, bool causal) {
  Dev<uint32_t> w(mask.words().data(), mask.words().size());
  adattn_stats st{};
  abi_check(adattn_b200_mask_sparsity(w.p, 1, mask.tile_rows(), mask.tile_cols(), causal ? 1 : 0,
                                      &st, nullptr));
  return st.block_sparsity;
}

}  // namespace adattn
