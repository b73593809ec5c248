// adattn_b200/attention.hpp -- C++ drop-in for the reference's tiled-attention
// interface (/root/reference/proj/include/adattn/attention.hpp:11-97 and
// bitpack.hpp:72-110), implemented on the B200 through the C-ABI in
// include/adattn_b200.h.  Same namespace, type and function names, value
// semantics and exceptions (std::invalid_argument with the reference's
// messages), so a reference caller recompiles against this header and links
// libadattn_b200.so instead of libadattn.a.
//
// Doubles are uploaded as fp64 and run on the EXACT path, which reproduces the
// reference's operation order (bit-identical results; pow() for alpha outside
// {1.5, 2} may differ in the last bit).  `threads` is accepted and ignored
// (work runs on the GPU); PhaseTimings::ms[0..3] receive the forward's
// per-phase device time when threads <= 1, as in the reference.  Every problem the
// reference's validate() accepts runs on the GPU (any tile size and width; a CUDA
// failure throws std::runtime_error) -- there is no CPU fallback.
#pragma once

#include <cstdint>
#include <vector>

namespace adattn {

// Mirrors Matrix (attention.hpp:11-22).
struct Matrix {
  int rows = 0, cols = 0;
  std::vector<double> data;

  Matrix() = default;
  Matrix(int r, int c) : rows(r), cols(c), data(size_t(r) * c, 0.0) {}

  double* row(int i) { return data.data() + size_t(i) * cols; }
  const double* row(int i) const { return data.data() + size_t(i) * cols; }
  double& at(int i, int j) { return data[size_t(i) * cols + j]; }
  double at(int i, int j) const { return data[size_t(i) * cols + j]; }
};

// Mirrors PackedBlockMask (bitpack.hpp:72-110): t_r rows of ceil(t_c/32)
// little-endian u32 words, bit j%32 of word j/32 marks key tile j.
class PackedBlockMask {
 public:
  PackedBlockMask(int t_r, int t_c);

  void set(int i, int j);
  bool test(int i, int j) const;
  int row_popcount(int i) const;
  uint64_t total_popcount() const;

  template <typename Fn>
  void for_each_set(int i, Fn&& fn) const {
    const uint32_t* row = words_.data() + size_t(i) * words_per_row_;
    for (int m = 0; m < words_per_row_; ++m)
      for (uint32_t w = row[m]; w; w &= w - 1) fn(32 * m + __builtin_ctz(w));
  }

  PackedBlockMask transposed() const;
  std::vector<uint8_t> serialize() const;
  static PackedBlockMask deserialize(const std::vector<uint8_t>& bytes);

  int tile_rows() const { return t_r_; }
  int tile_cols() const { return t_c_; }
  size_t byte_size() const { return words_.size() * 4; }
  const std::vector<uint32_t>& words() const { return words_; }
  std::vector<uint32_t>& mutable_words() { return words_; }

  bool operator==(const PackedBlockMask& o) const {
    return t_r_ == o.t_r_ && t_c_ == o.t_c_ && words_ == o.words_;
  }

 private:
  int t_r_, t_c_, words_per_row_;
  std::vector<uint32_t> words_;
};

// Mirrors AttentionProblem (attention.hpp:24-36).
struct AttentionProblem {
  Matrix q, k, v;
  double alpha = 1.5;
  double scale = 0.0;  // 0 means 1/sqrt(d)
  bool causal = false;
  int block_r = 64;
  int block_c = 64;
  int bins = 8;
  int refine_iters = 2;
  double refine_tol = 1e-6;
};

struct AttentionStats {
  double block_sparsity = 0.0;
  uint64_t blocks_visited_fwd = 0;
  uint64_t blocks_visited_bwd = 0;
  uint64_t flushes = 0;
};

struct AttentionResult {
  Matrix out;
  std::vector<double> tau;      // centred-scale thresholds (attention.hpp:46-49)
  std::vector<double> row_max;  // scaled-score row maxima
  PackedBlockMask mask;
  AttentionStats stats;
};

struct AttentionGradients {
  Matrix dq, dk, dv;
  std::vector<double> delta;
};

struct PhaseTimings {
  double ms[4] = {0.0, 0.0, 0.0, 0.0};
};

AttentionResult forward(const AttentionProblem& p, int threads = 1,
                        PhaseTimings* timings = nullptr);

std::vector<double> compute_delta(const AttentionProblem& p, const AttentionResult& res,
                                  const Matrix& dout, int threads = 1);

AttentionGradients backward(const AttentionProblem& p, AttentionResult& res, const Matrix& dout,
                            int threads = 1);

double block_sparsity(const PackedBlockMask& mask, bool causal);

}  // namespace adattn
