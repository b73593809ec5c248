// test_shim.cpp -- the reference's own test_attention.cpp scenarios
// (/root/reference/proj/tests/test_attention.cpp) compiled against the C++
// drop-in (include/adattn_b200/attention.hpp) and run on the B200.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "adattn_b200/attention.hpp"

using namespace adattn;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (cond) ++g_pass;                                                    \
    else {                                                                 \
      ++g_fail;                                                            \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
    }                                                                      \
  } while (0)
#define CHECK_THROWS(expr, Exc)                                            \
  do {                                                                     \
    bool _t = false;                                                       \
    try { (void)(expr); } catch (const Exc&) { _t = true; } catch (...) {} \
    CHECK(_t);                                                             \
  } while (0)

// splitmix64-seeded deterministic gaussians (Box-Muller); the values, not the
// generator, matter here
struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double u() { return double(next() >> 11) * 0x1.0p-53; }
  double g() {
    double a = u(), b = u();
    if (a < 1e-300) a = 1e-300;
    return std::sqrt(-2.0 * std::log(a)) * std::cos(6.283185307179586 * b);
  }
};

static Matrix gauss(Rng& r, int rows, int cols, double scale = 1.0) {
  Matrix m(rows, cols);
  for (double& x : m.data) x = scale * r.g();
  return m;
}
static Matrix from(int rows, int cols, std::vector<double> v) {
  Matrix m(rows, cols);
  m.data = std::move(v);
  return m;
}
static AttentionProblem problem(Rng& r, int n, int d, double alpha, int br, int bc, bool causal,
                                double qs = 1.0) {
  AttentionProblem p;
  p.q = gauss(r, n, d, qs);
  p.k = gauss(r, n, d);
  p.v = gauss(r, n, d);
  p.alpha = alpha;
  p.causal = causal;
  p.block_r = br;
  p.block_c = bc;
  return p;
}
static double prob_at(const AttentionProblem& p, const AttentionResult& res, int i, int j) {
  if (p.causal && j > i) return 0.0;
  const int d = p.q.cols;
  double s = 0.0;
  for (int x = 0; x < d; ++x) s += p.q.at(i, x) * p.k.at(j, x);
  s *= p.scale != 0.0 ? p.scale : 1.0 / std::sqrt(double(d));
  const double z = s == res.row_max[i] ? 1.0 : (p.alpha - 1.0) * (s - res.row_max[i]) + 1.0;
  const double t = z - res.tau[i];
  return t > 0.0 ? std::pow(t, 1.0 / (p.alpha - 1.0)) : 0.0;
}

int main() {
  {  // shape and parameter validation (test_attention.cpp:67-105)
    Rng rng(1);
    AttentionProblem p = problem(rng, 8, 4, 1.5, 4, 4, false);
    AttentionProblem bad = p;
    bad.k = gauss(rng, 8, 3);
    CHECK_THROWS(forward(bad), std::invalid_argument);
    bad = p;
    bad.v = gauss(rng, 7, 4);
    CHECK_THROWS(forward(bad), std::invalid_argument);
    bad = p;
    bad.k = gauss(rng, 6, 4);
    bad.v = gauss(rng, 6, 4);
    bad.causal = true;
    CHECK_THROWS(forward(bad), std::invalid_argument);
    bad = p;
    bad.alpha = 1.0;
    CHECK_THROWS(forward(bad), std::invalid_argument);
    bad = p;
    bad.block_r = 0;
    CHECK_THROWS(forward(bad), std::invalid_argument);
    bad = p;
    bad.refine_tol = 0.0;
    CHECK_THROWS(forward(bad), std::invalid_argument);
    bad = p;
    bad.bins = 5;
    CHECK_THROWS(forward(bad), std::invalid_argument);
    AttentionProblem wide = p;
    wide.bins = 32;
    bool ok = true;
    try { forward(wide); } catch (...) { ok = false; }
    CHECK(ok);
    // tiles and widths beyond the tiled kernels' envelope run too (exact_generic.cu)
    Rng r2(12);
    AttentionProblem big = problem(r2, 150, 160, 1.5, 128, 96, true);
    ok = true;
    try {
      AttentionResult res = forward(big);
      const Matrix dout = gauss(r2, 150, 160);
      const AttentionGradients g = backward(big, res, dout);
      for (int i = 0; i < big.q.rows; ++i) {
        double sum = 0.0;
        for (int j = 0; j < big.k.rows; ++j) sum += prob_at(big, res, i, j);
        ok &= std::isfinite(sum) && std::abs(sum - 1.0) < 1e-4 && std::isfinite(g.dq.at(i, 0));
      }
    } catch (...) {
      ok = false;
    }
    CHECK(ok);
  }
  {  // single query and key reduces to a point mass (107-131)
    AttentionProblem p;
    p.q = from(1, 1, {2.0});
    p.k = from(1, 1, {1.0});
    p.v = from(1, 1, {5.0});
    p.alpha = 2.0;
    p.scale = 1.0;
    AttentionResult res = forward(p);
    CHECK(res.out.at(0, 0) == 5.0);
    CHECK(res.tau[0] == 0.0);
    CHECK(res.row_max[0] == 2.0);
    CHECK(res.mask.test(0, 0));
    CHECK(res.stats.blocks_visited_fwd == 1);
    CHECK(res.stats.block_sparsity == 0.0);
    const AttentionGradients g = backward(p, res, from(1, 1, {1.0}));
    CHECK(g.delta[0] == 5.0);
    CHECK(g.dv.at(0, 0) == 1.0);
    CHECK(g.dk.at(0, 0) == 0.0);
    CHECK(g.dq.at(0, 0) == 0.0);
    CHECK(res.stats.blocks_visited_bwd == 2);
  }
  {  // two key sparsemax rows come out exact (133-163)
    AttentionProblem p;
    p.q = from(2, 1, {1.0, 1.0});
    p.k = from(2, 1, {1.0, 0.5});
    p.v = from(2, 2, {2.0, 0.0, 0.0, 4.0});
    p.alpha = 2.0;
    p.scale = 1.0;
    AttentionResult res = forward(p);
    CHECK(res.tau[0] == 0.25 && res.tau[1] == 0.25);
    CHECK(res.out.at(0, 0) == 1.5 && res.out.at(0, 1) == 1.0);
    CHECK(res.out.at(1, 0) == 1.5 && res.out.at(1, 1) == 1.0);
    const AttentionGradients g = backward(p, res, from(2, 2, {1.0, 0.0, 0.0, 1.0}));
    CHECK(g.delta[0] == 1.0 && g.delta[1] == 2.0);
    CHECK(std::abs(g.dq.at(0, 0) - 0.5) < 1e-12 && std::abs(g.dq.at(1, 0) + 1.0) < 1e-12);
    CHECK(std::abs(g.dk.at(0, 0) + 1.0) < 1e-12 && std::abs(g.dk.at(1, 0) - 1.0) < 1e-12);
    CHECK(std::abs(g.dv.at(0, 0) - 0.75) < 1e-12 && std::abs(g.dv.at(1, 1) - 0.25) < 1e-12);
  }
  {  // row sums and off-mask probabilities (217-237)
    Rng rng(7);
    AttentionProblem p = problem(rng, 50, 6, 1.5, 8, 8, true);
    p.refine_iters = 8;
    p.refine_tol = 1e-10;
    const AttentionResult res = forward(p);
    for (int i = 0; i < 50; ++i) {
      double sum = 0.0;
      for (int j = 0; j < 50; ++j) sum += prob_at(p, res, i, j);
      CHECK(std::abs(sum - 1.0) < 1e-8);
    }
    for (int i = 0; i < res.mask.tile_rows(); ++i)
      for (int j = 0; j < res.mask.tile_cols(); ++j) {
        if (res.mask.test(i, j)) continue;
        for (int r = i * 8; r < std::min(50, (i + 1) * 8); ++r)
          for (int c = j * 8; c < std::min(50, (j + 1) * 8); ++c) CHECK(prob_at(p, res, r, c) == 0.0);
      }
  }
  {  // forward visits exactly the set mask bits (239-250)
    Rng rng(99);
    for (const bool causal : {false, true}) {
      AttentionProblem p = problem(rng, 70, 4, 1.5, 16, 8, causal, 2.0);
      AttentionResult res = forward(p);
      CHECK(res.stats.blocks_visited_fwd == res.mask.total_popcount());
      backward(p, res, gauss(rng, 70, 4));
      CHECK(res.stats.blocks_visited_bwd == 2 * res.mask.total_popcount());
    }
  }
  {  // block sparsity counts addressable blocks (252-263)
    PackedBlockMask mask(2, 2);
    mask.set(0, 0);
    mask.set(1, 0);
    mask.set(1, 1);
    CHECK(std::abs(block_sparsity(mask, false) - 0.25) < 1e-15);
    CHECK(block_sparsity(mask, true) == 0.0);
    PackedBlockMask empty(2, 2);
    CHECK(block_sparsity(empty, false) == 1.0 && block_sparsity(empty, true) == 1.0);
  }
  {  // threads do not change a single bit (287-307)
    Rng rng(555);
    AttentionProblem p = problem(rng, 120, 8, 1.5, 16, 16, true);
    const AttentionResult one = forward(p, 1);
    const AttentionResult many = forward(p, 7);
    CHECK(one.out.data == many.out.data && one.tau == many.tau && one.mask == many.mask);
    const Matrix dout = gauss(rng, 120, 8);
    AttentionResult r1 = one, r4 = one;
    const AttentionGradients g1 = backward(p, r1, dout, 1), g4 = backward(p, r4, dout, 4);
    CHECK(g1.dq.data == g4.dq.data && g1.dk.data == g4.dk.data && g1.dv.data == g4.dv.data);
  }
  {  // zero upstream gradient zeroes every output gradient (309-319)
    Rng rng(3);
    AttentionProblem p = problem(rng, 20, 4, 2.0, 8, 8, false);
    AttentionResult res = forward(p);
    const AttentionGradients g = backward(p, res, Matrix(20, 4));
    bool zero = true;
    for (double x : g.dq.data) zero &= x == 0.0;
    for (double x : g.dk.data) zero &= x == 0.0;
    for (double x : g.dv.data) zero &= x == 0.0;
    for (double x : g.delta) zero &= x == 0.0;
    CHECK(zero);
  }
  {  // mask serialization layout is frozen (test_bitpack.cpp:231-251)
    PackedBlockMask mask(2, 40);
    mask.set(0, 0);
    mask.set(0, 33);
    mask.set(1, 39);
    const std::vector<uint8_t> want = {2, 0, 0, 0, 40, 0, 0, 0, 1, 0, 0, 0,
                                       2, 0, 0, 0, 0, 0, 0, 0, 0x80, 0, 0, 0};
    CHECK(mask.serialize() == want);
    CHECK(PackedBlockMask::deserialize(want) == mask);
    CHECK(mask.transposed().transposed() == mask);
  }
  {  // PhaseTimings: filled per phase when threads <= 1, untouched otherwise (attention.cpp:170)
    Rng rng(8);
    AttentionProblem p = problem(rng, 256, 32, 1.5, 64, 64, true);
    PhaseTimings t;
    const AttentionResult a = forward(p, 1, &t);
    bool all = true;
    for (double ms : t.ms) all &= ms > 0.0;
    CHECK(all);
    PhaseTimings u;
    const AttentionResult b = forward(p, 4, &u);
    CHECK(u.ms[0] == 0.0 && u.ms[1] == 0.0 && u.ms[2] == 0.0 && u.ms[3] == 0.0);
    CHECK(a.out.data == b.out.data && a.tau == b.tau);
  }
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
