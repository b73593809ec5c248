// exact_generic.cu -- EXACT path for problems outside the tiled fp64 kernels'
// shared-memory envelope (block_r or block_c > 64, d or dv > 128): one thread
// per query row (forward, delta, dQ) or per key (dK/dV), walking the
// reference's loops in their order (/root/reference/proj/src/attention.cpp),
// so results stay bit-identical to the reference like the tiled kernels'.
//
// Every reference quantity except two is tiling-independent: a row's max,
// histogram counts, O, delta and dQ accumulate over its keys in ascending
// order (inactive blocks hold only t < 0 terms), and a key's dK / dV over its
// rows in ascending order.  The two exceptions are honoured explicitly: the
// refinement sums f, f', f'' add one partial per block_c key tile
// (attention.cpp:250-282), and the mask bit of block (i, j) is the OR over the
// block_r x block_c block at the final thresholds (atomicOr over the tile's rows).
// Compiled with -fmad=false: a*b+c rounds like the reference except where
// fma() is written and the product is exact (fp32 / bf16 inputs).
#include <math_constants.h>

#include "common.cuh"
#include "exact.cuh"

namespace adattn_b200 {
namespace {

constexpr int kGenThreads = 128;
constexpr double kSlack = 1e-9;            // attention.cpp:25
constexpr double kDerivFloor = 1e-12;      // attention.cpp:27

// dot (attention.cpp:29-33) of rows a[0..d) and b[0..d): s += a[x] * b[x] in order;
// fused only when every product is exact (fp32 / bf16 operands)
__device__ __forceinline__ double gdot(const void* A, size_t a0, const void* Bm, size_t b0, int d,
                                       int dt) {
  double s = 0.0;
  if (dt == ADATTN_F64) {
    const double* a = reinterpret_cast<const double*>(A) + a0;
    const double* b = reinterpret_cast<const double*>(Bm) + b0;
    for (int x = 0; x < d; ++x) s = s + a[x] * b[x];
  } else {
    for (int x = 0; x < d; ++x) s = fma(load_elem(A, a0 + x, dt), load_elem(Bm, b0 + x, dt), s);
  }
  return s;
}

__device__ __forceinline__ double gmax(double a, double b) { return (a < b) ? b : a; }

// compute_z_block (attention.cpp:68-84) for one element
__device__ __forceinline__ double gz(const Geom& g, const void* q, const void* k, int bh, int r,
                                     int c, double m) {
  if (g.causal && c > r) return -CUDART_INF;
  const double s = g.scale * gdot(q, ((size_t)bh * g.n + r) * g.d, k, ((size_t)bh * g.m + c) * g.d,
                                  g.d, g.in_dtype);
  return s == m ? 1.0 : (g.alpha - 1.0) * (s - m) + 1.0;
}

__device__ __forceinline__ bool gbit(const uint32_t* mask, const Geom& g, int bh, int i, int j) {
  return (mask[((size_t)bh * g.t_r + i) * g.wpr + (j >> 5)] >> (j & 31)) & 1u;
}

// ------------------------------------------------------------------ forward
// oacc: fp64 accumulator rows [bh][n][dv] (the caller's out when it is fp64)
__global__ void __launch_bounds__(kGenThreads)
    gen_forward_kernel(Geom g, const void* __restrict__ q, const void* __restrict__ k,
                       const void* __restrict__ v, double* __restrict__ oacc,
                       double* __restrict__ tau_out, double* __restrict__ rmax_out,
                       uint32_t* __restrict__ mask_out, int32_t* __restrict__ steps_out) {
  const int bh = blockIdx.y;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= g.n) return;
  const int it = r / g.block_r;
  // the reference tile's key range: causal tiles stop at the tile's last row
  const int rt1 = min(g.n, (it + 1) * g.block_r);
  const int jlim = g.causal ? (rt1 - 1) / g.block_c : g.t_c - 1;
  const int cend = min(g.m, (jlim + 1) * g.block_c);
  const double e0 = g.e0, e1 = e0 - 1.0, e2 = e0 - 2.0;

  // Phase 1: row max (attention.cpp:182-195)
  double m = -CUDART_INF;
  for (int c = 0; c < cend; ++c) {
    if (g.causal && c > r) break;
    m = gmax(m, g.scale * gdot(q, ((size_t)bh * g.n + r) * g.d, k, ((size_t)bh * g.m + c) * g.d,
                               g.d, g.in_dtype));
  }
  // Phase 2: histogram (attention.cpp:201-210)
  uint32_t cnt[32];
  for (int b = 0; b < 32; ++b) cnt[b] = 0u;
  for (int c = 0; c < cend; ++c) {
    const double z = gz(g, q, k, bh, r, c, m);
    if (!(z >= 0.0)) continue;
    ++cnt[min((int)(g.bins * z), g.bins - 1)];
  }
  RowSolve rs;
  {
    double th, lo, hi;
    solve_histogram_dev(cnt, g.bins, g.alpha, th, lo, hi);
    if (g.tau_h_out) g.tau_h_out[(size_t)bh * g.n + r] = th;
    rs.tau = th;
    rs.lo = lo;
    rs.hi = hi;
    rs.f = rs.f1 = rs.f2 = rs.f_hi = 0.0;
    rs.sec_tau = rs.sec_f = rs.best_tau = 0.0;
    rs.best_af = CUDART_INF;
    rs.steps = 0;
    rs.sec_seeded = false;
    rs.done = false;
  }
  // Phase 3: refinement passes (attention.cpp:234-332); a row's passes do not
  // depend on the other rows, and a finished row keeps its tau
  const bool need_sec = g.alpha > 2.0;
  bool first_pass = true;
  for (;;) {
    rs.f = -1.0;
    rs.f1 = 0.0;
    rs.f2 = 0.0;
    if (first_pass) rs.f_hi = -1.0;
    for (int jt = 0; jt <= jlim; ++jt) {  // one partial per reference key tile
      const int c0 = jt * g.block_c, c1 = min(g.m, c0 + g.block_c);
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, shi = 0.0;
      for (int c = c0; c < c1; ++c) {
        const double z = gz(g, q, k, bh, r, c, m);
        const double t = z - rs.tau;
        if (t > 0.0) {
          s0 += pow_e(t, e0);
          s1 += pow_e(e1 < 0.0 ? gmax(t, kDerivFloor) : t, e1);
          s2 += pow_e(e2 < 0.0 ? gmax(t, kDerivFloor) : t, e2);
        }
        if (first_pass && need_sec) {
          const double th = z - rs.hi;
          if (th > 0.0) shi += pow_e(th, e0);
        }
      }
      rs.f += s0;
      rs.f1 -= e0 * s1;
      rs.f2 += e0 * (e0 - 1.0) * s2;
      if (first_pass && need_sec) rs.f_hi += shi;
    }
    first_pass = false;
    if (!row_step(rs, g.alpha, g.refine_tol, g.refine_iters, need_sec)) break;
  }
  const size_t row = (size_t)bh * g.n + r;
  tau_out[row] = rs.tau;
  rmax_out[row] = m;
  if (steps_out) steps_out[row] = rs.steps;
  // mask at the final tau (attention.cpp:254-266, 326-328): OR over the block
  for (int jt = 0; jt <= jlim; ++jt) {
    const int c0 = jt * g.block_c, c1 = min(g.m, c0 + g.block_c);
    bool any = false;
    for (int c = c0; c < c1 && !any; ++c) any = gz(g, q, k, bh, r, c, m) - rs.tau > -kSlack;
    if (any) atomicOr(&mask_out[((size_t)bh * g.t_r + it) * g.wpr + (jt >> 5)], 1u << (jt & 31));
  }
  // Phase 4: O over the row's keys with t > 0, ascending (attention.cpp:334-352)
  double* orow = oacc + row * g.dv;
  for (int x = 0; x < g.dv; ++x) orow[x] = 0.0;
  for (int c = 0; c < cend; ++c) {
    const double t = gz(g, q, k, bh, r, c, m) - rs.tau;
    if (t <= 0.0) continue;
    const double pv = pow_e(t, e0);
    const size_t vr = ((size_t)bh * g.m + c) * g.dv;
    for (int x = 0; x < g.dv; ++x) orow[x] = orow[x] + pv * load_elem(v, vr + x, g.in_dtype);
  }
}

// ---------------------------------------------------------- compute_delta
__global__ void __launch_bounds__(kGenThreads)
    gen_delta_kernel(Geom g, const void* __restrict__ q, const void* __restrict__ k,
                     const void* __restrict__ v, const double* __restrict__ tau,
                     const double* __restrict__ row_max, const uint32_t* __restrict__ mask,
                     const void* __restrict__ dout, double* __restrict__ delta) {
  const int bh = blockIdx.y;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= g.n) return;
  const int it = r / g.block_r;
  const size_t row = (size_t)bh * g.n + r;
  const double m = row_max[row], tr = tau[row];
  double num = 0.0, den = 0.0;
  for (int jt = 0; jt < g.t_c; ++jt) {  // for_each_set (attention.cpp:420-444)
    if (!gbit(mask, g, bh, it, jt)) continue;
    const int c0 = jt * g.block_c, c1 = min(g.m, c0 + g.block_c);
    for (int c = c0; c < c1; ++c) {
      const double t = gz(g, q, k, bh, r, c, m) - tr;
      if (t <= 0.0) continue;
      const double pv = pow_e(t, g.e0);
      const double u = pow_e(pv, 2.0 - g.alpha);
      num += u * gdot(dout, row * g.dv, v, ((size_t)bh * g.m + c) * g.dv, g.dv, g.in_dtype);
      den += u;
    }
  }
  delta[row] = den > 0.0 ? num / den : 0.0;
}

// ------------------------------------------------------------------- dK / dV
// key-major (attention.cpp:464-506): one thread per key, its active query tiles
// ascending (the transposed mask), rows ascending; fp64 accumulators dka, dva
__global__ void __launch_bounds__(kGenThreads)
    gen_dkdv_kernel(Geom g, const void* __restrict__ q, const void* __restrict__ k,
                    const void* __restrict__ v, const double* __restrict__ tau,
                    const double* __restrict__ row_max, const uint32_t* __restrict__ mask,
                    const void* __restrict__ dout, const double* __restrict__ delta,
                    double* __restrict__ dka, double* __restrict__ dva,
                    unsigned long long* visited) {
  const int bh = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.m) return;
  const int jt = c / g.block_c;
  const size_t key = (size_t)bh * g.m + c;
  double* dkr = dka + key * g.d;
  double* dvr = dva + key * g.dv;
  for (int x = 0; x < g.d; ++x) dkr[x] = 0.0;
  for (int x = 0; x < g.dv; ++x) dvr[x] = 0.0;
  unsigned long long nvis = 0;
  for (int it = 0; it < g.t_r; ++it) {
    if (!gbit(mask, g, bh, it, jt)) continue;
    ++nvis;
    const int r0 = it * g.block_r, r1 = min(g.n, r0 + g.block_r);
    for (int r = r0; r < r1; ++r) {
      const size_t row = (size_t)bh * g.n + r;
      const double t = gz(g, q, k, bh, r, c, row_max[row]) - tau[row];
      if (t <= 0.0) continue;
      const double pv = pow_e(t, g.e0);
      const double u = pow_e(pv, 2.0 - g.alpha);
      const double dp = gdot(dout, row * g.dv, v, key * g.dv, g.dv, g.in_dtype);
      const double ds = u * (dp - delta[row]);
      if (pv != 0.0)
        for (int x = 0; x < g.dv; ++x)
          dvr[x] = dvr[x] + pv * load_elem(dout, row * g.dv + x, g.in_dtype);
      if (ds != 0.0) {
        const double w = g.scale * ds;
        for (int x = 0; x < g.d; ++x) dkr[x] = dkr[x] + w * load_elem(q, row * g.d + x, g.in_dtype);
      }
    }
  }
  if (c % g.block_c == 0 && nvis) atomicAdd(visited, nvis);  // one count per block
}

// --------------------------------------------------------------------- dQ
__global__ void __launch_bounds__(kGenThreads)
    gen_dq_kernel(Geom g, const void* __restrict__ q, const void* __restrict__ k,
                  const void* __restrict__ v, const double* __restrict__ tau,
                  const double* __restrict__ row_max, const uint32_t* __restrict__ mask,
                  const void* __restrict__ dout, const double* __restrict__ delta,
                  double* __restrict__ dqa, unsigned long long* visited) {
  const int bh = blockIdx.y;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= g.n) return;
  const int it = r / g.block_r;
  const size_t row = (size_t)bh * g.n + r;
  const double m = row_max[row], tr = tau[row], dl = delta[row];
  double* dqr = dqa + row * g.d;
  for (int x = 0; x < g.d; ++x) dqr[x] = 0.0;
  unsigned long long nvis = 0;
  for (int jt = 0; jt < g.t_c; ++jt) {  // attention.cpp:512-535
    if (!gbit(mask, g, bh, it, jt)) continue;
    ++nvis;
    const int c0 = jt * g.block_c, c1 = min(g.m, c0 + g.block_c);
    for (int c = c0; c < c1; ++c) {
      const double t = gz(g, q, k, bh, r, c, m) - tr;
      if (t <= 0.0) continue;
      const double u = pow_e(pow_e(t, g.e0), 2.0 - g.alpha);
      const size_t key = (size_t)bh * g.m + c;
      const double dp = gdot(dout, row * g.dv, v, key * g.dv, g.dv, g.in_dtype);
      const double w = g.scale * u * (dp - dl);
      for (int x = 0; x < g.d; ++x) dqr[x] = dqr[x] + w * load_elem(k, key * g.d + x, g.in_dtype);
    }
  }
  if (r % g.block_r == 0 && nvis) atomicAdd(visited, nvis);
}

// fp64 accumulators -> the caller's output dtype
__global__ void gen_store_kernel(const double* __restrict__ src, void* dst, size_t n, int dtype) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    store_elem(dst, i, dtype, src[i]);
}

dim3 rows_grid(int rows, int bh) { return dim3((unsigned)((rows + kGenThreads - 1) / kGenThreads), (unsigned)bh); }

// fp64 buffer for `elems` results: the destination itself when it is fp64
struct Acc {
  double* p = nullptr;
  bool own = false;
  cudaError_t init(void* dst, size_t elems, int dtype, cudaStream_t st) {
    if (dtype == ADATTN_F64) {
      p = reinterpret_cast<double*>(dst);
      return cudaSuccess;
    }
    own = true;
    return cudaMallocAsync(reinterpret_cast<void**>(&p), elems * sizeof(double), st);
  }
  cudaError_t finish(void* dst, size_t elems, int dtype, cudaStream_t st) {
    if (!own) return cudaSuccess;
    gen_store_kernel<<<592, 256, 0, st>>>(p, dst, elems, dtype);
    note_launch();
    cudaError_t e = cudaGetLastError();
    cudaFreeAsync(p, st);
    return e;
  }
};

}  // namespace

bool exact_generic_needed(const Geom& g) {
  return g.block_r > 64 || g.block_c > 64 || g.d > 128 || g.dv > 128;
}

cudaError_t exact_generic_forward(const Geom& g, const void* q, const void* k, const void* v,
                                  void* out, double* tau, double* row_max, uint32_t* mask,
                                  int32_t* steps, cudaStream_t st) {
  const size_t no = (size_t)g.bh * g.n * g.dv;
  Acc o;
  cudaError_t e = o.init(out, no, g.out_dtype, st);
  if (!e) e = cudaMemsetAsync(mask, 0, sizeof(uint32_t) * (size_t)g.bh * g.t_r * g.wpr, st);
  if (e) return e;
  prof_begin("exact_generic_fwd", st);
  gen_forward_kernel<<<rows_grid(g.n, g.bh), kGenThreads, 0, st>>>(g, q, k, v, o.p, tau, row_max,
                                                                   mask, steps);
  prof_end(st);
  note_launch();
  if ((e = cudaGetLastError())) return e;
  return o.finish(out, no, g.out_dtype, st);
}

cudaError_t exact_generic_delta(const Geom& g, const void* q, const void* k, const void* v,
                                const double* tau, const double* row_max, const uint32_t* mask,
                                const void* dout, double* delta, cudaStream_t st) {
  gen_delta_kernel<<<rows_grid(g.n, g.bh), kGenThreads, 0, st>>>(g, q, k, v, tau, row_max, mask,
                                                                 dout, delta);
  note_launch();
  return cudaGetLastError();
}

cudaError_t exact_generic_backward(const Geom& g, const void* q, const void* k, const void* v,
                                   const double* tau, const double* row_max, const uint32_t* mask,
                                   const void* dout, void* dq, void* dk, void* dv, double* delta,
                                   unsigned long long* visited, cudaStream_t st) {
  cudaError_t e = exact_generic_delta(g, q, k, v, tau, row_max, mask, dout, delta, st);
  if (e) return e;
  const size_t nq = (size_t)g.bh * g.n * g.d, nk = (size_t)g.bh * g.m * g.d;
  const size_t nv = (size_t)g.bh * g.m * g.dv;
  Acc aq, ak, av;
  if ((e = aq.init(dq, nq, g.out_dtype, st)) || (e = ak.init(dk, nk, g.out_dtype, st)) ||
      (e = av.init(dv, nv, g.out_dtype, st)))
    return e;
  gen_dkdv_kernel<<<rows_grid(g.m, g.bh), kGenThreads, 0, st>>>(g, q, k, v, tau, row_max, mask,
                                                                dout, delta, ak.p, av.p, visited);
  note_launch();
  gen_dq_kernel<<<rows_grid(g.n, g.bh), kGenThreads, 0, st>>>(g, q, k, v, tau, row_max, mask, dout,
                                                              delta, aq.p, visited);
  note_launch();
  if ((e = cudaGetLastError())) return e;
  if ((e = aq.finish(dq, nq, g.out_dtype, st)) || (e = ak.finish(dk, nk, g.out_dtype, st)) ||
      (e = av.finish(dv, nv, g.out_dtype, st)))
    return e;
  return cudaSuccess;
}

}  // namespace adattn_b200
