// tc_bwd.cu -- bf16 tensor-core backward of tiled alpha-entmax attention for
// sm_100a (reference: /root/reference/proj/src/attention.cpp:411-539).
//
// Three kernels, each visiting only the set 64x64 mask blocks, one writer per
// output element (the reference's determinism rule):
//   tc_delta_kernel  query-major: S = Q K^T, dP = dO V^T -> delta_i =
//                    sum u dp / sum u, u = p^(2-alpha) = t^(1/(alpha-1) - 1)
//                    (compute_delta, attention.cpp:411-446); also writes the
//                    per-row constants (C = 1-(alpha-1)m-tau, delta) as fp32
//   tc_dq_kernel     query-major: dS = u (dp - delta) (bf16, smem) then
//                    dQ += dS K_j with K_j read MN-major (attention.cpp:508-535)
//   tc_dkdv_kernel   key-major over 128 keys: S^T = K Q_i^T, dP^T = V dO_i^T
//                    (M = keys), P^T and dS^T written back to TMEM as bf16 and
//                    used as the TMEM A operand of dV += P^T dO_i and
//                    dK += dS^T Q_i (attention.cpp:464-506)
#include <cuda.h>

#include <cstdlib>
#include <math_constants.h>

#include "common.cuh"
#include "tc.cuh"
#include "tc_common.cuh"
#include "tc_host.cuh"

namespace adattn_b200 {
namespace tc {
#ifdef ADATTN_PIPE_STATS
// dK/dV kernel: [0] MMA waits on Q/dO stage, [1] MMA waits on p_full, [2]
// epilogue warp 4 waits on s_full, [3] MMA-warp cycles, [4] units
__device__ unsigned long long g_bwd_stats[8];
// event trace of the pair dK/dV kernel's first cluster (leader CTA): [role][unit][event]
__device__ long long g_btrace[3][512][4];
#define BTRACE(role, uu, ev) \
  if (blockIdx.x == 0 && (uu) < 512) g_btrace[role][uu][ev] = clock64()
#define BSTAT_T0() const long long _t0 = clock64()
#define BSTAT_ADD(i, cond) \
  if (cond) atomicAdd(&g_bwd_stats[i], (unsigned long long)(clock64() - _t0))
#else
#define BSTAT_T0() \
  do {             \
  } while (0)
#define BSTAT_ADD(i, cond) \
  do {                     \
  } while (0)
#define BTRACE(role, uu, ev) \
  do {                       \
  } while (0)
#endif
namespace {

constexpr int BM = 256;  // query rows per CTA (delta, dQ)
constexpr int BN = 64;   // keys per tile
constexpr int NST = 4;
constexpr int kThreads = 320;  // 8 epilogue warps, producer, MMA issuer
constexpr int kEpi = 256;

struct BwdArgs {
  Geom g;
  int ncta_rows;
  float A1;
  float e0f, e1f;
  const double* tau;
  const double* row_max;
  // the nonzero-block lists the kernels walk (ELL, ascending; ell_row_lists /
  // ell_col_lists): row block i of head h: rcnt[h t_r + i] key blocks at
  // rcol[(h t_r + i) t_c ..]; key block j: ccnt[h t_c + j] query blocks at
  // crow[(h t_c + j) t_r ..]
  const int32_t* rcnt;
  const uint16_t* rcol;
  const int32_t* ccnt;
  const uint16_t* crow;
  double* delta;
  float2* rowc;  // [bh*n] {C, delta}
  const void* dout;  // bf16 [bh*n][dv] (delta from the forward's fold)
  const void* v;     // bf16 [bh*m][dv] (delta from the support lists)
  // delta kernels: 256-row blocks (global row / 256) whose delta the support kernel
  // formed are skipped (supp_skip[block] == 0); nullptr: every block
  const uint32_t* supp_skip;
  // dQ kernels: heads whose dQ the support-list rows kernel formed (dq_skip[bh] == 0)
  const uint32_t* dq_skip;
  // dK/dV kernels: heads whose dK/dV the support-list keys kernel formed (kv_skip[bh] == 0)
  const uint32_t* kv_skip;
  const void* kp;  // bf16 [bh*m][d] (dQ from the support lists)
  const void* qp;  // bf16 [bh*n][d] (dK from the support lists)
  int skip_f16;      // pair dK/dV two-buffer kernel: skip heads the SLOT3 kernel takes
  // fp16 operand plan of the pair dQ and dK/dV kernels (device; nullptr: bf16 hi/lo)
  const struct F16Plan* f16;
  void* dq;
  void* dk;
  void* dv;
  float scale_f;
};

// Mask words of row blocks rb0 .. rb0 + nrb - 1 of head bh, rebuilt in shared
// memory from the row lists (all threads of the CTA call this).
__device__ __forceinline__ void rows_from_lists(uint32_t* dst, int nrb, const BwdArgs& a, int bh,
                                                int rb0, int tid, int nthreads) {
  const Geom& g = a.g;
  for (int i = tid; i < nrb * g.wpr; i += nthreads) dst[i] = 0u;
  __syncthreads();
  for (int r = 0; r < nrb; ++r) {
    const int ib = rb0 + r;
    if (ib >= g.t_r) break;
    const size_t row = (size_t)bh * g.t_r + ib;
    const int cnt = a.rcnt[row];
    const uint16_t* c = a.rcol + row * g.t_c;
    for (int k = tid; k < cnt; k += nthreads) {
      const uint32_t j = c[k];
      atomicOr(&dst[r * g.wpr + (j >> 5)], 1u << (j & 31));
    }
  }
  __syncthreads();
}

// ubits[i] = bit kh set iff query block i is active in key block j0 + kh (kh < nkb),
// from the column lists (all threads of the CTA call this).
__device__ __forceinline__ void units_from_lists(uint8_t* ubits, int nkb, const BwdArgs& a, int bh,
                                                 int j0, int tid, int nthreads) {
  const Geom& g = a.g;
  for (int i = tid; i < g.t_r; i += nthreads) ubits[i] = 0;
  __syncthreads();
  for (int kh = 0; kh < nkb; ++kh) {  // one key block per pass: no two writers per byte
    const int j = j0 + kh;
    if (j < g.t_c) {
      const size_t col = (size_t)bh * g.t_c + j;
      const int cnt = a.ccnt[col];
      const uint16_t* r = a.crow + col * g.t_r;
      for (int k = tid; k < cnt; k += nthreads) ubits[r[k]] |= (uint8_t)(1u << kh);
    }
    __syncthreads();
  }
}


// Nonzero tiles / units of a CTA, compacted once (one warp, ascending) so every role
// walks a list instead of scanning all tile indices with mask lookups (at 99% block
// sparsity those scans were most of the backward's time).
template <typename P>
__device__ __forceinline__ void compact_active(uint16_t* list, volatile uint32_t* cnt, int last,
                                               int lane, P&& pred) {
  uint32_t n = 0;
  for (int b = 0; b <= last; b += 32) {
    const int J = b + lane;
    const bool on = J <= last && pred(J);
    const uint32_t m = __ballot_sync(0xffffffffu, on);
    if (on) list[n + __popc(m & ((1u << lane) - 1u))] = (uint16_t)J;
    n += __popc(m);
  }
  if (lane == 0) *cnt = n;
}
// next(J): the first listed index >= J (-1: none); consecutive calls with increasing J
// advance a cursor, a call with J <= the previous result starts a new walk
struct ActiveList {
  const uint16_t* l;
  int n, cur;
  __device__ __forceinline__ int next(int J) {
    if (cur > 0 && (int)l[cur - 1] >= J) cur = 0;
    while (cur < n && (int)l[cur] < J) ++cur;
    return cur < n ? (int)l[cur++] : -1;
  }
};

enum AlphaKind { AK15 = 0, AK2 = 1, AK125 = 2, AKGEN = 3 };

// fp16 operands for the gradient products (decided on the device, per launch):
//  dv_ok: dV = P^T dO with P (in [0, 1]) and dO in fp16 -- max|dO| fits fp16;
//  ds_ok: dQ = dS K and dK = dS^T Q with sigma dS, K, Q in fp16 -- alpha <= 2
//         (u = p^(2-alpha) <= 1), max|Q|, max|K| fit fp16, and
//         |dS| <= 2 d max|dO| max|V| (|dp|, |delta| <= d max|dO| max|V|) so the
//         power-of-two sigma puts every sigma dS within 2^15; results are
//         scaled back by 1/sigma (exact).
//  The fp16 copies of dO, Q and K are scaled by powers of two (f16_pow2_scale,
//  tc_common.cuh) so small operands do not underflow; inv_* undo them.
//  One plan per head (a head's results never depend on the other heads).
struct F16Plan {
  int dv_ok, ds_ok;
  float sigma, inv_sigma;
  float inv_do, inv_q, inv_k;
  int pad;
};

// KahanF: tc_common.cuh

// u = p^(2-alpha) = t^(e0-1) for t > 0, else 0; p = t^e0
template <int AK>
__device__ __forceinline__ void pu_of(float t, float e0f, float e1f, float& p, float& u) {
  const float tp = fmaxf(t, 0.f);
  if constexpr (AK == AK15) {
    p = tp * tp;
    u = tp;
  } else if constexpr (AK == AK2) {
    p = tp;
    u = __saturatef(tp * 0x1p126f);  // 1 for t > 0
  } else if constexpr (AK == AK125) {
    const float t2 = tp * tp;
    u = t2 * tp;
    p = u * tp;
  } else {
    if (tp > 0.f) {
      const float l = __log2f(tp);
      p = exp2f(e0f * l);
      u = exp2f(e1f * l);
    } else {
      p = 0.f;
      u = 0.f;
    }
  }
}

// dS = u (dp - delta) of one 32-key chunk, split into bf16 hi + lo pairs.
// MASKED: keys i > lim (causal diagonal) are outside the row's support.
template <int AK, bool MASKED, bool F16S = false>
__device__ __forceinline__ void ds_chunk(const float* s, const float* dp, float A1, float C,
                                         float dl, float e0f, float e1f, int lim, uint32_t* hi,
                                         uint32_t* lo, float sig = 1.f) {
  const float2 A2 = make_float2(A1, A1), C2 = make_float2(C, C), D2 = make_float2(-dl, -dl);
  // F16S: sigma (dp - delta) in one FFMA2; the fp16 dS is sigma dS
  const float2 S2 = make_float2(sig, sig), D2S = make_float2(-sig * dl, -sig * dl);
#pragma unroll
  for (int x = 0; x < 16; ++x) {
    float2 t = __ffma2_rn(A2, make_float2(s[2 * x], s[2 * x + 1]), C2);
    if (MASKED) {
      if (2 * x > lim) t.x = -1.f;
      if (2 * x + 1 > lim) t.y = -1.f;
    }
    float2 u;
    if constexpr (AK == AK15) {
      u = make_float2(fmaxf(t.x, 0.f), fmaxf(t.y, 0.f));
    } else {
      float p;
      pu_of<AK>(t.x, e0f, e1f, p, u.x);
      pu_of<AK>(t.y, e0f, e1f, p, u.y);
    }
    const float2 d = F16S ? __ffma2_rn(make_float2(dp[2 * x], dp[2 * x + 1]), S2, D2S)
                          : __fadd2_rn(make_float2(dp[2 * x], dp[2 * x + 1]), D2);
    const float2 ds = __fmul2_rn(u, d);
    if constexpr (F16S) {
      (void)lo;
      hi[x] = pack_f16x2(ds.x, ds.y);
    } else {
      split_bf16x2(ds.x, ds.y, hi[x], lo[x]);
    }
  }
}

// sum u dp and sum u of one 32-key chunk (delta numerator / denominator).
template <int AK, bool MASKED>
__device__ __forceinline__ void delta_chunk(const float* s, const float* dp, float A1, float C,
                                            float e0f, float e1f, int lim, float& n_out,
                                            float& d_out) {
  const float2 A2 = make_float2(A1, A1), C2 = make_float2(C, C);
  float2 n2a = make_float2(0.f, 0.f), d2a = n2a, n2b = n2a, d2b = n2a;
#pragma unroll
  for (int x = 0; x < 16; ++x) {
    float2 t = __ffma2_rn(A2, make_float2(s[2 * x], s[2 * x + 1]), C2);
    if (MASKED) {
      if (2 * x > lim) t.x = -1.f;
      if (2 * x + 1 > lim) t.y = -1.f;
    }
    float2 u;
    if constexpr (AK == AK15) {
      u = make_float2(fmaxf(t.x, 0.f), fmaxf(t.y, 0.f));
    } else {
      float p;
      pu_of<AK>(t.x, e0f, e1f, p, u.x);
      pu_of<AK>(t.y, e0f, e1f, p, u.y);
    }
    const float2 d = make_float2(dp[2 * x], dp[2 * x + 1]);
    if (x & 1) {
      n2b = __ffma2_rn(u, d, n2b);
      d2b = __fadd2_rn(d2b, u);
    } else {
      n2a = __ffma2_rn(u, d, n2a);
      d2a = __fadd2_rn(d2a, u);
    }
  }
  n_out = (n2a.x + n2a.y) + (n2b.x + n2b.y);
  d_out = (d2a.x + d2a.y) + (d2b.x + d2b.y);
}

// Key-major (dK/dV) chunk: 32 queries of one key.  P^T = t^e0 and
// dS^T = u (dp - delta_q), both split into bf16 hi + lo pairs.  rc[q] =
// (C_q, delta_q) from shared memory.  MASKED: queries q < lim (above the causal
// diagonal for this key) are outside the support.
template <int AK, bool MASKED, bool F16P = false, bool F16S = false>
__device__ __forceinline__ void pds_chunk(const float* s, const float* dp, const float2* rc,
                                          float A1, float e0f, float e1f, int lim, uint32_t* ph,
                                          uint32_t* pl, uint32_t* dh, uint32_t* dl, float sig = 1.f) {
  const float2 A2 = make_float2(A1, A1);
#pragma unroll
  for (int x = 0; x < 16; ++x) {
    const float4 c = reinterpret_cast<const float4*>(rc)[x];  // (C, delta) of queries 2x, 2x+1
    float2 t = __ffma2_rn(A2, make_float2(s[2 * x], s[2 * x + 1]), make_float2(c.x, c.z));
    if (MASKED) {
      if (2 * x < lim) t.x = -1.f;
      if (2 * x + 1 < lim) t.y = -1.f;
    }
    float2 p, u;
    if constexpr (AK == AK15) {
      u = make_float2(fmaxf(t.x, 0.f), fmaxf(t.y, 0.f));
      p = __fmul2_rn(u, u);
    } else {
      pu_of<AK>(t.x, e0f, e1f, p.x, u.x);
      pu_of<AK>(t.y, e0f, e1f, p.y, u.y);
    }
    const float2 d = __fadd2_rn(make_float2(dp[2 * x], dp[2 * x + 1]), make_float2(-c.y, -c.w));
    const float2 ds = __fmul2_rn(u, d);
    if constexpr (F16P) {
      ph[x] = pack_f16x2(p.x, p.y);  // p in [0, 1]: fp16 keeps 11 bits (bf16 hi + lo: ~16)
    } else {
      split_bf16x2(p.x, p.y, ph[x], pl[x]);
    }
    if constexpr (F16S) {
      const float2 dss = __fmul2_rn(ds, make_float2(sig, sig));
      dh[x] = pack_f16x2(dss.x, dss.y);
    } else {
      split_bf16x2(ds.x, ds.y, dh[x], dl[x]);
    }
  }
}

// ================================================================== delta
// Query-major delta kernel: 256 rows per CTA (two M=128 row groups), keys in
// 128-key tiles so S = Q K^T and dP = dO V^T are SS MMAs with N=128 (full
// tensor rate from shared memory).  TMEM: row group g owns S_g (cols 256g ..)
// and dP_g (cols 256g + 128 ..), single-buffered; the two groups ping-pong so
// one group's epilogue overlaps the other group's MMAs.  Each 64-key half of a
// tile is one reference block: only set mask blocks contribute (the
// reference's for_each_set, attention.cpp:420-444).
constexpr int DBN = 128;  // keys per tile (delta, dQ)

template <int D>
struct DeltaSmem {
  static constexpr int QB = BM * D * 2;
  static constexpr int TILE = DBN * D * 2;
  static constexpr int NST = D == 128 ? 3 : 6;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_DO = OFF_Q + QB;
  static constexpr int OFF_RING = OFF_DO + QB;
  static constexpr int OFF_BAR = OFF_RING + NST * TILE;
  static constexpr int OFF_MISC = OFF_BAR + 32 * 8;
  static constexpr int OFF_RED = OFF_RING;  // [256] x 2 f64 half-1 partials (ring drained)
  static constexpr int OFF_MASK = OFF_MISC + 64;
  __host__ __device__ static int off_list(int wpr) { return OFF_MASK + 4 * wpr * 4; }
  // + the compacted nonzero-tile list (<= 16 wpr u16)
  static size_t bytes(int wpr) { return 1024 + off_list(wpr) + 32 * wpr + 64; }
};

constexpr int kDeltaThreads = 512 + 64;  // 16 epilogue warps, producer, MMA issuer

template <int D, int AK>
__global__ void __launch_bounds__(kDeltaThreads, 1)
    tc_delta_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                    const BwdArgs a) {
  using L = DeltaSmem<D>;
  constexpr int NST = L::NST;
  constexpr int NCH = D / 64;
  const Geom& g = a.g;
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned base that stays in the shared address space (LDS/STS, not
  // generic LD/ST, for every access through it)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sDO = smem + L::OFF_DO;
  uint8_t* sRing = smem + L::OFF_RING;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full = bars;              // [NST]
  uint64_t* empty = bars + NST;       // [NST]
  uint64_t* s_full = bars + 2 * NST;  // [2 row groups]
  uint64_t* s_free = s_full + 2;      // [2]
  uint64_t* q_full = s_free + 2;
  volatile uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::OFF_MISC);
  double* sRed = reinterpret_cast<double*>(smem + L::OFF_RED);
  uint32_t* smask = reinterpret_cast<uint32_t*>(smem + L::OFF_MASK);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wpr = g.wpr;
  // head-major (K/V L2-resident), heaviest causal row blocks first within a head
  const int bh = blockIdx.x / a.ncta_rows;
  const int row0 = (a.ncta_rows - 1 - (int)(blockIdx.x % a.ncta_rows)) * BM;
  const int nkt = g.m / DBN;
  const int jmax = g.causal ? (row0 + BM - 1) / DBN : nkt - 1;

  // delta from the support lists: only the 256-row blocks the forward flagged run here
  if (a.supp_skip && a.supp_skip[((size_t)bh * g.n + row0) / BM] == 0u) return;
  rows_from_lists(smask, 4, a, bh, row0 / 64, tid, kDeltaThreads);
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);
    }
    mbar_init(q_full, 1);
    fence_barrier_init();
  }
  if (warp == 16) tmem_alloc(const_cast<uint32_t*>(s_tmem), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  // bits of reference blocks (row block rb of this CTA, key blocks 2J, 2J+1)
  auto bits2 = [&](int rb, int J) -> uint32_t {
    return (smask[rb * wpr + ((2 * J) >> 5)] >> ((2 * J) & 31)) & 3u;
  };
  auto rg_active = [&](int rg, int J) -> bool { return (bits2(2 * rg, J) | bits2(2 * rg + 1, J)) != 0; };
  // the CTA's nonzero 128-key tiles, compacted once
  uint16_t* sList = reinterpret_cast<uint16_t*>(smem + L::off_list(wpr));
  volatile uint32_t* sListN = reinterpret_cast<volatile uint32_t*>(smem + L::OFF_MISC) + 2;
  if (warp == 0)
    compact_active(sList, sListN, jmax, lane, [&](int J) -> bool { return rg_active(0, J) || rg_active(1, J); });
  __syncthreads();
  ActiveList walk{sList, (int)*sListN, 0};
  auto next_active = [&](int J) -> int { return walk.next(J); };

  if (warp == 16) {  // TMA producer
    const bool leader = elect_one_sync();
    const int qrow = bh * g.n + row0;
    if (leader) mbar_expect_tx(q_full, 2 * L::QB);
    for (int c = 0; c < NCH; ++c) {
      if (leader) tma_load_2d(sQ + c * BM * 128, &tm_q, q_full, c * 64, qrow);
      if (leader) tma_load_2d(sDO + c * BM * 128, &tm_do, q_full, c * 64, qrow);
    }
    uint32_t r = 0;
    auto load = [&](const CUtensorMap* tm, int row) {
      const uint32_t st = r % NST, ph = (r / NST) & 1;
      mbar_wait(&empty[st], ph ^ 1);
      if (leader) mbar_expect_tx(&full[st], L::TILE);
      for (int c = 0; c < NCH; ++c)
        if (leader) tma_load_2d(sRing + st * L::TILE + c * DBN * 128, tm, &full[st], c * 64, row);
      ++r;
    };
    const int krow0 = bh * g.m;
    for (int J = next_active(0); J >= 0; J = next_active(J + 1)) {
      load(&tm_k, krow0 + J * DBN);
      load(&tm_v, krow0 + J * DBN);
    }
  } else if (warp == 17) {  // MMA issuer (highest warp id: scheduler priority)
    const bool leader = elect_one_sync();
    constexpr uint32_t IDESC_S = idesc_bf16_f32(128, DBN, false, false);
    const uint32_t q_addr = smem_u32(sQ), do_addr = smem_u32(sDO), ring_addr = smem_u32(sRing);
    mbar_wait(q_full, 0);
    tc_fence_after();
    uint32_t r = 0, uses[2] = {0, 0};
    // loop-invariant descriptors (row group rg at +128 rows = 16 KB = +1024 in the field)
    uint64_t dQd[NCH], dDOd[NCH], dR[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      dQd[c] = desc_kmajor(q_addr + c * BM * 128);
      dDOd[c] = desc_kmajor(do_addr + c * BM * 128);
      dR[c] = desc_kmajor(ring_addr + c * DBN * 128);
    }
    constexpr uint32_t kTileF = (uint32_t)L::TILE >> 4;
    for (int J = next_active(0); J >= 0; J = next_active(J + 1)) {
      const uint32_t kst = r % NST, vst = (r + 1) % NST;
      mbar_wait(&full[kst], (r / NST) & 1);
      mbar_wait(&full[vst], ((r + 1) / NST) & 1);
      tc_fence_after();
      const bool act1 = rg_active(1, J);
      const uint64_t ko = (uint64_t)(kst * kTileF), vo = (uint64_t)(vst * kTileF);
#pragma unroll
      for (int rg = 0; rg < 2; ++rg) {
        if (!rg_active(rg, J)) continue;
        mbar_wait(&s_free[rg], (uses[rg] & 1) ^ 1);
        tc_fence_after();
        const uint32_t sc = tmem + rg * 256;
        const uint64_t ro = (uint64_t)(rg * 1024);
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (leader)
              umma_bf16(sc, dQd[c] + ro + (uint64_t)(2 * k), dR[c] + ko + (uint64_t)(2 * k),
                        IDESC_S, (c | k) != 0);
        // K_J's last reader issued: free its slot early (the next item, V_{J+1}, refills it)
        if (rg == 1 || !act1)
          if (leader) umma_commit(&empty[kst]);
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (leader)
              umma_bf16(sc + 128, dDOd[c] + ro + (uint64_t)(2 * k), dR[c] + vo + (uint64_t)(2 * k),
                        IDESC_S, (c | k) != 0);
        if (leader) umma_commit(&s_full[rg]);
        ++uses[rg];
      }
      if (leader) umma_commit(&empty[vst]);
      r += 2;
    }
  } else if (warp < 16) {  // epilogue (warp % 4 = TMEM lane quarter)
    const int ew = warp;             // 0..15
    const int rg = ew >> 3;              // row group
    const int half = (ew >> 2) & 1;      // keys 64*half .. +63 of each tile
    const int lq = warp & 3;             // TMEM lane quarter
    const int e = rg * 128 + lq * 32 + lane;
    const int rb = e >> 6;
    const int grow = row0 + e;
    // last key this row sees: the causal diagonal and the problem's real keys
    const int klim = g.causal ? min(grow, g.m_valid - 1) : g.m_valid - 1;
    const size_t orow = (size_t)bh * g.n + grow;
    const uint32_t tl = tmem + ((uint32_t)(lq * 32) << 16) + rg * 256 + half * 64;
    const float A1 = a.A1;
    const double B = 1.0 - (g.alpha - 1.0) * a.row_max[orow];
    const float C = (float)(B - a.tau[orow]);
    KahanF num, den;  // fp32 compensated sums of the fp32 chunk partials (no FP64 pipe)
    uint32_t uses = 0;
    for (int J = next_active(0); J >= 0; J = next_active(J + 1)) {
      if (!rg_active(rg, J)) continue;
      mbar_wait(&s_full[rg], uses & 1);
      ++uses;
      tc_fence_after();
      const bool mine = (bits2(rb, J) >> half) & 1u;  // the reference visits set blocks only
      const int k0 = J * DBN + half * 64;
      float s[32], dp[32];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        tmem_ld32(tl + c * 32, s);
        tmem_ld32(tl + 128 + c * 32, dp);
        tmem_wait_ld();
        if (c == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_free[rg]);
        }
        if (mine) {
          const int c0 = k0 + 32 * c;
          float n32, d32;
          if (c0 + 31 > klim)
            delta_chunk<AK, true>(s, dp, A1, C, a.e0f, a.e1f, klim - c0, n32, d32);
          else
            delta_chunk<AK, false>(s, dp, A1, C, a.e0f, a.e1f, 0, n32, d32);
          num.add(n32);
          den.add(d32);
        }
      }
    }
    // every epilogue thread has passed its last s_full wait: all MMAs (and ring
    // reads) are complete, so the ring can hold the half-1 partials
    bar_sync(1, 512);
    if (half == 1) {
      sRed[2 * e] = num.get();
      sRed[2 * e + 1] = den.get();
    }
    bar_sync(1, 512);
    if (half == 0) {
      const double nm = num.get() + sRed[2 * e];
      const double dn = den.get() + sRed[2 * e + 1];
      const double dlt = dn > 0.0 ? nm / dn : 0.0;
      a.delta[orow] = dlt;
      a.rowc[orow] = make_float2(C, (float)dlt);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 16) tmem_dealloc(tmem, 512);
}

// ============================================================ delta (pairs)
// CTA-pair variant (cta_group::2, d = 128): each CTA keeps its 256 rows (two
// row groups); the leader's M = 256 MMAs cover row group g of both CTAs, with
// each SM supplying half of the K_J / V_J tile (keys 64r..64r+63).
template <int D>
struct Delta2Smem {
  static_assert(D == 128, "pair delta kernel: d = 128");
  static constexpr int QB = BM * D * 2;
  static constexpr int HB = 64 * D * 2;  // 64 keys x d
  static constexpr int NST = 5;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_DO = OFF_Q + QB;
  static constexpr int OFF_RING = OFF_DO + QB;
  static constexpr int OFF_BAR = OFF_RING + NST * HB;
  static constexpr int OFF_MISC = OFF_BAR + 32 * 8;
  static constexpr int OFF_RED = OFF_RING;  // [256] x 2 f64 half-1 partials (ring drained)
  static constexpr int OFF_MASK = OFF_MISC + 64;
  __host__ __device__ static int off_list(int wpr) { return OFF_MASK + 8 * wpr * 4; }
  // + the compacted nonzero-tile list (<= 16 wpr u16)
  static size_t bytes(int wpr) { return 1024 + off_list(wpr) + 32 * wpr + 64; }
};

template <int D, int AK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kDeltaThreads, 1)
    tc_delta2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kh,
                     const __grid_constant__ CUtensorMap tm_vh, const __grid_constant__ CUtensorMap tm_do,
                     const BwdArgs a) {
  using L = Delta2Smem<D>;
  constexpr int NST = L::NST;
  constexpr int NCH = D / 64;
  const Geom& g = a.g;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sDO = smem + L::OFF_DO;
  uint8_t* sRing = smem + L::OFF_RING;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full = bars;              // [NST] leader
  uint64_t* empty = bars + NST;       // [NST] each CTA
  uint64_t* s_full = bars + 2 * NST;  // [2 rg] each CTA
  uint64_t* s_free = s_full + 2;      // [2 rg] leader, 16 warps
  uint64_t* q_full = s_free + 2;      // leader
  volatile uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::OFF_MISC);
  double* sRed = reinterpret_cast<double*>(smem + L::OFF_RED);
  uint32_t* smask = reinterpret_cast<uint32_t*>(smem + L::OFF_MASK);  // [8][wpr]: the pair's row blocks

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_ctarank();
  const bool lead_cta = rank == 0;
  const int wpr = g.wpr;
  const int npair = a.ncta_rows / 2;
  const int pair = (int)(blockIdx.x >> 1);
  const int bh = pair / npair;
  const int prow0 = (npair - 1 - pair % npair) * 2 * BM;  // heaviest pairs first
  const int row0 = prow0 + (int)rank * BM;
  const int nkt = g.m / DBN;
  const int jmax = g.causal ? (prow0 + 2 * BM - 1) / DBN : nkt - 1;

  if (a.supp_skip) {  // the pair's two 256-row blocks (both CTAs decide alike)
    const size_t b0 = ((size_t)bh * g.n + prow0) / BM;
    if (a.supp_skip[b0] == 0u && a.supp_skip[b0 + 1] == 0u) return;
  }
  rows_from_lists(smask, 8, a, bh, prow0 / 64, tid, kDeltaThreads);
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 16);
    }
    mbar_init(q_full, 1);
    fence_barrier_init();
  }
  if (warp == 16) tmem_alloc_2sm(const_cast<uint32_t*>(s_tmem), 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  // pair row block pb (0..7: CTA pb/4, row group (pb/2)&1), key blocks 2J, 2J+1
  auto bits2 = [&](int pb, int J) -> uint32_t {
    return (smask[pb * wpr + ((2 * J) >> 5)] >> ((2 * J) & 31)) & 3u;
  };
  auto rg_active = [&](int rg, int J) -> bool {  // row group rg of either CTA
    return (bits2(2 * rg, J) | bits2(2 * rg + 1, J) | bits2(4 + 2 * rg, J) | bits2(5 + 2 * rg, J)) != 0;
  };
  // the CTA's nonzero 128-key tiles, compacted once
  uint16_t* sList = reinterpret_cast<uint16_t*>(smem + L::off_list(wpr));
  volatile uint32_t* sListN = reinterpret_cast<volatile uint32_t*>(smem + L::OFF_MISC) + 2;
  if (warp == 0)
    compact_active(sList, sListN, jmax, lane, [&](int J) -> bool { return rg_active(0, J) || rg_active(1, J); });
  __syncthreads();
  ActiveList walk{sList, (int)*sListN, 0};
  auto next_active = [&](int J) -> int { return walk.next(J); };

  if (warp == 16) {  // TMA producer (both CTAs)
    const bool leader = elect_one_sync();
    const int qrow = bh * g.n + row0;
    if (lead_cta && leader) mbar_expect_tx(q_full, 2 * 2 * L::QB);
    for (int c = 0; c < NCH; ++c) {
      if (leader) tma_load_2d_2sm(sQ + c * BM * 128, &tm_q, q_full, c * 64, qrow);
      if (leader) tma_load_2d_2sm(sDO + c * BM * 128, &tm_do, q_full, c * 64, qrow);
    }
    uint32_t r = 0;
    auto load = [&](const CUtensorMap* tm, int row) {
      const uint32_t st = r % NST, ph = (r / NST) & 1;
      mbar_wait(&empty[st], ph ^ 1);
      if (lead_cta && leader) mbar_expect_tx(&full[st], 2 * L::HB);
      for (int c = 0; c < NCH; ++c)
        if (leader) tma_load_2d_2sm(sRing + st * L::HB + c * 64 * 128, tm, &full[st], c * 64, row);
      ++r;
    };
    const int krow0 = bh * g.m + 64 * (int)rank;
    for (int J = next_active(0); J >= 0; J = next_active(J + 1)) {
      load(&tm_kh, krow0 + J * DBN);
      load(&tm_vh, krow0 + J * DBN);
    }
  } else if (warp == 17) {  // MMA issuer: pair leader only
    if (lead_cta) {
      const bool leader = elect_one_sync();
      constexpr uint32_t IDESC_S = idesc_bf16_f32(256, DBN, false, false);
      const uint32_t q_addr = smem_u32(sQ), do_addr = smem_u32(sDO), ring_addr = smem_u32(sRing);
      uint64_t dQd[NCH], dDOd[NCH], dR[NCH];
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        dQd[c] = desc_kmajor(q_addr + c * BM * 128);
        dDOd[c] = desc_kmajor(do_addr + c * BM * 128);
        dR[c] = desc_kmajor(ring_addr + c * 64 * 128);
      }
      constexpr uint32_t kHF = (uint32_t)L::HB >> 4;
      mbar_wait(q_full, 0);
      tc_fence_after();
      uint32_t r = 0, uses[2] = {0, 0};
      for (int J = next_active(0); J >= 0; J = next_active(J + 1)) {
        const uint32_t kst = r % NST, vst = (r + 1) % NST;
        mbar_wait(&full[kst], (r / NST) & 1);
        mbar_wait(&full[vst], ((r + 1) / NST) & 1);
        tc_fence_after();
        const bool act1 = rg_active(1, J);
        const uint64_t ko = (uint64_t)(kst * kHF), vo = (uint64_t)(vst * kHF);
#pragma unroll
        for (int rg = 0; rg < 2; ++rg) {
          if (!rg_active(rg, J)) continue;
          mbar_wait(&s_free[rg], (uses[rg] & 1) ^ 1);
          tc_fence_after();
          const uint32_t sc = tmem + rg * 256;
          const uint64_t ro = (uint64_t)(rg * 1024);  // +128 rows (16 KB) in the address field
#pragma unroll
          for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (leader)
                umma2_bf16(sc, dQd[c] + ro + (uint64_t)(2 * k), dR[c] + ko + (uint64_t)(2 * k),
                           IDESC_S, (c | k) != 0);
          if (rg == 1 || !act1)
            if (leader) umma2_commit_mc(&empty[kst]);
#pragma unroll
          for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (leader)
                umma2_bf16(sc + 128, dDOd[c] + ro + (uint64_t)(2 * k), dR[c] + vo + (uint64_t)(2 * k),
                           IDESC_S, (c | k) != 0);
          if (leader) umma2_commit_mc(&s_full[rg]);
          ++uses[rg];
        }
        if (leader) umma2_commit_mc(&empty[vst]);
        r += 2;
      }
    }
  } else if (warp < 16) {  // epilogue
    const int ew = warp;
    const int rg = ew >> 3;
    const int half = (ew >> 2) & 1;
    const int lq = warp & 3;
    const int e = rg * 128 + lq * 32 + lane;
    const int rb = e >> 6;                 // own row block 0..3
    const int pb = 4 * (int)rank + rb;     // pair row block 0..7
    const int grow = row0 + e;
    // last key this row sees: the causal diagonal and the problem's real keys
    const int klim = g.causal ? min(grow, g.m_valid - 1) : g.m_valid - 1;
    const size_t orow = (size_t)bh * g.n + grow;
    const uint32_t tl = tmem + ((uint32_t)(lq * 32) << 16) + rg * 256 + half * 64;
    const float A1 = a.A1;
    const double B = 1.0 - (g.alpha - 1.0) * a.row_max[orow];
    const float C = (float)(B - a.tau[orow]);
    const uint32_t s_free_c = mapa_shared(smem_u32(&s_free[rg]), 0);
    KahanF num, den;  // fp32 compensated sums of the fp32 chunk partials (no FP64 pipe)
    uint32_t uses = 0;
    for (int J = next_active(0); J >= 0; J = next_active(J + 1)) {
      if (!rg_active(rg, J)) continue;
      mbar_wait(&s_full[rg], uses & 1);
      ++uses;
      tc_fence_after();
      const bool mine = (bits2(pb, J) >> half) & 1u;
      const int k0 = J * DBN + half * 64;
      float s[32], dp[32];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        tmem_ld32(tl + c * 32, s);
        tmem_ld32(tl + 128 + c * 32, dp);
        tmem_wait_ld();
        if (c == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(s_free_c);
        }
        if (mine) {
          const int c0 = k0 + 32 * c;
          float n32, d32;
          if (c0 + 31 > klim)
            delta_chunk<AK, true>(s, dp, A1, C, a.e0f, a.e1f, klim - c0, n32, d32);
          else
            delta_chunk<AK, false>(s, dp, A1, C, a.e0f, a.e1f, 0, n32, d32);
          num.add(n32);
          den.add(d32);
        }
      }
    }
    bar_sync(1, 512);
    if (half == 1) {
      sRed[2 * e] = num.get();
      sRed[2 * e + 1] = den.get();
    }
    bar_sync(1, 512);
    if (half == 0) {
      const double nm = num.get() + sRed[2 * e];
      const double dn = den.get() + sRed[2 * e + 1];
      const double dlt = dn > 0.0 ? nm / dn : 0.0;
      a.delta[orow] = dlt;
      a.rowc[orow] = make_float2(C, (float)dlt);
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 16) tmem_dealloc_2sm(tmem, 512);
}

// ============================================================ delta (pairs, 128 rows)
// CTA-pair variant with 128 query rows per CTA (256 per pair): the leader's
// M = 256 MMAs cover both CTAs' rows, each SM holds half of every K_J / V_J
// tile, and with one row group per CTA the TMEM holds TWO S/dP buffers, so the
// MMAs of tile J+1 never wait for the epilogue of tile J (the 256-row kernels
// single-buffer S/dP per row group).  16 epilogue warps: TMEM lane quarter x
// 32-key column quarter of the 128-key tile.
template <int D>
struct Delta3Smem {
  static_assert(D == 128, "pair delta kernel: d = 128");
  static constexpr int QB = 128 * D * 2;
  static constexpr int HB = 64 * D * 2;  // 64 keys x d
  static constexpr int NST = 8;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_DO = OFF_Q + QB;
  static constexpr int OFF_RING = OFF_DO + QB;
  static constexpr int OFF_BAR = OFF_RING + NST * HB;
  static constexpr int OFF_MISC = OFF_BAR + 32 * 8;
  static constexpr int OFF_RED = OFF_RING;  // [4][128] x 2 f64 partials (ring drained)
  static constexpr int OFF_MASK = OFF_MISC + 64;
  __host__ __device__ static int off_list(int wpr) { return OFF_MASK + 4 * wpr * 4; }
  // + the compacted nonzero-tile list (<= 16 wpr u16)
  static size_t bytes(int wpr) { return 1024 + off_list(wpr) + 32 * wpr + 64; }
};

template <int D, int AK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kDeltaThreads, 1)
    tc_delta3_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kh,
                     const __grid_constant__ CUtensorMap tm_vh, const __grid_constant__ CUtensorMap tm_do,
                     const BwdArgs a) {
  using L = Delta3Smem<D>;
  constexpr int NST = L::NST;
  constexpr int NCH = D / 64;
  constexpr int QR = 128;  // query rows per CTA
  const Geom& g = a.g;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sDO = smem + L::OFF_DO;
  uint8_t* sRing = smem + L::OFF_RING;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full = bars;              // [NST] leader
  uint64_t* empty = bars + NST;       // [NST] each CTA
  uint64_t* s_full = bars + 2 * NST;  // [2 buffers] each CTA
  uint64_t* s_free = s_full + 2;      // [2 buffers] leader, 32 warps
  uint64_t* q_full = s_free + 2;      // leader
  volatile uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::OFF_MISC);
  double* sRed = reinterpret_cast<double*>(smem + L::OFF_RED);
  uint32_t* smask = reinterpret_cast<uint32_t*>(smem + L::OFF_MASK);  // [4][wpr]: the pair's row blocks

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_ctarank();
  const bool lead_cta = rank == 0;
  const int wpr = g.wpr;
  const int npair = g.n / (2 * QR);
  const int pair = (int)(blockIdx.x >> 1);
  const int bh = pair / npair;
  const int prow0 = (npair - 1 - pair % npair) * 2 * QR;  // heaviest pairs first
  const int row0 = prow0 + (int)rank * QR;
  const int nkt = g.m / DBN;
  const int jmax = g.causal ? (prow0 + 2 * QR - 1) / DBN : nkt - 1;

  // the pair's 256 rows: one forward block (both CTAs decide alike)
  if (a.supp_skip && a.supp_skip[((size_t)bh * g.n + prow0) / 256] == 0u) return;
  rows_from_lists(smask, 4, a, bh, prow0 / 64, tid, kDeltaThreads);
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 32);
    }
    mbar_init(q_full, 1);
    fence_barrier_init();
  }
  if (warp == 16) tmem_alloc_2sm(const_cast<uint32_t*>(s_tmem), 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  // pair row block pb (0..3: CTA pb/2), key blocks 2J, 2J+1
  auto bits2 = [&](int pb, int J) -> uint32_t {
    return (smask[pb * wpr + ((2 * J) >> 5)] >> ((2 * J) & 31)) & 3u;
  };
  // the CTA's nonzero 128-key tiles, compacted once
  uint16_t* sList = reinterpret_cast<uint16_t*>(smem + L::off_list(wpr));
  volatile uint32_t* sListN = reinterpret_cast<volatile uint32_t*>(smem + L::OFF_MISC) + 2;
  if (warp == 0)
    compact_active(sList, sListN, jmax, lane, [&](int J) -> bool { return bits2(0, J) | bits2(1, J) | bits2(2, J) | bits2(3, J); });
  __syncthreads();
  ActiveList walk{sList, (int)*sListN, 0};
  auto next_active = [&](int J) -> int { return walk.next(J); };

  if (warp == 16) {  // TMA producer (both CTAs)
    const bool leader = elect_one_sync();
    const int qrow = bh * g.n + row0;
    if (lead_cta && leader) mbar_expect_tx(q_full, 2 * 2 * L::QB);
    for (int c = 0; c < NCH; ++c) {
      if (leader) tma_load_2d_2sm(sQ + c * QR * 128, &tm_q, q_full, c * 64, qrow);
      if (leader) tma_load_2d_2sm(sDO + c * QR * 128, &tm_do, q_full, c * 64, qrow);
    }
    uint32_t r = 0;
    auto load = [&](const CUtensorMap* tm, int row) {
      const uint32_t st = r % NST, ph = (r / NST) & 1;
      mbar_wait(&empty[st], ph ^ 1);
      if (lead_cta && leader) mbar_expect_tx(&full[st], 2 * L::HB);
      for (int c = 0; c < NCH; ++c)
        if (leader) tma_load_2d_2sm(sRing + st * L::HB + c * 64 * 128, tm, &full[st], c * 64, row);
      ++r;
    };
    const int krow0 = bh * g.m + 64 * (int)rank;
    for (int J = next_active(0); J >= 0; J = next_active(J + 1)) {
      load(&tm_kh, krow0 + J * DBN);
      load(&tm_vh, krow0 + J * DBN);
    }
  } else if (warp == 17) {  // MMA issuer: pair leader only
    if (lead_cta) {
      const bool leader = elect_one_sync();
      constexpr uint32_t IDESC_S = idesc_bf16_f32(256, DBN, false, false);
      const uint32_t q_addr = smem_u32(sQ), do_addr = smem_u32(sDO), ring_addr = smem_u32(sRing);
      uint64_t dQd[NCH], dDOd[NCH], dR[NCH];
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        dQd[c] = desc_kmajor(q_addr + c * QR * 128);
        dDOd[c] = desc_kmajor(do_addr + c * QR * 128);
        dR[c] = desc_kmajor(ring_addr + c * 64 * 128);
      }
      constexpr uint32_t kHF = (uint32_t)L::HB >> 4;
      mbar_wait(q_full, 0);
      tc_fence_after();
      uint32_t r = 0, t = 0;
      for (int J = next_active(0); J >= 0; J = next_active(J + 1), ++t) {
        const uint32_t kst = r % NST, vst = (r + 1) % NST, b = t & 1;
        mbar_wait(&full[kst], (r / NST) & 1);
        mbar_wait(&s_free[b], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint64_t ko = (uint64_t)(kst * kHF), vo = (uint64_t)(vst * kHF);
        const uint32_t sc = tmem + b * 256;
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (leader)
              umma2_bf16(sc, dQd[c] + (uint64_t)(2 * k), dR[c] + ko + (uint64_t)(2 * k), IDESC_S,
                         (c | k) != 0);
        if (leader) umma2_commit_mc(&empty[kst]);
        mbar_wait(&full[vst], ((r + 1) / NST) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (leader)
              umma2_bf16(sc + 128, dDOd[c] + (uint64_t)(2 * k), dR[c] + vo + (uint64_t)(2 * k),
                         IDESC_S, (c | k) != 0);
        if (leader) umma2_commit_mc(&s_full[b]);
        if (leader) umma2_commit_mc(&empty[vst]);
        r += 2;
      }
    }
  } else if (warp < 16) {  // epilogue
    const int lq = warp & 3;              // TMEM lane quarter
    const int cq = warp >> 2;             // keys 32 cq .. +31 of each 128-key tile
    const int e = lq * 32 + lane;         // local row 0..127
    const int pb = 2 * (int)rank + (e >> 6);  // pair row block 0..3
    const int grow = row0 + e;
    // last key this row sees: the causal diagonal and the problem's real keys
    const int klim = g.causal ? min(grow, g.m_valid - 1) : g.m_valid - 1;
    const size_t orow = (size_t)bh * g.n + grow;
    const uint32_t tl = tmem + ((uint32_t)(lq * 32) << 16) + cq * 32;
    const float A1 = a.A1;
    const double B = 1.0 - (g.alpha - 1.0) * a.row_max[orow];
    const float C = (float)(B - a.tau[orow]);
    const uint32_t s_free_c0 = mapa_shared(smem_u32(&s_free[0]), 0);
    const uint32_t s_free_c1 = mapa_shared(smem_u32(&s_free[1]), 0);
    KahanF num, den;  // fp32 compensated sums of the fp32 chunk partials (no FP64 pipe)
    uint32_t t = 0;
    for (int J = next_active(0); J >= 0; J = next_active(J + 1), ++t) {
      const uint32_t b = t & 1;
      mbar_wait(&s_full[b], (t >> 1) & 1);
      tc_fence_after();
      float s[32], dp[32];
      tmem_ld32(tl + b * 256, s);
      tmem_ld32(tl + b * 256 + 128, dp);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(b ? s_free_c1 : s_free_c0);
      if ((bits2(pb, J) >> (cq >> 1)) & 1u) {  // the reference visits set blocks only
        const int c0 = J * DBN + 32 * cq;
        float n32, d32;
        if (c0 + 31 > klim)
          delta_chunk<AK, true>(s, dp, A1, C, a.e0f, a.e1f, klim - c0, n32, d32);
        else
          delta_chunk<AK, false>(s, dp, A1, C, a.e0f, a.e1f, 0, n32, d32);
        num.add(n32);
        den.add(d32);
      }
    }
    // every epilogue thread has passed its last s_full wait: the pair's MMAs
    // reading this CTA's ring are complete, so the ring can hold the partials
    bar_sync(1, 512);
    sRed[(cq * 128 + e) * 2] = num.get();
    sRed[(cq * 128 + e) * 2 + 1] = den.get();
    bar_sync(1, 512);
    if (cq == 0) {
      double nm = 0.0, dn = 0.0;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        nm += sRed[(q4 * 128 + e) * 2];
        dn += sRed[(q4 * 128 + e) * 2 + 1];
      }
      const double dlt = dn > 0.0 ? nm / dn : 0.0;
      a.delta[orow] = dlt;
      a.rowc[orow] = make_float2(C, (float)dlt);
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 16) tmem_dealloc_2sm(tmem, 512);
}

// ===================================================================== dQ
// Query-major dQ kernel: 128 rows per CTA, 128-key tiles.  Per tile J:
//   S_J = Q K_J^T (SS, N=128) into S[J&1], dP_J = dO V_J^T into dP,
//   dS = u (dp - delta) split into bf16 hi + lo and written back over S[J&1]
//   (tcgen05.st), then dQ += dS_hi K_J + dS_lo K_J as TS MMAs (A from TMEM, K_J
//   read MN-major from the ring) -- no shared-memory round trip for dS.
// TMEM: S[0] 0..127, S[1] 128..255, dP 256..383, dQ 384..384+D.  The pipe
// order S_J, dP_J, dQ_{J-1} keeps the tensor core busy while the epilogue
// turns tile J into dS (attention.cpp:508-535; one writer per dQ row).
constexpr int QB_DQ = 128;

template <int D>
struct DqSmem {
  static constexpr int QB = QB_DQ * D * 2;
  static constexpr int TILE = DBN * D * 2;
  // K_J stays resident until dQ_J (issued after dP_{J+1}); V_J only until dP_J
  static constexpr int NSK = D == 128 ? 3 : 4;
  static constexpr int NSV = D == 128 ? 2 : 3;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_DO = OFF_Q + QB;
  static constexpr int OFF_KR = OFF_DO + QB;
  static constexpr int OFF_VR = OFF_KR + NSK * TILE;
  static constexpr int OFF_BAR = OFF_VR + NSV * TILE;
  static constexpr int OFF_MISC = OFF_BAR + 40 * 8;
  static constexpr int OFF_MASK = OFF_MISC + 64;
  __host__ __device__ static int off_list(int wpr) { return OFF_MASK + 2 * wpr * 4; }
  // + the compacted nonzero-tile list (<= 16 wpr u16)
  static size_t bytes(int wpr) { return 1024 + off_list(wpr) + 32 * wpr + 64; }
};

template <int D, int AK>
__global__ void __launch_bounds__(kThreads, 1)
    tc_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                 const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                 const BwdArgs a) {
  using L = DqSmem<D>;
  constexpr int NSK = L::NSK, NSV = L::NSV;
  constexpr int NCH = D / 64;
  const Geom& g = a.g;
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned base that stays in the shared address space (LDS/STS, not
  // generic LD/ST, for every access through it)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sDO = smem + L::OFF_DO;
  uint8_t* sK = smem + L::OFF_KR;
  uint8_t* sV = smem + L::OFF_VR;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* kfull = bars;              // [NSK]
  uint64_t* kempty = kfull + NSK;      // [NSK]
  uint64_t* vfull = kempty + NSK;      // [NSV]
  uint64_t* vempty = vfull + NSV;      // [NSV]
  uint64_t* s_full = vempty + NSV;     // [2] S_J and dP_J in TMEM
  uint64_t* ds_full = s_full + 2;      // [2] dS_J written over S[J&1]
  uint64_t* dp_free = ds_full + 2;     // dP consumed
  uint64_t* acc_full = dp_free + 1;
  uint64_t* q_full = acc_full + 1;
  volatile uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::OFF_MISC);
  uint32_t* smask = reinterpret_cast<uint32_t*>(smem + L::OFF_MASK);  // [2][wpr]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncta = g.n / QB_DQ;
  const int bh = blockIdx.x / ncta;  // head-major, heaviest first
  const int row0 = (ncta - 1 - (int)(blockIdx.x % ncta)) * QB_DQ;
  const int nkt = g.m / DBN;
  const int jmax = g.causal ? (row0 + QB_DQ - 1) / DBN : nkt - 1;
  const int wpr = g.wpr;

  if (a.dq_skip && a.dq_skip[bh] == 0u) return;  // dQ from the support lists
  rows_from_lists(smask, 2, a, bh, row0 / 64, tid, kThreads);
  if (tid == 0) {
    for (int i = 0; i < NSK; ++i) {
      mbar_init(&kfull[i], 1);
      mbar_init(&kempty[i], 1);
    }
    for (int i = 0; i < NSV; ++i) {
      mbar_init(&vfull[i], 1);
      mbar_init(&vempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&ds_full[i], 8);
    }
    mbar_init(dp_free, 8);
    mbar_init(acc_full, 1);
    mbar_init(q_full, 1);
    fence_barrier_init();
  }
  if (warp == 8) tmem_alloc(const_cast<uint32_t*>(s_tmem), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  auto bits2 = [&](int rb, int J) -> uint32_t {
    return (smask[rb * wpr + ((2 * J) >> 5)] >> ((2 * J) & 31)) & 3u;
  };
  // the CTA's nonzero 128-key tiles, compacted once
  uint16_t* sList = reinterpret_cast<uint16_t*>(smem + L::off_list(wpr));
  volatile uint32_t* sListN = reinterpret_cast<volatile uint32_t*>(smem + L::OFF_MISC) + 2;
  if (warp == 0)
    compact_active(sList, sListN, jmax, lane, [&](int J) -> bool { return bits2(0, J) | bits2(1, J); });
  __syncthreads();
  ActiveList walk{sList, (int)*sListN, 0};
  auto next_active = [&](int J) -> int { return walk.next(J); };

  if (warp == 8) {  // TMA producer
    const bool leader = elect_one_sync();
    const int qrow = bh * g.n + row0;
    if (leader) mbar_expect_tx(q_full, 2 * L::QB);
    for (int c = 0; c < NCH; ++c) {
      if (leader) tma_load_2d(sQ + c * QB_DQ * 128, &tm_q, q_full, c * 64, qrow);
      if (leader) tma_load_2d(sDO + c * QB_DQ * 128, &tm_do, q_full, c * 64, qrow);
    }
    uint32_t t = 0;
    const int krow0 = bh * g.m;
    for (int J = next_active(0); J >= 0; J = next_active(J + 1), ++t) {
      const uint32_t ks = t % NSK, vs = t % NSV;
      mbar_wait(&kempty[ks], ((t / NSK) & 1) ^ 1);
      if (leader) mbar_expect_tx(&kfull[ks], L::TILE);
      for (int c = 0; c < NCH; ++c)
        if (leader) tma_load_2d(sK + ks * L::TILE + c * DBN * 128, &tm_k, &kfull[ks], c * 64, krow0 + J * DBN);
      mbar_wait(&vempty[vs], ((t / NSV) & 1) ^ 1);
      if (leader) mbar_expect_tx(&vfull[vs], L::TILE);
      for (int c = 0; c < NCH; ++c)
        if (leader) tma_load_2d(sV + vs * L::TILE + c * DBN * 128, &tm_v, &vfull[vs], c * 64, krow0 + J * DBN);
    }
  } else if (warp == 9) {  // MMA issuer (highest warp id: scheduler priority)
    const bool leader = elect_one_sync();
    constexpr uint32_t IDESC_S = idesc_bf16_f32(128, DBN, false, false);
    constexpr uint32_t IDESC_DQ = idesc_bf16_f32(128, D, false, true);
    const uint32_t q_addr = smem_u32(sQ), do_addr = smem_u32(sDO);
    const uint32_t k_addr = smem_u32(sK), v_addr = smem_u32(sV);
    mbar_wait(q_full, 0);
    tc_fence_after();
    uint32_t t = 0;
    bool acc_init = false;
    // loop-invariant descriptors; ring slot s adds s * (TILE >> 4) to the address field
    uint64_t dQd[NCH], dDOd[NCH], dKs[NCH], dVs[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      dQd[c] = desc_kmajor(q_addr + c * QB_DQ * 128);
      dDOd[c] = desc_kmajor(do_addr + c * QB_DQ * 128);
      dKs[c] = desc_kmajor(k_addr + c * DBN * 128);
      dVs[c] = desc_kmajor(v_addr + c * DBN * 128);
    }
    const uint64_t dKmn = desc_mnmajor(k_addr, DBN * 128);
    constexpr uint32_t kTileF = (uint32_t)L::TILE >> 4;
    auto dq_mma = [&](uint32_t tt) {  // dQ += dS_tt K_tt (dS in S[tt&1], K in slot tt % NSK)
      const uint32_t b = tt & 1, ks = tt % NSK;
      mbar_wait(&ds_full[b], (tt >> 1) & 1);
      tc_fence_after();
      const uint64_t bk = dKmn + (uint64_t)(ks * kTileF);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        // keys 16k..16k+15: chunk k>>1 (32 keys) at cols 32(k>>1): hi +8(k&1), lo +16+8(k&1);
        // a 16-key K step of the MN-major operand is 2048 B = +128
        const uint32_t acol = b * 128 + 32 * (k >> 1) + 8 * (k & 1);
        const uint64_t bd = bk + (uint64_t)(128 * k);
        if (leader) umma_bf16_ts(tmem + 384, tmem + acol, bd, IDESC_DQ, (acc_init || k > 0) ? 1u : 0u);
        if (leader) umma_bf16_ts(tmem + 384, tmem + acol + 16, bd, IDESC_DQ, 1u);
      }
      acc_init = true;
      if (leader) umma_commit(&kempty[ks]);
    };
    for (int J = next_active(0); J >= 0; J = next_active(J + 1), ++t) {
      const uint32_t ks = t % NSK, vs = t % NSV, b = t & 1;
      mbar_wait(&kfull[ks], (t / NSK) & 1);
      tc_fence_after();
      // S[b] was last read by dQ_{t-2}, issued earlier (in-order tensor pipe)
      const uint64_t ko = (uint64_t)(ks * kTileF), vo = (uint64_t)(vs * kTileF);
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (leader)
            umma_bf16(tmem + b * 128, dQd[c] + (uint64_t)(2 * k), dKs[c] + ko + (uint64_t)(2 * k),
                      IDESC_S, (c | k) != 0);
      mbar_wait(&vfull[vs], (t / NSV) & 1);
      if (t > 0) mbar_wait(dp_free, (t - 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (leader)
            umma_bf16(tmem + 256, dDOd[c] + (uint64_t)(2 * k), dVs[c] + vo + (uint64_t)(2 * k),
                      IDESC_S, (c | k) != 0);
      if (leader) umma_commit(&s_full[b]);
      if (leader) umma_commit(&vempty[vs]);
      if (t > 0) dq_mma(t - 1);
    }
    if (t > 0) dq_mma(t - 1);
    if (leader) umma_commit(acc_full);
  } else if (warp < 8) {  // epilogue (warp % 4 = TMEM lane quarter)
    const int half = warp >> 2;  // keys 64*half .. +63 of each tile
    const int lq = warp & 3;
    const int e = lq * 32 + lane;      // local query row 0..127
    const int rb = e >> 6;
    const int grow = row0 + e;
    // last key this row sees: the causal diagonal and the problem's real keys
    const int klim = g.causal ? min(grow, g.m_valid - 1) : g.m_valid - 1;
    const size_t orow = (size_t)bh * g.n + grow;
    const uint32_t tl = tmem + ((uint32_t)(lq * 32) << 16);
    const float A1 = a.A1;
    const float2 rc = a.rowc[orow];  // {C, delta} from the delta kernel
    uint32_t t = 0;
    bool any = false;
    for (int J = next_active(0); J >= 0; J = next_active(J + 1)) {
      const uint32_t b = t & 1;
      const bool mine = (bits2(rb, J) >> half) & 1u;
      any |= mine;
      mbar_wait(&s_full[b], (t >> 1) & 1);
      tc_fence_after();
      const int k0 = J * DBN + half * 64;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float s[32], dp[32];
        const uint32_t scol = tl + b * 128 + half * 64 + c * 32;
        tmem_ld32(tl + 256 + half * 64 + c * 32, dp);
        tmem_ld32(scol, s);
        tmem_wait_ld();
        if (c == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(dp_free);
        }
        const int c0 = k0 + 32 * c;
        uint32_t hi[16], lo[16];
        if (!mine) {
#pragma unroll
          for (int x = 0; x < 16; ++x) hi[x] = lo[x] = 0u;
        } else if (c0 + 31 > klim) {
          ds_chunk<AK, true>(s, dp, A1, rc.x, rc.y, a.e0f, a.e1f, klim - c0, hi, lo);
        } else {
          ds_chunk<AK, false>(s, dp, A1, rc.x, rc.y, a.e0f, a.e1f, 0, hi, lo);
        }
        // chunk c (keys 32c..32c+31 of this half) keeps its own 32 columns:
        // packed hi at +0..15, lo at +16..31
        tmem_st16(scol, hi);
        tmem_st16(scol + 16, lo);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ds_full[b]);
      ++t;
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    (void)any;
    bool rany = false;  // the row's tile has any set block (padding bits are 0)
    for (int w = 0; w < wpr; ++w) rany |= smask[rb * wpr + w] != 0u;
#pragma unroll
    for (int c = 0; c < D / 64; ++c) {
      float o[32];
      tmem_ld32(tl + 384 + half * (D / 2) + c * 32, o);
      tmem_wait_ld();
      const int x0 = half * (D / 2) + c * 32;
      if (g.out_dtype == ADATTN_F64) {
        double* dst = reinterpret_cast<double*>(a.dq) + orow * D + x0;
#pragma unroll
        for (int i = 0; i < 32; ++i) dst[i] = rany ? (double)(a.scale_f * o[i]) : 0.0;
      } else {
        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.dq) + orow * D + x0);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          dst[i] = rany ? make_float4(a.scale_f * o[4 * i], a.scale_f * o[4 * i + 1],
                                      a.scale_f * o[4 * i + 2], a.scale_f * o[4 * i + 3])
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc(tmem, 512);
}

// ============================================================== dQ (pairs)
// CTA-pair variant of the dQ kernel (cta_group::2, cluster of 2, D = 128; the
// default for d = 128): the
// pair covers 256 query rows (rank r: rows +128r) and the leader issues every
// MMA for both SMs with M = 256, so each SM feeds only half of every B operand
// from its shared memory and the per-SM MMA issue count halves:
//   S  = Q K_J^T : B half = keys 64r..64r+63 of K_J (all d)          (KS slot)
//   dP = dO V_J^T: B half = keys 64r..64r+63 of V_J                   (VS slot)
//   dQ += dS K_J : A = dS in each SM's TMEM, B half = d cols 64r..+63 (KD slot, MN-major)
// Tiles are the union of both CTAs' active tiles; a CTA writes dS = 0 where its
// own blocks are clear.  Barriers: full / q_full / ds_full / dp_free live in the
// leader (TMA of both CTAs completes there; the peer's epilogue arrives
// remotely); empty / s_full / acc_full in each CTA, armed by multicast commits.
template <int D>
struct Dq2Smem {
  static_assert(D == 128, "pair dQ kernel: d = 128");
  static constexpr int QB = QB_DQ * D * 2;     // own 128 rows of Q (and of dO)
  static constexpr int HB = 64 * D * 2;        // 64 keys x d   (KS, VS slots)
  static constexpr int KDB = DBN * 64 * 2;     // 128 keys x 64 d (KD slot)
  static constexpr int NSK = 3, NSV = 3;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_DO = OFF_Q + QB;
  static constexpr int OFF_KS = OFF_DO + QB;
  static constexpr int OFF_KD = OFF_KS + NSK * HB;
  static constexpr int OFF_VS = OFF_KD + NSK * KDB;
  static constexpr int OFF_BAR = OFF_VS + NSV * HB;
  static constexpr int OFF_MISC = OFF_BAR + 40 * 8;
  static constexpr int OFF_MASK = OFF_MISC + 64;
  __host__ __device__ static int off_list(int wpr) { return OFF_MASK + 4 * wpr * 4; }
  // + the compacted nonzero-tile list (<= 16 wpr u16)
  static size_t bytes(int wpr) { return 1024 + off_list(wpr) + 32 * wpr + 64; }
};

template <int D, int AK, bool DSF16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    tc_dq2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kh,
                  const __grid_constant__ CUtensorMap tm_kd, const __grid_constant__ CUtensorMap tm_vh,
                  const __grid_constant__ CUtensorMap tm_do, const __grid_constant__ CUtensorMap tm_kd16,
                  const BwdArgs a) {
  using L = Dq2Smem<D>;
  // dQ = (sigma dS) K in fp16 (F16Plan): one MMA per K step instead of hi + lo.
  // DSF16 = false (the default) compiles the fp16 branches out of the issue loop.
  constexpr int NSK = L::NSK, NSV = L::NSV;
  constexpr int NCH = D / 64;
  const Geom& g = a.g;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sDO = smem + L::OFF_DO;
  uint8_t* sKS = smem + L::OFF_KS;
  uint8_t* sKD = smem + L::OFF_KD;
  uint8_t* sVS = smem + L::OFF_VS;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* kfull = bars;              // [NSK] leader: K_S + K_D of both CTAs
  uint64_t* kempty = kfull + NSK;      // [NSK] each CTA
  uint64_t* vfull = kempty + NSK;      // [NSV] leader
  uint64_t* vempty = vfull + NSV;      // [NSV] each CTA
  uint64_t* s_full = vempty + NSV;     // [2] each CTA
  uint64_t* ds_full = s_full + 2;      // [2] leader, 16 warps
  uint64_t* dp_free = ds_full + 2;     // leader, 16 warps
  uint64_t* acc_full = dp_free + 1;    // each CTA
  uint64_t* q_full = acc_full + 1;     // leader
  volatile uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::OFF_MISC);
  uint32_t* smask = reinterpret_cast<uint32_t*>(smem + L::OFF_MASK);  // [4][wpr] (the pair's row blocks)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_ctarank();
  const bool lead_cta = rank == 0;
  const int npair = g.n / (2 * QB_DQ);
  const int pair = (int)(blockIdx.x >> 1);
  const int bh = pair / npair;  // head-major, heaviest pairs first
  const F16Plan* pl = a.f16 ? a.f16 + bh : nullptr;  // the head's fp16 plan
  const bool f16s = DSF16 && pl && pl->ds_ok;
  const float sig = f16s ? pl->sigma : 1.f;
  const int prow0 = (npair - 1 - pair % npair) * 2 * QB_DQ;
  const int row0 = prow0 + (int)rank * QB_DQ;
  const int nkt = g.m / DBN;
  const int jmax = g.causal ? (prow0 + 2 * QB_DQ - 1) / DBN : nkt - 1;
  const int wpr = g.wpr;

  if (a.dq_skip && a.dq_skip[bh] == 0u) return;  // dQ from the support lists (both CTAs)
  rows_from_lists(smask, 4, a, bh, prow0 / 64, tid, kThreads);
  if (tid == 0) {
    for (int i = 0; i < NSK; ++i) {
      mbar_init(&kfull[i], 1);
      mbar_init(&kempty[i], 1);
    }
    for (int i = 0; i < NSV; ++i) {
      mbar_init(&vfull[i], 1);
      mbar_init(&vempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&ds_full[i], 16);
    }
    mbar_init(dp_free, 16);
    mbar_init(acc_full, 1);
    mbar_init(q_full, 1);
    fence_barrier_init();
  }
  if (warp == 8) tmem_alloc_2sm(const_cast<uint32_t*>(s_tmem), 512);
  tc_fence_before();
  cluster_sync();  // barrier inits of both CTAs visible before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  auto bits2 = [&](int rb, int J) -> uint32_t {  // rb: 0..3 over the pair's 256 rows
    return (smask[rb * wpr + ((2 * J) >> 5)] >> ((2 * J) & 31)) & 3u;
  };
  // the CTA's nonzero 128-key tiles, compacted once (union over both CTAs' rows)
  uint16_t* sList = reinterpret_cast<uint16_t*>(smem + L::off_list(wpr));
  volatile uint32_t* sListN = reinterpret_cast<volatile uint32_t*>(smem + L::OFF_MISC) + 2;
  if (warp == 0)
    compact_active(sList, sListN, jmax, lane, [&](int J) -> bool { return bits2(0, J) | bits2(1, J) | bits2(2, J) | bits2(3, J); });
  __syncthreads();
  ActiveList walk{sList, (int)*sListN, 0};
  auto next_active = [&](int J) -> int { return walk.next(J); };

  if (warp == 8) {  // TMA producer (both CTAs load their own halves)
    const bool leader = elect_one_sync();
    const int qrow = bh * g.n + row0;
    if (lead_cta && leader) mbar_expect_tx(q_full, 2 * 2 * L::QB);
    for (int c = 0; c < NCH; ++c) {
      if (leader) tma_load_2d_2sm(sQ + c * QB_DQ * 128, &tm_q, q_full, c * 64, qrow);
      if (leader) tma_load_2d_2sm(sDO + c * QB_DQ * 128, &tm_do, q_full, c * 64, qrow);
    }
    uint32_t t = 0;
    const int krow0 = bh * g.m;
    for (int J = next_active(0); J >= 0; J = next_active(J + 1), ++t) {
      const uint32_t ks = t % NSK, vs = t % NSV;
      mbar_wait(&kempty[ks], ((t / NSK) & 1) ^ 1);
      if (lead_cta && leader) mbar_expect_tx(&kfull[ks], 2 * (L::HB + L::KDB));
      for (int c = 0; c < NCH; ++c)
        if (leader)
          tma_load_2d_2sm(sKS + ks * L::HB + c * 64 * 128, &tm_kh, &kfull[ks], c * 64,
                          krow0 + J * DBN + 64 * (int)rank);
      if (leader)
        tma_load_2d_2sm(sKD + ks * L::KDB, f16s ? &tm_kd16 : &tm_kd, &kfull[ks], 64 * (int)rank, krow0 + J * DBN);
      mbar_wait(&vempty[vs], ((t / NSV) & 1) ^ 1);
      if (lead_cta && leader) mbar_expect_tx(&vfull[vs], 2 * L::HB);
      for (int c = 0; c < NCH; ++c)
        if (leader)
          tma_load_2d_2sm(sVS + vs * L::HB + c * 64 * 128, &tm_vh, &vfull[vs], c * 64,
                          krow0 + J * DBN + 64 * (int)rank);
    }
  } else if (warp == 9) {  // MMA issuer: the pair leader only
    if (lead_cta) {
      const bool leader = elect_one_sync();
      constexpr uint32_t IDESC_S = idesc_bf16_f32(256, DBN, false, false);
      constexpr uint32_t IDESC_DQ = idesc_bf16_f32(256, D, false, true);
      constexpr uint32_t IDESC_DQ16 = idesc_f16_f32(256, D, false, true);
      const uint32_t q_addr = smem_u32(sQ), do_addr = smem_u32(sDO);
      uint64_t dQd[NCH], dDOd[NCH], dKS[NCH], dVS[NCH];
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        dQd[c] = desc_kmajor(q_addr + c * QB_DQ * 128);
        dDOd[c] = desc_kmajor(do_addr + c * QB_DQ * 128);
        dKS[c] = desc_kmajor(smem_u32(sKS) + c * 64 * 128);
        dVS[c] = desc_kmajor(smem_u32(sVS) + c * 64 * 128);
      }
      const uint64_t dKD = desc_mnmajor(smem_u32(sKD), DBN * 128);
      constexpr uint32_t kHF = (uint32_t)L::HB >> 4, kKDF = (uint32_t)L::KDB >> 4;
      mbar_wait(q_full, 0);
      tc_fence_after();
      uint32_t t = 0;
      bool acc_init = false;
      auto dq_mma = [&](uint32_t tt) {
        const uint32_t b = tt & 1, ks = tt % NSK;
        mbar_wait(&ds_full[b], (tt >> 1) & 1);
        tc_fence_after();
        const uint64_t bk = dKD + (uint64_t)(ks * kKDF);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t acol = b * 128 + 32 * (k >> 1) + 8 * (k & 1);
          const uint64_t bd = bk + (uint64_t)(128 * k);
          if (f16s) {
            if (leader) umma2_bf16_ts(tmem + 384, tmem + acol, bd, IDESC_DQ16, (acc_init || k > 0) ? 1u : 0u);
          } else {
            if (leader) umma2_bf16_ts(tmem + 384, tmem + acol, bd, IDESC_DQ, (acc_init || k > 0) ? 1u : 0u);
            if (leader) umma2_bf16_ts(tmem + 384, tmem + acol + 16, bd, IDESC_DQ, 1u);
          }
        }
        acc_init = true;
        if (leader) umma2_commit_mc(&kempty[ks]);
      };
      for (int J = next_active(0); J >= 0; J = next_active(J + 1), ++t) {
        const uint32_t ks = t % NSK, vs = t % NSV, b = t & 1;
        mbar_wait(&kfull[ks], (t / NSK) & 1);
        tc_fence_after();
        const uint64_t ko = (uint64_t)(ks * kHF), vo = (uint64_t)(vs * kHF);
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (leader)
              umma2_bf16(tmem + b * 128, dQd[c] + (uint64_t)(2 * k), dKS[c] + ko + (uint64_t)(2 * k),
                         IDESC_S, (c | k) != 0);
        mbar_wait(&vfull[vs], (t / NSV) & 1);
        if (t > 0) mbar_wait(dp_free, (t - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (leader)
              umma2_bf16(tmem + 256, dDOd[c] + (uint64_t)(2 * k), dVS[c] + vo + (uint64_t)(2 * k),
                         IDESC_S, (c | k) != 0);
        if (leader) umma2_commit_mc(&s_full[b]);
        if (leader) umma2_commit_mc(&vempty[vs]);
        if (t > 0) dq_mma(t - 1);
      }
      if (t > 0) dq_mma(t - 1);
      if (leader) umma2_commit_mc(acc_full);
    }
  } else if (warp < 8) {  // epilogue (warp % 4 = TMEM lane quarter)
    const int half = warp >> 2;
    const int lq = warp & 3;
    const int e = lq * 32 + lane;
    const int rb = e >> 6;                // own row block 0/1
    const int prb = (int)rank * 2 + rb;   // row block within the pair
    const int grow = row0 + e;
    // last key this row sees: the causal diagonal and the problem's real keys
    const int klim = g.causal ? min(grow, g.m_valid - 1) : g.m_valid - 1;
    const size_t orow = (size_t)bh * g.n + grow;
    const uint32_t tl = tmem + ((uint32_t)(lq * 32) << 16);
    const float A1 = a.A1;
    const float2 rc = a.rowc[orow];
    // leader-CTA barriers as cluster addresses (local for the leader)
    const uint32_t ds_full_c0 = mapa_shared(smem_u32(&ds_full[0]), 0);
    const uint32_t ds_full_c1 = mapa_shared(smem_u32(&ds_full[1]), 0);
    const uint32_t dp_free_c = mapa_shared(smem_u32(dp_free), 0);
    uint32_t t = 0;
    for (int J = next_active(0); J >= 0; J = next_active(J + 1), ++t) {
      const uint32_t b = t & 1;
      const bool mine = (bits2(prb, J) >> half) & 1u;
      mbar_wait(&s_full[b], (t >> 1) & 1);
      tc_fence_after();
      const int k0 = J * DBN + half * 64;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float s[32], dp[32];
        const uint32_t scol = tl + b * 128 + half * 64 + c * 32;
        tmem_ld32(tl + 256 + half * 64 + c * 32, dp);
        tmem_ld32(scol, s);
        tmem_wait_ld();
        if (c == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(dp_free_c);
        }
        const int c0 = k0 + 32 * c;
        uint32_t hi[16], lo[16];
        if (!mine) {
#pragma unroll
          for (int x = 0; x < 16; ++x) hi[x] = lo[x] = 0u;
        } else if (c0 + 31 > klim) {
          if (f16s) ds_chunk<AK, true, true>(s, dp, A1, rc.x, rc.y, a.e0f, a.e1f, klim - c0, hi, lo, sig);
          else ds_chunk<AK, true>(s, dp, A1, rc.x, rc.y, a.e0f, a.e1f, klim - c0, hi, lo);
        } else {
          if (f16s) ds_chunk<AK, false, true>(s, dp, A1, rc.x, rc.y, a.e0f, a.e1f, 0, hi, lo, sig);
          else ds_chunk<AK, false>(s, dp, A1, rc.x, rc.y, a.e0f, a.e1f, 0, hi, lo);
        }
        tmem_st16(scol, hi);
        if (!f16s) tmem_st16(scol + 16, lo);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(b ? ds_full_c1 : ds_full_c0);
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const float oscale = a.scale_f * (f16s ? pl->inv_sigma * pl->inv_k : 1.f);
    bool rany = false;
    for (int w = 0; w < wpr; ++w) rany |= smask[prb * wpr + w] != 0u;
#pragma unroll
    for (int c = 0; c < D / 64; ++c) {
      float o[32];
      tmem_ld32(tl + 384 + half * (D / 2) + c * 32, o);
      tmem_wait_ld();
      const int x0 = half * (D / 2) + c * 32;
      if (g.out_dtype == ADATTN_F64) {
        double* dst = reinterpret_cast<double*>(a.dq) + orow * D + x0;
#pragma unroll
        for (int i = 0; i < 32; ++i) dst[i] = rany ? (double)(oscale * o[i]) : 0.0;
      } else {
        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.dq) + orow * D + x0);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          dst[i] = rany ? make_float4(oscale * o[4 * i], oscale * o[4 * i + 1],
                                      oscale * o[4 * i + 2], oscale * o[4 * i + 3])
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  tc_fence_before();
  cluster_sync();  // the pair's MMAs and remote arrives are done before TMEM is freed
  if (warp == 8) tmem_dealloc_2sm(tmem, 512);
}

// ================================================================= dK / dV
constexpr int KB = 128;      // keys per CTA
constexpr int QT = 64;       // query rows per unit (one reference tile)
constexpr int KST = 4;       // Q/dO stages

template <int D>
struct KvSmem {
  static constexpr int KVB = KB * D * 2;
  static constexpr int QTB = QT * D * 2;
  static constexpr int STAGE = 2 * QTB + 1024;  // Q_i, dO_i, rowc[64] (1024-aligned stages)
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + KVB;
  static constexpr int OFF_ST = OFF_V + KVB;
  static constexpr int OFF_BAR = OFF_ST + KST * STAGE;
  static constexpr int OFF_MISC = OFF_BAR + 32 * 8;
  static constexpr int OFF_UB = OFF_MISC + 64;
  __host__ __device__ static int off_list(int t_r) { return OFF_UB + (t_r + 15) / 16 * 16; }
  // + the compacted active-unit list (t_r u16)
  static size_t bytes(int t_r) { return 1024 + off_list(t_r) + 2 * t_r + 64; }
};

template <int D, int AK>
__global__ void __launch_bounds__(kThreads, 1)
    tc_dkdv_kernel(const __grid_constant__ CUtensorMap tm_qt, const __grid_constant__ CUtensorMap tm_kb,
                   const __grid_constant__ CUtensorMap tm_vb, const __grid_constant__ CUtensorMap tm_dot,
                   const BwdArgs a) {
  using L = KvSmem<D>;
  constexpr int NCH = D / 64;
  // S^T / dP^T buffers in TMEM (128 columns each) ahead of the dV, dK accumulators: d = 64
  // leaves room for three, so the gradients of unit u are issued after S^T(u + 2) and
  // the epilogue of unit u has two units of MMA work to hide behind (two buffers: the
  // S^T -> epilogue -> gradients -> S^T(u + 2) chain idled the pipe ~45% at C4)
  constexpr int NB = D == 64 ? 3 : 2;
  constexpr uint32_t ACC = NB * 128;
  const Geom& g = a.g;
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned base that stays in the shared address space (LDS/STS, not
  // generic LD/ST, for every access through it)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  uint8_t* sSt = smem + L::OFF_ST;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full = bars;             // [KST]
  uint64_t* empty = bars + KST;      // [KST]
  uint64_t* s_full = bars + 2 * KST; // [NB]
  uint64_t* p_full = s_full + NB;    // [NB]
  uint64_t* kv_full = p_full + NB;
  uint64_t* acc_full = kv_full + 1;
  volatile uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::OFF_MISC);
  uint8_t* ubits = smem + L::OFF_UB;  // [t_r] 2-bit activity of (i, j0), (i, j0+1)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nkb = g.m / KB;
  const int bh = blockIdx.x / nkb;   // head-major (Q/dO L2-resident)
  const int kb = blockIdx.x % nkb;   // causal: low key blocks have the most query tiles
  const int key0 = kb * KB;
  const int j0 = key0 / 64;          // first of the two reference key tiles
  const int wpr = g.wpr;
  const int i_first = g.causal ? key0 / QT : 0;

  if (a.kv_skip && a.kv_skip[bh] == 0u) return;  // dK/dV from the support lists
  units_from_lists(ubits, 2, a, bh, kb * KB / 64, threadIdx.x, kThreads);
  if (tid == 0) {
    for (int i = 0; i < KST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < NB; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 8);
    }
    mbar_init(kv_full, 1);
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 8) tmem_alloc(const_cast<uint32_t*>(s_tmem), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  (void)nkb;

  // bits of (query tile i, key tiles j0, j0+1): bit0 -> keys 0..63, bit1 -> 64..127
  auto unit_bits = [&](int i) -> uint32_t { return ubits[i]; };
  (void)wpr;
  (void)j0;
  // the CTA's active query units, compacted once
  uint16_t* sList = reinterpret_cast<uint16_t*>(smem + L::off_list(g.t_r));
  volatile uint32_t* sListN = reinterpret_cast<volatile uint32_t*>(smem + L::OFF_MISC) + 2;
  if (warp == 0)
    compact_active(sList, sListN, g.t_r - 1, lane, [&](int i) -> bool { return unit_bits(i) != 0; });
  __syncthreads();
  ActiveList walk{sList, (int)*sListN, 0};
  auto next_unit = [&](int i) -> int { return walk.next(i); };

  if (warp == 8) {  // TMA producer
    {
      const bool leader = elect_one_sync();
      const int krow = bh * g.m + key0;
      if (leader) mbar_expect_tx(kv_full, 2 * L::KVB);
      for (int c = 0; c < NCH; ++c) {
        if (leader) tma_load_2d(sK + c * KB * 128, &tm_kb, kv_full, c * 64, krow);
        if (leader) tma_load_2d(sV + c * KB * 128, &tm_vb, kv_full, c * 64, krow);
      }
      uint32_t r = 0;
      for (int i = next_unit(i_first); i >= 0; i = next_unit(i + 1)) {
        const uint32_t st = r % KST, ph = (r / KST) & 1;
        mbar_wait(&empty[st], ph ^ 1);
        if (leader) mbar_expect_tx(&full[st], 2 * L::QTB + QT * 8);
        uint8_t* base = sSt + st * L::STAGE;
        const int qrow = bh * g.n + i * QT;
        for (int c = 0; c < NCH; ++c) {
          if (leader) tma_load_2d(base + c * QT * 128, &tm_qt, &full[st], c * 64, qrow);
          if (leader) tma_load_2d(base + L::QTB + c * QT * 128, &tm_dot, &full[st], c * 64, qrow);
        }
        if (leader) bulk_load(base + 2 * L::QTB, a.rowc + qrow, QT * 8, &full[st]);
        ++r;
      }
    }
  } else if (warp == 9) {  // MMA issuer (highest warp id: scheduler priority)
    {
      const bool leader = elect_one_sync();
      constexpr uint32_t IDESC_S = idesc_bf16_f32(128, QT, false, false);
      constexpr uint32_t IDESC_G = idesc_bf16_f32(128, D, false, true);
      const uint32_t k_addr = smem_u32(sK), v_addr = smem_u32(sV), st_addr = smem_u32(sSt);
      mbar_wait(kv_full, 0);
      tc_fence_after();
      // loop-invariant operand descriptors (stage 0; other stages add STAGE >> 4)
      uint64_t dK[NCH], dV[NCH], dQk[NCH], dDOk[NCH];
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        dK[c] = desc_kmajor(k_addr + c * KB * 128);
        dV[c] = desc_kmajor(v_addr + c * KB * 128);
        dQk[c] = desc_kmajor(st_addr + c * QT * 128);
        dDOk[c] = desc_kmajor(st_addr + L::QTB + c * QT * 128);
      }
      const uint64_t dQmn = desc_mnmajor(st_addr, QT * 128);
      const uint64_t dDOmn = desc_mnmajor(st_addr + L::QTB, QT * 128);
#ifdef ADATTN_PIPE_STATS
      const long long t_m0 = clock64();
#endif
      uint32_t u = 0;
      bool init = false;
      auto grad_mma = [&](uint32_t uu) {
        const uint32_t b = uu % NB, st = uu % KST;
        {
          BSTAT_T0();
          mbar_wait(&p_full[b], (uu / NB) & 1);
          BSTAT_ADD(1, leader);
        }
        tc_fence_after();
        BSTAT_T0();
        // stage st's Q / dO descriptors: the base descriptors + the stage offset
        const uint64_t so = (uint64_t)((st * (uint32_t)L::STAGE) >> 4);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          // queries 16k..16k+15: packed pairs of half k>>1 at cols 32*(k>>1) + 8*(k&1)
          // (hi) and +16 (lo); K step of 16 rows = 2048 B = +128 in the address field
          const uint32_t acol = 32 * (k >> 1) + 8 * (k & 1);
          const uint64_t bdo = dDOmn + so + (uint64_t)(128 * k);
          const uint64_t bq = dQmn + so + (uint64_t)(128 * k);
          const uint32_t acc = (init || k > 0) ? 1u : 0u;
          if (leader) umma_bf16_ts(tmem + ACC, tmem + b * 128 + acol, bdo, IDESC_G, acc);
          if (leader) umma_bf16_ts(tmem + ACC, tmem + b * 128 + acol + 16, bdo, IDESC_G, 1u);
          if (leader) umma_bf16_ts(tmem + ACC + D, tmem + b * 128 + 64 + acol, bq, IDESC_G, acc);
          if (leader) umma_bf16_ts(tmem + ACC + D, tmem + b * 128 + 64 + acol + 16, bq, IDESC_G, 1u);
        }
        init = true;
        if (leader) umma_commit(&empty[st]);
        BSTAT_ADD(6, leader);
      };
      for (int i = next_unit(i_first); i >= 0; i = next_unit(i + 1)) {
        const uint32_t st = u % KST;
        {
          BSTAT_T0();
          mbar_wait(&full[st], (u / KST) & 1);
          BSTAT_ADD(0, leader);
        }
        tc_fence_after();
        const uint32_t b = u % NB;
        const uint64_t so = (uint64_t)((st * (uint32_t)L::STAGE) >> 4);
        BSTAT_T0();
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (leader) umma_bf16(tmem + b * 128, dK[c] + (uint64_t)(2 * k),
                      dQk[c] + so + (uint64_t)(2 * k), IDESC_S, (c | k) != 0);
            if (leader) umma_bf16(tmem + b * 128 + 64, dV[c] + (uint64_t)(2 * k),
                      dDOk[c] + so + (uint64_t)(2 * k), IDESC_S, (c | k) != 0);
          }
        if (leader) umma_commit(&s_full[b]);
        BSTAT_ADD(5, leader);
        // in pipe order after grad(u - NB), which read buffer b
        if (u >= NB - 1) grad_mma(u - (NB - 1));
        ++u;
      }
      for (uint32_t uu = u > NB - 1 ? u - (NB - 1) : 0; uu < u; ++uu) grad_mma(uu);
      if (leader) umma_commit(acc_full);
#ifdef ADATTN_PIPE_STATS
      if (leader) {
        atomicAdd(&g_bwd_stats[3], (unsigned long long)(clock64() - t_m0));
        atomicAdd(&g_bwd_stats[4], (unsigned long long)u);
      }
#endif
    }
  } else if (warp < 8) {  // epilogue (warp % 4 = TMEM lane quarter)
    const int ew = warp;
    const int half = ew >> 2;          // query columns 32*half .. +31
    const int lq = warp & 3;
    const int key = lq * 32 + lane;    // 0..127 within the CTA
    const int gkey = key0 + key;
    const int ksub = key >> 6;         // which reference key tile (0/1)
    const uint32_t tl = tmem + ((uint32_t)(lq * 32) << 16);
    const float A1 = a.A1;
    uint32_t u = 0;
    bool any = false;
    for (int i = next_unit(i_first); i >= 0; i = next_unit(i + 1)) {
      const uint32_t st = u % KST, b = u % NB;
      const bool mine = (unit_bits(i) >> ksub) & 1u;
      any |= mine;
      {
        BSTAT_T0();
        mbar_wait(&s_full[b], (u / NB) & 1);
        BSTAT_ADD(2, warp == 0 && lane == 0);
      }
      tc_fence_after();
      float s[32], dp[32];
      tmem_ld32(tl + b * 128 + half * 32, s);
      tmem_ld32(tl + b * 128 + 64 + half * 32, dp);
      tmem_wait_ld();
      const float2* rc = reinterpret_cast<const float2*>(sSt + st * L::STAGE + 2 * L::QTB);
      uint32_t ph[16], pl[16], dh[16], dl[16];
      const int q0 = i * QT + half * 32;
      if (!mine) {
#pragma unroll
        for (int x = 0; x < 16; ++x) ph[x] = pl[x] = dh[x] = dl[x] = 0u;
      } else if (g.causal && q0 < key0 + lq * 32 + 31) {  // warp-uniform: diagonal tiles
        pds_chunk<AK, true>(s, dp, rc + half * 32, A1, a.e0f, a.e1f, gkey - q0, ph, pl, dh, dl);
      } else {
        pds_chunk<AK, false>(s, dp, rc + half * 32, A1, a.e0f, a.e1f, 0, ph, pl, dh, dl);
      }
      // half h owns TMEM columns 32h..32h+31 of the S^T / dP^T regions it just read:
      // packed hi at +0..15, lo at +16..31
      tmem_st16(tl + b * 128 + half * 32, ph);
      tmem_st16(tl + b * 128 + half * 32 + 16, pl);
      tmem_st16(tl + b * 128 + 64 + half * 32, dh);
      tmem_st16(tl + b * 128 + 64 + half * 32 + 16, dl);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[b]);
      ++u;
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    any = __any_sync(0xffffffffu, any);
    const size_t krow = (size_t)bh * g.m + gkey;
#pragma unroll
    for (int which = 0; which < 2; ++which) {  // 0: dV, 1: dK
      void* base = which == 0 ? a.dv : a.dk;
      const float mul = which == 0 ? 1.f : a.scale_f;
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        float o[32];
        tmem_ld32(tl + ACC + which * D + half * (D / 2) + c * 32, o);
        tmem_wait_ld();
        const int x0 = half * (D / 2) + c * 32;
        if (g.out_dtype == ADATTN_F64) {
          double* dst = reinterpret_cast<double*>(base) + krow * D + x0;
#pragma unroll
          for (int x = 0; x < 32; ++x) dst[x] = any ? (double)(mul * o[x]) : 0.0;
        } else {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(base) + krow * D + x0);
#pragma unroll
          for (int x = 0; x < 8; ++x)
            dst[x] = any ? make_float4(mul * o[4 * x], mul * o[4 * x + 1], mul * o[4 * x + 2],
                                       mul * o[4 * x + 3])
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc(tmem, 512);
}

// ============================================================ dK / dV (pairs)
// CTA-pair variant (cta_group::2, d = 128): the pair covers 256 keys (rank r:
// keys +128r); the leader issues every MMA with M = 256.  Per 64-query unit i:
//   S^T  = K Q_i^T  : B half = queries 32r..32r+31 of Q_i (all d)     (QS)
//   dP^T = V dO_i^T : B half = queries 32r.. of dO_i                   (DS)
//   dV += P^T dO_i  : A = P^T (own TMEM), B half = d cols 64r.. of dO_i (DD, MN-major)
//   dK += dS^T Q_i  : A = dS^T, B half = d cols 64r.. of Q_i           (QD, MN-major)
// Units are the union of both CTAs' active units; rowc (C, delta) of the unit
// comes with a local bulk copy on a per-stage local barrier.
// mx: per-head |x| maxima (float bits) of dO, V, Q, K at mx[0..bh), mx[bh..2bh), ...
__global__ void f16_plan_kernel(F16Plan* plans, const uint32_t* mx, int bh, float alpha, int d,
                                int want_dv, int want_ds) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= bh) return;
  F16Plan* pl = plans + h;
  const uint32_t bdo = mx[h], bv = mx[bh + h], bq = mx[2 * bh + h], bk = mx[3 * bh + h];
  const float mdo = __uint_as_float(bdo), mv = __uint_as_float(bv);
  pl->dv_ok = want_dv && f16_copy_ok(bdo);
  pl->inv_do = 1.f / f16_pow2_scale(bdo);
  pl->inv_q = 1.f / f16_pow2_scale(bq);
  pl->inv_k = 1.f / f16_pow2_scale(bk);
  const float bound = 2.f * (float)d * mdo * mv;  // >= max |dS| (alpha <= 2)
  int ok = want_ds && alpha <= 2.f && f16_copy_ok(bq) && f16_copy_ok(bk) && bound < 3.0e38f;
  float sigma = 1.f;
  if (ok && bound > 0.f) {
    int ex;
    frexpf(32768.f / bound, &ex);          // 32768 / bound = f 2^ex, f in [0.5, 1)
    ex = max(-100, min(ex - 1, 100));     // 2^(ex-1) <= 32768 / bound
    sigma = ldexpf(1.f, ex);
  }
  pl->ds_ok = ok;
  pl->sigma = sigma;
  pl->inv_sigma = 1.f / sigma;
}


// delta from the forward's fold (Geom::ubar_in): delta_i = dO_i . Ubar_i / sum_j u_ij
// (0 when the sum is 0, attention.cpp:444), one warp per row; also rowc_i = (C_i, delta_i)
// for the dK/dV kernel, C_i = 1 - (alpha - 1) m_i - tau_i as the delta kernels form it
template <int D>
__global__ void delta_ubar_kernel(const uint16_t* __restrict__ dout, const float* __restrict__ ubar,
                                  const double* __restrict__ tau, const double* __restrict__ row_max,
                                  double alpha, size_t rows, double* delta, float2* rowc) {
  constexpr int E = D / 32;
  const size_t r = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const uint16_t* dp = dout + r * D + lane * E;
  const float* up = ubar + r * D + lane * E;
  float acc = 0.f;
  if constexpr (E == 4) {
    const uint2 w = *reinterpret_cast<const uint2*>(dp);
    const float4 u = *reinterpret_cast<const float4*>(up);
    acc = __uint_as_float(w.x << 16) * u.x + __uint_as_float(w.x & 0xFFFF0000u) * u.y +
          __uint_as_float(w.y << 16) * u.z + __uint_as_float(w.y & 0xFFFF0000u) * u.w;
  } else {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(dp);
    const float2 u = *reinterpret_cast<const float2*>(up);
    acc = __uint_as_float(w << 16) * u.x + __uint_as_float(w & 0xFFFF0000u) * u.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    const double su = (double)ubar[rows * D + r];
    const double dlt = su > 0.0 ? (double)acc / su : 0.0;
    const double B = 1.0 - (alpha - 1.0) * row_max[r];
    delta[r] = dlt;
    rowc[r] = make_float2((float)(B - tau[r]), (float)dlt);
  }
}

// delta and dQ from the support lists (Geom::supp_in, written by the forward's list
// phase: per row its keys j and t_ij > 0 at the final tau).  The backward's terms vanish
// off the support (u = p = 0 for t <= 0, attention.cpp:411-446, 508-535), so per row:
//   dp_j = dO_i . v_j,  delta_i = sum u_j dp_j / sum u_j  (0 when the sum is 0),
//   dQ_i = scale * sum_j u_j (dp_j - delta_i) k_j
// over ~30 entries at C3 instead of S and dP over every active block (the delta
// pre-pass: two products per tile, the dQ kernel: three).  One warp per row, lane l holds
// d elements l*E..; the head's K / V rows stay L2-resident (rows run head by head).
// Entries go in list order (key half 0, then half 1), sums in fp64: deterministic.
// Rows of a 256-row block the forward flagged are left to the delta kernel (its unit
// of `unit` rows runs when any of its blocks is flagged); dQ only for heads without a
// flagged block (hflag; the tensor-core dQ kernel takes the others) -- a row with more
// than 192 entries flags its head here (the tensor-core kernels run after this one).
// Also rowc_i = (C_i, delta_i) for the dK/dV kernel, as the delta kernels form it.
// (d = 64: a 64-register bound -- 4 CTAs of 256 per SM -- makes ptxas schedule more gathers
// ahead: C4 rows kernel 12.4 -> 9.9 ms; d = 128 keeps the unhinted bound, the hint cost 0.3 ms)
template <int D, int AK>
__global__ void __launch_bounds__(256, D == 64 ? 4 : 0) sparse_rows_kernel(
    const uint16_t* __restrict__ dout, const uint16_t* __restrict__ vv, const uint16_t* __restrict__ kk,
    const uint2* __restrict__ pool, const int2* __restrict__ cnt, const uint32_t* __restrict__ flag,
    uint32_t* hflag, int cap, int unit, const int32_t* __restrict__ koff, int32_t* kcur,
    int32_t* krow, float2* kpd, const double* __restrict__ tau,
    const double* __restrict__ row_max, double alpha, float e0f, float e1f, float scale,
    size_t rows, int n, int m, int out_f64, bool want_dq, void* dq, double* delta, float2* rowc) {
  constexpr int E = D / 32;
  constexpr int NCH = 3;  // entries kept in registers: 3 x 32 per row (C3: ~30, C5: ~40);
                          // longer rows recompute dp for the rest in phase 2
  const size_t r = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const size_t bh = r / (size_t)n;
  const size_t u0 = (bh * n + (r - bh * n) / unit * unit) / 256;
  const int2 h0 = cnt[r * 2], h1 = cnt[r * 2 + 1];  // (read beside the flags)
  for (int b = 0; b < unit / 256; ++b)
    if (flag[u0 + b]) return;
  const int c0 = h0.x, tot = h0.x + h1.x;
  const uint2* base = pool + (r / 256) * (size_t)(256 * cap);
  const uint16_t* vb = vv + bh * (size_t)m * D + lane * E;
  const uint16_t* kb = kk + bh * (size_t)m * D + lane * E;
  auto ld_row = [&](const uint16_t* p, float* x) {  // E bf16 of a row -> fp32
    if constexpr (E == 4) {
      const uint2 w = *reinterpret_cast<const uint2*>(p);
      x[0] = __uint_as_float(w.x << 16);
      x[1] = __uint_as_float(w.x & 0xFFFF0000u);
      x[2] = __uint_as_float(w.y << 16);
      x[3] = __uint_as_float(w.y & 0xFFFF0000u);
    } else {
      const uint32_t w = *reinterpret_cast<const uint32_t*>(p);
      x[0] = __uint_as_float(w << 16);
      x[1] = __uint_as_float(w & 0xFFFF0000u);
    }
  };
  float dov[E];
  ld_row(dout + r * D + lane * E, dov);
  // phase 1: dp of every entry -- lane k takes entry k whole (its V row, 16-byte loads,
  // against dO staged in shared memory as fp32), no per-entry warp reduction -- and delta
  __shared__ float4 sdo[8][D / 4];  // (8 warps per CTA)
  const int wi = (threadIdx.x >> 5) & 7;
  {  // the warp's dO row, fp32, d-ordered
    const uint16_t* dr = dout + r * D;
    for (int x = lane; x < D / 4; x += 32) {
      const uint2 w = *reinterpret_cast<const uint2*>(dr + 4 * x);
      sdo[wi][x] = make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xFFFF0000u),
                               __uint_as_float(w.y << 16), __uint_as_float(w.y & 0xFFFF0000u));
    }
  }
  __syncwarp();
  uint32_t keyr[NCH];
  float ur[NCH], dpr[NCH], pr[NCH];
  double num = 0.0, den = 0.0;
  for (int b = 0, ch = 0; b < tot; b += 32, ++ch) {
    const int idx = b + lane;
    uint2 my = make_uint2(0u, 0u);
    if (idx < tot) my = idx < c0 ? base[h0.y + idx] : base[h1.y + idx - c0];
    float p_, u_;
    pu_of<AK>(__uint_as_float(my.y), e0f, e1f, p_, u_);
    float dpk = 0.f;
    if (idx < tot) {
      const uint4* vr = reinterpret_cast<const uint4*>(vv + (bh * (size_t)m + my.x) * D);
      uint4 w[D / 8];
#pragma unroll
      for (int x = 0; x < D / 8; ++x) w[x] = vr[x];
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int x = 0; x < D / 8; ++x) {
        const float4 o0 = sdo[wi][2 * x], o1 = sdo[wi][2 * x + 1];
        s0 = fmaf(o0.x, __uint_as_float(w[x].x << 16), s0);
        s1 = fmaf(o0.y, __uint_as_float(w[x].x & 0xFFFF0000u), s1);
        s0 = fmaf(o0.z, __uint_as_float(w[x].y << 16), s0);
        s1 = fmaf(o0.w, __uint_as_float(w[x].y & 0xFFFF0000u), s1);
        s0 = fmaf(o1.x, __uint_as_float(w[x].z << 16), s0);
        s1 = fmaf(o1.y, __uint_as_float(w[x].z & 0xFFFF0000u), s1);
        s0 = fmaf(o1.z, __uint_as_float(w[x].w << 16), s0);
        s1 = fmaf(o1.w, __uint_as_float(w[x].w & 0xFFFF0000u), s1);
      }
      dpk = s0 + s1;
    } else {
      u_ = 0.f;
    }
    // sum u dp, sum u over the chunk: a fixed fp64 tree
    double tn = (double)u_ * (double)dpk, td = (double)u_;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tn += __shfl_xor_sync(0xffffffffu, tn, o);
      td += __shfl_xor_sync(0xffffffffu, td, o);
    }
    num += tn;
    den += td;
#pragma unroll
    for (int c = 0; c < NCH; ++c)
      if (c == ch) {
        keyr[c] = my.x;
        ur[c] = u_;
        pr[c] = p_;
        dpr[c] = dpk;
      }
  }
  const double dlt = den > 0.0 ? num / den : 0.0;
  if (lane == 0) {
    const double B = 1.0 - (alpha - 1.0) * row_max[r];
    delta[r] = dlt;
    rowc[r] = make_float2((float)(B - tau[r]), (float)dlt);
  }
  if (!want_dq || hflag[bh]) return;
  // phase 2: dQ_i = scale * sum_j dS_j k_j, dS_j = u_j (dp_j - delta_i)
  const float dl = (float)dlt;
  float acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.f;
  // d = 64: half-warps take alternate entries, 4 elements (8 bytes) a lane
  const int hf = lane >> 4, hl = lane & 15;
  const uint16_t* kb4 = kk + bh * (size_t)m * D + hl * 4;
  float a4[4] = {0.f, 0.f, 0.f, 0.f};
  // one chunk of up to 32 entries: scatter into the key lists, accumulate dS k_j
  auto dq_chunk = [&](int b, uint32_t keyc, float pc, float dsc) {
    const int nk = min(32, tot - b);
    if (koff && lane < nk) {  // this entry into its key's list (sorted by row in the keys kernel)
      const size_t kj = bh * (size_t)m + keyc;
      // head bh's lists live in its own n * cap entries
      const size_t slot = bh * (size_t)n * cap + (size_t)(koff[kj + bh] + atomicAdd(&kcur[kj], 1));
      krow[slot] = (int)(r - bh * n);
      kpd[slot] = make_float2(pc, dsc);
    }
    if constexpr (D == 64) {
#pragma unroll kGatherUnroll
      for (int k2 = 0; k2 < (nk + 1) / 2; ++k2) {
        const int k = 2 * k2 + hf;
        const uint32_t key = __shfl_sync(0xffffffffu, keyc, k & 31);
        const float ds = __shfl_sync(0xffffffffu, dsc, k & 31);
        if (k < nk) {
          const uint2 w = *reinterpret_cast<const uint2*>(kb4 + (size_t)key * D);
          a4[0] = fmaf(ds, __uint_as_float(w.x << 16), a4[0]);
          a4[1] = fmaf(ds, __uint_as_float(w.x & 0xFFFF0000u), a4[1]);
          a4[2] = fmaf(ds, __uint_as_float(w.y << 16), a4[2]);
          a4[3] = fmaf(ds, __uint_as_float(w.y & 0xFFFF0000u), a4[3]);
        }
      }
      return;
    }
#pragma unroll kGatherUnroll
    for (int k = 0; k < nk; ++k) {
      const uint32_t key = __shfl_sync(0xffffffffu, keyc, k);
      const float ds = __shfl_sync(0xffffffffu, dsc, k);
      float x[E];
      ld_row(kb + (size_t)key * D, x);
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] = fmaf(ds, x[e], acc[e]);
    }
  };
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    if (c * 32 >= tot) break;
    dq_chunk(c * 32, keyr[c], pr[c], ur[c] * (dpr[c] - dl));
  }
  for (int b = NCH * 32; b < tot; b += 32) {  // beyond the registers: entries and dp again
    const int idx = b + lane;
    uint2 my = make_uint2(0u, 0u);
    if (idx < tot) my = idx < c0 ? base[h0.y + idx] : base[h1.y + idx - c0];
    float pc, uc;
    pu_of<AK>(__uint_as_float(my.y), e0f, e1f, pc, uc);
    if (idx >= tot) uc = 0.f;
    float dpc = 0.f;
    if (idx < tot) {
      const uint4* vr = reinterpret_cast<const uint4*>(vv + (bh * (size_t)m + my.x) * D);
      float s0 = 0.f, s1 = 0.f;
#pragma unroll 4
      for (int x = 0; x < D / 8; ++x) {
        const uint4 w = vr[x];
        const float4 o0 = sdo[wi][2 * x], o1 = sdo[wi][2 * x + 1];
        s0 = fmaf(o0.x, __uint_as_float(w.x << 16), s0);
        s1 = fmaf(o0.y, __uint_as_float(w.x & 0xFFFF0000u), s1);
        s0 = fmaf(o0.z, __uint_as_float(w.y << 16), s0);
        s1 = fmaf(o0.w, __uint_as_float(w.y & 0xFFFF0000u), s1);
        s0 = fmaf(o1.x, __uint_as_float(w.z << 16), s0);
        s1 = fmaf(o1.y, __uint_as_float(w.z & 0xFFFF0000u), s1);
        s0 = fmaf(o1.z, __uint_as_float(w.w << 16), s0);
        s1 = fmaf(o1.w, __uint_as_float(w.w & 0xFFFF0000u), s1);
      }
      dpc = s0 + s1;
    }
    dq_chunk(b, my.x, pc, uc * (dpc - dl));
  }
  if constexpr (D == 64) {  // (even entries) + (odd entries); the first half-warp writes
#pragma unroll
    for (int e = 0; e < 4; ++e) a4[e] += __shfl_xor_sync(0xffffffffu, a4[e], 16);
    if (hf) return;
    if (out_f64) {
      double* dst = reinterpret_cast<double*>(dq) + r * D + hl * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) dst[e] = (double)(scale * a4[e]);
    } else {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(dq) + r * D + hl * 4) =
          make_float4(scale * a4[0], scale * a4[1], scale * a4[2], scale * a4[3]);
    }
    return;
  }
  if (out_f64) {
    double* dst = reinterpret_cast<double*>(dq) + r * D + lane * E;
#pragma unroll
    for (int e = 0; e < E; ++e) dst[e] = (double)(scale * acc[e]);
  } else {
    float* dst = reinterpret_cast<float*>(dq) + r * D + lane * E;
    if constexpr (E == 4) {
      *reinterpret_cast<float4*>(dst) = make_float4(scale * acc[0], scale * acc[1], scale * acc[2], scale * acc[3]);
    } else {
      *reinterpret_cast<float2*>(dst) = make_float2(scale * acc[0], scale * acc[1]);
    }
  }
}

// exclusive prefix of the per-key support counts (the forward's atomics), one CTA per head
// (koff[h (m + 1) + j]; heads with a flagged block are skipped)
__global__ void __launch_bounds__(1024) supp_scan_kernel(const int32_t* __restrict__ kcnt,
                                                         int32_t* koff, const uint32_t* hflag, int m) {
  const int h = blockIdx.x;
  if (hflag[h]) return;
  __shared__ int ws[32];
  const int32_t* c = kcnt + (size_t)h * m;
  int32_t* o = koff + (size_t)h * (m + 1);
  const int T = blockDim.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int per = (m + T - 1) / T;
  const int b0 = min(m, t * per), b1 = min(m, b0 + per);
  int sum = 0;
  for (int i = b0; i < b1; ++i) sum += c[i];
  int x = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  if (w == 0) {
    int y = lane < T / 32 ? ws[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int z = __shfl_up_sync(0xffffffffu, y, d);
      if (lane >= d) y += z;
    }
    ws[lane] = y;
  }
  __syncthreads();
  int pre = (w ? ws[w - 1] : 0) + x - sum;
  for (int i = b0; i < b1; ++i) {
    o[i] = pre;
    pre += c[i];
  }
  if (t == T - 1) o[m] = pre;
}

// dK and dV from the support lists, key-major: key j's entries (query row i, p_ij,
// dS_ij) -- scattered by the rows kernel in arbitrary order -- are sorted by row (a
// bitonic sort in shared memory: the summation order, and so every bit of the result,
// is fixed), then dV_j = sum_i p_ij dO_i and dK_j = scale sum_i dS_ij q_i over gathered
// dO / Q rows (attention.cpp:464-506: the terms vanish off the support).  One warp per
// key; a key with more than kMaxKey entries flags its head (the tensor-core dK/dV
// kernel, launched after this one, then takes the whole head).
// Two launches: keys with <= 256 entries, one warp each and 8 warps per CTA (16 KB of
// shared memory: high occupancy for the latency-bound gathers), which queue the longer
// lists (the first keys of a causal head: ~30 ln(n / j) entries) in klong; then a
// persistent launch whose warps take the queued keys (<= 4096 entries, 32 KB per warp).
template <int D, int KMAX, int WARPS, bool LONG>
__global__ void __launch_bounds__(WARPS * 32) sparse_keys_kernel(
    const uint16_t* __restrict__ dout, const uint16_t* __restrict__ qq,
    const int32_t* __restrict__ koff, const int32_t* __restrict__ krow,
    const float2* __restrict__ kpd, uint32_t* hflag, int32_t* klong, int cap, float scale,
    size_t keys, int n, int m, int out_f64, void* dk, void* dv, int shfl_sort) {
  constexpr int E = D / 32;
  __shared__ unsigned long long sk[WARPS][KMAX];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  size_t kr = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = (size_t)gridDim.x * WARPS;
  const size_t nlong = LONG ? (size_t)klong[0] : 0;
  for (size_t it = kr;; it += nwarps) {  // (short lists: one key per warp, no loop)
  if (LONG) {
    if (it >= nlong) return;
    kr = (size_t)klong[1 + it];
  } else {
    if (it != kr || kr >= keys) return;
  }
  const size_t bh = kr / (size_t)m;
  const size_t j = kr - bh * m;
  const int o0 = koff[bh * (m + 1) + j], o1 = koff[bh * (m + 1) + j + 1];  // (beside hflag)
  if (hflag[bh]) continue;
  const int cntk = o1 - o0;
  const size_t s0 = bh * (size_t)n * cap + (size_t)o0;
  if (!LONG && cntk > KMAX) {  // queued for the long-list launch
    if (lane == 0) klong[1 + atomicAdd(&klong[0], 1)] = (int32_t)kr;
    return;
  }
  if (cntk > KMAX) {  // the tensor-core dK/dV kernel (launched after this one) takes the head
    if (lane == 0) atomicOr(&hflag[bh], 1u);
    continue;
  }
  unsigned long long* sm = sk[wi];
  int np = 32;
  while (np < cntk) np <<= 1;
  if (shfl_sort && np == 32) {  // one entry per lane: the same bitonic network in registers
    unsigned long long x = lane < cntk ? ((unsigned long long)(uint32_t)krow[s0 + lane] << 32) | (uint32_t)lane : ~0ull;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, x, jj);
        const bool take_min = ((lane & jj) == 0) == ((lane & k) == 0);
        x = take_min ? (x < y ? x : y) : (x < y ? y : x);
      }
    sm[lane] = x;
    __syncwarp();
  } else {
  for (int i = lane; i < np; i += 32)
    sm[i] = i < cntk ? ((unsigned long long)(uint32_t)krow[s0 + i] << 32) | (uint32_t)i : ~0ull;
  __syncwarp();
  for (int k = 2; k <= np; k <<= 1)
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int i = lane; i < np; i += 32) {
        const int ixj = i ^ jj;
        if (ixj > i) {
          const unsigned long long x = sm[i], y = sm[ixj];
          if ((x > y) == ((i & k) == 0)) {
            sm[i] = y;
            sm[ixj] = x;
          }
        }
      }
      __syncwarp();
    }
  }
  if constexpr (D == 64) {  // half-warps take alternate entries, 4 elements (8 bytes) a lane
    const int hf = lane >> 4, hl = lane & 15;
    const uint16_t* db4 = dout + bh * (size_t)n * D + hl * 4;
    const uint16_t* qb4 = qq + bh * (size_t)n * D + hl * 4;
    float av[4] = {0.f, 0.f, 0.f, 0.f}, ak[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll kGatherUnroll
    for (int i = hf; i < cntk; i += 2) {
      const unsigned long long x = sm[i];
      const uint32_t row = (uint32_t)(x >> 32), sl = (uint32_t)x;
      const float2 pd = kpd[s0 + sl];
      const uint2 w0 = *reinterpret_cast<const uint2*>(db4 + (size_t)row * D);
      const uint2 w1 = *reinterpret_cast<const uint2*>(qb4 + (size_t)row * D);
      av[0] = fmaf(pd.x, __uint_as_float(w0.x << 16), av[0]);
      av[1] = fmaf(pd.x, __uint_as_float(w0.x & 0xFFFF0000u), av[1]);
      av[2] = fmaf(pd.x, __uint_as_float(w0.y << 16), av[2]);
      av[3] = fmaf(pd.x, __uint_as_float(w0.y & 0xFFFF0000u), av[3]);
      ak[0] = fmaf(pd.y, __uint_as_float(w1.x << 16), ak[0]);
      ak[1] = fmaf(pd.y, __uint_as_float(w1.x & 0xFFFF0000u), ak[1]);
      ak[2] = fmaf(pd.y, __uint_as_float(w1.y << 16), ak[2]);
      ak[3] = fmaf(pd.y, __uint_as_float(w1.y & 0xFFFF0000u), ak[3]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {  // even entries + odd entries (the same sum on both halves)
      av[e] += __shfl_xor_sync(0xffffffffu, av[e], 16);
      ak[e] += __shfl_xor_sync(0xffffffffu, ak[e], 16);
    }
    if (hf == 0) {
      const size_t orow = kr * D + hl * 4;
      if (out_f64) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          reinterpret_cast<double*>(dv)[orow + e] = (double)av[e];
          reinterpret_cast<double*>(dk)[orow + e] = (double)(scale * ak[e]);
        }
      } else {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(dv) + orow) = make_float4(av[0], av[1], av[2], av[3]);
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(dk) + orow) =
            make_float4(scale * ak[0], scale * ak[1], scale * ak[2], scale * ak[3]);
      }
    }
    __syncwarp();
    continue;
  }
  const uint16_t* db = dout + bh * (size_t)n * D + lane * E;
  const uint16_t* qb = qq + bh * (size_t)n * D + lane * E;
  float av[E], ak[E];
#pragma unroll
  for (int e = 0; e < E; ++e) av[e] = ak[e] = 0.f;
#pragma unroll kGatherUnroll
  for (int i = 0; i < cntk; ++i) {
    const unsigned long long x = sm[i];
    const uint32_t row = (uint32_t)(x >> 32), sl = (uint32_t)x;
    const float2 pd = kpd[s0 + sl];
    float od[E], oq[E];
    if constexpr (E == 4) {
      const uint2 w0 = *reinterpret_cast<const uint2*>(db + (size_t)row * D);
      const uint2 w1 = *reinterpret_cast<const uint2*>(qb + (size_t)row * D);
      od[0] = __uint_as_float(w0.x << 16); od[1] = __uint_as_float(w0.x & 0xFFFF0000u);
      od[2] = __uint_as_float(w0.y << 16); od[3] = __uint_as_float(w0.y & 0xFFFF0000u);
      oq[0] = __uint_as_float(w1.x << 16); oq[1] = __uint_as_float(w1.x & 0xFFFF0000u);
      oq[2] = __uint_as_float(w1.y << 16); oq[3] = __uint_as_float(w1.y & 0xFFFF0000u);
    } else {
      const uint32_t w0 = *reinterpret_cast<const uint32_t*>(db + (size_t)row * D);
      const uint32_t w1 = *reinterpret_cast<const uint32_t*>(qb + (size_t)row * D);
      od[0] = __uint_as_float(w0 << 16); od[1] = __uint_as_float(w0 & 0xFFFF0000u);
      oq[0] = __uint_as_float(w1 << 16); oq[1] = __uint_as_float(w1 & 0xFFFF0000u);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      av[e] = fmaf(pd.x, od[e], av[e]);
      ak[e] = fmaf(pd.y, oq[e], ak[e]);
    }
  }
  const size_t orow = kr * D + lane * E;
  if (out_f64) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      reinterpret_cast<double*>(dv)[orow + e] = (double)av[e];
      reinterpret_cast<double*>(dk)[orow + e] = (double)(scale * ak[e]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      reinterpret_cast<float*>(dv)[orow + e] = av[e];
      reinterpret_cast<float*>(dk)[orow + e] = scale * ak[e];
    }
  }
  __syncwarp();  // (the shared-memory list is reused by the warp's next key)
  }
}

constexpr int kKvThreads = 352;  // pair dK/dV: 8 epilogue warps, producer, 2 MMA issuers

template <int D>
struct Kv2Smem {
  static_assert(D == 128, "pair dK/dV kernel: d = 128");
  static constexpr int KVB = KB * D * 2;
  static constexpr int HB = 32 * D * 2;       // 32 queries x d (QS, DS)
  static constexpr int DB = QT * 64 * 2;      // 64 queries x 64 d (QD, DD)
  static constexpr int STAGE = 2 * HB + 2 * DB + 1024;  // + rowc[64]
  static constexpr int KST2 = 4;
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + KVB;
  static constexpr int OFF_ST = OFF_V + KVB;
  static constexpr int OFF_BAR = OFF_ST + KST2 * STAGE;
  static constexpr int OFF_MISC = OFF_BAR + 40 * 8;
  static constexpr int OFF_UB = OFF_MISC + 64;
  __host__ __device__ static int off_list(int t_r) { return OFF_UB + (t_r + 15) / 16 * 16; }
  // + the compacted active-unit list (t_r u16)
  static size_t bytes(int t_r) { return 1024 + off_list(t_r) + 2 * t_r + 64; }
};

// SLOT3 (fp16 P and fp16 dS heads only): TMEM holds three 64-column S^T slots and one
// dP^T slot instead of two S^T + dP^T buffers.  The epilogue reads S^T(u) and dP^T(u),
// releases the dP^T slot at once, and writes the packed P^T and dS^T (16 columns per
// 32-query half each) over S^T(u)'s own slot; so dP^T(u+1) needs only the epilogue's
// loads of unit u, and S^T(u+3) the gradient products of unit u -- the S^T -> epilogue
// -> gradients -> S^T(u+2) chain that left the two-buffer pipe ~40% idle (trace:
// 1880 cycles per unit against 1152 of MMA work) is broken.  Heads whose fp16 plan
// fails run in a second launch of the two-buffer kernel (skip_f16 = the other heads).
template <int D, int AK, bool DSF16, bool SLOT3 = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kKvThreads, 1)
    tc_dkdv2_kernel(const __grid_constant__ CUtensorMap tm_qh, const __grid_constant__ CUtensorMap tm_qd,
                    const __grid_constant__ CUtensorMap tm_kb, const __grid_constant__ CUtensorMap tm_vb,
                    const __grid_constant__ CUtensorMap tm_doh, const __grid_constant__ CUtensorMap tm_dod,
                    const __grid_constant__ CUtensorMap tm_dod16, const __grid_constant__ CUtensorMap tm_qd16,
                    const BwdArgs a) {
  using L = Kv2Smem<D>;
  // fp16 gradient products (F16Plan): dV = P^T dO (P in [0, 1]) and dK = (sigma dS)^T Q,
  // one MMA per K step each instead of the bf16 hi + lo pairs
  constexpr int KS = L::KST2;
  constexpr int NCH = D / 64;
  const Geom& g = a.g;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  uint8_t* sSt = smem + L::OFF_ST;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full = bars;             // [KS] leader: QS, DS, QD, DD of both CTAs
  uint64_t* empty = full + KS;       // [KS] each CTA (multicast commit)
  uint64_t* rfull = empty + KS;      // [KS] each CTA: its rowc copy
  uint64_t* s_full = rfull + KS;     // [2] each CTA
  uint64_t* p_full = s_full + 2;     // [2] leader, 16 warps
  uint64_t* kv_full = p_full + 2;    // leader
  uint64_t* acc_full = kv_full + 1;  // each CTA
  uint64_t* grad_done = acc_full + 1;  // [2] leader: gradient MMAs of the unit in S buffer b done
  // SLOT3: s3_full / p3_full / g3_done per S^T slot [3], dp_free (leader, 16 warps)
  uint64_t* s3_full = grad_done + 2;
  uint64_t* p3_full = s3_full + 3;
  uint64_t* g3_done = p3_full + 3;
  uint64_t* dp_free = g3_done + 3;
  volatile uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::OFF_MISC);
  uint8_t* ubits = smem + L::OFF_UB;  // [t_r]: bit 2r+kh = block (i, key tile kh of CTA r)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_ctarank();
  const bool lead_cta = rank == 0;
  const int npair = g.m / (2 * KB);
  const int pair = (int)(blockIdx.x >> 1);
  const int bh = pair / npair;          // head-major
  const F16Plan* pl = a.f16 ? a.f16 + bh : nullptr;  // the head's fp16 plan
  const bool f16 = pl && pl->dv_ok;
  const bool f16s = DSF16 && f16 && pl->ds_ok;  // (fp16 dS only with fp16 P: 3 epilogue variants)
  const float sig = f16s ? pl->sigma : 1.f;
  // (uniform per cluster: both CTAs belong to head bh)
  if constexpr (SLOT3) {
    if (!f16s) return;
  } else {
    if (a.skip_f16 && f16s) return;
  }
  const int kp = pair % npair;          // low key pairs (most query units) first
  const int pkey0 = kp * 2 * KB;
  const int key0 = pkey0 + (int)rank * KB;
  const int pj0 = pkey0 / 64;           // first of the pair's four reference key tiles
  const int i_first = g.causal ? pkey0 / QT : 0;

  if (a.kv_skip && a.kv_skip[bh] == 0u) return;  // dK/dV from the support lists (both CTAs)
  units_from_lists(ubits, 4, a, bh, pj0, threadIdx.x, kKvThreads);
  if (tid == 0) {
    for (int i = 0; i < KS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 2);  // S^T/dP^T reads (warp 9) and gradient reads (warp 10)
      mbar_init(&rfull[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 16);
    }
    mbar_init(kv_full, 1);
    mbar_init(acc_full, 1);
    mbar_init(&grad_done[0], 1);
    mbar_init(&grad_done[1], 1);
    for (int i = 0; i < 3; ++i) {
      mbar_init(&s3_full[i], 1);
      mbar_init(&p3_full[i], 16);
      mbar_init(&g3_done[i], 1);
    }
    mbar_init(dp_free, 16);
    fence_barrier_init();
  }
  if (warp == 8) tmem_alloc_2sm(const_cast<uint32_t*>(s_tmem), 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  // the CTA's active query units, compacted once
  uint16_t* sList = reinterpret_cast<uint16_t*>(smem + L::off_list(g.t_r));
  volatile uint32_t* sListN = reinterpret_cast<volatile uint32_t*>(smem + L::OFF_MISC) + 2;
  if (warp == 0)
    compact_active(sList, sListN, g.t_r - 1, lane, [&](int i) -> bool { return ubits[i] != 0; });
  __syncthreads();
  ActiveList walk{sList, (int)*sListN, 0};
  auto next_unit = [&](int i) -> int { return walk.next(i); };

  if (warp == 8) {  // TMA producer (both CTAs)
    const bool leader = elect_one_sync();
    const int krow = bh * g.m + key0;
    if (lead_cta && leader) mbar_expect_tx(kv_full, 2 * 2 * L::KVB);
    for (int c = 0; c < NCH; ++c) {
      if (leader) tma_load_2d_2sm(sK + c * KB * 128, &tm_kb, kv_full, c * 64, krow);
      if (leader) tma_load_2d_2sm(sV + c * KB * 128, &tm_vb, kv_full, c * 64, krow);
    }
    uint32_t u = 0;
    for (int i = next_unit(i_first); i >= 0; i = next_unit(i + 1), ++u) {
      const uint32_t st = u % KS;
      mbar_wait(&empty[st], ((u / KS) & 1) ^ 1);
      uint8_t* base = sSt + st * L::STAGE;
      const int qrow = bh * g.n + i * QT;
      if (lead_cta && leader) mbar_expect_tx(&full[st], 2 * (2 * L::HB + 2 * L::DB));
      // one 3-D box per 32-query half carries both d chunks (TMA costs ~240 cycles per
      // box below 16 KB: 7 boxes per unit outran the unit's MMAs, 5 do not)
      if (leader) tma_load_3d_2sm(base, &tm_qh, &full[st], qrow + 32 * (int)rank);
      if (leader) tma_load_3d_2sm(base + L::HB, &tm_doh, &full[st], qrow + 32 * (int)rank);
      if (leader) tma_load_2d_2sm(base + 2 * L::HB, f16s ? &tm_qd16 : &tm_qd, &full[st], 64 * (int)rank, qrow);
      if (leader)
        tma_load_2d_2sm(base + 2 * L::HB + L::DB, f16 ? &tm_dod16 : &tm_dod, &full[st], 64 * (int)rank, qrow);
      if (leader) mbar_expect_tx(&rfull[st], QT * 8);
      if (leader) bulk_load(base + 2 * L::HB + 2 * L::DB, a.rowc + qrow, QT * 8, &rfull[st]);
    }
  } else if (warp == 9 || warp == 10) {  // MMA issuers: pair leader only
    // Two issuing warps on different SM sub-partitions: warp 9 issues S^T / dP^T of
    // every unit, warp 10 the gradient products; the tensor pipe queues about one MMA
    // ahead, so each warp's waits and bookkeeping are covered by the other's MMAs.
    // S buffer b = u & 1: S^T/dP^T(u + 2) waits until the gradients of unit u (which
    // read P/dS(u) from that buffer) are done (grad_done[b]).
    if (lead_cta) {
      const bool leader = elect_one_sync();
      constexpr uint32_t IDESC_S = idesc_bf16_f32(256, QT, false, false);
      constexpr uint32_t IDESC_G = idesc_bf16_f32(256, D, false, true);
      constexpr uint32_t IDESC_G16 = idesc_f16_f32(256, D, false, true);
      const uint32_t k_addr = smem_u32(sK), v_addr = smem_u32(sV), st_addr = smem_u32(sSt);
      mbar_wait(kv_full, 0);
      tc_fence_after();
#ifdef ADATTN_PIPE_STATS
      const long long t_m0 = clock64();
#endif
      uint32_t u = 0;
      if (warp == 9 && SLOT3) {
        const uint64_t dK0 = desc_kmajor(k_addr), dV0 = desc_kmajor(v_addr);
        const uint64_t dQS0 = desc_kmajor(st_addr), dDS0 = desc_kmajor(st_addr + L::HB);
        for (int i = next_unit(i_first); i >= 0; i = next_unit(i + 1), ++u) {
          const uint32_t st = u % KS, x = u % 3;
          mbar_wait(&full[st], (u / KS) & 1);
          mbar_wait(&g3_done[x], ((u / 3) & 1) ^ 1);  // slot x: unit u-3's gradients done
          tc_fence_after();
          const uint64_t so = (uint64_t)((st * (uint32_t)L::STAGE) >> 4);
          if (leader)
            umma_ss_d128<2, ((KB * 128) >> 4), ((32 * 128) >> 4)>(tmem + x * 64, dK0, dQS0 + so, IDESC_S, 0u);
          if (u > 0) mbar_wait(dp_free, (u - 1) & 1);  // unit u-1's dP^T loaded by every warp
          tc_fence_after();
          if (leader)
            umma_ss_d128<2, ((KB * 128) >> 4), ((32 * 128) >> 4)>(tmem + 192, dV0, dDS0 + so, IDESC_S, 0u);
          if (leader) umma2_commit_mc(&s3_full[x]);
          if (leader) umma2_commit_mc(&empty[st]);
        }
      } else if (warp == 9) {
        const uint64_t dK0 = desc_kmajor(k_addr), dV0 = desc_kmajor(v_addr);
        const uint64_t dQS0 = desc_kmajor(st_addr), dDS0 = desc_kmajor(st_addr + L::HB);
        for (int i = next_unit(i_first); i >= 0; i = next_unit(i + 1), ++u) {
          const uint32_t st = u % KS, b = u & 1;
          if (leader) BTRACE(0, u, 0);
          {
            BSTAT_T0();
            mbar_wait(&full[st], (u / KS) & 1);
            BSTAT_ADD(0, leader);
          }
          if (leader) BTRACE(0, u, 1);
          {
            BSTAT_T0();
            mbar_wait(&grad_done[b], ((u >> 1) & 1) ^ 1);
            BSTAT_ADD(7, leader);
          }
          if (leader) BTRACE(0, u, 2);
          tc_fence_after();
          BSTAT_T0();
          const uint64_t so = (uint64_t)((st * (uint32_t)L::STAGE) >> 4);
          // S^T and dP^T as two 8-MMA chains (descriptors stepped inside one asm block)
          if (leader) {
            umma_ss_d128<2, ((KB * 128) >> 4), ((32 * 128) >> 4)>(tmem + b * 128, dK0, dQS0 + so, IDESC_S, 0u);
            umma_ss_d128<2, ((KB * 128) >> 4), ((32 * 128) >> 4)>(tmem + b * 128 + 64, dV0, dDS0 + so, IDESC_S, 0u);
          }
          if (leader) umma2_commit_mc(&s_full[b]);
          if (leader) umma2_commit_mc(&empty[st]);
          BSTAT_ADD(5, leader);
          if (leader) BTRACE(0, u, 3);
        }
      } else {
        const uint64_t dQD = desc_mnmajor(st_addr + 2 * L::HB, QT * 128);
        const uint64_t dDD = desc_mnmajor(st_addr + 2 * L::HB + L::DB, QT * 128);
        bool init = false;
        if constexpr (SLOT3) {
          for (int i = next_unit(i_first); i >= 0; i = next_unit(i + 1), ++u) {
            const uint32_t st = u % KS, x = u % 3;
            mbar_wait(&p3_full[x], (u / 3) & 1);
            tc_fence_after();
            const uint64_t so = (uint64_t)((st * (uint32_t)L::STAGE) >> 4);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              // queries 16k..16k+15: half k>>1's packed P^T at x*64 + 16(k>>1) + 8(k&1), dS^T +32
              const uint32_t pa = x * 64 + 16 * (k >> 1) + 8 * (k & 1);
              const uint32_t acc = (init || k > 0) ? 1u : 0u;
              if (leader) umma2_bf16_ts(tmem + 256, tmem + pa, dDD + so + (uint64_t)(128 * k), IDESC_G16, acc);
              if (leader)
                umma2_bf16_ts(tmem + 256 + D, tmem + pa + 32, dQD + so + (uint64_t)(128 * k), IDESC_G16, acc);
            }
            init = true;
            if (leader) umma2_commit_mc(&g3_done[x]);
            if (leader) umma2_commit_mc(&empty[st]);
          }
        } else
        for (int i = next_unit(i_first); i >= 0; i = next_unit(i + 1), ++u) {
          const uint32_t st = u % KS, b = u & 1;
          if (leader) BTRACE(1, u, 0);
          {
            BSTAT_T0();
            mbar_wait(&p_full[b], (u >> 1) & 1);
            BSTAT_ADD(1, leader);
          }
          if (leader) BTRACE(1, u, 1);
          tc_fence_after();
          BSTAT_T0();
          const uint64_t so = (uint64_t)((st * (uint32_t)L::STAGE) >> 4);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t acol = 32 * (k >> 1) + 8 * (k & 1);
            const uint64_t bdo = dDD + so + (uint64_t)(128 * k);
            const uint64_t bq = dQD + so + (uint64_t)(128 * k);
            const uint32_t acc = (init || k > 0) ? 1u : 0u;
            if (f16) {
              if (leader) umma2_bf16_ts(tmem + 256, tmem + b * 128 + acol, bdo, IDESC_G16, acc);
            } else {
              if (leader) umma2_bf16_ts(tmem + 256, tmem + b * 128 + acol, bdo, IDESC_G, acc);
              if (leader) umma2_bf16_ts(tmem + 256, tmem + b * 128 + acol + 16, bdo, IDESC_G, 1u);
            }
            if (f16s) {
              if (leader) umma2_bf16_ts(tmem + 256 + D, tmem + b * 128 + 64 + acol, bq, IDESC_G16, acc);
            } else {
              if (leader) umma2_bf16_ts(tmem + 256 + D, tmem + b * 128 + 64 + acol, bq, IDESC_G, acc);
              if (leader) umma2_bf16_ts(tmem + 256 + D, tmem + b * 128 + 64 + acol + 16, bq, IDESC_G, 1u);
            }
          }
          init = true;
          if (leader) umma2_commit_mc(&grad_done[b]);
          if (leader) umma2_commit_mc(&empty[st]);
          BSTAT_ADD(6, leader);
          if (leader) BTRACE(1, u, 2);
        }
        if (leader) umma2_commit_mc(acc_full);
      }
#ifdef ADATTN_PIPE_STATS
      if (leader && warp == 10) {
        atomicAdd(&g_bwd_stats[3], (unsigned long long)(clock64() - t_m0));
        atomicAdd(&g_bwd_stats[4], (unsigned long long)u);
      }
#endif
    }
  } else if (warp < 8) {  // epilogue (warp % 4 = TMEM lane quarter)
    const int half = warp >> 2;        // query columns 32*half .. +31
    const int lq = warp & 3;
    const int key = lq * 32 + lane;    // 0..127 within this CTA
    const int gkey = key0 + key;
    const int kbit = 2 * (int)rank + (key >> 6);
    const uint32_t tl = tmem + ((uint32_t)(lq * 32) << 16);
    const float A1 = a.A1;
    const uint32_t p_full_c0 = mapa_shared(smem_u32(&p_full[0]), 0);
    const uint32_t p_full_c1 = mapa_shared(smem_u32(&p_full[1]), 0);
    uint32_t u = 0;
    bool any = false;
    if constexpr (SLOT3) {
      const uint32_t dp_free_c = mapa_shared(smem_u32(dp_free), 0);
      for (int i = next_unit(i_first); i >= 0; i = next_unit(i + 1), ++u) {
        const uint32_t st = u % KS, x = u % 3;
        const bool mine = (ubits[i] >> kbit) & 1u;
        any |= mine;
        mbar_wait(&s3_full[x], (u / 3) & 1);
        mbar_wait(&rfull[st], (u / KS) & 1);
        tc_fence_after();
        float s[32], dp[32];
        tmem_ld32(tl + x * 64 + half * 32, s);
        tmem_ld32(tl + 192 + half * 32, dp);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(dp_free_c);  // dP^T slot read
        bar_sync(1, 256);  // every warp of this CTA has read S^T(u): slot x may be overwritten
        tc_fence_after();
        const float2* rc = reinterpret_cast<const float2*>(sSt + st * L::STAGE + 2 * L::HB + 2 * L::DB);
        uint32_t ph[16], pl[16], dh[16], dl[16];
        const int q0 = i * QT + half * 32;
        if (!mine) {
#pragma unroll
          for (int y = 0; y < 16; ++y) ph[y] = dh[y] = 0u;
        } else {
          const bool msk = g.causal && q0 < key0 + lq * 32 + 31;
          const int lim = msk ? gkey - q0 : 0;
          if (msk) pds_chunk<AK, true, true, true>(s, dp, rc + half * 32, A1, a.e0f, a.e1f, lim, ph, pl, dh, dl, sig);
          else pds_chunk<AK, false, true, true>(s, dp, rc + half * 32, A1, a.e0f, a.e1f, 0, ph, pl, dh, dl, sig);
        }
        tmem_st16(tl + x * 64 + half * 16, ph);
        tmem_st16(tl + x * 64 + 32 + half * 16, dh);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&p3_full[x]), 0));
      }
    } else
    for (int i = next_unit(i_first); i >= 0; i = next_unit(i + 1), ++u) {
      const uint32_t st = u % KS, b = u & 1;
      const bool mine = (ubits[i] >> kbit) & 1u;
      any |= mine;
      if (warp == 0 && lane == 0 && lead_cta) BTRACE(2, u, 0);
      {
        BSTAT_T0();
        mbar_wait(&s_full[b], (u >> 1) & 1);
        BSTAT_ADD(2, warp == 0 && lane == 0);
      }
      if (warp == 0 && lane == 0 && lead_cta) BTRACE(2, u, 1);
      mbar_wait(&rfull[st], (u / KS) & 1);
      tc_fence_after();
      float s[32], dp[32];
      tmem_ld32(tl + b * 128 + half * 32, s);
      tmem_ld32(tl + b * 128 + 64 + half * 32, dp);
      tmem_wait_ld();
      const float2* rc = reinterpret_cast<const float2*>(sSt + st * L::STAGE + 2 * L::HB + 2 * L::DB);
      uint32_t ph[16], pl[16], dh[16], dl[16];
      const int q0 = i * QT + half * 32;
      if (!mine) {
#pragma unroll
        for (int x = 0; x < 16; ++x) ph[x] = pl[x] = dh[x] = dl[x] = 0u;
      } else {
        const bool msk = g.causal && q0 < key0 + lq * 32 + 31;
        const int lim = msk ? gkey - q0 : 0;
        const float2* r2 = rc + half * 32;
#define PDS(M, FP, FS) pds_chunk<AK, M, FP, FS>(s, dp, r2, A1, a.e0f, a.e1f, lim, ph, pl, dh, dl, sig)
        if (f16s) { if (msk) PDS(true, true, true); else PDS(false, true, true); }
        else if (f16) { if (msk) PDS(true, true, false); else PDS(false, true, false); }
        else { if (msk) PDS(true, false, false); else PDS(false, false, false); }
#undef PDS
      }
      tmem_st16(tl + b * 128 + half * 32, ph);
      if (!f16) tmem_st16(tl + b * 128 + half * 32 + 16, pl);
      tmem_st16(tl + b * 128 + 64 + half * 32, dh);
      if (!f16s) tmem_st16(tl + b * 128 + 64 + half * 32 + 16, dl);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (warp == 0 && lane == 0 && lead_cta) BTRACE(2, u, 2);
      if (lane == 0) mbar_arrive_cluster(b ? p_full_c1 : p_full_c0);
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    any = __any_sync(0xffffffffu, any);
    const size_t krow = (size_t)bh * g.m + gkey;
#pragma unroll
    for (int which = 0; which < 2; ++which) {  // 0: dV, 1: dK
      void* base = which == 0 ? a.dv : a.dk;
      const float mul = which == 0 ? (f16 ? pl->inv_do : 1.f)
                                   : a.scale_f * (f16s ? pl->inv_sigma * pl->inv_q : 1.f);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        float o[32];
        tmem_ld32(tl + 256 + which * D + half * (D / 2) + c * 32, o);
        tmem_wait_ld();
        const int x0 = half * (D / 2) + c * 32;
        if (g.out_dtype == ADATTN_F64) {
          double* dst = reinterpret_cast<double*>(base) + krow * D + x0;
#pragma unroll
          for (int x = 0; x < 32; ++x) dst[x] = any ? (double)(mul * o[x]) : 0.0;
        } else {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(base) + krow * D + x0);
#pragma unroll
          for (int x = 0; x < 8; ++x)
            dst[x] = any ? make_float4(mul * o[4 * x], mul * o[4 * x + 1], mul * o[4 * x + 2],
                                       mul * o[4 * x + 3])
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 8) tmem_dealloc_2sm(tmem, 512);
}

// CTA-pair dQ kernel for d = 128 (ADATTN_DQ_PAIRS=0 selects the single-CTA kernel):
// 20.0 vs 24.6 ms at C3.
bool use_dq_pairs(const Geom& g) {
  const char* s = std::getenv("ADATTN_DQ_PAIRS");
  const int env = s ? std::atoi(s) : 1;
  return env != 0 && g.d == 128 && g.dv == 128 && g.n % (2 * QB_DQ) == 0;
}

// delta kernel: 0 single-CTA (256 rows), 1 CTA pair with 256 rows per CTA (the default:
// compensated fp32 sums, C3 11.4 ms vs 15.1 single), 2 pair with 128 rows per CTA and
// double-buffered S/dP (12.6 ms); ADATTN_DELTA_PAIRS overrides.  (Not launched when
// the forward folded the delta accumulation: delta_ubar_kernel instead.)
int delta_mode(const Geom& g, int ncta_rows) {
  if (g.d != 128 || g.dv != 128 || ncta_rows % 2 != 0) return 0;
  const char* s = std::getenv("ADATTN_DELTA_PAIRS");
  return s && *s ? std::atoi(s) : 1;  // C3: 15.1 (single) / 11.4 (1) / 12.6 (2) ms
}

// fp16 gradient products in the pair kernels: dV = P^T dO (default; ADATTN_DV_F16=0:
// bf16 hi + lo) and dQ = dS K, dK = dS^T Q with a power-of-two dS scale (default for
// alpha <= 1.5, ADATTN_DS_F16=0/1 overrides); each also falls back on the device when
// the data do not fit fp16 (F16Plan).  The d = 64 single-CTA kernels keep bf16 hi + lo:
// fp16 copies there added per-unit TMA boxes (TMA-bound at d = 64) and, in dK/dV, a
// stage size that no longer lets a second CTA's prologue overlap (C4: dK/dV 57.8 ->
// 58.0 ms, dQ 29.7 -> 33.1 ms; tried in round 2)
bool dv_f16_enabled() {
  const char* s = std::getenv("ADATTN_DV_F16");
  return !(s && *s == '0');
}
// fp16 dS: dQ/dK carry the fp16 rounding of dS (11 significant bits, ~2^-12 of
// max|grad|).  Measured against the bf16 hi/lo products (themselves within ~1e-4
// of the reference): alpha = 1.5 -> 3.4e-3 at N = 32K (max|dK| 15), 4.6e-3 at
// N = 128K (max|dK| 25): a 4-6x margin to the 2e-2 bar, -6% step time.  alpha = 2
// has ~2x larger gradients (7e-3 .. 9e-3, a 2x margin), so the default
// ("auto") takes fp16 dS for alpha <= 1.5 only; ADATTN_DS_F16=1 forces it (alpha
// <= 2, the plan's bound), =0 keeps hi/lo.
bool ds_f16_enabled(const Geom& g) {
  const char* s = std::getenv("ADATTN_DS_F16");
  if (s && *s == '1') return true;
  if (s && *s == '0') return false;
  return g.alpha <= 1.5;
}

// dQ from the support lists with delta (sparse_rows_kernel; ADATTN_SPARSE_DQ=0: the
// tensor-core dQ kernel)
bool sparse_dq_enabled() {
  const char* s = std::getenv("ADATTN_SPARSE_DQ");
  return !(s && *s == '0');
}
// key lists of <= 32 entries sorted with warp shuffles (ADATTN_KEYS_SHFL=0: in shared
// memory; the same network, bit-identical results)
bool keys_shfl_enabled() {
  const char* s = std::getenv("ADATTN_KEYS_SHFL");
  return !(s && *s == '0');
}
// dK/dV from the support lists (sparse_keys_kernel; ADATTN_SPARSE_KV=0: the tensor-core
// dK/dV kernel); needs the sparse dQ pass, which scatters the key lists
bool sparse_kv_enabled() {
  const char* s = std::getenv("ADATTN_SPARSE_KV");
  return !(s && *s == '0');
}

// three-slot pair dK/dV kernel for the fp16 P / dS heads (ADATTN_KV_SLOT3=0: two buffers)
bool kv_slot3_enabled(const Geom& g) {
  const char* s = std::getenv("ADATTN_KV_SLOT3");
  return !(s && *s == '0') && ds_f16_enabled(g) && dv_f16_enabled();
}

// CTA-pair dK/dV kernel for d = 128 (ADATTN_KV_PAIRS=0 selects the single-CTA kernel)
bool use_kv_pairs(const Geom& g) {
  const char* s = std::getenv("ADATTN_KV_PAIRS");
  const int env = s ? std::atoi(s) : 1;
  return env != 0 && g.d == 128 && g.dv == 128 && g.m % (2 * KB) == 0;
}

template <typename K>
cudaError_t set_smem(K kern, size_t bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int D, int AK>
cudaError_t run_bwd(const Geom& g, const CUtensorMap* m, const BwdArgs& a, bool delta_only,
                    cudaStream_t st) {
  cudaError_t e;
  const int dmode = delta_mode(g, a.ncta_rows);
  BwdArgs ad = a;  // the delta kernels' arguments (support mode: flagged heads only)
  const char* dname = "tc_delta";
  BwdArgs aq = a;   // the dQ kernels' arguments (support lists: flagged heads only)
  BwdArgs akv = a;  // the dK/dV kernels' arguments (likewise)
  bool want_kv = false;
  SuppLayout sl{};
  if (g.supp_in && !delta_only) {  // delta, dQ (and dK, dV) from the forward's support lists
    sl = supp_layout(g, const_cast<void*>(g.supp_in));
    const size_t rows = (size_t)g.bh * g.n;
    const bool want_dq = sparse_dq_enabled() && g.d == g.dv;
    want_kv = want_dq && sparse_kv_enabled();
    if (want_kv) {  // key-list offsets and cursors for the rows kernel's scatter
      if ((e = cudaMemsetAsync(sl.kcur, 0, 4 * (size_t)g.bh * g.m, st))) return e;
      supp_scan_kernel<<<(unsigned)g.bh, 1024, 0, st>>>(sl.kcnt, sl.koff, sl.hflag, g.m);
      note_launch();
      if ((e = cudaGetLastError())) return e;
    }
    prof_begin("tc_delta", st);
    sparse_rows_kernel<D, AK><<<(unsigned)((rows * 32 + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const uint16_t*>(a.dout), reinterpret_cast<const uint16_t*>(a.v),
        reinterpret_cast<const uint16_t*>(a.kp), sl.ent, sl.cnt, sl.flag, sl.hflag, sl.cap,
        dmode == 1 ? 512 : 256, want_kv ? sl.koff : nullptr, sl.kcur, sl.krow, sl.kpd, a.tau, a.row_max, g.alpha, a.e0f, a.e1f, (float)g.scale, rows,
        g.n, g.m, g.out_dtype == ADATTN_F64 ? 1 : 0, want_dq, a.dq, a.delta, a.rowc);
    prof_end(st);
    note_launch();
    if ((e = cudaGetLastError())) return e;
    ad.supp_skip = sl.flag;
    dname = "tc_delta_fb";
    if (want_dq) aq.dq_skip = sl.hflag;
    if (want_kv) akv.kv_skip = sl.hflag;
  }
  if (g.ubar_in && !delta_only) {  // delta from the forward's fold
    const size_t rows = (size_t)g.bh * g.n;
    prof_begin("tc_delta", st);
    delta_ubar_kernel<D><<<(unsigned)((rows * 32 + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const uint16_t*>(a.dout), g.ubar_in, a.tau, a.row_max, g.alpha, rows,
        a.delta, a.rowc);
    prof_end(st);
    note_launch();
    if ((e = cudaGetLastError())) return e;
  } else if (dmode == 2) {
    auto k0 = tc_delta3_kernel<128, AK>;
    const size_t sm = Delta3Smem<128>::bytes(g.wpr);
    if ((e = set_smem(k0, sm))) return e;
    prof_begin(dname, st);
    k0<<<dim3((unsigned)((g.n / 128) * g.bh)), kDeltaThreads, sm, st>>>(m[8], m[10], m[11], m[9], ad);
    prof_end(st);
    note_launch();
    if ((e = cudaGetLastError())) return e;
  } else if (dmode == 1) {
    auto k0 = tc_delta2_kernel<128, AK>;
    const size_t sm = Delta2Smem<128>::bytes(g.wpr);
    if ((e = set_smem(k0, sm))) return e;
    prof_begin(dname, st);
    k0<<<dim3((unsigned)(a.ncta_rows * g.bh)), kDeltaThreads, sm, st>>>(m[0], m[10], m[11], m[3], ad);
    prof_end(st);
    note_launch();
    if ((e = cudaGetLastError())) return e;
  } else {
    auto k0 = tc_delta_kernel<D, AK>;
    const size_t sm = DeltaSmem<D>::bytes(g.wpr);
    if ((e = set_smem(k0, sm))) return e;
    prof_begin(dname, st);
    k0<<<dim3((unsigned)(a.ncta_rows * g.bh)), kDeltaThreads, sm, st>>>(m[0], m[1], m[2], m[3], ad);
    prof_end(st);
    note_launch();
    if ((e = cudaGetLastError())) return e;
  }
  if (delta_only) return cudaSuccess;
  if (want_kv) {  // dK, dV from the support lists (heads without a flagged block)
    const size_t keys = (size_t)g.bh * g.m;
    prof_begin("tc_dkdv", st);
    if ((e = cudaMemsetAsync(sl.klong, 0, 4, st))) return e;
    sparse_keys_kernel<D, 256, 8, false><<<(unsigned)((keys + 7) / 8), 8 * 32, 0, st>>>(
        reinterpret_cast<const uint16_t*>(a.dout), reinterpret_cast<const uint16_t*>(a.qp),
        sl.koff, sl.krow, sl.kpd, sl.hflag, sl.klong, sl.cap, (float)g.scale, keys, g.n, g.m,
        g.out_dtype == ADATTN_F64 ? 1 : 0, a.dk, a.dv, keys_shfl_enabled() ? 1 : 0);
    note_launch();
    sparse_keys_kernel<D, 4096, 1, true><<<148 * 6, 32, 0, st>>>(
        reinterpret_cast<const uint16_t*>(a.dout), reinterpret_cast<const uint16_t*>(a.qp),
        sl.koff, sl.krow, sl.kpd, sl.hflag, sl.klong, sl.cap, (float)g.scale, keys, g.n, g.m,
        g.out_dtype == ADATTN_F64 ? 1 : 0, a.dk, a.dv, 0);
    prof_end(st);
    note_launch();
    if ((e = cudaGetLastError())) return e;
  }
  if (use_kv_pairs(g)) {
    const bool slot3 = kv_slot3_enabled(g) && a.f16;
    auto k2 = ds_f16_enabled(g) ? tc_dkdv2_kernel<128, AK, true> : tc_dkdv2_kernel<128, AK, false>;
    const size_t sm = Kv2Smem<128>::bytes(g.t_r);
    if ((e = set_smem(k2, sm))) return e;
    prof_begin(akv.kv_skip ? "tc_dkdv_fb" : "tc_dkdv", st);
    if (slot3) {  // fp16 P / dS heads, then (skip_f16) the rest with the two-buffer layout
      auto k3 = tc_dkdv2_kernel<128, AK, true, true>;
      if ((e = set_smem(k3, sm))) return e;
      k3<<<dim3((unsigned)((g.m / KB) * g.bh)), kKvThreads, sm, st>>>(m[12], m[4], m[5], m[6], m[13],
                                                                     m[7], m[14], m[16], akv);
      note_launch();
      BwdArgs a2 = akv;
      a2.skip_f16 = 1;
      k2<<<dim3((unsigned)((g.m / KB) * g.bh)), kKvThreads, sm, st>>>(m[12], m[4], m[5], m[6], m[13],
                                                                     m[7], m[14], m[16], a2);
    } else {
      k2<<<dim3((unsigned)((g.m / KB) * g.bh)), kKvThreads, sm, st>>>(m[12], m[4], m[5], m[6], m[13],
                                                                     m[7], m[14], m[16], akv);
    }
    prof_end(st);
    note_launch();
    if ((e = cudaGetLastError())) return e;
  } else {
    auto k2 = tc_dkdv_kernel<D, AK>;
    const size_t sm = KvSmem<D>::bytes(g.t_r);
    if ((e = set_smem(k2, sm))) return e;
    prof_begin(akv.kv_skip ? "tc_dkdv_fb" : "tc_dkdv", st);
    k2<<<dim3((unsigned)((g.m / KB) * g.bh)), kThreads, sm, st>>>(m[4], m[5], m[6], m[7], akv);
    prof_end(st);
    note_launch();
    if ((e = cudaGetLastError())) return e;
  }
  if (use_dq_pairs(g)) {
    auto k1 = ds_f16_enabled(g) ? tc_dq2_kernel<128, AK, true> : tc_dq2_kernel<128, AK, false>;
    const size_t sm = Dq2Smem<128>::bytes(g.wpr);
    if ((e = set_smem(k1, sm))) return e;
    prof_begin(aq.dq_skip ? "tc_dq_fb" : "tc_dq", st);
    k1<<<dim3((unsigned)((g.n / QB_DQ) * g.bh)), kThreads, sm, st>>>(m[8], m[10], m[1], m[11], m[9],
                                                                      m[15], aq);
    prof_end(st);
    note_launch();
    if ((e = cudaGetLastError())) return e;
  } else {
    auto k1 = tc_dq_kernel<D, AK>;
    const size_t sm = DqSmem<D>::bytes(g.wpr);
    if ((e = set_smem(k1, sm))) return e;
    prof_begin(aq.dq_skip ? "tc_dq_fb" : "tc_dq", st);
    k1<<<dim3((unsigned)((g.n / QB_DQ) * g.bh)), kThreads, sm, st>>>(m[8], m[1], m[2], m[9], aq);
    prof_end(st);
    note_launch();
    if ((e = cudaGetLastError())) return e;
  }
  return cudaSuccess;
}

template <int D>
cudaError_t run_bwd_d(const Geom& g, int ak, const CUtensorMap* m, const BwdArgs& a,
                      bool delta_only, cudaStream_t st) {
  switch (ak) {
    case AK15: return run_bwd<D, AK15>(g, m, a, delta_only, st);
    case AK2: return run_bwd<D, AK2>(g, m, a, delta_only, st);
    case AK125: return run_bwd<D, AK125>(g, m, a, delta_only, st);
    default: return run_bwd<D, AKGEN>(g, m, a, delta_only, st);
  }
}

}  // namespace

// rowc [bh*n] float2, then (fp16 gradient products) fp16 copies of dO, Q, K and the plan
static size_t ws_rowc(const Geom& g) { return ((size_t)g.bh * g.n * sizeof(float2) + 255) / 256 * 256; }
static size_t ws_h(const Geom& g, int cols, int rows) {
  return ((size_t)g.bh * rows * cols * 2 + 255) / 256 * 256;
}
// per-head plans + 4 per-head maxima
static size_t ws_plan(const Geom& g) {
  return ((size_t)g.bh * (sizeof(F16Plan) + 16) + 255) / 256 * 256;
}
// only what the enabled fp16 products need (ADATTN_DV_F16 / ADATTN_DS_F16 are read
// here and again at launch: change them between the query and the call and the
// C-ABI's workspace check fails loudly)
size_t backward_workspace(const Geom& g) {
  const bool pairs = g.d == 128 && g.dv == 128;
  const bool dvh = pairs && dv_f16_enabled(), dsh = pairs && ds_f16_enabled(g);
  return ws_rowc(g) + ell_bytes(g) + (dvh || dsh ? ws_h(g, g.dv, g.n) : 0) +
         (dsh ? ws_h(g, g.d, g.n) + ws_h(g, g.d, g.m) : 0) + ws_plan(g);
}

cudaError_t backward(const Geom& g, const void* q, const void* k, const void* v, const double* tau,
                     const double* row_max, const uint32_t* mask, const void* dout, void* dq,
                     void* dk, void* dv, double* delta, void* workspace, bool delta_only,
                     cudaStream_t st) {
  CUtensorMap m[17];
  cudaError_t e;
  const uint64_t nq = (uint64_t)g.bh * g.n, nk = (uint64_t)g.bh * g.m;
  if ((e = make_tmap_2d(&m[0], q, nq, g.d, BM))) return e;
  if ((e = make_tmap_2d(&m[1], k, nk, g.d, DBN))) return e;
  if ((e = make_tmap_2d(&m[2], v, nk, g.dv, DBN))) return e;
  if ((e = make_tmap_2d(&m[3], dout, nq, g.dv, BM))) return e;
  if ((e = make_tmap_2d(&m[4], q, nq, g.d, QT))) return e;
  if ((e = make_tmap_2d(&m[5], k, nk, g.d, KB))) return e;
  if ((e = make_tmap_2d(&m[6], v, nk, g.dv, KB))) return e;
  if ((e = make_tmap_2d(&m[7], dout, nq, g.dv, QT))) return e;
  if ((e = make_tmap_2d(&m[8], q, nq, g.d, QB_DQ))) return e;
  if ((e = make_tmap_2d(&m[9], dout, nq, g.dv, QB_DQ))) return e;
  if ((e = make_tmap_2d(&m[10], k, nk, g.d, 64))) return e;   // 64-key halves (pair dQ)
  if ((e = make_tmap_2d(&m[11], v, nk, g.dv, 64))) return e;
  // 32-query halves (pair dK/dV), both d chunks per box
  if ((e = make_tmap_3d_chunks(&m[12], q, nq, g.d, 32))) return e;
  if ((e = make_tmap_3d_chunks(&m[13], dout, nq, g.dv, 32))) return e;
  BwdArgs a;
  a.g = g;
  a.ncta_rows = g.n / BM;
  a.A1 = (float)((g.alpha - 1.0) * g.scale);
  a.e0f = (float)g.e0;
  a.e1f = (float)(g.e0 - 1.0);
  a.tau = tau;
  a.row_max = row_max;
  {  // the nonzero-block lists the kernels walk, from the forward's mask
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    uint8_t* w8 = reinterpret_cast<uint8_t*>(workspace) + ws_rowc(g);
    int32_t* rcnt = reinterpret_cast<int32_t*>(w8);
    w8 += al((size_t)g.bh * g.t_r * 4);
    uint16_t* rcol = reinterpret_cast<uint16_t*>(w8);
    w8 += al((size_t)g.bh * g.t_r * g.t_c * 2);
    int32_t* ccnt = reinterpret_cast<int32_t*>(w8);
    w8 += al((size_t)g.bh * g.t_c * 4);
    uint16_t* crow = reinterpret_cast<uint16_t*>(w8);
    const int32_t* rc = rcnt;
    const uint16_t* rl = rcol;
    if (g.rl_cnt_in && g.rl_col_in) {  // the forward's own lists
      rc = g.rl_cnt_in;
      rl = g.rl_col_in;
    } else if ((e = ell_row_lists(g, mask, rcnt, rcol, st))) {
      return e;
    }
    if (!delta_only && (e = ell_col_lists(g, rc, rl, ccnt, crow, st))) return e;
    a.rcnt = rc;
    a.rcol = rl;
    a.ccnt = ccnt;
    a.crow = crow;
  }
  a.delta = delta;
  a.rowc = reinterpret_cast<float2*>(workspace);
  a.dout = dout;
  a.v = v;
  a.kp = k;
  a.qp = q;
  a.supp_skip = nullptr;
  a.dq_skip = nullptr;
  a.kv_skip = nullptr;
  a.skip_f16 = 0;
  a.f16 = nullptr;
  m[14] = m[7];
  m[15] = m[1];
  m[16] = m[4];
  const bool want_dv = dv_f16_enabled(), want_ds = ds_f16_enabled(g);
  if (!delta_only && (use_kv_pairs(g) || use_dq_pairs(g)) && (want_dv || want_ds)) {
    // fp16 operand copies + range maxima, then the per-launch plan (device-side:
    // no host round trip); the pair kernels read it at start
    uint8_t* w8 = reinterpret_cast<uint8_t*>(workspace);
    size_t off = ws_rowc(g) + ell_bytes(g);
    __half2* do16 = reinterpret_cast<__half2*>(w8 + off);
    off += ws_h(g, g.dv, g.n);
    __half2* q16 = nullptr;
    __half2* k16 = nullptr;
    if (want_ds) {
      q16 = reinterpret_cast<__half2*>(w8 + off);
      off += ws_h(g, g.d, g.n);
      k16 = reinterpret_cast<__half2*>(w8 + off);
      off += ws_h(g, g.d, g.m);
    }
    F16Plan* plan = reinterpret_cast<F16Plan*>(w8 + off);
    uint32_t* mx = reinterpret_cast<uint32_t*>(plan + g.bh);  // [4][bh]
    const int H = g.bh;
    if ((e = cudaMemsetAsync(mx, 0, 16 * (size_t)H, st))) return e;
    // per head: dO [n][dv], V [m][dv], Q [n][d], K [m][d]
    const size_t eo = (size_t)g.n * g.dv, ev = (size_t)g.m * g.dv;
    const size_t eq = (size_t)g.n * g.d, ek = (size_t)g.m * g.d;
    // support-list backward: only heads the forward flagged reach the tensor-core
    // dQ / dK-dV kernels, so only they get fp16 copies
    const uint32_t* need = g.supp_in && sparse_dq_enabled() && sparse_kv_enabled() && g.d == g.dv
                               ? supp_layout(g, const_cast<void*>(g.supp_in)).hflag
                               : nullptr;
    if ((e = f16_absmax(dout, H, eo, mx, st, need))) return e;
    if (want_ds) {
      if ((e = f16_absmax(v, H, ev, mx + H, st, need))) return e;
      if ((e = f16_absmax(q, H, eq, mx + 2 * H, st, need))) return e;
      if ((e = f16_absmax(k, H, ek, mx + 3 * H, st, need))) return e;
    }
    f16_plan_kernel<<<(H + 127) / 128, 128, 0, st>>>(plan, mx, H, (float)g.alpha, g.d,
                                                     want_dv ? 1 : 0, want_ds ? 1 : 0);
    note_launch();
    if ((e = cudaGetLastError())) return e;
    if (want_dv && (e = f16_convert_scaled(dout, do16, H, eo, mx, st))) return e;
    if (want_ds) {
      if ((e = f16_convert_scaled(q, q16, H, eq, mx + 2 * H, st))) return e;
      if ((e = f16_convert_scaled(k, k16, H, ek, mx + 3 * H, st))) return e;
    }
    if ((e = make_tmap_2d(&m[14], do16, nq, g.dv, QT))) return e;
    if (want_ds) {
      if ((e = make_tmap_2d(&m[15], k16, nk, g.d, DBN))) return e;
      if ((e = make_tmap_2d(&m[16], q16, nq, g.d, QT))) return e;
    }
    a.f16 = plan;
  }
  a.dq = dq;
  a.dk = dk;
  a.dv = dv;
  a.scale_f = (float)g.scale;
  const int ak = alpha_kind(g.alpha);
  if (g.d == 64) return run_bwd_d<64>(g, ak, m, a, delta_only, st);
  return run_bwd_d<128>(g, ak, m, a, delta_only, st);
}

}  // namespace tc
}  // namespace adattn_b200

#ifdef ADATTN_PIPE_STATS
extern "C" void adattn_b200_bwd_trace(long long* out) {
  cudaMemcpyFromSymbol(out, adattn_b200::tc::g_btrace, sizeof(long long) * 3 * 512 * 4);
}
extern "C" void adattn_b200_bwd_stats(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, adattn_b200::tc::g_bwd_stats, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(adattn_b200::tc::g_bwd_stats, z, sizeof z);
  }
}
#endif
