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
#include <math_constants.h>

#include "common.cuh"
#include "tc.cuh"
#include "tc_common.cuh"
#include "tc_host.cuh"

namespace adattn_b200 {
namespace tc {
namespace {

constexpr int BM = 256;  // query rows per CTA (delta, dQ)
constexpr int BN = 64;   // keys per tile
constexpr int NST = 4;
constexpr int kThreads = 384;
constexpr int kEpi = 256;

struct BwdArgs {
  Geom g;
  int ncta_rows;
  float A1;
  float e0f, e1f;
  const double* tau;
  const double* row_max;
  const uint32_t* mask;
  double* delta;
  float2* rowc;  // [bh*n] {C, delta}
  void* dq;
  void* dk;
  void* dv;
  float scale_f;
};

enum AlphaKind { AK15 = 0, AK2 = 1, AK125 = 2, AKGEN = 3 };

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

// Shared geometry of the query-major kernels.
struct QmGeom {
  int bh, row0, jmax;
  int rg_jlim[2];
};

__device__ __forceinline__ QmGeom qm_geom(const Geom& g, int ncta_rows) {
  QmGeom q;
  q.bh = blockIdx.x % g.bh;
  const int crow = ncta_rows - 1 - blockIdx.x / g.bh;
  q.row0 = crow * BM;
  q.jmax = g.causal ? (q.row0 + BM - 1) / BN : g.t_c - 1;
  q.rg_jlim[0] = g.causal ? (q.row0 + 127) / BN : g.t_c - 1;
  q.rg_jlim[1] = q.jmax;
  return q;
}

// ================================================================== delta
// Query-major delta kernel: 256 rows per CTA (two M=128 row groups), S and dP
// double-buffered in TMEM (4 x 128 columns).
template <int D>
struct DeltaSmem {
  static constexpr int QB = BM * D * 2;
  static constexpr int TILE = BN * D * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_DO = OFF_Q + QB;
  static constexpr int OFF_RING = OFF_DO + QB;
  static constexpr int OFF_BAR = OFF_RING + NST * TILE;
  static constexpr int OFF_MISC = OFF_BAR + 32 * 8;
  static constexpr int OFF_MASK = OFF_MISC + 64;
  static size_t bytes(int wpr) { return 1024 + OFF_MASK + 4 * wpr * 4 + 64; }
};

template <int D, int AK>
__global__ void __launch_bounds__(kThreads, 1)
    tc_delta_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                    const BwdArgs a) {
  using L = DeltaSmem<D>;
  constexpr int NCH = D / 64;
  const Geom& g = a.g;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sDO = smem + L::OFF_DO;
  uint8_t* sRing = smem + L::OFF_RING;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full = bars;              // [NST]
  uint64_t* empty = bars + NST;       // [NST]
  uint64_t* s_full = bars + 2 * NST;  // [2]
  uint64_t* s_empty = s_full + 2;     // [2]
  uint64_t* q_full = s_empty + 2;
  volatile uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::OFF_MISC);
  uint32_t* smask = reinterpret_cast<uint32_t*>(smem + L::OFF_MASK);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const QmGeom G = qm_geom(g, a.ncta_rows);
  const int wpr = g.wpr;

  for (int i = tid; i < 4 * wpr; i += kThreads) {
    const int rbi = i / wpr, w = i - rbi * wpr;
    smask[i] = a.mask[((size_t)G.bh * g.t_r + (G.row0 / 64 + rbi)) * wpr + w];
  }
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 8);
    }
    mbar_init(q_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(const_cast<uint32_t*>(s_tmem), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  auto rb_active = [&](int rb, int j) -> bool {
    return (smask[rb * wpr + (j >> 5)] >> (j & 31)) & 1u;
  };
  auto rg_active = [&](int rg, int j) -> bool { return rb_active(2 * rg, j) || rb_active(2 * rg + 1, j); };
  auto next_active = [&](int j) -> int {
    for (; j <= G.jmax; ++j)
      if (rg_active(0, j) || rg_active(1, j)) return j;
    return -1;
  };

  if (warp == 0) {
    {
      const bool leader = elect_one_sync();
      const int qrow = G.bh * g.n + G.row0;
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
          if (leader) tma_load_2d(sRing + st * L::TILE + c * BN * 128, tm, &full[st], c * 64, row);
        ++r;
      };
      const int krow0 = G.bh * g.m;
      for (int j = next_active(0); j >= 0; j = next_active(j + 1)) {
        load(&tm_k, krow0 + j * BN);
        load(&tm_v, krow0 + j * BN);
      }
    }
  } else if (warp == 1) {
    {
      const bool leader = elect_one_sync();
      constexpr uint32_t IDESC_S = idesc_bf16_f32(128, BN, false, false);
      const uint32_t q_addr = smem_u32(sQ), do_addr = smem_u32(sDO), ring_addr = smem_u32(sRing);
      mbar_wait(q_full, 0);
      tc_fence_after();
      uint32_t item = 0, r = 0;
      for (int j = next_active(0); j >= 0; j = next_active(j + 1)) {
        const uint32_t b = item & 1;
        mbar_wait(&s_empty[b], ((item >> 1) & 1) ^ 1);
        const uint32_t kst = r % NST, vst = (r + 1) % NST;
        mbar_wait(&full[kst], (r / NST) & 1);
        mbar_wait(&full[vst], ((r + 1) / NST) & 1);
        tc_fence_after();
        for (int rg = 0; rg < 2; ++rg) {
          if (!rg_active(rg, j)) continue;
          const uint32_t sc = tmem + b * 256 + rg * 64;
          for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (leader) umma_bf16(sc, desc_kmajor(q_addr + c * BM * 128 + rg * 128 * 128 + k * 32),
                        desc_kmajor(ring_addr + kst * L::TILE + c * BN * 128 + k * 32), IDESC_S,
                        (c | k) != 0);
              if (leader) umma_bf16(sc + 128, desc_kmajor(do_addr + c * BM * 128 + rg * 128 * 128 + k * 32),
                        desc_kmajor(ring_addr + vst * L::TILE + c * BN * 128 + k * 32), IDESC_S,
                        (c | k) != 0);
            }
        }
        if (leader) umma_commit(&empty[kst]);
        if (leader) umma_commit(&empty[vst]);
        if (leader) umma_commit(&s_full[b]);
        ++item;
        r += 2;
      }
    }
  } else if (warp >= 4) {
    const int e = tid - 128;
    const int rg = e >> 7, lq = warp & 3, rb = e >> 6;
    const int grow = G.row0 + e;
    const size_t orow = (size_t)G.bh * g.n + grow;
    const uint32_t tl = tmem + ((uint32_t)(lq * 32) << 16);
    const float A1 = a.A1;
    const double B = 1.0 - (g.alpha - 1.0) * a.row_max[orow];
    const float C = (float)(B - a.tau[orow]);
    double num = 0.0, den = 0.0;
    uint32_t item = 0;
    for (int j = next_active(0); j >= 0; j = next_active(j + 1)) {
      const bool need = rg_active(rg, j);
      const bool mine = rb_active(rb, j);  // the reference visits set blocks only
      const uint32_t b = item & 1;
      mbar_wait(&s_full[b], (item >> 1) & 1);
      tc_fence_after();
      float s[64], dp[64];
      if (need) {
        tmem_ld32(tl + b * 256 + rg * 64, s);
        tmem_ld32(tl + b * 256 + rg * 64 + 32, s + 32);
        tmem_ld32(tl + b * 256 + 128 + rg * 64, dp);
        tmem_ld32(tl + b * 256 + 128 + rg * 64 + 32, dp + 32);
        tmem_wait_ld();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[b]);
      if (need && mine) {
        const bool diag = g.causal && j * BN + BN - 1 > grow;
        float n32 = 0.f, d32 = 0.f;
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          float t = fmaf(A1, s[i], C);
          if (diag && j * BN + i > grow) t = -1.f;
          float p, u;
          pu_of<AK>(t, a.e0f, a.e1f, p, u);
          n32 = fmaf(u, dp[i], n32);
          d32 += u;
        }
        num += (double)n32;
        den += (double)d32;
      }
      ++item;
    }
    const double dlt = den > 0.0 ? num / den : 0.0;
    a.delta[orow] = dlt;
    a.rowc[orow] = make_float2(C, (float)dlt);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// ===================================================================== dQ
// Query-major dQ kernel: 128 rows per CTA (one M=128 row group); the 8
// epilogue warps split each 64-key tile into two 32-column halves.
// dS = u (dp - delta) is split into bf16 hi + lo and both halves feed the
// dQ += dS K_j MMA (K_j read MN-major), so the bf16 rounding of dS drops out.
constexpr int QB_DQ = 128;

template <int D>
struct DqSmem {
  static constexpr int QB = QB_DQ * D * 2;
  static constexpr int TILE = BN * D * 2;
  static constexpr int DSB = QB_DQ * BN * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_DO = OFF_Q + QB;
  static constexpr int OFF_RING = OFF_DO + QB;
  static constexpr int OFF_DS = OFF_RING + NST * TILE;  // hi, lo
  static constexpr int OFF_BAR = OFF_DS + 2 * DSB;
  static constexpr int OFF_MISC = OFF_BAR + 32 * 8;
  static constexpr int OFF_MASK = OFF_MISC + 64;
  static size_t bytes(int wpr) { return 1024 + OFF_MASK + 2 * wpr * 4 + 64; }
};

template <int D, int AK>
__global__ void __launch_bounds__(kThreads, 1)
    tc_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                 const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                 const BwdArgs a) {
  using L = DqSmem<D>;
  constexpr int NCH = D / 64;
  const Geom& g = a.g;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sDO = smem + L::OFF_DO;
  uint8_t* sRing = smem + L::OFF_RING;
  uint8_t* sDS = smem + L::OFF_DS;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full = bars;              // [NST]
  uint64_t* empty = bars + NST;       // [NST]
  uint64_t* s_full = bars + 2 * NST;  // [2]
  uint64_t* s_empty = s_full + 2;     // [2]
  uint64_t* ds_full = s_empty + 2;
  uint64_t* ds_empty = ds_full + 1;
  uint64_t* acc_full = ds_empty + 1;
  uint64_t* q_full = acc_full + 1;
  volatile uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::OFF_MISC);
  uint32_t* smask = reinterpret_cast<uint32_t*>(smem + L::OFF_MASK);  // [2][wpr]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncta = g.n / QB_DQ;
  const int bh = blockIdx.x % g.bh;
  const int row0 = (ncta - 1 - blockIdx.x / g.bh) * QB_DQ;
  const int jmax = g.causal ? (row0 + QB_DQ - 1) / BN : g.t_c - 1;
  const int wpr = g.wpr;

  for (int i = tid; i < 2 * wpr; i += kThreads) {
    const int rbi = i / wpr, w = i - rbi * wpr;
    smask[i] = a.mask[((size_t)bh * g.t_r + (row0 / 64 + rbi)) * wpr + w];
  }
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 8);
    }
    mbar_init(ds_full, 8);
    mbar_init(ds_empty, 1);
    mbar_init(acc_full, 1);
    mbar_init(q_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(const_cast<uint32_t*>(s_tmem), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  auto rb_active = [&](int rb, int j) -> bool {
    return (smask[rb * wpr + (j >> 5)] >> (j & 31)) & 1u;
  };
  auto next_active = [&](int j) -> int {
    for (; j <= jmax; ++j)
      if (rb_active(0, j) || rb_active(1, j)) return j;
    return -1;
  };

  if (warp == 0) {
    {
      const bool leader = elect_one_sync();
      const int qrow = bh * g.n + row0;
      if (leader) mbar_expect_tx(q_full, 2 * L::QB);
      for (int c = 0; c < NCH; ++c) {
        if (leader) tma_load_2d(sQ + c * QB_DQ * 128, &tm_q, q_full, c * 64, qrow);
        if (leader) tma_load_2d(sDO + c * QB_DQ * 128, &tm_do, q_full, c * 64, qrow);
      }
      uint32_t r = 0;
      auto load = [&](const CUtensorMap* tm, int row) {
        const uint32_t st = r % NST, ph = (r / NST) & 1;
        mbar_wait(&empty[st], ph ^ 1);
        if (leader) mbar_expect_tx(&full[st], L::TILE);
        for (int c = 0; c < NCH; ++c)
          if (leader) tma_load_2d(sRing + st * L::TILE + c * BN * 128, tm, &full[st], c * 64, row);
        ++r;
      };
      const int krow0 = bh * g.m;
      for (int j = next_active(0); j >= 0; j = next_active(j + 1)) {
        load(&tm_k, krow0 + j * BN);
        load(&tm_v, krow0 + j * BN);
      }
    }
  } else if (warp == 1) {
    {
      const bool leader = elect_one_sync();
      constexpr uint32_t IDESC_S = idesc_bf16_f32(128, BN, false, false);
      constexpr uint32_t IDESC_DQ = idesc_bf16_f32(128, D, false, true);
      const uint32_t q_addr = smem_u32(sQ), do_addr = smem_u32(sDO);
      const uint32_t ring_addr = smem_u32(sRing), ds_addr = smem_u32(sDS);
      mbar_wait(q_full, 0);
      tc_fence_after();
      uint32_t item = 0, r = 0;
      bool acc_init = false;
      int prev = -1;
      uint32_t prev_kst = 0;
      auto dq_mma = [&](uint32_t kst, uint32_t it) {
        mbar_wait(ds_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t bd = desc_mnmajor(ring_addr + kst * L::TILE + k * 16 * 128, BN * 128);
          if (leader) umma_bf16(tmem + 256, desc_kmajor(ds_addr + k * 32), bd, IDESC_DQ,
                    (acc_init || k > 0) ? 1u : 0u);
          if (leader) umma_bf16(tmem + 256, desc_kmajor(ds_addr + L::DSB + k * 32), bd, IDESC_DQ, 1u);
        }
        acc_init = true;
        if (leader) umma_commit(&empty[kst]);
        if (leader) umma_commit(ds_empty);
      };
      for (int j = next_active(0); j >= 0; j = next_active(j + 1)) {
        const uint32_t b = item & 1;
        mbar_wait(&s_empty[b], ((item >> 1) & 1) ^ 1);
        const uint32_t kst = r % NST, vst = (r + 1) % NST;
        mbar_wait(&full[kst], (r / NST) & 1);
        mbar_wait(&full[vst], ((r + 1) / NST) & 1);
        tc_fence_after();
        const uint32_t sc = tmem + b * 128;
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (leader) umma_bf16(sc, desc_kmajor(q_addr + c * QB_DQ * 128 + k * 32),
                      desc_kmajor(ring_addr + kst * L::TILE + c * BN * 128 + k * 32), IDESC_S,
                      (c | k) != 0);
            if (leader) umma_bf16(sc + 64, desc_kmajor(do_addr + c * QB_DQ * 128 + k * 32),
                      desc_kmajor(ring_addr + vst * L::TILE + c * BN * 128 + k * 32), IDESC_S,
                      (c | k) != 0);
          }
        if (leader) umma_commit(&empty[vst]);
        if (leader) umma_commit(&s_full[b]);
        if (prev >= 0) dq_mma(prev_kst, item - 1);
        prev = j;
        prev_kst = kst;
        ++item;
        r += 2;
      }
      if (prev >= 0) dq_mma(prev_kst, item - 1);
      if (leader) umma_commit(acc_full);
    }
  } else if (warp >= 4) {
    const int half = (warp - 4) >> 2;  // key columns 32*half .. +31 of each tile
    const int lq = warp & 3;
    const int e = lq * 32 + lane;      // local query row 0..127
    const int rb = e >> 6;
    const int grow = row0 + e;
    const size_t orow = (size_t)bh * g.n + grow;
    const uint32_t tl = tmem + ((uint32_t)(lq * 32) << 16);
    const float A1 = a.A1;
    const float2 rc = a.rowc[orow];  // {C, delta} from the delta kernel
    uint32_t item = 0;
    const uint32_t ds_row = smem_u32(sDS) + (uint32_t)e * 128u;
    for (int j = next_active(0); j >= 0; j = next_active(j + 1)) {
      const bool mine = rb_active(rb, j);
      const uint32_t b = item & 1;
      mbar_wait(&s_full[b], (item >> 1) & 1);
      tc_fence_after();
      float s[32], dp[32];
      tmem_ld32(tl + b * 128 + half * 32, s);
      tmem_ld32(tl + b * 128 + 64 + half * 32, dp);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[b]);
      const int c0 = j * BN + half * 32;
      const bool diag = g.causal && c0 + 31 > grow;
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int x = 0; x < 16; ++x) {
        float ds2[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = 2 * x + h;
          float t = fmaf(A1, s[i], rc.x);
          if (!mine || (diag && c0 + i > grow)) t = -1.f;
          float p, u;
          pu_of<AK>(t, a.e0f, a.e1f, p, u);
          ds2[h] = u * (dp[i] - rc.y);
        }
        split_bf16x2(ds2[0], ds2[1], hi[x], lo[x]);
      }
      mbar_wait(ds_empty, (item & 1) ^ 1);
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {
        const uint32_t off = (((uint32_t)(half * 4 + qq)) ^ (uint32_t)(e & 7)) << 4;
        st_shared_v4(ds_row + off, hi[4 * qq], hi[4 * qq + 1], hi[4 * qq + 2], hi[4 * qq + 3]);
        st_shared_v4(ds_row + L::DSB + off, lo[4 * qq], lo[4 * qq + 1], lo[4 * qq + 2],
                     lo[4 * qq + 3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
      ++item;
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    bool any = false;
    for (int j = 0; j <= jmax; ++j) any |= rb_active(rb, j);
#pragma unroll
    for (int c = 0; c < D / 64; ++c) {
      float o[32];
      tmem_ld32(tl + 256 + half * (D / 2) + c * 32, o);
      tmem_wait_ld();
      const int x0 = half * (D / 2) + c * 32;
      if (g.out_dtype == ADATTN_F64) {
        double* dst = reinterpret_cast<double*>(a.dq) + orow * D + x0;
#pragma unroll
        for (int i = 0; i < 32; ++i) dst[i] = any ? (double)(a.scale_f * o[i]) : 0.0;
      } else {
        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.dq) + orow * D + x0);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          dst[i] = any ? make_float4(a.scale_f * o[4 * i], a.scale_f * o[4 * i + 1],
                                     a.scale_f * o[4 * i + 2], a.scale_f * o[4 * i + 3])
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// ================================================================= dK / dV
constexpr int KB = 128;      // keys per CTA
constexpr int QT = 64;       // query rows per unit (one reference tile)
constexpr int KST = 3;       // Q/dO stages

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
  static size_t bytes(int t_r) { return 1024 + OFF_UB + t_r + 64; }
};

template <int D, int AK>
__global__ void __launch_bounds__(kThreads, 1)
    tc_dkdv_kernel(const __grid_constant__ CUtensorMap tm_qt, const __grid_constant__ CUtensorMap tm_kb,
                   const __grid_constant__ CUtensorMap tm_vb, const __grid_constant__ CUtensorMap tm_dot,
                   const BwdArgs a) {
  using L = KvSmem<D>;
  constexpr int NCH = D / 64;
  const Geom& g = a.g;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  uint8_t* sSt = smem + L::OFF_ST;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full = bars;             // [KST]
  uint64_t* empty = bars + KST;      // [KST]
  uint64_t* s_full = bars + 2 * KST; // [2]
  uint64_t* p_full = s_full + 2;     // [2]
  uint64_t* kv_full = p_full + 2;
  uint64_t* acc_full = kv_full + 1;
  volatile uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::OFF_MISC);
  uint8_t* ubits = smem + L::OFF_UB;  // [t_r] 2-bit activity of (i, j0), (i, j0+1)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nkb = g.m / KB;
  const int bh = blockIdx.x % g.bh;
  const int kb = blockIdx.x / g.bh;  // causal: low key blocks have the most query tiles
  const int key0 = kb * KB;
  const int j0 = key0 / 64;          // first of the two reference key tiles
  const int wpr = g.wpr;
  const int i_first = g.causal ? key0 / QT : 0;

  {
    const int jw = (blockIdx.x / g.bh) * KB / 64;
    const int bhh = blockIdx.x % g.bh;
    for (int i = threadIdx.x; i < g.t_r; i += kThreads) {
      const uint32_t w = a.mask[((size_t)bhh * g.t_r + i) * g.wpr + (jw >> 5)];
      ubits[i] = (uint8_t)((w >> (jw & 31)) & 3u);
    }
  }
  if (tid == 0) {
    for (int i = 0; i < KST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 8);
    }
    mbar_init(kv_full, 1);
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(const_cast<uint32_t*>(s_tmem), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  (void)nkb;

  // bits of (query tile i, key tiles j0, j0+1): bit0 -> keys 0..63, bit1 -> 64..127
  auto unit_bits = [&](int i) -> uint32_t { return ubits[i]; };
  (void)wpr;
  (void)j0;
  auto next_unit = [&](int i) -> int {
    for (; i < g.t_r; ++i)
      if (unit_bits(i)) return i;
    return -1;
  };

  if (warp == 0) {
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
  } else if (warp == 1) {
    {
      const bool leader = elect_one_sync();
      constexpr uint32_t IDESC_S = idesc_bf16_f32(128, QT, false, false);
      constexpr uint32_t IDESC_G = idesc_bf16_f32(128, D, false, true);
      const uint32_t k_addr = smem_u32(sK), v_addr = smem_u32(sV), st_addr = smem_u32(sSt);
      mbar_wait(kv_full, 0);
      tc_fence_after();
      uint32_t u = 0;
      bool init = false;
      int prev = -1;
      uint32_t prev_st = 0;
      auto grad_mma = [&](uint32_t uu, uint32_t st) {
        const uint32_t b = uu & 1;
        mbar_wait(&p_full[b], (uu >> 1) & 1);
        tc_fence_after();
        const uint32_t qb = st_addr + st * L::STAGE;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          // queries 16k..16k+15: packed pairs of half k>>1 at cols 32*(k>>1) + 8*(k&1)
          // (hi) and +16 (lo)
          const uint32_t acol = 32 * (k >> 1) + 8 * (k & 1);
          const uint64_t bdo = desc_mnmajor(qb + L::QTB + k * 16 * 128, QT * 128);
          const uint64_t bq = desc_mnmajor(qb + k * 16 * 128, QT * 128);
          const uint32_t acc = (init || k > 0) ? 1u : 0u;
          if (leader) umma_bf16_ts(tmem + 256, tmem + b * 128 + acol, bdo, IDESC_G, acc);
          if (leader) umma_bf16_ts(tmem + 256, tmem + b * 128 + acol + 16, bdo, IDESC_G, 1u);
          if (leader) umma_bf16_ts(tmem + 256 + D, tmem + b * 128 + 64 + acol, bq, IDESC_G, acc);
          if (leader) umma_bf16_ts(tmem + 256 + D, tmem + b * 128 + 64 + acol + 16, bq, IDESC_G, 1u);
        }
        init = true;
        if (leader) umma_commit(&empty[st]);
      };
      for (int i = next_unit(i_first); i >= 0; i = next_unit(i + 1)) {
        const uint32_t st = u % KST;
        mbar_wait(&full[st], (u / KST) & 1);
        tc_fence_after();
        const uint32_t b = u & 1;
        const uint32_t qb = st_addr + st * L::STAGE;
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (leader) umma_bf16(tmem + b * 128, desc_kmajor(k_addr + c * KB * 128 + k * 32),
                      desc_kmajor(qb + c * QT * 128 + k * 32), IDESC_S, (c | k) != 0);
            if (leader) umma_bf16(tmem + b * 128 + 64, desc_kmajor(v_addr + c * KB * 128 + k * 32),
                      desc_kmajor(qb + L::QTB + c * QT * 128 + k * 32), IDESC_S, (c | k) != 0);
          }
        if (leader) umma_commit(&s_full[b]);
        if (prev >= 0) grad_mma(u - 1, prev_st);
        prev = i;
        prev_st = st;
        ++u;
      }
      if (prev >= 0) grad_mma(u - 1, prev_st);
      if (leader) umma_commit(acc_full);
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
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
      const uint32_t st = u % KST, b = u & 1;
      const bool mine = (unit_bits(i) >> ksub) & 1u;
      any |= mine;
      mbar_wait(&s_full[b], (u >> 1) & 1);
      tc_fence_after();
      float s[32], dp[32];
      tmem_ld32(tl + b * 128 + half * 32, s);
      tmem_ld32(tl + b * 128 + 64 + half * 32, dp);
      tmem_wait_ld();
      const float2* rc = reinterpret_cast<const float2*>(sSt + st * L::STAGE + 2 * L::QTB);
      uint32_t ph[16], pl[16], dh[16], dl[16];
      const int q0 = i * QT + half * 32;
#pragma unroll
      for (int x = 0; x < 16; ++x) {
        float pp[2], dd[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int qi = 2 * x + h;
          const float2 c = rc[half * 32 + qi];
          float t = fmaf(A1, s[qi], c.x);
          if (!mine || (g.causal && gkey > q0 + qi)) t = -1.f;
          float p, uu;
          pu_of<AK>(t, a.e0f, a.e1f, p, uu);
          pp[h] = p;
          dd[h] = uu * (dp[qi] - c.y);
        }
        split_bf16x2(pp[0], pp[1], ph[x], pl[x]);
        split_bf16x2(dd[0], dd[1], dh[x], dl[x]);
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
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

template <typename K>
cudaError_t set_smem(K kern, size_t bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int D, int AK>
cudaError_t run_bwd(const Geom& g, const CUtensorMap* m, const BwdArgs& a, bool delta_only,
                    cudaStream_t st) {
  cudaError_t e;
  {
    auto k0 = tc_delta_kernel<D, AK>;
    const size_t sm = DeltaSmem<D>::bytes(g.wpr);
    if ((e = set_smem(k0, sm))) return e;
    prof_begin("tc_delta", st);
    k0<<<dim3((unsigned)(a.ncta_rows * g.bh)), kThreads, sm, st>>>(m[0], m[1], m[2], m[3], a);
    prof_end(st);
    note_launch();
    if ((e = cudaGetLastError())) return e;
  }
  if (delta_only) return cudaSuccess;
  {
    auto k2 = tc_dkdv_kernel<D, AK>;
    const size_t sm = KvSmem<D>::bytes(g.t_r);
    if ((e = set_smem(k2, sm))) return e;
    prof_begin("tc_dkdv", st);
    k2<<<dim3((unsigned)((g.m / KB) * g.bh)), kThreads, sm, st>>>(m[4], m[5], m[6], m[7], a);
    prof_end(st);
    note_launch();
    if ((e = cudaGetLastError())) return e;
  }
  {
    auto k1 = tc_dq_kernel<D, AK>;
    const size_t sm = DqSmem<D>::bytes(g.wpr);
    if ((e = set_smem(k1, sm))) return e;
    prof_begin("tc_dq", st);
    k1<<<dim3((unsigned)((g.n / QB_DQ) * g.bh)), kThreads, sm, st>>>(m[8], m[1], m[2], m[9], a);
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

size_t backward_workspace(const Geom& g) { return (size_t)g.bh * g.n * sizeof(float2) + 256; }

cudaError_t backward(const Geom& g, const void* q, const void* k, const void* v, const double* tau,
                     const double* row_max, const uint32_t* mask, const void* dout, void* dq,
                     void* dk, void* dv, double* delta, void* workspace, bool delta_only,
                     cudaStream_t st) {
  CUtensorMap m[10];
  cudaError_t e;
  const uint64_t nq = (uint64_t)g.bh * g.n, nk = (uint64_t)g.bh * g.m;
  if ((e = make_tmap_2d(&m[0], q, nq, g.d, BM))) return e;
  if ((e = make_tmap_2d(&m[1], k, nk, g.d, BN))) return e;
  if ((e = make_tmap_2d(&m[2], v, nk, g.dv, BN))) return e;
  if ((e = make_tmap_2d(&m[3], dout, nq, g.dv, BM))) return e;
  if ((e = make_tmap_2d(&m[4], q, nq, g.d, QT))) return e;
  if ((e = make_tmap_2d(&m[5], k, nk, g.d, KB))) return e;
  if ((e = make_tmap_2d(&m[6], v, nk, g.dv, KB))) return e;
  if ((e = make_tmap_2d(&m[7], dout, nq, g.dv, QT))) return e;
  if ((e = make_tmap_2d(&m[8], q, nq, g.d, QB_DQ))) return e;
  if ((e = make_tmap_2d(&m[9], dout, nq, g.dv, QB_DQ))) return e;
  BwdArgs a;
  a.g = g;
  a.ncta_rows = g.n / BM;
  a.A1 = (float)((g.alpha - 1.0) * g.scale);
  a.e0f = (float)g.e0;
  a.e1f = (float)(g.e0 - 1.0);
  a.tau = tau;
  a.row_max = row_max;
  a.mask = mask;
  a.delta = delta;
  a.rowc = reinterpret_cast<float2*>(workspace);
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
