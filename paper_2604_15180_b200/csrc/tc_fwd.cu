// tc_fwd.cu -- bf16 tensor-core forward of tiled alpha-entmax attention for
// sm_100a (reference: /root/reference/proj/src/attention.cpp:157-361).
//
// One CTA = 256 query rows (four 64-row reference tiles, two M=128 UMMA row
// groups) of one head; keys stream in 64-key tiles (one reference key tile).
// Warp roles (384 threads):
//   warp 0      TMA producer: Q once, then K (and V in the output pass) tiles
//               into a 4-stage SWIZZLE_128B ring
//   warp 1      MMA issuer: S_g = Q_g K_j^T (M=128, N=64) into TMEM (double
//               buffered), O_g += P_g V_j (M=128, N=dv) in the output pass
//   warp 2      TMEM allocator (512 columns)
//   warps 4-11  epilogue, one thread per query row (tcgen05.ld 32x32b):
//               pass MAX  -> row max
//               pass HIST -> bin counts of z >= 0 -> solve_histogram -> tau_h
//               pass REF  -> f, f', f'' partial sums + 64x64 activity bits;
//                            safeguarded step per row (repeats until no row moves)
//               pass OUT  -> P = [z - tau]_+^(1/(alpha-1)) (bf16) into smem for
//                            the P*V MMA, over the set mask bits only
// Per-row refinement state and the step rules run in fp64 exactly as the
// reference; score-element math is fp32 (z = A1*acc + B, one FFMA).
#include <cuda.h>
#include <math_constants.h>

#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "tc.cuh"
#include "tc_common.cuh"
#include "tc_host.cuh"

namespace adattn_b200 {
namespace tc {
namespace {

constexpr int BM = 256;       // query rows per CTA
constexpr int BN = 64;        // keys per tile
constexpr int NST = 4;        // ring stages
constexpr int kThreads = 384;
constexpr int kEpi = 256;     // epilogue threads
constexpr int DEC_REF = 0, DEC_OUT = 1;

enum AlphaKind { AK15 = 0, AK2 = 1, AK125 = 2, AKGEN = 3 };

struct FwdArgs {
  Geom g;
  int ncta_rows;  // query CTAs per head = n / 256
  float A1;       // (alpha - 1) * scale
  float scale_f;
  float e0f, e1f, e2f;
  void* out;
  double* tau;
  double* row_max;
  uint32_t* mask;
  int32_t* steps;
};

template <int D>
struct FwdSmem {
  static constexpr int QBYTES = BM * D * 2;
  static constexpr int TILE = BN * D * 2;
  static constexpr int PBYTES = 2 * BM * BN * 2;  // P_hi, P_lo
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_RING = OFF_Q + QBYTES;
  static constexpr int OFF_P = OFF_RING + NST * TILE;
  static constexpr int OFF_BAR = OFF_P + PBYTES;
  static constexpr int NBAR = 2 * NST + 10;
  static constexpr int OFF_MISC = OFF_BAR + NBAR * 8;
  static constexpr int OFF_MASK = OFF_MISC + 64;
  static size_t bytes(int wpr) { return 1024 + OFF_MASK + 4 * wpr * 4 + 64; }
};

template <int AK>
__device__ __forceinline__ void ref_accumulate(float t, float e0f, float e1f, float e2f,
                                               float& s0, float& s1, float& s2) {
  const float tp = fmaxf(t, 0.f);
  if constexpr (AK == AK15) {  // e0=2, e1=1, e2=0
    s0 = fmaf(tp, tp, s0);
    s1 += tp;
    s2 += (t > 0.f) ? 1.f : 0.f;
  } else if constexpr (AK == AK2) {  // e0=1, e1=0 (e2 unused by Newton)
    s0 += tp;
    s1 += (t > 0.f) ? 1.f : 0.f;
  } else if constexpr (AK == AK125) {  // e0=4, e1=3, e2=2
    const float t2 = tp * tp;
    s0 = fmaf(t2, t2, s0);
    s1 = fmaf(t2, tp, s1);
    s2 += t2;
  } else {
    if (t > 0.f) {
      const float lt = __log2f(t);
      s0 += exp2f(e0f * lt);
      const float l1 = e1f < 0.f ? __log2f(fmaxf(t, 1e-12f)) : lt;
      s1 += (e1f == 0.f) ? 1.f : exp2f(e1f * l1);
      s2 += (e2f == 0.f) ? 1.f : exp2f(e2f * (e2f < 0.f ? __log2f(fmaxf(t, 1e-12f)) : lt));
    }
  }
}

template <int AK>
__device__ __forceinline__ float p_of(float t, float e0f) {
  const float tp = fmaxf(t, 0.f);
  if constexpr (AK == AK15) return tp * tp;
  else if constexpr (AK == AK2) return tp;
  else if constexpr (AK == AK125) {
    const float t2 = tp * tp;
    return t2 * t2;
  } else {
    return tp > 0.f ? exp2f(e0f * __log2f(tp)) : 0.f;
  }
}

template <int D, int AK>
__global__ void __launch_bounds__(kThreads, 1)
    tc_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const FwdArgs a) {
  using L = FwdSmem<D>;
  constexpr int NCH = D / 64;  // 128-byte chunks along d
  const Geom& g = a.g;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sRing = smem + L::OFF_RING;
  uint8_t* sP = smem + L::OFF_P;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full = bars;
  uint64_t* empty = bars + NST;
  uint64_t* s_full = bars + 2 * NST;
  uint64_t* s_empty = s_full + 2;
  uint64_t* p_full = s_empty + 2;
  uint64_t* p_empty = p_full + 1;
  uint64_t* o_full = p_empty + 1;
  uint64_t* q_full = o_full + 1;
  uint64_t* dec_bar = q_full + 1;
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + L::OFF_MISC);
  volatile uint32_t* s_tmem = misc;         // TMEM base
  volatile uint32_t* s_decision = misc + 1;
  uint32_t* smask = reinterpret_cast<uint32_t*>(smem + L::OFF_MASK);  // [4][wpr]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int bh = blockIdx.x % g.bh;
  const int crow = a.ncta_rows - 1 - blockIdx.x / g.bh;  // heaviest causal tiles first
  const int row0 = crow * BM;
  const int jmax = g.causal ? (row0 + BM - 1) / BN : g.t_c - 1;
  const int wpr = g.wpr;
  int rg_jlim[2];
  rg_jlim[0] = g.causal ? (row0 + 127) / BN : g.t_c - 1;
  rg_jlim[1] = jmax;

  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 8);
    }
    mbar_init(p_full, 8);
    mbar_init(p_empty, 1);
    mbar_init(o_full, 1);
    mbar_init(q_full, 1);
    mbar_init(dec_bar, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(const_cast<uint32_t*>(s_tmem), 512);
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  // activity of row group rg for key tile j in the output pass
  auto out_active = [&](int rg, int j) -> bool {
    const uint32_t bit = 1u << (j & 31);
    return ((smask[(2 * rg) * wpr + (j >> 5)] | smask[(2 * rg + 1) * wpr + (j >> 5)]) & bit) != 0;
  };
  auto any_active = [&](int j) -> bool { return out_active(0, j) || out_active(1, j); };
  auto next_active = [&](int j) -> int {  // first active key tile >= j, or -1
    for (; j <= jmax; ++j)
      if (any_active(j)) return j;
    return -1;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const int qrow = bh * g.n + row0;
      mbar_expect_tx(q_full, L::QBYTES);
      for (int c = 0; c < NCH; ++c) tma_load_2d(sQ + c * BM * 128, &tm_q, q_full, c * 64, qrow);
      uint32_t r = 0;
      auto load = [&](const CUtensorMap* tm, int row) {
        const uint32_t st = r % NST, ph = (r / NST) & 1;
        mbar_wait(&empty[st], ph ^ 1);
        mbar_expect_tx(&full[st], L::TILE);
        for (int c = 0; c < NCH; ++c)
          tma_load_2d(sRing + st * L::TILE + c * BN * 128, tm, &full[st], c * 64, row);
        ++r;
      };
      const int krow0 = bh * g.m;
      for (int pass = 0; pass < 2; ++pass)
        for (int j = 0; j <= jmax; ++j) load(&tm_k, krow0 + j * BN);
      for (uint32_t ref = 0;; ++ref) {
        for (int j = 0; j <= jmax; ++j) load(&tm_k, krow0 + j * BN);
        mbar_wait(dec_bar, ref & 1);
        if (*s_decision == DEC_OUT) break;
      }
      int prev = -1;
      for (int j = next_active(0); j >= 0; j = next_active(j + 1)) {
        load(&tm_k, krow0 + j * BN);
        if (prev >= 0) load(&tm_v, krow0 + prev * BN);
        prev = j;
      }
      if (prev >= 0) load(&tm_v, krow0 + prev * BN);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC_S = idesc_bf16_f32(128, BN, false, false);
      constexpr uint32_t IDESC_PV = idesc_bf16_f32(128, D, false, true);
      const uint32_t q_addr = smem_u32(sQ), ring_addr = smem_u32(sRing), p_addr = smem_u32(sP);
      mbar_wait(q_full, 0);
      tc_fence_after();
      uint32_t item = 0, r = 0;
      auto s_tile = [&](int j, bool out_pass) {
        const uint32_t b = item & 1;
        mbar_wait(&s_empty[b], ((item >> 1) & 1) ^ 1);
        const uint32_t st = r % NST;
        mbar_wait(&full[st], (r / NST) & 1);
        tc_fence_after();
        for (int rg = 0; rg < 2; ++rg) {
          const bool need = out_pass ? out_active(rg, j) : (j <= rg_jlim[rg]);
          if (!need) continue;
          const uint32_t d_t = tmem + b * 128 + rg * 64;
          for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(d_t, desc_kmajor(q_addr + c * BM * 128 + rg * 128 * 128 + k * 32),
                        desc_kmajor(ring_addr + st * L::TILE + c * BN * 128 + k * 32), IDESC_S,
                        (c | k) != 0);
        }
        umma_commit(&empty[st]);
        umma_commit(&s_full[b]);
        ++item;
        ++r;
      };
      bool o_init[2] = {false, false};
      uint32_t pi = 0;
      auto pv_tile = [&](int j) {
        const uint32_t st = r % NST;
        mbar_wait(&full[st], (r / NST) & 1);
        mbar_wait(p_full, pi & 1);
        tc_fence_after();
        for (int rg = 0; rg < 2; ++rg) {
          if (!out_active(rg, j)) continue;
          const uint32_t d_t = tmem + 256 + rg * D;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t bd = desc_mnmajor(ring_addr + st * L::TILE + k * 16 * 128, BN * 128);
            umma_bf16(d_t, desc_kmajor(p_addr + rg * 128 * 128 + k * 32), bd, IDESC_PV,
                      (o_init[rg] || k > 0) ? 1u : 0u);
            umma_bf16(d_t, desc_kmajor(p_addr + BM * BN * 2 + rg * 128 * 128 + k * 32), bd,
                      IDESC_PV, 1u);
          }
          o_init[rg] = true;
        }
        umma_commit(&empty[st]);
        umma_commit(p_empty);
        ++r;
        ++pi;
      };
      for (int pass = 0; pass < 2; ++pass)
        for (int j = 0; j <= jmax; ++j) s_tile(j, false);
      for (uint32_t ref = 0;; ++ref) {
        for (int j = 0; j <= jmax; ++j) s_tile(j, false);
        mbar_wait(dec_bar, ref & 1);
        if (*s_decision == DEC_OUT) break;
      }
      int prev = -1;
      for (int j = next_active(0); j >= 0; j = next_active(j + 1)) {
        s_tile(j, true);
        if (prev >= 0) pv_tile(prev);
        prev = j;
      }
      if (prev >= 0) pv_tile(prev);
      umma_commit(o_full);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int e = tid - 128;          // 0..255 == local query row
    const int rg = e >> 7;            // row group
    const int lq = warp & 3;          // TMEM lane quarter
    const int grow = row0 + e;        // query row within the head
    const int rb = e >> 6;            // 64-row reference tile within the CTA
    const uint32_t tl = tmem + ((uint32_t)(lq * 32) << 16);
    const int jl = rg_jlim[rg];
    const float A1 = a.A1;
    uint32_t item = 0;

    // Fetch S for (item, key tile j) into v[64]; release the TMEM buffer.
    float v[64];
    auto fetch = [&](int j, bool need) {
      const uint32_t b = item & 1;
      mbar_wait(&s_full[b], (item >> 1) & 1);
      tc_fence_after();
      if (need) {
        tmem_ld32(tl + b * 128 + rg * 64, v);
        tmem_ld32(tl + b * 128 + rg * 64 + 32, v + 32);
        tmem_wait_ld();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[b]);
      ++item;
      if (need && g.causal && j * BN + BN - 1 > grow) {
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (j * BN + i > grow) v[i] = -CUDART_INF_F;
      }
    };

    // pass MAX (attention.cpp:182-195): max of raw dot products, scaled once
    float mraw = -CUDART_INF_F;
    for (int j = 0; j <= jmax; ++j) {
      const bool need = j <= jl;
      fetch(j, need);
      if (need) {
#pragma unroll
        for (int i = 0; i < 64; ++i) mraw = fmaxf(mraw, v[i]);
      }
    }
    const float m_f = a.scale_f * mraw;  // == max(scale * s): rounding is monotone
    const double B = 1.0 - (g.alpha - 1.0) * (double)m_f;  // z = A1*acc + B
    const float Bf = (float)B;

    // pass HIST (attention.cpp:201-232): counts of bin min(floor(B*z), B-1), z >= 0
    const int nb = g.bins;
    uint32_t cnt[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) cnt[k] = 0;
    {
      const float An = A1 * (float)nb, Bn = Bf * (float)nb;  // exact: nb is a power of 2
      for (int j = 0; j <= jmax; ++j) {
        const bool need = j <= jl;
        fetch(j, need);
        if (!need) continue;
        if (nb <= 8) {
          uint32_t lo = 0, hi = 0;  // 8-bit fields, <= 64 per tile
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            const float y = fmaf(An, v[i], Bn);
            if (y >= 0.f) {
              int b = (int)(__float_as_uint(__fadd_rd(y, 8388608.f)) & 0x3Fu);
              b = min(b, nb - 1);
              const uint32_t inc = 1u << ((b & 3) << 3);
              if (b < 4) lo += inc;
              else hi += inc;
            }
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            cnt[k] += (lo >> (8 * k)) & 0xFFu;
            cnt[k + 4] += (hi >> (8 * k)) & 0xFFu;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            const float y = fmaf(An, v[i], Bn);
            if (y >= 0.f) {
              int b = (int)(__float_as_uint(__fadd_rd(y, 8388608.f)) & 0x3Fu);
              b = min(b, nb - 1);
#pragma unroll
              for (int k = 0; k < 32; ++k)
                if (k == b) cnt[k] += 1;
            }
          }
        }
      }
    }
    RowSolve rs;
    {
      uint32_t c32[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) c32[k] = cnt[k];
      double th, lo, hi;
      solve_histogram_dev(c32, nb, g.alpha, th, lo, hi);
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

    // passes REF (attention.cpp:234-332)
    const bool need_sec = g.alpha > 2.0;
    const double e0 = g.e0;
    bool first_pass = true;
    for (uint32_t ref = 0;; ++ref) {
      for (int i = e; i < 4 * wpr; i += kEpi) smask[i] = 0u;
      bar_sync(1, kEpi);
      double f = -1.0, f1 = 0.0, f2 = 0.0, fhi = -1.0;
      const float C = (float)(B - rs.tau);
      const float Chi = (float)(B - rs.hi);
      for (int j = 0; j <= jmax; ++j) {
        const bool need = j <= jl;
        fetch(j, need);
        bool act = false;
        if (need) {
          float s0 = 0.f, s1 = 0.f, s2 = 0.f, shi = 0.f, mx = -CUDART_INF_F;
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            const float t = fmaf(A1, v[i], C);
            mx = fmaxf(mx, t);
            ref_accumulate<AK>(t, a.e0f, a.e1f, a.e2f, s0, s1, s2);
          }
          if (first_pass && need_sec) {
#pragma unroll
            for (int i = 0; i < 64; ++i) {
              const float th = fmaf(A1, v[i], Chi);
              if (th > 0.f) shi += exp2f(a.e0f * __log2f(th));
            }
          }
          f += (double)s0;
          f1 -= e0 * (double)s1;
          f2 += e0 * (e0 - 1.0) * (double)s2;
          if (first_pass && need_sec) fhi += (double)shi;
          act = mx > -1e-9f;
        }
        if (__any_sync(0xffffffffu, act) && lane == 0)
          atomicOr(&smask[rb * wpr + (j >> 5)], 1u << (j & 31));
      }
      bool stepped = false;
      if (!rs.done) {
        rs.f = f;
        rs.f1 = f1;
        rs.f2 = f2;
        if (first_pass) rs.f_hi = fhi;
        stepped = row_step(rs, g.alpha, g.refine_tol, g.refine_iters, need_sec);
      }
      first_pass = false;
      const bool any = bar_red_or(2, kEpi, stepped);
      if (e == 0) {
        *s_decision = any ? DEC_REF : DEC_OUT;
        mbar_arrive(dec_bar);
      }
      if (!any) break;
    }

    // pass OUT (attention.cpp:334-352): P over the active 64x64 blocks
    {
      const float C = (float)(B - rs.tau);
      uint32_t pi = 0;
      const uint32_t p_row = smem_u32(sP) + (uint32_t)e * 128u;
      bool any_out = false;
      for (int j = next_active(0); j >= 0; j = next_active(j + 1)) {
        const bool need = out_active(rg, j);
        any_out |= need;
        fetch(j, need);
        uint32_t ph[32], pl[32];
        if (need) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            split_bf16x2(p_of<AK>(fmaf(A1, v[2 * i], C), a.e0f),
                         p_of<AK>(fmaf(A1, v[2 * i + 1], C), a.e0f), ph[i], pl[i]);
        }
        mbar_wait(p_empty, (pi & 1) ^ 1);
        if (need) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint32_t off = (q ^ (e & 7)) << 4;
            st_shared_v4(p_row + off, ph[4 * q], ph[4 * q + 1], ph[4 * q + 2], ph[4 * q + 3]);
            st_shared_v4(p_row + BM * BN * 2 + off, pl[4 * q], pl[4 * q + 1], pl[4 * q + 2],
                         pl[4 * q + 3]);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        ++pi;
      }
      // write O (fp32 or fp64), tau, row_max, steps
      const size_t orow = (size_t)bh * g.n + grow;
      mbar_wait(o_full, 0);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        float o[32];
        tmem_ld32(tl + 256 + rg * D + c * 32, o);
        tmem_wait_ld();
        if (!__any_sync(0xffffffffu, any_out)) {
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = 0.f;
        }
        if (g.out_dtype == ADATTN_F64) {
          double* dst = reinterpret_cast<double*>(a.out) + orow * D + c * 32;
#pragma unroll
          for (int i = 0; i < 32; ++i) dst[i] = (double)o[i];
        } else {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + orow * D + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) dst[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
        }
      }
      a.tau[orow] = rs.tau;
      a.row_max[orow] = (double)m_f;
      if (a.steps) a.steps[orow] = rs.steps;
      for (int i = e; i < 4 * wpr; i += kEpi) {
        const int rbi = i / wpr, w = i - rbi * wpr;
        a.mask[((size_t)bh * g.t_r + (row0 / 64 + rbi)) * wpr + w] = smask[i];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

template <int D, int AK>
cudaError_t launch_fwd(const Geom& g, const CUtensorMap& tq, const CUtensorMap& tk,
                       const CUtensorMap& tv, const FwdArgs& a, cudaStream_t st) {
  const size_t smem = FwdSmem<D>::bytes(g.wpr);
  auto kern = tc_fwd_kernel<D, AK>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e) return e;
  const dim3 grid((unsigned)(a.ncta_rows * g.bh));
  kern<<<grid, kThreads, smem, st>>>(tq, tk, tv, a);
  note_launch();
  return cudaGetLastError();
}

template <int D>
cudaError_t launch_fwd_d(const Geom& g, int ak, const CUtensorMap& tq, const CUtensorMap& tk,
                         const CUtensorMap& tv, const FwdArgs& a, cudaStream_t st) {
  switch (ak) {
    case AK15: return launch_fwd<D, AK15>(g, tq, tk, tv, a, st);
    case AK2: return launch_fwd<D, AK2>(g, tq, tk, tv, a, st);
    case AK125: return launch_fwd<D, AK125>(g, tq, tk, tv, a, st);
    default: return launch_fwd<D, AKGEN>(g, tq, tk, tv, a, st);
  }
}

}  // namespace

int alpha_kind(double alpha) {
  if (alpha == 1.5) return AK15;
  if (alpha == 2.0) return AK2;
  if (alpha == 1.25) return AK125;
  return AKGEN;
}

cudaError_t forward(const Geom& g, const void* q, const void* k, const void* v, void* out,
                    double* tau, double* row_max, uint32_t* mask, int32_t* steps,
                    cudaStream_t st) {
  CUtensorMap tq, tk, tv;
  cudaError_t e;
  if ((e = make_tmap_2d(&tq, q, (uint64_t)g.bh * g.n, g.d, BM))) return e;
  if ((e = make_tmap_2d(&tk, k, (uint64_t)g.bh * g.m, g.d, BN))) return e;
  if ((e = make_tmap_2d(&tv, v, (uint64_t)g.bh * g.m, g.dv, BN))) return e;
  FwdArgs a;
  a.g = g;
  a.ncta_rows = g.n / BM;
  a.A1 = (float)((g.alpha - 1.0) * g.scale);
  a.scale_f = (float)g.scale;
  a.e0f = (float)g.e0;
  a.e1f = (float)(g.e0 - 1.0);
  a.e2f = (float)(g.e0 - 2.0);
  a.out = out;
  a.tau = tau;
  a.row_max = row_max;
  a.mask = mask;
  a.steps = steps;
  const int ak = alpha_kind(g.alpha);
  if (g.d == 64) return launch_fwd_d<64>(g, ak, tq, tk, tv, a, st);
  return launch_fwd_d<128>(g, ak, tq, tk, tv, a, st);
}

}  // namespace tc
}  // namespace adattn_b200
