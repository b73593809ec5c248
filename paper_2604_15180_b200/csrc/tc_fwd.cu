// tc_fwd.cu -- bf16 tensor-core forward of tiled alpha-entmax attention for
// sm_100a (reference: /root/reference/proj/src/attention.cpp:157-361).
//
// One CTA = 256 query rows (four 64-row reference tiles, two M=128 UMMA row
// groups RG0/RG1) of one head.  Keys stream in 128-key tiles (two reference
// key tiles): S_g = Q_g K_J^T is an SS MMA with N=128, which is the smallest N
// that runs at the full tensor rate from shared memory (tools/mma_bench.cu:
// SMEM operand bandwidth is 128 B/cycle), and every K tile fetched from L2
// feeds both row groups.
//
// Warp roles (640 threads):
//   warp 0      TMA producer: Q once, then K (and V in the output pass) tiles
//               into a 3-stage SWIZZLE_128B ring
//   warp 1      MMA issuer (converged warp, one elected lane issues)
//   warp 2      TMEM allocator (512 columns)
//   warps 4-19  epilogue: 8 warps per row group, one thread per (row, 64-key
//               half of the tile); each row group has its own S barriers so
//               the two groups drift apart and hide each other's latency.
// TMEM: threshold passes: S[b][g] at b*256 + g*128 (double buffered);
//       output pass:      S[g] at g*128, O[g] at 256 + g*128.  P (bf16) is
//       written back over the thread's own S columns (tcgen05.st) and read as
//       the TMEM A operand of O_g += P_g V_J (TS MMA, no shared-memory trip).
// Passes (per CTA, in order):
//   MAX  -> row max; HIST -> bin counts of z >= 0 -> solve_histogram -> tau_h;
//   REF  -> f, f', f'' partial sums + 64x64 activity bits, one safeguarded step
//           per row, repeated until no row moves (the last pass's bits are the
//           mask); OUT -> P over the set mask bits, O = P V.
// Per-row refinement state and the step rules run in fp64 exactly as the
// reference; score-element math is fp32 (z = A1*acc + B, one FFMA) with packed
// f32x2 arithmetic.
#include <cuda.h>
#include <math_constants.h>

#include <cstdlib>

#include "common.cuh"
#include "tc.cuh"
#include "tc_common.cuh"
#include "tc_host.cuh"

namespace adattn_b200 {
namespace tc {
namespace {

#ifdef ADATTN_FWD_SLEEP
#define MBAR_WAIT mbar_wait_sleep
#else
#define MBAR_WAIT mbar_wait
#endif

constexpr int BM = 256;        // query rows per CTA
constexpr int BN = 128;        // keys per S tile (two 64-key reference tiles)
constexpr int NST = 4;         // ring stages
constexpr int kEpiWarps = 16;
constexpr int kEpi = kEpiWarps * 32;
// Warp roles: 0..15 epilogue (warp % 4 = TMEM lane quarter), 16 TMA producer
// (also TMEM alloc), 17 MMA issuer.  The MMA warp has the highest id: the
// scheduler's arbitration favours high warp ids, so MMA issue is not starved
// by the ALU-heavy epilogue warps sharing its SM sub-partition.
// Two MMA-issuing warps (17: row group 0, 18: row group 1), on different SM
// sub-partitions: the tensor pipe queues only about one MMA ahead, so every
// cycle an issuing warp spends outside tcgen05.mma (barrier waits, commits,
// bookkeeping -- and the issue slots it loses to the ALU-heavy epilogue warps
// of its sub-partition) idles the pipe; two independent issuers fill each
// other's gaps.
constexpr bool kDualMma = true;
constexpr int kWarpProd = kEpiWarps, kWarpMma = kEpiWarps + 1;
constexpr int kThreads = (kEpiWarps + (kDualMma ? 3 : 2)) * 32;
constexpr int DEC_REF = 0, DEC_OUT = 1;
constexpr int kTop = 8;  // list mode: largest per-tile maxima kept per thread in the MAX sweep
// output pass: all 16 epilogue warps write each row group's P in turn (0: 8 warps per group)
#ifndef ADATTN_OUT_ALL16
#define ADATTN_OUT_ALL16 1
#endif

enum AlphaKind { AK15 = 0, AK2 = 1, AK125 = 2, AKGEN = 3 };

}  // namespace
// Optional wait-cycle accounting (build with -DADATTN_PIPE_STATS): [0] MMA waits
// on TMA-full, [1] MMA waits on S-empty, [2] MMA waits on P-full, [3] producer
// waits on ring-empty, [4] epilogue warp 4 waits on S-full, [6] MMA-warp cycles,
// [7] ring items.
#ifdef ADATTN_PIPE_STATS
__device__ unsigned long long g_pipe_stats[64];
__device__ int g_cur_sweep_dummy;
#endif
#ifdef ADATTN_PIPE_TRACE
// event trace of CTA 0 (dev tool): per tracing thread a private 16K-entry
// region (role), fire-and-forget stores of type << 56 | tile << 40 | clock64
__device__ unsigned long long g_trace[64 << 12];
__device__ unsigned int g_trace_n;
inline void* g_trace_ptr() {
  void* p = nullptr;
  cudaGetSymbolAddress(&p, g_trace);
  return p;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// role: 0 producer, 1 MMA, 2 + warp (epilogue warps); +32 for CTA 1 of the pair
#define TRACE(role, type, J)                                                                \
  if (blockIdx.x < 2 && _tn < (1u << 12)) {                                                 \
    g_trace[(((role) + 32 * blockIdx.x) << 12) + _tn++] =                                   \
        ((unsigned long long)(type) << 56) | ((unsigned long long)((J) & 0xFFFF) << 40) |   \
        ((unsigned long long)clock64() & 0xFFFFFFFFFFull);                                  \
  }
#define TRACE_DECL unsigned _tn = 0
#else
#define TRACE(role, type, J) \
  do {                       \
  } while (0)
#define TRACE_DECL \
  do {             \
  } while (0)
#endif
namespace {
#ifdef ADATTN_PIPE_STATS
#define PSTAT_T0() const long long _t0 = clock64()
#define PSTAT_ADD(i) \
  if (leader) atomicAdd(&g_pipe_stats[i], (unsigned long long)(clock64() - _t0))
// epilogue phase marks (thread 128): [8+k] = cycles spent before mark k since the previous one
#define PASS_MARK(k)                                                                  \
  if (tid == 0) {                                                                     \
    const long long _n = clock64();                                                   \
    atomicAdd(&g_pipe_stats[8 + (k)], (unsigned long long)(_n - _pm));                \
    _pm = _n;                                                                         \
  }
// list-phase sub-marks (thread 0): [48+k] cycles before mark k since the previous one
#define LIST_MARK(k)                                                                  \
  if (tid == 0) {                                                                     \
    const long long _n = clock64();                                                   \
    atomicAdd(&g_pipe_stats[48 + (k)], (unsigned long long)(_n - _pm));               \
    _pm = _n;                                                                         \
  }
#else
#define LIST_MARK(k) \
  do {               \
  } while (0)
#define PASS_MARK(k) \
  do {               \
  } while (0)
#define PSTAT_T0() \
  do {             \
  } while (0)
#define PSTAT_ADD(i) \
  do {               \
  } while (0)
#endif

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
  // candidate lists (REF from lists instead of sweeps): per resident CTA slot
  // (%smid) and epilogue thread, `cand_cap` entries of (raw score, block)
  uint2* cand;
  int cand_cap;
  int cand_slots;
  int list_stage;  // 1: whole lists staged in the ring when they fit (ADATTN_LIST_STAGE=0: off)
  // support lists (list mode, delta from the support): the keys and u = p^(2 - alpha) of
  // the scores with t > 0 at the final tau, per 256-row CTA block in a pool of
  // 256 * supp_cap entries; per row and key half (count, pool offset); supp_flag[block] = 1
  // when the block's pool overflowed or the CTA fell back to the sweeps; nullptr: off
  uint2* supp;           // entries (key, t bits): t > 0 at the final tau
  int2* supp_cnt;
  uint32_t* supp_flag;   // per 256-row block
  uint32_t* supp_hflag;  // per head: any of its blocks flagged
  int32_t* supp_kcnt;    // per key of every head: support entries (the backward's transpose)
  int supp_cap;
  // O from the support lists (sparse_out_kernel after this kernel): CTAs whose lists went
  // into the pool skip the output pass and the O store
  int supp_o;
  // fp16 P V: per head, max |V| (float bits) of the scaled fp16 V copy; nullptr -> bf16 P
  const uint32_t* v16_max;
  // optional output (delta fold): Ubar [bh][n][dv] fp32, then sum u [bh][n] fp32
  float* ubar;
  // per resident CTA slot (%smid) and epilogue warp: the warp's maximum raw score of
  // every 128-key tile (its 32 rows x its 64 keys), nkt floats; nullptr: no skipping
  float* wtm;
  int wtm_slots;
  // optional output: per row block its active key blocks (ELL, ascending; ell_bytes layout)
  int32_t* rcnt;
  uint16_t* rcol;
};

template <int D>
struct FwdSmem {
  static constexpr int QBYTES = BM * D * 2;
  static constexpr int TILE = BN * D * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_RING = OFF_Q + QBYTES;
  static constexpr int OFF_CNT = OFF_RING + NST * TILE;   // [256][16] u32 (HIST combine)
  static constexpr int OFF_PART = OFF_CNT;                // [256][4] f64 (REF combine, reuses)
  static constexpr int OFF_BAR = OFF_CNT + BM * 16 * 4;
  static constexpr int NBAR = 4 * NST + 20;  // pair ring: 2*NST items of TILE/2
  static constexpr int OFF_MISC = OFF_BAR + NBAR * 8;
  static constexpr int OFF_ROW = OFF_MISC + 64;  // [256][4] f32 per-row scratch
  static constexpr int OFF_MASK = OFF_ROW + BM * 4 * 4;
  // after the mask ([4][wpr] u32): per-warp activity words [2 sets][16 warps][aw] u32,
  // thresholds [4] u32, activity sets [2 sets][2 row groups][aw] u32
  __host__ __device__ static int off_wact(int wpr) { return OFF_MASK + 4 * wpr * 4; }
  __host__ __device__ static int off_thr(int wpr, int nkt) { return off_wact(wpr) + 2 * kEpiWarps * ((nkt + 31) / 32) * 4; }
  __host__ __device__ static int off_act(int wpr, int nkt) { return off_thr(wpr, nkt) + 16; }
  // CTA pairs: union activity sets [2][2][aw], union mask [4][wpr], exchange flags [2]
  __host__ __device__ static int off_actu(int wpr, int nkt) { return off_act(wpr, nkt) + 4 * ((nkt + 31) / 32) * 4; }
  __host__ __device__ static int off_pm(int wpr, int nkt) { return off_actu(wpr, nkt) + 4 * ((nkt + 31) / 32) * 4; }
  __host__ __device__ static int off_xf(int wpr, int nkt) { return off_pm(wpr, nkt) + 4 * wpr * 4; }
  // the output pass's active 128-key tiles (ascending u16), after the exchange flags
  __host__ __device__ static int off_tiles(int wpr, int nkt) { return off_xf(wpr, nkt) + 16; }
  // list staging: the 16 epilogue warps' list totals (prefix sum)
  __host__ __device__ static int off_scan(int wpr, int nkt) { return (off_tiles(wpr, nkt) + 2 * nkt + 15) & ~15; }
  static size_t bytes(int wpr, int nkt) { return 1024 + off_scan(wpr, nkt) + 4 * kEpiWarps + 64; }
};

// Order-preserving float <-> u32 (atomicMax / atomicMin on floats in smem).
__device__ __forceinline__ uint32_t f2ord(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}
__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}
__device__ __forceinline__ float warp_min(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fminf(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
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

// Partial sums of one 32-element slice for the refinement pass: two
// independent accumulator sets of packed f32x2 for ILP.
template <int AK>
__device__ __forceinline__ void ref_slice(const float* v, float A1, float C, float e0f, float e1f,
                                          float e2f, float& s0o, float& s1o, float& s2o,
                                          float& mxo) {
  const float2 A2 = make_float2(A1, A1), C2 = make_float2(C, C);
  float2 s0a = make_float2(0.f, 0.f), s1a = s0a, s2a = s0a, s0b = s0a, s1b = s0a, s2b = s0a;
  float mxa = -CUDART_INF_F, mxb = -CUDART_INF_F;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float2 t = __ffma2_rn(A2, make_float2(v[2 * i], v[2 * i + 1]), C2);
    float2& s0 = (i & 1) ? s0b : s0a;
    float2& s1 = (i & 1) ? s1b : s1a;
    float2& s2 = (i & 1) ? s2b : s2a;
    float& mx = (i & 1) ? mxb : mxa;
    mx = fmaxf(mx, fmaxf(t.x, t.y));
    const float2 tp = make_float2(fmaxf(t.x, 0.f), fmaxf(t.y, 0.f));
    if constexpr (AK == AK15) {  // e0=2, e1=1, e2=0
      s0 = __ffma2_rn(tp, tp, s0);
      s1 = __fadd2_rn(s1, tp);
      s2 = __fadd2_rn(s2, make_float2(__saturatef(tp.x * 0x1p126f), __saturatef(tp.y * 0x1p126f)));
    } else if constexpr (AK == AK2) {  // e0=1, e1=0; f2 is unused by Newton
      s0 = __fadd2_rn(s0, tp);
      s1 = __fadd2_rn(s1, make_float2(__saturatef(tp.x * 0x1p126f), __saturatef(tp.y * 0x1p126f)));
    } else if constexpr (AK == AK125) {  // e0=4, e1=3, e2=2
      const float2 t2 = __fmul2_rn(tp, tp);
      s0 = __ffma2_rn(t2, t2, s0);
      s1 = __ffma2_rn(t2, tp, s1);
      s2 = __fadd2_rn(s2, t2);
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float x = h ? tp.y : tp.x;
        if (x > 0.f) {
          const float lt = __log2f(x);
          const float l1 = e1f < 0.f ? __log2f(fmaxf(x, 1e-12f)) : lt;
          const float l2 = e2f < 0.f ? __log2f(fmaxf(x, 1e-12f)) : lt;
          const float a0 = exp2f(e0f * lt), a1 = (e1f == 0.f) ? 1.f : exp2f(e1f * l1);
          const float a2 = (e2f == 0.f) ? 1.f : exp2f(e2f * l2);
          if (h) {
            s0.y += a0;
            s1.y += a1;
            s2.y += a2;
          } else {
            s0.x += a0;
            s1.x += a1;
            s2.x += a2;
          }
        }
      }
    }
  }
  s0o = (s0a.x + s0a.y) + (s0b.x + s0b.y);
  s1o = (s1a.x + s1a.y) + (s1b.x + s1b.y);
  s2o = (s2a.x + s2a.y) + (s2b.x + s2b.y);
  mxo = fmaxf(mxa, mxb);
}

// 1 << s with PTX clamp semantics (s >= 32 -> 0).
__device__ __forceinline__ uint32_t shl_clamp(uint32_t a, uint32_t s) {
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(s));
  return r;
}

// HIST binning of a 32-element slice, nibble-packed.  w = nb c (z + 1) with
// c = 1 - 2^-20 maps bin k of z (k/nb <= z < (k+1)/nb) to floor(w) = nb + k and
// z < 0 below nb; F = fadd.rd(w, 2^23) = 2^23 + floor(w) exactly, and
// G = F 2^-147 - (2^23 + nb) 2^-147 = 4k 2^-149 exactly: a denormal whose bit
// pattern IS the nibble shift 4k (z < 0: negative, sign bit set -> a clamped
// shift, counted nowhere).  Per element pair: FFMA2 + FADD2.RD + FFMA2 on the
// FMA pipe and 2 SHF + 1 IADD3 on the ALU pipe (the integer shift-amount
// arithmetic of a bit-pattern approach would load the ALU pipe, which bounds
// this sweep).  Needs denormals preserved (no -ftz).
// Three nibble accumulators (<= 11 elements each) fold into the 8-bit
// even/odd-bin fields hE (bins 0,2,4,6) / hO (1,3,5,7).
template <int NW>  // nibble words: bins <= 8 (1) or <= 16 (2)
__device__ __forceinline__ void hist_nib(const float* v, float2 Aw, float2 Bw, float2 Kf,
                                         uint32_t* hE, uint32_t* hO) {
  uint32_t n[3][NW];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int w = 0; w < NW; ++w) n[a][w] = 0;
  const float2 M = make_float2(8388608.f, 8388608.f);
  const float2 S = make_float2(0x1p-147f, 0x1p-147f);
#pragma unroll
  for (int x = 0; x < 16; ++x) {
    const float2 wv = __ffma2_rn(Aw, make_float2(v[2 * x], v[2 * x + 1]), Bw);
    const float2 F = __fadd2_rd(wv, M);
    const float2 G = __ffma2_rn(F, S, Kf);
    const uint32_t s0 = __float_as_uint(G.x);
    const uint32_t s1 = __float_as_uint(G.y);
    const int a0 = (2 * x) < 11 ? 0 : ((2 * x) < 22 ? 1 : 2);
    const int a1 = (2 * x + 1) < 11 ? 0 : ((2 * x + 1) < 22 ? 1 : 2);
#pragma unroll
    for (int w = 0; w < NW; ++w) {  // word w holds bins 8w .. 8w+7
      n[a0][w] += shl_clamp(1u, s0 - 32u * w);
      n[a1][w] += shl_clamp(1u, s1 - 32u * w);
    }
  }
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    hE[w] += (n[0][w] & 0x0F0F0F0Fu) + (n[1][w] & 0x0F0F0F0Fu) + (n[2][w] & 0x0F0F0F0Fu);
    hO[w] += ((n[0][w] >> 4) & 0x0F0F0F0Fu) + ((n[1][w] >> 4) & 0x0F0F0F0Fu) +
             ((n[2][w] >> 4) & 0x0F0F0F0Fu);
  }
}

// Whole HIST sweep of one thread (64 keys per tile) for nb <= 8 NW: counts of
// bins 0..8NW-1 into cnt[].  Per tile the 8-bit fields (<= 64) fold into
// 16-bit fields, drained to cnt every 512 tiles.
template <int NW, typename ActFn, typename TileFn>
__device__ __forceinline__ void hist_sweep(int jl, float2 Aw, float2 Bw, float2 Kf, uint32_t* cnt,
                                           ActFn&& active, TileFn&& tile) {
  uint32_t W[NW][4];
#pragma unroll
  for (int w = 0; w < NW; ++w) W[w][0] = W[w][1] = W[w][2] = W[w][3] = 0;
  auto drain = [&]() {
#pragma unroll
    for (int w = 0; w < NW; ++w) {  // fields: W0 (0,4) W1 (2,6) W2 (1,5) W3 (3,7)
      cnt[8 * w + 0] += W[w][0] & 0xFFFFu; cnt[8 * w + 4] += W[w][0] >> 16;
      cnt[8 * w + 2] += W[w][1] & 0xFFFFu; cnt[8 * w + 6] += W[w][1] >> 16;
      cnt[8 * w + 1] += W[w][2] & 0xFFFFu; cnt[8 * w + 5] += W[w][2] >> 16;
      cnt[8 * w + 3] += W[w][3] & 0xFFFFu; cnt[8 * w + 7] += W[w][3] >> 16;
      W[w][0] = W[w][1] = W[w][2] = W[w][3] = 0;
    }
  };
  for (int J = 0; J <= jl; ++J) {
    if (!active(J)) continue;
    uint32_t hE[NW], hO[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) hE[w] = hO[w] = 0;
    tile(J, hE, hO);
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      W[w][0] += hE[w] & 0x00FF00FFu;
      W[w][1] += (hE[w] >> 8) & 0x00FF00FFu;
      W[w][2] += hO[w] & 0x00FF00FFu;
      W[w][3] += (hO[w] >> 8) & 0x00FF00FFu;
    }
    if ((J & 511) == 511) drain();  // 16-bit fields hold < 1024 tiles of 64
  }
  drain();
}

// NB32: bins = 32 (the reference's 128-bit histogram words, attention.cpp:35) -- a
// separate instantiation, so the 4-word HIST counters' registers do not weigh on
// the default kernels
// CAND appends of one 32-key chunk, unrolled at compile time (the key offset of each
// 4-score group is an immediate of the append path, so the vote path carries no key math)
template <int I>
struct CandGroups {
  static __device__ __forceinline__ void run(uint32_t& lo, const float* v, float theta, uint32_t kc,
                                             uint32_t hi) {
    asm volatile(
        "{\n\t.reg .pred p0, p1, p2, p3, pa, q;\n\t.reg .f32 m;\n\t.reg .u64 a;\n\t"
        ".reg .b32 k0, k1, k2, k3;\n\t"
        "max.f32 m, %1, %2, %3;\n\t"
        "max.f32 m, m, %4;\n\t"
        "setp.gt.f32 pa, m, %5;\n\t"
        "vote.sync.any.pred q, pa, 0xffffffff;\n\t"
        "@!q bra.uni CANDL_SKIP_%=;\n\t"
        "setp.gt.f32 p0, %1, %5;\n\t"
        "setp.gt.f32 p1, %2, %5;\n\t"
        "setp.gt.f32 p2, %3, %5;\n\t"
        "setp.gt.f32 p3, %4, %5;\n\t"
        "add.u32 k0, %10, %11;\n\t"
        "add.u32 k1, k0, 1;\n\t"
        "add.u32 k2, k0, 2;\n\t"
        "add.u32 k3, k0, 3;\n\t"
        "mov.b64 a, {%0, %12};\n\t"
        "@p0 st.global.v2.b32 [a], {%6, k0};\n\t"
        "@p0 add.u32 %0, %0, 8;\n\t"
        "mov.b64 a, {%0, %12};\n\t"
        "@p1 st.global.v2.b32 [a], {%7, k1};\n\t"
        "@p1 add.u32 %0, %0, 8;\n\t"
        "mov.b64 a, {%0, %12};\n\t"
        "@p2 st.global.v2.b32 [a], {%8, k2};\n\t"
        "@p2 add.u32 %0, %0, 8;\n\t"
        "mov.b64 a, {%0, %12};\n\t"
        "@p3 st.global.v2.b32 [a], {%9, k3};\n\t"
        "@p3 add.u32 %0, %0, 8;\n\t"
        "CANDL_SKIP_%=:\n\t}"
        : "+r"(lo)
        : "f"(v[I]), "f"(v[I + 1]), "f"(v[I + 2]), "f"(v[I + 3]), "f"(theta),
          "r"(__float_as_uint(v[I])), "r"(__float_as_uint(v[I + 1])),
          "r"(__float_as_uint(v[I + 2])), "r"(__float_as_uint(v[I + 3])), "r"(kc), "n"(I),
          "r"(hi)
        : "memory");
    CandGroups<I + 4>::run(lo, v, theta, kc, hi);
  }
};
template <>
struct CandGroups<32> {
  static __device__ __forceinline__ void run(uint32_t&, const float*, float, uint32_t, uint32_t) {}
};

template <int D, int AK, bool PAIR, bool NB32 = false>
__global__ void __launch_bounds__(kThreads, 1)
    tc_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_kh, const __grid_constant__ CUtensorMap tm_v,
                  const __grid_constant__ CUtensorMap tm_v16, const FwdArgs a) {
  using L = FwdSmem<D>;
  static_assert(!PAIR || D == 128, "CTA pairs split K and V tiles in 64-row / 64-column halves");
  // ring: NST tiles, or (pairs) 2*NST items of half a tile (this CTA's half of K or V)
  constexpr int NSTR = PAIR ? 2 * NST : NST;
  constexpr uint32_t ITEM = PAIR ? L::TILE / 2 : L::TILE;
  constexpr int NCH = D / 64;  // 128-byte chunks along d
  const Geom& g = a.g;
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned base that stays in the shared address space (LDS/STS, not
  // generic LD/ST, for every access through it)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sRing = smem + L::OFF_RING;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full = bars;               // [NSTR]
  uint64_t* empty = bars + NSTR;       // [NSTR]
  uint64_t* s_full = bars + 2 * NSTR;  // [2 buffers][2 row groups]
  uint64_t* s_empty = s_full + 4;      // [2][2]
  uint64_t* p_full = s_empty + 4;      // [2 row groups]
  uint64_t* o_full = p_full + 2;
  uint64_t* q_full = o_full + 1;
  uint64_t* dec_bar = q_full + 1;
  uint64_t* plan_bar = dec_bar + 1;  // activity set published (phase 0: HIST, 1: CAND)
  uint64_t* xbar = plan_bar + 1;     // [2] pair exchanges (the peer arrives)
  // delta-fold output pass: S full [2], P+U full [2], O / Ubar full, O / Ubar read
  uint64_t* fs_full = xbar + 2;
  uint64_t* fp_full = fs_full + 2;
  uint64_t* fo_full = fp_full + 2;
  uint64_t* fo_empty = fo_full + 1;
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + L::OFF_MISC);
  volatile uint32_t* s_tmem = misc;  // TMEM base
  volatile uint32_t* s_decision = misc + 1;
  volatile uint32_t* s_ntiles = misc + 2;  // entries of sTiles
  uint32_t* sCnt = reinterpret_cast<uint32_t*>(smem + L::OFF_CNT);
  double* sPart = reinterpret_cast<double*>(smem + L::OFF_PART);
  float* sRow = reinterpret_cast<float*>(smem + L::OFF_ROW);
  uint32_t* smask = reinterpret_cast<uint32_t*>(smem + L::OFF_MASK);  // [4][wpr]
  const int nkt_ = g.m / BN, aw = (nkt_ + 31) / 32;
  uint32_t* sWAct = reinterpret_cast<uint32_t*>(smem + L::off_wact(g.wpr));   // [2][16][aw]
  uint32_t* sThr = reinterpret_cast<uint32_t*>(smem + L::off_thr(g.wpr, nkt_));  // [2 sets][2 rg]
  uint32_t* sAct = reinterpret_cast<uint32_t*>(smem + L::off_act(g.wpr, nkt_));  // [2][2][aw]
  // pairs: the MMAs are joint, so sweeps and the output pass run over the union
  // of both CTAs' activity sets / masks (extra tiles only add exact zeros)
  uint32_t* sActU = PAIR ? reinterpret_cast<uint32_t*>(smem + L::off_actu(g.wpr, nkt_)) : sAct;
  uint32_t* sPm = PAIR ? reinterpret_cast<uint32_t*>(smem + L::off_pm(g.wpr, nkt_)) : smask;
  volatile uint32_t* xflag = reinterpret_cast<volatile uint32_t*>(smem + L::off_xf(g.wpr, nkt_));
  uint16_t* sTiles = reinterpret_cast<uint16_t*>(smem + L::off_tiles(g.wpr, nkt_));
  int* sScan = reinterpret_cast<int*>(smem + L::off_scan(g.wpr, nkt_));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // head-major (the head's K/V stay L2-resident across its CTAs' sweeps),
  // heaviest causal row blocks first within a head
  uint32_t rank = 0;
  if constexpr (PAIR) rank = cluster_ctarank();
  const bool lead_cta = rank == 0;
  int bh, row0, lim0;  // lim0: first row of the rows whose causal limits the MMAs follow
  if constexpr (PAIR) {  // a pair = 512 rows: CTA r owns rows prow0 + 256 r ..
    const int npair = a.ncta_rows >> 1, pair = (int)(blockIdx.x >> 1);
    bh = pair / npair;
    const int prow0 = (npair - 1 - pair % npair) * 2 * BM;
    row0 = prow0 + (int)rank * BM;
    lim0 = prow0 + BM;
  } else {
    bh = blockIdx.x / a.ncta_rows;
    row0 = (a.ncta_rows - 1 - (int)(blockIdx.x % a.ncta_rows)) * BM;
    lim0 = row0;
  }
  // O = P V in fp16 (P in [0, 1], the head's V copied to fp16 scaled by a power of
  // two s, undone on O) unless the head's V holds a non-finite value
  const bool pvf16 = a.v16_max != nullptr && f16_copy_ok(a.v16_max[bh]);
  // delta fold in the output pass (single-CTA kernel; the C-ABI passes ubar only then)
  bool fold = false;
  if constexpr (!PAIR) fold = a.ubar != nullptr;
  const float oinv = pvf16 ? 1.f / f16_pow2_scale(a.v16_max[bh]) : 1.f;
  const int nkt = g.m / BN;                              // 128-key tiles
  const int Jmax = g.causal ? (lim0 + BM - 1) / BN : nkt - 1;
  const int wpr = g.wpr;
  int rg_jlim[2], own_jlim[2];  // tiles issued per row group (pair: CTA 1's rows) / own rows'
  rg_jlim[0] = g.causal ? (lim0 + 127) / BN : nkt - 1;
  rg_jlim[1] = Jmax;
  own_jlim[0] = g.causal ? (row0 + 127) / BN : nkt - 1;
  own_jlim[1] = g.causal ? (row0 + BM - 1) / BN : nkt - 1;

  if (tid == 0) {
    for (int i = 0; i < NSTR; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kDualMma ? 2 : 1);  // a commit from each MMA warp
    }
    constexpr uint32_t kArr = PAIR ? 16 : 8;  // epilogue warps of a row group (both CTAs)
    for (int i = 0; i < 4; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], kArr);
    }
    // output pass: all 16 epilogue warps (both CTAs: 32) write each row group's P
    mbar_init(&p_full[0], ADATTN_OUT_ALL16 ? 2 * kArr : kArr);
    mbar_init(&p_full[1], ADATTN_OUT_ALL16 ? 2 * kArr : kArr);
    mbar_init(o_full, kDualMma ? 2 : 1);
    mbar_init(q_full, 1);
    mbar_init(dec_bar, 1);
    mbar_init(plan_bar, 1);
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    if constexpr (!PAIR) {
      for (int i = 0; i < 2; ++i) {
        mbar_init(&fs_full[i], 1);
        mbar_init(&fp_full[i], kEpiWarps);
      }
      mbar_init(fo_full, 1);
      mbar_init(fo_empty, kEpiWarps);
    }
    fence_barrier_init();
  }
  if (tid < 4) sThr[tid] = 0xFFFFFFFFu;
  if (warp == kWarpProd) {
    if constexpr (PAIR) tmem_alloc_2sm(const_cast<uint32_t*>(s_tmem), 512);
    else tmem_alloc(const_cast<uint32_t*>(s_tmem), 512);
  }
  if (warp == kWarpProd && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(PAIR ? &tm_kh : &tm_k);
    prefetch_tmap(&tm_v);
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();  // both CTAs' barriers initialised before remote arrives / TMA
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  // threshold-sweep activity: set s (0: HIST, 1: CAND / REF), row group rg, tile J
  auto act = [&](int s, int rg, int J) -> bool {  // union (pairs) -- the tiles issued
    return (sActU[(s * 2 + rg) * aw + (J >> 5)] >> (J & 31)) & 1u;
  };
  auto act_any = [&](int s, int J) -> bool { return act(s, 0, J) || act(s, 1, J); };

  // output-pass activity of row group rg for 128-key tile J (reference blocks
  // (2rg, 2J), (2rg, 2J+1), (2rg+1, 2J), (2rg+1, 2J+1))
  auto out_active_m = [&](const uint32_t* m, int rg, int J) -> bool {
    const uint32_t bits = 3u << ((2 * J) & 31);
    const int w = (2 * J) >> 5;
    return ((m[(2 * rg) * wpr + w] | m[(2 * rg + 1) * wpr + w]) & bits) != 0;
  };
  auto out_active = [&](int rg, int J) -> bool { return out_active_m(sPm, rg, J); };
  // The output pass walks the CTA's nonzero-tile list: the 128-key tiles that hold an
  // active block of one of its four row blocks (pairs: of either CTA), ascending --
  // the union of the row blocks' nonzero-block lists (attention.cpp:334-352).
  // Built by epilogue warp 0 once the mask is final, before the decision barrier.
  auto build_tiles = [&]() {
    uint32_t n = 0;
    for (int J0 = 0; J0 <= Jmax; J0 += 32) {
      const int J = J0 + lane;
      const bool on = J <= Jmax && (out_active(0, J) || out_active(1, J));
      const uint32_t b = __ballot_sync(0xffffffffu, on);
      if (on) sTiles[n + __popc(b & ((1u << lane) - 1u))] = (uint16_t)J;
      n += __popc(b);
    }
    if (lane == 0) *s_ntiles = n;
    __syncwarp();
  };

  if (warp == kWarpProd) {
    // ------------------------------------------------------------ producer
    const bool leader = elect_one_sync();
    const int qrow = bh * g.n + row0;
    if (leader && lead_cta) mbar_expect_tx(q_full, (PAIR ? 2 : 1) * L::QBYTES);
    for (int c = 0; c < NCH; ++c) {
      if constexpr (PAIR) {
        if (leader) tma_load_2d_2sm(sQ + c * BM * 128, &tm_q, q_full, c * 64, qrow);
      } else {
        if (leader) tma_load_2d(sQ + c * BM * 128, &tm_q, q_full, c * 64, qrow);
      }
    }
    uint32_t r = 0;
    TRACE_DECL;
    const int krow0 = bh * g.m;
    // one ring item: K or V of 128-key tile J (pairs: this CTA's half -- keys
    // 64 rank .. +63 of K, columns 64 rank .. +63 of V -- completing on the
    // leader's barrier)
    auto load = [&](bool is_v, int J) {
      const uint32_t st = r % NSTR, ph = (r / NSTR) & 1;
      {
        PSTAT_T0();
        MBAR_WAIT(&empty[st], ph ^ 1);
        PSTAT_ADD(3);
        if (leader) TRACE(0, 1, J);
      }
      uint8_t* dst = sRing + st * ITEM;
      const int row = krow0 + J * BN;
      if constexpr (PAIR) {
        if (leader && lead_cta) mbar_expect_tx(&full[st], 2 * ITEM);
        if (is_v) {
          if (leader) tma_load_2d_2sm(dst, pvf16 ? &tm_v16 : &tm_v, &full[st], 64 * (int)rank, row);
        } else {
          if (leader) tma_load_3d_2sm(dst, &tm_kh, &full[st], row + 64 * (int)rank);
        }
      } else {
        if (leader) mbar_expect_tx(&full[st], L::TILE);
        for (int c = 0; c < NCH; ++c)
          if (leader)
            tma_load_2d(dst + c * BN * 128, is_v ? (pvf16 ? &tm_v16 : &tm_v) : &tm_k, &full[st], c * 64, row);
      }
      ++r;
    };
    for (int J = 0; J <= Jmax; ++J) load(false, J);  // MAX
    MBAR_WAIT(plan_bar, 0);
    uint32_t dround = 0;
    bool out_now = false;
    auto hist_loads = [&]() {  // HIST: tiles that can hold z >= 0
      for (int J = 0; J <= Jmax; ++J)
        if (act_any(0, J)) load(false, J);
    };
    if (!a.cand) {
      hist_loads();
      MBAR_WAIT(plan_bar, 1);
    } else {  // CAND sweep (list mode): tiles that can hold z > k_s / B - eps
      for (int J = 0; J <= Jmax; ++J)
        if (act_any(1, J)) load(false, J);
      MBAR_WAIT(dec_bar, 0);
      dround = 1;
      out_now = *s_decision == DEC_OUT;
      if (!out_now) hist_loads();  // list overflow: HIST, then REF sweeps
    }
    if (!out_now)
      for (uint32_t ref = 0;; ++ref) {
        for (int J = 0; J <= Jmax; ++J)
          if (act_any(1, J)) load(false, J);
        MBAR_WAIT(dec_bar, (dround + ref) & 1);
        if (*s_decision == DEC_OUT) break;
      }
    if (fold) {  // output pass, one row group at a time: K(item i), then V(item i - 1)
      int prevf = -1;
      for (int g2 = 0; g2 < 2; ++g2)
        for (uint32_t t = 0, nt_ = *s_ntiles; t < nt_; ++t) {
          const int J = sTiles[t];
          if (!out_active(g2, J)) continue;
          load(false, J);
          if (prevf >= 0) load(true, prevf);
          prevf = J;
        }
      if (prevf >= 0) load(true, prevf);
    }
    int prev = -1;
    for (uint32_t t = 0, nt_ = fold ? 0u : *s_ntiles; t < nt_; ++t) {
      const int J = sTiles[t];
      load(false, J);
      if (prev >= 0) load(true, prev);
      prev = J;
    }
    if (prev >= 0) load(true, prev);
  } else if ((warp == kWarpMma || (kDualMma && warp == kWarpMma + 1)) && (!PAIR || lead_cta)) {
    // ------------------------------------------------------------ MMA issuers
    // (pairs: the leader issues M=256 MMAs over both CTAs' rows).  rgm: the row
    // groups this warp issues for; both warps walk every ring item.
    const uint32_t rgm = kDualMma ? (1u << (warp - kWarpMma)) : 3u;
    const bool leader = elect_one_sync();
    constexpr uint32_t IDESC_S = idesc_bf16_f32(PAIR ? 256 : 128, BN, false, false);
    constexpr uint32_t IDESC_PV_BF = idesc_bf16_f32(PAIR ? 256 : 128, D, false, true);
    constexpr uint32_t IDESC_PV16 = idesc_f16_f32(PAIR ? 256 : 128, D, false, true);
    const uint32_t IDESC_PV = pvf16 ? IDESC_PV16 : IDESC_PV_BF;
    auto commit = [&](uint64_t* bar) {
      if constexpr (PAIR) {
        if (leader) umma2_commit_mc(bar);
      } else {
        if (leader) umma_commit(bar);
      }
    };
    const uint32_t q_addr = smem_u32(sQ), ring_addr = smem_u32(sRing);
    MBAR_WAIT(q_full, 0);
    tc_fence_after();
#ifdef ADATTN_PIPE_STATS
    const long long t_mma0 = clock64();
#endif
    // it[rg]: threshold tiles issued to row group rg (S buffer b = it & 1, that
    // buffer's previous uses = it >> 1); indices stay compile-time (no local memory)
    uint32_t it[2] = {0, 0}, r = 0, nt = 0;  // nt: row-group tiles issued (stats)
    TRACE_DECL;
    // operand descriptors, precomputed: the start-address field advances 2 (32 B)
    // per 16-element K step
    uint64_t dQ[2][NCH];
#pragma unroll
    for (int g2 = 0; g2 < 2; ++g2)
#pragma unroll
      for (int c = 0; c < NCH; ++c) dQ[g2][c] = desc_kmajor(q_addr + c * BM * 128 + g2 * 128 * 128);
    const uint64_t dK0 = desc_kmajor(ring_addr);
    int cur_sweep = 0;  // stats: [32+2s] ring waits, [33+2s] S-buffer waits of sweep s
    (void)cur_sweep;
    auto wait_ring = [&]() -> uint32_t {
      const uint32_t st = r % NSTR;
      PSTAT_T0();
      MBAR_WAIT(&full[st], (r / NSTR) & 1);
      PSTAT_ADD(0);
      PSTAT_ADD(32 + 2 * cur_sweep);
      tc_fence_after();
      return st;
    };
    auto issue_s = [&](uint32_t d_t, int rg, uint32_t st) {
      const uint64_t dk = dK0 + (uint64_t)((st * ITEM) >> 4);
      constexpr uint32_t CH = (PAIR ? 64 : BN) * 128;  // bytes per 64-column chunk of d
      if constexpr (D == 128) {
        if (leader)
          umma_ss_d128<(PAIR ? 2 : 1), ((BM * 128) >> 4), ((int)(CH >> 4))>(d_t, dQ[rg][0], dk, IDESC_S, 0u);
      } else {
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t bk = dk + (uint64_t)(((uint32_t)(c * CH) >> 4) + 2 * k);
            if constexpr (PAIR) {
              if (leader) umma2_bf16(d_t, dQ[rg][c] + (uint64_t)(2 * k), bk, IDESC_S, (c | k) != 0);
            } else {
              if (leader) umma_bf16(d_t, dQ[rg][c] + (uint64_t)(2 * k), bk, IDESC_S, (c | k) != 0);
            }
          }
      }
    };
    // threshold passes: S double buffered per row group
    // Both row groups' S buffers are claimed before either group's MMAs are
    // issued, so the 16 MMAs of a tile go out back to back (the tensor pipe
    // queues only about one MMA ahead: any gap in the issue stream idles it).
    auto s_tile = [&](int J, int set) {  // set < 0: every tile (MAX)
      const uint32_t st = wait_ring();
      if (leader) TRACE(1, 2, J);
      bool doit[2];
#pragma unroll
      for (int rg = 0; rg < 2; ++rg) {
        doit[rg] = ((rgm >> rg) & 1u) && !(J > rg_jlim[rg] || (set >= 0 && !act(set, rg, J)));
        if (!doit[rg]) continue;
        PSTAT_T0();
        if (leader) TRACE(1, 12 + rg, J);
        MBAR_WAIT(&s_empty[(it[rg] & 1) * 2 + rg], ((it[rg] >> 1) & 1) ^ 1);
        if (leader) TRACE(1, 14 + rg, J);
        PSTAT_ADD(1);
        PSTAT_ADD(33 + 2 * cur_sweep);
      }
      if (leader) TRACE(1, 3, J);
      tc_fence_after();
#pragma unroll
      for (int rg = 0; rg < 2; ++rg) {
        if (!doit[rg]) continue;
        const uint32_t b = it[rg] & 1;
        {
          PSTAT_T0();
          issue_s(tmem + b * 256 + rg * 128, rg, st);
          commit(&s_full[b * 2 + rg]);
          PSTAT_ADD(44 + (cur_sweep == 0 ? 0 : 1));  // [44] MAX, [45] other sweeps: issue cycles
          if (leader) TRACE(1, 4 + rg, J);
        }
        ++it[rg];
        ++nt;
      }
      commit(&empty[st]);
      ++r;
    };
#ifdef ADATTN_PIPE_STATS
    // MMA-side sweep cost: [16+2s] MMA-warp cycles of sweep s, [17+2s] row-group tiles issued
    long long _sw = clock64();
    auto sweep_mark = [&](int s) {
      const long long n = clock64();
      if (leader) {
        atomicAdd(&g_pipe_stats[16 + 2 * s], (unsigned long long)(n - _sw));
        atomicAdd(&g_pipe_stats[17 + 2 * s], (unsigned long long)nt);
      }
      _sw = n;
      nt = 0;
      cur_sweep = s + 1;
    };
#else
    auto sweep_mark = [&](int) { (void)nt; };
#endif
    for (int J = 0; J <= Jmax; ++J) s_tile(J, -1);  // MAX
    sweep_mark(0);
    MBAR_WAIT(plan_bar, 0);
    uint32_t dround = 0;
    bool out_now = false;
    auto hist_tiles = [&]() {
      for (int J = 0; J <= Jmax; ++J)
        if (act_any(0, J)) s_tile(J, 0);  // HIST
      sweep_mark(1);
    };
    if (!a.cand) {
      hist_tiles();
      MBAR_WAIT(plan_bar, 1);
    } else {  // CAND sweep (list mode)
      for (int J = 0; J <= Jmax; ++J)
        if (act_any(1, J)) s_tile(J, 1);
      sweep_mark(2);
      MBAR_WAIT(dec_bar, 0);
      dround = 1;
      out_now = *s_decision == DEC_OUT;
      if (!out_now) hist_tiles();  // list overflow: HIST, then REF sweeps
    }
    if (!out_now)
      for (uint32_t ref = 0;; ++ref) {
        for (int J = 0; J <= Jmax; ++J)
          if (act_any(1, J)) s_tile(J, 1);
        MBAR_WAIT(dec_bar, (dround + ref) & 1);
        if (*s_decision == DEC_OUT) break;
      }
    sweep_mark(3);  // REF sweeps (fallback) + waiting for the decision
    if (fold) {
      // Output pass with the delta fold: one row group at a time;
      // per active tile (item i) S(i) into buffer i & 1, then -- once the
      // epilogue has written P(i-1) and U(i-1) over buffer (i-1) & 1 --
      // O += P V and Ubar += U V.  TMEM: S buffers at 0 / 128, O at 256, Ubar at
      // 384.  Warp kWarpMma issues everything in order (S(i+1) before the
      // products of item i, so the epilogue of i+1 overlaps them); the other
      // MMA warp only releases ring slots.
      const uint64_t dVf = desc_mnmajor(ring_addr, BN * 128);
      if (warp != kWarpMma) {
        for (int g2 = 0; g2 < 2; ++g2)
          for (uint32_t t = 0, nt_ = *s_ntiles; t < nt_; ++t) {
            if (!out_active(g2, sTiles[t])) continue;
            for (int x = 0; x < 2; ++x) {  // K(i), V(i): one release each
              const uint32_t st = wait_ring();
              if (elect_one_sync()) mbar_arrive(&empty[st]);
              __syncwarp();
              ++r;
            }
          }
      } else {
        uint32_t fi = 0;        // items issued
        int pg = -1;            // group of item fi - 1 (-1: none yet)
        bool p_first = false;   // item fi - 1 is the first of its group
        bool g0_any = false;    // row group 0 has items (its O / Ubar must be read first)
        // the products of item fi - 1 (V(item) in ring slot vst)
        auto products = [&](uint32_t vst, bool last_of_group) {
          const uint32_t pb = (fi - 1) & 1;
          MBAR_WAIT(&fp_full[pb], ((fi - 1) >> 1) & 1);
          // group 1's first products overwrite the accumulators group 0's O / Ubar
          // were read from
          if (p_first && pg == 1 && g0_any) MBAR_WAIT(fo_empty, 0);
          tc_fence_after();
          const uint64_t bv = dVf + (uint64_t)((vst * ITEM) >> 4);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            // keys 16k..16k+15: P at pb*128 + 32*(k>>1) + 8*(k&1), U 16 columns on
            const uint32_t acol = pb * 128 + 32 * (k >> 1) + 8 * (k & 1);
            const uint32_t acc = (!p_first || k > 0) ? 1u : 0u;
            if (leader) umma_bf16_ts(tmem + 256, tmem + acol, bv + (uint64_t)(128 * k), IDESC_PV, acc);
            if (leader) umma_bf16_ts(tmem + 384, tmem + acol + 16, bv + (uint64_t)(128 * k), IDESC_PV, acc);
          }
          if (last_of_group) commit(fo_full);
          commit(&empty[vst]);
          ++r;
        };
        for (int g2 = 0; g2 < 2; ++g2) {
          bool first = true;
          for (uint32_t t = 0, nt_ = *s_ntiles; t < nt_; ++t) {
            const int J = sTiles[t];
            if (!out_active(g2, J)) continue;
            const uint32_t kst = wait_ring();  // K(J)
            issue_s(tmem + (fi & 1) * 128, g2, kst);
            commit(&fs_full[fi & 1]);
            commit(&empty[kst]);
            ++r;
            ++nt;
            if (pg >= 0) products(wait_ring(), pg != g2);  // V(item fi - 1)
            if (g2 == 0) g0_any = true;
            p_first = first;
            first = false;
            pg = g2;
            ++fi;
          }
        }
        if (pg >= 0) products(wait_ring(), true);
      }
    } else {
    // output pass: S[g] at g*128 (buffer 0 of each group), O[g] at 256 + g*128.
    // Per active tile J, per group g: PV_g(prev) then S_g(J) -- in tensor-pipe
    // order, so S_g(J) overwrites P_g(prev) only after PV_g(prev) has read it,
    // and one group's P computation overlaps the other group's MMAs.
    bool o_init[2] = {false, false};
    uint32_t pcnt[2] = {0, 0};
    const uint64_t dVmn = desc_mnmajor(ring_addr, BN * 128);  // (pairs: one 64-column chunk)
    auto pv = [&](int rg, uint32_t vst) {
      {
        PSTAT_T0();
        MBAR_WAIT(&p_full[rg], pcnt[rg] & 1);
        PSTAT_ADD(2);
      }
      ++pcnt[rg];
      tc_fence_after();
      const uint64_t bv = dVmn + (uint64_t)((vst * ITEM) >> 4);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        // keys 16k..16k+15: packed P pairs at TMEM cols rg*128 + 32*(k>>1) + 8*(k&1)
        // (each 32-key chunk's P over the first half of its own S columns);
        // a 16-key step of the MN-major V operand is 2048 B = +128
        const uint32_t acol = rg * 128 + 32 * (k >> 1) + 8 * (k & 1);
        const uint32_t acc = (o_init[rg] || k > 0) ? 1u : 0u;
        if constexpr (PAIR) {
          if (leader) umma2_bf16_ts(tmem + 256 + rg * D, tmem + acol, bv + (uint64_t)(128 * k), IDESC_PV, acc);
        } else {
          if (leader) umma_bf16_ts(tmem + 256 + rg * D, tmem + acol, bv + (uint64_t)(128 * k), IDESC_PV, acc);
        }
      }
      o_init[rg] = true;
    };
    int prev = -1;
    bool prev_act[2] = {false, false};
    for (uint32_t t = 0, nt_ = *s_ntiles; t < nt_; ++t) {
      const int J = sTiles[t];
      const uint32_t kst = wait_ring();  // K(J) is ring item r
      uint32_t vst = 0;
      if (prev >= 0) {
        vst = (r + 1) % NSTR;  // V(prev) follows K(J) in the producer's order
        PSTAT_T0();
        MBAR_WAIT(&full[vst], ((r + 1) / NSTR) & 1);
        PSTAT_ADD(0);
        tc_fence_after();
      }
      bool act[2];
#pragma unroll
      for (int rg = 0; rg < 2; ++rg) {
        if (!((rgm >> rg) & 1u)) {
          act[rg] = false;
          continue;
        }
        if (prev >= 0 && prev_act[rg]) pv(rg, vst);
        act[rg] = out_active(rg, J);
        if (act[rg]) {
          ++nt;
          issue_s(tmem + rg * 128, rg, kst);
          commit(&s_full[rg]);
        }
      }
      commit(&empty[kst]);
      ++r;
      if (prev >= 0) {
        commit(&empty[vst]);
        ++r;
      }
      prev = J;
      prev_act[0] = act[0];
      prev_act[1] = act[1];
    }
    if (prev >= 0) {
      const uint32_t vst = wait_ring();
#pragma unroll
      for (int rg = 0; rg < 2; ++rg)
        if (prev_act[rg]) pv(rg, vst);
      commit(&empty[vst]);
      ++r;
    }
    commit(o_full);
    }  // !fold
    sweep_mark(4);
#ifdef ADATTN_PIPE_STATS
    if (leader) {
      atomicAdd(&g_pipe_stats[6], (unsigned long long)(clock64() - t_mma0));
      atomicAdd(&g_pipe_stats[7], (unsigned long long)r);
    }
#endif
  } else if (warp < kEpiWarps) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp;              // 0..15
    const int rg = ew >> 3;           // row group
    const int half = (ew >> 2) & 1;   // keys 64*half .. +63 of each 128-key tile
    const int lq = warp & 3;          // TMEM lane quarter
    const int e = rg * 128 + lq * 32 + lane;  // local query row 0..255
    const int grow = row0 + e;        // query row within the head
    const int rb = e >> 6;            // 64-row reference tile within the CTA
    const uint32_t tl = tmem + ((uint32_t)(lq * 32) << 16) + rg * 128 + half * 64;
    const int jl = rg_jlim[rg];       // tiles the MMA warp issues to this row group
    const int own_jl = own_jlim[rg];  // ... of which this CTA's rows can see (causal)
    const int bar_rg = 1 + rg;        // named barrier of this row group (256 threads)
    uint32_t smid_e;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_e));
    float* const wt = (a.wtm && (int)smid_e < a.wtm_slots)
                          ? a.wtm + ((size_t)smid_e * kEpiWarps + ew) * (size_t)nkt_ : nullptr;
    // this warp's activity for set s, tile J (publish_set)
    auto wact = [&](int s, int J) -> bool {
      return (sWAct[(s * kEpiWarps + ew) * aw + (J >> 5)] >> (J & 31)) & 1u;
    };
    // S-buffer / P handshakes go to the pair leader's barriers (its MMA warp waits on them)
    auto arrive_mma = [&](uint64_t* bar) {
      if (PAIR && !lead_cta) mbar_arrive_cluster(mapa_shared(smem_u32(bar), 0));
      else mbar_arrive(bar);
    };
    // pair exchanges (all epilogue threads): afterwards the peer's shared-memory
    // state written before its matching exchange is visible through DSMEM
    uint32_t xk = 0;
    auto pair_xchg = [&]() {
      bar_sync(3, kEpi);
      if (tid == 0) {
        uint64_t* xb = &xbar[xk & 1];
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        mbar_arrive_cluster_release(mapa_shared(smem_u32(xb), rank ^ 1u));
        mbar_wait_cluster(xb, (xk >> 1) & 1);
      }
      ++xk;
      bar_sync(3, kEpi);
    };
    auto peer_ld = [&](const volatile uint32_t* p) -> uint32_t {
      return ld_shared_cluster(mapa_shared(smem_u32(const_cast<const uint32_t*>(p)), rank ^ 1u));
    };
    auto pair_or = [&](bool v) -> bool {  // v: CTA-uniform
      if (tid == 0) xflag[xk & 1] = v ? 1u : 0u;
      pair_xchg();
      return v || peer_ld(&xflag[(xk - 1) & 1]) != 0u;
    };
    auto pair_or_words = [&](uint32_t* dst, const uint32_t* src, int n) {  // dst = src | peer src
      pair_xchg();
      for (int i = tid; i < n; i += kEpi) dst[i] = src[i] | peer_ld(&src[i]);
      bar_sync(3, kEpi);
    };
    (void)pair_or;
    (void)pair_or_words;
    const float A1 = a.A1;
    uint32_t it = 0;                  // threshold tiles consumed (S buffer it & 1, its use it >> 1)
    TRACE_DECL;

    float v[32];
    // 32-key chunk c (0/1) of this thread's 64 keys of tile J, from buffer column base
    // keys beyond the row (causal) or beyond the problem (padding of a ragged m)
    const int klim = g.causal ? min(grow, g.m_valid - 1) : g.m_valid - 1;
    const bool row_real = grow < g.n_valid;  // padding rows of a ragged n: no mask bits
    auto mask_chunk = [&](float* x, int J, int c) {
      const int k0 = J * BN + half * 64 + c * 32;
      if (k0 + 31 > klim) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (k0 + i > klim) x[i] = -CUDART_INF_F;
      }
    };
    auto load_chunk = [&](uint32_t col, int J, int c) {
#ifdef ADATTN_PIPE_STATS
      const long long _tl = clock64();
#endif
      tmem_ld32(tl + col + c * 32, v);
      tmem_wait_ld();
#ifdef ADATTN_PIPE_STATS
      if (tid == 0) {  // [46] TMEM load + wait cycles of thread 0, [47] loads
        atomicAdd(&g_pipe_stats[46], (unsigned long long)(clock64() - _tl));
        atomicAdd(&g_pipe_stats[47], 1ull);
      }
#endif
      mask_chunk(v, J, c);
    };
    // threshold-pass tile: wait, run body on chunks 0 and 1, release the buffer
    // (own == false: a tile issued for the peer CTA's rows only -- release it unread)
    auto tau_tile = [&](int J, bool own, auto&& body) {
      const uint32_t b = it & 1;
      if (!own) {  // not this warp's tile (no candidate rows; pairs: the peer's rows only)
        MBAR_WAIT(&s_full[b * 2 + rg], (it >> 1) & 1);
        ++it;
        __syncwarp();
        if (lane == 0) arrive_mma(&s_empty[b * 2 + rg]);
        return;
      }
      {
#ifdef ADATTN_PIPE_STATS
        const long long _tw = clock64();
#endif
        MBAR_WAIT(&s_full[b * 2 + rg], (it >> 1) & 1);
#ifdef ADATTN_PIPE_STATS
        if (warp == 0 && lane == 0) atomicAdd(&g_pipe_stats[4], (unsigned long long)(clock64() - _tw));
#endif
        if (lane == 0) TRACE(2 + warp, 6 + rg, J);
      }
      ++it;
      tc_fence_after();
      load_chunk(b * 256, J, 0);
      body(static_cast<const float*>(v));
      load_chunk(b * 256, J, 1);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_mma(&s_empty[b * 2 + rg]);
      if (lane == 0) TRACE(2 + warp, 8 + rg, J);
      body(static_cast<const float*>(v));
      if (lane == 0) TRACE(2 + warp, 10 + rg, J);
    };

#ifdef ADATTN_PIPE_STATS
    long long _pm = clock64();
#endif
    // PhaseTimings: epilogue thread 0 attributes its time to the reference phases
    unsigned long long* const pacc = tid == 0 ? g.phase_ns : nullptr;
    unsigned long long pt = pacc ? global_ns() : 0ull;
    // ---- pass MAX (attention.cpp:182-195): max of raw dot products, scaled once
    // Also the per-(row group, tile) maximum raw score, for the activity sets
    // of the later sweeps (tiles whose every score is below every row's
    // threshold are skipped there).
    // List mode (candidate lists enabled): the thread also keeps the kTop largest
    // of its per-tile maxima (distinct scores); their histogram bounds the
    // bracket floor from below (f_h only grows with more entries), which sets
    // the candidate threshold of the single CAND sweep that replaces the HIST
    // sweep (see the CAND pass below).
    const bool list_mode = a.cand != nullptr;
    float top[kTop];
#pragma unroll
    for (int i = 0; i < kTop; ++i) top[i] = -CUDART_INF_F;
    float mraw = -CUDART_INF_F;
    for (int J = 0; J <= jl; ++J) {
      float tmx = -CUDART_INF_F;
      const bool own = J <= own_jl;
      tau_tile(J, own, [&](const float* v) {
#pragma unroll
        for (int i = 0; i < 32; i += 2) tmx = fmaxf(tmx, fmaxf(v[i], v[i + 1]));
      });
      if (!own) continue;
      if (list_mode) {  // sorted insert (descending) of the tile's max: 2 kTop - 1 FMNMX
#pragma unroll
        for (int t = kTop - 1; t > 0; --t) top[t] = fmaxf(top[t], fminf(top[t - 1], tmx));
        top[0] = fmaxf(top[0], tmx);
      }
      mraw = fmaxf(mraw, tmx);
      tmx = warp_max(tmx);
      if (lane == 0 && wt) wt[J] = tmx;  // the warp's tile maximum (its rows x its 64 keys)
    }
    sRow[e * 4 + half] = mraw;
    bar_sync(bar_rg, 256);
    mraw = fmaxf(sRow[e * 4], sRow[e * 4 + 1]);
    PASS_MARK(0);
    phase_tick(pacc, 0, pt);
    const float m_f = a.scale_f * mraw;  // == max(scale * s): rounding is monotone
    const double B = 1.0 - (g.alpha - 1.0) * (double)m_f;  // z = A1*acc + B
    const float Bf = (float)B;

    // activity sets: tile J matters to epilogue warp w only if w's tile maximum (its
    // 32 rows x its 64 keys, from the MAX sweep) reaches the lowest threshold of its
    // rows (lowered by a few ulps: a superset); set 0 (HIST): z >= 0 <=>
    // acc >= -B/A1; set 1 (CAND / REF): z > lo - eps.  A warp skips the epilogue work
    // of the tiles outside its set (it only releases the S buffer), and the MMAs of a
    // row group skip the tiles outside the union of its 8 warps' sets.
    auto publish_set = [&](int s, float thr, bool arrive) {
      thr = warp_min(thr);
      for (int i = tid; i < 2 * aw; i += kEpi) sAct[s * 2 * aw + i] = 0u;
      bar_sync(3, kEpi);
      for (int w0 = 0; w0 < aw; ++w0) {
        const int J = 32 * w0 + lane;
        const bool on = J <= own_jl && (!wt || wt[J] >= thr);
        const uint32_t bits = __ballot_sync(0xffffffffu, on);
        if (lane == 0) {
          sWAct[(s * kEpiWarps + ew) * aw + w0] = bits;
          if (bits) atomicOr(&sAct[(s * 2 + rg) * aw + w0], bits);
        }
      }
      bar_sync(3, kEpi);
      if constexpr (PAIR) pair_or_words(sActU + s * 2 * aw, sAct + s * 2 * aw, 2 * aw);
      if (arrive && tid == 0) mbar_arrive(plan_bar);
    };
    // (list mode: one plan_bar arrival after both sets -- consecutive arrivals
    // could run a waiter's parity two phases behind)
    {
      float th = (float)(-B / (double)A1);
      th -= 4e-7f * fabsf(th) + 1e-30f;
      publish_set(0, th, !list_mode);
    }

    // combine the two key halves' counts (bins < kmin dropped: incomplete in
    // list mode) and solve; the half-0 thread owns the row's solver state
    const int nb = g.bins;  // 2..16 on this path (tc_supported)
    uint32_t* row_cnt = sCnt + e * 16;
    RowSolve rs;
    rs.tau = 0.0;
    rs.lo = rs.hi = 0.0;
    rs.steps = 0;
    rs.done = true;
    // half 0: the row's solver state from its full counts c32 (solve_histogram +
    // refine_bracket, histogram.cpp:73-165)
    auto solve_c32 = [&](const uint32_t* c32) {
      double th, lo, hi;
      solve_histogram_dev(c32, nb, g.alpha, th, lo, hi);
      if (g.tau_h_out) g.tau_h_out[(size_t)bh * g.n + grow] = th;
      rs.tau = th;
      rs.lo = lo;
      rs.hi = hi;
      rs.f = rs.f1 = rs.f2 = rs.f_hi = 0.0;
      rs.sec_tau = rs.sec_f = rs.best_tau = 0.0;
      rs.best_af = CUDART_INF;
      rs.steps = 0;
      rs.sec_seeded = false;
      rs.done = false;
      sRow[e * 4 + 2] = (float)(B - rs.tau);
      sRow[e * 4 + 3] = (float)(B - rs.hi);
    };
    // the two key halves' HIST counts (cnt[16] per thread, nb <= 16 or the low /
    // high 16 bins of nb = 32), combined through row_cnt, then solved by half 0
    auto solve_counts = [&](const uint32_t* cnt, const uint32_t* cnt_hi) {
      uint32_t c32[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) c32[k] = 0u;
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        const uint32_t* c = part ? cnt_hi : cnt;
        if (!c) break;
        if (half == 1) {
#pragma unroll
          for (int k = 0; k < 16; ++k) row_cnt[k] = c[k];
        }
        bar_sync(bar_rg, 256);
        if (half == 0) {
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (16 * part + k < nb) c32[16 * part + k] = c[k] + row_cnt[k];
        }
        bar_sync(bar_rg, 256);
      }
      if (half == 0) solve_c32(c32);
    };

    // ---- pass HIST (attention.cpp:201-232): counts of min(floor(B z), B-1), z >= 0
    auto hist_solve = [&]() {
      const float cw = 1.0f - 0x1p-20f;  // keeps z = 1 (the row max) inside bin nb-1
      const float2 Aw = make_float2(A1 * (float)nb * cw, A1 * (float)nb * cw);
      const float bw = (float)((B + 1.0) * (double)nb * (double)cw);
      const float2 Bw = make_float2(bw, bw);
      const float kf = -(0x1p-124f + (float)nb * 0x1p-147f);  // -(2^23 + nb) 2^-147, exact
      const float2 K = make_float2(kf, kf);
      if (nb <= 16) {
        uint32_t cnt[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) cnt[k] = 0;
        if (nb <= 8)
          hist_sweep<1>(jl, Aw, Bw, K, cnt, [&](int J) { return act(0, rg, J); },
                        [&](int J, uint32_t* hE, uint32_t* hO) {
            tau_tile(J, wact(0, J), [&](const float* v) { hist_nib<1>(v, Aw, Bw, K, hE, hO); });
          });
        else
          hist_sweep<2>(jl, Aw, Bw, K, cnt, [&](int J) { return act(0, rg, J); },
                        [&](int J, uint32_t* hE, uint32_t* hO) {
            tau_tile(J, wact(0, J), [&](const float* v) { hist_nib<2>(v, Aw, Bw, K, hE, hO); });
          });
        PASS_MARK(1);
        solve_counts(cnt, nullptr);
      } else {
        if constexpr (NB32) {  // bins = 32: four nibble words
          uint32_t cnt[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) cnt[k] = 0;
          hist_sweep<4>(jl, Aw, Bw, K, cnt, [&](int J) { return act(0, rg, J); },
                        [&](int J, uint32_t* hE, uint32_t* hO) {
            tau_tile(J, wact(0, J), [&](const float* v) { hist_nib<4>(v, Aw, Bw, K, hE, hO); });
          });
          PASS_MARK(1);
          solve_counts(cnt, cnt + 16);
        }
      }
      phase_tick(pacc, 1, pt);
    };

    const bool need_sec = g.alpha > 2.0;
    const double e0 = g.e0;
    bool first_pass = true;
    uint32_t dround = 0;
    bool list_ok = false;
    bool so = false;  // O from the support lists (this CTA's rows all in the pool)

    // ---- pass CAND: every score that can matter for the histogram solve, for
    // tau in [lo, hi] or for the mask is appended to a per-thread list as (raw
    // score, 64-key block); histogram, solve_histogram and the refinement
    // (attention.cpp:201-332) then run on the lists with no further sweeps.
    //
    // List mode skips the HIST sweep.  The rows' kTop-per-thread largest scores
    // form a subset histogram whose bracket floor k_s bounds the full
    // histogram's floor k from below: f_h(e) = -1 + sum over bins above e of
    // count * (edge - e)^e0 only grows when entries are added, so the largest
    // edge with f_h >= 0 only moves up.  solve_histogram reads only the bins
    // above its floor (histogram.cpp:104-159), so the bins >= k_s -- complete in
    // a list of every score with z > k_s / B - eps -- give the exact tau_h, and
    // tau >= tau_h >= k_s / B covers f, f', f'' and the mask (z > tau - 1e-9).
    // Sweep mode (alpha < 1.4: lists too long) keeps HIST and the REF sweeps;
    // a list overflow falls back to them too.
    // Each listed term is evaluated with the sweeps' formula t = A1*acc + (B - tau).
    int k_s = 0;  // (half 0, list mode) subset floor: bins >= k_s are complete
    if (!list_mode) hist_solve();
    if (list_mode) {
      float* row_top = reinterpret_cast<float*>(row_cnt);
      if (half == 1) {
#pragma unroll
        for (int i = 0; i < kTop; ++i) row_top[i] = top[i];
      }
      bar_sync(bar_rg, 256);
      if (half == 0) {
        uint32_t c32[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) c32[k] = 0u;
        auto bin_in = [&](float acc) {
          const float z = fmaf(A1, acc, Bf);
          if (z >= 0.f) ++c32[min((int)((float)nb * z), nb - 1)];
        };
#pragma unroll
        for (int i = 0; i < kTop; ++i) {
          bin_in(top[i]);
          bin_in(row_top[i]);
        }
        double th, lo, hi;
        int fl;
        solve_histogram_dev(c32, nb, g.alpha, th, lo, hi, &fl);
        k_s = fl > 0 ? fl : 0;
      }
    }
    // activity set 1 (CAND / REF sweeps): scores with z <= lo - eps (sweep mode:
    // lo = tau_h; list mode: k_s / B <= tau_h) reach neither the solve, nor
    // f, f', f'' (tau >= lo), nor the mask (z > tau - 1e-9)
    if (half == 0) {
      const float eps_t = 1e-6f * (2.f + fabsf(Bf));  // fp32 slack of z (|B| scale)
      const double lo_set = list_mode ? (double)k_s / nb : rs.lo;
      sRow[e * 4 + 0] = (float)(B - lo_set) + eps_t;
    }
    bar_sync(bar_rg, 256);
    // z > lo - eps  <=>  acc > theta (A1 > 0), lowered by a few ulps (superset)
    float theta = -sRow[e * 4 + 0] / A1;
    theta -= 4e-7f * fabsf(theta) + 1e-30f;
    if (!row_real) theta = 3.0e38f;  // padding rows list nothing
    publish_set(1, theta, true);

    if (a.cand) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      const int cap = a.cand_cap;
      uint2* lst = a.cand + ((size_t)smid * kEpi + (size_t)(tid)) * (size_t)cap;
      bool ovf = (int)smid >= a.cand_slots;  // (uniform: one CTA per SM)
      int cnt = 0;
      {
        // carry-free 32-bit append offsets: a list never crosses a 4 GB boundary
        // (4 KB-aligned regions of cap * 8 bytes); a region that would is treated
        // as an overflow (the CTA's sweeps take over)
        const uint64_t lst64 = reinterpret_cast<uint64_t>(lst);
        const uint32_t lo0 = (uint32_t)lst64, hi = (uint32_t)(lst64 >> 32);
        uint32_t lo = lo0;
        if ((uint64_t)lo0 + (uint64_t)cap * 8u > 0x100000000ull) ovf = true;
#define CAND_USED ((int)((lo - lo0) >> 3))
        for (int J = 0; J <= jl; ++J) {
          if (!act(1, rg, J)) continue;
          // entries carry the key index (its 64-key block is key >> 6)
          const uint32_t key0 = (uint32_t)(J * BN + half * 64);
          int ck = 0;  // 32-key chunk of the tile the body is called for
          // a tile appends <= 64 entries; warp-uniform (the append votes are warp-collective)
          ovf = __any_sync(0xffffffffu, ovf || CAND_USED > cap - 64);
          tau_tile(J, wact(1, J), [&](const float* v) {
            const uint32_t kc = key0 + 32u * (uint32_t)(ck++);
            if (ovf) return;
            // candidates are rare (~0.4% of scores): one 3-input max + warp vote per
            // 4 scores keeps the common path at 2 FMNMX + compare + vote + branch; the
            // appends advance a 32-bit offset (no 64-bit carry chains, measured -0.9 ms)
            CandGroups<0>::run(lo, v, theta, kc, hi);
          });
        }
        cnt = CAND_USED;
#undef CAND_USED
#ifdef ADATTN_PIPE_STATS
        // [26] listed entries, [27] listing threads, [28] longest list, [29] overflowed threads
        atomicAdd(&g_pipe_stats[26], (unsigned long long)cnt);
        atomicAdd(&g_pipe_stats[27], 1ull);
        atomicMax(&g_pipe_stats[28], (unsigned long long)cnt);
        if (ovf) atomicAdd(&g_pipe_stats[29], 1ull);
#endif
      }
      PASS_MARK(2);
      bool ovf_any = bar_red_or(4, kEpi, ovf);
      LIST_MARK(0);  // all warps done with CAND
      if constexpr (PAIR) ovf_any = pair_or(ovf_any);  // both CTAs take the same path
      if (!ovf_any) {
        // The K ring is idle until the decision (producer and MMA warps wait on
        // dec_bar): stage each thread's first `lcap` listed scores there
        // ([i][thread] layout, conflict-free) so the refinement rounds read
        // shared memory instead of waiting on L2 per entry.
        float* sl = reinterpret_cast<float*>(sRing);
        constexpr int lcap = NST * L::TILE / (kEpi * 4);
        // Whole-list staging: the CTA's lists packed back to back in the ring (an
        // exclusive prefix sum of the counts; scores f32, then their 64-key blocks u16)
        // when they all fit (C3 gaussian: ~17K entries, room for 21.8K).  The
        // refinement rounds and the mask pass then read shared memory only -- with
        // per-thread staging the longest lists of a CTA (up to ~230 entries) were read
        // from L2 in every round and the barriers waited on them.  Otherwise each
        // thread's first lcap scores ([i][thread], conflict-free) and L2 beyond.
        // entries: f32 score + u16 key (m <= 65536: 21.8K entries at d = 128), else
        // f32 score + u16 key >> 6 + u8 key & 63 (18.7K)
        const bool k16 = g.m <= 65536;
        const int kEmax = k16 ? NST * L::TILE / 6 : NST * L::TILE / 7;
        uint16_t* sblk = reinterpret_cast<uint16_t*>(sRing + 4 * kEmax);  // key (k16) or key >> 6
        uint8_t* sko = sRing + 6 * kEmax;                                   // key & 63 (!k16)
        int sbase = 0;
        bool full;
        {
          int x = cnt;  // inclusive warp scan of the counts
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
          }
          if (lane == 31) sScan[warp] = x;
          bar_sync(3, kEpi);
          int pre = 0, tot = 0;
#pragma unroll
          for (int w = 0; w < kEpiWarps; ++w) {
            const int t = sScan[w];
            pre += w < warp ? t : 0;
            tot += t;
          }
          sbase = pre + x - cnt;
          full = a.list_stage != 0 && tot <= kEmax;  // CTA-uniform
        }
        const int ns = full ? cnt : (cnt < lcap ? cnt : lcap);
        auto sidx = [&](int i) { return full ? sbase + i : i * kEpi + tid; };
        // the histogram of the listed scores (list mode), read in the same pass:
        // both halves of a row add into its 32 packed 16-bit counters in row_cnt
        // (a row lists <= 2 x 512 scores)
        if (half == 0) {
#pragma unroll
          for (int k = 0; k < 16; ++k) row_cnt[k] = 0u;
        }
        bar_sync(bar_rg, 256);
        // 16 entries (8 x 16-byte loads) in flight from L2; lists start 4 KB-aligned and
        // an odd count reads one entry past its end, inside the thread's region
        for (int i0 = 0; i0 < cnt; i0 += 16) {
          uint4 q8[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            q8[j] = i0 + 2 * j < cnt ? reinterpret_cast<const uint4*>(lst + i0)[j]
                                     : make_uint4(0xFF800000u, 0u, 0xFF800000u, 0u);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int i = i0 + j;
            const uint32_t sx = (j & 1) ? q8[j >> 1].z : q8[j >> 1].x;
            const uint32_t sy = (j & 1) ? q8[j >> 1].w : q8[j >> 1].y;
            if (i < ns) {
              sl[sidx(i)] = __uint_as_float(sx);
              if (full) {
                if (k16) {
                  sblk[sbase + i] = (uint16_t)sy;
                } else {
                  sblk[sbase + i] = (uint16_t)(sy >> 6);
                  sko[sbase + i] = (uint8_t)(sy & 63u);
                }
              }
            }
            const float z = fmaf(A1, __uint_as_float(sx), Bf);
            if (i < cnt && z >= 0.f) {
              const int k = min((int)((float)nb * z), nb - 1);
              atomicAdd(&row_cnt[k >> 1], 1u << (16 * (k & 1)));
            }
          }
        }
        LIST_MARK(1);  // staging + histogram
        if (list_mode) {
          bar_sync(bar_rg, 256);
          if (half == 0) {  // bins >= k_s are complete in the lists
            uint32_t c32[32];
#pragma unroll
            for (int k = 0; k < 32; ++k)
              c32[k] = (k < nb && k >= k_s) ? (row_cnt[k >> 1] >> (16 * (k & 1))) & 0xFFFFu : 0u;
            solve_c32(c32);
          }
          // sPart (refinement partials) aliases the count rows of the OTHER row
          // group (sCnt): both groups finish reading counts before any writes them
          bar_sync(3, kEpi);
          phase_tick(pacc, 1, pt);
        }
        LIST_MARK(2);  // histogram solve
        // refinement rounds on the lists (same RowSolve / row_step as the sweeps)
        for (;;) {
          bar_sync(bar_rg, 256);  // C / Chi published
          const float C = sRow[e * 4 + 2];
          const float Chi = sRow[e * 4 + 3];
          double f = 0.0, f1 = 0.0, f2 = 0.0, fhi = 0.0;
          for (int i0 = 0; i0 < cnt; i0 += 8) {
            // 8 loads in flight (entries past the staged ones come from L2)
            float accs[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int i = i0 + j;
              accs[j] = i < ns ? sl[sidx(i)]
                               : (i < cnt ? __uint_as_float(lst[i].x) : -CUDART_INF_F);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
            const float acc = accs[j];
            const float t = fmaf(A1, acc, C);
            if (t > 0.f) {
              if constexpr (AK == AK15) {
                f += (double)(t * t);
                f1 += (double)t;
                f2 += 1.0;
              } else if constexpr (AK == AK2) {
                f += (double)t;
                f1 += 1.0;
              } else if constexpr (AK == AK125) {
                const float t2 = t * t;
                f += (double)(t2 * t2);
                f1 += (double)(t2 * t);
                f2 += (double)t2;
              } else {
                const float lt = __log2f(t);
                const float l1 = a.e1f < 0.f ? __log2f(fmaxf(t, 1e-12f)) : lt;
                const float l2 = a.e2f < 0.f ? __log2f(fmaxf(t, 1e-12f)) : lt;
                f += (double)exp2f(a.e0f * lt);
                f1 += a.e1f == 0.f ? 1.0 : (double)exp2f(a.e1f * l1);
                f2 += a.e2f == 0.f ? 1.0 : (double)exp2f(a.e2f * l2);
              }
            }
            if (first_pass && need_sec) {
              const float th = fmaf(A1, acc, Chi);
              if (th > 0.f) fhi += (double)exp2f(a.e0f * __log2f(th));
            }
            }
          }
          if (half == 1) {
            sPart[e * 4 + 0] = f;
            sPart[e * 4 + 1] = f1;
            sPart[e * 4 + 2] = f2;
            sPart[e * 4 + 3] = fhi;
          }
          bar_sync(bar_rg, 256);
          bool stepped = false;
          if (half == 0 && !rs.done) {
            rs.f = -1.0 + (f + sPart[e * 4 + 0]);
            rs.f1 = -e0 * (f1 + sPart[e * 4 + 1]);
            rs.f2 = e0 * (e0 - 1.0) * (f2 + sPart[e * 4 + 2]);
            if (first_pass) rs.f_hi = -1.0 + (fhi + sPart[e * 4 + 3]);
            stepped = row_step(rs, g.alpha, g.refine_tol, g.refine_iters, need_sec);
            sRow[e * 4 + 2] = (float)(B - rs.tau);
          }
          first_pass = false;
          const bool more = bar_red_or(4, kEpi, stepped);
          LIST_MARK(3);  // refinement rounds
          if (!more) break;
        }
        // mask at the final tau: block active iff any z > tau - 1e-9 (attention.cpp:254-266)
        for (int i = tid; i < 4 * wpr; i += kEpi) smask[i] = 0u;
        bar_sync(3, kEpi);
        {
          const float C = sRow[e * 4 + 2];
          // support lists (delta from the support in the backward): the entries with
          // t > 0 at the final tau, in list order, packed per CTA (256 rows) in a pool of
          // supp_cap entries per row: counted in the mask pass, placed by a prefix sum over
          // the CTA's threads, written by a second pass over the staged list
          const bool sup = a.supp != nullptr;
          int ns_ = 0;
          if (full) {
            for (int i0 = 0; i0 < cnt; i0 += 8) {
              float accs[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) accs[j] = i0 + j < cnt ? sl[sbase + i0 + j] : -CUDART_INF_F;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float t = fmaf(A1, accs[j], C);
                if (row_real && t > -1e-9f) {
                  const uint32_t bk = k16 ? (uint32_t)sblk[sbase + i0 + j] >> 6 : sblk[sbase + i0 + j];
                  atomicOr(&smask[rb * wpr + (bk >> 5)], 1u << (bk & 31));
                  ns_ += t > 0.f;
                }
              }
            }
          } else {
            for (int i0 = 0; i0 < cnt; i0 += 8) {
              uint2 en[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) en[j] = i0 + j < cnt ? lst[i0 + j] : make_uint2(0xFF800000u, 0u);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float t = fmaf(A1, __uint_as_float(en[j].x), C);
                if (row_real && t > -1e-9f) {
                  const uint32_t bk = en[j].y >> 6;
                  atomicOr(&smask[rb * wpr + (bk >> 5)], 1u << (bk & 31));
                  ns_ += t > 0.f;
                }
              }
            }
          }
          if (sup) {
            int x = ns_;  // inclusive warp scan, then the 16 warp totals
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int y = __shfl_up_sync(0xffffffffu, x, o);
              if (lane >= o) x += y;
            }
            bar_sync(3, kEpi);  // (sScan of the staging scan consumed)
            if (lane == 31) sScan[warp] = x;
            bar_sync(3, kEpi);
            int pre = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < kEpiWarps; ++w) {
              const int tw = sScan[w];
              pre += w < warp ? tw : 0;
              tot += tw;
            }
            const int pc = BM * a.supp_cap;  // the CTA's pool
            const size_t blk256 = ((size_t)bh * g.n + row0) / BM;
            const size_t srow = (size_t)bh * g.n + grow;
            so = a.supp_o != 0 && tot <= pc;  // (CTA-uniform)
            if (tot > pc) {
              if (tid == 0) {  // the delta kernel (and the tensor-core backward) take these rows
                a.supp_flag[blk256] = 1u;
                a.supp_hflag[bh] = 1u;
              }
            } else {
              int off = pre + x - ns_;
              a.supp_cnt[srow * 2 + half] = make_int2(ns_, off);
              uint2* pool = a.supp + blk256 * (size_t)pc;
              for (int i0 = 0; i0 < cnt; i0 += 8) {  // 8 entries in flight
                float accs[8];
                uint32_t keys[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  const int i = i0 + j;
                  if (i >= cnt) {
                    accs[j] = -CUDART_INF_F;
                    keys[j] = 0u;
                  } else if (full) {
                    accs[j] = sl[sbase + i];
                    keys[j] = k16 ? (uint32_t)sblk[sbase + i]
                                  : ((uint32_t)sblk[sbase + i] << 6) | sko[sbase + i];
                  } else {
                    const uint2 en = lst[i];
                    accs[j] = __uint_as_float(en.x);
                    keys[j] = en.y;
                  }
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  const float t = fmaf(A1, accs[j], C);
                  if (row_real && t > 0.f) {
                    pool[off++] = make_uint2(keys[j], __float_as_uint(t));
                    atomicAdd(&a.supp_kcnt[(size_t)bh * g.m + keys[j]], 1);  // (the transpose)
                  }
                }
              }
            }
          }
        }
        fence_proxy_async_smem();  // generic writes to the ring before its next TMA loads
        list_ok = true;
        phase_tick(pacc, 2, pt);
        LIST_MARK(4);  // mask
      }
      PASS_MARK(3);
      bar_sync(3, kEpi);
      if (PAIR && list_ok) pair_or_words(sPm, smask, 4 * wpr);
      if (list_ok) {
        if (so) {  // no output pass: sparse_out_kernel forms O from the support lists
          if (tid == 0) *s_ntiles = 0u;
        } else if (warp == 0) {
          build_tiles();
        }
        bar_sync(3, kEpi);
      }
      if (tid == 0) {
        *s_decision = list_ok ? DEC_OUT : DEC_REF;
        mbar_arrive(dec_bar);
      }
      LIST_MARK(5);  // tile list + decision
      dround = 1;
      if (!list_ok) {
        // no support lists for this CTA's rows: the backward's delta kernel takes the head
        if (tid == 0 && a.supp) {
          a.supp_flag[((size_t)bh * g.n + row0) / BM] = 1u;
          a.supp_hflag[bh] = 1u;
        }
        hist_solve();  // fallback: the exact histogram by the HIST sweep
      }
    }

    // ---- passes REF (attention.cpp:234-332): sweeps (no lists, or a list overflowed)
    for (uint32_t ref = 0; !list_ok; ++ref) {
      for (int i = tid; i < 4 * wpr; i += kEpi) smask[i] = 0u;
      bar_sync(3, kEpi);  // C/Chi published, masks cleared, counts consumed
      const float C = sRow[e * 4 + 2];
      const float Chi = sRow[e * 4 + 3];
      KahanF f, f1, f2, fhi;  // compensated fp32 over the fp32 slice sums
      for (int J = 0; J <= jl; ++J) {
        if (!act(1, rg, J)) continue;
        float mx_t = -CUDART_INF_F;
        tau_tile(J, wact(1, J), [&](const float* v) {
          float s0, s1, s2, mx;
          ref_slice<AK>(v, A1, C, a.e0f, a.e1f, a.e2f, s0, s1, s2, mx);
          if (first_pass && need_sec) {
            float shi = 0.f;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float th = fmaf(A1, v[i], Chi);
              if (th > 0.f) shi += exp2f(a.e0f * __log2f(th));
            }
            fhi.add(shi);
          }
          f.add(s0);
          f1.add(s1);
          f2.add(s2);
          mx_t = fmaxf(mx_t, mx);
        });
        const int jt = 2 * J + half;  // reference key tile of this thread's half
        if (__any_sync(0xffffffffu, row_real && mx_t > -1e-9f) && lane == 0)
          atomicOr(&smask[rb * wpr + (jt >> 5)], 1u << (jt & 31));
      }
      if (half == 1) {
        sPart[e * 4 + 0] = f.get();
        sPart[e * 4 + 1] = f1.get();
        sPart[e * 4 + 2] = f2.get();
        sPart[e * 4 + 3] = fhi.get();
      }
      bar_sync(bar_rg, 256);
      bool stepped = false;
      if (half == 0 && !rs.done) {
        rs.f = -1.0 + (f.get() + sPart[e * 4 + 0]);
        rs.f1 = -e0 * (f1.get() + sPart[e * 4 + 1]);
        rs.f2 = e0 * (e0 - 1.0) * (f2.get() + sPart[e * 4 + 2]);
        if (first_pass) rs.f_hi = -1.0 + (fhi.get() + sPart[e * 4 + 3]);
        stepped = row_step(rs, g.alpha, g.refine_tol, g.refine_iters, need_sec);
        sRow[e * 4 + 2] = (float)(B - rs.tau);
      }
      first_pass = false;
      bool any = bar_red_or(4, kEpi, stepped);
      if constexpr (PAIR) {
        any = pair_or(any);
        if (!any) pair_or_words(sPm, smask, 4 * wpr);
      }
      if (!any) {
        if (warp == 0) build_tiles();
        bar_sync(3, kEpi);
      }
      if (tid == 0) {
        *s_decision = any ? DEC_REF : DEC_OUT;
        mbar_arrive(dec_bar);
      }
      if (!any) break;
    }

    PASS_MARK(4);
    if (!list_ok) phase_tick(pacc, 2, pt);
    // ---- pass OUT (attention.cpp:334-352): P over the active blocks, O = P V
#if ADATTN_OUT_ALL16
    {
      // All 16 epilogue warps work on each row group's tile in turn (warp w: TMEM
      // lane quarter w % 4, keys 32 (w / 4) .. +31 of the tile), so a group's P is
      // ready in half the time one group's 8 warps need: with a single S buffer per
      // group in this pass, that turnaround is what the other group's MMAs must cover.
      // P of a 32-key chunk goes over the first 16 of the chunk's own S columns.
      const int qq = ew >> 2;  // 32-key chunk of the tile
      if ((ew & 7) == 0 && lane == 0) misc[4 + rg] = it;
      bar_sync(3, kEpi);
      uint32_t ob[2], gC[2];
      int gklim[2];
#pragma unroll
      for (int g2 = 0; g2 < 2; ++g2) {
        ob[g2] = (misc[4 + g2] + 1) >> 1;  // previous uses of S buffer 0 of group g2
        const int eg = g2 * 128 + lq * 32 + lane;
        gC[g2] = __float_as_uint(sRow[eg * 4 + 2]);
        const int gr = row0 + eg;
        gklim[g2] = g.causal ? min(gr, g.m_valid - 1) : g.m_valid - 1;
      }
      bool any_out = false;  // for the O write: tiles of this thread's own group rg
      const uint32_t tq = tmem + ((uint32_t)(lq * 32) << 16) + 32 * qq;
      for (uint32_t t = 0, nt_ = fold ? 0u : *s_ntiles; t < nt_; ++t) {
        const int J = sTiles[t];
#pragma unroll
        for (int g2 = 0; g2 < 2; ++g2) {
          if (!out_active(g2, J)) continue;
          if (g2 == rg) any_out = true;
          // pairs: a tile active for the peer's rows only gets P = 0 without reading S
          const bool own = !PAIR || out_active_m(smask, g2, J);
          MBAR_WAIT(&s_full[g2], ob[g2] & 1);  // output-pass S lives in buffer 0
          ++ob[g2];
          tc_fence_after();
          uint32_t pk[16];
          if (own) {
            tmem_ld32(tq + g2 * 128, v);
            tmem_wait_ld();
            const int k0 = J * BN + 32 * qq;
            if (k0 + 31 > gklim[g2]) {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (k0 + i > gklim[g2]) v[i] = -CUDART_INF_F;
            }
            const float C = __uint_as_float(gC[g2]);
            const float2 A2 = make_float2(A1, A1), C2 = make_float2(C, C);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float2 t = __ffma2_rn(A2, make_float2(v[2 * i], v[2 * i + 1]), C2);
              float2 pp;
              if constexpr (AK == AK15 || AK == AK125 || AK == AK2) {  // packed powers
                const float2 tp = make_float2(fmaxf(t.x, 0.f), fmaxf(t.y, 0.f));
                if constexpr (AK == AK2) {
                  pp = tp;
                } else {
                  pp = __fmul2_rn(tp, tp);
                  if constexpr (AK == AK125) pp = __fmul2_rn(pp, pp);
                }
              } else {
                pp = make_float2(p_of<AK>(t.x, a.e0f), p_of<AK>(t.y, a.e0f));
              }
              pk[i] = pvf16 ? pack_f16x2(pp.x, pp.y) : pack_bf16x2(pp.x, pp.y);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = 0u;
          }
          tmem_st16(tq + g2 * 128, pk);
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_mma(&p_full[g2]);
        }
      }
#else
    {
      const float C = sRow[e * 4 + 2];
      const float2 A2 = make_float2(A1, A1), C2 = make_float2(C, C);
      bool any_out = false;
      uint32_t ob = (it + 1) >> 1;  // previous uses of S buffer 0 of this group
      for (uint32_t t = 0, nt_ = fold ? 0u : *s_ntiles; t < nt_; ++t) {
        const int J = sTiles[t];
        if (!out_active(rg, J)) continue;
        any_out = true;
        const bool own = !PAIR || out_active_m(smask, rg, J);
        MBAR_WAIT(&s_full[rg], ob & 1);
        ++ob;
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t pk[16];
          if (own) {
            load_chunk(0, J, c);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float2 t = __ffma2_rn(A2, make_float2(v[2 * i], v[2 * i + 1]), C2);
              float2 pp;
              if constexpr (AK == AK15 || AK == AK125 || AK == AK2) {
                const float2 tp = make_float2(fmaxf(t.x, 0.f), fmaxf(t.y, 0.f));
                if constexpr (AK == AK2) {
                  pp = tp;
                } else {
                  pp = __fmul2_rn(tp, tp);
                  if constexpr (AK == AK125) pp = __fmul2_rn(pp, pp);
                }
              } else {
                pp = make_float2(p_of<AK>(t.x, a.e0f), p_of<AK>(t.y, a.e0f));
              }
              pk[i] = pvf16 ? pack_f16x2(pp.x, pp.y) : pack_bf16x2(pp.x, pp.y);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = 0u;
          }
          // keys 64*half + 32c .. +31 -> the first 16 of that chunk's own S columns
          tmem_st16(tl + c * 32, pk);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_mma(&p_full[rg]);
      }
#endif
      if (fold) {
        // delta fold: P and U = p^(2 - alpha) of item i over the first /
        // second 16 columns of each 32-key chunk of S buffer i & 1; the MMA warp
        // accumulates O += P V and Ubar += U V; per row group, O, Ubar and sum u go
        // to HBM (the backward forms delta = dO . Ubar / sum u, attention.cpp:411-446)
        const int qq = ew >> 2;  // 32-key chunk of the tile
        const uint32_t tq = tmem + ((uint32_t)(lq * 32) << 16) + 32 * qq;
        float* sUs = reinterpret_cast<float*>(sCnt);  // [256][4] partial sums of u
        uint32_t fi = 0, ndone = 0;
        for (int g2 = 0; g2 < 2; ++g2) {
          const int eg = g2 * 128 + lq * 32 + lane;
          const int gr = row0 + eg;
          const float Cg = sRow[eg * 4 + 2];
          const int klg = g.causal ? min(gr, g.m_valid - 1) : g.m_valid - 1;
          const float2 A2 = make_float2(A1, A1), C2 = make_float2(Cg, Cg);
          float us = 0.f;
          bool anyg = false;
          for (uint32_t t = 0, nt_ = *s_ntiles; t < nt_; ++t) {
            const int J = sTiles[t];
            if (!out_active(g2, J)) continue;
            anyg = true;
            const uint32_t b = fi & 1;
            MBAR_WAIT(&fs_full[b], (fi >> 1) & 1);
            ++fi;
            tc_fence_after();
            tmem_ld32(tq + b * 128, v);
            tmem_wait_ld();
            const int k0 = J * BN + 32 * qq;
            if (k0 + 31 > klg) {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (k0 + i > klg) v[i] = -CUDART_INF_F;
            }
            float2 u2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {  // keys 16 hh .. +15: P -> cols 8 hh, U -> 16 + 8 hh
              uint32_t pk[8], uk[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int x = 8 * hh + i;
                const float2 t = __ffma2_rn(A2, make_float2(v[2 * x], v[2 * x + 1]), C2);
                const float2 tp = make_float2(fmaxf(t.x, 0.f), fmaxf(t.y, 0.f));
                float2 pp, uu;
                if constexpr (AK == AK15) {
                  uu = tp;
                  pp = __fmul2_rn(tp, tp);
                } else if constexpr (AK == AK2) {
                  pp = tp;
                  uu = make_float2(__saturatef(tp.x * 0x1p126f), __saturatef(tp.y * 0x1p126f));
                } else if constexpr (AK == AK125) {
                  const float2 t2 = __fmul2_rn(tp, tp);
                  uu = __fmul2_rn(t2, tp);
                  pp = __fmul2_rn(t2, t2);  // (t^2)^2 like the P of the other output passes
                } else {
                  uu.x = tp.x > 0.f ? exp2f(a.e1f * __log2f(tp.x)) : 0.f;
                  uu.y = tp.y > 0.f ? exp2f(a.e1f * __log2f(tp.y)) : 0.f;
                  pp = make_float2(p_of<AK>(t.x, a.e0f), p_of<AK>(t.y, a.e0f));
                }
                u2 = __fadd2_rn(u2, uu);
                pk[i] = pvf16 ? pack_f16x2(pp.x, pp.y) : pack_bf16x2(pp.x, pp.y);
                uk[i] = pvf16 ? pack_f16x2(uu.x, uu.y) : pack_bf16x2(uu.x, uu.y);
              }
              tmem_st8(tq + b * 128 + 8 * hh, pk);
              tmem_st8(tq + b * 128 + 16 + 8 * hh, uk);
            }
            us += u2.x + u2.y;
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&fp_full[b]);
          }
          // O and Ubar of this row group: lane quarter lq, columns 32 qq .. +31
          const bool rd = 32 * qq < D;
          const size_t orow_g = (size_t)bh * g.n + gr;
          if (anyg) {
            MBAR_WAIT(fo_full, ndone & 1);
            ++ndone;
            tc_fence_after();
          }
#pragma unroll
          for (int which = 0; which < 2; ++which) {  // 0: O, 1: Ubar
            float o[32];
            if (anyg && rd) {
              tmem_ld32(tmem + ((uint32_t)(lq * 32) << 16) + 256 + 128 * which + 32 * qq, o);
              tmem_wait_ld();
            }
            if (which == 1 && anyg) {  // both read: group 1's products may overwrite them
              tc_fence_before();
              __syncwarp();
              if (g2 == 0 && lane == 0) mbar_arrive(fo_empty);
            }
            if (!rd) continue;
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = anyg ? o[i] * oinv : 0.f;
            if (which == 0 && g.out_dtype == ADATTN_F64) {
              double* dst = reinterpret_cast<double*>(a.out) + orow_g * D + 32 * qq;
#pragma unroll
              for (int i = 0; i < 32; ++i) dst[i] = (double)o[i];
            } else {
              float* base = which == 0 ? reinterpret_cast<float*>(a.out) : a.ubar;
              float4* dst = reinterpret_cast<float4*>(base + orow_g * D + 32 * qq);
#pragma unroll
              for (int i = 0; i < 8; ++i) dst[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
            }
          }
          sUs[eg * 4 + qq] = us;
        }
        bar_sync(3, kEpi);
        if (tid < BM) {
          const float* su = sUs + tid * 4;
          a.ubar[(size_t)g.bh * g.n * D + (size_t)bh * g.n + row0 + tid] = (su[0] + su[1]) + (su[2] + su[3]);
        }
      }
      // write O (fp32 or fp64): this thread's half of the row's dv columns
      const size_t orow = (size_t)bh * g.n + grow;
      if (!fold) MBAR_WAIT(o_full, 0);
      PASS_MARK(5);
      tc_fence_after();
      const bool written = __any_sync(0xffffffffu, any_out);
      const uint32_t to = tmem + ((uint32_t)(lq * 32) << 16) + 256 + rg * D + half * (D / 2);
#pragma unroll
      for (int c = 0; c < (fold || so ? 0 : D / 64); ++c) {
        float o[32];
        tmem_ld32(to + c * 32, o);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = written ? o[i] * oinv : 0.f;
        const int x0 = half * (D / 2) + c * 32;
        if (g.out_dtype == ADATTN_F64) {
          double* dst = reinterpret_cast<double*>(a.out) + orow * D + x0;
#pragma unroll
          for (int i = 0; i < 32; ++i) dst[i] = (double)o[i];
        } else {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + orow * D + x0);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            dst[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
        }
      }
      if (half == 0) {
        a.tau[orow] = rs.tau;
        a.row_max[orow] = (double)m_f;
        if (a.steps) a.steps[orow] = rs.steps;
      }
      for (int i = tid; i < 4 * wpr; i += kEpi) {
        const int rbi = i / wpr, w = i - rbi * wpr;
        a.mask[((size_t)bh * g.t_r + (row0 / 64 + rbi)) * wpr + w] = smask[i];
      }
      // the nonzero-block lists of the four row blocks (ELL, ascending key blocks),
      // emitted for the backward; laid out in the caller's (unpadded) geometry
      if (a.rcnt && warp < 4) {
        const int t_r_v = (g.n_valid + 63) / 64, t_c_v = (g.m_valid + 63) / 64;
        const int ib = row0 / 64 + warp;
        if (ib < t_r_v) {
          const size_t row = (size_t)bh * t_r_v + ib;
          uint16_t* out = a.rcol + row * t_c_v;
          uint32_t n = 0;
          for (int w0 = 0; w0 < wpr; w0 += 32) {
            const int w = w0 + lane;
            uint32_t bits = w < wpr ? smask[warp * wpr + w] : 0u;
            const int top = t_c_v - 32 * w;  // key blocks >= t_c_v are padding
            if (top < 32) bits &= top <= 0 ? 0u : ((1u << top) - 1u);
            const uint32_t c = __popc(bits);
            uint32_t pre = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t x = __shfl_up_sync(0xffffffffu, pre, o);
              if (lane >= o) pre += x;
            }
            uint32_t k = n + pre - c;
            for (; bits; bits &= bits - 1) out[k++] = (uint16_t)(32 * w + __ffs(bits) - 1);
            n += __shfl_sync(0xffffffffu, pre, 31);
          }
          if (lane == 0) a.rcnt[row] = (int32_t)n;
        }
      }
    }
    PASS_MARK(6);
    phase_tick(pacc, 3, pt);
  }
  tc_fence_before();
  if constexpr (PAIR) {
    cluster_sync();  // the pair's MMAs, remote arrives and DSMEM reads are done
    if (warp == kWarpProd) tmem_dealloc_2sm(tmem, 512);
  } else {
    __syncthreads();
    if (warp == kWarpProd) tmem_dealloc(tmem, 512);
  }
}

template <int D, int AK, bool PAIR>
cudaError_t launch_fwd(const Geom& g, const CUtensorMap& tq, const CUtensorMap& tk,
                       const CUtensorMap& tkh, const CUtensorMap& tv, const CUtensorMap& tv16,
                       const FwdArgs& a, cudaStream_t st) {
  const size_t smem = FwdSmem<D>::bytes(g.wpr, g.m / BN);
  auto kern = tc_fwd_kernel<D, AK, PAIR>;
  if constexpr (!PAIR) {
    if (g.bins > 16) kern = tc_fwd_kernel<D, AK, false, true>;
  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e) return e;
  const dim3 grid((unsigned)(a.ncta_rows * g.bh));
  prof_begin("tc_fwd", st);
  if constexpr (PAIR) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, tq, tk, tkh, tv, tv16, a);
  } else {
    kern<<<grid, kThreads, smem, st>>>(tq, tk, tkh, tv, tv16, a);
  }
  prof_end(st);
  note_launch();
  return e ? e : cudaGetLastError();
}

template <int D, bool PAIR>
cudaError_t launch_fwd_d(const Geom& g, int ak, const CUtensorMap& tq, const CUtensorMap& tk,
                         const CUtensorMap& tkh, const CUtensorMap& tv, const CUtensorMap& tv16,
                         const FwdArgs& a, cudaStream_t st) {
  switch (ak) {
    case AK15: return launch_fwd<D, AK15, PAIR>(g, tq, tk, tkh, tv, tv16, a, st);
    case AK2: return launch_fwd<D, AK2, PAIR>(g, tq, tk, tkh, tv, tv16, a, st);
    case AK125: return launch_fwd<D, AK125, PAIR>(g, tq, tk, tkh, tv, tv16, a, st);
    default: return launch_fwd<D, AKGEN, PAIR>(g, tq, tk, tkh, tv, tv16, a, st);
  }
}

// CTA pairs for the forward (ADATTN_FWD_PAIRS=0/1 overrides the default)
bool use_fwd_pairs(const Geom& g) {
  if (g.d != 128 || g.dv != 128 || (g.n / BM) % 2 != 0 || g.bins > 16) return false;
  const char* s = std::getenv("ADATTN_FWD_PAIRS");
  if (s && *s) return s[0] != '0';
  // With two MMA-issuing warps the single-CTA forward is the faster one at C3
  // (35.4 vs 37.9 ms, tools/ab.py); before, pairs won (37.0 vs 41.1 ms).
  return false;
}

}  // namespace

// The output pass folds the delta accumulation (single-CTA kernel only).  U goes
// through the tensor cores as fp16, so Ubar carries u's 2^-11 relative rounding:
// exact for alpha = 2 (u in {0, 1}), but at alpha = 1.5 delta moves by ~5e-3 on
// rows with small supports (a coherent per-row shift of dS), which exceeds the
// gradient bar on peaked inputs.  The support lists (list mode) are cheaper still
// (C3 alpha = 2: 83.6 vs 89.5 ms per step), so the fold is the default only for
// alpha = 2 without them (ADATTN_DELTA_FOLD=1 forces it on, 0 off).
bool fwd_delta_fold(const Geom& g) {
  if (!g.ubar_out || g.d != g.dv) return false;
  if (g.d == 128 && use_fwd_pairs(g)) return false;
  const char* s = std::getenv("ADATTN_DELTA_FOLD");
  if (s && *s) return *s != '0';
  return g.alpha == 2.0 && !delta_supp_possible(g);
}

int alpha_kind(double alpha) {
  if (alpha == 1.5) return AK15;
  if (alpha == 2.0) return AK2;
  if (alpha == 1.25) return AK125;
  return AKGEN;
}

// O from the support lists: O_i = sum_j p_ij v_j over the row's entries (key, t_ij > 0 at
// the final tau) -- the output pass's P V without the zero terms (attention.cpp:334-352),
// exact bf16 products summed in fp32 in list order.  One warp per row, lane l holds dv
// elements l*E..; rows of blocks the forward flagged (their CTA ran the output pass) are
// left alone.
template <int D, int AK>
__global__ void __launch_bounds__(256) sparse_out_kernel(
    const uint16_t* __restrict__ vv, const uint2* __restrict__ pool, const int2* __restrict__ cnt,
    const uint32_t* __restrict__ flag, int cap, float e0f, size_t rows, int n, int m, int out_f64,
    void* out) {
  constexpr int E = D / 32;
  const size_t r = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int2 h0 = cnt[r * 2], h1 = cnt[r * 2 + 1];  // (read beside the flag: one L2 trip)
  if (flag[r / 256]) return;
  const size_t bh = r / (size_t)n;
  const int c0 = h0.x, tot = h0.x + h1.x;
  const uint2* base = pool + (r / 256) * (size_t)(256 * cap);
  const uint16_t* vb = vv + bh * (size_t)m * D + lane * E;
  if constexpr (D == 64) {  // half-warps take alternate entries, 4 elements (8 bytes) a lane
    const int hf = lane >> 4, hl = lane & 15;
    const uint16_t* vb4 = vv + bh * (size_t)m * D + hl * 4;
    float a4[4] = {0.f, 0.f, 0.f, 0.f};
    for (int b = 0; b < tot; b += 32) {
      const int idx = b + lane;
      uint2 my = make_uint2(0u, 0u);
      if (idx < tot) my = idx < c0 ? base[h0.y + idx] : base[h1.y + idx - c0];
      const float pl = idx < tot ? p_of<AK>(__uint_as_float(my.y), e0f) : 0.f;
      const int nk = min(32, tot - b);
#pragma unroll kGatherUnroll
      for (int k2 = 0; k2 < (nk + 1) / 2; ++k2) {
        const int k = 2 * k2 + hf;
        const uint32_t key = __shfl_sync(0xffffffffu, my.x, k & 31);
        const float p = __shfl_sync(0xffffffffu, pl, k & 31);
        if (k < nk) {
          const uint2 w = *reinterpret_cast<const uint2*>(vb4 + (size_t)key * D);
          a4[0] = fmaf(p, __uint_as_float(w.x << 16), a4[0]);
          a4[1] = fmaf(p, __uint_as_float(w.x & 0xFFFF0000u), a4[1]);
          a4[2] = fmaf(p, __uint_as_float(w.y << 16), a4[2]);
          a4[3] = fmaf(p, __uint_as_float(w.y & 0xFFFF0000u), a4[3]);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) a4[e] += __shfl_xor_sync(0xffffffffu, a4[e], 16);
    if (hf == 0) {
      if (out_f64) {
        double* dst = reinterpret_cast<double*>(out) + r * D + hl * 4;
#pragma unroll
        for (int e = 0; e < 4; ++e) dst[e] = (double)a4[e];
      } else {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + r * D + hl * 4) =
            make_float4(a4[0], a4[1], a4[2], a4[3]);
      }
    }
    return;
  }
  float acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.f;
  for (int b = 0; b < tot; b += 32) {
    const int idx = b + lane;
    uint2 my = make_uint2(0u, 0u);
    if (idx < tot) my = idx < c0 ? base[h0.y + idx] : base[h1.y + idx - c0];
    const float pl = idx < tot ? p_of<AK>(__uint_as_float(my.y), e0f) : 0.f;
    const int nk = min(32, tot - b);
#pragma unroll kGatherUnroll
    for (int k = 0; k < nk; ++k) {
      const uint32_t key = __shfl_sync(0xffffffffu, my.x, k);
      const float p = __shfl_sync(0xffffffffu, pl, k);
      const uint16_t* vr = vb + (size_t)key * D;
      if constexpr (E == 4) {
        const uint2 w = *reinterpret_cast<const uint2*>(vr);
        acc[0] = fmaf(p, __uint_as_float(w.x << 16), acc[0]);
        acc[1] = fmaf(p, __uint_as_float(w.x & 0xFFFF0000u), acc[1]);
        acc[2] = fmaf(p, __uint_as_float(w.y << 16), acc[2]);
        acc[3] = fmaf(p, __uint_as_float(w.y & 0xFFFF0000u), acc[3]);
      } else {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(vr);
        acc[0] = fmaf(p, __uint_as_float(w << 16), acc[0]);
        acc[1] = fmaf(p, __uint_as_float(w & 0xFFFF0000u), acc[1]);
      }
    }
  }
  if (out_f64) {
    double* dst = reinterpret_cast<double*>(out) + r * D + lane * E;
#pragma unroll
    for (int e = 0; e < E; ++e) dst[e] = (double)acc[e];
  } else {
    float* dst = reinterpret_cast<float*>(out) + r * D + lane * E;
#pragma unroll
    for (int e = 0; e < E; ++e) dst[e] = acc[e];
  }
}

template <int D>
cudaError_t launch_sparse_out(const Geom& g, int ak, const FwdArgs& a, const void* v,
                              cudaStream_t st) {
  const SuppLayout sl = supp_layout(g, g.supp_out);
  const size_t rows = (size_t)g.bh * g.n;
  const unsigned grid = (unsigned)((rows * 32 + 255) / 256);
  const int f64 = g.out_dtype == ADATTN_F64 ? 1 : 0;
  const uint16_t* vb = reinterpret_cast<const uint16_t*>(v);
  prof_begin("tc_fwd_out", st);
  switch (ak) {
    case AK15: sparse_out_kernel<D, AK15><<<grid, 256, 0, st>>>(vb, sl.ent, sl.cnt, sl.flag, sl.cap, a.e0f, rows, g.n, g.m, f64, a.out); break;
    case AK2: sparse_out_kernel<D, AK2><<<grid, 256, 0, st>>>(vb, sl.ent, sl.cnt, sl.flag, sl.cap, a.e0f, rows, g.n, g.m, f64, a.out); break;
    case AK125: sparse_out_kernel<D, AK125><<<grid, 256, 0, st>>>(vb, sl.ent, sl.cnt, sl.flag, sl.cap, a.e0f, rows, g.n, g.m, f64, a.out); break;
    default: sparse_out_kernel<D, AKGEN><<<grid, 256, 0, st>>>(vb, sl.ent, sl.cnt, sl.flag, sl.cap, a.e0f, rows, g.n, g.m, f64, a.out); break;
  }
  prof_end(st);
  note_launch();
  return cudaGetLastError();
}

// O from the support lists (ADATTN_SPARSE_OUT=0: the output pass on the tensor cores);
// needs the support lists and the single-CTA forward
bool sparse_out_enabled() {
  const char* s = std::getenv("ADATTN_SPARSE_OUT");
  return !(s && *s == '0');
}

cudaError_t forward(const Geom& g, const void* q, const void* k, const void* v, void* out,
                    double* tau, double* row_max, uint32_t* mask, int32_t* steps, void* ws,
                    cudaStream_t st) {
  CUtensorMap tq, tk, tkh, tv, tv16;
  cudaError_t e;
  if ((e = make_tmap_2d(&tq, q, (uint64_t)g.bh * g.n, g.d, BM))) return e;
  if ((e = make_tmap_2d(&tk, k, (uint64_t)g.bh * g.m, g.d, BN))) return e;
  if ((e = make_tmap_3d_chunks(&tkh, k, (uint64_t)g.bh * g.m, g.d, 64))) return e;
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
  a.ubar = fwd_delta_fold(g) ? g.ubar_out : nullptr;
  a.wtm = ws ? reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + forward_wtm_offset(g)) : nullptr;
  a.wtm_slots = a.wtm ? forward_wtm_slots() : 0;
  a.rcnt = g.rl_cnt_out;
  a.rcol = g.rl_col_out;
  const CandPlan cp = cand_plan(g);
  // lists start 4 KB-aligned (forward_cand_bytes keeps 4 KB of slack): the appends'
  // 32-bit offsets then never carry with the default cap (4 KB regions; any other
  // region that would cross a 4 GB boundary takes the overflow path)
  a.cand = (cp.cap > 0 && ws)
               ? reinterpret_cast<uint2*>((reinterpret_cast<uintptr_t>(ws) + 4095) & ~uintptr_t(4095))
               : nullptr;
  a.cand_cap = cp.cap;
  a.cand_slots = cp.slots;
  a.supp = nullptr;
  a.supp_cnt = nullptr;
  a.supp_flag = nullptr;
  a.supp_hflag = nullptr;
  a.supp_kcnt = nullptr;
  a.supp_cap = 0;
  a.supp_o = 0;
  if (!a.ubar && a.cand && g.supp_out && delta_supp_enabled(g)) {  // (list mode only)
    const SuppLayout sl = supp_layout(g, g.supp_out);
    if ((e = cudaMemsetAsync(sl.flag, 0, 4 * sl.nblk, st))) return e;
    a.supp = sl.ent;
    a.supp_cnt = sl.cnt;
    a.supp_flag = sl.flag;
    a.supp_hflag = sl.hflag;
    a.supp_kcnt = sl.kcnt;
    a.supp_cap = sl.cap;
    if ((e = cudaMemsetAsync(sl.hflag, 0, 4 * (size_t)g.bh, st))) return e;
    if ((e = cudaMemsetAsync(sl.kcnt, 0, 4 * (size_t)g.bh * g.m, st))) return e;
  } else if (g.supp_out && delta_supp_enabled(g)) {  // no lists written: every head flagged
    const SuppLayout sl = supp_layout(g, g.supp_out);
    if ((e = cudaMemsetAsync(sl.flag, 1, 4 * sl.nblk, st))) return e;
    if ((e = cudaMemsetAsync(sl.hflag, 1, 4 * (size_t)g.bh, st))) return e;
  }
  {
    const char* ls = std::getenv("ADATTN_LIST_STAGE");
    a.list_stage = (ls && *ls == '0') ? 0 : 1;
  }
  a.v16_max = nullptr;
  tv16 = tv;
  // O from the support lists: the output pass runs only in flagged CTAs, which then take
  // bf16 P and V (no fp16 V copy for them)
  const bool pairs = g.d == 128 && use_fwd_pairs(g);
  const bool supp_o = a.supp && !pairs && g.d == g.dv && sparse_out_enabled();
  if (pv_f16_enabled() && ws && !supp_o) {
    uint8_t* w8 = reinterpret_cast<uint8_t*>(ws) + forward_cand_bytes(g);
    __half2* v16 = reinterpret_cast<__half2*>(w8);
    uint32_t* vmax = reinterpret_cast<uint32_t*>(w8 + ((size_t)g.bh * g.m * g.dv * 2 + 255) / 256 * 256);
    const size_t ve = (size_t)g.m * g.dv;  // per head
    if ((e = cudaMemsetAsync(vmax, 0, 4 * (size_t)g.bh, st))) return e;
    if ((e = f16_absmax(v, g.bh, ve, vmax, st))) return e;
    if ((e = f16_convert_scaled(v, v16, g.bh, ve, vmax, st))) return e;
    if ((e = make_tmap_2d(&tv16, v16, (uint64_t)g.bh * g.m, g.dv, BN))) return e;
    a.v16_max = vmax;
  }

  const int ak = alpha_kind(g.alpha);
  a.supp_o = supp_o ? 1 : 0;
  if (g.d == 64) e = launch_fwd_d<64, false>(g, ak, tq, tk, tkh, tv, tv16, a, st);
  else if (pairs) e = launch_fwd_d<128, true>(g, ak, tq, tk, tkh, tv, tv16, a, st);
  else e = launch_fwd_d<128, false>(g, ak, tq, tk, tkh, tv, tv16, a, st);
  if (e || !a.supp_o) return e;
  return g.dv == 64 ? launch_sparse_out<64>(g, ak, a, v, st) : launch_sparse_out<128>(g, ak, a, v, st);
}

}  // namespace tc
}  // namespace adattn_b200

#ifdef ADATTN_PIPE_TRACE
extern "C" unsigned adattn_b200_trace_read(unsigned long long* out, int reset) {
  const unsigned n = 64u << 12;
  if (out) cudaMemcpyFromSymbol(out, adattn_b200::tc::g_trace, sizeof(unsigned long long) * n);
  if (reset) cudaMemset(adattn_b200::tc::g_trace_ptr(), 0, sizeof(unsigned long long) * n);
  return n;
}
#endif
#ifdef ADATTN_PIPE_STATS
extern "C" void adattn_b200_pipe_stats(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, adattn_b200::tc::g_pipe_stats, sizeof(unsigned long long) * 64);
  if (reset) {
    unsigned long long z[64] = {};
    cudaMemcpyToSymbol(adattn_b200::tc::g_pipe_stats, z, sizeof z);
  }
}
#endif
