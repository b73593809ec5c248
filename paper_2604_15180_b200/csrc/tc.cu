// tc.cu -- dispatch for the bf16 tensor-core path and its TMA descriptor helper.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "tc.cuh"
#include "tc_common.cuh"
#include "tc_host.cuh"

namespace adattn_b200 {
namespace tc {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

cudaError_t make_tmap_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                         uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// [rows x cols] bf16 row-major viewed as (64 cols, rows, cols/64 chunks): one
// box of `box_rows` rows carries every 64-column chunk, landing in shared memory
// chunk-major ([chunk][row][64 cols], SWIZZLE_128B) -- the layout of
// cols/64 separate 2-D boxes, in one TMA instruction.
cudaError_t make_tmap_3d_chunks(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                                uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[3] = {64, rows, cols / 64};
  cuuint64_t strides[2] = {cols * 2, 128};
  cuuint32_t box[3] = {64, box_rows, (cuuint32_t)(cols / 64)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

namespace {
__global__ void nsmid_probe(int* out) {
  uint32_t v;
  asm volatile("mov.u32 %0, %%nsmid;" : "=r"(v));
  *out = (int)v;
}
}  // namespace

// Number of %smid values of the current device (one list slot per resident CTA).
static int nsmid_slots() {
  static int cache[64];
  static std::once_flag once[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
  std::call_once(once[dev], [dev] {
    int* d = nullptr;
    int h = 0;
    if (cudaMalloc(&d, sizeof(int)) == cudaSuccess) {
      nsmid_probe<<<1, 1>>>(d);
      if (cudaMemcpy(&h, d, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) h = 0;
      cudaFree(d);
    }
    cudaGetLastError();
    cache[dev] = h;
  });
  return cache[dev];
}

// Lists pay off when few scores fall in the refinement window; alpha < 1.4
// (e.g. 1.25: thousands of candidates per row at N=32K) keeps the sweeps.
// ADATTN_CAND_CAP overrides the per-thread capacity (0 disables the lists).
CandPlan cand_plan(const Geom& g) {
  CandPlan p{0, 0};
  int cap = 512;
  if (const char* s = std::getenv("ADATTN_CAND_CAP")) cap = std::atoi(s);
  const char* force = std::getenv("ADATTN_CAND_FORCE");  // experiment: lists for any alpha
  if (cap < 64 || (g.alpha < 1.4 && !(force && *force == '1'))) return p;
  cap = (cap + 63) / 64 * 64;
  p.slots = nsmid_slots();
  if (p.slots <= 0) return p;
  p.cap = cap;
  return p;
}

// O = P V with fp16 P (in [0, 1]) and an fp16 copy of V (ADATTN_PV_F16=0: bf16 P)
bool pv_f16_enabled() {
  const char* s = std::getenv("ADATTN_PV_F16");
  return !(s && *s == '0');
}

// blocks [h * bpp, (h + 1) * bpp) cover head h's n8 groups of 8 bf16 (16-byte
// loads: 4-byte accesses left these HBM-bound passes at ~1.2 TB/s)
__global__ void absmax_bf16_kernel(const uint4* __restrict__ src, size_t n8, int bpp,
                                   uint32_t* maxbits, const uint32_t* need) {
  const int h = blockIdx.x / bpp, b = blockIdx.x - h * bpp;
  if (need && need[h] == 0u) {  // no tensor-core kernel reads this head: no copy (a
    if (b == 0 && threadIdx.x == 0) maxbits[h] = 0xFFFFFFFFu;  // non-finite: bf16 plan)
    return;
  }
  src += (size_t)h * n8;
  uint32_t m = 0;
  for (size_t i = b * (size_t)blockDim.x + threadIdx.x; i < n8; i += (size_t)bpp * blockDim.x) {
    const uint4 u = __ldg(src + i);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)  // |bf16| as float bits: (w << 16) & 0x7FFF0000 per half
      m = max(m, max((w[j] << 16) & 0x7FFF0000u, w[j] & 0x7FFF0000u));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(maxbits + h, m);
}

__global__ void f16_scaled_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                  size_t n8, int bpp, const uint32_t* maxbits) {
  const int h = blockIdx.x / bpp, b = blockIdx.x - h * bpp;
  const uint32_t mb = maxbits[h];
  if (!f16_copy_ok(mb)) return;  // the kernels keep the head's bf16 operand
  const float s = f16_pow2_scale(mb);
  src += (size_t)h * n8;
  dst += (size_t)h * n8;
  for (size_t i = b * (size_t)blockDim.x + threadIdx.x; i < n8; i += (size_t)bpp * blockDim.x) {
    const uint4 u = __ldg(src + i);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float lo = __uint_as_float(w[j] << 16), hi = __uint_as_float(w[j] & 0xFFFF0000u);
      const __half2 hv = __floats2half2_rn(lo * s, hi * s);
      o[j] = *reinterpret_cast<const uint32_t*>(&hv);
    }
    dst[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

static int blocks_per_head(int heads) { return std::max(2, std::min(128, 8 * 148 / heads)); }

cudaError_t f16_absmax(const void* src, int heads, size_t elems, uint32_t* maxbits,
                       cudaStream_t st, const uint32_t* need) {
  const int bpp = blocks_per_head(heads);
  absmax_bf16_kernel<<<heads * bpp, 256, 0, st>>>(reinterpret_cast<const uint4*>(src),
                                                  elems / 8, bpp, maxbits, need);
  note_launch();
  return cudaGetLastError();
}

cudaError_t f16_convert_scaled(const void* src, void* dst, int heads, size_t elems,
                               const uint32_t* maxbits, cudaStream_t st) {
  const int bpp = blocks_per_head(heads);
  f16_scaled_kernel<<<heads * bpp, 256, 0, st>>>(reinterpret_cast<const uint4*>(src),
                                                 reinterpret_cast<uint4*>(dst), elems / 8, bpp,
                                                 maxbits);
  note_launch();
  return cudaGetLastError();
}

// candidate lists, then (fp16 P V) the fp16 copy of V and its range maximum
// delta from the support lists: list mode only (every score with t > 0
// at the final tau is in the candidate lists), and not when the forward folds delta
bool delta_supp_possible(const Geom& g) {
  const char* s = std::getenv("ADATTN_DELTA_SUPP");
  if (s && *s == '0') return false;
  return cand_plan(g).cap > 0 && (g.dv == 64 || g.dv == 128);
}
bool delta_supp_enabled(const Geom& g) {
  if (!delta_supp_possible(g)) return false;
  Geom gf = g;
  float dummy = 0.f;
  gf.ubar_out = &dummy;
  return !fwd_delta_fold(gf);
}
static int supp_cap_of() {
  // support entries per row, pooled per 256-row block (C3 gaussian: ~30 per row, C5 ~40; a
  // block whose rows need more than 256 * cap in total falls back to the tensor cores)
  int cap = 64;
  if (const char* s = std::getenv("ADATTN_SUPP_CAP")) cap = std::max(1, std::atoi(s));
  return cap;
}
// layout (tc_host.cuh SuppLayout), 256-byte aligned sections
static size_t supp_sections(const Geom& g, size_t off[10]) {
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t rows = (size_t)g.bh * g.n, nblk = (rows + 255) / 256;
  const size_t ent = nblk * 256 * (size_t)supp_cap_of();
  const size_t sz[10] = {nblk * 4, (size_t)g.bh * 4, rows * 2 * 8, ent * 8,
                        (size_t)g.bh * g.m * 4, (size_t)g.bh * (g.m + 1) * 4,
                        (size_t)g.bh * g.m * 4, ent * 4, ent * 8, ((size_t)g.bh * g.m + 1) * 4};
  size_t o = 0;
  for (int i = 0; i < 10; ++i) {
    off[i] = o;
    o += al(sz[i]);
  }
  return o;
}
size_t supp_bytes(const Geom& g) {
  if (!delta_supp_enabled(g)) return 0;
  size_t off[10];
  return supp_sections(g, off);
}
SuppLayout supp_layout(const Geom& g, void* base) {
  size_t off[10];
  supp_sections(g, off);
  uint8_t* p = reinterpret_cast<uint8_t*>(base);
  SuppLayout l;
  l.flag = reinterpret_cast<uint32_t*>(p + off[0]);
  l.hflag = reinterpret_cast<uint32_t*>(p + off[1]);
  l.cnt = reinterpret_cast<int2*>(p + off[2]);
  l.ent = reinterpret_cast<uint2*>(p + off[3]);
  l.kcnt = reinterpret_cast<int32_t*>(p + off[4]);
  l.koff = reinterpret_cast<int32_t*>(p + off[5]);
  l.kcur = reinterpret_cast<int32_t*>(p + off[6]);
  l.krow = reinterpret_cast<int32_t*>(p + off[7]);
  l.kpd = reinterpret_cast<float2*>(p + off[8]);
  l.klong = reinterpret_cast<int32_t*>(p + off[9]);
  l.cap = supp_cap_of();
  l.nblk = ((size_t)g.bh * g.n + 255) / 256;
  return l;
}

size_t forward_cand_bytes(const Geom& g) {
  const CandPlan p = cand_plan(g);
  return p.cap > 0 ? ((size_t)p.slots * 512 * (size_t)p.cap * 8 + 4096 + 255) / 256 * 256 : 0;
}
// then per resident CTA slot and epilogue warp the warp's tile maxima (activity sets)
size_t forward_wtm_offset(const Geom& g) {
  return forward_cand_bytes(g) +
         (pv_f16_enabled() ? ((size_t)g.bh * g.m * g.dv * 2 + 255) / 256 * 256 +
                                 ((size_t)g.bh * 4 + 255) / 256 * 256 : 0);
}
int forward_wtm_slots() { return std::max(0, nsmid_slots()); }
size_t forward_workspace(const Geom& g) {
  return forward_wtm_offset(g) +
         ((size_t)forward_wtm_slots() * 16 * (size_t)(g.m / 128) * 4 + 255) / 256 * 256;
}

}  // namespace tc

// Envelope of the tensor-core path: bf16 inputs, 64x64 reference
// tiles, d, dv <= 128, a positive scale (the kernels rank raw scores), bins <= 32.
// The kernels run d = dv in {64, 128} with n % 256 == 0, m % 128 == 0; other
// sizes run on zero-padded copies (capi.cu tc_ragged).
bool tc_supported(const Geom& g) {
  return g.in_dtype == ADATTN_BF16 && g.block_r == 64 && g.block_c == 64 && g.d <= 128 &&
         g.dv <= 128 && g.scale > 0.0 && g.bins <= 32 && g.bins >= 2;
}
std::string tc_envelope() {
  return "bf16 inputs, block_r=block_c=64, d, dv <= 128, scale>0, 2<=bins<=32";
}
size_t tc_forward_workspace(const Geom& g) { return tc::forward_workspace(g); }
size_t tc_backward_workspace(const Geom& g) { return tc::backward_workspace(g); }
bool tc_delta_fold(const Geom& g) { return tc::fwd_delta_fold(g); }
size_t tc_delta_supp_bytes(const Geom& g) { return tc::supp_bytes(g); }

cudaError_t tc_forward(const Geom& g, const void* q, const void* k, const void* v, void* out,
                       double* tau, double* row_max, uint32_t* mask, int32_t* steps, void* ws,
                       cudaStream_t st) {
  return tc::forward(g, q, k, v, out, tau, row_max, mask, steps, ws, st);
}
cudaError_t tc_delta(const Geom& g, const void* q, const void* k, const void* v,
                     const double* tau, const double* row_max, const uint32_t* mask,
                     const void* dout, double* delta, void* ws, cudaStream_t st) {
  return tc::backward(g, q, k, v, tau, row_max, mask, dout, nullptr, nullptr, nullptr, delta, ws,
                      true, st);
}
cudaError_t tc_backward(const Geom& g, const void* q, const void* k, const void* v,
                        const double* tau, const double* row_max, const uint32_t* mask,
                        const void* dout, void* dq, void* dk, void* dv, double* delta, void* ws,
                        cudaStream_t st) {
  return tc::backward(g, q, k, v, tau, row_max, mask, dout, dq, dk, dv, delta, ws, false, st);
}

}  // namespace adattn_b200
