// tma_bench.cu -- TMA tile-load throughput per SM from L2 (dev tool, not product).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2604_15180_b200/csrc
//        -I../include tools/tma_bench.cu -o tma_bench -lcuda
// One producer warp streams [rows x 64 cols] bf16 boxes (SWIZZLE_128B) through an
// NST-stage ring; one consumer warp releases each stage as soon as it lands.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>

#include "tc_common.cuh"

using namespace adattn_b200::tc;

template <int NST, int BOXR>
__global__ void __launch_bounds__(64, 1) tma_bench(const __grid_constant__ CUtensorMap tm,
                                                 unsigned long long* out, int iters, int rows_total) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[NST], empty[NST];
  constexpr int BYTES = BOXR * 128;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const long long t0 = clock64();
  if (warp == 0) {
    const bool leader = elect_one_sync();
    for (int r = 0; r < iters; ++r) {
      const int st = r % NST;
      mbar_wait(&empty[st], ((r / NST) & 1) ^ 1);
      if (leader) mbar_expect_tx(&full[st], BYTES);
      const int row = ((blockIdx.x * 7919 + r * BOXR) % (rows_total - BOXR));
      if (leader) tma_load_2d(smem + st * BYTES, &tm, &full[st], 0, row);
    }
  } else {
    for (int r = 0; r < iters; ++r) {
      const int st = r % NST;
      mbar_wait(&full[st], (r / NST) & 1);
      if (elect_one_sync()) mbar_arrive(&empty[st]);
    }
    const long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
}

template <int NST, int BOXR>
void run(PFN_cuTensorMapEncodeTiled_v12000 enc, void* base, int rows, const char* name, int nblk = 148) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {64, (cuuint64_t)rows};
  cuuint64_t strides[1] = {64 * 2};
  cuuint32_t box[2] = {64, BOXR};
  cuuint32_t es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int iters = 2000;
  auto k = tma_bench<NST, BOXR>;
  const int sm = NST * BOXR * 128;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  k<<<nblk, 64, sm>>>(tm, d, iters, rows);
  k<<<nblk, 64, sm>>>(tm, d, iters, rows);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < nblk; ++i) avg += (double)h[i] / nblk;
  printf("%-28s %s  %.1f B/cycle/SM  (%.0f cycles per %d B box)\n", name,
         e ? cudaGetErrorString(e) : "ok", (double)iters * BOXR * 128 / avg, avg / iters, BOXR * 128);
  cudaFree(d);
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  const int rows = 1 << 19;  // 512K rows x 128 B = 64 MB (L2-resident)
  void* base;
  cudaMalloc(&base, (size_t)rows * 128);
  cudaMemset(base, 0, (size_t)rows * 128);
  run<4, 128>(enc, base, rows, "box 128x64 (16 KB), 4 stages");
  run<8, 128>(enc, base, rows, "box 128x64 (16 KB), 8 stages");
  run<8, 128>(enc, base, rows, "16 KB boxes, 8 st, 16 CTAs", 16);
  run<4, 256>(enc, base, rows, "box 256x64 (32 KB), 4 stages");
  run<4, 64>(enc, base, rows, "box 64x64 (8 KB), 4 stages");
  run<16, 64>(enc, base, rows, "box 64x64 (8 KB), 16 stages");
  return 0;
}
