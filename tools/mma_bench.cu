// mma_bench.cu -- microbenchmark of tcgen05.mma issue throughput per SM for the
// operand sources / shapes the attention kernels use (dev tool, not product).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2604_15180_b200/csrc
//        -I../include tools/mma_bench.cu -o mma_bench -lcuda
#include <cstdio>
#include <cstdlib>

#include "tc_common.cuh"

using namespace adattn_b200::tc;

// MODE bit0: commit to a side barrier every 8 MMAs; bit1: tcgen05 fence::after
// every 8; bit2: mbarrier try_wait on an already-complete barrier every 8;
// bit5: the bit2 wait uses mbarrier.test_wait (non-blocking spin) instead of try_wait;
// bit6: warps 2-3 stream st.shared.v4 writes into a separate 32 KB region while
// the MMAs run (the TMA tile arrivals' share of shared-memory bandwidth);
// bit7 (with bit6): the side warps stream tcgen05.ld of 32 columns instead of smem writes
// bit3: B operand MN-major (SW128, 64-element MN chunks 16 KB apart); bit4:
// alternate two accumulators every 2 MMAs (hi/lo pairs into dV then dK)
template <int N, bool TS, int NMMA, int MODE = 0>
__global__ void __launch_bounds__(256, 1) bench(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, side, done;
  __shared__ uint32_t tbase;
  __shared__ volatile uint32_t stop;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += 256) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&side, 1);
    mbar_init(&done, 1);
    mbar_arrive(&done);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) stop = 0;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == 1) {
    const bool leader = elect_one_sync();
    const uint32_t a_addr = smem_u32(smem), b_addr = smem_u32(smem + 32768);
    constexpr bool BMN = (MODE & 8) != 0;
    constexpr uint32_t IDESC = idesc_bf16_f32(128, N, false, BMN);
    const long long t0 = clock64();
    for (int i = 0; i < NMMA; ++i) {
      const int k = i & 3;
      if ((i & 7) == 0 && i) {
        if (MODE & 1)
          if (leader) umma_commit(&side);
        if (MODE & 4) {
          if (MODE & 32) {
            uint32_t ok = 0;
            while (!ok)
              asm volatile(
                  "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                  "selp.u32 %0, 1, 0, p;\n\t}"
                  : "=r"(ok)
                  : "r"(smem_u32(&done)), "r"(0u)
                  : "memory");
          } else {
            mbar_wait(&done, 0);
          }
        }
        if (MODE & 2) tc_fence_after();
        if (MODE & 1024) {  // issuing warp stalls ~256 cycles every 8 MMAs
          const long long w0 = clock64();
          while (clock64() - w0 < 256) {
          }
        }
      }
      const uint64_t bdesc = BMN ? desc_mnmajor(b_addr + k * 2048, 16384)
                                 : desc_kmajor(b_addr + k * 32);
      const uint32_t dt = (MODE & 16) ? tmem + 256 + ((i >> 1) & 1) * 128 : tmem + 256;
      if (leader) {
        if constexpr (TS) {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dt),
              "r"(tmem + 8 * k), "l"(bdesc), "r"(IDESC), "r"(1u));
        } else {
          umma_bf16(dt, desc_kmajor(a_addr + k * 32), bdesc, IDESC, 1u);
        }
      }
    }
    if (leader) umma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (leader) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    stop = 1;
  } else if ((MODE & 64) && warp >= 2 && (warp < 4 || (MODE & 512))) {
    unsigned long long nbytes = 0;
    if (MODE & 128) {  // warps 2,3 read TMEM lanes 64-127, columns 0..127 (not the accumulator)
      float acc = 0.f;
      while (!stop) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          float v[32];
          tmem_ld32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + ((MODE & 256) ? 256 + r * 32 : r * 32), v);
          tmem_wait_ld();
          acc += v[0] + v[31];
        }
        nbytes += 4 * 32 * 32 * 4 * ((MODE & 512) ? 6 : 2);  // side warps
      }
      if (acc == 12345.f) out[0] = 0;
    } else {
      const uint32_t base = smem_u32(smem + 65536) + (threadIdx.x - 64) * 16;
      while (!stop) {
#pragma unroll
        for (int r = 0; r < 8; ++r) st_shared_v4(base + r * 1024 % 32768, r, r, r, r);
        nbytes += 8 * 16 * 64;
      }
    }
    if (threadIdx.x == 64) out[148 + blockIdx.x] = nbytes;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int N, bool TS, int MODE = 0>
void run(const char* name) {
  constexpr int NMMA = 4096;
  unsigned long long* d;
  cudaMalloc(&d, 2 * 148 * 8);
  cudaMemset(d, 0, 2 * 148 * 8);
  auto k = bench<N, TS, NMMA, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<148, 256, 100 * 1024>>>(d);
  k<<<148, 256, 100 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2 * 148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += (double)h[i] / 148.0;
  const double cyc = avg / NMMA;
  const double macs = 128.0 * N * 16;
  printf("%-18s %s  cycles/MMA %7.1f  MAC/cycle/SM %7.0f  (%.0f%% of 4096)  side-writes %.1f B/cycle\n", name,
         e ? cudaGetErrorString(e) : "ok", cyc, macs / cyc, 100.0 * macs / cyc / 4096.0,
         (double)h[148] / avg);
  cudaFree(d);
}


// The dK/dV kernel's per-unit MMA sequence, no epilogue or TMA: per unit 8 x
// (SS M128 N64 S^T, SS M128 N64 dP^T) interleaved, then 16 TS M128 N128
// (dV hi/lo, dK hi/lo).  MODE bit0: commit after the S/dP block and after the
// grads (the kernel's commits).
template <int MODE>
__global__ void __launch_bounds__(384, 1) bench_kv(unsigned long long* out, int units) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, side, side2;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  __shared__ volatile uint32_t stop;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += 384) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&side, 1);
    mbar_init(&side2, 1);
    mbar_arrive(&side2);
    fence_barrier_init();
    stop = 0;
  }
  if (warp == 0) tmem_alloc(&tbase, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == 1) {
    const bool leader = elect_one_sync();
    const uint32_t k_addr = smem_u32(smem), v_addr = smem_u32(smem + 32768),
                   q_addr = smem_u32(smem + 65536), do_addr = smem_u32(smem + 65536 + 16384);
    constexpr uint32_t IS = idesc_bf16_f32(128, 64, false, false);
    constexpr uint32_t IG = idesc_bf16_f32(128, 128, false, true);
    const long long t0 = clock64();
    for (int u = 0; u < units; ++u) {
      const uint32_t b = u & 1;
      for (int c = 0; c < 2; ++c)
        for (int k = 0; k < 4; ++k) {
          if (leader) umma_bf16(tmem + b * 128, desc_kmajor(k_addr + c * 16384 + k * 32),
                                desc_kmajor(q_addr + c * 8192 + k * 32), IS, (c | k) != 0);
          if (leader) umma_bf16(tmem + b * 128 + 64, desc_kmajor(v_addr + c * 16384 + k * 32),
                                desc_kmajor(do_addr + c * 8192 + k * 32), IS, (c | k) != 0);
        }
      if (MODE & 1) if (leader) umma_commit(&side);
      if (MODE & 32) {  // a satisfied mbarrier wait + tcgen05 fence between the groups
        mbar_wait(&side2, 0);
        tc_fence_after();
      }
      if (MODE & 8) {  // the issuing warp stalls ~200 cycles between the groups
        const long long w0 = clock64();
        while (clock64() - w0 < 200) {
        }
      }
      for (int k = 0; k < 4; ++k) {
        const uint32_t acol = 32 * (k >> 1) + 8 * (k & 1);
        const uint64_t bdo = desc_mnmajor(do_addr + k * 2048, 8192);
        const uint64_t bq = desc_mnmajor(q_addr + k * 2048, 8192);
        if (leader) umma_bf16_ts(tmem + 256, tmem + (b ^ 1) * 128 + acol, bdo, IG, 1u);
        if (leader) umma_bf16_ts(tmem + 256, tmem + (b ^ 1) * 128 + acol + 16, bdo, IG, 1u);
        if (leader) umma_bf16_ts(tmem + 384, tmem + (b ^ 1) * 128 + 64 + acol, bq, IG, 1u);
        if (leader) umma_bf16_ts(tmem + 384, tmem + (b ^ 1) * 128 + 64 + acol + 16, bq, IG, 1u);
      }
      if (MODE & 1) if (leader) umma_commit(&side);
      if (MODE & 32) {
        mbar_wait(&side2, 0);
        tc_fence_after();
      }
      if (MODE & 16) {  // and ~400 cycles after the grads
        const long long w0 = clock64();
        while (clock64() - w0 < 400) {
        }
      }
    }
    if (leader) umma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (leader) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    stop = 1;
  } else if (warp >= 4 && (MODE & 2)) {
    // epilogue-like TMEM traffic: 8 warps, per round ld 2 x 32 cols, st 4 x 16 cols
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16) + ((warp >> 2) & 1) * 32;
    uint32_t r[16];
    float v[32];
    float acc = 0.f;
    while (!stop) {
      tmem_ld32(tl, v);
      tmem_ld32(tl + 64, v);
      tmem_wait_ld();
      for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(v[i] + v[i + 16]);
      acc += v[3];
      tmem_st16(tl, r);
      tmem_st16(tl + 16, r);
      tmem_st16(tl + 64, r);
      tmem_st16(tl + 80, r);
      tmem_wait_st();
      if (MODE & 4)
        for (int i = 0; i < 8; ++i)
          st_shared_v4(smem_u32(smem) + 98304 + ((threadIdx.x * 16 + i * 4096) & 4095), i, i, i, i);
    }
    if (acc == 1234.f) out[0] = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int MODE>
void run_kv(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  auto k = bench_kv<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int units = 512;
  k<<<148, 384, 100 * 1024>>>(d, units);
  k<<<148, 384, 100 * 1024>>>(d, units);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += (double)h[i] / 148.0;
  printf("%-22s %s  cycles/unit %7.1f  (ideal 1792 at 67%% SS N64 + 100%% TS)\n", name,
         e ? cudaGetErrorString(e) : "ok", avg / units);
  cudaFree(d);
}

int main() {
  run<64, false>("SS M128 N64");
  run<128, false>("SS M128 N128");
  run<256, false>("SS M128 N256");
  run<64, true>("TS M128 N64");
  run<128, true>("TS M128 N128");
  run<256, true>("TS M128 N256");
  run<64, false, 1>("SS N64 +commit/8");
  run<64, false, 2>("SS N64 +fence/8");
  run<64, false, 4>("SS N64 +wait/8");
  run<64, false, 7>("SS N64 +all/8");
  run<64, true, 7>("TS N64 +all/8");
  run<128, false, 8>("SS N128 Bmn");
  run<128, true, 8>("TS N128 Bmn");
  run<128, true, 24>("TS N128 Bmn alt2");
  run<64, false, 8>("SS N64 Bmn");
  run<128, false, 64>("SS N128 +smemwr");
  run<128, false, 192>("SS N128 +tmemld");
  run<128, true, 192>("TS N128 +tmemld");
  run<128, false, 192 + 512>("SS N128 +tmemld6w");
  run<128, false, 192 + 512 + 256>("SS N128 +tmemld6w-acc");
  run<128, true, 64>("TS N128 +smemwr");
  run<64, true, 64>("TS N64 +smemwr");
  run<128, false, 4>("SS N128 +wait/8");
  run<128, false, 1024>("SS N128 +256cyc gap/8");
  run<128, true, 1024>("TS N128 +256cyc gap/8");
  run<256, false, 1024>("SS N256 +256cyc gap/8");
  run<128, false, 36>("SS N128 +testwait/8");
  run<128, true, 4>("TS N128 +wait/8");
  run<128, true, 36>("TS N128 +testwait/8");
  run_kv<0>("dkdv MMA sequence");
  run_kv<1>("dkdv MMA seq +commits");
  run_kv<2>("dkdv MMA seq +tmem ld/st");
  run_kv<6>("dkdv MMA +tmem +smemwr");
  run_kv<8>("dkdv MMA +200cyc gap");
  run_kv<24>("dkdv MMA +200+400 gaps");
  run_kv<33>("dkdv MMA +wait+fence x2");
  run<64, true, 8>("TS N64 Bmn");
  return 0;
}
