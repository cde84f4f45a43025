// Microbenchmark: TMEM bandwidth per SM on B200 (sm_100a).
//   mode 0: tcgen05.ld 32x32b.x32 by W warps (each warp its lane quarter)
//   mode 1: tcgen05.st 32x32b.x32 by W warps
//   mode 2: tcgen05.mma kind::f16 M128 N32 K16 with A from TMEM (PV shape),
//           one thread issuing back to back (A read: 128 lanes x 8 cols x 4 B)
//   mode 3: same MMA shape with A from shared memory (SS)
// One CTA per SM, all 148 SMs; clock64 deltas per CTA.  Prints bytes/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2604_27441_b200/csrc
//        ubench_tmem.cu -o ubench_tmem -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace nvrec::sm100;

constexpr int kIters = 2048;

template <int kMode, int kN = 32, int kAcc = 1>
__global__ void __launch_bounds__(512, 1) tmem_bench(unsigned long long* cyc, uint32_t* sink,
                                                     int warps) {
  __shared__ uint32_t tbase;
  __shared__ __align__(1024) uint8_t a_smem[128 * 16 * 2];
  __shared__ __align__(1024) uint8_t b_smem[256 * 16 * 2];
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < int(sizeof(a_smem)); i += blockDim.x) a_smem[i] = 0;
  for (int i = threadIdx.x; i < int(sizeof(b_smem)); i += blockDim.x) b_smem[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tbase;
  uint32_t acc = 0;
  unsigned long long t0 = clock64();
  if (kMode == 0 || kMode == 1) {
    if (warp < warps) {
      const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
      const uint32_t col0 = (warp >> 2) * 128;
      uint32_t r[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = i;
      for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (kMode == 0) tmem_ld32(t + lane_off + ((col0 + 32 * c) & 511), r);
          else tmem_st32(t + lane_off + ((col0 + 32 * c) & 511), r);
        }
        if (kMode == 0) {
          tmem_wait_ld();
          acc ^= r[it & 31];
        } else {
          tmem_wait_st();
        }
      }
    }
  } else {
    if (threadIdx.x == 0) {
      const uint32_t idesc = idesc_bf16(128, kN);
      const uint64_t bd = sdesc(smem_u32(b_smem), 128, kSwizzleNone, 256);
      const uint64_t ad = sdesc(smem_u32(a_smem), 128, kSwizzleNone, 2048);
      for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          // kAcc independent accumulators of kN columns (cols 256.. / 0.. for N=256)
          const uint32_t d = kN >= 256 ? t + (c % kAcc) * 256 : t + 256 + (c % kAcc) * kN;
          if (kMode == 2) mma_ts(d, t + 8 * (c % 4), bd, idesc, 1);
          else mma_ss(d, ad, bd, idesc, 1);
        }
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 0xdeadbeef) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(t);
}

template <int kMode, int kN = 32, int kAcc = 1>
void run(const char* name, int warps, double bytes_per_cta) {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 4);
  tmem_bench<kMode, kN, kAcc><<<148, 512>>>(cyc, sink, warps);
  cudaDeviceSynchronize();
  tmem_bench<kMode, kN, kAcc><<<148, 512>>>(cyc, sink, warps);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < 148; ++i) mean += double(h[i]) / 148;
  printf("%-34s N=%3d acc=%d warps=%2d  %8.1f bytes/clk/SM  (%.0f clk, %.1f clk/MMA, %s)\n", name,
         kN, kAcc, warps, bytes_per_cta / mean, mean, mean / (kIters * 8.0), cudaGetErrorString(e));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  for (int w : {1, 2, 4, 8, 16}) {
    const double bytes = double(w) * kIters * 4 * 32 * 32 * 4;   // warps x iters x 4 x (32 lanes x 32 cols x 4 B)
    run<0>("tcgen05.ld 32x32b.x32", w, bytes);
  }
  for (int w : {4, 8, 16}) {
    const double bytes = double(w) * kIters * 4 * 32 * 32 * 4;
    run<1>("tcgen05.st 32x32b.x32", w, bytes);
  }
  // A operand bytes read per MMA: 128 rows x 16 bf16 = 4 KB
  const double ab = double(kIters) * 8 * 4096;
  run<2, 32, 1>("mma A=TMEM", 1, ab);
  run<2, 32, 2>("mma A=TMEM", 1, ab);
  run<2, 32, 4>("mma A=TMEM", 1, ab);
  run<3, 32, 1>("mma A=SMEM", 1, ab);
  run<3, 32, 4>("mma A=SMEM", 1, ab);
  run<3, 64, 1>("mma A=SMEM", 1, ab);
  run<3, 64, 2>("mma A=SMEM", 1, ab);
  run<3, 128, 1>("mma A=SMEM", 1, ab);
  run<3, 128, 2>("mma A=SMEM", 1, ab);
  run<3, 256, 1>("mma A=SMEM", 1, ab);
  run<3, 256, 2>("mma A=SMEM", 1, ab);
  run<2, 64, 1>("mma A=TMEM", 1, ab);
  run<2, 128, 1>("mma A=TMEM", 1, ab);
  return 0;
}
