// Microbenchmark: per-SM throughput of the instructions in the attention
// softmax inner loop (ex2 variants, f32 -> 16-bit packs), to find which
// issue pipe binds.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

constexpr int kIters = 4096;

__device__ __forceinline__ float ex2f(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t ex2bf2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t cvtbf2(float a, float b) { uint32_t y; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(a), "f"(b)); return y; }
__device__ __forceinline__ uint32_t cvth2(float a, float b) { uint32_t y; asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(a), "f"(b)); return y; }

template <int kOp>
__global__ void bench(float* out, float seed) {
  float a[8];
  uint32_t u[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = seed * (threadIdx.x + i) * 1e-6f; u[i] = __float_as_uint(a[i]) ^ i; }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (kOp == 0) a[i] = ex2f(a[i]);
      if (kOp == 1) u[i] = ex2h2(u[i]);
      if (kOp == 2) u[i] = ex2bf2(u[i]);
      if (kOp == 3) u[i] = cvtbf2(a[i], __uint_as_float(u[i]));
      if (kOp == 4) u[i] = cvth2(a[i], __uint_as_float(u[i]));
      if (kOp == 5) { a[i] = fmaxf(a[i], __uint_as_float(u[i])); }
      if (kOp == 6) { a[i] = fmaf(a[i], 1.0001f, -0.5f); }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(u[i]);
  if (s == 1.2345f) out[threadIdx.x] = s;
}

template <int kOp>
void run(const char* name, int blocks, int threads) {
  float* out; cudaMalloc(&out, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  bench<kOp><<<blocks, threads>>>(out, 1.f);
  cudaEventRecord(e0);
  bench<kOp><<<blocks, threads>>>(out, 1.f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = double(blocks) * threads * kIters * 8;
  int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("%-22s %8.3f ms  %8.2f Gop/s  %6.2f lane-ops/clk/SM (at %d MHz)\n", name, ms, ops / ms * 1e-6,
         ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  cudaFree(out);
}

int main() {
  int blocks = 148 * 4, threads = 512;
  run<0>("ex2.approx.f32", blocks, threads);
  run<1>("ex2.approx.f16x2", blocks, threads);
  run<2>("ex2.approx.bf16x2", blocks, threads);
  run<3>("cvt.rn.bf16x2.f32", blocks, threads);
  run<4>("cvt.rn.f16x2.f32", blocks, threads);
  run<5>("fmax", blocks, threads);
  run<6>("ffma", blocks, threads);
  return 0;
}
