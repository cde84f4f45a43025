// ubench_issue.cu -- issue cost of tcgen05.mma: one thread (`if (lane == 0)`,
// ptxas wraps every UTCHMMA in an ELECT loop over the active threads) versus
// the whole warp executing the issue loop with the MMA predicated on
// elect.sync inside the same asm block.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../paper_2604_27441_b200/csrc ubench_issue.cu -o ubench_issue
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace nvrec::sm100;

constexpr int kIters = 4096;

__device__ __forceinline__ void mma_ss_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                             uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc,
                                             uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

// mode 0: N-wide SS MMAs, lane 0 issues; mode 1: same, whole warp + elect.sync
// mode 2: the x3w stream (6 S + 8 x (N64 + N32) PV per S tile), lane 0
// mode 3: the x3w stream, whole warp + elect.sync
template <int kMode, int kN>
__global__ void __launch_bounds__(128, 1) issue_bench(unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  uint8_t* base = dsm + ((1024 - (smem_u32(dsm) & 1023)) & 1023);
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tbase;
  const unsigned long long t0 = clock64();
  const uint32_t q0 = smem_u32(base), k0 = q0 + 16384, v0 = k0 + 16384;
  if (kMode <= 1 && threadIdx.x < 32 && (kMode == 1 || threadIdx.x == 0)) {
    const uint32_t idesc = idesc_bf16(128, kN);
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint64_t ad = sdesc(q0 + (c & 3) * 32, 1024, kSwizzle128B);
        const uint64_t bd = sdesc(k0 + (c & 3) * 32, 1024, kSwizzle128B);
        if (kMode == 0) mma_ss(t + 256, ad, bd, idesc, 1);
        else mma_ss_elect(t + 256, ad, bd, idesc, 1);
      }
    }
    if (kMode == 0) mma_commit(&bar);
    else commit_elect(&bar);
    mbar_wait(&bar, 0);
  }
  if (kMode >= 2 && threadIdx.x < 32 && (kMode == 3 || threadIdx.x == 0)) {
    constexpr uint32_t idS = idesc_bf16(128, 128), idP64 = idesc_bf16(128, 64),
                       idP32 = idesc_bf16(128, 32);
    constexpr int qa[6] = {0, 1, 0, 1, 2, 3}, kc[6] = {0, 1, 2, 3, 0, 1};
    for (int n = 0; n < kIters; ++n) {
      const uint32_t sc = t + (n % 3) * 128;
      const uint32_t qb = q0 + (n & 1) * 8192;
#pragma unroll
      for (int u = 0; u < 6; ++u) {
        const uint64_t ad = sdesc(qb + qa[u] * 32, 1024, kSwizzle128B);
        const uint64_t bd = sdesc(k0 + kc[u] * 32, 1024, kSwizzle128B);
        if (kMode == 2) mma_ss(sc, ad, bd, idS, u);
        else mma_ss_elect(sc, ad, bd, idS, u);
      }
      if (n >= 2) {
        const int m = n - 2;
        const uint32_t bc = t + (m % 3) * 128, oc = t + 384 + 64 * (m & 1);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t ah = bc + (kk >> 2) * 64 + (kk & 3) * 8;
          const uint64_t vd = sdesc(v0 + (kk >> 2) * 8192 + (kk & 3) * 32, 1024, kSwizzle128B);
          if (kMode == 2) {
            mma_ts(oc, ah, vd, idP64, kk);
            mma_ts(oc, ah + 32, vd, idP32, 1);
          } else {
            mma_ts_elect(oc, ah, vd, idP64, kk);
            mma_ts_elect(oc, ah + 32, vd, idP32, 1);
          }
        }
      }
    }
    if (kMode == 2) mma_commit(&bar);
    else commit_elect(&bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(t);
}

template <int kMode, int kN>
void run(const char* name) {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  const int smem = 64 * 1024 + 1024;
  cudaFuncSetAttribute(issue_bench<kMode, kN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  issue_bench<kMode, kN><<<148, 128, smem>>>(cyc);
  cudaDeviceSynchronize();
  issue_bench<kMode, kN><<<148, 128, smem>>>(cyc);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < 148; ++i) mean += double(h[i]) / 148;
  const double per = kMode <= 1 ? mean / (kIters * 8.0) : mean / kIters;
  printf("%-44s N=%3d  %7.1f clk/%s (%s)\n", name, kN, per, kMode <= 1 ? "MMA" : "S tile",
         cudaGetErrorString(e));
  cudaFree(cyc);
}

int main() {
  run<0, 32>("SS MMAs, lane 0 issues");
  run<1, 32>("SS MMAs, warp + elect.sync");
  run<0, 64>("SS MMAs, lane 0 issues");
  run<1, 64>("SS MMAs, warp + elect.sync");
  run<0, 128>("SS MMAs, lane 0 issues");
  run<1, 128>("SS MMAs, warp + elect.sync");
  run<2, 128>("x3w stream (per-MMA descriptors), lane 0");
  run<3, 128>("x3w stream (per-MMA descriptors), warp+elect");
  return 0;
}
