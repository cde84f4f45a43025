// Microbenchmark: TMEM bandwidth per SM on B200 (sm_100a).
//   mode 0: tcgen05.ld 32x32b.x32 by W warps (each warp its lane quarter)
//   mode 1: tcgen05.st 32x32b.x32 by W warps
//   mode 2: tcgen05.mma kind::f16 M128 N32 K16 with A from TMEM (PV shape),
//           one thread issuing back to back (A read: 128 lanes x 8 cols x 4 B)
//   mode 3: same MMA shape with A from shared memory (SS)
//   mode 4: SS MMAs issued by one thread in each of `warps` warps (own
//           accumulators): is the ~44 clk/MMA floor at small N per issuer?
//   mode 6: the dense precise attention's MMA stream per S tile, no softmax:
//           S = 6 x (M128 N128 K16, SWIZZLE_128B Q/K) into buffer n % 3, then
//           PV = 8 x (N64 A=TMEM + N32 A=TMEM) into O; clk per S tile
//   mode 7: mode 6 while warps 4.. stream the softmax's TMEM traffic (two
//           tcgen05.ld x32 + four tcgen05.st x16 per 64 columns) over the S buffers
//   mode 8: mode 6 with the kernel's per-S-tile tcgen05.commit pattern (after
//           the S MMAs, after the PV MMAs, and a K/V-release commit)
//   mode 5: SS MMAs by warp 0 while warps 1..warps-1 stream tcgen05.ld over
//           TMEM columns 0-255 (the softmax's S reads): TMEM contention
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
  __shared__ __align__(1024) uint8_t q_smem[kMode >= 6 ? 32768 + 16384 - 8192 : 16];
  __shared__ uint64_t bar, bars[16];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < int(sizeof(a_smem)); i += blockDim.x) a_smem[i] = 0;
  for (int i = threadIdx.x; i < int(sizeof(b_smem)); i += blockDim.x) b_smem[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 16; ++i) mbar_init(&bars[i], 1);
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
  } else if (kMode == 4) {
    if ((threadIdx.x & 31) == 0 && warp < warps) {
      const uint32_t idesc = idesc_bf16(128, kN);
      const uint64_t bd = sdesc(smem_u32(b_smem), 128, kSwizzleNone, 256);
      const uint64_t ad = sdesc(smem_u32(a_smem), 128, kSwizzleNone, 2048);
      const uint32_t d = t + warp * kN;
      for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) mma_ss(d, ad, bd, idesc, 1);
      }
      mma_commit(&bars[warp]);
      mbar_wait(&bars[warp], 0);
    }
  } else if (kMode == 8) {
    if (threadIdx.x == 0) {
      const uint32_t qb = smem_u32(q_smem), kb = qb + 8192, vb = qb + 24576;
      constexpr uint32_t idS = idesc_bf16(128, 128), idP64 = idesc_bf16(128, 64),
                         idP32 = idesc_bf16(128, 32);
      constexpr int qa[6] = {0, 1, 0, 1, 2, 3}, kc[6] = {0, 1, 2, 3, 0, 1};
      for (int n = 0; n < kIters; ++n) {
        const uint32_t sc = t + (n % 3) * 128;
        if (warps & 8) tc_fence_after();
        if (warps & 16) mbar_wait_fast(&bars[15], 1);     // an already-completed phase
#pragma unroll
        for (int u = 0; u < 6; ++u)
          mma_ss(sc, sdesc(qb + qa[u] * 32, 1024, kSwizzle128B),
                 sdesc(kb + kc[u] * 32, 1024, kSwizzle128B), idS, u);
        if (warps & 1) mma_commit(&bars[n % 3]);
        if (warps & 8) tc_fence_after();
        if (warps & 16) mbar_wait_fast(&bars[15], 1);
        if (n >= 2) {
          const uint32_t bc = t + ((n - 2) % 3) * 128, oc = t + 384;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t ah = bc + (kk >> 2) * 64 + (kk & 3) * 8;
            const uint32_t vh = vb + (kk >> 2) * 8192 + (kk & 3) * 32;
            mma_ts(oc, ah, sdesc(vh, 1024, kSwizzle128B), idP64, kk);
            mma_ts(oc, ah + 32, sdesc(vh, 1024, kSwizzle128B), idP32, 1);
          }
          if (warps & 2) mma_commit(&bars[3 + (n & 1)]);
          if (warps & 4) mma_commit(&bars[5 + (n & 3)]);
        }
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
    }
  } else if (kMode == 6 || kMode == 7) {
    if (kMode == 7 && warp >= 4 && warp < 4 + warps) {
      const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
      uint32_t r[64];
      volatile uint32_t* flag = sink + 1;
      for (int it = 0; it < 64 * kIters && *flag == 0; ++it) {
        const uint32_t c0 = ((it + warp) % 6) * 64;
        tmem_ld32(t + lane_off + c0, r);
        tmem_ld32(t + lane_off + c0 + 32, r + 32);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] ^= r[i + 32];
        tmem_st16(t + lane_off + c0, r);
        tmem_st16(t + lane_off + c0 + 16, r + 16);
        tmem_st16(t + lane_off + c0 + 32, r);
        tmem_st16(t + lane_off + c0 + 48, r + 16);
        tmem_wait_st();
        acc ^= r[it & 31];
      }
    }
    if (threadIdx.x == 0) {
      const uint32_t qb = smem_u32(q_smem), kb = qb + 8192, vb = qb + 24576;   // overlapping: timing only
      constexpr uint32_t idS = idesc_bf16(128, 128), idP64 = idesc_bf16(128, 64),
                         idP32 = idesc_bf16(128, 32);
      constexpr int qa[6] = {0, 1, 0, 1, 2, 3}, kc[6] = {0, 1, 2, 3, 0, 1};
      for (int n = 0; n < kIters; ++n) {
        const uint32_t sc = t + (n % 3) * 128;
#pragma unroll
        for (int u = 0; u < 6; ++u)
          mma_ss(sc, sdesc(qb + qa[u] * 32, 1024, kSwizzle128B),
                 sdesc(kb + kc[u] * 32, 1024, kSwizzle128B), idS, u);
        if (n >= 2) {
          const uint32_t bc = t + ((n - 2) % 3) * 128, oc = t + 384;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t ah = bc + (kk >> 2) * 64 + (kk & 3) * 8;
            const uint32_t vh = vb + (kk >> 2) * 8192 + (kk & 3) * 32;
            mma_ts(oc, ah, sdesc(vh, 1024, kSwizzle128B), idP64, kk);
            mma_ts(oc, ah + 32, sdesc(vh, 1024, kSwizzle128B), idP32, 1);
          }
        }
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      sink[1] = 1;
    }
  } else if (kMode == 5) {
    if (threadIdx.x == 0) {
      const uint32_t idesc = idesc_bf16(128, kN);
      const uint64_t bd = sdesc(smem_u32(b_smem), 128, kSwizzleNone, 256);
      const uint64_t ad = sdesc(smem_u32(a_smem), 128, kSwizzleNone, 2048);
      for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) mma_ss(t + 256 + (c & 1) * 128, ad, bd, idesc, 1);
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      sink[1] = 1;
    } else if (warp >= 4 && warp < 4 + warps) {
      const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
      uint32_t r[32];
      volatile uint32_t* flag = sink + 1;
      for (int it = 0; it < 4 * kIters && *flag == 0; ++it) {
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(t + lane_off + ((64 * c + 32 * (warp >> 2)) & 255), r);
        tmem_wait_ld();
        acc ^= r[it & 31];
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
  cudaMalloc(&sink, 8);
  cudaMemset(sink, 0, 8);
  tmem_bench<kMode, kN, kAcc><<<148, 512>>>(cyc, sink, warps);
  cudaDeviceSynchronize();
  cudaMemset(sink, 0, 8);
  tmem_bench<kMode, kN, kAcc><<<148, 512>>>(cyc, sink, warps);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < 148; ++i) mean += double(h[i]) / 148;
  printf("%-34s N=%3d acc=%d warps=%2d  %8.1f bytes/clk/SM  (%.0f clk, %.1f clk/%s, %s)\n", name,
         kN, kAcc, warps, bytes_per_cta / mean, mean, mean / (kIters * (kMode >= 6 ? 1.0 : 8.0)),
         kMode >= 6 ? "S tile" : "MMA", cudaGetErrorString(e));
  cudaFree(cyc);
  cudaFree(sink);
}


// mode R: the dense precise attention's MMA stream with the kernel's operand
// addresses: Q of 2 query tiles (16 KB each), K/V in a 4-stage ring (16 KB +
// 16 KB per key tile, key tile j = n / 2), S buffers n % 3, O' per tile.  rot = 0
// reuses stage 0 every time (operands possibly cached), rot = 1 rotates.
__global__ void __launch_bounds__(512, 1) rot_bench(unsigned long long* cyc, int rot, int qtmem, int rnd, int fix) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  uint8_t* base = dsm + ((1024 - (smem_u32(dsm) & 1023)) & 1023);
  // operands: zeros, or (rnd) bf16 values in [-2, 2) from a hash, so that the
  // tensor datapath toggles as it does on real data
  const int nw = (fix & 16) ? 40 * 1024 / 4 : 160 * 1024 / 4;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) {
    uint32_t h = (uint32_t(i) + 0x9e3779b9u * (blockIdx.x + 1)) * 0x85ebca6bu;
    h ^= h >> 13; h *= 0xc2b2ae35u; h ^= h >> 16;
    const uint32_t v = rnd ? ((0x3f80u | (h & 0x807fu)) | ((0x3f80u | ((h >> 16) & 0x807fu)) << 16)) : 0u;
    reinterpret_cast<uint32_t*>(base)[i] = v;
  }
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
  if (rnd) {   // P/S columns: the same kind of bf16 pairs (each warp its lane quarter)
    const uint32_t lo = uint32_t((threadIdx.x >> 5) * 32) << 16;
    for (int c = 0; c < 512; c += 32) {
      uint32_t r[32];
      for (int e = 0; e < 32; ++e) {
        uint32_t h = (uint32_t(threadIdx.x * 512 + c + e) + 0x7f4a7c15u * (blockIdx.x + 1)) * 0x85ebca6bu;
        h ^= h >> 15;
        r[e] = (0x3f00u | (h & 0x807fu)) | ((0x3f00u | ((h >> 16) & 0x807fu)) << 16);
      }
      tmem_st32(t + lo + c, r);
    }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t q0 = smem_u32(base), k0 = q0 + 32768, v0 = k0 + 4 * 16384;
    constexpr uint32_t idS = idesc_bf16(128, 128), idP64 = idesc_bf16(128, 64),
                       idP32 = idesc_bf16(128, 32);
    constexpr int qa[6] = {0, 1, 0, 1, 2, 3}, kc[6] = {0, 1, 2, 3, 0, 1};
    for (int n = 0; n < 2048; ++n) {
      const int tq = (fix & 1) ? 0 : (n & 1), j = n >> 1, st = rot ? (j & 3) : 0;
      const uint32_t sc = t + (n % 3) * 128;
      uint32_t qb = q0 + tq * 16384, kb = k0 + st * 16384;
      if (fix & 4) { qb = q0; kb = q0 + 8192; }        // mode 6's overlapping operands
#pragma unroll
      for (int u = 0; u < 6; ++u) {
        if (qtmem)   // A (Q) from TMEM columns of the O' area (timing only)
          mma_ts(sc, t + 384 + 8 * (u & 3), sdesc(kb + kc[u] * 32, 1024, kSwizzle128B), idS, u);
        else
          mma_ss(sc, sdesc(qb + qa[u] * 32, 1024, kSwizzle128B),
                 sdesc(kb + kc[u] * 32, 1024, kSwizzle128B), idS, u);
      }
      if (n >= 2) {
        const int m = n - 2, jm = m >> 1, sv = rot ? (jm & 3) : 0;
        const uint32_t bc = t + (m % 3) * 128, oc = t + 384 + ((fix & 2) ? 0 : 64 * (m & 1));
        uint32_t vb = v0 + sv * 16384;
        if (fix & 4) vb = q0 + 24576;
        if (fix & 8) vb = k0 + sv * 16384;              // V = the K stage (same lines)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t ah = bc + (kk >> 2) * 64 + (kk & 3) * 8;
          const uint32_t vh = vb + (kk >> 2) * 8192 + (kk & 3) * 32;
          mma_ts(oc, ah, sdesc(vh, 1024, kSwizzle128B), idP64, kk);
          mma_ts(oc, ah + 32, sdesc(vh, 1024, kSwizzle128B), idP32, 1);
        }
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(t);
}

void run_rot(int rot, int qtmem, int rnd = 0, int fix = 0) {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  // fix & 16 (with fix & 4: operands inside 40 KB): 41 KB of dynamic smem; fix & 32: 512 threads
  const int smem = (fix & 16) ? 41 * 1024 : 160 * 1024 + 1024;
  const int thr = (fix & 32) ? 512 : 128;
  cudaFuncSetAttribute(rot_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024 + 1024);
  rot_bench<<<148, thr, smem>>>(cyc, rot, qtmem, rnd, fix);
  cudaDeviceSynchronize();
  rot_bench<<<148, thr, smem>>>(cyc, rot, qtmem, rnd, fix);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < 148; ++i) mean += double(h[i]) / 148;
  printf("x3w MMA stream, kernel operand layout, rotate=%d Q-in-TMEM=%d operands=%s fixQ=%d fixO=%d fix=%d: %.1f clk/S tile (%s)\n",
         rot, qtmem, rnd ? "random" : "zero", fix & 1, fix >> 1 & 1, fix, mean / 2048.0, cudaGetErrorString(e));
  cudaFree(cyc);
}

int main() {
  run_rot(0, 0);
  run_rot(1, 0);
  run_rot(1, 1);
  run_rot(1, 0, 1);
  run_rot(1, 1, 1);
  run_rot(0, 0, 1);
  run_rot(0, 0, 0, 32);
  run_rot(0, 0, 0, 16 + 4);
  run_rot(0, 0, 0, 16 + 4 + 3);
  run_rot(0, 0, 0, 16 + 32 + 4 + 3);
  const double ab0 = double(kIters) * 8 * 4096;
  run<6, 128, 1>("x3w MMA stream (S 6xN128 + PV 8x(N64+N32))", 1, ab0);
  run<8, 128, 1>("x3w MMA stream + commits (mask)", 0, ab0);
  return 0;
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
  for (int w : {1, 2, 4})
    run<4, 32, 1>("mma SS N32, one issuer per warp", w, ab * w);
  for (int w : {1, 2, 4})
    run<4, 64, 1>("mma SS N64, one issuer per warp", w, ab * w);
  for (int w : {0, 4, 8})
    run<5, 128, 1>("mma SS N128 + LDTM warps", w, ab);
  run<6, 128, 1>("x3w MMA stream (S 6xN128 + PV 8x(N64+N32))", 1, ab);
  for (int w : {4, 8})
    run<7, 128, 1>("x3w MMA stream + softmax TMEM ld/st", w, ab);
  for (int w : {0, 1, 3, 7, 15, 23, 31})   // bit 0: commit after S, 1: after PV, 2: K/V release, 3: fence::after_thread_sync x2, 4: mbarrier try_wait x2
    run<8, 128, 1>("x3w MMA stream + commits (mask)", w, ab);
  run<2, 64, 1>("mma A=TMEM", 1, ab);
  run<2, 128, 1>("mma A=TMEM", 1, ab);
  return 0;
}
