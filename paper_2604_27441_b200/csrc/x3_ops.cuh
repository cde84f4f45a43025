// x3_ops.cuh -- per-row helpers of the split-operand ("x3", fp32-class)
// tensor-core kernels: fp16/bf16 hi/lo splits, a 64-wide row written as the
// [hi | lo] K-major no-swizzle UMMA A operand of a 128-row tile, LayerNorm.
#pragma once

#include "sm100.cuh"

namespace nvrec {
namespace x3 {

using namespace sm100;

constexpr uint32_t kABytes = 128 * 64 * 2;       // one fp16 [128 x 64] operand copy

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
// fp16 hi/lo split of a pair
__device__ __forceinline__ void split_h2(float x, float y, uint32_t& hi, uint32_t& lo) {
  hi = pack_h2(x, y);
  const float2 h = __half22float2(*reinterpret_cast<const __half2*>(&hi));
  lo = pack_h2(x - h.x, y - h.y);
}
// bf16 hi/lo split of a pair (the attention operands)
__device__ __forceinline__ void split_bf16(float x, float y, uint32_t& hi, uint32_t& lo) {
  hi = pack_bf16(x, y);
  const float2 h = unpack_bf16(hi);
  lo = pack_bf16(x - h.x, y - h.y);
}

// row m of 64 fp32 -> [hi | lo] fp16 K-major core-matrix operands; cols
// [c0, c0 + 8 nk) only (the temporal attention writes one head at a time)
__device__ __forceinline__ void put_row_x3(uint8_t* base, int m, const float* y, int k0 = 0,
                                           int nk = 8) {
#pragma unroll
  for (int ki = 0; ki < 8; ++ki) {
    if (ki >= nk) break;
    uint32_t h[4], l[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) split_h2(y[8 * ki + 2 * j], y[8 * ki + 2 * j + 1], h[j], l[j]);
    *reinterpret_cast<uint4*>(base + (k0 + ki) * 2048 + m * 16) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(base + kABytes + (k0 + ki) * 2048 + m * 16) =
        make_uint4(l[0], l[1], l[2], l[3]);
  }
}

__device__ __forceinline__ void layernorm64(const float* x, float* y, const float* g,
                                            const float* bt) {
  float mean = 0.f;
#pragma unroll
  for (int o = 0; o < 64; ++o) mean += x[o];
  mean *= (1.f / 64.f);
  float var = 0.f;
#pragma unroll
  for (int o = 0; o < 64; ++o) var = fmaf(x[o] - mean, x[o] - mean, var);
  const float rstd = rsqrtf(var * (1.f / 64.f) + 1e-5f);
#pragma unroll
  for (int o = 0; o < 64; ++o) y[o] = (x[o] - mean) * rstd * g[o] + bt[o];
}

// LayerNorm of a 64-wide row written straight into the [hi | lo] A operand
// (no 64-float output array: 8 values at a time)
__device__ __forceinline__ void ln_put_row_x3(uint8_t* base, int m, const float* x, const float* g,
                                              const float* bt) {
  float mean = 0.f;
#pragma unroll
  for (int o = 0; o < 64; ++o) mean += x[o];
  mean *= (1.f / 64.f);
  float var = 0.f;
#pragma unroll
  for (int o = 0; o < 64; ++o) var = fmaf(x[o] - mean, x[o] - mean, var);
  const float rstd = rsqrtf(var * (1.f / 64.f) + 1e-5f);
#pragma unroll
  for (int ki = 0; ki < 8; ++ki) {
    float y[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int o = 8 * ki + j;
      y[j] = (x[o] - mean) * rstd * __ldg(g + o) + __ldg(bt + o);
    }
    uint32_t h[4], l[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) split_h2(y[2 * j], y[2 * j + 1], h[j], l[j]);
    *reinterpret_cast<uint4*>(base + ki * 2048 + m * 16) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(base + kABytes + ki * 2048 + m * 16) = make_uint4(l[0], l[1], l[2], l[3]);
  }
}

}  // namespace x3
}  // namespace nvrec
