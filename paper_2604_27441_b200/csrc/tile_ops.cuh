// tile_ops.cuh -- CTA-level fp32 building blocks shared by the token kernels:
// small GEMMs against K-major weights, LayerNorm, and the Q/K/V scatter into
// the spatial-attention layouts.
#pragma once

#include "common.cuh"

namespace nvrec {

// out(t, n) = sum_k in[t*ldi + k] * Wt[k*N + n] + bias[n], for t < ntok,
// n < N (N % 4 == 0).  `in` lives in shared memory; Wt/bias in global (L1/L2
// resident: the whole model is ~1.5 MB).  Each work item is a 4-token x
// 4-column register tile: per k one 16-byte coalesced weight load, four
// broadcast shared loads and 16 FMAs.  epi(t, n, v) consumes each result.
template <class Epi>
__device__ __forceinline__ void tile_gemm(const float* in, int ldi, int ntok, int K,
                                          const float* __restrict__ Wt,
                                          const float* __restrict__ bias, int N,
                                          Epi epi) {
  const int nq = N >> 2;
  const int tq = (ntok + 3) >> 2;
  for (int item = threadIdx.x; item < nq * tq; item += blockDim.x) {
    const int cq = item % nq, tg = item / nq;
    const int t0 = tg * 4;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    const float* a0 = in + min(t0 + 0, ntok - 1) * ldi;
    const float* a1 = in + min(t0 + 1, ntok - 1) * ldi;
    const float* a2 = in + min(t0 + 2, ntok - 1) * ldi;
    const float* a3 = in + min(t0 + 3, ntok - 1) * ldi;
    const float* w = Wt + cq * 4;
#pragma unroll 4
    for (int k = 0; k < K; ++k) {
      const float4 wv = __ldg(reinterpret_cast<const float4*>(w + size_t(k) * N));
      const float x0 = a0[k], x1 = a1[k], x2 = a2[k], x3 = a3[k];
      acc[0][0] = fmaf(x0, wv.x, acc[0][0]); acc[0][1] = fmaf(x0, wv.y, acc[0][1]);
      acc[0][2] = fmaf(x0, wv.z, acc[0][2]); acc[0][3] = fmaf(x0, wv.w, acc[0][3]);
      acc[1][0] = fmaf(x1, wv.x, acc[1][0]); acc[1][1] = fmaf(x1, wv.y, acc[1][1]);
      acc[1][2] = fmaf(x1, wv.z, acc[1][2]); acc[1][3] = fmaf(x1, wv.w, acc[1][3]);
      acc[2][0] = fmaf(x2, wv.x, acc[2][0]); acc[2][1] = fmaf(x2, wv.y, acc[2][1]);
      acc[2][2] = fmaf(x2, wv.z, acc[2][2]); acc[2][3] = fmaf(x2, wv.w, acc[2][3]);
      acc[3][0] = fmaf(x3, wv.x, acc[3][0]); acc[3][1] = fmaf(x3, wv.y, acc[3][1]);
      acc[3][2] = fmaf(x3, wv.z, acc[3][2]); acc[3][3] = fmaf(x3, wv.w, acc[3][3]);
    }
    const float4 bv = __ldg(reinterpret_cast<const float4*>(bias + cq * 4));
    const float bb[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (t0 + i < ntok) {
#pragma unroll
        for (int j = 0; j < 4; ++j) epi(t0 + i, cq * 4 + j, acc[i][j] + bb[j]);
      }
    }
  }
}

// Same contract as tile_gemm for a CTA holding only a handful of tokens
// (pruned last block): work items are (token, 4 columns, K slice); the K
// slices shorten the serial dependence chain ks-fold and are summed through
// `red` (shared, >= blockDim.x * 4 floats).  All threads must call it.
template <class Epi>
__device__ __forceinline__ void tile_gemm_narrow(const float* in, int ldi, int ntok, int K,
                                                 const float* __restrict__ Wt,
                                                 const float* __restrict__ bias, int N,
                                                 float* red, Epi epi) {
  const int nq = N >> 2;
  const int items = nq * ntok;
  int ks = 1;
  while (ks * 2 * items <= int(blockDim.x) && ks * 2 * 8 <= K) ks *= 2;
  for (int base = 0; base < items; base += blockDim.x) {
    const int active = min(items - base, int(blockDim.x) / ks);
    const int t_id = threadIdx.x;
    const int it = t_id % active, slice = t_id / active;
    if (t_id < active * ks) {
      const int item = base + it;
      const int cq = item % nq, t = item / nq;
      const int k0 = slice * (K / ks), k1 = (slice + 1 == ks) ? K : k0 + K / ks;
      const float* a0 = in + t * ldi;
      const float* w = Wt + cq * 4;
      float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
      // 16 weight rows in flight per batch (the phase is L2-latency bound);
      // same accumulation order as the plain loop
      int k = k0;
      for (; k + 16 <= k1; k += 16) {
        float4 wv[16];
        float xv[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          wv[u] = __ldg(reinterpret_cast<const float4*>(w + size_t(k + u) * N));
          xv[u] = a0[k + u];
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          c0 = fmaf(xv[u], wv[u].x, c0); c1 = fmaf(xv[u], wv[u].y, c1);
          c2 = fmaf(xv[u], wv[u].z, c2); c3 = fmaf(xv[u], wv[u].w, c3);
        }
      }
      for (; k < k1; ++k) {
        const float4 wv = __ldg(reinterpret_cast<const float4*>(w + size_t(k) * N));
        const float x0 = a0[k];
        c0 = fmaf(x0, wv.x, c0); c1 = fmaf(x0, wv.y, c1);
        c2 = fmaf(x0, wv.z, c2); c3 = fmaf(x0, wv.w, c3);
      }
      float* r = red + 4 * (slice * active + it);
      r[0] = c0; r[1] = c1; r[2] = c2; r[3] = c3;
    }
    __syncthreads();
    for (int o = threadIdx.x; o < active * 4; o += blockDim.x) {
      const int it2 = o >> 2, j = o & 3;
      float acc = 0.f;
      for (int sl = 0; sl < ks; ++sl) acc += red[4 * (sl * active + it2) + j];
      const int item = base + it2;
      const int cq = item % nq, t = item / nq;
      epi(t, cq * 4 + j, acc + __ldg(bias + cq * 4 + j));
    }
    __syncthreads();
  }
}

// LayerNorm (eps 1e-5, biased variance, affine) of rows of width d <= 128,
// one warp per row: out[r*ldo + :] = LN(in[r*ldi + :]).  nn.LayerNorm
// (model.py:47-52,79).
__device__ __forceinline__ void tile_layernorm(const float* in, int ldi, float* out, int ldo,
                                               int nrows, int d,
                                               const float* __restrict__ g,
                                               const float* __restrict__ bta) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  for (int r = warp; r < nrows; r += nwarps) {
    const float* x = in + r * ldi;
    float v[4];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int c = lane + 32 * i;
      v[i] = c < d ? x[c] : 0.f;
      s += v[i];
    }
    const float mean = warp_sum(s) / float(d);
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int c = lane + 32 * i;
      float t = c < d ? v[i] - mean : 0.f;
      q = fmaf(t, t, q);
    }
    const float rstd = rsqrtf(warp_sum(q) / float(d) + 1e-5f);
    float* o = out + r * ldo;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int c = lane + 32 * i;
      if (c < d) o[c] = (v[i] - mean) * rstd * __ldg(g + c) + __ldg(bta + c);
    }
  }
}

// Scatter one qkv feature (model.py:37: reshape(b, t, 3, heads, hd)) of the
// token (b, it, s) into the spatial-attention operand layouts.
struct QkvDst {
  float* q; float* k; float* v;                     // SIMT attention (fp32) layouts
  __nv_bfloat16* qh; __nv_bfloat16* kh; __nv_bfloat16* vth;  // tensor-core layouts
  const int* rank;   // non-null: Q rows are compact (pruned consumer block)
  int nt, ns, ns_pad, d, heads, hd;
  int x3;            // tensor-core precise path: bf16 hi/lo split, Q/K rows
                     // [hi(hd) | lo(hd)], V^T rows hi 0..hd-1, lo hd..2hd-1
};

__device__ __forceinline__ void qkv_store(const QkvDst& o, int b, int it, int s, int n, float v) {
  const int which = n / o.d;
  const int f = n - which * o.d;
  const int hh = f / o.hd, e = f - hh * o.hd;
  const size_t seq = size_t(b * o.nt + it) * o.heads + hh;
  int row = s;
  if (which == 0 && o.rank) {
    row = o.rank[b * o.ns + s];
    if (row < 0) return;
  }
  if (o.qh && o.x3) {
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    const __nv_bfloat16 lo = __float2bfloat16_rn(v - __bfloat162float(hi));
    if (which < 2) {
      __nv_bfloat16* r = (which == 0 ? o.qh : o.kh) + (seq * o.ns_pad + row) * 2 * o.hd;
      r[e] = hi;
      r[o.hd + e] = lo;
    } else {
      o.vth[(seq * 2 * o.hd + e) * o.ns_pad + row] = hi;
      o.vth[(seq * 2 * o.hd + o.hd + e) * o.ns_pad + row] = lo;
    }
  } else if (o.qh) {
    if (which == 0) o.qh[(seq * o.ns_pad + row) * o.hd + e] = __float2bfloat16_rn(v);
    else if (which == 1) o.kh[(seq * o.ns_pad + row) * o.hd + e] = __float2bfloat16_rn(v);
    else o.vth[(seq * o.hd + e) * o.ns_pad + row] = __float2bfloat16_rn(v);
  } else {
    float* dst = which == 0 ? o.q : (which == 1 ? o.k : o.v);
    dst[(seq * o.ns_pad + row) * o.hd + e] = v;
  }
}

__device__ __forceinline__ float gelu_erf(float x) {   // nn.GELU() default
  return 0.5f * x * (1.f + erff(x * 0.70710678118654752440f));
}

// nn.GELU() (erf form) with erf from Abramowitz-Stegun 7.1.26 (|err| < 1.5e-7;
// GELU |err| < 5e-7 measured over [-12, 12]): one MUFU rcp + one MUFU ex2 +
// 10 FMA-pipe ops instead of erff's ~30.  Used where the result is rounded
// to fp16 anyway (tensor-core operands).
__device__ __forceinline__ float gelu_as(float v) {
  float t;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(fabsf(v), 0.3275911f * 0.70710678118654752440f, 1.f)));
  float p = fmaf(t, 0.5f * 1.061405429f, 0.5f * -1.453152027f);
  p = fmaf(p, t, 0.5f * 1.421413741f);
  p = fmaf(p, t, 0.5f * -0.284496736f);
  p = fmaf(p, t, 0.5f * 0.254829592f);
  p *= t;
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"((v * v) * (-0.5f * 1.4426950408889634f)));
  const float h = p * e;                       // (1 - erf(|v|/sqrt 2)) / 2
  return v * (v >= 0.f ? 1.f - h : h);
}

// Stage the 12 block-tail parameter vectors (biases and LayerNorm affines,
// concatenated in `par` order, vector q ending at tail_par_end(q)) into shared
// memory with every global load in flight at once: one flat, unrolled pass
// (a struct-array loop indexed at run time lands in local memory and
// serialises twelve load round trips at every CTA start).
__host__ __device__ constexpr int tail_par_end(int q) {
  return q < 3 ? 64 * (q + 1) : q == 3 ? 384 : q < 7 ? 448 + 64 * (q - 4) : q == 7 ? 832
       : 896 + 64 * (q - 8) > 1024 ? 1216 : 896 + 64 * (q - 8);
}
static_assert(tail_par_end(0) == 64 && tail_par_end(3) == 384 && tail_par_end(6) == 576 &&
              tail_par_end(7) == 832 && tail_par_end(10) == 1024 && tail_par_end(11) == 1216,
              "tail parameter layout");
template <int kThreadsT>
__device__ __forceinline__ void stage_tail_params(float* par, const float* const (&src)[12]) {
  constexpr int kN = tail_par_end(11);
  constexpr int kPer = (kN + kThreadsT - 1) / kThreadsT;
  float v[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int i = int(threadIdx.x) + k * kThreadsT;
    const float* p = src[11];
    int base = tail_par_end(10);
#pragma unroll
    for (int q = 10; q >= 0; --q)
      if (i < tail_par_end(q)) {
        p = src[q];
        base = q ? tail_par_end(q - 1) : 0;
      }
    v[k] = i < kN ? __ldg(p + (i - base)) : 0.f;
  }
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int i = int(threadIdx.x) + k * kThreadsT;
    if (i < kN) par[i] = v[k];
  }
}

}  // namespace nvrec
