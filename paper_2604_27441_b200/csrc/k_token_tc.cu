// k_token_tc.cu -- tensor-core (tcgen05) version of the fused block tail for
// a NON-LAST block on the fast path: everything between one spatial
// attention and the next (model.py:60-64 then :59/:37 of the next block):
//
//   x += proj_s(ao)                    [128 x 64]  . [64 x 64]
//   t  = LN_t(x); qkv = qkv_t(t)       [128 x 64]  . [64 x 192]
//   a  = attn over the nt slices of each position (CUDA cores, fp32)
//   x += proj_t(a)                     [128 x 64]  . [64 x 64]
//   h  = GELU(fc1(LN_m(x)))            [128 x 64]  . [64 x 256]
//   x += fc2(h)                        [128 x 256] . [256 x 64]
//   q,k,v = qkv_s'(LN_s'(x))           [128 x 64]  . [64 x 192]  -> bf16 attention operands
//
// Persistent CTAs (one per SM) keep all six fp16 weight matrices of the block
// resident in shared memory (128 KB, loaded once by bulk copies) and loop over
// tiles of 128 rows = P positions x nt slices (P = 128/nt; siblings of a
// position are adjacent rows).  Warps 0-3 own one row each per thread (TMEM
// lane = row): they keep the fp32 residual x in registers, do LayerNorm, bias,
// GELU (erf) and the 3-token temporal softmax on CUDA cores, and write the
// fp16 A operands (no-swizzle K-major core matrices); warp 4 issues the MMAs
// (fp32 accumulation in TMEM).
#include "launch.cuh"
#include "sm100.cuh"

namespace nvrec {

namespace {

using namespace sm100;

constexpr int kThreads = 160;
constexpr uint32_t kWBlockElems = 53248;          // proj_s..fc2 of one block
constexpr uint32_t kOffProjS = 0, kOffQkvT = 4096, kOffProjT = 16384, kOffFc1 = 20480,
                   kOffFc2 = 36864, kOffQkvS = 53248;
constexpr int kXStride = 68;                      // fp32 exchange row (bank spread)
// staged parameter vectors (floats): offsets into TokSmem::par
constexpr int kPBProjS = 0, kPLnTw = 64, kPLnTb = 128, kPBQkvT = 192, kPBProjT = 384,
              kPLnMw = 448, kPLnMb = 512, kPBFc1 = 576, kPBFc2 = 832, kPLnSw = 896,
              kPLnSb = 960, kPBQkvN = 1024, kParFloats = 1216;

struct __align__(128) TokSmem {
  __half w[kOffQkvS + 12288];     // 128 KB of weights
  uint8_t a[128 * 64 * 2];        // 16 KB fp16 A operand (K = 64)
  uint8_t h[128 * 256 * 2];       // 64 KB fp16 hidden (K = 256) / fp32 k,v exchange
  float par[kParFloats];          // biases + LN affine, staged once per CTA
  uint64_t bar_w, bar_a, bar_d;
  uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// one row of 64 fp32 -> fp16 K-major core-matrix layout (row m)
__device__ __forceinline__ void put_row64(uint8_t* base, int m, const float* y) {
#pragma unroll
  for (int ki = 0; ki < 8; ++ki)
    *reinterpret_cast<uint4*>(base + ki * 2048 + m * 16) =
        make_uint4(pack_h2(y[8 * ki], y[8 * ki + 1]), pack_h2(y[8 * ki + 2], y[8 * ki + 3]),
                   pack_h2(y[8 * ki + 4], y[8 * ki + 5]), pack_h2(y[8 * ki + 6], y[8 * ki + 7]));
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

__device__ __forceinline__ void named_sync() {
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
token_tc_kernel(TokenTcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  TokSmem& sm =
      *reinterpret_cast<TokSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = a.nt;
  const int P = 128 / nt;                  // positions per tile
  const int tiles_per_b = (a.ns + P - 1) / P;
  const int n_tiles = tiles_per_b * a.b;

  if (warp == 4 && lane == 0) {
    mbar_init(&sm.bar_w, 1);
    mbar_init(&sm.bar_a, 128);
    mbar_init(&sm.bar_d, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  // TMEM columns: fc1 accumulator [0,256); 192-wide [256,448); 64-wide [448,512)
  constexpr uint32_t kD256 = 0, kD192 = 256, kD64 = 448;

  if (warp == 4) {
    if (lane == 0) {
      mbar_expect_tx(&sm.bar_w, (kWBlockElems + 12288) * 2);
      bulk_load(sm.w, a.w_blk, kWBlockElems * 2, &sm.bar_w);
      bulk_load(sm.w + kOffQkvS, a.w_qkv_next, 12288 * 2, &sm.bar_w);
      mbar_wait(&sm.bar_w, 0);
      const uint32_t wb = smem_u32(sm.w), ab = smem_u32(sm.a), hb = smem_u32(sm.h);
      uint32_t pa = 0;
      auto gemm = [&](uint32_t dcol, uint32_t abase, uint32_t woff, int N, int K) {
        mbar_wait(&sm.bar_a, pa & 1);
        ++pa;
        tc_fence_after();
        const uint32_t idesc = idesc_f16(128, N), lbo_b = (N / 8) * 128;
        const uint32_t bbase = wb + woff * 2;
        for (int kk = 0; kk < K / 16; ++kk)
          mma_ss(tmem + dcol, sdesc(abase + kk * 4096, 128, kSwizzleNone, 2048),
                 sdesc(bbase + kk * 2 * lbo_b, 128, kSwizzleNone, lbo_b), idesc, kk != 0);
        mma_commit(&sm.bar_d);
      };
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        gemm(kD64, ab, kOffProjS, 64, 64);
        gemm(kD192, ab, kOffQkvT, 192, 64);
        gemm(kD64, ab, kOffProjT, 64, 64);
        gemm(kD256, ab, kOffFc1, 256, 64);
        gemm(kD64, hb, kOffFc2, 64, 256);
        gemm(kD192, ab, kOffQkvS, 192, 64);
      }
    }
  } else {
    {
      const struct { const float* src; int off, n; } vecs[12] = {
          {a.b_proj_s, kPBProjS, 64}, {a.ln_t_w, kPLnTw, 64}, {a.ln_t_b, kPLnTb, 64},
          {a.b_qkv_t, kPBQkvT, 192}, {a.b_proj_t, kPBProjT, 64}, {a.ln_m_w, kPLnMw, 64},
          {a.ln_m_b, kPLnMb, 64}, {a.b_fc1, kPBFc1, 256}, {a.b_fc2, kPBFc2, 64},
          {a.ln_s_next_w, kPLnSw, 64}, {a.ln_s_next_b, kPLnSb, 64}, {a.b_qkv_next, kPBQkvN, 192}};
#pragma unroll 1
      for (int v = 0; v < 12; ++v)
        for (int i = threadIdx.x; i < vecs[v].n; i += 128) sm.par[vecs[v].off + i] = vecs[v].src[i];
      named_sync();
    }
    const float* P_ = sm.par;
    const int m = threadIdx.x;                       // row == TMEM lane
    const uint32_t lane_off = uint32_t(warp * 32) << 16;
    const int j = m / nt, it = m - j * nt;           // position slot, slice
    uint32_t pd = 0;
    auto wait_d = [&]() {
      mbar_wait(&sm.bar_d, pd & 1);
      ++pd;
      tc_fence_after();
    };
    auto signal_a = [&]() {
      fence_proxy_async();
      mbar_arrive(&sm.bar_a);
    };
    // x += D[64 cols at col] + bias
    auto add64 = [&](float* x, uint32_t col, const float* bias) {
      uint32_t r[32];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        tmem_ld32(tmem + lane_off + col + 32 * h, r);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) x[32 * h + e] += __uint_as_float(r[e]) + bias[32 * h + e];
      }
    };
    const float scale = rsqrtf(32.f);
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const int b = tile / tiles_per_b;
      const int s0 = (tile - b * tiles_per_b) * P;
      const int s = s0 + j;
      const bool valid = m < P * nt && s < a.ns;
      const size_t xrow = (size_t(b * nt + it) * a.ns + s) * 64;
      float x[64], y[64];
      // ---- 1. x += proj_s(ao) ------------------------------------------------
      {
        const float4* ao = reinterpret_cast<const float4*>(a.ao + xrow);
        const float4* xi = reinterpret_cast<const float4*>(a.x + xrow);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          float4 v = valid ? ao[q] : make_float4(0.f, 0.f, 0.f, 0.f);
          float4 u = valid ? xi[q] : make_float4(0.f, 0.f, 0.f, 0.f);
          y[4 * q] = v.x; y[4 * q + 1] = v.y; y[4 * q + 2] = v.z; y[4 * q + 3] = v.w;
          x[4 * q] = u.x; x[4 * q + 1] = u.y; x[4 * q + 2] = u.z; x[4 * q + 3] = u.w;
        }
      }
      put_row64(sm.a, m, y);
      signal_a();
      wait_d();
      add64(x, kD64, P_ + kPBProjS);
      // ---- 2. qkv_t(LN_t(x)) -------------------------------------------------
      layernorm64(x, y, P_ + kPLnTw, P_ + kPLnTb);
      put_row64(sm.a, m, y);
      signal_a();
      wait_d();
      // q stays in registers (y), k and v of one head at a time go through smem
      {
        uint32_t r[32];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          tmem_ld32(tmem + lane_off + kD192 + 32 * h, r);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) y[32 * h + e] = __uint_as_float(r[e]) + P_[kPBQkvT + 32 * h + e];
        }
      }
      float* xch = reinterpret_cast<float*>(sm.h);   // [128][kXStride]: k(32) | v(32)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_off + kD192 + 64 + 32 * hh, r);       // k, head hh
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e)
          xch[m * kXStride + e] = __uint_as_float(r[e]) + P_[kPBQkvT + 64 + 32 * hh + e];
        tmem_ld32(tmem + lane_off + kD192 + 128 + 32 * hh, r);      // v, head hh
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e)
          xch[m * kXStride + 32 + e] = __uint_as_float(r[e]) + P_[kPBQkvT + 128 + 32 * hh + e];
        named_sync();
        float sc[8];
        float mx = -INFINITY;
#pragma unroll
        for (int ik = 0; ik < 8; ++ik) {
          if (ik >= nt) break;
          const float4* kr = reinterpret_cast<const float4*>(xch + min(j * nt + ik, 127) * kXStride);
          float acc = 0.f;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 kv = kr[q];
            acc = fmaf(y[32 * hh + 4 * q], kv.x, acc);
            acc = fmaf(y[32 * hh + 4 * q + 1], kv.y, acc);
            acc = fmaf(y[32 * hh + 4 * q + 2], kv.z, acc);
            acc = fmaf(y[32 * hh + 4 * q + 3], kv.w, acc);
          }
          sc[ik] = acc * scale;
          mx = fmaxf(mx, sc[ik]);
        }
        float den = 0.f;
#pragma unroll
        for (int ik = 0; ik < 8; ++ik) {
          if (ik >= nt) break;
          sc[ik] = __expf(sc[ik] - mx);
          den += sc[ik];
        }
        const float inv = 1.f / den;
        float o[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = 0.f;
#pragma unroll
        for (int ik = 0; ik < 8; ++ik) {
          if (ik >= nt) break;
          const float4* vr = reinterpret_cast<const float4*>(xch + min(j * nt + ik, 127) * kXStride + 32);
          const float p = sc[ik] * inv;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 vv = vr[q];
            o[4 * q] = fmaf(p, vv.x, o[4 * q]);
            o[4 * q + 1] = fmaf(p, vv.y, o[4 * q + 1]);
            o[4 * q + 2] = fmaf(p, vv.z, o[4 * q + 2]);
            o[4 * q + 3] = fmaf(p, vv.w, o[4 * q + 3]);
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)                // head hh -> A columns [32hh, 32hh+32)
          *reinterpret_cast<uint4*>(sm.a + (4 * hh + q) * 2048 + m * 16) =
              make_uint4(pack_h2(o[8 * q], o[8 * q + 1]), pack_h2(o[8 * q + 2], o[8 * q + 3]),
                         pack_h2(o[8 * q + 4], o[8 * q + 5]), pack_h2(o[8 * q + 6], o[8 * q + 7]));
        named_sync();                              // exchange buffer reused
      }
      // ---- 3. x += proj_t(o) ---------------------------------------------------
      signal_a();
      wait_d();
      add64(x, kD64, P_ + kPBProjT);
      // ---- 4. h = GELU(fc1(LN_m(x))) -------------------------------------------
      layernorm64(x, y, P_ + kPLnMw, P_ + kPLnMb);
      put_row64(sm.a, m, y);
      signal_a();
      wait_d();
#pragma unroll 1
      for (int c8 = 0; c8 < 8; ++c8) {               // 8 chunks of 32 hidden units
        uint32_t r[32];
        tmem_ld32(tmem + lane_off + kD256 + 32 * c8, r);
        tmem_wait_ld();
        float g[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) g[e] = gelu_erf(__uint_as_float(r[e]) + P_[kPBFc1 + 32 * c8 + e]);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<uint4*>(sm.h + (4 * c8 + q) * 2048 + m * 16) =
              make_uint4(pack_h2(g[8 * q], g[8 * q + 1]), pack_h2(g[8 * q + 2], g[8 * q + 3]),
                         pack_h2(g[8 * q + 4], g[8 * q + 5]), pack_h2(g[8 * q + 6], g[8 * q + 7]));
      }
      signal_a();
      wait_d();
      // ---- 5. x += fc2(h); store x -----------------------------------------------
      add64(x, kD64, P_ + kPBFc2);
      if (valid) {
        float4* xo = reinterpret_cast<float4*>(a.x + xrow);
#pragma unroll
        for (int q = 0; q < 16; ++q) xo[q] = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
      }
      // ---- 6. next block's LN_s + qkv_s -> bf16 attention operands ----------------
      layernorm64(x, y, P_ + kPLnSw, P_ + kPLnSb);
      put_row64(sm.a, m, y);
      signal_a();
      wait_d();
      int qrow = s;
      if (a.qrank) qrow = valid ? a.qrank[b * a.ns + s] : -1;
#pragma unroll 1
      for (int c6 = 0; c6 < 6; ++c6) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_off + kD192 + 32 * c6, r);
        tmem_wait_ld();
        if (!valid) continue;
        const int which = c6 >> 1, head = c6 & 1;
        const size_t seq = size_t(b * nt + it) * 2 + head;
        float v[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]) + P_[kPBQkvN + 32 * c6 + e];
        if (which < 2) {
          if (which == 0 && qrow < 0) continue;
          uint4* d4 = reinterpret_cast<uint4*>((which == 0 ? a.qh : a.kh) +
                                               (seq * a.ns_pad + (which == 0 ? qrow : s)) * 32);
#pragma unroll
          for (int e = 0; e < 32; e += 8)
            d4[e / 8] = make_uint4(pack_bf16(v[e], v[e + 1]), pack_bf16(v[e + 2], v[e + 3]),
                                   pack_bf16(v[e + 4], v[e + 5]), pack_bf16(v[e + 6], v[e + 7]));
        } else {
          __nv_bfloat16* dst = a.vth + seq * 32 * a.ns_pad + s;
#pragma unroll
          for (int e = 0; e < 32; ++e) dst[size_t(e) * a.ns_pad] = __float2bfloat16_rn(v[e]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

}  // namespace

bool token_tc_supported(const Dims& D) {
  return D.d == 64 && D.heads == 2 && D.nt <= 8 && D.hidden == 256;
}

cudaError_t launch_token_tc(const TokenTcArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(TokSmem) + 128;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(token_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr = true;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int P = 128 / a.nt;
  const int tiles = ((a.ns + P - 1) / P) * a.b;
  token_tc_kernel<<<tiles < sms ? tiles : sms, kThreads, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace nvrec
