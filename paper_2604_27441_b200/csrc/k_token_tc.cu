// k_token_tc.cu -- tensor-core (tcgen05) version of the fused block tail for
// a NON-LAST block on the fast path: everything between one spatial
// attention and the next (model.py:60-64 then :59/:37 of the next block):
//
//   x += proj_s(ao)                    [128 x 64]  . [64 x 64]
//   t  = LN_t(x); qkv = qkv_t(t)       [128 x 64]  . [64 x 192]
//   a  = attn over the nt slices of each position (CUDA cores, fp32)
//   x += proj_t(a)                     [128 x 64]  . [64 x 64]
//   h  = GELU(fc1(LN_m(x)))            [128 x 64]  . [64 x 256]
//   x += fc2(h)                        [128 x 256] . [256 x 64]   (h from TMEM)
//   q,k,v = qkv_s'(LN_s'(x))           [128 x 64]  . [64 x 192]  -> bf16 attention operands
//
// Persistent CTAs (one per SM) keep all six fp16 weight matrices of the block
// resident in shared memory (128 KB, loaded once by bulk copies).  Two tile
// slots per CTA, each a warpgroup that owns one 128-row tile at a time, so
// one slot's CUDA-core work (LayerNorm, bias, GELU, temporal softmax) overlaps
// the other's MMAs.  Every warp holds floor(32/nt) whole positions (lane =
// j*nt + slice; the leftover lanes are idle rows), so the temporal attention
// across the nt slices of a position is a handful of warp shuffles.  Each
// slot issues its own MMAs (elected thread after a 128-thread named barrier);
// fp32 accumulators live in the slot's 256 TMEM columns, and the GELU output
// is written back there as fp16 pairs and consumed by the fc2 MMA directly
// from TMEM (no shared-memory round trip for the 128 x 256 hidden tile).
#include "launch.cuh"
#include "sm100.cuh"

namespace nvrec {

namespace {

using namespace sm100;

constexpr int kSlots = 2;
constexpr int kThreads = 128 * kSlots;
constexpr uint32_t kWBlockElems = 53248;          // proj_s..fc2 of one block
constexpr uint32_t kOffProjS = 0, kOffQkvT = 4096, kOffProjT = 16384, kOffFc1 = 20480,
                   kOffFc2 = 36864, kOffQkvS = 53248;
// staged parameter vectors (floats): offsets into TokSmem::par
constexpr int kPBProjS = 0, kPLnTw = 64, kPLnTb = 128, kPBQkvT = 192, kPBProjT = 384,
              kPLnMw = 448, kPLnMb = 512, kPBFc1 = 576, kPBFc2 = 832, kPLnSw = 896,
              kPLnSb = 960, kPBQkvN = 1024, kParFloats = 1216;

struct __align__(128) TokSmem {
  __half w[kOffQkvS + 12288];     // 128 KB of weights
  uint8_t a[kSlots][128 * 64 * 2];// 16 KB fp16 A operand (K = 64) per slot
  float par[kParFloats];          // biases + LN affine, staged once per CTA
  uint64_t bar_w, bar_d[kSlots];
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

#ifdef NVREC_TRACE
__device__ unsigned long long g_tc_trace[2][16];
#define TT(i) \
  do { if (blockIdx.x == 0 && threadIdx.x == 0 && ntile < 2) g_tc_trace[ntile][i] = clock64(); } while (0)
#else
#define TT(i) do {} while (0)
#endif

__global__ void __launch_bounds__(kThreads, 1)
token_tc_kernel(TokenTcArgs a) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // pointer arithmetic (not integer casts) keeps the shared address space
  TokSmem& sm = *reinterpret_cast<TokSmem*>(smem_raw + ((128 - (smem_u32(smem_raw) & 127)) & 127));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = warp >> 2, wq = warp & 3;        // tile slot, TMEM lane quarter
  const int nt = a.nt;
  const int ppw = 32 / nt;                          // whole positions per warp
  const int P = 4 * ppw;                            // positions per tile
  const int tiles_per_b = (a.ns + P - 1) / P;
  const int n_tiles = tiles_per_b * a.b;

  if (threadIdx.x == 0) {
    mbar_init(&sm.bar_w, 1);
    for (int k = 0; k < kSlots; ++k) mbar_init(&sm.bar_d[k], 1);
    fence_mbar_init();
    mbar_expect_tx(&sm.bar_w, (kWBlockElems + 12288) * 2);
    bulk_load(sm.w, a.w_blk, kWBlockElems * 2, &sm.bar_w);
    bulk_load(sm.w + kOffQkvS, a.w_qkv_next, 12288 * 2, &sm.bar_w);
  }
  {
    const float* const src[12] = {a.b_proj_s, a.ln_t_w, a.ln_t_b, a.b_qkv_t, a.b_proj_t,
                                  a.ln_m_w, a.ln_m_b, a.b_fc1, a.b_fc2, a.ln_s_next_w,
                                  a.ln_s_next_b, a.b_qkv_next};
    static_assert(kPBProjS == 0 && kPLnTw == 64 && kPBQkvT == 192 && kPBFc1 == 576 &&
                  kPBQkvN == 1024 && kParFloats == 1216, "par layout == tail_par_end");
    stage_tail_params<kThreads>(sm.par, src);
  }
  if (warp == 0) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  mbar_wait(&sm.bar_w, 0);

  const float* P_ = sm.par;
  const int m = wq * 32 + lane;                     // row == TMEM lane
  const uint32_t lane_off = uint32_t(wq * 32) << 16;
  const uint32_t tbase = sm.tmem_base + 256 * slot; // this slot's 256 columns
  const int jl = lane / nt, it = lane - jl * nt;    // position in warp, slice
  const bool row_live = jl < ppw;
  uint8_t* A = sm.a[slot];
  const uint32_t ab = smem_u32(A), wb = smem_u32(sm.w);
  const bool issuer = wq == 0;                  // warp: one elected lane issues (*_w)
  uint32_t pd = 0;
  // all 128 threads of the slot have written their operands -> one warp
  // issues the GEMM, everybody waits for the accumulator
  auto run = [&](auto issue) {
    fence_proxy_async();
    tc_fence_before();
    asm volatile("bar.sync %0, 128;" ::"r"(1 + slot) : "memory");
    if (issuer) {
      tc_fence_after();
      issue();
      mma_commit_w(&sm.bar_d[slot]);
    }
    mbar_wait(&sm.bar_d[slot], pd & 1);
    ++pd;
    tc_fence_after();
  };
  auto gemm_a = [&](uint32_t dcol, uint32_t woff, int N) {   // D = A(smem, K=64) W
    run([&] {
      const uint32_t idesc = idesc_f16(128, N), lbo_b = (N / 8) * 128;
      const uint32_t bbase = wb + woff * 2;
      for (int kk = 0; kk < 4; ++kk)
        mma_ss_w(tbase + dcol, sdesc(ab + kk * 4096, 128, kSwizzleNone, 2048),
               sdesc(bbase + kk * 2 * lbo_b, 128, kSwizzleNone, lbo_b), idesc, kk != 0);
    });
  };
  // x += D[64 cols at col] + bias
  auto add64 = [&](float* x, uint32_t col, const float* bias) {
    uint32_t r[64];
    tmem_ld32(tbase + lane_off + col, r);
    tmem_ld32(tbase + lane_off + col + 32, r + 32);
    tmem_wait_ld();
#pragma unroll
    for (int e = 0; e < 64; ++e) x[e] += __uint_as_float(r[e]) + bias[e];
  };
  const float scale = rsqrtf(32.f);

  int ntile = 0;
  for (int tile = blockIdx.x * kSlots + slot; tile < n_tiles; tile += gridDim.x * kSlots, ++ntile) {
    TT(0);
    const int b = tile / tiles_per_b;
    const int s = (tile - b * tiles_per_b) * P + wq * ppw + jl;
    const bool valid = row_live && s < a.ns;
    const size_t xrow = (size_t(b * nt + it) * a.ns + s) * 64;
    float x[64], y[64];
    // ---- 1. x += proj_s(ao) ------------------------------------------------
    {
      // ao arrives in fp16 (attn_tc rounds it exactly as put_row64 would):
      // its 8 16-byte chunks go straight into the A operand rows
      const uint4* ao = reinterpret_cast<const uint4*>(a.ao + xrow);
#pragma unroll
      for (int ki = 0; ki < 8; ++ki)
        *reinterpret_cast<uint4*>(A + ki * 2048 + m * 16) = valid ? ao[ki] : make_uint4(0, 0, 0, 0);
      if (a.xh) {
        // block 0: the embedding handed the residual over in fp16
        const uint4* xi = reinterpret_cast<const uint4*>(a.xh + xrow);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint4 u = valid ? xi[q] : make_uint4(0, 0, 0, 0);
          const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w4[e]));
            x[8 * q + 2 * e] = f.x;
            x[8 * q + 2 * e + 1] = f.y;
          }
        }
      } else {
        const float4* xi = reinterpret_cast<const float4*>(a.x + xrow);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          float4 u = valid ? xi[q] : make_float4(0.f, 0.f, 0.f, 0.f);
          x[4 * q] = u.x; x[4 * q + 1] = u.y; x[4 * q + 2] = u.z; x[4 * q + 3] = u.w;
        }
      }
    }
    TT(1);
    gemm_a(0, kOffProjS, 64);
    TT(2);
    add64(x, 0, P_ + kPBProjS);
    // ---- 2. qkv_t(LN_t(x)); temporal attention by warp shuffles --------------
    layernorm64(x, y, P_ + kPLnTw, P_ + kPLnTb);
    put_row64(A, m, y);
    TT(3);
    gemm_a(0, kOffQkvT, 192);
    TT(4);
#pragma unroll 1
    for (int hh = 0; hh < 2; ++hh) {
      float q[32], kk_[32], vv[32];
      tmem_ld32(tbase + lane_off + 32 * hh, reinterpret_cast<uint32_t*>(q));
      tmem_ld32(tbase + lane_off + 64 + 32 * hh, reinterpret_cast<uint32_t*>(kk_));
      tmem_ld32(tbase + lane_off + 128 + 32 * hh, reinterpret_cast<uint32_t*>(vv));
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        q[e] += P_[kPBQkvT + 32 * hh + e];
        kk_[e] += P_[kPBQkvT + 64 + 32 * hh + e];
        vv[e] += P_[kPBQkvT + 128 + 32 * hh + e];
      }
      float sc[8];
      float mx = -INFINITY;
      const int l0 = jl * nt;                        // lane of slice 0
#pragma unroll
      for (int ik = 0; ik < 8; ++ik) {
        if (ik >= nt) break;
        float acc = 0.f;
#pragma unroll
        for (int e = 0; e < 32; ++e) acc = fmaf(q[e], __shfl_sync(0xffffffffu, kk_[e], l0 + ik), acc);
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
#pragma unroll
      for (int e = 0; e < 32; ++e) q[e] = 0.f;        // q -> output accumulator
#pragma unroll
      for (int ik = 0; ik < 8; ++ik) {
        if (ik >= nt) break;
        const float p = sc[ik] * inv;
#pragma unroll
        for (int e = 0; e < 32; ++e) q[e] = fmaf(p, __shfl_sync(0xffffffffu, vv[e], l0 + ik), q[e]);
      }
      if (!row_live) {
#pragma unroll
        for (int e = 0; e < 32; ++e) q[e] = 0.f;
      }
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4)                 // head hh -> A columns [32hh, 32hh+32)
        *reinterpret_cast<uint4*>(A + (4 * hh + c4) * 2048 + m * 16) =
            make_uint4(pack_h2(q[8 * c4], q[8 * c4 + 1]), pack_h2(q[8 * c4 + 2], q[8 * c4 + 3]),
                       pack_h2(q[8 * c4 + 4], q[8 * c4 + 5]), pack_h2(q[8 * c4 + 6], q[8 * c4 + 7]));
    }
    // ---- 3. x += proj_t(o) ---------------------------------------------------
    TT(5);
    gemm_a(0, kOffProjT, 64);
    TT(6);
    add64(x, 0, P_ + kPBProjT);
    // ---- 4. h = GELU(fc1(LN_m(x))), written back to TMEM as fp16 pairs -----
    layernorm64(x, y, P_ + kPLnMw, P_ + kPLnMb);
    put_row64(A, m, y);
    TT(7);
    gemm_a(0, kOffFc1, 256);
    TT(8);
#pragma unroll 1
    // 8 chunks of 32 hidden units; the TMEM load of chunk c+1 is in flight
    // while chunk c is computed and stored (stores go to [16c, 16c+16), below
    // every chunk still to be loaded)
    {
      uint32_t ra[32], rb[32];
      auto gelu_store = [&](const uint32_t* r, int c8) {
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float2 g = gelu_as2(make_float2(__uint_as_float(r[e]) + P_[kPBFc1 + 32 * c8 + e],
                                                __uint_as_float(r[e + 1]) + P_[kPBFc1 + 32 * c8 + e + 1]));
          pk[e / 2] = pack_h2(g.x, g.y);
        }
        tmem_st16(tbase + lane_off + 16 * c8, pk);   // columns [16 c8, 16 c8 + 16)
      };
      tmem_ld32(tbase + lane_off, ra);
      tmem_wait_ld32(ra);
#pragma unroll 1
      for (int c8 = 0; c8 < 8; c8 += 2) {
        tmem_ld32(tbase + lane_off + 32 * (c8 + 1), rb);
        gelu_store(ra, c8);
        tmem_wait_ld32(rb);
        if (c8 + 2 < 8) tmem_ld32(tbase + lane_off + 32 * (c8 + 2), ra);
        gelu_store(rb, c8 + 1);
        if (c8 + 2 < 8) tmem_wait_ld32(ra);
      }
    }
    tmem_wait_st();
    TT(9);
    // ---- 5. x += fc2(h) (A from TMEM columns [0,128)), store x ---------------
    run([&] {
      const uint32_t idesc = idesc_f16(128, 64), lbo_b = 8 * 128;
      const uint32_t bbase = wb + kOffFc2 * 2;
      for (int kk = 0; kk < 16; ++kk)
        mma_ts_w(tbase + 128, tbase + kk * 8, sdesc(bbase + kk * 2 * lbo_b, 128, kSwizzleNone, lbo_b),
               idesc, kk != 0);
    });
    TT(10);
    add64(x, 128, P_ + kPBFc2);
    int qrow = s;
    if (a.qrank) qrow = valid ? a.qrank[b * a.ns + s] : -1;
    // a pruned next block reads the residual rows of masked positions only
    if (valid && qrow >= 0) {
      float4* xo = reinterpret_cast<float4*>(a.x + xrow);
#pragma unroll
      for (int q = 0; q < 16; ++q) xo[q] = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
    }
    // ---- 6. next block's LN_s + qkv_s -> bf16 attention operands ----------------
    layernorm64(x, y, P_ + kPLnSw, P_ + kPLnSb);
    put_row64(A, m, y);
    TT(11);
    gemm_a(0, kOffQkvS, 192);
    TT(12);
    // V^T stores in 4-byte pairs: lanes of adjacent positions (same slice)
    // swap one value per dimension pair, so position pair (2i, 2i+1) of dims
    // (e, e+1) goes out as two 32-bit stores instead of four 16-bit ones
    const bool pairs = (ppw & 1) == 0;
    const bool even = (jl & 1) == 0;
    const int partner = even ? lane + nt : lane - nt;
    const bool pair_ok = row_live && (s & ~1) < a.ns;
#pragma unroll 1
    for (int c6 = 0; c6 < 6; ++c6) {
      uint32_t r[32];
      tmem_ld32(tbase + lane_off + 32 * c6, r);
      tmem_wait_ld();
      const int which = c6 >> 1, head = c6 & 1;
      const size_t seq = size_t(b * nt + it) * 2 + head;
      float v[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]) + P_[kPBQkvN + 32 * c6 + e];
      if (which < 2) {
        if (!valid || (which == 0 && qrow < 0)) continue;
        uint4* d4 = reinterpret_cast<uint4*>((which == 0 ? a.qh : a.kh) +
                                             (seq * a.ns_pad + (which == 0 ? qrow : s)) * 32);
#pragma unroll
        for (int e = 0; e < 32; e += 8)
          d4[e / 8] = make_uint4(pack_bf16(v[e], v[e + 1]), pack_bf16(v[e + 2], v[e + 3]),
                                 pack_bf16(v[e + 4], v[e + 5]), pack_bf16(v[e + 6], v[e + 7]));
      } else if (pairs) {
        __nv_bfloat16* col = a.vth + seq * 32 * a.ns_pad + (s & ~1);
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float mine = even ? v[e] : v[e + 1];
          const float theirs = __shfl_sync(0xffffffffu, even ? v[e + 1] : v[e], partner);
          const uint32_t w = even ? pack_bf16(mine, theirs) : pack_bf16(theirs, mine);
          if (pair_ok)
            *reinterpret_cast<uint32_t*>(col + size_t(even ? e : e + 1) * a.ns_pad) = w;
        }
      } else if (valid) {
        __nv_bfloat16* dst = a.vth + seq * 32 * a.ns_pad + s;
#pragma unroll
        for (int e = 0; e < 32; ++e) dst[size_t(e) * a.ns_pad] = __float2bfloat16_rn(v[e]);
      }
    }
    // every thread's TMEM reads precede the next tile's first MMA (run()'s barrier)
    TT(15);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(sm.tmem_base);
  pdl_trigger();
}

}  // namespace

#ifdef NVREC_TRACE
int token_tc_trace(unsigned long long* host, int n) {
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  const int m = n < 32 ? n : 32;
  return cudaMemcpyFromSymbol(host, g_tc_trace, m * 8) == cudaSuccess ? m : -1;
}
#endif

bool token_tc_supported(const Dims& D) {
  return D.d == 64 && D.heads == 2 && D.nt <= 8 && D.hidden == 256;
}

cudaError_t launch_token_tc(const TokenTcArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(TokSmem) + 128;
  if (cudaError_t e = smem_optin(token_tc_kernel, int(smem))) return e;
  const int sms = sm_count();
  const int P = 4 * (32 / a.nt);
  const int tiles = ((a.ns + P - 1) / P) * a.b;
  const int ctas = (tiles + kSlots - 1) / kSlots;
  launch_seq(token_tc_kernel, ctas < sms ? ctas : sms, kThreads, smem, s, a);
  return cudaGetLastError();
}

}  // namespace nvrec
