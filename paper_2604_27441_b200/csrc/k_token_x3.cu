// k_token_x3.cu -- the fused block tail of a NON-LAST block on the PRECISE
// path (model.py:60-64, then the next block's :59/:37), on tcgen05 with
// fp32-class products: every GEMM operand is split a = a_hi + a_lo (fp16,
// weights pre-scaled by 2^s so their lo parts stay normal, TcW::blk3) and
// D = A_hi W_hi + A_hi W_lo + A_lo W_hi, fp32 accumulation; LayerNorm,
// softmax, GELU and the residual stay fp32.
//
// The split weights of one block tail (256 KB) do not fit in shared memory
// together, so the tail runs as three persistent phase kernels, each with its
// phase's weights resident and the fp32 residual x handed over in HBM:
//   phase 0   x += proj_s(ao);  x += proj_t(attn_t(qkv_t(LN_t(x))))   80 KB
//   phase 1   x += fc2(GELU(fc1(LN_m(x))))                             128 KB
//   phase 2   q,k,v = qkv_s'(LN_s'(x)) -> split bf16 attention operands  48 KB
// Tiles, slots and the per-warp position layout follow k_token_tc.cu (lane =
// j*nt + slice, the temporal attention is warp shuffles); every row is held
// by two threads (warps w and w + 4 of its slot, 32 columns each: one head of
// the temporal attention and of q/k/v), which doubles the warps that hide the
// TMEM / L2 latencies of this per-row work.  fc1 -> fc2 runs in
// two halves of 128 hidden units: fc1 half -> TMEM, GELU written back in place
// as fp16 [hi 32 | lo 32] column groups, fc2 reads them as the A operand from
// TMEM; the accumulator sits beside the half (192 of the slot's 256 columns).
#include "launch.cuh"
#include "x3_ops.cuh"

namespace nvrec {

namespace {

using namespace sm100;
using namespace x3;

constexpr int kSlots = 2;
// two threads per row: warps 8 slot + 4 hf + wq, hf = the row's column half
// (32 of the 64 columns; one head of the temporal attention / of q, k, v)
constexpr int kSlotThreads = 256;
constexpr int kThreads = kSlotThreads * kSlots;
// element offsets of the [hi | lo] packs inside one block's blk3 pack
constexpr uint32_t kX3ProjS = 0, kX3QkvT = 8192, kX3ProjT = 32768, kX3Fc1 = 40960,
                   kX3Fc2 = 73728, kX3QkvS = 106496, kX3Blk = 131072;
// weights resident per phase (halves) and their offset inside the block pack
__host__ __device__ constexpr uint32_t ph_elems(int ph) {
  return ph == 0 ? kX3Fc1 : (ph == 1 ? kX3QkvS - kX3Fc1 : kX3Blk - kX3QkvS);
}
__host__ __device__ constexpr uint32_t ph_base(int ph) {
  return ph == 0 ? 0u : (ph == 1 ? kX3Fc1 : kX3QkvS);
}
// staged parameter vectors (floats), as k_token_tc.cu
constexpr int kPBProjS = 0, kPLnTw = 64, kPLnTb = 128, kPBQkvT = 192, kPBProjT = 384,
              kPLnMw = 448, kPLnMb = 512, kPBFc1 = 576, kPBFc2 = 832, kPLnSw = 896,
              kPLnSb = 960, kPBQkvN = 1024, kParFloats = 1216;
template <int PH>
struct __align__(128) X3Smem {
  __half w[ph_elems(PH)];
  uint8_t a[kSlots][2 * kABytes];   // per slot: A_hi | A_lo
  float par[kParFloats];
  float2 red[kSlots][2][128];       // LayerNorm (mean, M2) of each row half
  uint64_t bar_w, bar_d[kSlots];
  uint32_t tmem_base;
};

#ifdef NVREC_TRACE
// phase timestamps of CTA 0, slot 0, its first two tiles (tools/trace_token.py)
__device__ unsigned long long g_tx_trace[3][2][16];
#define TX(i) \
  do { \
    if (blockIdx.x == 0 && threadIdx.x == 0 && ntile < 2) g_tx_trace[PH][ntile][i] = clock64(); \
  } while (0)
#else
#define TX(i) do {} while (0)
#endif

template <int PH>
__global__ void __launch_bounds__(kThreads, 1)
token_x3_kernel(TokenX3Args a) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem_raw[];
  using S = X3Smem<PH>;
  S& sm = *reinterpret_cast<S*>(smem_raw + ((128 - (smem_u32(smem_raw) & 127)) & 127));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = warp >> 3, hf = (warp >> 2) & 1, wq = warp & 3;   // tile slot, half, lane quarter
  const int nt = a.nt;
  const int ppw = 32 / nt;                          // whole positions per warp
  const int P = 4 * ppw;                            // positions per tile
  const int tiles_per_b = (a.ns + P - 1) / P;
  const int n_tiles = tiles_per_b * a.b;

  if (threadIdx.x == 0) {
    mbar_init(&sm.bar_w, 1);
    for (int k = 0; k < kSlots; ++k) mbar_init(&sm.bar_d[k], 1);
    fence_mbar_init();
    constexpr uint32_t bytes = ph_elems(PH) * 2;
    mbar_expect_tx(&sm.bar_w, bytes);
    const __half* src = (PH == 2 ? a.w_next : a.w_blk) + ph_base(PH);
    // bulk copies of <= 64 KB each
    for (uint32_t off = 0; off < bytes; off += 65536)
      bulk_load(reinterpret_cast<uint8_t*>(sm.w) + off, reinterpret_cast<const uint8_t*>(src) + off,
                bytes - off < 65536 ? bytes - off : 65536, &sm.bar_w);
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
  const int c0 = 32 * hf;                           // this thread's first column
  const uint32_t lane_off = uint32_t(wq * 32) << 16;
  const uint32_t tbase = sm.tmem_base + 256 * slot; // this slot's 256 columns
  const int jl = lane / nt, it = lane - jl * nt;    // position in warp, slice
  const bool row_live = jl < ppw;
  uint8_t* A = sm.a[slot];
  const uint32_t ab = smem_u32(A);
  const uint32_t wb = smem_u32(sm.w) - ph_base(PH) * 2;   // + element offset * 2 = a block pack matrix
  const bool issuer = wq == 0 && hf == 0;       // warp: one elected lane issues (*_w)
  auto slot_sync = [&] { asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(kSlotThreads) : "memory"); };
  uint32_t pd = 0;
  auto run = [&](auto issue) {
    fence_proxy_async();
    tc_fence_before();
    slot_sync();
    if (issuer) {
      tc_fence_after();
      issue();
      mma_commit_w(&sm.bar_d[slot]);
    }
    mbar_wait(&sm.bar_d[slot], pd & 1);
    ++pd;
    tc_fence_after();
  };
  // D[dcol..] (=) A(smem [hi|lo], K = 64) . W ([hi|lo] at element offset woff
  // of the block pack, N x 64, rows n0.. of an Nfull-row matrix)
  auto issue_a = [&](uint32_t dcol, uint32_t woff, int N, int Nfull, int n0) {
    const uint32_t idesc = idesc_f16(128, N), lbo_b = (Nfull / 8) * 128;
    const uint32_t bh = wb + woff * 2 + (n0 / 8) * 128, bl = bh + Nfull * 64 * 2;
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t ah = sdesc(ab + kk * 4096, 128, kSwizzleNone, 2048);
      const uint64_t al = sdesc(ab + kABytes + kk * 4096, 128, kSwizzleNone, 2048);
      const uint64_t wh = sdesc(bh + kk * 2 * lbo_b, 128, kSwizzleNone, lbo_b);
      const uint64_t wl = sdesc(bl + kk * 2 * lbo_b, 128, kSwizzleNone, lbo_b);
      mma_ss_w(tbase + dcol, ah, wh, idesc, kk != 0);
      mma_ss_w(tbase + dcol, ah, wl, idesc, 1);
      mma_ss_w(tbase + dcol, al, wh, idesc, 1);
    }
  };
  auto gemm_a = [&](uint32_t dcol, uint32_t woff, int N) {
    run([&] { issue_a(dcol, woff, N, N, 0); });
  };
  // x (this half) += D[32 cols at col + c0] * sc + bias
  auto add32 = [&](float* x, uint32_t col, float sc, const float* bias) {
    uint32_t r[32];
    tmem_ld32(tbase + lane_off + col + c0, r);
    tmem_wait_ld();
#pragma unroll
    for (int e = 0; e < 32; ++e) x[e] += fmaf(__uint_as_float(r[e]), sc, bias[c0 + e]);
  };
  // LayerNorm of the row's 64 values held as two halves by two threads: local
  // two-pass mean and M2 per half, one exchange, merged (Chan et al.) the same
  // way in both threads; the normalised half goes straight into the A operand
  float2* red = &sm.red[slot][0][0];
  auto ln_put = [&](const float* x, const float* g, const float* bt) {
    float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int e = 0; e < 32; ++e) s4[e & 3] += x[e];
    const float mh = ((s4[0] + s4[1]) + (s4[2] + s4[3])) * (1.f / 32.f);
    float q4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int e = 0; e < 32; ++e) q4[e & 3] = fmaf(x[e] - mh, x[e] - mh, q4[e & 3]);
    const float m2 = (q4[0] + q4[1]) + (q4[2] + q4[3]);
    red[hf * 128 + m] = make_float2(mh, m2);
    slot_sync();
    const float2 o = red[(hf ^ 1) * 128 + m];
    const float d = mh - o.x;
    const float mean = 0.5f * (mh + o.x);
    const float rstd = rsqrtf((m2 + o.y + 16.f * d * d) * (1.f / 64.f) + 1e-5f);
#pragma unroll
    for (int ki = 0; ki < 4; ++ki) {
      float y[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int e = 8 * ki + j;
        y[j] = (x[e] - mean) * rstd * g[c0 + e] + bt[c0 + e];
      }
      put_row_x3(A, m, y, 4 * hf + ki, 1);
    }
  };
  const float scale = rsqrtf(32.f);

  int ntile = 0;
  for (int tile = blockIdx.x * kSlots + slot; tile < n_tiles; tile += gridDim.x * kSlots, ++ntile) {
    TX(0);
    const int b = tile / tiles_per_b;
    const int s = (tile - b * tiles_per_b) * P + wq * ppw + jl;
    const bool valid = row_live && s < a.ns;
    const size_t xrow = (size_t(b * nt + it) * a.ns + s) * 64 + c0;
    float x[32];
    {
      const float4* xi = reinterpret_cast<const float4*>(a.x + xrow);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 u = valid ? xi[q] : make_float4(0.f, 0.f, 0.f, 0.f);
        x[4 * q] = u.x; x[4 * q + 1] = u.y; x[4 * q + 2] = u.z; x[4 * q + 3] = u.w;
      }
    }
    if constexpr (PH == 0) {
      // ---- x += proj_s(ao) ---------------------------------------------------
      {
        float y[32];
        const float4* ai = reinterpret_cast<const float4*>(a.ao + xrow);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 u = valid ? ai[q] : make_float4(0.f, 0.f, 0.f, 0.f);
          y[4 * q] = u.x; y[4 * q + 1] = u.y; y[4 * q + 2] = u.z; y[4 * q + 3] = u.w;
        }
        TX(1);
        put_row_x3(A, m, y, 4 * hf, 4);
      }
      gemm_a(0, kX3ProjS, 64);
      TX(2);
      add32(x, 0, a.sc[0], P_ + kPBProjS);
      // ---- qkv_t(LN_t(x)); temporal attention (head hf) by warp shuffles -------
      ln_put(x, P_ + kPLnTw, P_ + kPLnTb);
      TX(3);
      gemm_a(0, kX3QkvT, 192);
      TX(4);
      const float sq = a.sc[1];
      const int l0 = jl * nt;                          // lane of slice 0
      float sc[8];
#pragma unroll
      for (int ik = 0; ik < 8; ++ik) sc[ik] = 0.f;
#pragma unroll
      for (int c = 0; c < 2; ++c) {                    // 16 of the head's 32 dims at a time
        float q[16], kk_[16];
        tmem_ld16(tbase + lane_off + c0 + 16 * c, reinterpret_cast<uint32_t*>(q));
        tmem_ld16(tbase + lane_off + 64 + c0 + 16 * c, reinterpret_cast<uint32_t*>(kk_));
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          q[e] = fmaf(q[e], sq, P_[kPBQkvT + c0 + 16 * c + e]);
          kk_[e] = fmaf(kk_[e], sq, P_[kPBQkvT + 64 + c0 + 16 * c + e]);
        }
#pragma unroll
        for (int ik = 0; ik < 8; ++ik) {
          if (ik >= nt) break;
#pragma unroll
          for (int e = 0; e < 16; ++e) sc[ik] = fmaf(q[e], __shfl_sync(0xffffffffu, kk_[e], l0 + ik), sc[ik]);
        }
      }
      float mx = -INFINITY;
#pragma unroll
      for (int ik = 0; ik < 8; ++ik) {
        if (ik >= nt) break;
        sc[ik] *= scale;
        mx = fmaxf(mx, sc[ik]);
      }
      float den = 0.f;
#pragma unroll
      for (int ik = 0; ik < 8; ++ik) {
        if (ik >= nt) break;
        sc[ik] = expf(sc[ik] - mx);
        den += sc[ik];
      }
      const float inv = 1.f / den;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float vv[16], o[16];
        tmem_ld16(tbase + lane_off + 128 + c0 + 16 * c, reinterpret_cast<uint32_t*>(vv));
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          vv[e] = fmaf(vv[e], sq, P_[kPBQkvT + 128 + c0 + 16 * c + e]);
          o[e] = 0.f;
        }
#pragma unroll
        for (int ik = 0; ik < 8; ++ik) {
          if (ik >= nt) break;
          const float p = sc[ik] * inv;
#pragma unroll
          for (int e = 0; e < 16; ++e) o[e] = fmaf(p, __shfl_sync(0xffffffffu, vv[e], l0 + ik), o[e]);
        }
        if (!row_live) {
#pragma unroll
          for (int e = 0; e < 16; ++e) o[e] = 0.f;
        }
        put_row_x3(A, m, o, 4 * hf + 2 * c, 2);        // head hf -> A columns [32hf, 32hf+32)
      }
      // ---- x += proj_t(o) ------------------------------------------------------
      TX(5);
      gemm_a(0, kX3ProjT, 64);
      TX(6);
      add32(x, 0, a.sc[2], P_ + kPBProjT);
      if (valid) {
        float4* xo = reinterpret_cast<float4*>(a.x + xrow);
#pragma unroll
        for (int q = 0; q < 8; ++q) xo[q] = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
      }
    } else if constexpr (PH == 1) {
      // ---- x += fc2(GELU(fc1(LN_m(x)))) in two halves of 128 hidden units ------
      TX(1);
      ln_put(x, P_ + kPLnMw, P_ + kPLnMb);
      TX(2);
      const float s1 = a.sc[3], s2 = a.sc[4];
      // fc2 K step kk (16 hidden units of half H) from the TMEM column groups
      auto issue_fc2 = [&](int H) {
        const uint32_t idesc = idesc_f16(128, 64), lbo_b = 8 * 128;
        const uint32_t bh = wb + kX3Fc2 * 2, bl = bh + 64 * 256 * 2;
        for (int kk = 0; kk < 8; ++kk) {
          const int kg = 8 * H + kk;                    // global K16 step
          const uint32_t ah = tbase + (kk >> 2) * 64 + (kk & 3) * 8;
          const uint64_t wh = sdesc(bh + kg * 2 * lbo_b, 128, kSwizzleNone, lbo_b);
          const uint64_t wl = sdesc(bl + kg * 2 * lbo_b, 128, kSwizzleNone, lbo_b);
          mma_ts_w(tbase + 128, ah, wh, idesc, kg != 0);
          mma_ts_w(tbase + 128, ah, wl, idesc, 1);
          mma_ts_w(tbase + 128, ah + 32, wh, idesc, 1);
        }
      };
      // GELU of the fc1 half in TMEM cols [0,128) -> [hi 32 | lo 32] per 64;
      // this thread's group is g = hf (cols 64 hf ..)
#pragma unroll 1
      for (int H = 0; H < 2; ++H) {
        if (H == 0) run([&] { issue_a(0, kX3Fc1, 128, 256, 0); });
        else run([&] { issue_fc2(0); issue_a(0, kX3Fc1, 128, 256, 128); });
        TX(3 + 2 * H);
        const uint32_t gcol = tbase + lane_off + 64 * hf;
        const float* bias = P_ + kPBFc1 + 128 * H + 64 * hf;
        // values 0-31 -> hi pairs at cols 0-15 (stored at once), lo pairs at
        // cols 32-47 (stored once values 32-63 have been read)
        uint32_t r0[32], lo0[16];
        tmem_ld32(gcol, r0);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float2 g = gelu_as2(make_float2(fmaf(__uint_as_float(r0[e]), s1, bias[e]),
                                                fmaf(__uint_as_float(r0[e + 1]), s1, bias[e + 1])));
          split_h2(g.x, g.y, r0[e / 2], lo0[e / 2]);
        }
        tmem_st16(gcol, r0);
        uint32_t r1[32], lo1[16];
        tmem_ld32(gcol + 32, r1);
        tmem_wait_ld();
        tmem_st16(gcol + 32, lo0);
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float2 g = gelu_as2(make_float2(fmaf(__uint_as_float(r1[e]), s1, bias[32 + e]),
                                                fmaf(__uint_as_float(r1[e + 1]), s1, bias[33 + e])));
          split_h2(g.x, g.y, r1[e / 2], lo1[e / 2]);
        }
        tmem_st16(gcol + 16, r1);
        tmem_st16(gcol + 48, lo1);
        tmem_wait_st();
        TX(4 + 2 * H);
      }
      run([&] { issue_fc2(1); });
      TX(7);
      add32(x, 128, s2, P_ + kPBFc2);
      if (valid) {
        float4* xo = reinterpret_cast<float4*>(a.x + xrow);
#pragma unroll
        for (int q = 0; q < 8; ++q) xo[q] = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
      }
    } else {
      // ---- next block's LN_s + qkv_s -> split bf16 attention operands ----------
      TX(1);
      ln_put(x, P_ + kPLnSw, P_ + kPLnSb);
      TX(2);
      gemm_a(0, kX3QkvS, 192);
      TX(3);
      int qrow = s;
      if (a.qrank) qrow = valid ? a.qrank[b * a.ns + s] : -1;
      const float sq = a.sc[5];
      __nv_bfloat16* vt = reinterpret_cast<__nv_bfloat16*>(A);
      const int jpos = wq * ppw + jl;                 // position inside the tile
      const int head = hf;
      const size_t seq = size_t(b * nt + it) * 2 + head;
#pragma unroll 1
      for (int which = 0; which < 3; ++which) {       // q, k, v of head hf: 32 columns
        const int c6 = 2 * which + head;
        uint32_t r[32];
        tmem_ld32(tbase + lane_off + 32 * c6, r);
        tmem_wait_ld();
        if (!valid) continue;
        float v[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = fmaf(__uint_as_float(r[e]), sq, P_[kPBQkvN + 32 * c6 + e]);
        if (which < 2) {
          if (which == 0 && qrow < 0) continue;
          uint4* d4 = reinterpret_cast<uint4*>((which == 0 ? a.qh : a.kh) +
                                               (seq * a.ns_pad + (which == 0 ? qrow : s)) * 64);
#pragma unroll
          for (int e = 0; e < 32; e += 8) {
            uint32_t h[4], l[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) split_bf16(v[e + 2 * j], v[e + 2 * j + 1], h[j], l[j]);
            d4[e / 8] = make_uint4(h[0], h[1], h[2], h[3]);
            d4[4 + e / 8] = make_uint4(l[0], l[1], l[2], l[3]);
          }
        } else {
          // V^T rows (hi e, lo 32 + e) staged in the slot's A buffer (the qkv_s
          // MMA has consumed it) as [slice, head][64][position]
          __nv_bfloat16* st = vt + ((it * 2 + head) * 64) * P + jpos;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const __nv_bfloat16 h = __float2bfloat16_rn(v[e]);
            st[e * P] = h;
            st[(32 + e) * P] = __float2bfloat16_rn(v[e] - __bfloat162float(h));
          }
        }
      }
      // coalesced V^T stores: 8 consecutive positions (16 bytes) per store
      slot_sync();
      {
        const int s0 = (tile - b * tiles_per_b) * P;
        const int nvalid = min(P, a.ns - s0);
        const int cpr = (P + 7) / 8;                     // chunks per staged row
        const int rows = nt * 2 * 64;
        // thread u of the slot owns chunk u % cpr of rows u / cpr, + 256 / cpr,
        // ... (no division inside the loop)
        const int u = hf * 128 + m;
        const int rstep = kSlotThreads / cpr, ch = u % cpr, row0 = u / cpr;
        for (int row = row0; row0 < rstep && row < rows; row += rstep) {
          const int sl = row >> 6, e = row & 63;
          const size_t sq2 = size_t(b * nt + (sl >> 1)) * 2 + (sl & 1);
          __nv_bfloat16* dst = a.vth + (sq2 * 64 + e) * a.ns_pad + s0 + 8 * ch;
          const __nv_bfloat16* src = vt + row * P + 8 * ch;
          if ((P & 7) == 0 && 8 * ch + 8 <= nvalid) {
            *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
          } else {
            for (int k = 0; k < 8 && 8 * ch + k < nvalid; ++k) dst[k] = src[k];
          }
        }
      }
      // the staging buffer is the next tile's A operand
      slot_sync();
    }
    // every thread's TMEM reads precede the next tile's first MMA (run()'s barrier)
    TX(15);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(sm.tmem_base);
  pdl_trigger();
}

template <int PH>
cudaError_t launch_phase(const TokenX3Args& a, cudaStream_t s) {
  const size_t smem = sizeof(X3Smem<PH>) + 128;
  if (cudaError_t e = smem_optin(token_x3_kernel<PH>, int(smem))) return e;
  const int sms = sm_count();
  const int P = 4 * (32 / a.nt);
  const int tiles = ((a.ns + P - 1) / P) * a.b;
  const int ctas = (tiles + kSlots - 1) / kSlots;
  launch_seq(token_x3_kernel<PH>, ctas < sms ? ctas : sms, kThreads, smem, s, a);
  return cudaGetLastError();
}

}  // namespace

#ifdef NVREC_TRACE
int token_x3_trace(unsigned long long* host, int n) {
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  const int m = n < 96 ? n : 96;
  return cudaMemcpyFromSymbol(host, g_tx_trace, m * 8) == cudaSuccess ? m : -1;
}
#endif

cudaError_t launch_token_x3(const TokenX3Args& a, cudaStream_t s) {
  cudaError_t e;
  if ((e = launch_phase<0>(a, s)) != cudaSuccess) return e;
  if ((e = launch_phase<1>(a, s)) != cudaSuccess) return e;
  return launch_phase<2>(a, s);
}

}  // namespace nvrec
