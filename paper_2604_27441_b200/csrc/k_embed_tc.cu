// k_embed_tc.cu -- tcgen05 implicit-GEMM tubelet embedding (the "encoder
// convolution", model.py:73-74,111) fused with its epilogue (x/255 scale,
// bias, time_pos, mask-channel rank-1 term, model.py:102-114) and with block
// 0's LN_s + qkv_s projection (model.py:59 -> :37), for the u8 server path.
//
// CTA = 128 tokens = an 8 x 16 rectangle of patches of one (stream, time
// slice); 6 warps:
//   warp 4     producer: per K stage (tubelet frame tt, kPy patch rows) one 5-D
//              TMA box of raw u8 pixels [8 ih][2 py][16 iw][16*c bytes]
//              straight from the HWC planes (zero-filled past the frame edge)
//              and one bulk copy of the stage's fp16 weight block
//   warps 0-3  converters: u8 -> fp16 (exact: byte_perm into 1024+v, then
//              -1024) written as the UMMA A operand (no-swizzle K-major core
//              matrices); masked patches of the corrupted frame become zeros
//   warp 5     MMA: D[128 x 64] += A[128 x 32c] W^T per stage (fp32 in TMEM;
//              the u8 / u16 split variants: D[128 x 128] = A [W_hi ; W_lo]^T),
//              then the qkv GEMM [128 x 64] x [64 x 192] on the LN output
//   warps 0-3  epilogue: TMEM -> registers (one token row per thread),
//              x = acc/255 + bias + time_pos (+ sum of mask-channel weights),
//              store x (fp32), LayerNorm in registers -> fp16 A2, then
//              q/k/v + bias -> bf16 attention operands (Q, K rows; V^T).
// GEMM per token: K = 512c (c = 3: 1536), N = 64; the u8 planes are read
// once from HBM by TMA.
//
// X3 (precise path): fp32-class products.  Pixels are exact in fp16, so the
// embedding is pix . W_hi + pix . W_lo (two MMAs per K step against the
// [hi | lo] weight packs, TcW::emb3, scaled by 2^s); the LN output is split
// y = y_hi + y_lo and the qkv GEMM is y_hi W_hi + y_hi W_lo + y_lo W_hi.  x
// leaves in fp32; q/k/v leave as bf16 hi/lo pairs in the split attention
// layouts (QkvDst::x3).  One CTA per SM (the doubled rings take ~135 KB).
//
// 16-bit depth (nvrec_recover_u16): C == 2 reads each u16 pixel as its two
// bytes (lo, hi) -- exact in fp16 like u8 pixels -- against weights W (lo) and
// 256 W (hi) (TcW::emb16 / emb16_3), and the epilogue divides by 65535: the
// same GEMM as W . (u16 / 65535), with no conversion pass over the planes.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "launch.cuh"
#include "sm100.cuh"

namespace nvrec {

namespace {

using namespace sm100;

constexpr int kRows = 128;
constexpr int kTh = 8, kTw = 16;   // patch rectangle per CTA
constexpr int kThreads = 192;

// RGB: two CTAs per SM (<= ~113 KB of shared memory each), so one CTA's
// epilogue and qkv GEMM overlap the other's pixel stream; the qkv weights
// reuse the A ring and the LN output reuses the raw-pixel ring once the K loop
// is done.  A K stage is kPy patch rows of one tubelet frame: 2 for RGB
// (K = 96), 4 for depth (K = 64) so a depth stage is not dominated by its
// barrier round trip.
template <int C, bool X3 = false, bool F32 = false>
struct __align__(128) EmbSmem {
  static constexpr int kX = X3 ? 2 : 1;                      // hi (+ lo) operand copies
  // patch rows per K stage; the split-operand (X3) variants use half-size
  // stages so that two CTAs fit on an SM (<= ~113 KB of shared memory each).
  // F32 (float module API): a stage is 2 pixel rows of ONE channel (K = 32).
  static constexpr int kPy = F32 ? 2 : X3 ? (C == 1 ? 2 : 1) : (C == 1 ? 4 : 2);
  static constexpr int kSpt = 16 / kPy;                      // K stages per tubelet frame (u8)
  static constexpr int kNst = 2;
  static constexpr int kKst = F32 ? 32 : 16 * kPy * C;      // K per stage
  static constexpr uint32_t kU8_ = F32 ? kTh * kPy * kTw * 16 * 4 : kTh * kPy * kTw * 16 * C;
  // raw-pixel TMA ring: the X3 variants fill the region the LN output (A2,
  // 32 KB) needs anyway -- 5-8 stages in flight against HBM latency; the
  // float boxes are 16 KB (2 or 3 stages)
  static constexpr int kNu8 = F32 ? (X3 ? 2 : 3) : X3 ? int(32768 / kU8_) : (C == 1 ? 4 : 3);
  static constexpr uint32_t kU8 = kU8_;                     // raw bytes per stage
  static constexpr uint32_t kA1 = kRows * kKst * 2;         // fp16 A per stage, one copy
  static constexpr uint32_t kA = F32 ? kA1 * kX : kA1;      // F32 X3: A_hi | A_lo
  static constexpr uint32_t kW1 = 64 * kKst * 2;            // fp16 W per stage (one copy)
  static constexpr uint32_t kW = kW1 * kX;                  // [hi | lo]
  static constexpr uint32_t kQkvW1 = 192 * 64 * 2, kA21 = kRows * 64 * 2;
  static constexpr uint32_t kQkvW = kQkvW1 * kX, kA2 = kA21 * kX;
  // Weight ring.  The per-stage weight blocks come from L2 and bound the K
  // loop when only two are in flight (measured: the MMA waited ~600 clk per
  // stage); the u8 split variants keep four in flight and park the qkv
  // weights in the weight region after the K loop (the A ring shrinks to two
  // stages), which still fits two CTAs per SM.
  static constexpr bool kQkvInW = X3 && !F32;
  static constexpr int kNw = kQkvInW ? 4 : kNst;
  static constexpr uint32_t kWRegion = kQkvInW && kNw * kW < kQkvW ? kQkvW : kNw * kW;
  static constexpr uint32_t kARegion =
      kQkvInW ? kNst * kA : (kNst * kA > kQkvW ? kNst * kA : kQkvW);
  static constexpr uint32_t kURegion = kNu8 * kU8 > kA2 ? kNu8 * kU8 : kA2;
  uint8_t a_raw[kARegion];        // A ring (then the qkv weights unless kQkvInW)
  uint8_t w_raw[kWRegion];        // weight ring (then the qkv weights if kQkvInW)
  uint8_t u8_raw[kURegion];       // pixel ring, then: LN output (A2) [128 x 64] fp16, then V^T staging
  float par[64 * 5 + 192];        // bias | time_pos[it] | wmsum | ln_w | ln_b | qkv_b
  uint64_t u8_full[kNu8], u8_empty[kNu8], w_full[kNw], w_empty[kNw], aready[kNst], empty[kNst];
  uint64_t acc_full, wq_full, a2_ready, qkv_full;
  uint32_t tmem_base;
  int slot[16];
  __device__ uint8_t* a(int i) { return a_raw + i * kA; }
  __device__ uint8_t* w(int i) { return w_raw + i * kW; }
  __device__ uint8_t* qkvw() { return kQkvInW ? w_raw : a_raw; }
  __device__ uint8_t* u8(int i) { return u8_raw + i * kU8; }
};

// two CTAs per SM (<= 113.5 KB each incl. alignment slack and the 1 KB the
// runtime reserves per CTA) for every u8 / u16 variant and the split float one
static_assert(sizeof(EmbSmem<3, true>) + 128 <= 112 * 1024, "RGB X3 embed: two CTAs per SM");
static_assert(sizeof(EmbSmem<1, true>) + 128 <= 112 * 1024, "depth X3 embed: two CTAs per SM");
static_assert(sizeof(EmbSmem<2, true>) + 128 <= 112 * 1024, "u16 X3 embed: two CTAs per SM");
static_assert(sizeof(EmbSmem<3, false>) + 128 <= 112 * 1024, "RGB embed: two CTAs per SM");

__device__ __forceinline__ uint32_t u8x2_to_h2(uint32_t w, uint32_t sel) {
  uint32_t p = __byte_perm(w, 0x64646464u, sel);     // fp16 1024 + byte
  __half2 h = *reinterpret_cast<__half2*>(&p);
  h = __hsub2(h, __half2half2(__ushort_as_half(0x6400)));
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// bf16 hi/lo split of a pair: hi = bf16(p), lo = bf16(p - hi)
__device__ __forceinline__ void split_bf16(float x, float y, uint32_t& hi, uint32_t& lo) {
  hi = pack_bf16(x, y);
  const float2 h = unpack_bf16(hi);
  lo = pack_bf16(x - h.x, y - h.y);
}

#ifdef NVREC_TRACE
// CTA 0: MMA-thread timestamps per stage (0: start, 1: A ready, 2: W ready) and
// converter-warp-0 lane-0 timestamps (3: pixels ready), tools/trace_embed.py
__device__ unsigned long long g_emb_trace[64][4];
__device__ unsigned long long g_emb_trace_end[8];
#define ET(st, e) \
  do { if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (st) < 64) g_emb_trace[st][e] = clock64(); } while (0)
#define EE(i) \
  do { if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) g_emb_trace_end[i] = clock64(); } while (0)
#else
#define ET(st, e) do {} while (0)
#define EE(i) do {} while (0)
#endif

template <int C, bool X3, bool F32 = false>
__global__ void __launch_bounds__(kThreads, 1)
embed_tc_kernel(const __grid_constant__ CUtensorMap tm_u8, EmbedTcArgs a, TcW tcw) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem_raw[];
  using S = EmbSmem<C, X3, F32>;
  // pointer arithmetic (not integer casts) keeps the shared address space
  S& sm = *reinterpret_cast<S*>(smem_raw + ((128 - (smem_u32(smem_raw) & 127)) & 127));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_w = (a.nw + kTw - 1) / kTw;
  const int ih0 = (blockIdx.x / tiles_w) * kTh, iw0 = (blockIdx.x % tiles_w) * kTw;
  const int it = blockIdx.y, b = blockIdx.z;
  const int T = a.D.T;
  // F32: T x C x 8 image stages (2 rows of one channel of one sub-frame), then
  // 8 mask-channel stages on the last slice (model.py:105-107: the mask channel
  // is nonzero only in the stack's last frame)
  // u8 / u16 split variants: [W_hi ; W_lo] stacked into one N = 128 operand
  constexpr bool kStacked = X3 && !F32;
  const bool last_slice_cta = it == a.D.nt - 1;
  const int nimg = F32 ? T * C * 8 : T * S::kSpt;
  const int nst = nimg + (F32 && last_slice_cta ? 8 : 0);

  if (warp == 4 && lane == 0) {
    for (int i = 0; i < S::kNu8; ++i) {
      mbar_init(&sm.u8_full[i], 1);
      mbar_init(&sm.u8_empty[i], 128);
    }
    for (int i = 0; i < S::kNst; ++i) {
      mbar_init(&sm.aready[i], 128);
      mbar_init(&sm.empty[i], 1);
    }
    for (int i = 0; i < S::kNw; ++i) {
      mbar_init(&sm.w_full[i], 1);
      mbar_init(&sm.w_empty[i], 1);
    }
    mbar_init(&sm.acc_full, 1);
    mbar_init(&sm.wq_full, 1);
    mbar_init(&sm.a2_ready, 128);
    mbar_init(&sm.qkv_full, 1);
    fence_mbar_init();
    tma_prefetch(&tm_u8);
  }
  if (!F32 && threadIdx.x < T) sm.slot[threadIdx.x] = a.frame_index[b * a.D.F + it * T + threadIdx.x];
  if (F32 && threadIdx.x < T) {
    // front padding (model.py:99-101): stack frame fr comes from input frame
    // max(0, fr - (F - f_in))
    const int fr = it * T + threadIdx.x, src = max(0, fr - (a.D.F - a.f_in));
    sm.slot[threadIdx.x] = (b * a.f_in + src) * C;     // plane index of channel 0
  }
  for (int i = threadIdx.x; i < 64; i += blockDim.x) {
    sm.par[i] = a.emb_b[i];
    sm.par[64 + i] = a.time_pos[it * 64 + i];
    sm.par[128 + i] = a.emb_wmsum[i];
    sm.par[192 + i] = a.ln_w[i];
    sm.par[256 + i] = a.ln_b[i];
  }
  for (int i = threadIdx.x; i < 192; i += blockDim.x) sm.par[320 + i] = a.qkv_b[i];
  if (warp == 0) tmem_alloc<256>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 4) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      // raw pixels run up to S::kNu8 stages ahead: their slots free as soon as
      // the converters have read them
      for (int st = 0; st < nimg; ++st) {
        const int pu = st % S::kNu8;
        mbar_wait(&sm.u8_empty[pu], ((st / S::kNu8) & 1) ^ 1);
        mbar_expect_tx(&sm.u8_full[pu], S::kU8);
        if constexpr (F32) {
          // (256 px, 2 rows, 8 patch rows) of plane (b, frame, ch)
          const int tt = st / (C * 8), ch = (st / 8) % C, rp = st % 8;
          tma_load_4d(sm.u8(pu), &tm_u8, &sm.u8_full[pu], iw0 * 16, 2 * rp, ih0,
                      sm.slot[tt] + ch);
        } else {
          tma_load_5d(sm.u8(pu), &tm_u8, &sm.u8_full[pu], 0, iw0, S::kPy * (st % S::kSpt), ih0,
                      sm.slot[st / S::kSpt]);
        }
      }
    } else if (lane == 1) {
      // weights: their own ring of kNw stages (independent thread, own waits)
      for (int st = 0; st < nst; ++st) {
        const int ps = st % S::kNw;
        mbar_wait(&sm.w_empty[ps], ((st / S::kNw) & 1) ^ 1);
        mbar_expect_tx(&sm.w_full[ps], S::kW);
        // the host packs 2-row stages back to back, so kPy/2 of them are one
        // block (X3: one [hi | lo] pair per kernel stage)
        const __half* src =
            F32 ? (X3 ? tcw.embf3 : tcw.embf) + size_t(st) * (S::kW / 2)
            : C == 2 ? (X3 ? tcw.emb16_3 + size_t(st) * (S::kW / 2) : tcw.emb16 + size_t(st) * (S::kW / 2))
                   : (X3 ? tcw.emb3 + size_t(st) * (S::kW / 2)
                         : tcw.emb + size_t(st) * (S::kPy / 2) * tcw.emb_stage_elems);
        bulk_load(sm.w(ps), src, S::kW, &sm.w_full[ps]);
      }
      // qkv weights into the A ring / weight ring once the last embed MMA has read it
      mbar_wait(&sm.acc_full, 0);
      mbar_expect_tx(&sm.wq_full, S::kQkvW);
      bulk_load(sm.qkvw(), X3 ? tcw.qkv0_3 : tcw.qkv0, S::kQkvW, &sm.wq_full);
    }
  } else if (warp == 5) {
    // ---------------------------------------------------------------- MMA
    {   // the whole warp runs the loop; one elected lane issues (*_w)
      const uint32_t idesc = idesc_f16(128, 64), idesc128 = idesc_f16(128, 128);
      for (int st = 0; st < nst; ++st) {
        const int ps = st % S::kNst, pw = st % S::kNw;
        ET(st, 0);
        mbar_wait(&sm.aready[ps], (st / S::kNst) & 1);
        ET(st, 1);
        mbar_wait(&sm.w_full[pw], (st / S::kNw) & 1);
        ET(st, 2);
        tc_fence_after();
        const uint32_t ab = smem_u32(sm.a(ps)), wb = smem_u32(sm.w(pw));
#pragma unroll
        for (int kk = 0; kk < S::kKst / 16; ++kk) {
          const uint64_t ad = sdesc(ab + kk * 4096, 128, kSwizzleNone, 2048);
          if constexpr (kStacked) {
            // pixels are exact: pix . [W_hi ; W_lo] as one N = 128 MMA (the
            // stacked pack, LBO 2048); D[0,64) + D[64,128) in the epilogue
            mma_ss_w(tmem, ad, sdesc(wb + kk * 4096, 128, kSwizzleNone, 2048), idesc128,
                     (st | kk) != 0);
          } else {
            mma_ss_w(tmem, ad, sdesc(wb + kk * 2048, 128, kSwizzleNone, 1024), idesc, (st | kk) != 0);
            if (F32 && X3)   // float inputs: + x_hi . W_lo + x_lo . W_hi
              mma_ss_w(tmem, ad, sdesc(wb + S::kW1 + kk * 2048, 128, kSwizzleNone, 1024), idesc, 1);
            if (F32 && X3)
              mma_ss_w(tmem, sdesc(ab + S::kA1 + kk * 4096, 128, kSwizzleNone, 2048),
                       sdesc(wb + kk * 2048, 128, kSwizzleNone, 1024), idesc, 1);
          }
        }
        mma_commit_w(&sm.empty[ps]);
        mma_commit_w(&sm.w_empty[pw]);
      }
      mma_commit_w(&sm.acc_full);
      mbar_wait(&sm.wq_full, 0);
      mbar_wait(&sm.a2_ready, 0);
      tc_fence_after();
      const uint32_t idesc2 = idesc_f16(128, 192);
      const uint32_t a2b = smem_u32(sm.u8(0)), wqb = smem_u32(sm.qkvw());
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t yh = sdesc(a2b + kk * 4096, 128, kSwizzleNone, 2048);
        const uint64_t wh = sdesc(wqb + kk * 6144, 128, kSwizzleNone, 3072);
        mma_ss_w(tmem + 64, yh, wh, idesc2, kk != 0);
        if (X3) {   // y_hi W_lo + y_lo W_hi
          mma_ss_w(tmem + 64, yh, sdesc(wqb + S::kQkvW1 + kk * 6144, 128, kSwizzleNone, 3072),
                 idesc2, 1);
          mma_ss_w(tmem + 64, sdesc(a2b + S::kA21 + kk * 4096, 128, kSwizzleNone, 2048), wh,
                 idesc2, 1);
        }
      }
      mma_commit_w(&sm.qkv_full);
    }
  } else {
    // ------------------------------------------------- converters, then epilogue
    const int m = threadIdx.x;
    const int ihl = m >> 4, iwl = m & 15;
    const int ih = ih0 + ihl, iw = iw0 + iwl;
    const bool valid = ih < a.nh && iw < a.nw;
    const int s = valid ? ih * a.nw + iw : 0;
    const bool masked = !F32 && valid && a.rank[b * a.ns + s] >= 0;
    const bool last_slice = it == a.D.nt - 1;
    if constexpr (F32) {
      // float module API: stage = 2 pixel rows of one channel; the corrupted
      // (last) frame is multiplied by (1 - mask) (model.py:108-109); the mask
      // channel is its own 8 stages (model.py:105-107)
      const uint8_t* mrow = a.pmask + size_t(b) * a.h * a.w;
      for (int st = 0; st < nst; ++st) {
        const int ps = st % S::kNst, pu = st % S::kNu8;
        const bool img = st < nimg;
        if (img) mbar_wait(&sm.u8_full[pu], (st / S::kNu8) & 1);
        if (st >= S::kNst) mbar_wait(&sm.empty[ps], ((st / S::kNst) & 1) ^ 1);
        const int tt = img ? st / (C * 8) : T - 1, rp = img ? st % 8 : st - nimg;
        const bool corrupted = last_slice && tt == T - 1;
        uint8_t* arow = sm.a(ps) + m * 16;
#pragma unroll
        for (int pyl = 0; pyl < 2; ++pyl) {
          const int y = ih * 16 + 2 * rp + pyl;
          uint4 mk = make_uint4(0u, 0u, 0u, 0u);
          if (valid && (corrupted || !img))
            mk = __ldg(reinterpret_cast<const uint4*>(mrow + size_t(y) * a.w + iw * 16));
          const uint32_t mw[4] = {mk.x, mk.y, mk.z, mk.w};
          float v[16];
          if (img) {
            const float4* src = reinterpret_cast<const float4*>(
                sm.u8(pu) + ((ihl * 2 + pyl) * 256 + iwl * 16) * 4);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 u = src[q];
              v[4 * q] = u.x; v[4 * q + 1] = u.y; v[4 * q + 2] = u.z; v[4 * q + 3] = u.w;
            }
            if (corrupted) {
#pragma unroll
              for (int e = 0; e < 16; ++e)
                if ((mw[e >> 2] >> (8 * (e & 3))) & 0xFFu) v[e] = 0.f;
            }
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = ((mw[e >> 2] >> (8 * (e & 3))) & 0xFFu) ? 1.f : 0.f;
          }
#pragma unroll
          for (int kh = 0; kh < 2; ++kh) {             // K chunk pyl * 2 + kh: 8 pixels
            uint32_t hi[4], lo[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              hi[j] = pack_h2(v[8 * kh + 2 * j], v[8 * kh + 2 * j + 1]);
              if (X3) {
                const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&hi[j]));
                lo[j] = pack_h2(v[8 * kh + 2 * j] - hf.x, v[8 * kh + 2 * j + 1] - hf.y);
              }
            }
            const int ki = pyl * 2 + kh;
            *reinterpret_cast<uint4*>(arow + ki * 2048) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
            if (X3)
              *reinterpret_cast<uint4*>(arow + S::kA1 + ki * 2048) =
                  make_uint4(lo[0], lo[1], lo[2], lo[3]);
          }
        }
        if (img) mbar_arrive(&sm.u8_empty[pu]);
        fence_proxy_async();
        mbar_arrive(&sm.aready[ps]);
      }
    }
    for (int st = 0; !F32 && st < nst; ++st) {
      const int ps = st % S::kNst, pu = st % S::kNu8;
      mbar_wait(&sm.u8_full[pu], (st / S::kNu8) & 1);
      if (threadIdx.x == 0) ET(st, 3);
      if (st >= S::kNst) mbar_wait(&sm.empty[ps], ((st / S::kNst) & 1) ^ 1);   // A slot drained
      const bool zero = last_slice && (st / S::kSpt) == T - 1 && masked;   // corrupted frame
      uint8_t* arow = sm.a(ps) + m * 16;
#pragma unroll
      for (int pyl = 0; pyl < S::kPy; ++pyl) {
        const uint4* src =
            reinterpret_cast<const uint4*>(sm.u8(pu) + ((ihl * S::kPy + pyl) * kTw + iwl) * 16 * C);
#pragma unroll
        for (int q = 0; q < C; ++q) {
          uint4 v = zero ? make_uint4(0, 0, 0, 0) : src[q];
          const int ki = (pyl * 16 * C + q * 16) / 8;
          uint4 h0, h1;
          h0.x = u8x2_to_h2(v.x, 0x4140); h0.y = u8x2_to_h2(v.x, 0x4342);
          h0.z = u8x2_to_h2(v.y, 0x4140); h0.w = u8x2_to_h2(v.y, 0x4342);
          h1.x = u8x2_to_h2(v.z, 0x4140); h1.y = u8x2_to_h2(v.z, 0x4342);
          h1.z = u8x2_to_h2(v.w, 0x4140); h1.w = u8x2_to_h2(v.w, 0x4342);
          *reinterpret_cast<uint4*>(arow + ki * 2048) = h0;
          *reinterpret_cast<uint4*>(arow + (ki + 1) * 2048) = h1;
        }
      }
      mbar_arrive(&sm.u8_empty[pu]);        // raw pixels consumed
      fence_proxy_async();
      mbar_arrive(&sm.aready[ps]);
    }
    // ---- epilogue 1: x = acc/255 + bias + time_pos (+ mask term) ------------
    const uint32_t lane_off = uint32_t(warp * 32) << 16;
    EE(0);
    mbar_wait(&sm.acc_full, 0);
    EE(1);
    tc_fence_after();
    float x[64];
    {
      uint32_t r[32];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        tmem_ld32(tmem + lane_off + 32 * h, r);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) x[32 * h + j] = __uint_as_float(r[j]);
        if constexpr (kStacked) {       // + pix . W_lo (columns 64..127)
          tmem_ld32(tmem + lane_off + 64 + 32 * h, r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) x[32 * h + j] += __uint_as_float(r[j]);
        }
      }
    }
    const bool mterm = !F32 && last_slice && masked;   // F32: the mask channel is in the GEMM
    // (X3: the weights were scaled by 2^s; 2^-s / 255 is exactly 2^-s fl(1/255));
    // u16 depth (C == 2: byte pairs, hi-byte weights x 256) is / 65535; float
    // stacks are already in [0, 1]
    const float pix_inv = F32 ? 1.f : C == 2 ? 1.f / 65535.f : 1.f / 255.f;
    const float inv255 =
        X3 ? (F32 ? tcw.sc_embf : C == 2 ? tcw.sc_emb16 : tcw.sc_emb) * pix_inv : pix_inv;
#pragma unroll
    for (int o = 0; o < 64; ++o) {
      float v = fmaf(x[o], inv255, sm.par[o]);
      if (mterm) v += sm.par[128 + o];
      x[o] = v + sm.par[64 + o];
    }
    if (valid && a.xh && !X3) {
      uint4* xo = reinterpret_cast<uint4*>(a.xh + (size_t(b * a.D.nt + it) * a.ns + s) * 64);
#pragma unroll
      for (int o = 0; o < 64; o += 8)
        xo[o / 8] = make_uint4(pack_h2(x[o], x[o + 1]), pack_h2(x[o + 2], x[o + 3]),
                               pack_h2(x[o + 4], x[o + 5]), pack_h2(x[o + 6], x[o + 7]));
    } else if (valid) {
      float4* xo = reinterpret_cast<float4*>(a.x + (size_t(b * a.D.nt + it) * a.ns + s) * 64);
#pragma unroll
      for (int o = 0; o < 64; o += 4) xo[o / 4] = make_float4(x[o], x[o + 1], x[o + 2], x[o + 3]);
    }
    // ---- LN_s (block 0) in registers -> fp16 A2 -----------------------------
    float mean = 0.f;
#pragma unroll
    for (int o = 0; o < 64; ++o) mean += x[o];
    mean *= (1.f / 64.f);
    float var = 0.f;
#pragma unroll
    for (int o = 0; o < 64; ++o) var = fmaf(x[o] - mean, x[o] - mean, var);
    const float rstd = rsqrtf(var * (1.f / 64.f) + 1e-5f);
    uint8_t* a2row = sm.u8(0) + m * 16;   // every pixel stage has been consumed
#pragma unroll
    for (int ki = 0; ki < 8; ++ki) {
      float y[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int o = ki * 8 + j;
        y[j] = (x[o] - mean) * rstd * sm.par[192 + o] + sm.par[256 + o];
      }
      uint32_t hi[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) hi[j] = pack_h2(y[2 * j], y[2 * j + 1]);
      *reinterpret_cast<uint4*>(a2row + ki * 2048) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      if (X3) {
        uint32_t lo[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 h = __half22float2(*reinterpret_cast<const __half2*>(&hi[j]));
          lo[j] = pack_h2(y[2 * j] - h.x, y[2 * j + 1] - h.y);
        }
        *reinterpret_cast<uint4*>(a2row + S::kA21 + ki * 2048) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
    }
    fence_proxy_async();
    tc_fence_before();     // the accumulator reads precede the qkv MMA (it reuses columns 64..127)
    mbar_arrive(&sm.a2_ready);
    EE(2);
    // ---- epilogue 2: q, k, v (+ bias) -> bf16 attention operands -----------
    // V^T staging over the LN output (A2), which the finished qkv MMA has read
    constexpr int kVtR = X3 ? 64 : 32;                 // V^T rows per head
    __nv_bfloat16* vst = reinterpret_cast<__nv_bfloat16*>(sm.u8(0));
    static_assert(2 * kVtR * kRows * 2 <= S::kURegion, "V^T staging fits the A2 region");
    mbar_wait(&sm.qkv_full, 0);
    EE(3);
    tc_fence_after();
    int qrow = s;
    if (a.qrank) qrow = valid ? a.qrank[b * a.ns + s] : -1;
#pragma unroll 1
    for (int c6 = 0; c6 < 6; ++c6) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_off + 64 + 32 * c6, r);
      tmem_wait_ld();
      if (!valid) continue;
      const int which = c6 >> 1, head = c6 & 1;
      const size_t seq = size_t(b * a.D.nt + it) * 2 + head;
      float v[32];
      const float qs = X3 ? tcw.sc_qkv0 : 1.f;
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] = fmaf(__uint_as_float(r[e]), qs, sm.par[320 + 32 * c6 + e]);
      if (X3) {
        // bf16 hi/lo pairs: Q/K rows [hi 32 | lo 32], V^T rows e (hi), 32 + e (lo)
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
          // V^T rows e (hi) and 32 + e (lo), staged per token (coalesced below)
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const __nv_bfloat16 h = __float2bfloat16_rn(v[e]);
            vst[(head * kVtR + e) * kRows + m] = h;
            vst[(head * kVtR + 32 + e) * kRows + m] = __float2bfloat16_rn(v[e] - __bfloat162float(h));
          }
        }
        continue;
      }
      if (which < 2) {
        if (which == 0 && qrow < 0) continue;
        __nv_bfloat16* dst = (which == 0 ? a.qh : a.kh) +
                             (seq * a.ns_pad + (which == 0 ? qrow : s)) * 32;
        uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
        for (int e = 0; e < 32; e += 8)
          d4[e / 8] = make_uint4(pack_bf16(v[e], v[e + 1]), pack_bf16(v[e + 2], v[e + 3]),
                                 pack_bf16(v[e + 4], v[e + 5]), pack_bf16(v[e + 6], v[e + 7]));
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) vst[(head * kVtR + e) * kRows + m] = __float2bfloat16_rn(v[e]);
      }
    }
    // V^T: the tile's 8 patch rows of 16 positions per (head, row), 16 bytes
    // (8 positions) per store instead of one 2-byte store per element
    asm volatile("bar.sync 1, 128;" ::: "memory");
    for (int idx = m; idx < 2 * kVtR * 16; idx += kRows) {
      const int half = idx & 1, r = (idx >> 1) & 7, row = idx >> 4;   // row = head * kVtR + e
      const int head = row / kVtR, e = row - head * kVtR;
      const int ihr = ih0 + r, iwc = iw0 + 8 * half;
      if (ihr >= a.nh || iwc >= a.nw) continue;
      const int s0 = ihr * a.nw + iwc;
      const size_t seq = size_t(b * a.D.nt + it) * 2 + head;
      __nv_bfloat16* dst = a.vth + (seq * kVtR + e) * a.ns_pad + s0;
      const __nv_bfloat16* src = vst + row * kRows + r * 16 + 8 * half;
      if (iwc + 8 <= a.nw && (s0 & 7) == 0) {
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
      } else {
        for (int k = 0; k < 8 && iwc + k < a.nw; ++k) dst[k] = src[k];
      }
    }
  }
  EE(4);
  tc_fence_before();
  __syncthreads();
  EE(5);
  if (warp == 0) tmem_dealloc<256>(tmem);
  pdl_trigger();
}

#ifdef NVREC_TRACE
}  // namespace
int embed_trace(unsigned long long* host, int n) {
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  if (cudaMemcpyFromSymbol(host, g_emb_trace, 64 * 4 * 8) != cudaSuccess) return -1;
  if (n > 256 && cudaMemcpyFromSymbol(host + 256, g_emb_trace_end, 8 * 8) != cudaSuccess) return -1;
  return n;
}
namespace {
#endif

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

template <int C, bool X3>
cudaError_t launch_c(const EmbedTcArgs& a, cudaStream_t s) {
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  // u8 HWC planes viewed as (16c bytes, iw, py, ih, slot)
  CUtensorMap tm;
  cuuint64_t dims[5] = {cuuint64_t(16 * C), cuuint64_t(a.nw), 16, cuuint64_t(a.nh),
                        cuuint64_t(a.n_slots)};
  cuuint64_t strides[4] = {cuuint64_t(16 * C), cuuint64_t(a.w) * C, cuuint64_t(16) * a.w * C,
                           cuuint64_t(a.h) * a.w * C};
  cuuint32_t box[5] = {cuuint32_t(16 * C), kTw, EmbSmem<C, X3>::kPy, kTh, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  if (fn(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, const_cast<uint8_t*>(a.frames), dims, strides,
         box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const size_t smem = sizeof(EmbSmem<C, X3>) + 128;
  if (cudaError_t e = smem_optin(embed_tc_kernel<C, X3>, int(smem))) return e;
  const int tiles = ((a.nh + kTh - 1) / kTh) * ((a.nw + kTw - 1) / kTw);
  launch_seq(embed_tc_kernel<C, X3>, dim3(tiles, a.D.nt, a.b), kThreads, smem, s, tm, a, *a.tcw);
  return cudaGetLastError();
}

}  // namespace

bool embed_tc_supported(const Dims& D) {
  return D.p == 16 && D.d == 64 && D.heads == 2 && (D.c == 1 || D.c == 3) && D.T <= 2;
}

// float module API: stack (b, f_in, c, h, w) planes viewed as (w, 16 rows,
// h/16 patch rows, plane) with boxes of (256 px, 2 rows, 8 patch rows)
template <int C, bool X3>
cudaError_t launch_f32(const EmbedTcArgs& a, cudaStream_t s) {
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  CUtensorMap tm;
  cuuint64_t dims[4] = {cuuint64_t(a.w), 16, cuuint64_t(a.nh), cuuint64_t(a.b) * a.f_in * C};
  cuuint64_t strides[3] = {cuuint64_t(a.w) * 4, cuuint64_t(16) * a.w * 4,
                           cuuint64_t(a.h) * a.w * 4};
  cuuint32_t box[4] = {cuuint32_t(kTw * 16), 2, kTh, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  if (fn(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(a.stack), dims, strides,
         box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const size_t smem = sizeof(EmbSmem<C, X3, true>) + 128;
  if (cudaError_t e = smem_optin(embed_tc_kernel<C, X3, true>, int(smem))) return e;
  const int tiles = ((a.nh + kTh - 1) / kTh) * ((a.nw + kTw - 1) / kTw);
  launch_seq(embed_tc_kernel<C, X3, true>, dim3(tiles, a.D.nt, a.b), kThreads, smem, s, tm, a,
             *a.tcw);
  return cudaGetLastError();
}

cudaError_t launch_embed_tc(const EmbedTcArgs& a, cudaStream_t s) {
  if (a.f32) {
    if (a.x3) return a.D.c == 3 ? launch_f32<3, true>(a, s) : launch_f32<1, true>(a, s);
    return a.D.c == 3 ? launch_f32<3, false>(a, s) : launch_f32<1, false>(a, s);
  }
  // 16-bit depth: the u16 plane is read as byte pairs (lo, hi), i.e. a
  // two-"channel" u8 image whose hi-byte weights carry the factor 256
  if (a.u16) return a.x3 ? launch_c<2, true>(a, s) : launch_c<2, false>(a, s);
  if (a.x3) return a.D.c == 3 ? launch_c<3, true>(a, s) : launch_c<1, true>(a, s);
  return a.D.c == 3 ? launch_c<3, false>(a, s) : launch_c<1, false>(a, s);
}

}  // namespace nvrec
