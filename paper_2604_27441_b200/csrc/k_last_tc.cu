// k_last_tc.cu -- the LAST transformer block, the final LayerNorm and the
// head (model.py:59-64 for block L-1, then :117-122) on tcgen05, for the
// masked patches only (exact pruning: only the last
// time slice reaches the head, and the merge keeps only masked patches,
// server.py:196).  Replaces the CUDA-core token_kernel<narrow>, whose cost
// grew linearly with the masked-patch count (563 us per 8 x 720p launch at
// 20 % block loss).
//
// Layout.  One tile = up to 128 masked positions gathered ACROSS streams (a
// prefix sum over the per-stream counts), tile row == TMEM lane.  The CTA has
// 16 warps: warp w serves TMEM lane quarter w % 4 (rows 32(w%4)..+31) and
// column group cg = w / 4, so each row is worked on by four threads, one per
// 16-column slice of the 64-wide rows (and per quarter of the wide GELU / head
// epilogues).  Row reductions (LayerNorm, temporal scores) are exchanged
// through shared memory.  Per tile:
//
//   proj_s    x_t += proj_s(ao_t)            t = 0..nt-1 (nt A operands)
//   qkv_t     LN_t(x_t) -> q|k|v of the last slice, k|v of the others
//   attn_t    last-slice query over the nt keys (a thread owns 16 dims of one
//             head; partial scores exchanged with its partner)
//   proj_t    x += proj_t(o)                 last slice only
//   mlp       x += fc2(GELU(fc1(LN_m(x))))   fc1 halves -> GELU -> TMEM (fp16
//             hi|lo) -> fc2 reads its A operand from TMEM
//   head      y = LN(x); sigmoid(head(y)) in 4 column chunks of 4 patch rows
//             (64c columns; thread cg owns patch row 4j + cg of chunk j), the
//             MMA of chunk j+1 overlapping the epilogue of chunk j; quantised
//             with numpy's two float32 roundings (server.py:194), 16 bytes per
//             store into the merged plane
//
// Every product is fp32-class: split fp16 operands (weights pre-scaled by
// 2^s, TcW::last3 / head3) and D = A_hi W_hi + A_hi W_lo + A_lo W_hi with fp32
// accumulation; LayerNorm, softmax, GELU (erf) and the residual stay fp32.
// The split weights (336 KB for RGB) stream through a two-stage 48 KB
// shared-memory ring (cp.async.bulk from L2), each chunk issued as soon as the
// previous user of its stage retired.  The attention's key-split partials
// arrive merged (attn_combine_kernel).  Few masked patches (few tiles): 2 or
// 4 CTAs share a tile, each repeating the block tail and running a disjoint
// subset of the head chunks, which halves / quarters the per-tile latency
// chain where the GPU would otherwise idle.
#include "launch.cuh"
#include "x3_ops.cuh"

namespace nvrec {

namespace {

using namespace sm100;
using namespace x3;

constexpr int kThreads = 512;
constexpr int kNtMax = 3;           // TMEM: (nt-1) x 128 + 192 columns <= 512
constexpr int kMaxStreams = 256;
constexpr uint32_t kStage = 49152;  // bytes per weight-ring stage
constexpr int kBlkChunks = 7;       // proj_s, qkv_t, proj_t, fc1 x 2, fc2 x 2
// [hi | lo] elements of the last3 chunks
__host__ __device__ constexpr uint32_t blk_chunk_elems(int k) {
  return k == 0 ? 8192u : k == 1 ? 24576u : k == 2 ? 8192u : 16384u;
}

struct __align__(128) LastSmem {
  uint8_t w[2][kStage];
  uint8_t a[kNtMax][2 * kABytes];   // per slice: A_hi | A_lo
  float4 red[2][kNtMax][128];       // per-row partials, one float per column group
  uint64_t bar_w[2], bar_d, bar_h[2];
  uint32_t tmem_base;
  int n_tiles, rows, hsplit;
  int pref[kMaxStreams + 1];
};

__device__ __forceinline__ void chunk_src(const LastTcArgs& a, int k, const uint8_t*& src,
                                          uint32_t& bytes) {
  if (k < kBlkChunks) {
    uint32_t off = 0;
    for (int i = 0; i < k; ++i) off += blk_chunk_elems(i);
    src = reinterpret_cast<const uint8_t*>(a.w_blk + off);
    bytes = blk_chunk_elems(k) * 2;
  } else {
    const uint32_t hb = uint32_t(a.c) * 64 * 64 * 2 * 2;   // [hi | lo] 64c x 64 fp16
    src = reinterpret_cast<const uint8_t*>(a.w_head) + size_t(k - kBlkChunks) * hb;
    bytes = hb;
  }
}

// 16 fp32 values -> columns [8 k0, 8 k0 + 16) of row m of a [hi | lo] A operand
__device__ __forceinline__ void put16_x3(uint8_t* base, int m, const float* y, int k0) {
#pragma unroll
  for (int ki = 0; ki < 2; ++ki) {
    uint32_t h[4], l[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) split_h2(y[8 * ki + 2 * j], y[8 * ki + 2 * j + 1], h[j], l[j]);
    *reinterpret_cast<uint4*>(base + (k0 + ki) * 2048 + m * 16) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(base + kABytes + (k0 + ki) * 2048 + m * 16) =
        make_uint4(l[0], l[1], l[2], l[3]);
  }
}

__device__ __forceinline__ float sum4(float4 v) { return (v.x + v.y) + (v.z + v.w); }
__device__ __forceinline__ float comp(float4 v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}
__device__ __forceinline__ void set_comp(float4* p, int i, float v) {
  reinterpret_cast<float*>(p)[i] = v;
}

#ifdef NVREC_TRACE
__device__ unsigned long long g_last_trace[64];
#define LT(i) \
  do { if (blockIdx.x == 0 && threadIdx.x == 0) g_last_trace[i] = clock64(); } while (0)
#else
#define LT(i) do {} while (0)
#endif

// sigmoid on MUFU without branches: ex2.approx (rel. err ~2^-22) and
// rcp.approx refined by one Newton step (~1 ulp); z is clamped at -80 so
// 1 + e^-z stays finite.  |error| < 3e-7 for |z| < 20, below the precise
// path's 1.5e-5 bar.
__device__ __forceinline__ float sigmoid_fast(float z) {
  const float d = 1.f + ex2(-1.4426950408889634f * fmaxf(z, -80.f));
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
  return fmaf(r, fmaf(-d, r, 1.f), r);
}

template <int NT, int C>
__global__ void __launch_bounds__(kThreads, 1)
last_tc_kernel(LastTcArgs a) {
  pdl_wait();
  LT(0);
  extern __shared__ __align__(128) uint8_t smem_raw[];
  LastSmem& sm =
      *reinterpret_cast<LastSmem*>(smem_raw + ((128 - (smem_u32(smem_raw) & 127)) & 127));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wq = warp & 3, cg = warp >> 2;          // lane quarter, column group
  const int m = wq * 32 + lane;                     // tile row == TMEM lane
  const uint32_t lane_off = uint32_t(wq * 32) << 16;
  constexpr int nt = NT, c = C;
  const bool t0 = threadIdx.x == 0;
  const int c0 = 16 * cg;                           // this thread's 16 columns

  if (t0) {
    mbar_init(&sm.bar_w[0], 1);
    mbar_init(&sm.bar_w[1], 1);
    mbar_init(&sm.bar_d, 1);
    mbar_init(&sm.bar_h[0], 1);
    mbar_init(&sm.bar_h[1], 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    // rows of stream b are [pref[b], pref[b+1]) of the gathered row space
    int run = 0;
#pragma unroll 1
    for (int b0 = 0; b0 < a.b; b0 += 32) {
      const int bi = b0 + lane;
      int v = bi < a.b ? (a.count ? a.count[bi] : a.ns) : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (bi < a.b) sm.pref[bi + 1] = run + v;
      run += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) {
      sm.pref[0] = 0;
      // spread the rows over the grid: 32..128 rows per tile; when tiles are
      // fewer than CTAs, 2 or 4 CTAs share a tile, each running the block
      // tail and a disjoint subset of the 4 head chunks
      int rows = (run + int(gridDim.x) - 1) / int(gridDim.x);
      rows = min(128, max(32, (rows + 31) & ~31));
      const int tiles = (run + rows - 1) / rows;
      const int per = tiles > 0 ? int(gridDim.x) / tiles : 1;
      sm.rows = rows;
      sm.n_tiles = tiles;
      const int cap = min(per, a.max_hsplit);
      sm.hsplit = cap >= 4 ? 4 : cap >= 2 ? 2 : 1;
    }
  }
  if (warp == 0) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  LT(1);
  const int n_tiles = sm.n_tiles, rows = sm.rows, total = sm.pref[a.b], hsplit = sm.hsplit;
  const int nh = 4 / hsplit;                        // head chunks per work item
  const int per_item = kBlkChunks + nh;             // weight chunks per work item
  const int n_items = n_tiles * hsplit;             // item = tile * hsplit + head part
  const uint32_t tbase = sm.tmem_base;
  const int my_items =
      int(blockIdx.x) < n_items ? (n_items - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;
  const int n_chunks = my_items * per_item;

  // ---- weight ring: chunk ci lives in stage ci & 1 --------------------------------
  auto load_chunk = [&](int ci) {      // thread 0, once the stage's last reader retired
    if (ci >= n_chunks) return;
    const uint8_t* src;
    uint32_t bytes;
    const int k = ci % per_item;
    const int hpart = (int(blockIdx.x) + (ci / per_item) * int(gridDim.x)) % hsplit;
    chunk_src(a, k < kBlkChunks ? k : kBlkChunks + hpart + hsplit * (k - kBlkChunks), src, bytes);
    uint64_t* bar = &sm.bar_w[ci & 1];
    mbar_expect_tx(bar, bytes);
    bulk_load(sm.w[ci & 1], src, bytes, bar);
  };
  auto wait_chunk = [&](int ci) { mbar_wait_fast(&sm.bar_w[ci & 1], (ci >> 1) & 1); };
  auto wsm = [&](int ci) { return smem_u32(sm.w[ci & 1]); };
  if (t0) {
    load_chunk(0);
    load_chunk(1);
  }

  uint32_t pd = 0, ph0 = 0, ph1 = 0;
  auto sync_mma = [&]() {              // operands written by every thread -> MMA issue
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  };
  const bool w0 = warp == 0;            // MMA issue: warp 0, one elected lane (*_w)
  auto run = [&](auto issue) {
    sync_mma();
    if (w0) {
      issue();
      mma_commit_w(&sm.bar_d);
    }
    mbar_wait(&sm.bar_d, pd & 1);
    ++pd;
    tc_fence_after();
  };
  // D[dcol..] (=) A_j (smem [hi|lo], K = 64) . W (smem [hi|lo] at w, N x 64)
  auto issue_a = [&](int j, uint32_t dcol, uint32_t w, int N) {
    const uint32_t ab = smem_u32(sm.a[j]);
    const uint32_t idesc = idesc_f16(128, N), lbo_b = (N / 8) * 128;
    const uint32_t bh = w, bl = w + N * 64 * 2;
#pragma unroll 1
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
  // x[16] += D[16 cols at col] * sc + bias
  auto add16 = [&](float* x, uint32_t col, float sc, const float* bias) {
    uint32_t r[16];
    tmem_ld16(tbase + lane_off + col, r);
    tmem_wait_ld();
#pragma unroll
    for (int e = 0; e < 16; ++e) x[e] += fmaf(__uint_as_float(r[e]), sc, __ldg(bias + e));
  };
  // LayerNorm over the row's four 16-column groups (two-pass, like
  // torch.layer_norm) of up to kNtMax rows at once; y = normalised own columns
  auto ln16 = [&](float (*x)[16], float (*y)[16], int n, const float* g, const float* bt) {
    float mean[kNtMax], rstd[kNtMax];
#pragma unroll
    for (int i = 0; i < kNtMax; ++i) {
      if (i >= n) break;
      float sacc = 0.f;
#pragma unroll
      for (int e = 0; e < 16; ++e) sacc += x[i][e];
      set_comp(&sm.red[0][i][m], cg, sacc);
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kNtMax; ++i) {
      if (i >= n) break;
      mean[i] = sum4(sm.red[0][i][m]) * (1.f / 64.f);
      float v = 0.f;
#pragma unroll
      for (int e = 0; e < 16; ++e) v = fmaf(x[i][e] - mean[i], x[i][e] - mean[i], v);
      set_comp(&sm.red[1][i][m], cg, v);
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kNtMax; ++i) {
      if (i >= n) break;
      rstd[i] = rsqrtf(sum4(sm.red[1][i][m]) * (1.f / 64.f) + 1e-5f);
#pragma unroll
      for (int e = 0; e < 16; ++e)
        y[i][e] = (x[i][e] - mean[i]) * rstd[i] * __ldg(g + c0 + e) + __ldg(bt + c0 + e);
    }
  };
  const float scale = rsqrtf(32.f);
  const int hh = cg >> 1, dh = cg & 1;              // temporal head and 16-dim half

  int ci0 = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x, ci0 += per_item) {
    const int tile = item / hsplit, hpart = item - tile * hsplit;
    const int g = tile * rows + m;
    const bool valid = m < rows && g < total;
    int b = 0, r = 0, s = 0;
    if (valid) {
      int lo = 0, hi = a.b - 1;        // last stream with pref <= g (skips empty ones)
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sm.pref[mid] <= g) lo = mid;
        else hi = mid - 1;
      }
      b = lo;
      r = g - sm.pref[b];
      s = a.list ? a.list[b * a.ns + r] : r;
    }
    float xs[kNtMax][16], ys[kNtMax][16];

    // ---- x_t += proj_s(ao_t), every slice ------------------------------------------
#pragma unroll
    for (int it = 0; it < kNtMax; ++it) {
      if (it >= nt) break;
      float* y = ys[it];
      if (!valid) {
#pragma unroll
        for (int e = 0; e < 16; ++e) y[e] = 0.f;
      } else {
        const float4* ai = reinterpret_cast<const float4*>(
            a.ao + (size_t(b * nt + it) * a.ns + r) * 64 + c0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 u = ai[q];
          y[4 * q] = u.x; y[4 * q + 1] = u.y; y[4 * q + 2] = u.z; y[4 * q + 3] = u.w;
        }
      }
      put16_x3(sm.a[it], m, y, 2 * cg);
      // the residual rows while the MMA runs
      if (valid) {
        const float4* xi = reinterpret_cast<const float4*>(
            a.x + (size_t(b * nt + it) * a.ns + s) * 64 + c0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 u = xi[q];
          xs[it][4 * q] = u.x; xs[it][4 * q + 1] = u.y; xs[it][4 * q + 2] = u.z;
          xs[it][4 * q + 3] = u.w;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) xs[it][e] = 0.f;
      }
    }
    LT(2);
    run([&] {
      wait_chunk(ci0);
#pragma unroll 1
      for (int it = 0; it < nt; ++it) issue_a(it, 64 * it, wsm(ci0), 64);
    });
    LT(3);
    if (t0) load_chunk(ci0 + 2);                                  // proj_t -> stage 0

    // ---- LN_t of every slice -> qkv_t (q|k|v of the last slice, k|v of the others) ---
#pragma unroll
    for (int it = 0; it < kNtMax; ++it) {
      if (it >= nt) break;
      add16(xs[it], 64 * it + c0, a.sc[0], a.b_proj_s + c0);
    }
    ln16(xs, ys, nt, a.ln_t_w, a.ln_t_b);
#pragma unroll
    for (int it = 0; it < kNtMax; ++it) {
      if (it >= nt) break;
      put16_x3(sm.a[it], m, ys[it], 2 * cg);
    }
    LT(4);
    run([&] {
      wait_chunk(ci0 + 1);
      const uint32_t wq3 = wsm(ci0 + 1);
      issue_a(nt - 1, 0, wq3, 192);                               // last slice -> [0, 192)
      // k|v = rows 64..191 of the qkv_t matrix (8-row groups are 128 B apart)
#pragma unroll 1
      for (int it = 0; it + 1 < nt; ++it) {
        const uint32_t ab = smem_u32(sm.a[it]);
        const uint32_t idesc = idesc_f16(128, 128), lbo_b = 24 * 128;
        const uint32_t bh = wq3 + 8 * 128, bl = wq3 + 192 * 128 + 8 * 128;
#pragma unroll 1
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ah = sdesc(ab + kk * 4096, 128, kSwizzleNone, 2048);
          const uint64_t al = sdesc(ab + kABytes + kk * 4096, 128, kSwizzleNone, 2048);
          const uint64_t wh = sdesc(bh + kk * 2 * lbo_b, 128, kSwizzleNone, lbo_b);
          const uint64_t wl = sdesc(bl + kk * 2 * lbo_b, 128, kSwizzleNone, lbo_b);
          const uint32_t d = tbase + 192 + 128 * it;
          mma_ss_w(d, ah, wh, idesc, kk != 0);
          mma_ss_w(d, ah, wl, idesc, 1);
          mma_ss_w(d, al, wh, idesc, 1);
        }
      }
    });
    LT(5);
    if (t0) load_chunk(ci0 + 3);                                  // fc1 rows 0-127 -> stage 1

    // ---- temporal attention of the last-slice query (head hh, dims 16 dh..) -----------
    float* xl = xs[nt - 1];
    {
      const float sq = a.sc[1];
      const float* bq = a.b_qkv_t + 32 * hh + 16 * dh;
      float q[16], kv[16], sc[kNtMax];
      {
        uint32_t rq[16];
        tmem_ld16(tbase + lane_off + 32 * hh + 16 * dh, rq);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e) q[e] = fmaf(__uint_as_float(rq[e]), sq, __ldg(bq + e));
      }
#pragma unroll
      for (int it = 0; it < kNtMax; ++it) {
        if (it >= nt) break;
        const uint32_t kc = (it == nt - 1 ? 64 : 192 + 128 * it) + 32 * hh + 16 * dh;
        uint32_t rk[16];
        tmem_ld16(tbase + lane_off + kc, rk);
        tmem_wait_ld();
        float acc = 0.f;
#pragma unroll
        for (int e = 0; e < 16; ++e)
          acc = fmaf(q[e], fmaf(__uint_as_float(rk[e]), sq, __ldg(bq + 64 + e)), acc);
        set_comp(&sm.red[0][it][m], cg, acc);
      }
      __syncthreads();
      float mx = -INFINITY;
#pragma unroll
      for (int it = 0; it < kNtMax; ++it) {
        if (it >= nt) break;
        const float4 pr = sm.red[0][it][m];
        sc[it] = (comp(pr, 2 * hh) + comp(pr, 2 * hh + 1)) * scale;
        mx = fmaxf(mx, sc[it]);
      }
      float den = 0.f;
#pragma unroll
      for (int it = 0; it < kNtMax; ++it) {
        if (it >= nt) break;
        sc[it] = expf(sc[it] - mx);
        den += sc[it];
      }
      const float inv = 1.f / den;
#pragma unroll
      for (int e = 0; e < 16; ++e) kv[e] = 0.f;                   // output accumulator
#pragma unroll
      for (int it = 0; it < kNtMax; ++it) {
        if (it >= nt) break;
        const uint32_t vc = (it == nt - 1 ? 128 : 192 + 128 * it + 64) + 32 * hh + 16 * dh;
        uint32_t rv[16];
        tmem_ld16(tbase + lane_off + vc, rv);
        tmem_wait_ld();
        const float p = sc[it] * inv;
#pragma unroll
        for (int e = 0; e < 16; ++e)
          kv[e] = fmaf(p, fmaf(__uint_as_float(rv[e]), sq, __ldg(bq + 128 + e)), kv[e]);
      }
      put16_x3(sm.a[0], m, kv, 2 * cg);                          // = columns 32 hh + 16 dh
    }

    LT(6);
    // ---- x += proj_t(o); LN_m -> fc1 ------------------------------------------------
    run([&] {
      wait_chunk(ci0 + 2);
      issue_a(0, 0, wsm(ci0 + 2), 64);
    });
    LT(7);
    if (t0) load_chunk(ci0 + 4);                                  // fc1 rows 128-255 -> stage 0
    add16(xl, c0, a.sc[2], a.b_proj_t + c0);
    ln16(reinterpret_cast<float(*)[16]>(xl), ys, 1, a.ln_m_w, a.ln_m_b);
    put16_x3(sm.a[0], m, ys[0], 2 * cg);

    // ---- x += fc2(GELU(fc1(.))) in two halves of 128 hidden units --------------------
    {
      LT(8);
      const float s1 = a.sc[3];
      // fc2 K-half H (its own [hi | lo] N = 64 x K = 128 chunk) from the TMEM
      // column groups [hi 32 | lo 32] of the half's GELU
      auto issue_fc2 = [&](int H, uint32_t w) {
        const uint32_t idesc = idesc_f16(128, 64), lbo_b = 8 * 128;
        const uint32_t bh = w, bl = w + 64 * 128 * 2;
#pragma unroll 1
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t ah = tbase + (kk >> 2) * 64 + (kk & 3) * 8;
          const uint64_t wh = sdesc(bh + kk * 2 * lbo_b, 128, kSwizzleNone, lbo_b);
          const uint64_t wl = sdesc(bl + kk * 2 * lbo_b, 128, kSwizzleNone, lbo_b);
          mma_ts_w(tbase + 128, ah, wh, idesc, H != 0 || kk != 0);
          mma_ts_w(tbase + 128, ah, wl, idesc, 1);
          mma_ts_w(tbase + 128, ah + 32, wh, idesc, 1);
        }
      };
#pragma unroll 1
      for (int H = 0; H < 2; ++H) {
        if (H == 0) {
          run([&] {
            wait_chunk(ci0 + 3);
            issue_a(0, 0, wsm(ci0 + 3), 128);
          });
          if (t0) load_chunk(ci0 + 5);                            // fc2 K 0-127 -> stage 1
        } else {
          run([&] {
            wait_chunk(ci0 + 5);
            issue_fc2(0, wsm(ci0 + 5));
            wait_chunk(ci0 + 4);
            issue_a(0, 0, wsm(ci0 + 4), 128);
          });
          if (t0) load_chunk(ci0 + 6);                            // fc2 K 128-255 -> stage 0
        }
        // GELU of the fc1 half in TMEM cols [0,128): group gq = cg / 2 (64
        // hidden units), this thread's 32 of them; written back in place as
        // [hi 32 | lo 32] columns once every thread has read its values
        LT(9 + 2 * H);
        const int gq = cg >> 1, sub = cg & 1;
        uint32_t rr[32], lo[16];
        tmem_ld32(tbase + lane_off + 64 * gq + 32 * sub, rr);
        tmem_wait_ld();
        const float* bias = a.b_fc1 + 128 * H + 64 * gq + 32 * sub;
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float2 g = gelu_as2(make_float2(fmaf(__uint_as_float(rr[e]), s1, __ldg(bias + e)),
                                                fmaf(__uint_as_float(rr[e + 1]), s1, __ldg(bias + e + 1))));
          split_h2(g.x, g.y, rr[e / 2], lo[e / 2]);
        }
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        tmem_st16(tbase + lane_off + 64 * gq + 16 * sub, rr);
        tmem_st16(tbase + lane_off + 64 * gq + 32 + 16 * sub, lo);
        tmem_wait_st();
        LT(10 + 2 * H);
      }
      run([&] {
        wait_chunk(ci0 + 6);
        issue_fc2(1, wsm(ci0 + 6));
      });
      LT(13);
      if (t0) load_chunk(ci0 + 7);                                // head 0 -> stage 1
      add16(xl, 128 + c0, a.sc[4], a.b_fc2 + c0);
    }

    // ---- final LN, head in 4 chunks of 4 patch rows, sigmoid, quantise, merge --------
    ln16(reinterpret_cast<float(*)[16]>(xl), ys, 1, a.norm_w, a.norm_b);
    put16_x3(sm.a[0], m, ys[0], 2 * cg);
    if (t0) load_chunk(ci0 + 8);                                  // head 1 -> stage 0
    const int nc = 64 * c;                                        // columns per chunk
    auto issue_head = [&](int i) {         // this item's i-th head chunk -> TMEM slot i & 1
      const int ci = ci0 + kBlkChunks + i;
      wait_chunk(ci);
      issue_a(0, 256 * (i & 1), wsm(ci), nc);
      mma_commit_w(&sm.bar_h[i & 1]);
    };
    LT(14);
    sync_mma();
    if (w0) issue_head(0);
    const int ih = s / a.nw, iw = s - (s / a.nw) * a.nw;
    uint8_t* ob = nullptr;
    const int pix_bytes = a.u16 ? 2 * c : c;                      // u16 depth: 2 bytes
    if (valid && !a.out_f32)
      ob = a.out_u8 ? a.out_u8 + size_t(b) * a.img_h * a.img_w * pix_bytes
                    : a.out_frames + size_t(a.out_slot[b * a.slot_stride]) * a.frame_bytes;
#pragma unroll 1
    for (int i = 0; i < nh; ++i) {
      const int j = hpart + hsplit * i;                           // head chunk
      if (i + 1 < nh) {
        // every thread has read chunk i-1's columns, which chunk i+1 reuses
        tc_fence_before();
        __syncthreads();
        if (w0) {
          tc_fence_after();
          issue_head(i + 1);
        }
      }
      if (i & 1) mbar_wait(&sm.bar_h[1], ph1++ & 1);
      else mbar_wait(&sm.bar_h[0], ph0++ & 1);
      tc_fence_after();
      LT(15 + 2 * (i & 3));
      // chunk i's stage retired: head i+2, then the next item's first chunks
      if (t0) load_chunk(ci0 + kBlkChunks + i + 2);
      const int py = 4 * j + cg, yy = ih * 16 + py;
#pragma unroll 1
      for (int q = 0; q < c; ++q) {
        uint32_t v[16];
        const int ul = (cg * c + q) * 16;                        // column inside the chunk
        tmem_ld16(tbase + lane_off + 256 * (i & 1) + ul, v);
        tmem_wait_ld();
        if (!valid) continue;
        const int u0 = nc * j + ul;                               // head column
        float sg[16];
        const float4* hb = reinterpret_cast<const float4*>(a.head_b + u0);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float4 bb = __ldg(hb + q4);
          sg[4 * q4] = bb.x; sg[4 * q4 + 1] = bb.y; sg[4 * q4 + 2] = bb.z; sg[4 * q4 + 3] = bb.w;
        }
#pragma unroll
        for (int e = 0; e < 16; ++e)
          sg[e] = sigmoid_fast(fmaf(__uint_as_float(v[e]), a.sc_head, sg[e]));
        if (a.out_f32) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int px = (q * 16 + e) / c, ch = (q * 16 + e) - px * c;
            a.out_f32[((size_t(b) * c + ch) * a.img_h + yy) * a.img_w + iw * 16 + px] = sg[e];
          }
        } else if (C == 1 && a.u16) {
          // np.clip(out * 65535.0 + 0.5, 0, 65535).astype(np.uint16) (16-bit
          // depth, the u8 rule at 16 bits): f32 mul, f32 add, truncate
          uint32_t wd[8];
#pragma unroll
          for (int e2 = 0; e2 < 8; ++e2) {
            float q0 = __fadd_rn(__fmul_rn(sg[2 * e2], 65535.f), 0.5f);
            float q1 = __fadd_rn(__fmul_rn(sg[2 * e2 + 1], 65535.f), 0.5f);
            q0 = fminf(fmaxf(q0, 0.f), 65535.f);
            q1 = fminf(fmaxf(q1, 0.f), 65535.f);
            wd[e2] = uint32_t(q0) | (uint32_t(q1) << 16);
          }
          uint4* o16 = reinterpret_cast<uint4*>(ob + (size_t(yy) * a.img_w + iw * 16) * 2);
          o16[0] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
          o16[1] = make_uint4(wd[4], wd[5], wd[6], wd[7]);
        } else {
          uint32_t wd[4];
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4) {
            uint32_t w = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              // np.clip(out * 255.0 + 0.5, 0, 255).astype(np.uint8): f32 mul, f32 add
              float qv = __fadd_rn(__fmul_rn(sg[4 * e4 + e], 255.f), 0.5f);
              qv = fminf(fmaxf(qv, 0.f), 255.f);
              w |= uint32_t(qv) << (8 * e);
            }
            wd[e4] = w;
          }
          *reinterpret_cast<uint4*>(ob + (size_t(yy) * a.img_w + iw * 16) * c + q * 16) =
              make_uint4(wd[0], wd[1], wd[2], wd[3]);
        }
      }
      LT(16 + 2 * (i & 3));
    }
    LT(23);
    // the next tile's first MMA follows run()'s barrier: every TMEM read above is done
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
  pdl_trigger();
}

}  // namespace

#ifdef NVREC_TRACE
int last_trace(unsigned long long* host, int n) {
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  const int m = n < 64 ? n : 64;
  return cudaMemcpyFromSymbol(host, g_last_trace, m * 8) == cudaSuccess ? m : -1;
}
#endif

bool last_tc_supported(const Dims& D, int b) {
  return D.d == 64 && D.heads == 2 && D.hd == 32 && D.hidden == 256 && D.nt >= 1 &&
         D.nt <= kNtMax && D.p == 16 && (D.c == 1 || D.c == 3) && b >= 1 && b <= kMaxStreams;
}

cudaError_t launch_last_tc(const LastTcArgs& a, int grid_rows, cudaStream_t s) {
  const size_t smem = sizeof(LastSmem) + 128;
  auto kern = a.c == 3 ? (a.nt == 3 ? last_tc_kernel<3, 3> : a.nt == 2 ? last_tc_kernel<2, 3>
                                                           : last_tc_kernel<1, 3>)
                       : (a.nt == 3 ? last_tc_kernel<3, 1> : a.nt == 2 ? last_tc_kernel<2, 1>
                                                           : last_tc_kernel<1, 1>);
  if (cudaError_t e = smem_optin(kern, int(smem))) return e;
  const int sms = sm_count();
  int grid = ceil_div(grid_rows, 32);
  if (grid > sms) grid = sms;
  if (grid < 1) grid = 1;
  launch_seq(kern, grid, kThreads, smem, s, a);
  return cudaGetLastError();
}

}  // namespace nvrec
