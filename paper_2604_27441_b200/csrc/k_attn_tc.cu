// k_attn_tc.cu -- tcgen05/TMEM flash attention for the spatial attention of
// the nvrec blocks (F.scaled_dot_product_attention at model.py:39, called on
// (b*nt, ns, d) at model.py:59-60): softmax(Q K^T / sqrt(32)) V per (stream,
// time slice, head), non-causal, unmasked, head_dim 32, bf16 operands, fp32
// scores / softmax / output.
//
// CTA = two 128-query tiles of one (slice, head) sequence; 10 warps:
//   warps 4t..4t+3  softmax of query tile t (TMEM lanes 0-127, one row/thread)
//   warp  8    TMA producer: Q tiles once, then K/V tiles through a 6-stage
//              ring (K: 128 keys x 64 B, SWIZZLE_64B; V^T: 32 dims x 2 x 128 B,
//              SWIZZLE_128B; the 3-D tensor maps zero-fill keys >= ns)
//   warp  9    MMA issuer (lane 0; the split-operand variants: the whole warp,
//              one lane elected per MMA, sm100.cuh mma_*_w)
// TMEM (512 columns): every query tile owns two 128-column S buffers, so the
// tensor core computes S(j+1) while the softmax warps work on S(j) -- the
// softmax never waits for a QK^T round trip.  Key tile j of tile t:
//   S(j)  = Q_t K_j^T            -> buf[t][j%2] (fp32, 128 columns)
//   P(j)  = 2^(S*scale - m)      softmax warps, bf16 pairs over buf cols 0-63
//   O'(j) = P(j) V_j             -> buf cols 64-95 (dead S columns; fresh
//                                  accumulator, M128 N32 K128, P from TMEM)
// and the softmax thread folds O'(j-1) into its register-resident output
// O = O * 2^(m(j-2) - m(j-1)) + O'(j-1) right after its row max of S(j), then
// releases the buffer for S(j+1).  No output rescaling round trips through
// TMEM, no spin on the tensor core.
//
// Barriers per tile t: s_full[t][2] (S(j) ready, tcgen05.commit), p_full[t]
// (P(j) stored, 128 arrivals), pv_full[t] (O'(j) ready, commit), o_read[t]
// (O'(j) folded, 128 arrivals: buf[j%2] may take S(j+2)).
//
// The exponentials bind (head_dim 32 gives 128 MMA FLOP per exp, SURVEY.md
// 8d): MUFU ex2 for most pairs, the FMA-pipe polynomial for one pair in
// kPolyOf4 of each four.
//
// kX3 (the precise path): fp32-class products from split bf16 operands,
// a = a_hi + a_lo with a_hi = bf16(a), a_lo = bf16(a - a_hi) (16 significant
// bits), every product formed as hi*hi + hi*lo + lo*hi with fp32
// accumulation:
//   Q, K  [seq][ns_pad][64] bf16, columns 0-31 hi, 32-63 lo (128-byte rows,
//         SWIZZLE_128B): S = Qh Kh^T + Qh Kl^T + Ql Kh^T = six K16 MMAs
//   V^T   [seq][64][ns_pad], rows 0-31 hi, 32-63 lo
//   P     split by the softmax warps: P_hi pairs over S columns 0-31, P_lo
//         pairs over 32-63; O'(j) = Ph Vh + Ph Vl + Pl Vh (12 K16 MMAs) into
//         a separate 32-column accumulator per query tile.
// Key tiles are 64 keys (the split P fills its S buffer), all exponentials on
// MUFU (ex2.approx.f32, rel. error ~2^-22).  TMEM: QT x (2 x 64 + 32) columns.
#include <cstdlib>
#include <type_traits>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "launch.cuh"
#include "sm100.cuh"

namespace nvrec {

namespace {

using namespace sm100;

// End-of-group rendezvous of the role-split loops (TMA/MMA warps and softmax
// warps run separate loops over the same work items, so the CTA meets at two
// different barrier instructions): the NON-aligned form, which PTX allows to
// be reached from different code locations (__syncthreads / bar.sync are
// .aligned: one instruction for the whole CTA).
__device__ __forceinline__ void group_barrier() {
  asm volatile("barrier.sync 1, %0;" ::"r"(blockDim.x) : "memory");
}

constexpr int kHd = 32;
constexpr int kTileQ = 128;
constexpr int kTileK = 128;
constexpr int kStages = 6;
// per-variant geometry (kX3: split-bf16 precise path, see the header)
template <bool X3> struct Geo {
  static constexpr int TK = X3 ? 64 : 128;              // keys per tile
  static constexpr uint32_t Row = X3 ? 128 : 64;        // bytes per Q/K row
  static constexpr uint32_t QBytes = kTileQ * Row;
  static constexpr uint32_t KBytes = TK * Row;
  static constexpr uint32_t VBytes = 8192;              // V^T tile: 32 dims x 128 keys | 64 rows x 64 keys
  static constexpr uint32_t Sw = X3 ? 2u /*kSwizzle128B*/ : 4u /*kSwizzle64B*/;
  static constexpr uint32_t Sbo = X3 ? 1024 : 512;
};
template <bool X3, int QT> __host__ __device__ constexpr int stages_for() { return X3 && QT == 1 ? 5 : kStages; }
template <bool X3, int QT> __host__ __device__ constexpr uint32_t tmem_cols() {
  return X3 ? (QT == 2 ? 512u : 256u) : uint32_t(QT * 256);
}
// QT = query tiles per CTA: 2 for dense launches (one CTA per SM, all 512 TMEM
// columns); 1 for pruned launches (a handful of masked-patch queries per
// sequence: latency-bound, so two CTAs share an SM and the key range is split
// twice as finely).
__host__ __device__ constexpr int threads_for(int QT) { return (4 * QT + 4) * 32; }
// Register split (setmaxnreg): QT = 2 launches 168 registers per thread (3
// warps per SMSP), QT = 1 launches 128 (two CTAs, 4 warps per SMSP); the
// TMA/MMA warpgroup drops to kRegsCtl and the softmax warpgroups rise to
// regs_softmax (per SMSP: ctl + softmax warps x registers <= 512).
constexpr int kRegsCtl = 40;
__host__ __device__ constexpr int regs_softmax(int QT) { return QT == 2 ? 232 : 216; }
constexpr int kPolyOf4 = 1;                            // FMA-pipe exp2 pairs per 4
constexpr uint32_t kQBytes = kTileQ * kHd * 2;         // 8 KB
constexpr uint32_t kKBytes = kTileK * kHd * 2;         // 8 KB
constexpr uint32_t kVBytes = kHd * kTileK * 2;         // 8 KB
constexpr uint32_t kIdescS = idesc_bf16(128, 128);
constexpr uint32_t kIdescPV = idesc_bf16(128, 32);
constexpr uint32_t kIdescPV64 = idesc_bf16(128, 64);
constexpr uint32_t kColOp = 64;                        // O'(j) inside its S buffer
constexpr float kSlackSum = 256.f;                     // speculative-max headroom: row sum of P
static_assert(2 * 2 * kTileK <= 512, "TMEM budget");

template <int QT, bool X3 = false>
struct __align__(1024) Smem {
  static constexpr int NS = stages_for<X3, QT>();
  uint8_t v[NS][Geo<X3>::VBytes];   // 1024-aligned (SWIZZLE_128B atoms)
  uint8_t q[QT][Geo<X3>::QBytes];   // 512/1024-aligned (SWIZZLE_64B/128B atoms)
  uint8_t k[NS][Geo<X3>::KBytes];
  uint64_t q_full;
  uint64_t kv_full[NS], kv_empty[NS];
  uint64_t s_full[QT][2], p_full[QT], pv_full[QT], o_read[QT], done;
  int redo[3];                      // per group iteration (mod 3): speculative max overflowed
  uint32_t tmem_base;
};

struct TcArgs {
  float* ao;          // [b][nt][ns][64]
  int ao_half;        // write ao as fp16 (same layout, the token_tc A operand format)
  const int* count;   // compact query count per stream, or null (= ns)
  float* part;        // KV-split partials [split][seq][ns][kPart] or null
  int nt, heads, ns, d, seqs;
  int splits;         // key-range splits (flash-decoding style) >= 1
  int groups;         // query groups launched per (seq, split); CTAs loop
  int mode;           // 0 speculative max (default), 1 exact maxima, 2 force redo (tests)
  int* redo_list;     // [0] = count, then work items whose speculative max overflowed
  float scale_log2;
};
constexpr int kPart = 36;
constexpr int kFixCtas = 32;                           // exact fix-up grid (grid-stride list walk)
__device__ unsigned long long g_fix_items;             // diagnostics: items redone so far                              // 32 output dims, m, l, 2 pad (16 B rows)

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <bool X3 = false>
__device__ __forceinline__ uint32_t buf_col(int t, int j) {
  return uint32_t((2 * t + (j & 1)) * Geo<X3>::TK);
}
// O'(j) of query tile t: inside its S buffer (fast) or its own 32 columns (kX3)
template <bool X3, int QT>
__device__ __forceinline__ uint32_t o_col(int t, int j) {
  return X3 ? uint32_t(2 * QT * Geo<X3>::TK + 32 * t) : buf_col<X3>(t, j) + kColOp;
}
// bf16 hi/lo split of a pair: hi = bf16(p), lo = bf16(p - hi)
__device__ __forceinline__ void split_bf16(float x, float y, uint32_t& hi, uint32_t& lo) {
  hi = pack_bf16(x, y);
  const float2 h = unpack_bf16(hi);
  lo = pack_bf16(x - h.x, y - h.y);
}

// Work item = (query group, key split, sequence), it = (group*splits + split)*seqs + seq.
// kMulti: the CTA may loop over several items (pruned launches step through a
// stream's query groups; the fix-up launch walks redo_list); the dense
// instantiation runs exactly one item and keeps every counter at 0.
// kExact: exact per-tile maxima (the fix-up); otherwise the speculative
// running max, and a CTA whose exponent overflowed records its item for the
// fix-up launch that follows on the same stream.
template <bool kMulti, bool kExact, bool kList, int kQT, bool kX3 = false>
__global__ void __launch_bounds__(threads_for(kQT), kQT == 1 ? 2 : 1)
attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q,
               const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_v, TcArgs a) {
  using G = Geo<kX3>;
  constexpr int TK = G::TK;
  constexpr int NS = stages_for<kX3, kQT>();
  pdl_wait();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem<kQT, kX3>& sm = *reinterpret_cast<Smem<kQT, kX3>*>(smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkv_all = (a.ns + TK - 1) / TK;
  const int n_list = kList ? *(volatile int*)a.redo_list : 0;
  // fix-up launch: the last CTA to leave re-arms the list (count and exit
  // counter back to 0) once every CTA has read the count
  auto fix_exit = [&]() {
    if (kList && threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(a.redo_list + 1, 1) == int(gridDim.x) - 1) {
        a.redo_list[0] = 0;
        a.redo_list[1] = 0;
      }
    }
  };
  if (kList && n_list > 0 && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(&g_fix_items, (unsigned long long)n_list);
  if (kList && n_list == 0) {                             // nothing overflowed (uniform)
    __syncthreads();
    fix_exit();
    return;
  }
  // the k-th work item of this CTA, or -1 when done
  auto item_at = [&](int k) -> int {
    if (kList) {
      const int i = int(blockIdx.x) + k * int(gridDim.x);
      return i < n_list ? a.redo_list[2 + i] : -1;
    }
    if (!kMulti && k > 0) return -1;
    return int(blockIdx.x) + k * int(gridDim.x);
  };
  struct Item { int seq, split, group, b, nq, j0, nkv; };
  auto decode = [&](int it) {
    Item w;
    w.seq = it % a.seqs;
    w.split = (it / a.seqs) % a.splits;
    w.group = it / (a.seqs * a.splits);
    w.b = w.seq / (a.nt * a.heads);
    w.nq = a.count ? a.count[w.b] : a.ns;
    w.j0 = w.split * nkv_all / a.splits;
    w.nkv = (w.split + 1) * nkv_all / a.splits - w.j0;
    return w;
  };
  // an item past its stream's queries: skip it (list) or stop (grid order)
  auto live = [&](const Item& w) { return w.group * kQT * kTileQ < w.nq; };
  if (!kList && !live(decode(blockIdx.x))) return;        // uniform across the CTA

  const int kProducer = 4 * kQT, kMma = 4 * kQT + 1;
  if (warp == kProducer && lane == 0) {
    mbar_init(&sm.done, 1);
    sm.redo[0] = (a.mode == 2 && !kExact) ? 1 : 0;   // mode 2: the first item is redone
    sm.redo[1] = sm.redo[2] = 0;
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm.kv_full[s], 1);
      mbar_init(&sm.kv_empty[s], 1);
    }
    for (int t = 0; t < kQT; ++t) {
      mbar_init(&sm.s_full[t][0], 1);
      mbar_init(&sm.s_full[t][1], 1);
      mbar_init(&sm.p_full[t], 128);
      mbar_init(&sm.pv_full[t], 1);
      mbar_init(&sm.o_read[t], 128);
    }
    fence_mbar_init();
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
  }
  if (warp == 0) tmem_alloc<tmem_cols<kX3, kQT>()>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  // Query groups group0, group0 + groups, ...: a pruned launch is sized for one
  // group per sequence and loops when a stream has more masked patches.  The
  // barriers are never re-initialised (a late tcgen05.commit arrival would
  // land on a fresh barrier); every role keeps running use counts instead:
  //   gkv    K/V tiles through the ring so far (stage, phase)
  //   gs[t]  S tiles of query slot t so far (buffer, s_full/p_full/pv_full phase)
  //   go[t]  O' folds of slot t so far (o_read phase)
  //   gq     groups so far (q_full, done phase)
  // Each role runs its own copy of the group loop so that the register
  // reallocation (setmaxnreg) covers disjoint code.
  int gkv = 0, gq = 0, gs[kQT] = {}, go[kQT] = {};
  if (warp >= 4 * kQT) {
    setmaxnreg_dec<kRegsCtl>();
  for (int kit = 0;; ++kit) {
    const int it = item_at(kit);
    if (it < 0) break;
    const Item w = decode(it);
    if (!live(w)) {
      if (kList) continue;
      break;
    }
    const int seq = w.seq, split = w.split, b = w.b, nq = w.nq, j0 = w.j0, nkv = w.nkv;
    const int q0 = w.group * kQT * kTileQ;
    const int ntq = min(kQT, (nq - q0 + kTileQ - 1) / kTileQ);   // live query tiles
    if (warp == kProducer) {
      // ---------------------------------------------------------- TMA producer
      if (lane == 0) {
        sm.redo[(gq + 1) % 3] = 0;                 // slot of iteration gq+1 (last read at gq-2)
        mbar_expect_tx(&sm.q_full, ntq * G::QBytes);
        for (int t = 0; t < ntq; ++t)
          tma_load_3d(sm.q[t], &tm_q, &sm.q_full, 0, q0 + t * kTileQ, seq);
        for (int j = 0; j < nkv; ++j) {
          const int g = gkv + j, s = g % NS;
          mbar_wait(&sm.kv_empty[s], ((g / NS) & 1) ^ 1);
          mbar_expect_tx(&sm.kv_full[s], G::KBytes + G::VBytes);
          const int key0 = (j0 + j) * TK;
          tma_load_3d(sm.k[s], &tm_k, &sm.kv_full[s], 0, key0, seq);
          tma_load_3d(sm.v[s], &tm_v, &sm.kv_full[s], key0, 0, seq);
          if (!kX3) tma_load_3d(sm.v[s] + G::VBytes / 2, &tm_v, &sm.kv_full[s], key0 + 64, 0, seq);
        }
      }
    } else if (warp == kMma) {
      // ---------------------------------------------------------- MMA issuer
      // x3 (split operands, 22 MMAs per key tile): the whole warp runs the
      // loop and one elected lane issues (*_w: no per-MMA ELECT loop); the
      // bf16 variant (3 MMAs per key tile, softmax-bound) measured faster
      // with lane 0 alone
      if (kX3 || lane == 0) {
        auto mss = [&](uint32_t d, uint64_t a_, uint64_t b_, uint32_t id, uint32_t acc) {
          if constexpr (kX3) mma_ss_w(d, a_, b_, id, acc);
          else mma_ss(d, a_, b_, id, acc);
        };
        auto mts = [&](uint32_t d, uint32_t a_, uint64_t b_, uint32_t id, uint32_t acc) {
          if constexpr (kX3) mma_ts_w(d, a_, b_, id, acc);
          else mma_ts(d, a_, b_, id, acc);
        };
        auto mcommit = [&](uint64_t* bar) {
          if constexpr (kX3) mma_commit_w(bar);
          else mma_commit(bar);
        };
        constexpr int QK = kX3 ? 4 : 2;            // K16 chunks per Q/K row
        uint64_t qdesc[kQT][QK];
        for (int t = 0; t < kQT; ++t)
          for (int kk = 0; kk < QK; ++kk)
            qdesc[t][kk] = sdesc(smem_u32(sm.q[t]) + kk * 32, G::Sbo, G::Sw);
        constexpr uint32_t idS = idesc_bf16(128, TK);
        mbar_wait(&sm.q_full, gq & 1);
        for (int j = 0; j <= nkv; ++j) {
          if (j < nkv) {
            // S_t(j) into buf[t][j%2] once O'(j-2) there has been folded
            // (kX3: once P(j-2) was read by PV(j-2), issued earlier in order)
            const int g = gkv + j, s = g % NS;
            mbar_wait_fast(&sm.kv_full[s], (g / NS) & 1);
            tc_fence_after();
            const uint32_t kb = smem_u32(sm.k[s]);
            for (int t = 0; t < ntq; ++t) {
              const uint32_t sc = tmem + buf_col<kX3>(t, gs[t] + j);
              if constexpr (kX3) {
                // hi.hi + hi.lo + lo.hi: (Q chunk, K chunk) over the 128-byte rows
                constexpr int qa[6] = {0, 1, 0, 1, 2, 3}, kb_[6] = {0, 1, 2, 3, 0, 1};
#pragma unroll
                for (int u = 0; u < 6; ++u)
                  mss(sc, qdesc[t][qa[u]], sdesc(kb + kb_[u] * 32, G::Sbo, G::Sw), idS, u);
              } else {
                if (j >= 2) {
                  mbar_wait_fast(&sm.o_read[t], (go[t] + j - 2) & 1);
                  tc_fence_after();
                }
                for (int kk = 0; kk < 2; ++kk)
                  mss(sc, qdesc[t][kk], sdesc(kb + kk * 32, G::Sbo, G::Sw), idS, kk);
              }
              mcommit(&sm.s_full[t][(gs[t] + j) & 1]);
            }
          }
          if (j >= 1) {
            // O'_t(j-1) = P_t(j-1) V_{j-1}: M128 N32, 16 keys per step
            const int jp = j - 1, sp = (gkv + jp) % NS;
            const uint32_t vb = smem_u32(sm.v[sp]);
            for (int t = 0; t < ntq; ++t) {
              mbar_wait_fast(&sm.p_full[t], (gs[t] + jp) & 1);
              tc_fence_after();
              const uint32_t bc = tmem + buf_col<kX3>(t, gs[t] + jp);
              const uint32_t oc = tmem + o_col<kX3, kQT>(t, gs[t] + jp);
              if constexpr (kX3) {
                // Ph Vh + Ph Vl + Pl Vh; V^T rows 32-63 (lo) sit 4 KB after hi
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                  const uint32_t vh = vb + kk * 32;
                  mts(oc, bc + kk * 8, sdesc(vh, 1024, kSwizzle128B), kIdescPV, kk);
                  mts(oc, bc + kk * 8, sdesc(vh + 4096, 1024, kSwizzle128B), kIdescPV, 1);
                  mts(oc, bc + 32 + kk * 8, sdesc(vh, 1024, kSwizzle128B), kIdescPV, 1);
                }
              } else {
                for (int kk = 0; kk < 8; ++kk) {   // chunk kk/4 of V^T, 32 B apart
                  const uint32_t addr = vb + (kk >> 2) * (G::VBytes / 2) + (kk & 3) * 32;
                  mts(oc, bc + kk * 8, sdesc(addr, 1024, kSwizzle128B), kIdescPV, kk);
                }
              }
              mcommit(&sm.pv_full[t]);
            }
            mcommit(&sm.kv_empty[sp]);               // K/V_{j-1} fully consumed
          }
        }
        mcommit(&sm.done);             // the group's MMAs (Q reads) are complete
        mbar_wait(&sm.done, gq & 1);
      }
    }
    // next group (or the same one again, exact, if a speculative max
    // overflowed): Q smem and TMEM are reused once everybody is done
    const int gq_done = gq;
    gkv += nkv;
    ++gq;
    for (int t = 0; t < ntq; ++t) {
      gs[t] += nkv;
      go[t] += nkv - 1;
    }
    tc_fence_before();
    __syncwarp();
    group_barrier();
    tc_fence_after();
    if (!kExact && warp == kProducer && lane == 0 && sm.redo[gq_done % 3] != 0) {
      const int idx = atomicAdd(a.redo_list, 1);     // overflowed: exact fix-up later
      a.redo_list[2 + idx] = it;
    }
  }
  } else {
    setmaxnreg_inc<regs_softmax(kQT)>();
  for (int kit = 0;; ++kit) {
    const int it = item_at(kit);
    if (it < 0) break;
    const Item w = decode(it);
    if (!live(w)) {
      if (kList) continue;
      break;
    }
    const int seq = w.seq, split = w.split, b = w.b, nq = w.nq, j0 = w.j0, nkv = w.nkv;
    const int q0 = w.group * kQT * kTileQ;
    const int ntq = min(kQT, (nq - q0 + kTileQ - 1) / kTileQ);   // live query tiles
    {
      // ---------------------------------------------------------- softmax warps
      const int t = warp >> 2;                 // query tile
      const int quarter = warp & 3;            // TMEM lane quarter
      const int row = quarter * 32 + lane;
      const uint32_t lane_off = uint32_t(quarter * 32) << 16;
      float m = -INFINITY, l = 0.f, a_prev = 0.f;
      float2 o2[kHd / 2];
#pragma unroll
      for (int e = 0; e < kHd / 2; ++e) o2[e] = make_float2(0.f, 0.f);
      const int jend = t < ntq ? nkv : 0;          // idle warpgroup: no live rows
      // a warp whose 32 query rows are all past the stream's queries (the
      // tail of the last group; most warps of a pruned launch) keeps the
      // barrier protocol but skips the exponentials -- rows are independent
      // in the MMAs, so its stale P/O rows are never read back
      const bool rows_live = q0 + t * kTileQ + quarter * 32 < nq;
      const int gst = gs[t];
      const float2 sc2 = make_float2(a.scale_log2, a.scale_log2);
      // fold O'(g) into the register-resident output
      auto fold = [&](int g) {
        mbar_wait(&sm.pv_full[t], g & 1);
        tc_fence_after();
        uint32_t ov[32];
        tmem_ld32(tmem + lane_off + o_col<kX3, kQT>(t, g), ov);
        tmem_wait_ld();
        const float2 ap = make_float2(a_prev, a_prev);
#pragma unroll
        for (int e = 0; e < kHd / 2; ++e)
          o2[e] = ffma2(o2[e], ap, make_float2(__uint_as_float(ov[2 * e]),
                                               __uint_as_float(ov[2 * e + 1])));
      };
      // the key-tile loop, specialised for speculative / exact maxima
      // (Z: counters known to be zero -- the single speculative pass of a
      // dense CTA -- so buffer/phase arithmetic folds at compile time)
      auto tiles = [&](auto ex_tag, auto zero_tag) {
        constexpr bool EX = decltype(ex_tag)::value;
        constexpr bool Z = decltype(zero_tag)::value;
        const int gst0 = Z ? 0 : gst;
        for (int j = 0; j < jend; ++j) {
          const int g = gst0 + j;
          const uint32_t t_s = tmem + lane_off + buf_col<kX3>(t, g);
          mbar_wait(&sm.s_full[t][g & 1], (g >> 1) & 1);
          tc_fence_after();
          const int valid = a.ns - (j0 + j) * TK;   // keys of this tile that exist
          // Running max: exact for the first key tile (pass 1), speculative
          // afterwards -- P is computed against the running max while the
          // tile's own max is tracked on the side; only a row whose max grew by
          // more than kSlack (P > 2^kSlack) rescales its stored P by an exact
          // power of two.  Softmax is shift-invariant, so this is the same sum.
          float mn = m;
          float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
          if constexpr (kX3) {
            // one 64-key chunk: S -> P = 2^(s*scale - mn) (MUFU) -> P_hi/P_lo
            // pairs over the S columns; then O'(j-1) is folded
            if (rows_live) {
              uint32_t r[64];
              tmem_ld32(t_s, r);
              tmem_ld32(t_s + 32, r + 32);
              tmem_wait_ld();
              if (valid < TK) {
#pragma unroll
                for (int c = 0; c < 64; ++c)
                  if (c >= valid) r[c] = __float_as_uint(-INFINITY);
              }
              if (j == 0 || EX) {
                float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int c = 0; c < 64; ++c) mx4[c & 3] = fmaxf(mx4[c & 3], __uint_as_float(r[c]));
                mn = fmaxf(m, fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * a.scale_log2);
              }
              const float2 nm2 = make_float2(-mn, -mn);
              uint32_t pl[32];
#pragma unroll
              for (int c = 0; c < 64; c += 2) {
                const float2 v = ffma2(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])),
                                       sc2, nm2);
                const float2 p = make_float2(ex2(v.x), ex2(v.y));
                sum2[(c >> 1) & 1] = fadd2(sum2[(c >> 1) & 1], p);
                split_bf16(p.x, p.y, r[c >> 1], pl[c >> 1]);   // r[c/2] already consumed
              }
              tmem_st16(t_s, r);
              tmem_st16(t_s + 16, r + 16);
              tmem_st16(t_s + 32, pl);
              tmem_st16(t_s + 48, pl + 16);
            }
            if (j > 0) fold(g - 1);
          } else {
          if ((j == 0 || EX) && rows_live) {
            float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  #pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint32_t r[64];
              tmem_ld32(t_s + 64 * h, r);
              tmem_ld32(t_s + 64 * h + 32, r + 32);
              tmem_wait_ld();
  #pragma unroll
              for (int c = 0; c < 64; ++c)
                mx4[c & 3] = fmaxf(mx4[c & 3], 64 * h + c < valid ? __uint_as_float(r[c]) : -INFINITY);
            }
            mn = fmaxf(m, fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * a.scale_log2);
          }
          // exp pass: p = 2^(s*scale - mn) as packed bf16 pairs, written over the
          // already-consumed S columns (chunk h2 reads S[64h2, 64h2+64) and
          // writes P pairs to columns [32h2, 32h2+32)); O'(j-1) is folded
          // between the two halves and its buffer handed back for S(j+1)
          const float2 nm2 = make_float2(-mn, -mn);
  #pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {             // two 32-column chunks per wait
            if (rows_live && h2 == 1 && valid <= 64) {
              // the key range's last tile ends inside its first half: P = 0
              // for the second half without exponentiating masked scores
              uint32_t z[16];
  #pragma unroll
              for (int c = 0; c < 16; ++c) z[c] = 0u;
              tmem_st16(t_s + 32, z);
              tmem_st16(t_s + 48, z);
            } else if (rows_live) {
            uint32_t r[64], pk[32];
            tmem_ld32(t_s + 64 * h2, r);
            tmem_ld32(t_s + 64 * h2 + 32, r + 32);
            tmem_wait_ld();
            if (valid < kTileK) {
  #pragma unroll
              for (int c = 0; c < 64; ++c)
                if (64 * h2 + c >= valid) r[c] = __float_as_uint(-INFINITY);
            }
  #pragma unroll
            for (int c = 0; c < 64; c += 2) {
              const float2 v = ffma2(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])),
                                     sc2, nm2);
              const float2 p = ((c >> 1) & 3) < kPolyOf4 ? exp2_poly2(v)
                                                         : make_float2(ex2(v.x), ex2(v.y));
              sum2[(c >> 1) & 1] = fadd2(sum2[(c >> 1) & 1], p);
              pk[c >> 1] = pack_bf16(p.x, p.y);
            }
            tmem_st16(t_s + 32 * h2, pk);
            tmem_st16(t_s + 32 * h2 + 16, pk + 16);
            }
            if (h2 == 0 && j > 0) {
              fold(g - 1);
              tc_fence_before();
              mbar_arrive(&sm.o_read[t]);
            }
          }
          }
          float2 sums = fadd2(sum2[0], sum2[1]);
          float tsum = sums.x + sums.y;
          if (!EX && j > 0 && __any_sync(0xffffffffu, !(tsum <= kSlackSum))) {
            // rare: the row sum exceeds 2^kSlack, so some p may too -- rescale
            // this row's P (and its sum) by 2^-k, k = ceil(log2 max p), exact
            // (kX3: P_hi over columns 0-31 sets the max, P_lo scales alike)
            tmem_wait_st();
            uint32_t pk[2][32];
            float pmax = 0.f;
  #pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              tmem_ld32(t_s + 32 * h2, pk[h2]);
              tmem_wait_ld();
              if (kX3 && h2 == 1) continue;
  #pragma unroll
              for (int c = 0; c < 32; ++c) {
                const float2 pv = unpack_bf16(pk[h2][c]);
                pmax = fmaxf(pmax, fmaxf(pv.x, pv.y));
              }
            }
            // p >= 2^100 (or inf from MUFU): the exponent overflowed, P is not
            // exact any more -> the whole query group is redone with exact maxima
            if (!(tsum <= kSlackSum) && !(pmax < 0x1p100f)) sm.redo[gq % 3] = 1;
            const float k = tsum > kSlackSum && pmax < 0x1p100f ? fmaxf(0.f, ceilf(__log2f(pmax)))
                                                                : 0.f;
            const float f = ex2(-k);
  #pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
  #pragma unroll
              for (int c = 0; c < 32; ++c) {
                const float2 pv = unpack_bf16(pk[h2][c]);
                pk[h2][c] = pack_bf16(pv.x * f, pv.y * f);
              }
              tmem_st16(t_s + 32 * h2, pk[h2]);
              tmem_st16(t_s + 32 * h2 + 16, pk[h2] + 16);
            }
            tsum *= f;
            mn += k;
          }
          const float alpha = ex2(m - mn);
          l = l * alpha + tsum;
          m = mn;
          a_prev = alpha;
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&sm.p_full[t]);
        }
      };
      tiles(std::integral_constant<bool, kExact>{}, std::integral_constant<bool, !kMulti>{});
      const int q = q0 + t * kTileQ + row;
      if (t < ntq) {
        const int g = gst + nkv - 1;
        mbar_wait(&sm.pv_full[t], g & 1);          // final O'
        tc_fence_after();
        uint32_t ov[32];
        tmem_ld32(tmem + lane_off + o_col<kX3, kQT>(t, g), ov);
        tmem_wait_ld();
        float o[kHd];
#pragma unroll
        for (int e = 0; e < kHd / 2; ++e) {
          const float2 x = ffma2(o2[e], make_float2(a_prev, a_prev),
                                 make_float2(__uint_as_float(ov[2 * e]), __uint_as_float(ov[2 * e + 1])));
          o[2 * e] = x.x;
          o[2 * e + 1] = x.y;
        }
        if (q < nq && a.splits > 1) {
          // unnormalised partial (O, m, l) of this key range; attn_combine merges
          float* dst = a.part + ((size_t(split) * a.seqs + seq) * a.ns + q) * kPart;
#pragma unroll
          for (int e = 0; e < kHd; e += 4)
            *reinterpret_cast<float4*>(dst + e) = make_float4(o[e], o[e + 1], o[e + 2], o[e + 3]);
          dst[32] = m;
          dst[33] = l;
        } else if (q < nq) {
          const int it = (seq / a.heads) % a.nt, hh = seq % a.heads;
          const float inv = 1.f / l;
          const size_t off = (size_t(b * a.nt + it) * a.ns + q) * a.d + hh * kHd;
          if (a.ao_half) {
            // fp16, rounded exactly as token_tc would round the fp32 value
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(a.ao) + off);
#pragma unroll
            for (int e = 0; e < kHd; e += 8)
              dst[e / 8] = make_uint4(pack_h2(o[e] * inv, o[e + 1] * inv),
                                      pack_h2(o[e + 2] * inv, o[e + 3] * inv),
                                      pack_h2(o[e + 4] * inv, o[e + 5] * inv),
                                      pack_h2(o[e + 6] * inv, o[e + 7] * inv));
          } else {
            float4* dst = reinterpret_cast<float4*>(a.ao + off);
#pragma unroll
            for (int e = 0; e < kHd; e += 4)
              dst[e / 4] = make_float4(o[e] * inv, o[e + 1] * inv, o[e + 2] * inv, o[e + 3] * inv);
          }
        }
      }
    }
    // next group (or the same one again, exact, if a speculative max
    // overflowed): Q smem and TMEM are reused once everybody is done
    const int gq_done = gq;
    gkv += nkv;
    ++gq;
    for (int t = 0; t < ntq; ++t) {
      gs[t] += nkv;
      go[t] += nkv - 1;
    }
    tc_fence_before();
    __syncwarp();
    group_barrier();
    tc_fence_after();
    (void)gq_done;
  }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<tmem_cols<kX3, kQT>()>(tmem);
  fix_exit();
  pdl_trigger();
}

// ---- dense split-bf16 attention with 128-key tiles (precise path) -------------
// The dense speculative launch of the precise path: same arithmetic as the
// kX3 variant of attn_tc_kernel, but 128-key tiles.  A split P fills its whole
// 128-column S buffer (per 64-key chunk h: P_hi pairs at 64h + [0,32), P_lo
// pairs at 64h + [32,64)), so the two query tiles share THREE rotating S
// buffers: S tile n (query tile t = n % ntq, key tile j = n / ntq) lives in
// buffer n % 3, and the MMA issuer runs PV two S tiles behind, i.e. the next S
// of a query tile is issued as soon as the OTHER tile's previous P is done --
// each softmax warpgroup finds its next S computed while it works.  O(t) has
// its own 64 columns and accumulates over ALL key tiles in TMEM (Ph [Vh | Vl]
// as one N = 64 MMA, then Pl Vh into the first half; the halves are added once
// at the end): with the speculative max, m only moves in the rare rescale,
// which scales O in place.  TMEM = 3 x 128 + 2 x 64 = 512 columns.  The MMA
// warp issues warp-wide (one elected lane per MMA).
constexpr int kWTK = 128, kWStages = 4;
#ifdef NVREC_TRACE
// phase timestamps of one CTA (tools/trace_attn.py): role r (0: softmax warp
// 0 = tile 0, 1: softmax warp 4 = tile 1, 2: MMA issuer), step i, event e
constexpr int kTraceCta = 300;
__device__ unsigned long long g_trace[3 * 128 * 8];
#define NVREC_TR(role, i, e)                                                          \
  do {                                                                                \
    if (blockIdx.x == kTraceCta && (i) < 128) g_trace[((role) * 128 + (i)) * 8 + (e)] = clock64(); \
  } while (0)
#else
#define NVREC_TR(role, i, e) do {} while (0)
#endif
constexpr uint32_t kWQBytes = 128 * 128, kWKBytes = 128 * 128, kWVBytes = 128 * 128;

struct __align__(1024) SmemW {
  uint8_t v[kWStages][kWVBytes];    // V^T: two (64 keys x 64 rows) boxes, rows 0-31 hi, 32-63 lo
  uint8_t q[2][kWQBytes];           // Q tile [128][64] bf16 (hi | lo), SWIZZLE_128B
  uint8_t k[kWStages][kWKBytes];    // K tile [128][64]
  uint64_t q_full, kv_full[kWStages], kv_empty[kWStages];
  uint64_t s_full[3], p_full[2], pv_full[2];
  int redo;
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(threads_for(2), 1)
attn_x3w_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v, TcArgs a) {
  pdl_wait();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  SmemW& sm = *reinterpret_cast<SmemW*>(smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkv_all = (a.ns + kWTK - 1) / kWTK;
  const int it = int(blockIdx.x);
  const int seq = it % a.seqs, split = (it / a.seqs) % a.splits, group = it / (a.seqs * a.splits);
  const int b = seq / (a.nt * a.heads);
  const int nq = a.ns;
  const int j0 = split * nkv_all / a.splits;
  const int nkv = (split + 1) * nkv_all / a.splits - j0;
  const int q0 = group * 2 * kTileQ;
  if (q0 >= nq) return;
  const int ntq = min(2, (nq - q0 + kTileQ - 1) / kTileQ);
  const int N = nkv * ntq;                                  // S tiles of this CTA
  constexpr uint32_t kOCol = 3 * kWTK;                      // O'(t) at 384 + 32 t
  constexpr int kProducer = 8, kMma = 9;
  if (warp == kProducer && lane == 0) {
    sm.redo = a.mode == 2 ? 1 : 0;
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < kWStages; ++s) {
      mbar_init(&sm.kv_full[s], 1);
      mbar_init(&sm.kv_empty[s], 1);
    }
    for (int i = 0; i < 3; ++i) mbar_init(&sm.s_full[i], 1);
    for (int t = 0; t < 2; ++t) {
      mbar_init(&sm.p_full[t], 128);
      mbar_init(&sm.pv_full[t], 1);
    }
    fence_mbar_init();
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
  }
  if (warp == 0) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp >= 8) {
    setmaxnreg_dec<kRegsCtl>();
    if (warp == kProducer && lane == 0) {
      // ------------------------------------------------------------ TMA producer
      mbar_expect_tx(&sm.q_full, ntq * kWQBytes);
      for (int t = 0; t < ntq; ++t) tma_load_3d(sm.q[t], &tm_q, &sm.q_full, 0, q0 + t * kTileQ, seq);
      for (int j = 0; j < nkv; ++j) {
        const int s = j % kWStages;
        mbar_wait(&sm.kv_empty[s], ((j / kWStages) & 1) ^ 1);
        mbar_expect_tx(&sm.kv_full[s], kWKBytes + kWVBytes);
        const int key0 = (j0 + j) * kWTK;
        tma_load_3d(sm.k[s], &tm_k, &sm.kv_full[s], 0, key0, seq);
        tma_load_3d(sm.v[s], &tm_v, &sm.kv_full[s], key0, 0, seq);
        tma_load_3d(sm.v[s] + kWVBytes / 2, &tm_v, &sm.kv_full[s], key0 + 64, 0, seq);
      }
    } else if (warp == kMma) {
      // ------------------------------------------------------------ MMA issuer
      // (the whole warp runs the loop; one elected lane issues: *_w)
      const uint32_t qbase = smem_u32(sm.q[0]);
      constexpr uint32_t idS = idesc_bf16(128, kWTK);
      mbar_wait(&sm.q_full, 0);
      for (int n = 0; n < N + 2; ++n) {
        NVREC_TR(2, n, 0);
        if (n < N) {
          // S(n) -> buffer n % 3 (its previous user, PV(n-3), was issued in
          // iteration n-1: the tensor pipe executes MMAs in issue order)
          const int t = n % ntq, j = n / ntq, s = j % kWStages;
          if (t == 0) {
            mbar_wait_fast(&sm.kv_full[s], (j / kWStages) & 1);
            tc_fence_after();
          }
          const uint32_t kb = smem_u32(sm.k[s]), qb = qbase + t * kWQBytes;
          const uint32_t sc = tmem + (n % 3) * kWTK;
          constexpr int qa[6] = {0, 1, 0, 1, 2, 3}, kc[6] = {0, 1, 2, 3, 0, 1};
#pragma unroll
          for (int u = 0; u < 6; ++u)
            mma_ss_w(sc, sdesc(qb + qa[u] * 32, 1024, kSwizzle128B),
                   sdesc(kb + kc[u] * 32, 1024, kSwizzle128B), idS, u);
          mma_commit_w(&sm.s_full[n % 3]);
        }
        NVREC_TR(2, n, 1);
        const int m = n - 2;
        if (m >= 0 && m < N) {
          // O'_t(m) = Ph Vh + Ph Vl + Pl Vh over 8 K16 chunks
          const int t = m % ntq, j = m / ntq, s = j % kWStages;
          mbar_wait_fast(&sm.p_full[t], j & 1);
          NVREC_TR(2, n, 2);
          tc_fence_after();
          const uint32_t vb = smem_u32(sm.v[s]);
          const uint32_t bc = tmem + (m % 3) * kWTK, oc = tmem + kOCol + 64 * t;
          // per 16 keys: Ph [Vh | Vl] (one N = 64 MMA: the V^T hi and lo rows
          // are adjacent) + Pl Vh (N = 32); O'(t) = D[0,32) + D[32,64)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t ah = bc + (kk >> 2) * 64 + (kk & 3) * 8;
            const uint32_t vh = vb + (kk >> 2) * (kWVBytes / 2) + (kk & 3) * 32;
            mma_ts_w(oc, ah, sdesc(vh, 1024, kSwizzle128B), kIdescPV64, (j | kk) != 0);
            mma_ts_w(oc, ah + 32, sdesc(vh, 1024, kSwizzle128B), kIdescPV, 1);
          }
          mma_commit_w(&sm.pv_full[t]);
          if (t == ntq - 1) mma_commit_w(&sm.kv_empty[s]);     // K/V(j) fully consumed
        }
        NVREC_TR(2, n, 3);
      }
    }
  } else {
    setmaxnreg_inc<regs_softmax(2)>();
    // ------------------------------------------------------------ softmax warps
    const int t = warp >> 2, quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    float m = -INFINITY, l = 0.f;
    const bool live_t = t < ntq;
    const bool rows_live = live_t && q0 + t * kTileQ + quarter * 32 < nq;
    const float2 sc2 = make_float2(a.scale_log2, a.scale_log2);
    // O(t) accumulates in TMEM over all key tiles (PV with enable-input from
    // the second tile on); the softmax only waits for PV(j-1) before handing
    // over P(j+1)... (bounds the p_full phases) and reads O once at the end
    const uint32_t o_t = tmem + lane_off + kOCol + 64 * t;
    const bool tr = quarter == 0 && lane == 0;
    for (int j = 0; live_t && j < nkv; ++j) {
      const int n = j * ntq + t;
      const uint32_t t_s = tmem + lane_off + (n % 3) * kWTK;
      if (tr) NVREC_TR(t, j, 0);
      mbar_wait(&sm.s_full[n % 3], (n / 3) & 1);
      if (tr) NVREC_TR(t, j, 1);
      tc_fence_after();
      const int valid = a.ns - (j0 + j) * kWTK;
      float mn = m;
      if (j == 0 && rows_live) {
        // exact max over the first key tile; speculative afterwards
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t r[64];
          tmem_ld32(t_s + 64 * h, r);
          tmem_ld32(t_s + 64 * h + 32, r + 32);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 64; ++c)
            mx4[c & 3] = fmaxf(mx4[c & 3], 64 * h + c < valid ? __uint_as_float(r[c]) : -INFINITY);
        }
        mn = fmaxf(m, fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * a.scale_log2);
      }
      float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      const float2 nm2 = make_float2(-mn, -mn);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (rows_live) {
          uint32_t r[64], pl[32];
          tmem_ld32(t_s + 64 * h, r);
          tmem_ld32(t_s + 64 * h + 32, r + 32);
          tmem_wait_ld();
          if (valid < kWTK) {
#pragma unroll
            for (int c = 0; c < 64; ++c)
              if (64 * h + c >= valid) r[c] = __float_as_uint(-INFINITY);
          }
#pragma unroll
          for (int c = 0; c < 64; c += 2) {
            const float2 v = ffma2(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])), sc2, nm2);
            const float2 p = make_float2(ex2(v.x), ex2(v.y));
            sum2[(c >> 1) & 1] = fadd2(sum2[(c >> 1) & 1], p);
            split_bf16(p.x, p.y, r[c >> 1], pl[c >> 1]);   // r[c/2] already consumed
          }
          tmem_st16(t_s + 64 * h, r);
          tmem_st16(t_s + 64 * h + 16, r + 16);
          tmem_st16(t_s + 64 * h + 32, pl);
          tmem_st16(t_s + 64 * h + 48, pl + 16);
        }
        if (tr) NVREC_TR(t, j, 2 + 2 * h);
      }
      float2 sums = fadd2(sum2[0], sum2[1]);
      float tsum = sums.x + sums.y;
      if (j > 0 && __any_sync(0xffffffffu, !(tsum <= kSlackSum))) {
        // rare: rescale this row's P (hi and lo) by 2^-k, exact
        tmem_wait_st();
        float pmax = 0.f;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          uint32_t pk[32];
          tmem_ld32(t_s + 64 * h, pk);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const float2 pv = unpack_bf16(pk[c]);
            pmax = fmaxf(pmax, fmaxf(pv.x, pv.y));
          }
        }
        if (!(tsum <= kSlackSum) && !(pmax < 0x1p100f)) sm.redo = 1;
        const float k = tsum > kSlackSum && pmax < 0x1p100f ? fmaxf(0.f, ceilf(__log2f(pmax))) : 0.f;
        const float f = ex2(-k);
#pragma unroll 1
        for (int g4 = 0; g4 < 4; ++g4) {        // hi and lo column groups alike
          uint32_t pk[32];
          tmem_ld32(t_s + 32 * g4, pk);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const float2 pv = unpack_bf16(pk[c]);
            pk[c] = pack_bf16(pv.x * f, pv.y * f);
          }
          tmem_st32(t_s + 32 * g4, pk);
        }
        tsum *= f;
        mn += k;
        // O (all earlier tiles) by 2^(m - mn) once PV(j-1) has landed
        mbar_wait(&sm.pv_full[t], (j - 1) & 1);
        tc_fence_after();
        const float al = ex2(m - mn);
#pragma unroll 1
        for (int g4 = 0; g4 < 2; ++g4) {
          uint32_t ov[32];
          tmem_ld32(o_t + 32 * g4, ov);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 32; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) * al);
          tmem_st32(o_t + 32 * g4, ov);
        }
      }
      const float alpha = ex2(m - mn);
      l = l * alpha + tsum;
      m = mn;
      // P(j) goes to the issuer only once PV(j-1) is done: the issuer has then
      // consumed p_full's previous phase (no parity aliasing), and a rescale
      // above never races an in-flight PV
      if (j > 0) {
        mbar_wait(&sm.pv_full[t], (j - 1) & 1);
        tc_fence_after();
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&sm.p_full[t]);
      if (tr) NVREC_TR(t, j, 5);
    }
    if (live_t) {
      mbar_wait(&sm.pv_full[t], (nkv - 1) & 1);
      tc_fence_after();
      float2 o2[kHd / 2];
      {
        uint32_t ov[64];
        tmem_ld32(o_t, ov);
        tmem_ld32(o_t + 32, ov + 32);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < kHd / 2; ++e)
          o2[e] = fadd2(make_float2(__uint_as_float(ov[2 * e]), __uint_as_float(ov[2 * e + 1])),
                        make_float2(__uint_as_float(ov[32 + 2 * e]), __uint_as_float(ov[33 + 2 * e])));
      }
      const int q = q0 + t * kTileQ + row;
      if (q < nq && a.splits > 1) {
        float* dst = a.part + ((size_t(split) * a.seqs + seq) * a.ns + q) * kPart;
#pragma unroll
        for (int e = 0; e < kHd / 2; e += 2)
          *reinterpret_cast<float4*>(dst + 2 * e) = make_float4(o2[e].x, o2[e].y, o2[e + 1].x, o2[e + 1].y);
        dst[32] = m;
        dst[33] = l;
      } else if (q < nq) {
        const int it2 = (seq / a.heads) % a.nt, hh = seq % a.heads;
        const float inv = 1.f / l;
        float4* dst = reinterpret_cast<float4*>(a.ao + (size_t(b * a.nt + it2) * a.ns + q) * a.d + hh * kHd);
#pragma unroll
        for (int e = 0; e < kHd / 2; e += 2)
          dst[e / 2] = make_float4(o2[e].x * inv, o2[e].y * inv, o2[e + 1].x * inv, o2[e + 1].y * inv);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
  if (warp == kProducer && lane == 0 && sm.redo != 0) {
    const int idx = atomicAdd(a.redo_list, 1);     // overflowed: exact fix-up later
    a.redo_list[2 + idx] = it;
  }
  pdl_trigger();
}

// Merge the key-range partials: O = sum_s O_s 2^(m_s - M) / sum_s l_s 2^(m_s - M).
// One thread per (row, output dim); 8 rows per 256-thread block, grid-stride.
__global__ void __launch_bounds__(256)
attn_combine_kernel(const float* __restrict__ part, float* __restrict__ ao,
                    const int* __restrict__ count, int seqs, int splits, int nt, int heads,
                    int ns, int d, int ao_half) {
  pdl_entry();
  const int seq = blockIdx.y;
  const int b = seq / (nt * heads);
  const int nq = count ? count[b] : ns;
  const int it = (seq / heads) % nt, hh = seq % heads;
  const int e = threadIdx.x & 31;
  for (int q = blockIdx.x * 8 + (threadIdx.x >> 5); q < nq; q += gridDim.x * 8) {
    // every split's loads in flight at once: unrolled to the maximum split
    // count, splits past `splits` re-read the last one with weight 0
    float ms[kAttnMaxSplits], ls[kAttnMaxSplits], os[kAttnMaxSplits];
    float M = -INFINITY;
#pragma unroll
    for (int sp = 0; sp < kAttnMaxSplits; ++sp) {
      const float* p = part + ((size_t(min(sp, splits - 1)) * seqs + seq) * ns + q) * kPart;
      ms[sp] = __ldg(p + 32);
      ls[sp] = __ldg(p + 33);
      os[sp] = __ldg(p + e);
      M = fmaxf(M, ms[sp]);
    }
    float o = 0.f, L = 0.f;
#pragma unroll
    for (int sp = 0; sp < kAttnMaxSplits; ++sp) {
      const float w = sp < splits ? ex2(ms[sp] - M) : 0.f;
      L = fmaf(ls[sp], w, L);
      o = fmaf(os[sp], w, o);
    }
    const size_t off = (size_t(b * nt + it) * ns + q) * d + hh * kHd + e;
    if (ao_half) reinterpret_cast<__half*>(ao)[off] = __float2half_rn(o / L);
    else ao[off] = o / L;
  }
}

// ---- host: tensor maps ---------------------------------------------------------
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

bool make_map_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                 uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0, uint32_t box1,
                 CUtensorMapSwizzle sw) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool tc_supported(const Dims& D) { return D.hd == kHd; }

#ifdef NVREC_TRACE
int attn_trace(unsigned long long* host, int n) {
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  const int m = n < int(sizeof(g_trace) / 8) ? n : int(sizeof(g_trace) / 8);
  return cudaMemcpyFromSymbol(host, g_trace, m * 8) == cudaSuccess ? m : -1;
}
#endif

int64_t attn_fixup_items() {
  unsigned long long v = 0;
  if (cudaDeviceSynchronize() != cudaSuccess ||
      cudaMemcpyFromSymbol(&v, g_fix_items, sizeof v) != cudaSuccess)
    return -1;
  return int64_t(v);
}

cudaError_t launch_attn_tc(const Act& A, const Dims& D, const int* count, cudaStream_t s,
                           int* n_kernels, bool defer_combine, int* splits_out, bool ao_half,
                           bool x3) {
  const int seqs = A.b * D.nt * D.heads;
  CUtensorMap tq, tk, tv;
  if (!x3) {
    const uint64_t row_b = kHd * 2, seq_b = uint64_t(A.ns_pad) * kHd * 2;
    // Q/K: [seq][ns_pad][32] bf16 viewed (32, ns, seq); rows >= ns read as zero
    if (!make_map_3d(&tq, A.qh, kHd, A.ns, seqs, row_b, seq_b, kHd, kTileQ,
                     CU_TENSOR_MAP_SWIZZLE_64B) ||
        !make_map_3d(&tk, A.kh, kHd, A.ns, seqs, row_b, seq_b, kHd, kTileK,
                     CU_TENSOR_MAP_SWIZZLE_64B) ||
        // V^T: [seq][32][ns_pad] viewed (ns, 32, seq), 64-key boxes (128 B rows)
        !make_map_3d(&tv, A.vth, A.ns, kHd, seqs, uint64_t(A.ns_pad) * 2, seq_b, 64, kHd,
                     CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  } else {
    // split operands: Q/K [seq][ns_pad][64] (hi | lo) as (64, ns, seq), 128-byte
    // rows; V^T [seq][64][ns_pad] (hi rows | lo rows) as (ns, 64, seq)
    const uint64_t row_b = 2 * kHd * 2, seq_b = uint64_t(A.ns_pad) * 2 * kHd * 2;
    if (!make_map_3d(&tq, A.qh, 2 * kHd, A.ns, seqs, row_b, seq_b, 2 * kHd, kTileQ,
                     CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_map_3d(&tk, A.kh, 2 * kHd, A.ns, seqs, row_b, seq_b, 2 * kHd, Geo<true>::TK,
                     CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_map_3d(&tv, A.vth, A.ns, 2 * kHd, seqs, uint64_t(A.ns_pad) * 2, seq_b,
                     Geo<true>::TK, 2 * kHd, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  // the dense precise launch runs attn_x3w_kernel (128-key tiles, K boxes of
  // 128 rows); NVREC_ATTN_X3W=0 keeps the 64-key variant (A/B)
  static int wide_env = -1;
  if (wide_env < 0) {
    const char* e = getenv("NVREC_ATTN_X3W");
    wide_env = e && e[0] == '0' ? 0 : 1;
  }
  const bool wide = x3 && !count && wide_env;
  CUtensorMap tkw;
  if (wide && !make_map_3d(&tkw, A.kh, 2 * kHd, A.ns, seqs, 2 * kHd * 2,
                           uint64_t(A.ns_pad) * 2 * kHd * 2, 2 * kHd, kWTK,
                           CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  TcArgs ta;
  ta.ao = A.ao;
  ta.ao_half = ao_half;
  ta.count = count;
  ta.part = A.part;
  ta.nt = D.nt;
  ta.heads = D.heads;
  ta.ns = A.ns;
  ta.d = D.d;
  ta.seqs = seqs;
  ta.scale_log2 = 1.4426950408889634f / sqrtf(float(kHd));
  const int sms = sm_count();
  // Dense launch: two query tiles per CTA, one CTA per SM (all of TMEM).  A
  // pruned launch (compact masked-patch queries, count on the device): one
  // query tile per CTA, two CTAs per SM, sized for one query group per
  // sequence and looping over further groups.  A short grid splits the key
  // range (flash-decoding partials merged by attn_combine_kernel) so every
  // SM slot works.
  const int qt = count ? 1 : 2, per_sm = count ? 2 : 1;
  const int nkv = ceil_div(A.ns, x3 && !wide ? Geo<true>::TK : kTileK);
  ta.groups = count ? 1 : ceil_div(A.ns, qt * kTileQ);
  int best = 1;
  double best_t = 1e30;
  for (int sp = 1; sp <= kAttnMaxSplits && sp <= nkv && A.part; ++sp) {
    const int ctas = ta.groups * seqs * sp;
    const double t = double(ceil_div(ctas, per_sm * sms)) / sp + (sp > 1 ? 0.05 : 0.0);
    if (t < best_t - 1e-9) { best_t = t; best = sp; }
  }
  static int force = -2;
  if (force == -2) {
    const char* e = getenv("NVREC_ATTN_SPLITS");      // debugging / experiments
    force = e ? atoi(e) : -1;
  }
  if (force >= 1 && force <= kAttnMaxSplits && force <= nkv && A.part) best = force;
  ta.splits = best;
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("NVREC_ATTN_MODE");        // tests: exact / redo
    mode = e && e[0] == 'e' ? 1 : (e && e[0] == 'r' ? 2 : 0);
  }
  ta.mode = mode;
  ta.redo_list = A.redo_list;
  const dim3 grid(ta.groups * seqs * ta.splits);
  cudaError_t err = cudaSuccess;
  auto run = [&](auto qt_tag, auto x3_tag) {
    constexpr int QT = decltype(qt_tag)::value;
    constexpr bool X3 = decltype(x3_tag)::value;
    const int nth = threads_for(QT);
    const size_t smem = sizeof(Smem<QT, X3>) + 1024;
    auto k_exact = attn_tc_kernel<true, true, false, QT, X3>;
    auto k_spec = attn_tc_kernel<QT == 1, false, false, QT, X3>;
    auto k_fix = attn_tc_kernel<true, true, true, QT, X3>;
    if ((err = smem_optin(k_exact, int(smem))) != cudaSuccess ||
        (err = smem_optin(k_spec, int(smem))) != cudaSuccess ||
        (err = smem_optin(k_fix, int(smem))) != cudaSuccess)
      return;
    if (mode == 1 || !A.redo_list) {
      // exact maxima throughout (tests), or no fix-up list available
      launch_seq(k_exact, grid, nth, smem, s, tq, tk, tv, ta);
    } else if (X3 && QT == 2 && wide) {
      // dense precise launch: 128-key tiles, rotating S buffers
      const size_t sw = sizeof(SmemW) + 1024;
      if ((err = smem_optin(attn_x3w_kernel, int(sw))) != cudaSuccess) return;
      launch_seq(attn_x3w_kernel, grid, nth, sw, s, tq, tkw, tv, ta);
      launch_pdl(k_fix, kFixCtas, nth, smem, s, tq, tk, tv, ta);
    } else {
      launch_seq(k_spec, grid, nth, smem, s, tq, tk, tv, ta);
      // exact fix-up of the (rare) items whose speculative exponent overflowed:
      // a grid-stride walk of the list; every CTA exits at once when it is
      // empty, and the last CTA out re-arms the list
      launch_pdl(k_fix, kFixCtas, nth, smem, s, tq, tk, tv, ta);
    }
  };
  if (qt == 1) {
    if (x3) run(std::integral_constant<int, 1>{}, std::true_type{});
    else run(std::integral_constant<int, 1>{}, std::false_type{});
  } else {
    if (x3) run(std::integral_constant<int, 2>{}, std::true_type{});
    else run(std::integral_constant<int, 2>{}, std::false_type{});
  }
  if (err != cudaSuccess) return err;
  const bool combine = ta.splits > 1 && !defer_combine;
  if (n_kernels) *n_kernels = (mode == 1 || !A.redo_list ? 1 : 2) + (combine ? 1 : 0);
  if (splits_out) *splits_out = ta.splits;
  if (combine) {
    // pruned launches: the compact row count is on the device; size for up to
    // 512 rows per sequence per pass (rows past the count exit at once)
    dim3 cg(ceil_div(count ? (A.ns < 512 ? A.ns : 512) : A.ns, 8), seqs);
    launch_pdl(attn_combine_kernel, cg, 256, 0, s, A.part, A.ao, count, seqs, ta.splits, D.nt,
               D.heads, A.ns, D.d, int(ao_half));
  }
  return cudaGetLastError();
}

}  // namespace nvrec
