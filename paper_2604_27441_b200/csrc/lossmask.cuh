// lossmask.cuh -- the codec-header parse + per-block corruption flags shared
// by the loss-mask kernel (k_lossmask.cu) and the frame decoder
// (k_decode.cu).  Restates, bit-exactly:
//   receiver.py:224-237   missing body shard i in [1, n_data) zero-fills
//                         payload bytes [(i-1)L, min(iL, body_len))
//   codec.py:180-201      parse_header (validation order kept as status codes;
//                         FrameKind(kind) is checked last, as _Header's
//                         constructor does)
//   codec.py:172-177      block_ranges: [off_j, off_{j+1}), last ends at
//                         payload_len
//   codec.py:274-278      short payload => extra zero range at the tail
//   codec.py:250-257      flag_j = OR_r (s_j < z1_r && e_j > z0_r), z1 > z0
//   codec.py:318-320      grid[present_ids[flagged]] = True
//   recovery.py:221       np.packbits(grid) (MSB-first) = the wire bitset
// One CTA per frame, one thread per bitmap byte (8 blocks).  For a
// well-formed block (s_j < e_j) only the shards overlapping [s_j, e_j) are
// tested (SURVEY.md Appendix B closed form); malformed ranges fall back to
// the literal loop over all shards, so the result is exact for every header
// the parser accepts.
#pragma once

#include <cstdint>

#include "nvrec_b200.h"

namespace nvrec {
namespace lm {

// status codes (nvrec_lossmask_job.status[0] / nvrec_decode_job status)
enum : int {
  kOk = 0,
  kHeaderTruncated = 1,        // "header truncated"
  kBadGeometry = 2,            // "inconsistent geometry in header"
  kHeaderTruncated2 = 3,       // "header truncated" (bitmap/offsets)
  kBitmapCount = 4,            // "bitmap disagrees with present count"
  kGridCapacity = 5,           // grid_capacity too small (caller error)
  kNotWholeRecords = 6,        // "payload range is not whole RLE records"
  kSampleCount = 7,            // "payload sample count disagrees with header"
  kNeedReference = 8,          // "P-frame decode requires a reference plane"
  kPlaneCapacity = 9,          // plane_capacity too small (caller error)
  kBadKind = 10,               // FrameKind(kind) ValueError
};

__device__ __forceinline__ uint32_t ld_u32le(const uint8_t* p) {
  return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) |
         (uint32_t(p[3]) << 24);
}

// Block-wide exclusive scan of one int per thread; returns the exclusive
// prefix and writes the block total to *total.
__device__ __forceinline__ int block_exclusive_scan(int v, int* total, int* sh /*[32]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int nw = blockDim.x >> 5;
    int w = lane < nw ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) sh[lane] = w;  // inclusive per-warp totals
  }
  __syncthreads();
  int warp_base = warp ? sh[warp - 1] : 0;
  *total = sh[(blockDim.x >> 5) - 1];
  __syncthreads();
  return warp_base + x - v;
}

struct ShardView {
  int i_cap;               // last body shard index with a non-empty range
  int64_t L, body_len;
  const uint8_t* received;
};

// Does payload range [s, e) intersect any zero-filled shard range?  Only the
// shards overlapping [s, e) can match, so the loop is 1-4 iterations for a
// well-formed block (a block payload is at most a few shard lengths).
__device__ __forceinline__ bool hits_shards(const ShardView& v, int64_t s, int64_t e) {
  if (v.i_cap < 1) return false;
  int64_t lo_i = 1, hi_i = v.i_cap;
  if (s < e) {
    if (v.body_len <= s) return false;
    if (s >= 0 && e <= 0xFFFFFFFFll && v.L > 0 && v.L <= 0xFFFFFFFFll) {
      // 32-bit unsigned division (a 64-bit one is a ~70-instruction routine)
      const uint32_t L32 = uint32_t(v.L);
      lo_i = int64_t(uint32_t(s) / L32) + 1;
      hi_i = int64_t(uint32_t(e - 1) / L32) + 1;
    } else {
      lo_i = s / v.L + 1;
      hi_i = (e - 1) / v.L + 1;
    }
    if (lo_i < 1) lo_i = 1;                             // first shard with hi_i > s
    if (hi_i > v.i_cap) hi_i = v.i_cap;                 // last shard with lo_i < e
  }
  for (int64_t i = lo_i; i <= hi_i; ++i) {
    if (v.received[i]) continue;
    int64_t z0 = (i - 1) * v.L;
    int64_t z1 = min(z0 + v.L, v.body_len);
    if (z1 <= z0) continue;
    if (s < z1 && e > z0) return true;
  }
  return false;
}

// Parsed fixed header fields (codec.py:26,183-189).
struct Header {
  int kind, channels, w, h, block, quant, n_present, n_blocks, bitmap_len;
  uint32_t payload_len;
  const uint8_t* bitmap;
  const uint8_t* offs;
};

// The whole mask job for one frame, executed by one CTA.  Writes grid,
// wire_bits and status exactly like nvrec_loss_mask.  When block_rank is
// non-null it also receives, per block j, the present rank r of the block
// (bit 30 set when flagged) or -1 for an absent block -- the index the
// decoder needs to find the block's payload range -- and present_id the
// inverse (present rank -> block, same flag bit).  Returns the status.
// stage: optional shared-memory buffer (stage_cap bytes); when the header and
// the received flags fit they are copied there once (one coalesced round
// trip) and every later parse step reads shared memory.
__device__ inline int lossmask_job(const nvrec_lossmask_job& job_in, int32_t* block_rank,
                                   Header* out_hdr, int* sh_scan /*[32]*/, int* sh_flagged,
                                   uint8_t* stage = nullptr, int stage_cap = 0,
                                   int32_t* present_id = nullptr) {
  nvrec_lossmask_job job = job_in;
  if (stage && job.header_len >= 0 && job.n_data >= 0 &&
      job.header_len + job.n_data <= stage_cap) {
    for (int i = threadIdx.x; i < job.header_len; i += blockDim.x) stage[i] = job.header[i];
    for (int i = threadIdx.x; i < job.n_data; i += blockDim.x)
      stage[job.header_len + i] = job.received[i];
    job.header = stage;
    job.received = stage + job.header_len;
  }
  const uint8_t* hdr = job.header;
  if (threadIdx.x == 0) *sh_flagged = 0;
  __syncthreads();

  // ---- parse_header (codec.py:180-201) -------------------------------------
  int err = kOk;
  Header H{};
  if (job.header_len < 14) {
    err = kHeaderTruncated;
  } else {
    H.kind = hdr[0];
    H.channels = hdr[1];
    H.w = hdr[2] | (hdr[3] << 8);
    H.h = hdr[4] | (hdr[5] << 8);
    H.block = hdr[6];
    H.quant = hdr[7];
    H.payload_len = ld_u32le(hdr + 8);
    H.n_present = hdr[12] | (hdr[13] << 8);
    if (H.block == 0 || H.w % H.block || H.h % H.block) {
      err = kBadGeometry;
    } else {
      H.n_blocks = (H.w / H.block) * (H.h / H.block);
      H.bitmap_len = (H.n_blocks + 7) / 8;
      if (job.header_len < 14 + H.bitmap_len + 4 * H.n_present) err = kHeaderTruncated2;
      else if (H.n_blocks > job.grid_capacity) err = kGridCapacity;
    }
  }
  H.bitmap = hdr + 14;
  H.offs = hdr + 14 + H.bitmap_len;

  const int nd = job.n_data;
  ShardView sv;
  sv.L = job.shard_len;
  sv.body_len = job.body_len;
  sv.received = job.received;
  {
    int64_t nonempty = job.body_len > 0 ? (job.body_len + sv.L - 1) / sv.L : 0;
    sv.i_cap = int(nonempty < int64_t(nd - 1) ? nonempty : int64_t(nd - 1));
  }
  const bool tail = !err && job.payload_received < int64_t(H.payload_len);

  // ---- per present block flags (codec.py:250-257,318-320) -------------------
  int rank_base = 0;
  for (int byte0 = 0; byte0 < H.bitmap_len && !err; byte0 += blockDim.x) {
    int t = byte0 + threadIdx.x;
    uint32_t bits = 0;
    if (t < H.bitmap_len) {
      bits = H.bitmap[t];
      int valid = H.n_blocks - 8 * t;                   // unpackbits(count=)
      if (valid < 8) bits &= (0xFFu << (8 - valid)) & 0xFFu;
    }
    int tot;
    int r = rank_base + block_exclusive_scan(__popc(bits), &tot, sh_scan);
    rank_base += tot;
    if (t < H.bitmap_len) {
      uint32_t wire = 0;
      int nflag = 0;
      for (int bit = 0; bit < 8; ++bit) {
        int j = 8 * t + bit;
        if (j >= H.n_blocks) break;
        uint8_t g = 0;
        int32_t br = -1;
        if (bits & (0x80u >> bit)) {
          if (r < H.n_present) {
            int64_t s = ld_u32le(H.offs + 4 * r);
            int64_t e = (r + 1 < H.n_present) ? int64_t(ld_u32le(H.offs + 4 * (r + 1)))
                                              : int64_t(H.payload_len);
            bool f = hits_shards(sv, s, e);
            if (!f && tail) f = s < int64_t(H.payload_len) && e > job.payload_received;
            for (int x = 0; x < job.n_extra && !f; ++x) {
              int64_t z0 = job.extra_ranges[2 * x], z1 = job.extra_ranges[2 * x + 1];
              if (z1 > z0 && s < z1 && e > z0) f = true;
            }
            g = f ? 1 : 0;
            br = r | (f ? (1 << 30) : 0);
            if (present_id) present_id[r] = j | (f ? (1 << 30) : 0);
          }
          ++r;
        }
        job.grid[j] = g;
        if (block_rank) block_rank[j] = br;
        wire |= uint32_t(g) << (7 - bit);
        nflag += g;
      }
      if (job.wire_bits) job.wire_bits[t] = uint8_t(wire);
      if (nflag) atomicAdd(sh_flagged, nflag);
    }
  }
  if (!err && rank_base != H.n_present) err = kBitmapCount;
  if (!err && H.kind > 1) err = kBadKind;
  __syncthreads();
  // an undecodable frame (LOST_FRAME in the reference, receiver.py:244-248)
  // recovers nothing: clear its wire bits so a recovery launch that consumes
  // them (graphs run unconditionally) leaves the plane untouched
  if (err && job.wire_bits)
    for (int t = threadIdx.x; t < (job.grid_capacity + 7) / 8; t += blockDim.x) job.wire_bits[t] = 0;
  if (threadIdx.x == 0) {
    job.status[0] = err;
    job.status[1] = err ? 0 : *sh_flagged;
    job.status[2] = (err || !H.block) ? 0 : H.h / H.block;
    job.status[3] = (err || !H.block) ? 0 : H.w / H.block;
  }
  if (out_hdr) {
    *out_hdr = H;
    out_hdr->bitmap = job_in.header + 14;               // global copies stay valid
    out_hdr->offs = job_in.header + 14 + H.bitmap_len;
  }
  return err;
}

}  // namespace lm
}  // namespace nvrec
