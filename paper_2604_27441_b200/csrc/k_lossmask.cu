// k_lossmask.cu -- integer loss-mask construction and masked-patch lists.
//
// lossmask_kernel restates, bit-exactly, the reference P-frame mask path:
//   receiver.py:224-237   missing body shard i in [1, n_data) zero-fills
//                         payload bytes [(i-1)L, min(iL, body_len))
//   codec.py:180-201      parse_header (validation order and messages kept
//                         as status codes)
//   codec.py:172-177      block_ranges: [off_j, off_{j+1}), last ends at
//                         payload_len
//   codec.py:274-278      short payload => extra zero range at the tail
//   codec.py:250-257      flag_j = OR_r (s_j < z1_r && e_j > z0_r), z1 > z0
//   codec.py:318-320      grid[present_ids[flagged]] = True
//   recovery.py:221       np.packbits(grid) (MSB-first) = the wire bitset
// One CTA per frame, one thread per bitmap byte (8 blocks).  For a
// well-formed block (s_j < e_j) only the shards overlapping [s_j, e_j) are
// tested (SURVEY.md Appendix B closed form); malformed ranges fall back to
// the literal loop over all shards, so the kernel is exact for every header
// the parser accepts.
//
// masklist_kernel turns a wire bitset into the ascending list of masked
// patches of one stream (+ inverse rank table), which the pruned last block
// and the head consume (server.py:196 discards every unmasked prediction).
#include "launch.cuh"

namespace nvrec {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t ld_u32le(const uint8_t* p) {
  return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) |
         (uint32_t(p[3]) << 24);
}

// Block-wide exclusive scan of one int per thread; returns the exclusive
// prefix and writes the block total to *total.
__device__ int block_exclusive_scan(int v, int* total, int* sh /*[32]*/) {
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
__device__ bool hits_shards(const ShardView& v, int64_t s, int64_t e) {
  if (v.i_cap < 1) return false;
  int64_t lo_i = 1, hi_i = v.i_cap;
  if (s < e) {
    if (v.body_len <= s) return false;
    lo_i = s / v.L + 1; if (lo_i < 1) lo_i = 1;       // first shard with hi_i > s
    hi_i = (e - 1) / v.L + 1; if (hi_i > v.i_cap) hi_i = v.i_cap;  // last shard with lo_i < e
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

}  // namespace

__global__ void __launch_bounds__(kThreads)
lossmask_kernel(const nvrec_lossmask_job* __restrict__ jobs) {
  __shared__ int sh_scan[32];
  __shared__ int sh_err, sh_flagged;
  const nvrec_lossmask_job job = jobs[blockIdx.x];
  const uint8_t* hdr = job.header;
  if (threadIdx.x == 0) { sh_err = 0; sh_flagged = 0; }
  __syncthreads();

  // ---- parse_header (codec.py:180-201) -------------------------------------
  int err = 0;
  int w = 0, h = 0, block = 0, n_present = 0, n_blocks = 0, bitmap_len = 0;
  uint32_t payload_len = 0;
  if (job.header_len < 14) {
    err = 1;                                   // "header truncated"
  } else {
    w = hdr[2] | (hdr[3] << 8);
    h = hdr[4] | (hdr[5] << 8);
    block = hdr[6];
    payload_len = ld_u32le(hdr + 8);
    n_present = hdr[12] | (hdr[13] << 8);
    if (block == 0 || w % block || h % block) {
      err = 2;                                 // "inconsistent geometry"
    } else {
      n_blocks = (w / block) * (h / block);
      bitmap_len = (n_blocks + 7) / 8;
      if (job.header_len < 14 + bitmap_len + 4 * n_present) err = 3;
      else if (n_blocks > job.grid_capacity) err = 5;
    }
  }
  const uint8_t* bitmap = hdr + 14;
  const uint8_t* offs = hdr + 14 + bitmap_len;

  const int nd = job.n_data;
  ShardView sv;
  sv.L = job.shard_len;
  sv.body_len = job.body_len;
  sv.received = job.received;
  {
    int64_t nonempty = job.body_len > 0 ? (job.body_len + sv.L - 1) / sv.L : 0;
    sv.i_cap = int(nonempty < int64_t(nd - 1) ? nonempty : int64_t(nd - 1));
  }
  const bool tail = !err && job.payload_received < int64_t(payload_len);

  // ---- per present block flags (codec.py:250-257,318-320) -------------------
  int rank_base = 0;
  for (int byte0 = 0; byte0 < bitmap_len && !err; byte0 += blockDim.x) {
    int t = byte0 + threadIdx.x;
    uint32_t bits = 0;
    if (t < bitmap_len) {
      bits = bitmap[t];
      int valid = n_blocks - 8 * t;                     // unpackbits(count=)
      if (valid < 8) bits &= (0xFFu << (8 - valid)) & 0xFFu;
    }
    int tot;
    int r = rank_base + block_exclusive_scan(__popc(bits), &tot, sh_scan);
    rank_base += tot;
    if (t < bitmap_len) {
      uint32_t wire = 0;
      int nflag = 0;
      for (int bit = 0; bit < 8; ++bit) {
        int j = 8 * t + bit;
        if (j >= n_blocks) break;
        uint8_t g = 0;
        if (bits & (0x80u >> bit)) {
          if (r < n_present) {
            int64_t s = ld_u32le(offs + 4 * r);
            int64_t e = (r + 1 < n_present) ? int64_t(ld_u32le(offs + 4 * (r + 1)))
                                            : int64_t(payload_len);
            bool f = hits_shards(sv, s, e);
            if (!f && tail) f = s < int64_t(payload_len) && e > job.payload_received;
            for (int x = 0; x < job.n_extra && !f; ++x) {
              int64_t z0 = job.extra_ranges[2 * x], z1 = job.extra_ranges[2 * x + 1];
              if (z1 > z0 && s < z1 && e > z0) f = true;
            }
            g = f ? 1 : 0;
          }
          ++r;
        }
        job.grid[j] = g;
        wire |= uint32_t(g) << (7 - bit);
        nflag += g;
      }
      if (job.wire_bits) job.wire_bits[t] = uint8_t(wire);
      if (nflag) atomicAdd(&sh_flagged, nflag);
    }
  }
  if (!err && rank_base != n_present) err = 4;   // "bitmap disagrees with present count"
  __syncthreads();
  if (threadIdx.x == 0) {
    job.status[0] = err;
    job.status[1] = err ? 0 : sh_flagged;
    job.status[2] = (err || !block) ? 0 : h / block;
    job.status[3] = (err || !block) ? 0 : w / block;
  }
}

// Wire bitset (b, nbytes) -> ascending masked-patch list, rank table, count.
__global__ void __launch_bounds__(kThreads)
masklist_kernel(const uint8_t* __restrict__ bits, int nbytes, int ns,
                int* __restrict__ list, int* __restrict__ rank, int* __restrict__ count) {
  __shared__ int sh_scan[32];
  const int b = blockIdx.x;
  const uint8_t* mb = bits + size_t(b) * nbytes;
  int* lst = list + size_t(b) * ns;
  int* rk = rank + size_t(b) * ns;
  int base = 0;
  for (int byte0 = 0; byte0 < nbytes; byte0 += blockDim.x) {
    int t = byte0 + threadIdx.x;
    uint32_t v = 0;
    if (t < nbytes) {
      v = mb[t];
      int valid = ns - 8 * t;
      if (valid < 8) v &= valid > 0 ? (0xFFu << (8 - valid)) & 0xFFu : 0u;
    }
    int tot;
    int r = base + block_exclusive_scan(__popc(v), &tot, sh_scan);
    base += tot;
    for (int bit = 0; bit < 8; ++bit) {
      int s = 8 * t + bit;
      if (t >= nbytes || s >= ns) break;
      if (v & (0x80u >> bit)) { lst[r] = s; rk[s] = r; ++r; }
      else rk[s] = -1;
    }
  }
  if (threadIdx.x == 0) count[b] = base;
}

// ---------------------------------------------------------------------------
cudaError_t launch_lossmask(const nvrec_lossmask_job* jobs, int n_jobs, cudaStream_t s) {
  if (n_jobs <= 0) return cudaSuccess;
  lossmask_kernel<<<n_jobs, kThreads, 0, s>>>(jobs);
  return cudaGetLastError();
}

cudaError_t launch_masklist(const uint8_t* bits, int b, int nbytes, int ns, int* list,
                            int* rank, int* count, cudaStream_t s) {
  masklist_kernel<<<b, kThreads, 0, s>>>(bits, nbytes, ns, list, rank, count);
  return cudaGetLastError();
}

}  // namespace nvrec
