// k_decode.cu -- zero-fill frame decode on the GPU:
// the corrupted plane and its corruption mask that the recovery path
// consumes, bit-exact with rgbdstream codec.decode (codec.py:260-321).
//
// Per frame the reference (1) parses the header and flags every present
// block whose payload range meets a zero-filled range (the loss mask),
// (2) concatenates the payload ranges of the clean blocks, RLE-decodes the
// concatenation (3-byte records: u8 run, u16 zigzag value, codec.py:25,
// 134-138) and (3) writes reference + unzigzag(v) * quant (int16 wrap,
// clip to [0,255]) -- or clip(int16(v) * quant) for an I-frame -- into the
// clean blocks, channel-planar within a block (codec.py:85-96,296-317);
// every other block keeps the reference (P) or zero (I).
//
// Four launches per batch of frames:
//   decode_parse_kernel   one CTA per frame: lm::lossmask_job (the mask path
//                         of k_lossmask.cu) + per-block present rank table.
//   decode_copy_kernel    base plane: the reference (P) or zeros (I), 16 B
//                         per thread, grid-stride (HBM-bound).
//   decode_present_kernel one warp per present block: RLE-decodes the block's
//                         own payload range
//                         (warp scan of the run lengths, run starts marked in
//                         shared memory, carry-forward scan) and writes the
//                         reconstructed pixels.  Exact whenever every clean
//                         block's range is whole records decoding to exactly
//                         block*block*c samples -- true for any stream the
//                         encoder produces, because runs break at block
//                         boundaries (codec.py:105-131).  Otherwise it raises
//                         the frame's slow flag.
//   decode_final_kernel   frames with the slow flag only: one thread replays
//                         the literal reference semantics (python slicing of
//                         each range, concatenation, records straddling
//                         ranges, the two error checks in reference order);
//                         then undecodable frames get the error policy
//                         (plane = decode reference, wire bits cleared).
// All four are stream-ordered and graph capturable; nothing syncs the host.
#include "launch.cuh"
#include "lossmask.cuh"

namespace nvrec {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxBs = 768;               // 16 x 16 x 3 samples per block (fast path)
constexpr int32_t kFlagBit = 1 << 30;
constexpr int kParseStage = 40 * 1024;    // header + received flags staged in smem
constexpr int kParseThreads = 1024;       // one bitmap byte per thread up to 8192 blocks

struct Fixed {
  int kind, c, w, h, block, quant, n_present;
  uint32_t payload_len;
  int bitmap_len, n_blocks;
};

__device__ __forceinline__ Fixed read_fixed(const uint8_t* hdr) {
  Fixed f;
  f.kind = hdr[0];
  f.c = hdr[1];
  f.w = hdr[2] | (hdr[3] << 8);
  f.h = hdr[4] | (hdr[5] << 8);
  f.block = hdr[6];
  f.quant = hdr[7];
  f.payload_len = lm::ld_u32le(hdr + 8);
  f.n_present = hdr[12] | (hdr[13] << 8);
  f.n_blocks = (f.w / f.block) * (f.h / f.block);
  f.bitmap_len = (f.n_blocks + 7) / 8;
  return f;
}

// codec.py:146-148 then * int16(quant) (int16 wrap) + reference (int16
// wrap), clip [0, 255]; I-frames: clip(int16(v) * int16(quant)).
__device__ __forceinline__ uint8_t reconstruct(int kind, uint32_t v, int quant, uint8_t ref) {
  int16_t x;
  if (kind == 0) {
    x = int16_t(int16_t(uint16_t(v)) * int16_t(quant));
  } else {
    const int16_t uz = int16_t(uint16_t(v >> 1)) ^ int16_t(-int16_t(v & 1));
    const int16_t d = int16_t(uz * int16_t(quant));
    x = int16_t(int16_t(ref) + d);
  }
  return uint8_t(x < 0 ? 0 : (x > 255 ? 255 : x));
}

__device__ __forceinline__ int64_t block_end(const Fixed& f, const uint8_t* offs, int r) {
  return r + 1 < f.n_present ? int64_t(lm::ld_u32le(offs + 4 * (r + 1))) : int64_t(f.payload_len);
}

}  // namespace

__global__ void __launch_bounds__(kParseThreads)
decode_parse_kernel(const nvrec_decode_job* __restrict__ jobs) {
  pdl_entry();
  __shared__ int sh_scan[32];
  __shared__ int sh_flagged;
  extern __shared__ uint8_t stage[];
  const nvrec_decode_job job = jobs[blockIdx.x];
  lm::Header H;
  int err = lm::lossmask_job(job.mask, job.scratch + 4, &H, sh_scan, &sh_flagged, stage,
                             kParseStage, job.scratch + 4 + job.mask.grid_capacity);
  if (threadIdx.x == 0) {
    if (!err && H.kind == 1 && !job.reference) err = lm::kNeedReference;
    if (!err && int64_t(H.h) * H.w * H.channels > job.plane_capacity) err = lm::kPlaneCapacity;
    if (err) job.mask.status[0] = err;
    job.scratch[0] = 0;                       // slow-path flag
  }
}

// Base plane: the reference (P) or zeros (I), grid-stride, 16 B per thread
// where aligned; clean present blocks are overwritten by the next kernel.
__global__ void __launch_bounds__(kThreads)
decode_copy_kernel(const nvrec_decode_job* __restrict__ jobs) {
  pdl_entry();
  const nvrec_decode_job& jr = jobs[blockIdx.y];
  if (jr.mask.status[0] != 0) return;
  const Fixed f = read_fixed(jr.mask.header);
  const uint8_t* ref = jr.reference;
  uint8_t* out = jr.plane;
  if (f.kind == 1 && ref == out) return;                 // in-place decode
  const size_t bytes = size_t(f.h) * f.w * f.c;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  const size_t t0 = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (((reinterpret_cast<uintptr_t>(ref) | reinterpret_cast<uintptr_t>(out) | bytes) & 15) == 0) {
    const uint4* src = reinterpret_cast<const uint4*>(ref);
    uint4* dst = reinterpret_cast<uint4*>(out);
    for (size_t i = t0; i < bytes / 16; i += stride)
      dst[i] = f.kind == 1 ? __ldg(src + i) : make_uint4(0, 0, 0, 0);
  } else {
    for (size_t i = t0; i < bytes; i += stride) out[i] = f.kind == 1 ? ref[i] : 0;
  }
}

// One present block (rank r) per warp: RLE-decode the block's own payload
// range and write reference + delta (P) / value (I).
__device__ __forceinline__ void decode_one(const nvrec_decode_job& jr, const Fixed& f, int r,
                                           uint32_t* mk, uint8_t* rec, int lane) {
  __syncwarp();                                        // previous block's buffers drained
  const int32_t pid = jr.scratch[4 + jr.mask.grid_capacity + r];
  if (pid & kFlagBit) return;                          // corrupted: keeps the base
  const int j = pid;
  const int wb = f.w / f.block;
  const int by = j / wb, bx = j - by * wb;
  const int rowb = f.block * f.c;                     // bytes per block row
  const size_t pitch = size_t(f.w) * f.c;
  const size_t base = size_t(by) * f.block * pitch + size_t(bx) * rowb;
  const uint8_t* ref = jr.reference;
  uint8_t* out = jr.plane;
  const int bs = f.block * f.block * f.c;

  // clean present block: decode its own payload range
  const uint8_t* offs = jr.mask.header + 14 + f.bitmap_len;
  const int64_t s = lm::ld_u32le(offs + 4 * r);
  const int64_t e = block_end(f, offs, r);
  const int64_t avail = jr.mask.payload_received;     // len(enc.payload)
  bool ok = bs <= kMaxBs && s < e && e <= avail && (e - s) % 3 == 0 && e - s <= 3 * kMaxBs;
  if (ok) {
    // the block's records in one round trip (all lanes' loads in flight)
    const uint8_t* src = jr.payload + s;
    for (int i = lane; i < int(e - s); i += 32) rec[i] = __ldg(src + i);
    for (int p = lane; p < bs; p += 32) mk[p] = 0;
    __syncwarp();
    const uint8_t* pay = rec;
    const int nrec = int((e - s) / 3);
    int pos = 0;                                       // samples so far
    for (int r0 = 0; r0 < nrec && pos <= bs; r0 += 32) {
      const int ri = r0 + lane;
      int run = 0;
      uint32_t val = 0;
      if (ri < nrec) {
        run = pay[3 * ri];
        val = uint32_t(pay[3 * ri + 1]) | (uint32_t(pay[3 * ri + 2]) << 8);
      }
      int incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int start = pos + incl - run;
      if (run > 0 && start < bs) mk[start] = 0x10000u | val;
      pos += __shfl_sync(0xffffffffu, incl, 31);
    }
    ok = pos == bs;
  }
  if (!ok) {
    if (lane == 0) atomicOr(jr.scratch, 1);
    return;
  }
  __syncwarp();
  // carry-forward: every sample position takes the value of the last run
  // start at or before it (position 0 always starts a run)
  const int per = (bs + 31) / 32;
  const int p0 = lane * per, p1 = min(bs, p0 + per);
  uint32_t last = 0;
  for (int p = p0; p < p1; ++p)
    if (mk[p]) last = mk[p];
  uint32_t incl = last;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o && !incl) incl = y;
  }
  uint32_t cur = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) cur = 0;
  for (int p = p0; p < p1; ++p) {
    if (mk[p]) cur = mk[p];
    mk[p] = cur;
  }
  __syncwarp();
  // one pixel (all channels) per lane step: samples are channel-planar
  // (sample = ch * block^2 + y * block + x), pixels interleaved in the plane
  const int bb = f.block * f.block;
  const int lg = f.block == 16 ? 4 : -1;             // shift instead of divide (16-px blocks)
  for (int q = lane; q < bb; q += 32) {
    const int y = lg > 0 ? q >> lg : q / f.block;
    const int x = q - y * f.block;
    const size_t off = base + size_t(y) * pitch + size_t(x) * f.c;
    for (int ch = 0; ch < f.c; ++ch) {
      const uint32_t v = mk[ch * bb + q] & 0xFFFFu;
      out[off + ch] = reconstruct(f.kind, v, f.quant, f.kind == 1 ? ref[off + ch] : 0);
    }
  }
}

// Warps stride over the present ranks (grid sized for ~1/4 of the blocks).
__global__ void __launch_bounds__(kThreads)
decode_present_kernel(const nvrec_decode_job* __restrict__ jobs) {
  pdl_entry();
  __shared__ uint32_t sh_mark[kWarps][kMaxBs];
  __shared__ uint8_t sh_rec[kWarps][3 * kMaxBs];
  const nvrec_decode_job& jr = jobs[blockIdx.y];
  if (jr.mask.status[0] != 0) return;
  const Fixed f = read_fixed(jr.mask.header);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = blockIdx.x * kWarps + warp; r < f.n_present; r += gridDim.x * kWarps) {
    decode_one(jr, f, r, sh_mark[warp], sh_rec[warp], lane);
  }
}

// Literal replay of codec.py:283-317 for frames the fast path rejected.
__device__ void decode_slow(const nvrec_decode_job& jr) {
  if (jr.mask.status[0] != 0 || jr.scratch[0] == 0) return;
  const Fixed f = read_fixed(jr.mask.header);
  const uint8_t* offs = jr.mask.header + 14 + f.bitmap_len;
  const int32_t* brank = jr.scratch + 4;
  const int64_t avail = jr.mask.payload_received;
  // payload after the tail pad (codec.py:274-278): max(len, payload_len) bytes
  const int64_t PL = avail > int64_t(f.payload_len) ? avail : int64_t(f.payload_len);
  auto byte_at = [&](int64_t x) -> uint32_t { return x < avail ? jr.payload[x] : 0u; };
  auto slice = [&](int j, int64_t* a, int64_t* b) {
    const int r = brank[j] & (kFlagBit - 1);
    const int64_t s = lm::ld_u32le(offs + 4 * r), e = block_end(f, offs, r);
    *a = s < PL ? s : PL;                              // python payload[s:e]
    const int64_t ee = e > s ? e : s;
    *b = ee < PL ? ee : PL;
  };
  auto clean = [&](int j) { return brank[j] >= 0 && !(brank[j] & kFlagBit); };
  int64_t total = 0, n_clean = 0;
  for (int j = 0; j < f.n_blocks; ++j) {
    if (!clean(j)) continue;
    int64_t a, b;
    slice(j, &a, &b);
    total += b - a;
    ++n_clean;
  }
  if (total % 3) { jr.mask.status[0] = lm::kNotWholeRecords; return; }
  const int64_t bs = int64_t(f.block) * f.block * f.c;

  // byte cursor over the concatenation of the clean slices
  struct Cursor { int j; int64_t x, b; };
  auto next_slice = [&](Cursor& cu) {
    while (cu.x >= cu.b) {
      ++cu.j;
      while (cu.j < f.n_blocks && !clean(cu.j)) ++cu.j;
      if (cu.j >= f.n_blocks) return false;
      slice(cu.j, &cu.x, &cu.b);
    }
    return true;
  };
  auto get = [&](Cursor& cu) -> uint32_t {
    next_slice(cu);
    return byte_at(cu.x++);
  };
  const int64_t nrec = total / 3;
  {
    Cursor cu{-1, 0, 0};
    int64_t samples = 0;
    for (int64_t k = 0; k < nrec; ++k) {
      samples += get(cu);
      get(cu);
      get(cu);
    }
    if (samples != n_clean * bs) { jr.mask.status[0] = lm::kSampleCount; return; }
  }
  // write: sample p belongs to the (p / bs)-th clean block, channel-planar
  Cursor cu{-1, 0, 0};
  int ob = -1;                                         // current output block
  int64_t p = 0;
  const int wb = f.w / f.block, bb = f.block * f.block;
  const size_t pitch = size_t(f.w) * f.c;
  for (int64_t k = 0; k < nrec; ++k) {
    const uint32_t run = get(cu);
    uint32_t v = get(cu);
    v |= get(cu) << 8;
    for (uint32_t t = 0; t < run; ++t, ++p) {
      const int64_t q = p % bs;
      if (q == 0) {
        ++ob;
        while (!clean(ob)) ++ob;
      }
      const int ch = int(q / bb), y = int((q % bb) / f.block), x = int(q % f.block);
      const int by = ob / wb, bx = ob - by * wb;
      const size_t off = (size_t(by) * f.block + y) * pitch + (size_t(bx) * f.block + x) * f.c + ch;
      jr.plane[off] = reconstruct(f.kind, v, f.quant, f.kind == 1 ? jr.reference[off] : 0);
    }
  }
}

// Last launch per batch: the slow path (thread 0), then the error policy.
// A frame whose decode failed (UndecodableError -> LOST_FRAME, receiver.py:
// 244-248) is not displayed by the reference and leaves its references
// alone; here its slot joins the cyclic ring, so it receives a copy of the
// decode reference (the newest displayable plane: the next P-frame decodes
// against the same plane as in the reference) and its wire bits are cleared
// (the recovery launch that follows in the same graph changes nothing).
__global__ void __launch_bounds__(256) decode_final_kernel(const nvrec_decode_job* __restrict__ jobs) {
  pdl_entry();
  const nvrec_decode_job& jr = jobs[blockIdx.x];
  if (threadIdx.x == 0) decode_slow(jr);
  __syncthreads();
  if (jr.mask.status[0] == 0) return;
  if (jr.mask.wire_bits)
    for (int t = threadIdx.x; t < (jr.mask.grid_capacity + 7) / 8; t += blockDim.x)
      jr.mask.wire_bits[t] = 0;
  const uint8_t* ref = jr.reference;
  uint8_t* out = jr.plane;
  if (!ref || ref == out) return;
  const size_t bytes = size_t(jr.plane_capacity);
  if (((reinterpret_cast<uintptr_t>(ref) | reinterpret_cast<uintptr_t>(out) | bytes) & 15) == 0) {
    for (size_t i = threadIdx.x; i < bytes / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(out)[i] = __ldg(reinterpret_cast<const uint4*>(ref) + i);
  } else {
    for (size_t i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = ref[i];
  }
}

cudaError_t launch_decode(const nvrec_decode_job* jobs, int n_jobs, int max_blocks,
                          cudaStream_t s) {
  if (n_jobs <= 0) return cudaSuccess;
  launch_pdl(decode_parse_kernel, n_jobs, kParseThreads, kParseStage, s, jobs);
  launch_pdl(decode_copy_kernel, dim3((2 * sm_count() + n_jobs - 1) / n_jobs * 2, n_jobs), kThreads, 0, s, jobs);
  dim3 grid((max_blocks + 4 * kWarps - 1) / (4 * kWarps), n_jobs);
  launch_pdl(decode_present_kernel, grid, kThreads, 0, s, jobs);
  launch_pdl(decode_final_kernel, n_jobs, 256, 0, s, jobs);
  return cudaGetLastError();
}

}  // namespace nvrec
