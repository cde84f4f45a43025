// k_baseline.cu -- the reference's timeout / fault fallback on the GPU,
// bit-exact (rgbdstream/recovery.py:94-196):
//
// baseline_match_kernel<C>  one CTA per masked 16-px block.  The +-8 px
//   search window of the most recent reference (34 x 34 px incl. the 1-px
//   ring, clamped at the frame edge) is staged in shared memory together
//   with the block's template: the intact pixels of its one-pixel border ring
//   in the corrupted plane (_ring_coords :94-106, in-bounds and not masked),
//   or -- when the whole ring is masked -- the block's own 256 pixels.  Each
//   of the 289 shifts is one thread: integer SAD over the in-bounds template
//   positions, score = SAD / #valid + 1e-6 (|dy| + |dx|) in float64 exactly
//   as numpy computes it (_best_shift :109-125), first minimum in (dy, dx)
//   raster order; the block is then copied from the shifted, edge-clamped
//   reference window.
// baseline_median_kernel    depth only (:162-184): on the masked bounding
//   box +-2 px, pixels on the two-pixel band straddling the mask boundary
//   (4-connected dilation, outside the box counts as unmasked-free) take the
//   3x3 median with 'nearest' edges at the box border.  32 x 32 output tiles
//   with a 1-px halo of the block-match result and of the mask staged in
//   shared memory.
#include <algorithm>
#include <cfloat>
#include <climits>

#include "launch.cuh"

namespace nvrec {

namespace {

constexpr int kB = 16, kR = 8;
constexpr int kWin = kB + 2 + 2 * kR;      // 34: ring + search radius on both sides

__device__ __forceinline__ bool masked_px(const uint8_t* bits, int gw, int y, int x) {
  const int j = (y >> 4) * gw + (x >> 4);
  return (bits[j >> 3] >> (7 - (j & 7))) & 1;
}

template <int C>
__global__ void __launch_bounds__(320)
baseline_match_kernel(const uint8_t* __restrict__ planes, const uint8_t* __restrict__ refs,
                      const uint8_t* __restrict__ mask_bits, const int* __restrict__ list,
                      const int* __restrict__ count, uint8_t* __restrict__ out, int h, int w,
                      int ns, int nbytes) {
  pdl_entry();
  __shared__ uint8_t win[kWin * kWin * C];
  __shared__ short ty[kB * kB], tx[kB * kB];
  __shared__ uint8_t tv[kB * kB * C];
  __shared__ int n_tmpl, n_ring_intact;
  __shared__ double score[(2 * kR + 1) * (2 * kR + 1)];
  __shared__ int best;
  const int b = blockIdx.y;
  const int gw = w / kB;
  const uint8_t* bits = mask_bits + size_t(b) * nbytes;
  const uint8_t* plane = planes + size_t(b) * h * w * C;
  const uint8_t* ref = refs + size_t(b) * h * w * C;
  uint8_t* o = out + size_t(b) * h * w * C;
  const int cnt = count[b];
  for (int r = blockIdx.x; r < cnt; r += gridDim.x) {
    const int s = list[b * ns + r];
    const int y0 = (s / gw) * kB, x0 = (s % gw) * kB;
    const int wy = y0 - 1 - kR, wx = x0 - 1 - kR;        // window origin
    // stage the reference window (clamped at the frame edge)
    for (int i = threadIdx.x; i < kWin * kWin; i += blockDim.x) {
      const int yy = min(max(wy + i / kWin, 0), h - 1);
      const int xx = min(max(wx + i % kWin, 0), w - 1);
#pragma unroll
      for (int ch = 0; ch < C; ++ch) win[i * C + ch] = ref[(size_t(yy) * w + xx) * C + ch];
    }
    // template: the intact in-bounds ring pixels, in _ring_coords order
    if (threadIdx.x == 0) {
      int n = 0;
      auto take = [&](int yy, int xx) {
        if (yy < 0 || yy >= h || xx < 0 || xx >= w) return;
        if (masked_px(bits, gw, yy, xx)) return;
        ty[n] = short(yy - y0);
        tx[n] = short(xx - x0);
        ++n;
      };
      for (int xx = x0 - 1; xx < x0 + kB + 1; ++xx) {
        take(y0 - 1, xx);
        take(y0 + kB, xx);
      }
      for (int yy = y0; yy < y0 + kB; ++yy) {
        take(yy, x0 - 1);
        take(yy, x0 + kB);
      }
      n_ring_intact = n;
      if (n == 0) {                 // fully masked neighbourhood: the block itself
        for (int i = 0; i < kB * kB; ++i) {
          ty[i] = short(i / kB);
          tx[i] = short(i % kB);
        }
        n = kB * kB;
      }
      n_tmpl = n;
    }
    __syncthreads();
    const int nt = n_tmpl;
    for (int i = threadIdx.x; i < nt; i += blockDim.x) {
      const int yy = y0 + ty[i], xx = x0 + tx[i];
#pragma unroll
      for (int ch = 0; ch < C; ++ch) tv[i * C + ch] = plane[(size_t(yy) * w + xx) * C + ch];
    }
    __syncthreads();
    // one shift per thread
    if (threadIdx.x < (2 * kR + 1) * (2 * kR + 1)) {
      const int dy = int(threadIdx.x) / (2 * kR + 1) - kR;
      const int dx = int(threadIdx.x) % (2 * kR + 1) - kR;
      long long sad = 0;
      int nvalid = 0;
      for (int i = 0; i < nt; ++i) {
        const int yy = y0 + ty[i] + dy, xx = x0 + tx[i] + dx;
        if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
        const uint8_t* c8 = win + ((yy - wy) * kWin + (xx - wx)) * C;
        int d = 0;
#pragma unroll
        for (int ch = 0; ch < C; ++ch) d += abs(int(c8[ch]) - int(tv[i * C + ch]));
        sad += d;
        ++nvalid;
      }
      double sc = nvalid > 0 ? double(sad) / double(nvalid) : __longlong_as_double(0x7ff0000000000000LL);
      sc += 1e-6 * double(abs(dy) + abs(dx));
      score[threadIdx.x] = sc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int bi = 0;
      double bs = score[0];
      for (int i = 1; i < (2 * kR + 1) * (2 * kR + 1); ++i)
        if (score[i] < bs) { bs = score[i]; bi = i; }
      best = bi;
    }
    __syncthreads();
    const int dy = best / (2 * kR + 1) - kR, dx = best % (2 * kR + 1) - kR;
    for (int i = threadIdx.x; i < kB * kB; i += blockDim.x) {
      const int py = i / kB, px = i % kB;
      // ref[clip(y0+py+dy), clip(x0+px+dx)]: the staged window is clamped too
      const uint8_t* src = win + ((py + 1 + kR + dy) * kWin + (px + 1 + kR + dx)) * C;
      uint8_t* dst = o + (size_t(y0 + py) * w + x0 + px) * C;
#pragma unroll
      for (int ch = 0; ch < C; ++ch) dst[ch] = src[ch];
    }
    __syncthreads();
  }
}

// masked bounding box +-2 px per stream: bbox[b] = {y0, y1, x0, x1} (y1/x1
// exclusive), all zero when nothing is masked
__global__ void baseline_bbox_kernel(const int* __restrict__ list, const int* __restrict__ count,
                                     int ns, int gw, int h, int w, int* __restrict__ bbox) {
  pdl_entry();
  const int b = blockIdx.x;
  int ymin = INT_MAX, ymax = -1, xmin = INT_MAX, xmax = -1;
  for (int r = threadIdx.x; r < count[b]; r += blockDim.x) {
    const int s = list[b * ns + r];
    const int by = s / gw, bx = s % gw;
    ymin = min(ymin, by); ymax = max(ymax, by);
    xmin = min(xmin, bx); xmax = max(xmax, bx);
  }
  for (int o = 16; o > 0; o >>= 1) {
    ymin = min(ymin, __shfl_xor_sync(0xffffffffu, ymin, o));
    xmin = min(xmin, __shfl_xor_sync(0xffffffffu, xmin, o));
    ymax = max(ymax, __shfl_xor_sync(0xffffffffu, ymax, o));
    xmax = max(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
  }
  if (threadIdx.x == 0) {
    int* bb = bbox + 4 * b;
    if (ymax < 0) { bb[0] = bb[1] = bb[2] = bb[3] = 0; return; }
    bb[0] = max(ymin * kB - 2, 0);
    bb[1] = min(ymax * kB + kB - 1 + 3, h);
    bb[2] = max(xmin * kB - 2, 0);
    bb[3] = min(xmax * kB + kB - 1 + 3, w);
  }
}

__device__ __forceinline__ uint8_t median9(uint8_t* v) {
  // partial selection: the 5th smallest of 9
#pragma unroll
  for (int i = 0; i < 5; ++i) {
#pragma unroll
    for (int j = i + 1; j < 9; ++j) {
      const uint8_t a = v[i], c = v[j];
      v[i] = min(a, c);
      v[j] = max(a, c);
    }
  }
  return v[4];
}

constexpr int kTile = 32;

// depth plane (c = 1): out = base except on the boundary band of the box
__global__ void __launch_bounds__(kTile * kTile / 4)
baseline_median_kernel(const uint8_t* __restrict__ base, const uint8_t* __restrict__ mask_bits,
                       const int* __restrict__ bbox, uint8_t* __restrict__ out, int h, int w,
                       int nbytes) {
  pdl_entry();
  __shared__ uint8_t sv[kTile + 2][kTile + 2];     // block-match result, 1-px halo
  __shared__ uint8_t sm[kTile + 2][kTile + 2];     // mask, 1-px halo (0 outside the box)
  const int b = blockIdx.z;
  const int gw = w / kB;
  const int* bb = bbox + 4 * b;
  const int by0 = bb[0], by1 = bb[1], bx0 = bb[2], bx1 = bb[3];
  const uint8_t* bits = mask_bits + size_t(b) * nbytes;
  const uint8_t* src = base + size_t(b) * h * w;
  uint8_t* dst = out + size_t(b) * h * w;
  const int ty0 = blockIdx.y * kTile, tx0 = blockIdx.x * kTile;
  for (int i = threadIdx.x; i < (kTile + 2) * (kTile + 2); i += blockDim.x) {
    const int ly = i / (kTile + 2), lx = i % (kTile + 2);
    const int y = ty0 + ly - 1, x = tx0 + lx - 1;
    // 'nearest' relative to the box: clamp into [by0, by1) x [bx0, bx1)
    const int cy = min(max(y, by0), by1 - 1), cx = min(max(x, bx0), bx1 - 1);
    const bool in_box = by1 > by0 && y >= by0 && y < by1 && x >= bx0 && x < bx1;
    sv[ly][lx] = (by1 > by0) ? src[size_t(min(max(cy, 0), h - 1)) * w + min(max(cx, 0), w - 1)] : 0;
    sm[ly][lx] = in_box ? (masked_px(bits, gw, y, x) ? 1 : 2) : 0;   // 0 = outside box
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kTile * kTile; i += blockDim.x) {
    const int ly = i / kTile + 1, lx = i % kTile + 1;
    const int y = ty0 + ly - 1, x = tx0 + lx - 1;
    if (y >= h || x >= w) continue;
    uint8_t v = src[size_t(y) * w + x];
    const uint8_t me = sm[ly][lx];
    if (me) {
      const uint8_t nb[4] = {sm[ly - 1][lx], sm[ly + 1][lx], sm[ly][lx - 1], sm[ly][lx + 1]};
      bool bnd = false;
#pragma unroll
      for (int q = 0; q < 4; ++q) bnd |= (me == 2 && nb[q] == 1) || (me == 1 && nb[q] == 2);
      if (bnd) {
        uint8_t nv[9];
        int k = 0;
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
          for (int dx = -1; dx <= 1; ++dx) nv[k++] = sv[ly + dy][lx + dx];
        v = median9(nv);
      }
    }
    dst[size_t(y) * w + x] = v;
  }
}

}  // namespace

cudaError_t launch_baseline(int depth, int b, int h, int w, int c, const uint8_t* planes,
                            const uint8_t* refs, const uint8_t* mask_bits, uint8_t* out,
                            uint8_t* base, int* list, int* rank, int* count, int* bbox,
                            cudaStream_t s) {
  const int ns = (h / kB) * (w / kB);
  const int nbytes = (ns + 7) / 8;
  cudaError_t e = launch_masklist(mask_bits, b, nbytes, ns, list, rank, count, s);
  if (e != cudaSuccess) return e;
  uint8_t* match_out = depth ? base : out;
  const size_t plane_bytes = size_t(h) * w * c;
  e = cudaMemcpyAsync(match_out, planes, plane_bytes * b, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return e;
  dim3 grid(std::min(ns, 2 * sm_count()), b);
  if (c == 3)
    launch_pdl(baseline_match_kernel<3>, grid, 320, 0, s, planes, refs, mask_bits, list, count,
                                                  match_out, h, w, ns, nbytes);
  else
    launch_pdl(baseline_match_kernel<1>, grid, 320, 0, s, planes, refs, mask_bits, list, count,
                                                  match_out, h, w, ns, nbytes);
  if ((e = cudaGetLastError()) != cudaSuccess || !depth) return e;
  launch_pdl(baseline_bbox_kernel, b, 32, 0, s, list, count, ns, w / kB, h, w, bbox);
  dim3 mg(ceil_div(w, kTile), ceil_div(h, kTile), b);
  launch_pdl(baseline_median_kernel, mg, kTile * kTile / 4, 0, s, base, mask_bits, bbox, out, h, w,
                                                           nbytes);
  return cudaGetLastError();
}

}  // namespace nvrec
