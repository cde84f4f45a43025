// k_embed.cu -- tubelet embedding (the "encoder convolution") and the
// pre-attention LayerNorm + QKV projection of block 0, fp32 CUDA-core path.
//
// embed_kernel<U8> computes, per token (b, it, ih, iw), model.py:99-114:
//   x[o] = bias[o] + time_pos[it][o]
//        + sum_{ci,tt,py,px} W[o,ci,tt,py,px] * in[ci, it*T+tt, ih*p+py, iw*p+px]
//        + sum_{py,px} W[o,c,T-1,py,px] * mask[ih*p+py, iw*p+px]   (it == nt-1)
// where the last frame's masked pixels are multiplied by (1 - mask)
// (model.py:108-109).  The Conv3d has kernel == stride, so it is a GEMM over
// non-overlapping patches: M = tokens, K = c*T*p*p (+ mask rows), N = dim.
//   U8  = RecoveryServer path: u8 HWC planes addressed through a per-stream
//         frame-slot table (front padding = repeated slot, model.py:99-101),
//         normalised with the exact f32 u8/255 of server.py:189 (LUT), and a
//         block mask (the mask channel collapses to a per-token rank-1 term).
//   F32 = MaskedVideoModel.forward path: f32 (b, f, c, h, w) stack, arbitrary
//         per-pixel mask.
// The contraction K is ordered (tt, py, px, ci) so each K chunk (one patch
// row of one frame) is p*c contiguous bytes of the HWC plane.
#include "launch.cuh"

namespace nvrec {


constexpr int kEmbTok = 64;      // tokens per CTA
constexpr int kEmbThreads = 256;

template <bool U8>
__global__ void __launch_bounds__(kEmbThreads)
embed_kernel(EmbedArgs a) {
  pdl_entry();
  extern __shared__ float smem[];
  const Dims& D = a.D;
  const int kc_max = D.p * D.c > D.p ? D.p * D.c : D.p;
  float* As = smem;                              // [kc_max][kEmbTok + 1]
  float* Ws = As + kc_max * (kEmbTok + 1);       // [kc_max][d]
  float* lut = Ws + kc_max * D.d;                // [256]
  __shared__ int s_masked[kEmbTok];

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int s0 = blockIdx.x * kEmbTok;
  const int it = blockIdx.y, b = blockIdx.z;
  const int d = D.d, p = D.p, c = D.c;
  const int nj = d >> 4;                         // outputs per thread (<= 8)
  const bool last_slice = (it == D.nt - 1);

  if (U8) {
    for (int v = tid; v < 256; v += blockDim.x) lut[v] = __fdiv_rn(float(v), 255.f);
  }
  for (int t = tid; t < kEmbTok; t += blockDim.x) {
    int s = s0 + t;
    s_masked[t] = (U8 && s < a.ns && a.rank) ? (a.rank[b * a.ns + s] >= 0) : 0;
  }

  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  auto fma_chunk = [&](int kc) {
    for (int kk = 0; kk < kc; ++kk) {
      float av[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk * (kEmbTok + 1) + ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < nj) {
          const float wv = Ws[kk * d + tx + 16 * j];
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[i][j] = fmaf(av[i], wv, acc[i][j]);
        }
      }
    }
  };

  const int kc = p * c;
  for (int tt = 0; tt < D.T; ++tt) {
    const int f = it * D.T + tt;
    const bool last_frame = (f == D.F - 1);
    const uint8_t* src8 = nullptr;
    const float* srcf = nullptr;
    if (U8) {
      src8 = a.frames + size_t(a.frame_index[b * D.F + f]) * a.frame_bytes;
    } else {
      int fs = f - (D.F - a.f_in);
      if (fs < 0) fs = 0;                        // front pad with frame 0
      srcf = a.stack + size_t(b * a.f_in + fs) * c * a.h * a.w;
    }
    for (int py = 0; py < p; ++py) {
      __syncthreads();
      for (int idx = tid; idx < kEmbTok * kc; idx += blockDim.x) {
        const int t = idx / kc, kk = idx - t * kc;
        const int s = s0 + t;
        float v = 0.f;
        if (s < a.ns) {
          const int ih = s / a.nw, iw = s - ih * a.nw;
          const int y = ih * p + py;
          if (U8) {
            if (!(last_frame && s_masked[t]))
              v = lut[src8[(size_t(y) * a.w + iw * p) * c + kk]];
          } else {
            const int px = kk / c, ci = kk - px * c;
            const int xx = iw * p + px;
            v = srcf[(size_t(ci) * a.h + y) * a.w + xx];
            if (last_frame) {
              float m = a.pmask[(size_t(b) * a.h + y) * a.w + xx] ? 1.f : 0.f;
              v = v * (1.f - m);
            }
          }
        }
        As[kk * (kEmbTok + 1) + t] = v;
      }
      const float* wsrc = a.emb_w + size_t((tt * p + py) * kc) * d;
      for (int idx = tid; idx < kc * d; idx += blockDim.x) Ws[idx] = __ldg(wsrc + idx);
      __syncthreads();
      fma_chunk(kc);
    }
  }
  // mask channel on the last frame (model.py:105-107)
  if (!U8 && last_slice) {
    for (int py = 0; py < p; ++py) {
      __syncthreads();
      for (int idx = tid; idx < kEmbTok * p; idx += blockDim.x) {
        const int t = idx / p, px = idx - t * p;
        const int s = s0 + t;
        float v = 0.f;
        if (s < a.ns) {
          const int ih = s / a.nw, iw = s - ih * a.nw;
          v = a.pmask[(size_t(b) * a.h + ih * p + py) * a.w + iw * p + px] ? 1.f : 0.f;
        }
        As[px * (kEmbTok + 1) + t] = v;
      }
      const float* wsrc = a.emb_wmask + size_t(py * p) * d;
      for (int idx = tid; idx < p * d; idx += blockDim.x) Ws[idx] = __ldg(wsrc + idx);
      __syncthreads();
      fma_chunk(p);
    }
  }
  // epilogue: bias + time_pos (+ block-mask rank-1 term) -> x
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = ty + 16 * i, s = s0 + t;
    if (s >= a.ns) continue;
    const bool mterm = U8 && last_slice && s_masked[t];
    float* xo = a.x + (size_t(b * D.nt + it) * a.ns + s) * d;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j < nj) {
        const int o = tx + 16 * j;
        float v = acc[i][j] + __ldg(a.emb_b + o);
        if (mterm) v += __ldg(a.emb_wmsum + o);
        xo[o] = v + __ldg(a.time_pos + it * d + o);
      }
    }
  }
}

// LN_s + qkv_s of block 0 (model.py:59 -> _Attention.qkv, model.py:37) for
// 32 consecutive positions of one time slice per CTA.

constexpr int kLnTok = 32;

__global__ void __launch_bounds__(256)
ln_qkv_kernel(LnQkvArgs a) {
  pdl_entry();
  extern __shared__ float smem[];
  const int d = a.D.d;
  float* Xs = smem;               // [kLnTok][d]
  float* Ts = Xs + kLnTok * d;    // [kLnTok][d]
  const int s0 = blockIdx.x * kLnTok, it = blockIdx.y, b = blockIdx.z;
  const int n = min(kLnTok, a.ns - s0);
  const float* xin = a.x + (size_t(b * a.D.nt + it) * a.ns + s0) * d;
  for (int i = threadIdx.x; i < n * d; i += blockDim.x) Xs[i] = xin[i];
  __syncthreads();
  tile_layernorm(Xs, d, Ts, d, n, d, a.ln_w, a.ln_b);
  __syncthreads();
  tile_gemm(Ts, d, n, d, a.qkv_w, a.qkv_b, 3 * d, [&](int t, int col, float v) {
    qkv_store(a.dst, b, it, s0 + t, col, v);
  });
}

// out[b] = corrupted plane (the merge's pass-through half, server.py:196);
// the head then overwrites the masked patches.
__global__ void copy_plane_kernel(const uint8_t* __restrict__ frames,
                                  const int32_t* __restrict__ frame_index, int F,
                                  size_t frame_bytes, uint8_t* __restrict__ out) {
  pdl_entry();
  const int b = blockIdx.y;
  const uint4* src = reinterpret_cast<const uint4*>(
      frames + size_t(frame_index[b * F + F - 1]) * frame_bytes);
  uint4* dst = reinterpret_cast<uint4*>(out + size_t(b) * frame_bytes);
  const size_t n16 = frame_bytes / 16;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16;
       i += size_t(gridDim.x) * blockDim.x)
    dst[i] = __ldg(src + i);
}

// ---------------------------------------------------------------------------
size_t embed_smem_bytes(const Dims& D) {
  int kc_max = D.p * D.c > D.p ? D.p * D.c : D.p;
  return sizeof(float) * (size_t(kc_max) * (kEmbTok + 1) + size_t(kc_max) * D.d + 256);
}

cudaError_t launch_embed(const EmbedArgs& a, bool u8, int b, cudaStream_t s) {
  dim3 grid(ceil_div(a.ns, kEmbTok), a.D.nt, b);
  size_t smem = embed_smem_bytes(a.D);
  if (u8) {
    if (cudaError_t e = smem_optin(embed_kernel<true>, int(smem))) return e;
    launch_seq(embed_kernel<true>, grid, kEmbThreads, smem, s, a);
  } else {
    if (cudaError_t e = smem_optin(embed_kernel<false>, int(smem))) return e;
    launch_seq(embed_kernel<false>, grid, kEmbThreads, smem, s, a);
  }
  return cudaGetLastError();
}

cudaError_t launch_ln_qkv(const LnQkvArgs& a, int b, cudaStream_t s) {
  dim3 grid(ceil_div(a.ns, kLnTok), a.D.nt, b);
  size_t smem = sizeof(float) * 2 * kLnTok * a.D.d;
  launch_seq(ln_qkv_kernel, grid, 256, smem, s, a);
  return cudaGetLastError();
}

cudaError_t launch_copy_plane(const uint8_t* frames, const int32_t* frame_index, int F,
                              size_t frame_bytes, uint8_t* out, int b, cudaStream_t s) {
  int blocks = int((frame_bytes / 16 + 255) / 256);
  if (blocks > sm_count() * 4) blocks = sm_count() * 4;
  launch_pdl(copy_plane_kernel, dim3(blocks, b), 256, 0, s, frames, frame_index, F, frame_bytes, out);
  return cudaGetLastError();
}

}  // namespace nvrec
