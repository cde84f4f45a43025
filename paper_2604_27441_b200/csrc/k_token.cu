// k_token.cu -- everything of one transformer block after its spatial
// attention, fused per group of spatial positions (fp32 CUDA cores):
//
//   x += proj_s(ao)                          model.py:60 (residual), :40
//   x += proj_t(attn_t(LN_t(x)))             model.py:61-62 over nt slices
//   x += fc2(GELU(fc1(LN_m(x))))             model.py:53-54,64
//   then either the next block's LN_s + qkv_s (scattered into the spatial
//   attention operands), or -- after the last block --
//   out = sigmoid(head(LN(x[:, -1])))        model.py:117-122, unpatchified
//   and for the u8 server path quantised with numpy's two float32 roundings
//   (server.py:194) straight into the merged output plane.
//
// Temporal attention only mixes the nt tokens of one spatial position, so a
// CTA owning P positions x nt slices is closed under the whole block tail.
// Exact pruning: in the LAST block only the last
// slice reaches the head, so its temporal query, proj_t and MLP run for that
// slice only; on the server path the CTA walks the masked-patch list instead
// of all positions (the merge discards every other prediction, server.py:196).
#include <algorithm>

#include "launch.cuh"

namespace nvrec {


template <bool kNarrow>
__device__ __forceinline__ void token_tile(const TokenArgs& a, int b, int r0, int cnt,
                                           float* smem, int* spos) {
  const Dims& D = a.D;
  const int d = D.d, nt = D.nt;
  const int P = a.P;
  const int npos = min(P, cnt - r0);
  const int ntok = npos * nt;
  const int ntok_max = P * nt;
  float* Xs = smem;                    // [ntok][d]   token t = j*nt + it
  float* As = Xs + ntok_max * d;       // [ntok][d]
  float* Ts = As + ntok_max * d;       // [ntok][d]
  float* Hs = Ts + ntok_max * d;       // [ntok][4d]
  auto gemm = [&](const float* in, int ldi, int ntok_, int K, const float* Wt, const float* bias,
                  int N, auto epi) {
    if (kNarrow) tile_gemm_narrow(in, ldi, ntok_, K, Wt, bias, N, Hs + ntok_max * 4 * d, epi);
    else tile_gemm(in, ldi, ntok_, K, Wt, bias, N, epi);
  };

  for (int j = threadIdx.x; j < npos; j += blockDim.x)
    spos[j] = a.list ? a.list[b * a.ns + r0 + j] : r0 + j;
  __syncthreads();
  for (int i = threadIdx.x; i < ntok * d; i += blockDim.x) {
    const int t = i / d, o = i - t * d;
    const int j = t / nt, it = t - j * nt;
    const size_t slice = size_t(b * nt + it) * a.ns;
    Xs[i] = a.x[(slice + spos[j]) * d + o];
    if (a.splits > 1) {
      // merge the key-range partials of this row and head (attn_combine_kernel's
      // O = sum_s O_s 2^(m_s - M) / sum_s l_s 2^(m_s - M), fused into the load)
      const int hh = o / D.hd, e = o - hh * D.hd;
      const size_t seqs = size_t(gridDim.y) * nt * D.heads;
      const size_t seq = size_t(b * nt + it) * D.heads + hh;
      const float* p0 = a.part + (seq * a.ns + r0 + j) * 36;
      const size_t sstride = seqs * a.ns * 36;
      float M = -INFINITY;
      for (int sp = 0; sp < a.splits; ++sp) M = fmaxf(M, __ldg(p0 + sp * sstride + 32));
      float acc = 0.f, L = 0.f;
      for (int sp = 0; sp < a.splits; ++sp) {
        const float* p = p0 + sp * sstride;
        const float wgt = exp2f(__ldg(p + 32) - M);
        L = fmaf(__ldg(p + 33), wgt, L);
        acc = fmaf(__ldg(p + e), wgt, acc);
      }
      As[i] = acc / L;
    } else {
      As[i] = a.ao[(slice + r0 + j) * d + o];
    }
  }
  __syncthreads();

  // 1. spatial-attention output projection + residual
  gemm(As, d, ntok, d, a.w.proj_s_w, a.w.proj_s_b, d,
            [&](int t, int n, float v) { Xs[t * d + n] += v; });
  __syncthreads();
  // 2-3. LN_t and qkv_t for every slice (keys/values of all slices needed)
  tile_layernorm(Xs, d, Ts, d, ntok, d, a.w.ln_t_w, a.w.ln_t_b);
  __syncthreads();
  const int d3 = 3 * d;
  gemm(Ts, d, ntok, d, a.w.qkv_t_w, a.w.qkv_t_b, d3,
            [&](int t, int n, float v) { Hs[t * d3 + n] = v; });
  __syncthreads();
  // 4. temporal attention over nt slices per (position, head)
  const int hd = D.hd, heads = D.heads;
  const int q_first = a.last ? nt - 1 : 0;       // last block: last-slice query only
  const int nq = nt - q_first;
  const float scale = rsqrtf(float(hd));
  for (int item = threadIdx.x; item < npos * heads * nq; item += blockDim.x) {
    const int iq = q_first + item % nq;
    const int hh = (item / nq) % heads;
    const int j = item / (nq * heads);
    const float* qv = Hs + (j * nt + iq) * d3 + hh * hd;
    float sc[kMaxNt];
    float mx = -INFINITY;
    for (int ik = 0; ik < nt; ++ik) {
      const float* kv = Hs + (j * nt + ik) * d3 + d + hh * hd;
      float acc = 0.f;
      for (int e = 0; e < hd; ++e) acc = fmaf(qv[e], kv[e], acc);
      sc[ik] = acc * scale;
      mx = fmaxf(mx, sc[ik]);
    }
    float den = 0.f;
    for (int ik = 0; ik < nt; ++ik) { sc[ik] = expf(sc[ik] - mx); den += sc[ik]; }
    const float inv = 1.f / den;
    float* o = As + (j * nt + iq) * d + hh * hd;
    for (int e = 0; e < hd; ++e) {
      float acc = 0.f;
      for (int ik = 0; ik < nt; ++ik)
        acc = fmaf(sc[ik], Hs[(j * nt + ik) * d3 + 2 * d + hh * hd + e], acc);
      o[e] = acc * inv;
    }
  }
  __syncthreads();
  // rows that continue: all tokens, or (last block) the last slice only
  const int roff = a.last ? (nt - 1) * d : 0;
  const int rld = a.last ? nt * d : d;
  const int rows = a.last ? npos : ntok;
  auto rowmap = [&](int t) { return a.last ? t * nt + nt - 1 : t; };
  // 5. temporal output projection + residual
  gemm(As + roff, rld, rows, d, a.w.proj_t_w, a.w.proj_t_b, d,
            [&](int t, int n, float v) { Xs[rowmap(t) * d + n] += v; });
  __syncthreads();
  // 6. MLP
  tile_layernorm(Xs + roff, rld, Ts + roff, rld, rows, d, a.w.ln_m_w, a.w.ln_m_b);
  __syncthreads();
  const int d4 = D.hidden;
  gemm(Ts + roff, rld, rows, d, a.w.fc1_w, a.w.fc1_b, d4,
            [&](int t, int n, float v) { Hs[t * d4 + n] = gelu_erf(v); });
  __syncthreads();
  gemm(Hs, d4, rows, d4, a.w.fc2_w, a.w.fc2_b, d,
            [&](int t, int n, float v) { Xs[rowmap(t) * d + n] += v; });
  __syncthreads();

  if (!a.last) {
    // 7a. write back the residual stream; next block's LN_s + qkv_s
    for (int i = threadIdx.x; i < ntok * d; i += blockDim.x) {
      const int t = i / d, o = i - t * d;
      const int j = t / nt, it = t - j * nt;
      a.x[(size_t(b * nt + it) * a.ns + spos[j]) * d + o] = Xs[i];
    }
    tile_layernorm(Xs, d, Ts, d, ntok, d, a.wn.ln_s_w, a.wn.ln_s_b);
    __syncthreads();
    gemm(Ts, d, ntok, d, a.wn.qkv_s_w, a.wn.qkv_s_b, d3, [&](int t, int n, float v) {
      const int j = t / nt, it = t - j * nt;
      qkv_store(a.dst, b, it, spos[j], n, v);
    });
    return;
  }
  // 7b. final LN on the last slice, head, sigmoid, unpatchify (+ quantise)
  tile_layernorm(Xs + roff, rld, Ts, d, npos, d, a.norm_w, a.norm_b);
  __syncthreads();
  const int p = D.p, c = D.c, pc = p * c;
  gemm(Ts, d, npos, d, a.head_w, a.head_b, D.used, [&](int j, int u, float v) {
    const float sg = 1.f / (1.f + expf(-v));
    const int py = u / pc, rem = u - py * pc, px = rem / c, ch = rem - px * c;
    const int s = spos[j];
    const int ih = s / a.nw, iw = s - ih * a.nw;
    const int y = ih * p + py, xx = iw * p + px;
    if (a.out_f32) {
      a.out_f32[((size_t(b) * c + ch) * a.img_h + y) * a.img_w + xx] = sg;
    } else {
      // np.clip(out * 255.0 + 0.5, 0, 255).astype(np.uint8): f32 mul, f32 add
      float q = __fadd_rn(__fmul_rn(sg, 255.f), 0.5f);
      q = fminf(fmaxf(q, 0.f), 255.f);
      uint8_t* ob = a.out_u8 ? a.out_u8 + size_t(b) * a.img_h * a.img_w * c
                             : a.out_frames + size_t(a.out_slot[b * a.slot_stride]) * a.frame_bytes;
      ob[(size_t(y) * a.img_w + xx) * c + ch] = uint8_t(q);
    }
  });
}

// Dense blocks: one tile per CTA.  The pruned last block: a grid-stride loop
// over the stream's masked-patch list (the count lives on the device, so the
// grid is sized for the GPU, not for the worst case).
template <bool kNarrow>
__global__ void __launch_bounds__(256, kNarrow ? 1 : 2)
token_kernel(TokenArgs a) {
  pdl_wait();
  extern __shared__ float smem[];
  __shared__ int spos[48];
  const int b = blockIdx.y;
  const int cnt = a.list ? a.count[b] : a.ns;
  for (int r0 = blockIdx.x * a.P; r0 < cnt; r0 += gridDim.x * a.P) {
    token_tile<kNarrow>(a, b, r0, cnt, smem, spos);
    __syncthreads();
  }
  pdl_trigger();
}

size_t token_smem_bytes(const Dims& D, int P) {
  const size_t ntok = size_t(P) * D.nt;
  const size_t hcols = D.hidden > 3 * D.d ? D.hidden : 3 * D.d;
  return sizeof(float) * (3 * ntok * D.d + ntok * hcols + 256 * 4);   // + split-K scratch
}

cudaError_t launch_token(const TokenArgs& a_in, int b, int max_rows, cudaStream_t s) {
  TokenArgs a = a_in;
  // dense blocks: 48 tokens per CTA; the pruned last block walks a short
  // list of masked patches, so one position per CTA spreads it over the GPU
  const bool narrow = a.list != nullptr;
  a.P = narrow ? 1 : max(1, 48 / a.D.nt);
  size_t smem = token_smem_bytes(a.D, a.P);
  dim3 grid(ceil_div(max_rows, a.P), b);
  if (narrow) grid.x = std::min<int>(grid.x, std::max(1, 2 * sm_count() / b));
  if (narrow) {
    if (cudaError_t e = smem_optin(token_kernel<true>, int(smem))) return e;
    launch_seq(token_kernel<true>, grid, 256, smem, s, a);
  } else {
    if (cudaError_t e = smem_optin(token_kernel<false>, int(smem))) return e;
    launch_seq(token_kernel<false>, grid, 256, smem, s, a);
  }
  return cudaGetLastError();
}

}  // namespace nvrec
