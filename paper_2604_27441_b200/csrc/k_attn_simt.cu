// k_attn_simt.cu -- fp32 spatial attention on CUDA cores (precise mode and
// every head size the tensor-core kernel does not cover).
//
// softmax(Q K^T / sqrt(hd)) V per (stream, time slice, head) over all ns
// patches, unmasked and non-causal: F.scaled_dot_product_attention at
// model.py:39 as called from the spatial half of _Block (model.py:59-60).
// One thread owns one query row (q and the running output in registers);
// K/V tiles of 64 keys are staged in shared memory and read as broadcasts;
// online softmax in base 2.  Queries may be a compact list (pruned last
// block): row r of Q/AO then belongs to masked patch list[r].
#include "launch.cuh"

namespace nvrec {


constexpr int kKeyTile = 64;

template <int HD>
__global__ void __launch_bounds__(128)
attn_simt_kernel(AttnArgs a) {
  pdl_entry();
  __shared__ __align__(16) float Ks[kKeyTile * HD];
  __shared__ __align__(16) float Vs[kKeyTile * HD];
  const int seq = blockIdx.y;
  const int b = seq / (a.nt * a.heads);
  const int it = (seq / a.heads) % a.nt;
  const int hh = seq % a.heads;
  const int nq = a.count ? a.count[b] : a.ns;
  const int q0 = blockIdx.x * 128;
  if (q0 >= nq) return;
  const int r = q0 + threadIdx.x;
  const bool active = r < nq;

  float q[HD], o[HD];
  const float* qp = a.q + (size_t(seq) * a.ns_pad + (active ? r : 0)) * HD;
#pragma unroll
  for (int e = 0; e < HD; ++e) { q[e] = qp[e] * a.scale_log2; o[e] = 0.f; }
  float m = -INFINITY, l = 0.f;

  const float* kbase = a.k + size_t(seq) * a.ns_pad * HD;
  const float* vbase = a.v + size_t(seq) * a.ns_pad * HD;
  for (int k0 = 0; k0 < a.ns; k0 += kKeyTile) {
    __syncthreads();
    const int nk = min(kKeyTile, a.ns - k0);
    for (int i = threadIdx.x; i < kKeyTile * HD / 4; i += blockDim.x) {
      float4 kv = make_float4(0.f, 0.f, 0.f, 0.f), vv = kv;
      if (i * 4 < nk * HD) {     // rows past ns are never written: zero them
        kv = reinterpret_cast<const float4*>(kbase + size_t(k0) * HD)[i];
        vv = reinterpret_cast<const float4*>(vbase + size_t(k0) * HD)[i];
      }
      reinterpret_cast<float4*>(Ks)[i] = kv;
      reinterpret_cast<float4*>(Vs)[i] = vv;
    }
    __syncthreads();
    float s[kKeyTile];
    float mt = -INFINITY;
#pragma unroll
    for (int j = 0; j < kKeyTile; ++j) {
      float acc = 0.f;
#pragma unroll
      for (int e = 0; e < HD; ++e) acc = fmaf(q[e], Ks[j * HD + e], acc);
      s[j] = j < nk ? acc : -INFINITY;
      mt = fmaxf(mt, s[j]);
    }
    const float mn = fmaxf(m, mt);
    const float alpha = exp2f(m - mn);
    l *= alpha;
#pragma unroll
    for (int e = 0; e < HD; ++e) o[e] *= alpha;
#pragma unroll
    for (int j = 0; j < kKeyTile; ++j) {
      const float pj = exp2f(s[j] - mn);
      l += pj;
#pragma unroll
      for (int e = 0; e < HD; ++e) o[e] = fmaf(pj, Vs[j * HD + e], o[e]);
    }
    m = mn;
  }
  if (!active) return;
  const float inv = 1.f / l;
  float* out = a.ao + (size_t(b * a.nt + it) * a.ns + r) * a.d + hh * HD;
#pragma unroll
  for (int e = 0; e < HD; ++e) out[e] = o[e] * inv;
}

cudaError_t launch_attn_simt(const AttnArgs& a, int b, int max_rows, cudaStream_t s) {
  dim3 grid(ceil_div(max_rows, 128), b * a.nt * a.heads);
  const int hd = a.d / a.heads;
  switch (hd) {
    case 8: launch_seq(attn_simt_kernel<8>, grid, 128, 0, s, a); break;
    case 16: launch_seq(attn_simt_kernel<16>, grid, 128, 0, s, a); break;
    case 32: launch_seq(attn_simt_kernel<32>, grid, 128, 0, s, a); break;
    case 64: launch_seq(attn_simt_kernel<64>, grid, 128, 0, s, a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace nvrec
