// common.cuh -- shared definitions for the nvrec B200 kernels.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <utility>

#include "nvrec_b200.h"

namespace nvrec {

// ---- programmatic dependent launch ---------------------------------------------------
// Every kernel is launched by launch_pdl with programmatic stream serialisation:
// its CTAs may be scheduled (and run their launch overhead) while the previous
// kernel on the stream drains.  pdl_entry() is the first statement of every
// kernel: it blocks until the predecessor grid has completed and its memory is
// visible, then allows the successor to start launching.  Because every CTA
// passes the wait before it can exit, completion stays transitive down the chain.
// Heavy kernels (many waves of big CTAs) call pdl_wait() first and pdl_trigger()
// only as they finish, so a light successor's CTAs are not parked on an SM
// through the heavy kernel's last wave.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_entry() {
  pdl_wait();
  pdl_trigger();
}
bool pdl_enabled();   // NVREC_PDL=0 turns the attribute off (A/B, debugging)

// Per-device launch facts (capi.cu).  The dynamic shared-memory opt-in is a
// property of the device context, so it is recorded per (kernel, device)
// under a mutex and marked done only after cudaFuncSetAttribute succeeded:
// a second GPU in the same process, or two host threads racing to the first
// launch, still launch with the attribute set.
cudaError_t smem_optin(const void* kernel, int bytes);
template <typename... P>
inline cudaError_t smem_optin(void (*kernel)(P...), int bytes) {
  return smem_optin(reinterpret_cast<const void*>(kernel), bytes);
}
int sm_count();       // multiprocessors of the current device

// Only light kernels (small CTAs, a few SMs' worth of resources) take the
// attribute: a heavy successor launched early parks CTAs on every SM while it
// waits, which starves the concurrent stream of the other modality (measured:
// -2% step throughput when every launch used it).  Heavy kernels use
// launch_seq, i.e. plain stream order; their pdl_entry() still releases light
// successors early.
template <bool kPdl = true, typename... P, typename... A>
inline cudaError_t launch_pdl(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, A&&... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = kPdl && pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<P>(args)...);
}
template <typename... P, typename... A>
inline cudaError_t launch_seq(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, A&&... args) {
  return launch_pdl<false>(kernel, grid, block, smem, s, std::forward<A>(args)...);
}

constexpr int kMaxDim = 128;
constexpr int kMaxNt = 16;
constexpr int kAttnQTile = 128;     // queries per attention CTA / key padding unit

// Model geometry derived from nvrec ModelConfig + channels
// (model.py:70-80; config.py:35-41).
struct Dims {
  int c;        // image channels (3 RGB / 1 depth)
  int d;        // dim
  int heads, hd;
  int T, p;     // tubelet frames, patch edge
  int F, nt;    // stack_len, time slices
  int layers;
  int hidden;   // 4*d
  int kimg;     // c*T*p*p   (image part of the embed contraction)
  int used;     // p*p*c     (head columns of the last tubelet frame)
};

// Per-block weights, all fp32, weight matrices stored K-major ("Wt[k][n]",
// the transpose of nn.Linear's (out, in)), so a warp reading one k row for
// consecutive n is coalesced.
struct BlockW {
  const float *ln_s_w, *ln_s_b, *qkv_s_w, *qkv_s_b, *proj_s_w, *proj_s_b;
  const float *ln_t_w, *ln_t_b, *qkv_t_w, *qkv_t_b, *proj_t_w, *proj_t_b;
  const float *ln_m_w, *ln_m_b, *fc1_w, *fc1_b, *fc2_w, *fc2_b;
};

// fp16 operands of the tensor-core (fast) path, pre-packed in the UMMA
// no-swizzle K-major "interleaved" layout: element (n, k) of an N x K block at
// ((k/8)*(N/8) + n/8)*64 + (n%8)*8 + k%8 (core matrices of 8 rows x 16 B).
struct TcW {
  const __half* emb;            // [T*8 stages][64 x 32c] embed weight blocks
  const __half* qkv0;           // [192 x 64] block-0 qkv_s weight
  int emb_stage_elems;          // 64 * 32c
  // per block, contiguous: proj_s [64x64] | qkv_t [192x64] | proj_t [64x64] |
  // fc1 [256x64] | fc2 [64x256] | qkv_s [192x64]
  const __half* blk[8];
  // Precise path (split fp16): every matrix W is packed as [hi | lo] blocks of
  // W * 2^s (hi = fp16(W 2^s), lo = fp16(W 2^s - hi); s per matrix puts
  // max|W| 2^s near 2^14 so lo stays a normal number); sc = 2^-s undoes it in
  // the epilogue.  Same element order as the fast packs.
  const __half* emb3;           // [T*16/kPy stages][hi 64 x 16 kPy c | lo ...], kPy = 1 (RGB) / 2
  const __half* qkv0_3;         // [hi 192x64 | lo 192x64] block-0 qkv_s
  const __half* blk3[8];        // per block: proj_s | qkv_t | proj_t | fc1 | fc2 | qkv_s, each [hi | lo]
  // head rows of the last tubelet frame in 4 chunks of 4 patch rows (64c
  // columns), each [hi 64c x 64 | lo 64c x 64] (k_last_tc.cu)
  const __half* head3;
  float sc_head;
  // 16-bit depth embedding (channels == 1): per 2-patch-row stage the K axis is
  // (py, px, byte) with byte 0 = lo (W) and byte 1 = hi (256 W); fp16 packs
  // (emb16) and [hi | lo] split packs scaled by 2^s16 (emb16_3, sc = 2^-s16)
  const __half* emb16;
  const __half* emb16_3;
  float sc_emb16;
  // float module-API embedding (k_embed_tc.cu, F32): per stage 2 pixel rows
  // (K = 32) of one channel of one sub-frame, T x c x 8 stages, then 8
  // mask-channel stages (last sub-frame); fp16 (embf) and [hi | lo] x 2^s (embf3)
  const __half* embf;
  const __half* embf3;
  float sc_embf;
  // the last block's matrices as k_last_tc.cu streams them: proj_s | qkv_t |
  // proj_t | fc1 rows 0-127 | fc1 rows 128-255 | fc2 K 0-127 | fc2 K 128-255,
  // each [hi | lo] (scales sc_blk[layers - 1])
  const __half* last3;
  float sc_emb, sc_qkv0;
  float sc_blk[8][6];
};

struct ModelW {
  TcW tc;
  const float* emb_w;      // [kimg][d], k = ((tt*p+py)*p+px)*c+ci
  const float* emb_wmask;  // [p*p][d] mask-channel weights at tt = T-1
  const float* emb_wmsum;  // [d]      sum of emb_wmask over pixels
  const float* emb_b;      // [d]
  const float* time_pos;   // [nt][d]
  BlockW blk[8];
  const float* norm_w;
  const float* norm_b;
  const float* head_w;     // [d][used] last-tubelet-frame columns only
  const float* head_b;     // [used]
};

// Token-stream buffers of one forward (workspace carve-up).
struct Act {
  float* x;          // [b][nt][ns][d] residual stream
  __half* xh;        // fast path: fp16 copy of the embedding output for block 0's
  bool x_half;       //   tensor-core tail (set when the embed wrote xh instead of x)
  float* ao;         // [b][nt][nrow][d] spatial-attention output (compact rows
                     //   when `list` is set: row r <-> list[r])
  float* q;          // f32 path: [b*nt*heads][nq_pad][hd]; rows compact when
  float* k;          //   the consuming block is pruned
  float* v;          // [b*nt*heads][ns_pad][hd]
  __nv_bfloat16* qh; // bf16 path: Q,K [seq][ns_pad][32]; Vt [seq][32][ns_pad]
  __nv_bfloat16* kh;
  __nv_bfloat16* vth;
  int* list;         // [b][ns] masked positions (ascending) or nullptr = dense
  int* rank;         // [b][ns] position -> row in list, -1 if absent
  int* count;        // [b] entries in list
  float* part;       // bf16 path: key-split attention partials [split][seq][ns][36]
  int* redo_list;    // bf16 path: [0] count + attention work items for the exact fix-up
  int b, ns, nh, nw, ns_pad;
};
constexpr int kAttnMaxSplits = 6;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__host__ __device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int round_up(int a, int b) { return ceil_div(a, b) * b; }

}  // namespace nvrec
