// launch.cuh -- kernel argument blocks and host launchers shared between the
// kernel translation units and the C-ABI (capi.cu).
#pragma once

#include "tile_ops.cuh"

namespace nvrec {

struct EmbedArgs {
  Dims D;
  const float* emb_w;      // [kimg][d]
  const float* emb_wmask;  // [p*p][d]
  const float* emb_wmsum;  // [d]
  const float* emb_b;      // [d]
  const float* time_pos;   // [nt][d]
  // U8 path
  const uint8_t* frames;
  const int32_t* frame_index;  // [b][F]
  size_t frame_bytes;
  const int* rank;             // [b][ns] >= 0 <=> patch masked
  // F32 path
  const float* stack;          // (b, f_in, c, h, w)
  int f_in;
  const uint8_t* pmask;        // (b, h, w)
  int h, w, nh, nw, ns;
  float* x;                    // [b][nt][ns][d]
};

struct LnQkvArgs {
  Dims D;
  const float* x;
  const float* ln_w; const float* ln_b; const float* qkv_w; const float* qkv_b;
  QkvDst dst;
  int ns;
};

struct TokenArgs {
  Dims D;
  BlockW w;             // this block
  BlockW wn;            // next block (ln_s/qkv_s used) when !last
  const float* norm_w; const float* norm_b;
  const float* head_w; const float* head_b;
  int last;
  const int* list;      // masked positions (ascending) or null = dense
  const int* count;
  float* x;             // [b][nt][ns][d]
  const float* ao;      // [b][nt][ns][d], row r (compact when list)
  const float* part;    // or: key-split attention partials [split][seq][ns][36] to
  int splits;           //     merge on load (splits > 1; the combine kernel is skipped)
  QkvDst dst;           // next block's Q/K/V
  int img_h, img_w, nh, nw, ns;
  float* out_f32;       // (b, c, h, w) or null
  uint8_t* out_u8;      // (b, h, w, c) or null
  uint8_t* out_frames;  // or: merge in place into stream b's corrupted plane,
  const int32_t* out_slot;  // frames + out_slot[b * slot_stride] * frame_bytes
  int slot_stride;
  size_t frame_bytes;
  int P;                // positions per CTA (set by launch_token)
};

struct AttnArgs {
  const float* q; const float* k; const float* v;
  float* ao;              // [b][nt][ns][d] rows r
  const int* count;       // compact query count per stream or null (= ns)
  int nt, heads, ns, ns_pad, d;
  float scale_log2;       // log2(e) / sqrt(hd)
};

// tensor-core spatial attention envelope (k_attn_tc.cu)
bool tc_supported(const Dims& D);
// tensor-core embedding (+ block-0 LN/QKV) envelope (k_embed_tc.cu)
bool embed_tc_supported(const Dims& D);
struct EmbedTcArgs {
  Dims D;
  const TcW* tcw;                 // host copy of the packed-weight pointers
  const float* emb_wmsum; const float* emb_b; const float* time_pos;
  const float* ln_w; const float* ln_b; const float* qkv_b;
  const uint8_t* frames; const int32_t* frame_index; int n_slots;
  const int* rank;                // masked patches (block mask), required
  const int* qrank;               // compact Q rows (block 0 pruned) or null
  float* x;
  __half* xh;                     // or: the embedding output in fp16 (token_tc input)
  __nv_bfloat16* qh; __nv_bfloat16* kh; __nv_bfloat16* vth;
  int b, h, w, nh, nw, ns, ns_pad;
  int x3;                         // precise: split operands (TcW emb3/qkv0_3), fp32 x
  int u16;                        // frames are u16 depth planes (TcW emb16 / emb16_3)
  // or: the float module API (TcW embf / embf3): stack (b, f_in, c, h, w) in
  // [0, 1] (front-padded to F frames on the fly), pixel mask (b, h, w)
  int f32;
  const float* stack; int f_in;
  const uint8_t* pmask;
};
cudaError_t launch_embed_tc(const EmbedTcArgs& a, cudaStream_t s);

// tensor-core tail of a non-last block (k_token_tc.cu)
bool token_tc_supported(const Dims& D);
struct TokenTcArgs {
  int b, ns, ns_pad, nt;
  float* x; const __half* ao;   // ao in fp16 (written so by attn_tc for this consumer)
  const __half* xh;             // residual input in fp16 (from embed_tc) or null = x
  const __half* w_blk;          // this block's fp16 pack (proj_s..fc2)
  const __half* w_qkv_next;     // next block's qkv_s pack
  const float *b_proj_s, *ln_t_w, *ln_t_b, *b_qkv_t, *b_proj_t, *ln_m_w, *ln_m_b;
  const float *b_fc1, *b_fc2, *ln_s_next_w, *ln_s_next_b, *b_qkv_next;
  __nv_bfloat16* qh; __nv_bfloat16* kh; __nv_bfloat16* vth;
  const int* qrank;             // compact Q rows for a pruned next block, or null
};
cudaError_t launch_token_tc(const TokenTcArgs& a, cudaStream_t s);

// precise (split-fp16) tensor-core tail of a non-last block (k_token_x3.cu):
// three phase kernels, same envelope as token_tc
struct TokenX3Args {
  int b, ns, ns_pad, nt;
  float* x; const float* ao;    // fp32 residual (in/out) and attention output
  const __half* w_blk;          // this block's [hi | lo] pack (TcW::blk3)
  const __half* w_next;         // next block's pack (its qkv_s)
  float sc[6];                  // 2^-s: proj_s, qkv_t, proj_t, fc1, fc2, next qkv_s
  const float *b_proj_s, *ln_t_w, *ln_t_b, *b_qkv_t, *b_proj_t, *ln_m_w, *ln_m_b;
  const float *b_fc1, *b_fc2, *ln_s_next_w, *ln_s_next_b, *b_qkv_next;
  __nv_bfloat16* qh; __nv_bfloat16* kh; __nv_bfloat16* vth;   // split layouts (QkvDst::x3)
  const int* qrank;             // compact Q rows for a pruned next block, or null
};
cudaError_t launch_token_x3(const TokenX3Args& a, cudaStream_t s);

// tensor-core LAST block + final LayerNorm + head on the masked patches
// (k_last_tc.cu); split-fp16 (fp32-class) products on both precision paths
struct LastTcArgs {
  int b, ns, nt, c;             // streams, positions per slice, time slices, channels
  int img_h, img_w, nw;
  const int* list;              // [b][ns] masked positions (ascending), or null = all
  const int* count;             // [b] entries of list, or null
  const float* x;               // [b][nt][ns][64] residual stream (positions)
  const float* ao;              // [b][nt][ns][64] attention output, row r <-> list[r]
  const __half* w_blk;          // the last block's streaming pack (TcW::last3)
  const __half* w_head;         // TcW::head3
  float sc[5];                  // 2^-s: proj_s, qkv_t, proj_t, fc1, fc2
  float sc_head;
  const float *b_proj_s, *ln_t_w, *ln_t_b, *b_qkv_t, *b_proj_t, *ln_m_w, *ln_m_b;
  const float *b_fc1, *b_fc2, *norm_w, *norm_b, *head_b;
  float* out_f32;               // (b, c, h, w) or null
  uint8_t* out_u8;              // (b, h, w, c) or null
  uint8_t* out_frames;          // or: in place into stream b's corrupted plane,
  const int32_t* out_slot;      //   frames + out_slot[b * slot_stride] * frame_bytes
  int slot_stride;
  size_t frame_bytes;
  int u16;                      // u16 depth planes: out * 65535 quantisation, 2-byte pixels
  int max_hsplit;                // CTAs that may share a tile (1, 2 or 4)
};
bool last_tc_supported(const Dims& D, int b);
// grid_rows: an upper bound of the gathered rows (sizes the grid)
cudaError_t launch_last_tc(const LastTcArgs& a, int grid_rows, cudaStream_t s);

cudaError_t launch_embed(const EmbedArgs& a, bool u8, int b, cudaStream_t s);
cudaError_t launch_ln_qkv(const LnQkvArgs& a, int b, cudaStream_t s);
cudaError_t launch_copy_plane(const uint8_t* frames, const int32_t* frame_index, int F,
                              size_t frame_bytes, uint8_t* out, int b, cudaStream_t s);
cudaError_t launch_token(const TokenArgs& a, int b, int max_rows, cudaStream_t s);
cudaError_t launch_attn_simt(const AttnArgs& a, int b, int max_rows, cudaStream_t s);
// defer_combine: the consumer merges key-split partials itself (token_kernel);
// *splits_out receives the split count (1 = ao written directly); x3: the
// precise path's split-bf16 operand layouts (QkvDst::x3)
cudaError_t launch_attn_tc(const Act& A, const Dims& D, const int* count, cudaStream_t s,
                           int* n_kernels = nullptr, bool defer_combine = false,
                           int* splits_out = nullptr, bool ao_half = false,
                           bool x3 = false);
int64_t attn_fixup_items();   // -1 on a CUDA error
#ifdef NVREC_TRACE
int attn_trace(unsigned long long* host, int n);   // trace build (tools/trace_attn.py)
int last_trace(unsigned long long* host, int n);   // trace build (tools/trace_last.py)
int token_x3_trace(unsigned long long* host, int n);   // trace build (tools/trace_token.py)
int embed_trace(unsigned long long* host, int n);      // trace build (tools/trace_embed.py)
int token_tc_trace(unsigned long long* host, int n);   // trace build (tools/trace_token.py fast)
#endif
cudaError_t launch_lossmask(const nvrec_lossmask_job* jobs, int n_jobs, cudaStream_t s);
cudaError_t launch_baseline(int depth, int b, int h, int w, int c, const uint8_t* planes,
                            const uint8_t* refs, const uint8_t* mask_bits, uint8_t* out,
                            uint8_t* base, int* list, int* rank, int* count, int* bbox,
                            cudaStream_t s);
cudaError_t launch_decode(const nvrec_decode_job* jobs, int n_jobs, int max_blocks,
                          cudaStream_t s);
int rs_plan_host(int n, int r, const uint8_t* present, uint8_t* coef, int32_t* sources,
                 int32_t* missing, int32_t* m_out);
cudaError_t launch_rs(const nvrec_rs_job* jobs, int n_jobs, int max_shard_len, int max_coef,
                      bool word, cudaStream_t s);
cudaError_t launch_masklist(const uint8_t* bits, int b, int nbytes, int ns, int* list,
                            int* rank, int* count, cudaStream_t s);

}  // namespace nvrec
