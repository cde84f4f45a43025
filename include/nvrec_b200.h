/*
 * nvrec_b200.h -- C-ABI of the B200-native nvrec recovery path.
 *
 * One shared library (libnvrec_b200.so, sm_100a) exports plain-pointer
 * entry points; no torch types cross this boundary.  Every function returns
 * 0 on success or a negative NVREC_E* code; nvrec_last_error() then holds a
 * message (thread-local).  Device pointers are caller-owned; nothing is
 * allocated on the hot path (workspaces are sized by nvrec_workspace_bytes
 * and passed in), and every launch goes to the caller's cudaStream_t, so the
 * calls are CUDA-graph capturable.
 *
 * Reference interfaces replaced (arxiv 2604.27441, /root/reference/pkg):
 *   nvrec_model_create/load  <- nvrec/train.py:40-43  Checkpoint.build_model
 *                               + nn.Module.load_state_dict of
 *                               nvrec/model.py:67-80  MaskedVideoModel.__init__
 *   nvrec_forward_f32        <- nvrec/model.py:82-122 MaskedVideoModel.forward
 *   nvrec_recover_u8         <- nvrec/server.py:181-196 RecoveryServer._recover
 *                               (u8 stack/normalise, forward, quantise, merge)
 *   nvrec_baseline_u8        <- rgbdstream/recovery.py:94-196 recover_baseline
 *   nvrec_decode             <- rgbdstream/codec.py:260-321 decode (zero-fill
 *                               P-frame / I-frame decode + its mask), fed by
 *                               receiver.py:222-237 (_finalize_p body)
 *   nvrec_rs_plan/           <- rgbdstream/fec.py:144-163 rs_reconstruct
 *   nvrec_rs_reconstruct        (receiver.py:180-209 _finalize_i)
 *   nvrec_loss_mask          <- rgbdstream/receiver.py:224-237 zero-fill +
 *                               rgbdstream/codec.py:159-201,250-257,274-281,
 *                               318-320 (parse_header, block_ranges,
 *                               _corrupted_blocks, decode mask) +
 *                               rgbdstream/recovery.py:221 (wire bitset)
 */
#ifndef NVREC_B200_H
#define NVREC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NVREC_ABI_VERSION 5

enum {
  NVREC_OK = 0,
  NVREC_E_INVALID = -1,      /* bad argument (maps to ValueError)          */
  NVREC_E_UNSUPPORTED = -2,  /* config the kernels do not implement        */
  NVREC_E_CUDA = -3,         /* CUDA runtime / launch failure              */
  NVREC_E_WORKSPACE = -4,    /* workspace too small                        */
  NVREC_E_STATE = -5         /* weights not loaded                         */
};

/* Precision of the arithmetic on the forward path.
 *   NVREC_PREC_FAST:    bf16/fp16 tensor-core (tcgen05) operands, fp32
 *                       accumulation/softmax/LN/GELU; RGB and u8 depth.
 *   NVREC_PREC_PRECISE: fp32-class: every tensor-core product from split bf16
 *                       operands (a = hi + lo, hi*hi + hi*lo + lo*hi, fp32
 *                       accumulation; ~16 significant bits per operand), all
 *                       other arithmetic fp32; shapes outside the tensor-core
 *                       envelope run fp32 CUDA-core kernels.  The 16-bit
 *                       depth mode (<= 1/65535 of full scale). */
enum { NVREC_PREC_FAST = 0, NVREC_PREC_PRECISE = 1 };

/* Architecture fields of nvrec ModelConfig (config.py:14-19,35-41). */
typedef struct nvrec_config {
  int32_t k;          /* reference frames                                   */
  int32_t tubelet_t;  /* frames per temporal token                          */
  int32_t patch;      /* spatial patch edge (== mask block, 16)             */
  int32_t dim;        /* token width                                        */
  int32_t layers;     /* transformer blocks                                 */
  int32_t heads;      /* attention heads                                    */
} nvrec_config;

typedef struct nvrec_model nvrec_model;   /* opaque; weights on one device */

int nvrec_abi_version(void);
const char* nvrec_last_error(void);

/* Create a model for `channels` (3 = RGB, 1 = depth) on the current CUDA
 * device.  Fails with NVREC_E_UNSUPPORTED for architectures outside the
 * kernels' envelope (dim % 16, dim <= 128, dim/heads in {8,16,32,64}). */
int nvrec_model_create(const nvrec_config* cfg, int32_t channels, nvrec_model** out);
int nvrec_model_destroy(nvrec_model* m);

/* Load fp32 HOST tensors in MaskedVideoModel state-dict order
 * (time_pos, embed.weight, embed.bias, blocks.i.{norm_s, attn_s.qkv,
 * attn_s.proj, norm_t, attn_t.qkv, attn_t.proj, norm_m, mlp.0, mlp.2}
 * .{weight,bias}..., norm.weight, norm.bias, head.weight, head.bias).
 * numel[i] is checked against the architecture.  Synchronous. */
int nvrec_model_load(nvrec_model* m, const float* const* tensors,
                     const int64_t* numel, int32_t n_tensors);

/* Bytes of device workspace a forward/recover of this shape needs. */
int64_t nvrec_workspace_bytes(const nvrec_model* m, int32_t batch,
                              int32_t height, int32_t width, int32_t precision);

/* MaskedVideoModel.forward: stack f32 (b, f, c, h, w) in [0,1] oldest first
 * (f <= stack_len, front-padded with frame 0), mask u8 (b, h, w) nonzero =
 * corrupted (any pixel pattern).  out f32 (b, c, h, w).  Device pointers. */
int nvrec_forward_f32(const nvrec_model* m, const float* stack, int32_t b,
                      int32_t f, int32_t c, int32_t h, int32_t w,
                      const uint8_t* mask, float* out, void* workspace,
                      int64_t workspace_bytes, int32_t precision, void* stream);

/* RecoveryServer._recover over a batch of independent streams (block mask).
 * frames: n_slots u8 planes (h, w, c) packed at `frames + slot * h*w*c`;
 * frame_index: int32 (b, stack_len) slot (< n_slots) of each stacked frame, oldest first,
 *   already front-padded, the last entry the corrupted plane;
 * mask_bits: u8 (b, ceil(gh*gw/8)) wire bitset (MSB-first, row-major);
 * out: u8 (b, h, w, c) merged planes (unmasked pixels = corrupted plane).
 * Only masked patches are decoded (exact: the merge discards the rest).
 * The stacked frames are read before `out` is written, so `out` may alias
 * the planes of one reference slot (in-place ring update).  out == NULL merges
 * in place: each stream's corrupted plane (slot frame_index[b*F + F-1], which
 * must then be writable) receives the recovered patches and becomes the merged
 * plane -- no pass-through copy. */
int nvrec_recover_u8(const nvrec_model* m, int32_t b, int32_t h, int32_t w,
                     const uint8_t* frames, int32_t n_slots, const int32_t* frame_index,
                     const uint8_t* mask_bits, uint8_t* out, void* workspace,
                     int64_t workspace_bytes, int32_t precision, void* stream);

/* 16-bit depth extension of nvrec_recover_u8 (the reference's wire format is
 * u8 only; SPEC.md:74 names 16-bit depth an extension point): frames are u16
 * planes (h, w) of a channels == 1 model at `frames + slot * h*w` (elements),
 * normalised as u16 / 65535 and quantised as clip(out * 65535 + 0.5, 0,
 * 65535) -- the u8 rule of server.py:189-194 at 16 bits -- then merged through
 * the block mask.  Same slot table, mask bits, aliasing and in-place (out ==
 * NULL) rules as nvrec_recover_u8.  Needs the tensor-core envelope
 * (dim 64, 2 heads, patch 16, stack slices <= 3): NVREC_E_UNSUPPORTED
 * otherwise. */
int nvrec_recover_u16(const nvrec_model* m, int32_t b, int32_t h, int32_t w,
                      const uint16_t* frames, int32_t n_slots, const int32_t* frame_index,
                      const uint8_t* mask_bits, uint16_t* out, void* workspace,
                      int64_t workspace_bytes, int32_t precision, void* stream);

/* One P-frame's loss-mask job (all pointers are DEVICE pointers). */
typedef struct nvrec_lossmask_job {
  const uint8_t* header;      /* codec header bytes (shard 0 payload)        */
  int32_t header_len;
  int32_t n_data;             /* data shards incl. header shard 0            */
  const uint8_t* received;    /* u8[n_data], nonzero = shard arrived         */
  int32_t shard_len;          /* body shard payload length L                 */
  int64_t body_len;           /* encoded_len - header_len (receiver.py:225)  */
  int64_t payload_received;   /* len(assembled body); < payload_len => tail
                                 zero-fill (codec.py:274-278)                */
  const int64_t* extra_ranges;/* optional explicit [lo,hi) pairs or NULL     */
  int32_t n_extra;
  uint8_t* grid;              /* out u8[gh*gw] 0/1 (CorruptionMask.grid)     */
  uint8_t* wire_bits;         /* out u8[ceil(gh*gw/8)] (np.packbits) or NULL */
  int32_t* status;            /* out: 0 ok, else UndecodableError reason;
                                 [1] = flagged count, [2] = gh, [3] = gw     */
  int32_t grid_capacity;      /* bytes available at grid                    */
} nvrec_lossmask_job;

/* Batched loss-mask kernel: jobs is a DEVICE array of n_jobs descriptors.
 * Bit-exact with the reference receiver+codec.  A job whose status is
 * nonzero gets all ceil(grid_capacity/8) wire-bit bytes cleared, so a
 * recovery launch consuming them leaves that stream's plane untouched. */
int nvrec_loss_mask(const nvrec_lossmask_job* jobs, int32_t n_jobs, void* stream);

/* Status codes written to nvrec_lossmask_job.status[0] (0 = ok):
 *   1, 3 "header truncated"; 2 "inconsistent geometry in header";
 *   4 "bitmap disagrees with present count"   (codec.UndecodableError)
 *   10 invalid FrameKind                      (ValueError in parse_header)
 *   5 grid_capacity too small                 (caller error)
 * and, from nvrec_decode only:
 *   6 "payload range is not whole RLE records";
 *   7 "payload sample count disagrees with header"   (UndecodableError)
 *   8 "P-frame decode requires a reference plane"    (ValueError)
 *   9 plane_capacity too small                       (caller error) */

/* One frame of codec.decode(enc, reference, zero_fill_ranges)
 * (codec.py:260-321).  DEVICE pointers.  `mask` describes the header and
 * the zero-filled ranges exactly as for nvrec_loss_mask and receives the
 * grid / wire bits / status; mask.payload_received = len(enc.payload), the
 * number of bytes at `payload` (the receiver's assembled body, zero chunks
 * included, receiver.py:228-237).  The output plane is (h, w, c) u8 from
 * the header; reference has the same shape and is required for P-frames
 * (it may alias plane: in-place decode into a reference ring slot). */
typedef struct nvrec_decode_job {
  nvrec_lossmask_job mask;
  const uint8_t* payload;
  const uint8_t* reference;
  uint8_t* plane;
  int64_t plane_capacity;     /* bytes available at plane                     */
  int32_t* scratch;           /* int32[2 * mask.grid_capacity + 4] device scratch */
} nvrec_decode_job;

/* Batched decode: jobs is a DEVICE array; max_blocks >= every job's block
 * count (h/block * w/block).  Bit-exact with the reference.  Error policy
 * (LOST_FRAME, receiver.py:244-248): a job that ends with a nonzero status
 * has its wire bits cleared and, when it has a reference distinct from
 * plane, plane_capacity bytes of the reference copied into plane (the
 * reference must span plane_capacity bytes), so the slot repeats the newest
 * displayable plane instead of holding a stale one. */
int nvrec_decode(const nvrec_decode_job* jobs, int32_t n_jobs, int32_t max_blocks, void* stream);

/* Reed-Solomon erasure reconstruction (fec.rs_reconstruct, fec.py:144-163).
 * nvrec_rs_plan runs on the HOST: given n data + r parity shards and
 * present (u8[n+r], nonzero = received) it picks the first n present shards
 * (sources, int32[n]; index < n = data shard, >= n = parity shard), lists
 * the m missing data shards (missing, int32[>= r]) and writes the m x n GF(2^8)
 * decode coefficients (coef, u8[>= r*n]).  Returns NVREC_E_INVALID with
 * "only %d of %d required shards present" when fewer than n survive
 * (UnrecoverableError).  m == 0 means the systematic fast path (no work). */
int nvrec_rs_plan(int32_t n, int32_t r, const uint8_t* present, uint8_t* coef,
                  int32_t* sources, int32_t* missing, int32_t* m_out);

typedef struct nvrec_rs_job {
  uint8_t* data;              /* n x shard_len: present data shards in place;
                                 the m missing rows are written              */
  const uint8_t* parity;      /* r x shard_len received parity shards        */
  const uint8_t* coef;        /* m x n (nvrec_rs_plan)                       */
  const int32_t* sources;     /* n                                            */
  const int32_t* missing;     /* m                                            */
  int32_t n, r, m, shard_len;
} nvrec_rs_job;

/* Batched GF(2^8) reconstruction of the missing data rows (DEVICE jobs
 * array); max_shard_len >= every shard_len, max_coef >= every m*n. */
int nvrec_rs_reconstruct(const nvrec_rs_job* jobs, int32_t n_jobs, int32_t max_shard_len,
                         int32_t max_coef, int32_t aligned4, void* stream);

/* Timeout / fault fallback on the GPU, bit-exact with the reference
 * recover_baseline_rgb / recover_baseline_depth (rgbdstream/recovery.py:94-196):
 * +-8 px SAD block match of every masked 16-px block against the most recent
 * reference on its intact border ring; depth adds the 3x3 median on the
 * mask-boundary band.  planes/refs/out: (b, h, w, c) u8 device; mask_bits as
 * in nvrec_recover_u8.  (No references => the caller returns the plane.) */
int64_t nvrec_baseline_workspace_bytes(int32_t b, int32_t h, int32_t w, int32_t c);
int nvrec_baseline_u8(int32_t depth, int32_t b, int32_t h, int32_t w, int32_t c,
                      const uint8_t* planes, const uint8_t* refs, const uint8_t* mask_bits,
                      uint8_t* out, void* workspace, int64_t workspace_bytes, void* stream);

/* Optional per-stage timing for benchmarks: between begin and end every
 * kernel launch is bracketed by CUDA events on its stream; end synchronises
 * and returns the summed milliseconds and kernel-launch counts per
 * NVREC_STAGE_*.  Returns the number of kernels launched.  Not thread-safe;
 * off by default. */
enum {
  NVREC_STAGE_LOSSMASK = 0, NVREC_STAGE_MASKLIST = 1, NVREC_STAGE_COPY = 2,
  NVREC_STAGE_EMBED = 3, NVREC_STAGE_LNQKV = 4, NVREC_STAGE_ATTN_SIMT = 5,
  NVREC_STAGE_ATTN_TC = 6, NVREC_STAGE_TOKEN = 7, NVREC_STAGE_BASELINE = 8,
  NVREC_STAGE_DECODE = 9, NVREC_STAGE_RS = 10, NVREC_STAGE_LAST_TC = 11,
  NVREC_NUM_STAGES = 12
};
int nvrec_profile_begin(void);
int nvrec_profile_end(float* ms_per_stage, int32_t* launches_per_stage, int32_t n_stages);

/* Diagnostics: attention work items (query group x key split x sequence) the
 * exact fix-up launch has recomputed on the current device since the process
 * started (the speculative running max overflowed for them).  Synchronises
 * the device. */
int64_t nvrec_attn_fixup_items(void);

#ifdef __cplusplus
}
#endif
#endif /* NVREC_B200_H */
