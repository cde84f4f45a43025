// capi.cu -- the C-ABI (include/nvrec_b200.h): model objects, weight
// packing, workspace carve-up and the per-forward launch sequence.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cstdarg>
#include <cmath>

#include "launch.cuh"

#include <cstdlib>

#include <map>
#include <mutex>
#include <utility>

cudaError_t nvrec::smem_optin(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;   // (kernel, device) -> bytes
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_pair(kernel, dev);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done[key] = bytes;
  return e;
}

int nvrec::sm_count() {
  static std::mutex mu;
  static std::map<int, int> sms;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lock(mu);
  auto it = sms.find(dev);
  if (it != sms.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1)
    return 148;
  sms[dev] = n;
  return n;
}

bool nvrec::pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("NVREC_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(NVREC_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK(expr, what)                                  \
  do {                                                  \
    cudaError_t _e = (expr);                            \
    if (_e != cudaSuccess) return cuda_fail(_e, what);  \
  } while (0)

}  // namespace


// ---- optional per-stage timing (bench.py roofline) ----------------------------
// When enabled, every kernel launch of the library is bracketed by a pair of
// CUDA events recorded on the launching stream; nvrec_profile_end sums the
// durations per stage.  Off by default (zero overhead on the hot path).
namespace {
constexpr int kProfMax = 8192;
struct ProfRec { cudaEvent_t a, b; int kind, kernels; };
bool g_prof = false;
std::vector<ProfRec> g_prof_pool;
int g_prof_n = 0;

struct ProfScope {
  ProfRec* r = nullptr;
  cudaStream_t s;
  ProfScope(int kind, cudaStream_t st) : s(st) {
    if (!g_prof || g_prof_n >= int(g_prof_pool.size())) return;
    r = &g_prof_pool[g_prof_n++];
    r->kind = kind;
    r->kernels = 1;
    cudaEventRecord(r->a, s);
  }
  // kernels launched inside this scope (default one)
  void kernels(int n) { if (r) r->kernels = n; }
  ~ProfScope() { if (r) cudaEventRecord(r->b, s); }
};
}  // namespace

struct nvrec_model {
  nvrec_config cfg;
  nvrec::Dims D;
  int device = 0;
  float* blob = nullptr;        // all packed fp32 weights
  size_t blob_floats = 0;
  __half* blob_bf16 = nullptr;          // tensor-core operand packs (fast path, fp16)
  __half* blob_x3 = nullptr;            // split-fp16 [hi | lo] packs (precise path)
  nvrec::ModelW W{};
  bool loaded = false;
};

namespace {

using nvrec::Dims;

Dims make_dims(const nvrec_config& c, int channels) {
  Dims D;
  D.c = channels;
  D.d = c.dim;
  D.heads = c.heads;
  D.hd = c.dim / c.heads;
  D.T = c.tubelet_t;
  D.p = c.patch;
  int raw = c.k + 1;
  D.F = raw + ((c.tubelet_t - raw % c.tubelet_t) % c.tubelet_t);
  D.nt = D.F / D.T;
  D.layers = c.layers;
  D.hidden = 4 * c.dim;
  D.kimg = channels * D.T * D.p * D.p;
  D.used = D.p * D.p * channels;
  return D;
}

// expected numel of each state-dict tensor, in state-dict order
std::vector<int64_t> expected_numel(const Dims& D) {
  std::vector<int64_t> v;
  const int64_t d = D.d;
  v.push_back(int64_t(D.nt) * d);                                  // time_pos
  v.push_back(d * (D.c + 1) * D.T * D.p * D.p);                    // embed.weight
  v.push_back(d);                                                  // embed.bias
  for (int i = 0; i < D.layers; ++i) {
    const int64_t blk[18] = {d, d, 3 * d * d, 3 * d, d * d, d,     // norm_s, attn_s
                             d, d, 3 * d * d, 3 * d, d * d, d,     // norm_t, attn_t
                             d, d, 4 * d * d, 4 * d, 4 * d * d, d};// norm_m, mlp
    v.insert(v.end(), blk, blk + 18);
  }
  v.push_back(d);
  v.push_back(d);                                                  // norm
  v.push_back(int64_t(D.T) * D.p * D.p * D.c * d);                 // head.weight
  v.push_back(int64_t(D.T) * D.p * D.p * D.c);                     // head.bias
  return v;
}

// nn.Linear weight (out, in) -> K-major [in][out]
void transpose_into(std::vector<float>& dst, const float* w, int out, int in) {
  for (int k = 0; k < in; ++k)
    for (int n = 0; n < out; ++n) dst.push_back(w[size_t(n) * in + k]);
}

struct WorkspaceLayout {
  size_t x, ao, q, k, v, qh, kh, vth, list, rank, count, part, redo, xh, total;
};

// Attention variant of a forward: 0 = fp32 SIMT (shapes outside the tensor-
// core envelope), 1 = bf16 tensor cores (fast), 2 = split-bf16 tensor cores
// (precise: hi*hi + hi*lo + lo*hi, fp32-class products).
// NVREC_PRECISE_SIMT=1: the precise path's embedding and block tails on the
// fp32 CUDA-core kernels (A/B of the split-operand tensor-core kernels)
bool precise_simt() {
  static const bool on = [] {
    const char* e = getenv("NVREC_PRECISE_SIMT");
    return e && e[0] == '1';
  }();
  return on;
}

bool f32_embed_simt() {   // NVREC_F32_EMBED_SIMT=1: the float API embeds on CUDA cores (A/B)
  static const bool on = [] {
    const char* e = getenv("NVREC_F32_EMBED_SIMT");
    return e && e[0] == '1';
  }();
  return on;
}

bool last_simt() {
  static const bool on = [] {
    const char* e = getenv("NVREC_LAST_SIMT");
    return e && e[0] == '1';
  }();
  return on;
}

int attn_mode(const Dims& D, int precision) {
  if (!nvrec::tc_supported(D)) return 0;
  return precision == NVREC_PREC_FAST ? 1 : 2;
}

WorkspaceLayout layout_ws(const Dims& D, int b, int h, int w, int precision) {
  const int ns = (h / D.p) * (w / D.p);
  const int ns_pad = nvrec::round_up(ns, nvrec::kAttnQTile);
  WorkspaceLayout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t tok = size_t(b) * D.nt * ns;
  const size_t seqrows = size_t(b) * D.nt * D.heads * ns_pad * D.hd;
  L.x = take(tok * D.d * 4);
  L.ao = take(tok * D.d * 4);
  const int am = attn_mode(D, precision);
  if (am) {
    L.xh = am == 1 ? take(tok * D.d * 2) : SIZE_MAX;
    const size_t sz = seqrows * 2 * (am == 2 ? 2 : 1);   // x3: hi and lo
    L.qh = take(sz);
    L.kh = take(sz);
    L.vth = take(sz);
    L.q = L.k = L.v = SIZE_MAX;
    L.part = take(size_t(nvrec::kAttnMaxSplits) * b * D.nt * D.heads * ns * 36 * 4);
    // work items: query groups (>= one 128-query tile) x splits x sequences
    // (+ the count and the fix-up exit counter)
    L.redo = take((2 + size_t(nvrec::kAttnMaxSplits) * b * D.nt * D.heads *
                   ((ns + nvrec::kAttnQTile - 1) / nvrec::kAttnQTile)) * 4);
  } else {
    L.q = take(seqrows * 4);
    L.k = take(seqrows * 4);
    L.v = take(seqrows * 4);
    L.qh = L.kh = L.vth = L.part = L.redo = L.xh = SIZE_MAX;
  }
  L.list = take(size_t(b) * ns * 4);
  L.rank = take(size_t(b) * ns * 4);
  L.count = take(size_t(b) * 4);
  L.total = off;
  return L;
}

template <class T>
T* at(void* base, size_t off) {
  return off == SIZE_MAX ? nullptr : reinterpret_cast<T*>(static_cast<char*>(base) + off);
}

int check_arch(const nvrec_config* cfg, int channels) {
  if (!cfg) return fail(NVREC_E_INVALID, "null config");
  if (channels != 1 && channels != 3) return fail(NVREC_E_INVALID, "channels must be 1 or 3");
  if (cfg->k < 1 || cfg->tubelet_t < 1 || cfg->patch < 1 || cfg->dim < 1 ||
      cfg->layers < 1 || cfg->heads < 1 || cfg->dim % cfg->heads)
    return fail(NVREC_E_INVALID, "invalid ModelConfig");
  const int hd = cfg->dim / cfg->heads;
  if (cfg->dim % 16 || cfg->dim > nvrec::kMaxDim || !(hd == 8 || hd == 16 || hd == 32 || hd == 64))
    return fail(NVREC_E_UNSUPPORTED, "unsupported dim/heads (dim %% 16 == 0, dim <= 128, "
                "dim/heads in {8,16,32,64}); got dim=%d heads=%d", cfg->dim, cfg->heads);
  if (cfg->layers > 8) return fail(NVREC_E_UNSUPPORTED, "layers > 8 unsupported");
  int raw = cfg->k + 1;
  int F = raw + ((cfg->tubelet_t - raw % cfg->tubelet_t) % cfg->tubelet_t);
  if (F / cfg->tubelet_t > nvrec::kMaxNt) return fail(NVREC_E_UNSUPPORTED, "too many time slices");
  if ((cfg->patch * cfg->patch * channels) % 4)
    return fail(NVREC_E_UNSUPPORTED, "patch*patch*channels must be a multiple of 4");
  return 0;
}

// Shared launch sequence after the embedding: blocks, attention, head.
// In-place merge target (out_u8 == null on the u8 path): stream b's corrupted
// plane, frames + frame_index[b * F + F - 1] * frame_bytes.
struct InPlace {
  uint8_t* frames = nullptr;
  const int32_t* frame_index = nullptr;
};

int run_blocks(const nvrec_model* m, nvrec::Act& A, const WorkspaceLayout& L, int am,
               bool pruned, int h, int w, float* out_f32, uint8_t* out_u8,
               cudaStream_t s, InPlace ip = {}, bool u16 = false) {
  const Dims& D = m->D;
  const int b = A.b;
  const bool fast = am == 1;
  nvrec::QkvDst dst{};
  dst.nt = D.nt; dst.ns = A.ns; dst.ns_pad = A.ns_pad; dst.d = D.d;
  dst.heads = D.heads; dst.hd = D.hd;
  dst.q = A.q; dst.k = A.k; dst.v = A.v; dst.qh = A.qh; dst.kh = A.kh; dst.vth = A.vth;
  dst.x3 = am == 2;
  // arm the attention fix-up list once per forward (every fix-up launch
  // leaves it empty again)
  if (am && A.redo_list) CK(cudaMemsetAsync(A.redo_list, 0, 2 * sizeof(int), s), "memset");
  for (int li = 0; li < D.layers; ++li) {
    const bool last = li == D.layers - 1;
    const bool prune_here = last && pruned;
    // block li's spatial attention: Q/K/V were written by the previous stage
    cudaError_t e;
    int splits = 1;
    // tensor-core tail of a non-last block: token_tc (fast) / token_x3 (precise)
    const bool tc_tail = !last && nvrec::token_tc_supported(D) &&
                         (fast ? m->W.tc.blk[li] != nullptr
                               : (am == 2 && m->W.tc.blk3[li] != nullptr && !precise_simt()));
    // tensor-core last block + head (k_last_tc.cu); NVREC_LAST_SIMT=1 keeps the
    // CUDA-core token_kernel (A/B)
    const bool last_tc = last && am != 0 && m->W.tc.last3 != nullptr && !precise_simt() &&
                         !last_simt() && nvrec::last_tc_supported(D, b);
    if (am) {
      ProfScope ps(NVREC_STAGE_ATTN_TC, s);
      int nk = 1;
      // the SIMT token kernel merges key-split partials itself; the tensor-core
      // last block reads merged rows (attn_combine_kernel: one thread per
      // element instead of a serial per-row merge on the last block's lanes)
      const bool defer = !tc_tail && !last_tc;
      e = nvrec::launch_attn_tc(A, D, prune_here ? A.count : nullptr, s, &nk, defer, &splits,
                                fast && tc_tail,   // token_tc reads ao as fp16
                                am == 2);
      ps.kernels(nk);
    } else {
      nvrec::AttnArgs aa{};
      aa.q = A.q; aa.k = A.k; aa.v = A.v; aa.ao = A.ao;
      aa.count = prune_here ? A.count : nullptr;
      aa.nt = D.nt; aa.heads = D.heads; aa.ns = A.ns; aa.ns_pad = A.ns_pad; aa.d = D.d;
      aa.scale_log2 = 1.4426950408889634f / sqrtf(float(D.hd));
      ProfScope ps(NVREC_STAGE_ATTN_SIMT, s);
      e = nvrec::launch_attn_simt(aa, b, A.ns, s);
    }
    if (e != cudaSuccess) return cuda_fail(e, "spatial attention launch");
    nvrec::TokenArgs ta{};
    ta.D = D;
    ta.w = m->W.blk[li];
    if (!last) ta.wn = m->W.blk[li + 1];
    ta.norm_w = m->W.norm_w; ta.norm_b = m->W.norm_b;
    ta.head_w = m->W.head_w; ta.head_b = m->W.head_b;
    ta.last = last;
    ta.list = prune_here ? A.list : nullptr;
    ta.count = A.count;
    ta.x = A.x; ta.ao = A.ao;
    ta.part = A.part; ta.splits = splits;
    ta.dst = dst;
    // the next block is the last: its Q rows are compact when pruned
    ta.dst.rank = (!last && li + 1 == D.layers - 1 && pruned) ? A.rank : nullptr;
    ta.img_h = h; ta.img_w = w; ta.nh = A.nh; ta.nw = A.nw; ta.ns = A.ns;
    ta.out_f32 = out_f32; ta.out_u8 = out_u8;
    ta.out_frames = ip.frames;
    ta.out_slot = ip.frame_index ? ip.frame_index + (D.F - 1) : nullptr;
    ta.slot_stride = D.F;
    ta.frame_bytes = size_t(h) * w * D.c * (u16 ? 2 : 1);
    if (last_tc) {
      const nvrec::BlockW& bw = m->W.blk[li];
      nvrec::LastTcArgs la{};
      la.b = b; la.ns = A.ns; la.nt = D.nt; la.c = D.c;
      la.img_h = h; la.img_w = w; la.nw = A.nw;
      la.list = ta.list;
      la.count = ta.list ? A.count : nullptr;
      la.x = A.x; la.ao = A.ao;
      la.w_blk = m->W.tc.last3;
      la.w_head = m->W.tc.head3;
      for (int j = 0; j < 5; ++j) la.sc[j] = m->W.tc.sc_blk[li][j];
      la.sc_head = m->W.tc.sc_head;
      la.b_proj_s = bw.proj_s_b; la.ln_t_w = bw.ln_t_w; la.ln_t_b = bw.ln_t_b;
      la.b_qkv_t = bw.qkv_t_b; la.b_proj_t = bw.proj_t_b; la.ln_m_w = bw.ln_m_w;
      la.ln_m_b = bw.ln_m_b; la.b_fc1 = bw.fc1_b; la.b_fc2 = bw.fc2_b;
      la.norm_w = m->W.norm_w; la.norm_b = m->W.norm_b; la.head_b = m->W.head_b;
      la.out_f32 = out_f32; la.out_u8 = out_u8;
      la.out_frames = ip.frames; la.out_slot = ta.out_slot;
      la.slot_stride = D.F; la.frame_bytes = ta.frame_bytes;
      la.u16 = u16;
      static const int hs_env = [] {
        const char* e = getenv("NVREC_LAST_HSPLIT");   // A/B: CTAs per tile cap
        return e ? atoi(e) : 4;
      }();
      la.max_hsplit = hs_env;
      ProfScope ps(NVREC_STAGE_LAST_TC, s);
      e = nvrec::launch_last_tc(la, b * A.ns, s);
    } else if (tc_tail && am == 2) {
      const nvrec::BlockW& bw = m->W.blk[li];
      const nvrec::BlockW& bn = m->W.blk[li + 1];
      nvrec::TokenX3Args tt{};
      tt.b = b; tt.ns = A.ns; tt.ns_pad = A.ns_pad; tt.nt = D.nt;
      tt.x = A.x; tt.ao = A.ao;
      tt.w_blk = m->W.tc.blk3[li];
      tt.w_next = m->W.tc.blk3[li + 1];
      for (int j = 0; j < 5; ++j) tt.sc[j] = m->W.tc.sc_blk[li][j];
      tt.sc[5] = m->W.tc.sc_blk[li + 1][5];
      tt.b_proj_s = bw.proj_s_b; tt.ln_t_w = bw.ln_t_w; tt.ln_t_b = bw.ln_t_b;
      tt.b_qkv_t = bw.qkv_t_b; tt.b_proj_t = bw.proj_t_b; tt.ln_m_w = bw.ln_m_w;
      tt.ln_m_b = bw.ln_m_b; tt.b_fc1 = bw.fc1_b; tt.b_fc2 = bw.fc2_b;
      tt.ln_s_next_w = bn.ln_s_w; tt.ln_s_next_b = bn.ln_s_b; tt.b_qkv_next = bn.qkv_s_b;
      tt.qh = A.qh; tt.kh = A.kh; tt.vth = A.vth;
      tt.qrank = ta.dst.rank;
      ProfScope ps(NVREC_STAGE_TOKEN, s);
      ps.kernels(3);
      e = nvrec::launch_token_x3(tt, s);
    } else if (tc_tail) {
      const nvrec::BlockW& bw = m->W.blk[li];
      const nvrec::BlockW& bn = m->W.blk[li + 1];
      nvrec::TokenTcArgs tt{};
      tt.b = b; tt.ns = A.ns; tt.ns_pad = A.ns_pad; tt.nt = D.nt;
      tt.x = A.x; tt.ao = reinterpret_cast<const __half*>(A.ao);
      tt.xh = (li == 0 && A.x_half) ? A.xh : nullptr;
      tt.w_blk = m->W.tc.blk[li];
      tt.w_qkv_next = m->W.tc.blk[li + 1] + 53248;
      tt.b_proj_s = bw.proj_s_b; tt.ln_t_w = bw.ln_t_w; tt.ln_t_b = bw.ln_t_b;
      tt.b_qkv_t = bw.qkv_t_b; tt.b_proj_t = bw.proj_t_b; tt.ln_m_w = bw.ln_m_w;
      tt.ln_m_b = bw.ln_m_b; tt.b_fc1 = bw.fc1_b; tt.b_fc2 = bw.fc2_b;
      tt.ln_s_next_w = bn.ln_s_w; tt.ln_s_next_b = bn.ln_s_b; tt.b_qkv_next = bn.qkv_s_b;
      tt.qh = A.qh; tt.kh = A.kh; tt.vth = A.vth;
      tt.qrank = ta.dst.rank;
      ProfScope ps(NVREC_STAGE_TOKEN, s);
      e = nvrec::launch_token_tc(tt, s);
    } else {
      ProfScope ps(NVREC_STAGE_TOKEN, s);
      e = nvrec::launch_token(ta, b, A.ns, s);
    }
    if (e != cudaSuccess) return cuda_fail(e, "token kernel launch");
  }
  return 0;
}

}  // namespace

extern "C" {

int nvrec_abi_version(void) { return NVREC_ABI_VERSION; }
const char* nvrec_last_error(void) { return g_err.c_str(); }

int nvrec_model_create(const nvrec_config* cfg, int32_t channels, nvrec_model** out) {
  if (!out) return fail(NVREC_E_INVALID, "null out");
  int rc = check_arch(cfg, channels);
  if (rc) return rc;
  nvrec_model* m = new nvrec_model();
  m->cfg = *cfg;
  m->D = make_dims(*cfg, channels);
  cudaGetDevice(&m->device);
  *out = m;
  return 0;
}

int nvrec_model_destroy(nvrec_model* m) {
  if (!m) return 0;
  if (m->blob) cudaFree(m->blob);
  if (m->blob_bf16) cudaFree(m->blob_bf16);
  if (m->blob_x3) cudaFree(m->blob_x3);
  delete m;
  return 0;
}

int nvrec_model_load(nvrec_model* m, const float* const* t, const int64_t* numel,
                     int32_t n) {
  if (!m || !t || !numel) return fail(NVREC_E_INVALID, "null argument");
  const Dims& D = m->D;
  std::vector<int64_t> want = expected_numel(D);
  if (n != int(want.size()))
    return fail(NVREC_E_INVALID, "expected %d state tensors, got %d", int(want.size()), n);
  for (int i = 0; i < n; ++i)
    if (numel[i] != want[i])
      return fail(NVREC_E_INVALID, "state tensor %d has %lld elements, expected %lld", i,
                  (long long)numel[i], (long long)want[i]);
  const int d = D.d, p = D.p, c = D.c, T = D.T;
  std::vector<float> h;
  std::vector<size_t> off;
  auto mark = [&]() { off.push_back(h.size()); };
  // embed: W[o][ci][tt][py][px] -> [((tt*p+py)*p+px)*c+ci][o]
  const float* ew = t[1];
  auto ew_at = [&](int o, int ci, int tt, int py, int px) {
    return ew[((((size_t)o * (c + 1) + ci) * T + tt) * p + py) * p + px];
  };
  mark();  // 0 emb_w
  for (int tt = 0; tt < T; ++tt)
    for (int py = 0; py < p; ++py)
      for (int px = 0; px < p; ++px)
        for (int ci = 0; ci < c; ++ci)
          for (int o = 0; o < d; ++o) h.push_back(ew_at(o, ci, tt, py, px));
  mark();  // 1 emb_wmask [p*p][d] at tt = T-1, channel c
  for (int py = 0; py < p; ++py)
    for (int px = 0; px < p; ++px)
      for (int o = 0; o < d; ++o) h.push_back(ew_at(o, c, T - 1, py, px));
  mark();  // 2 emb_wmsum
  for (int o = 0; o < d; ++o) {
    float sacc = 0.f;
    for (int py = 0; py < p; ++py)
      for (int px = 0; px < p; ++px) sacc += ew_at(o, c, T - 1, py, px);
    h.push_back(sacc);
  }
  mark();  // 3 emb_b
  h.insert(h.end(), t[2], t[2] + d);
  mark();  // 4 time_pos
  h.insert(h.end(), t[0], t[0] + size_t(D.nt) * d);
  std::vector<size_t> blk_off;
  for (int i = 0; i < D.layers; ++i) {
    const float* const* bt = t + 3 + 18 * i;
    // order inside BlockW: ln_s_w, ln_s_b, qkv_s_w, qkv_s_b, proj_s_w, proj_s_b,
    //   ln_t_w, ln_t_b, qkv_t_w, qkv_t_b, proj_t_w, proj_t_b,
    //   ln_m_w, ln_m_b, fc1_w, fc1_b, fc2_w, fc2_b
    const int outs[18] = {0, 0, 3 * d, 0, d, 0, 0, 0, 3 * d, 0, d, 0, 0, 0, 4 * d, 0, d, 0};
    const int ins[18] = {0, 0, d, 0, d, 0, 0, 0, d, 0, d, 0, 0, 0, d, 0, 4 * d, 0};
    for (int j = 0; j < 18; ++j) {
      blk_off.push_back(h.size());
      if (outs[j]) transpose_into(h, bt[j], outs[j], ins[j]);
      else h.insert(h.end(), bt[j], bt[j] + want[3 + 18 * i + j]);
      while (h.size() % 4) h.push_back(0.f);   // keep float4 alignment
    }
  }
  const int tail = 3 + 18 * D.layers;
  mark();  // 5 norm_w
  h.insert(h.end(), t[tail], t[tail] + d);
  mark();  // 6 norm_b
  h.insert(h.end(), t[tail + 1], t[tail + 1] + d);
  // head: keep rows ((T-1)*p*p + py*p + px)*c + ch (model.py:119-120), K-major
  mark();  // 7 head_w [d][used]
  const float* hw = t[tail + 2];
  const size_t base_row = size_t(T - 1) * p * p * c;
  for (int k = 0; k < d; ++k)
    for (int u = 0; u < D.used; ++u) h.push_back(hw[(base_row + u) * d + k]);
  while (h.size() % 4) h.push_back(0.f);   // head_b read as float4 (k_last_tc.cu)
  mark();  // 8 head_b
  for (int u = 0; u < D.used; ++u) h.push_back(t[tail + 3][base_row + u]);

  if (m->blob) { cudaFree(m->blob); m->blob = nullptr; }
  CK(cudaSetDevice(m->device), "cudaSetDevice");
  CK(cudaMalloc(&m->blob, h.size() * sizeof(float)), "cudaMalloc(weights)");
  CK(cudaMemcpy(m->blob, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice),
     "cudaMemcpy(weights)");
  m->blob_floats = h.size();
  float* B = m->blob;
  m->W.emb_w = B + off[0];
  m->W.emb_wmask = B + off[1];
  m->W.emb_wmsum = B + off[2];
  m->W.emb_b = B + off[3];
  m->W.time_pos = B + off[4];
  for (int i = 0; i < D.layers; ++i) {
    const float* p18[18];
    for (int j = 0; j < 18; ++j) p18[j] = B + blk_off[18 * i + j];
    nvrec::BlockW& bw = m->W.blk[i];
    bw.ln_s_w = p18[0]; bw.ln_s_b = p18[1]; bw.qkv_s_w = p18[2]; bw.qkv_s_b = p18[3];
    bw.proj_s_w = p18[4]; bw.proj_s_b = p18[5];
    bw.ln_t_w = p18[6]; bw.ln_t_b = p18[7]; bw.qkv_t_w = p18[8]; bw.qkv_t_b = p18[9];
    bw.proj_t_w = p18[10]; bw.proj_t_b = p18[11];
    bw.ln_m_w = p18[12]; bw.ln_m_b = p18[13]; bw.fc1_w = p18[14]; bw.fc1_b = p18[15];
    bw.fc2_w = p18[16]; bw.fc2_b = p18[17];
  }
  m->W.norm_w = B + off[5];
  m->W.norm_b = B + off[6];
  m->W.head_w = B + off[7];
  m->W.head_b = B + off[8];
  // ---- bf16 UMMA packs for the tensor-core path ----------------------------
  if (m->blob_bf16) { cudaFree(m->blob_bf16); m->blob_bf16 = nullptr; }
  if (nvrec::embed_tc_supported(D)) {
    // fp16 operands: u8 pixels are exact in fp16 and fp16 keeps 3 more
    // mantissa bits of the weights than bf16
    std::vector<__half> hb;
    auto pack = [&](int N, int K, auto at) {   // at(n, k) -> float
      size_t base = hb.size();
      hb.resize(base + size_t(N) * K);
      for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k)
          hb[base + (size_t(k / 8) * (N / 8) + n / 8) * 64 + (n % 8) * 8 + k % 8] =
              __float2half_rn(at(n, k));
      return base;
    };
    const int kst = 32 * c;                         // K per stage: 2 patch rows
    std::vector<size_t> stage_off;
    for (int st = 0; st < T * 8; ++st) {
      const int tt = st / 8, py0 = 2 * (st % 8);
      stage_off.push_back(pack(d, kst, [&](int n, int k) {
        const int pyl = k / (16 * c), rem = k % (16 * c), px = rem / c, ci = rem % c;
        return ew_at(n, ci, tt, py0 + pyl, px);
      }));
    }
    const float* q0 = t[3 + 2];                      // blocks.0.attn_s.qkv.weight (3d, d)
    size_t qoff = pack(3 * d, d, [&](int n, int k) { return q0[size_t(n) * d + k]; });
    std::vector<size_t> blk_pack;
    for (int i = 0; i < D.layers; ++i) {
      const float* const* bt = t + 3 + 18 * i;
      auto lin = [&](const float* wt, int N, int K) {
        return pack(N, K, [&](int n, int k) { return wt[size_t(n) * K + k]; });
      };
      blk_pack.push_back(lin(bt[4], d, d));            // attn_s.proj
      lin(bt[8], 3 * d, d);                            // attn_t.qkv
      lin(bt[10], d, d);                               // attn_t.proj
      lin(bt[14], 4 * d, d);                           // mlp.0
      lin(bt[16], d, 4 * d);                           // mlp.2
      lin(bt[2], 3 * d, d);                            // attn_s.qkv
    }
    // 16-bit depth embedding (k_embed_tc.cu, C == 2): per 2-patch-row stage,
    // K = (py, px, byte), byte 0 = lo (W), byte 1 = hi (256 W)
    auto at16 = [&](int tt, int py0) {
      return [&, tt, py0](int n, int k) {
        const int pyl = k / 32, rem = k % 32, px = rem / 2;
        return ew_at(n, 0, tt, py0 + pyl, px) * ((rem & 1) ? 256.f : 1.f);
      };
    };
    size_t emb16_off = SIZE_MAX;
    if (c == 1)
      for (int st = 0; st < T * 8; ++st) {
        const size_t o = pack(d, 64, at16(st / 8, 2 * (st % 8)));
        if (st == 0) emb16_off = o;
      }
    // float module-API embedding (k_embed_tc.cu, F32): stages of 2 rows of one
    // channel (tt, ch, rp), then the mask channel's 8 stages (last sub-frame)
    auto atf = [&](int st) {
      const int nimg = T * c * 8;
      const int tt = st < nimg ? st / (c * 8) : T - 1;
      const int ch = st < nimg ? (st / 8) % c : c;
      const int rp = st < nimg ? st % 8 : st - nimg;
      return [&, tt, ch, rp](int n, int k) { return ew_at(n, ch, tt, 2 * rp + k / 16, k % 16); };
    };
    const int nstf = T * c * 8 + 8;
    size_t embf_off = 0;
    for (int st = 0; st < nstf; ++st) {
      const size_t o = pack(d, 32, atf(st));
      if (st == 0) embf_off = o;
    }
    CK(cudaMalloc(&m->blob_bf16, hb.size() * sizeof(__half)), "cudaMalloc(fp16)");
    CK(cudaMemcpy(m->blob_bf16, hb.data(), hb.size() * sizeof(__half),
                  cudaMemcpyHostToDevice), "cudaMemcpy(fp16)");
    m->W.tc.emb = m->blob_bf16 + stage_off[0];
    m->W.tc.emb_stage_elems = d * kst;
    m->W.tc.qkv0 = m->blob_bf16 + qoff;
    for (int i = 0; i < D.layers; ++i) m->W.tc.blk[i] = m->blob_bf16 + blk_pack[i];
    m->W.tc.emb16 = emb16_off == SIZE_MAX ? nullptr : m->blob_bf16 + emb16_off;
    m->W.tc.embf = m->blob_bf16 + embf_off;

    // ---- split-fp16 [hi | lo] packs for the precise path ----------------------
    // W * 2^s with max|W| 2^s in [2^13, 2^14): hi = fp16(W 2^s) and lo =
    // fp16(W 2^s - hi) keep 22 significant bits and lo stays normal; the
    // kernels multiply their accumulators by 2^-s (TcW::sc_*).
    if (m->blob_x3) { cudaFree(m->blob_x3); m->blob_x3 = nullptr; }
    std::vector<__half> h3;
    auto exponent_for = [](float mx) {
      if (!(mx > 0.f) || !std::isfinite(mx)) return 0;
      const int s = int(std::floor(std::log2(16384.0 / double(mx))));
      return s < -60 ? -60 : (s > 60 ? 60 : s);
    };
    auto pack2 = [&](int N, int K, auto at, int sexp) {
      const size_t base = h3.size();
      h3.resize(base + 2 * size_t(N) * K);
      for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) {
          const size_t idx = (size_t(k / 8) * (N / 8) + n / 8) * 64 + (n % 8) * 8 + k % 8;
          const float v = std::ldexp(at(n, k), sexp);
          const __half hi = __float2half_rn(v);
          h3[base + idx] = hi;
          h3[base + size_t(N) * K + idx] = __float2half_rn(v - __half2float(hi));
        }
      return base;
    };
    // [hi ; lo] stacked as ONE 2N-row B operand (N = 64 -> an N = 128 MMA
    // computes A W_hi and A W_lo side by side; the epilogue adds the halves):
    // the same core-matrix layout as pack2 with 2N rows
    auto pack2m = [&](int N, int K, auto at, int sexp) {
      const size_t base = h3.size();
      h3.resize(base + 2 * size_t(N) * K);
      for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) {
          const float v = std::ldexp(at(n, k), sexp);
          const __half hi = __float2half_rn(v);
          for (int part = 0; part < 2; ++part) {
            const int r = n + part * N;
            const size_t idx = (size_t(k / 8) * (2 * N / 8) + r / 8) * 64 + (r % 8) * 8 + k % 8;
            h3[base + idx] = part ? __float2half_rn(v - __half2float(hi)) : hi;
          }
        }
      return base;
    };
    auto maxabs = [](int N, int K, auto at) {
      float mx = 0.f;
      for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) mx = std::fmax(mx, std::fabs(at(n, k)));
      return mx;
    };
    // embedding: one exponent for the whole image part of the weight
    float emx = 0.f;
    for (int o = 0; o < d; ++o)
      for (int ci = 0; ci < c; ++ci)
        for (int tt = 0; tt < T; ++tt)
          for (int py = 0; py < p; ++py)
            for (int px = 0; px < p; ++px) emx = std::fmax(emx, std::fabs(ew_at(o, ci, tt, py, px)));
    const int se = exponent_for(emx);
    m->W.tc.sc_emb = std::ldexp(1.f, -se);
    const int kpy3 = c == 3 ? 1 : 2, kst3 = 16 * kpy3 * c;   // embed_tc's X3 K stage (EmbSmem::kPy)
    size_t emb3_off = 0;
    for (int st = 0; st < T * 16 / kpy3; ++st) {
      const int tt = st / (16 / kpy3), py0 = kpy3 * (st % (16 / kpy3));
      const size_t o = pack2m(d, kst3, [&](int n, int k) {
        const int pyl = k / (16 * c), rem = k % (16 * c), px = rem / c, ci = rem % c;
        return ew_at(n, ci, tt, py0 + pyl, px);
      }, se);
      if (st == 0) emb3_off = o;
    }
    auto lin3 = [&](const float* wt, int N, int K, float* sc) {
      auto at = [&](int n, int k) { return wt[size_t(n) * K + k]; };
      const int sx = exponent_for(maxabs(N, K, at));
      *sc = std::ldexp(1.f, -sx);
      return pack2(N, K, at, sx);
    };
    const size_t q3off = lin3(t[3 + 2], 3 * d, d, &m->W.tc.sc_qkv0);
    std::vector<size_t> blk3;
    for (int i = 0; i < D.layers; ++i) {
      const float* const* bt = t + 3 + 18 * i;
      float* sc = m->W.tc.sc_blk[i];
      blk3.push_back(lin3(bt[4], d, d, sc + 0));          // attn_s.proj
      lin3(bt[8], 3 * d, d, sc + 1);                      // attn_t.qkv
      lin3(bt[10], d, d, sc + 2);                         // attn_t.proj
      lin3(bt[14], 4 * d, d, sc + 3);                     // mlp.0
      lin3(bt[16], d, 4 * d, sc + 4);                     // mlp.2
      lin3(bt[2], 3 * d, d, sc + 5);                      // attn_s.qkv
    }
    // 16-bit depth embedding, split: one exponent for lo and hi (x 256) bytes
    size_t emb16_3_off = SIZE_MAX;
    if (c == 1) {
      const int s16 = exponent_for(256.f * emx);
      m->W.tc.sc_emb16 = std::ldexp(1.f, -s16);
      for (int st = 0; st < T * 16; ++st) {             // one patch row per X3 stage
        const size_t o = pack2m(d, 32, at16(st / 16, st % 16), s16);
        if (st == 0) emb16_3_off = o;
      }
    }
    // float module-API embedding, split: one exponent over image + mask channels
    size_t embf3_off = 0;
    {
      float fmx = emx;
      for (int o = 0; o < d; ++o)
        for (int py = 0; py < p; ++py)
          for (int px = 0; px < p; ++px) fmx = std::fmax(fmx, std::fabs(ew_at(o, c, T - 1, py, px)));
      const int sf = exponent_for(fmx);
      m->W.tc.sc_embf = std::ldexp(1.f, -sf);
      for (int st = 0; st < nstf; ++st) {
        const size_t o = pack2(d, 32, atf(st), sf);
        if (st == 0) embf3_off = o;
      }
    }
    // head (last tubelet frame rows, model.py:119-120) in 4 chunks of 4 patch
    // rows = 64c columns: the last-block kernel streams one chunk at a time
    const float* hw3 = t[tail + 2];
    const size_t hrow0 = size_t(T - 1) * p * p * c;
    auto head_at = [&](int n, int k) { return hw3[(hrow0 + n) * d + k]; };
    const int sh = exponent_for(maxabs(D.used, d, head_at));
    m->W.tc.sc_head = std::ldexp(1.f, -sh);
    size_t head3_off = 0;
    const int hchunk = D.used / 4;
    for (int j = 0; j < 4; ++j) {
      const size_t o = pack2(hchunk, d, [&](int n, int k) { return head_at(hchunk * j + n, k); }, sh);
      if (j == 0) head3_off = o;
    }
    // the last block re-packed as the streaming chunks of k_last_tc.cu (each a
    // contiguous [hi | lo] block <= 48 KB): proj_s, qkv_t, proj_t, fc1 rows
    // 0-127 / 128-255, fc2 K 0-127 / 128-255 (same exponents as blk3)
    size_t last3_off = 0;
    {
      const int li = D.layers - 1;
      const float* const* bt = t + 3 + 18 * li;
      const float* sc = m->W.tc.sc_blk[li];
      auto ex = [](float scv) { return -int(std::lround(std::log2(double(scv)))); };
      auto mat = [&](const float* wt, int K, int n0, int k0) {
        return [=](int n, int k) { return wt[size_t(n0 + n) * K + k0 + k]; };
      };
      last3_off = pack2(d, d, mat(bt[4], d, 0, 0), ex(sc[0]));             // proj_s
      pack2(3 * d, d, mat(bt[8], d, 0, 0), ex(sc[1]));                      // qkv_t
      pack2(d, d, mat(bt[10], d, 0, 0), ex(sc[2]));                         // proj_t
      pack2(2 * d, d, mat(bt[14], d, 0, 0), ex(sc[3]));                     // fc1 rows 0..127
      pack2(2 * d, d, mat(bt[14], d, 2 * d, 0), ex(sc[3]));                 // fc1 rows 128..255
      pack2(d, 2 * d, mat(bt[16], 4 * d, 0, 0), ex(sc[4]));                 // fc2 K 0..127
      pack2(d, 2 * d, mat(bt[16], 4 * d, 0, 2 * d), ex(sc[4]));             // fc2 K 128..255
    }
    CK(cudaMalloc(&m->blob_x3, h3.size() * sizeof(__half)), "cudaMalloc(x3)");
    CK(cudaMemcpy(m->blob_x3, h3.data(), h3.size() * sizeof(__half), cudaMemcpyHostToDevice),
       "cudaMemcpy(x3)");
    m->W.tc.emb3 = m->blob_x3 + emb3_off;
    m->W.tc.qkv0_3 = m->blob_x3 + q3off;
    for (int i = 0; i < D.layers; ++i) m->W.tc.blk3[i] = m->blob_x3 + blk3[i];
    m->W.tc.head3 = m->blob_x3 + head3_off;
    m->W.tc.emb16_3 = emb16_3_off == SIZE_MAX ? nullptr : m->blob_x3 + emb16_3_off;
    m->W.tc.embf3 = m->blob_x3 + embf3_off;
    m->W.tc.last3 = m->blob_x3 + last3_off;
  }
  m->loaded = true;
  return 0;
}

int64_t nvrec_workspace_bytes(const nvrec_model* m, int32_t b, int32_t h, int32_t w,
                              int32_t precision) {
  if (!m || b < 1 || h < 1 || w < 1) return fail(NVREC_E_INVALID, "bad shape");
  return int64_t(layout_ws(m->D, b, h, w, precision).total);
}

static int common_checks(const nvrec_model* m, int b, int h, int w, void* ws,
                         int64_t ws_bytes, int precision, WorkspaceLayout* L) {
  if (!m) return fail(NVREC_E_INVALID, "null model");
  if (!m->loaded) return fail(NVREC_E_STATE, "weights not loaded");
  if (b < 1) return fail(NVREC_E_INVALID, "batch must be >= 1");
  if (h % m->D.p || w % m->D.p || h < 1 || w < 1)
    return fail(NVREC_E_INVALID, "frame size must be a multiple of the patch edge");
  if (precision != NVREC_PREC_FAST && precision != NVREC_PREC_PRECISE)
    return fail(NVREC_E_INVALID, "unknown precision %d", precision);
  *L = layout_ws(m->D, b, h, w, precision);
  if (!ws || ws_bytes < int64_t(L->total))
    return fail(NVREC_E_WORKSPACE, "workspace too small: %lld < %lld", (long long)ws_bytes,
                (long long)L->total);
  return 0;
}

static nvrec::Act make_act(const nvrec_model* m, void* ws, const WorkspaceLayout& L, int b,
                           int h, int w) {
  nvrec::Act A{};
  A.x = at<float>(ws, L.x);
  A.xh = L.xh == SIZE_MAX ? nullptr : at<__half>(ws, L.xh);
  A.x_half = false;
  A.ao = at<float>(ws, L.ao);
  A.q = at<float>(ws, L.q);
  A.k = at<float>(ws, L.k);
  A.v = at<float>(ws, L.v);
  A.qh = at<__nv_bfloat16>(ws, L.qh);
  A.kh = at<__nv_bfloat16>(ws, L.kh);
  A.vth = at<__nv_bfloat16>(ws, L.vth);
  A.list = at<int>(ws, L.list);
  A.rank = at<int>(ws, L.rank);
  A.count = at<int>(ws, L.count);
  A.part = at<float>(ws, L.part);
  A.redo_list = at<int>(ws, L.redo);
  A.b = b;
  A.nh = h / m->D.p;
  A.nw = w / m->D.p;
  A.ns = A.nh * A.nw;
  A.ns_pad = nvrec::round_up(A.ns, nvrec::kAttnQTile);
  return A;
}

static int embed_and_qkv0(const nvrec_model* m, nvrec::Act& A, bool u8, const float* stack,
                          int f, const uint8_t* pmask, const uint8_t* frames,
                          const int32_t* frame_index, int h, int w, bool pruned,
                          int precision, cudaStream_t s) {
  const Dims& D = m->D;
  nvrec::EmbedArgs ea{};
  ea.D = D;
  ea.emb_w = m->W.emb_w; ea.emb_wmask = m->W.emb_wmask; ea.emb_wmsum = m->W.emb_wmsum;
  ea.emb_b = m->W.emb_b; ea.time_pos = m->W.time_pos;
  ea.frames = frames; ea.frame_index = frame_index;
  ea.frame_bytes = size_t(h) * w * D.c;
  ea.rank = u8 ? A.rank : nullptr;
  ea.stack = stack; ea.f_in = f; ea.pmask = pmask;
  ea.h = h; ea.w = w; ea.nh = A.nh; ea.nw = A.nw; ea.ns = A.ns;
  ea.x = A.x;
  cudaError_t e;
  {
    ProfScope ps(NVREC_STAGE_EMBED, s);
    e = nvrec::launch_embed(ea, u8, A.b, s);
  }
  if (e != cudaSuccess) return cuda_fail(e, "embed launch");
  nvrec::LnQkvArgs la{};
  la.D = D;
  la.x = A.x;
  la.ln_w = m->W.blk[0].ln_s_w; la.ln_b = m->W.blk[0].ln_s_b;
  la.qkv_w = m->W.blk[0].qkv_s_w; la.qkv_b = m->W.blk[0].qkv_s_b;
  la.dst.q = A.q; la.dst.k = A.k; la.dst.v = A.v;
  la.dst.qh = A.qh; la.dst.kh = A.kh; la.dst.vth = A.vth;
  la.dst.rank = (pruned && D.layers == 1) ? A.rank : nullptr;
  la.dst.nt = D.nt; la.dst.ns = A.ns; la.dst.ns_pad = A.ns_pad; la.dst.d = D.d;
  la.dst.heads = D.heads; la.dst.hd = D.hd;
  la.dst.x3 = attn_mode(D, precision) == 2;
  la.ns = A.ns;
  {
    ProfScope ps(NVREC_STAGE_LNQKV, s);
    e = nvrec::launch_ln_qkv(la, A.b, s);
  }
  if (e != cudaSuccess) return cuda_fail(e, "ln_qkv launch");
  return 0;
}

int nvrec_forward_f32(const nvrec_model* m, const float* stack, int32_t b, int32_t f,
                      int32_t c, int32_t h, int32_t w, const uint8_t* mask, float* out,
                      void* ws, int64_t ws_bytes, int32_t precision, void* stream) {
  if (m && c != m->D.c)
    return fail(NVREC_E_INVALID, "expected %d channels, got %d", m->D.c, c);
  WorkspaceLayout L;
  int rc = common_checks(m, b, h, w, ws, ws_bytes, precision, &L);
  if (rc) return rc;
  if (f < 1 || f > m->D.F) return fail(NVREC_E_INVALID, "stack longer than configured length");
  if (!stack || !mask || !out) return fail(NVREC_E_INVALID, "null tensor pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  nvrec::Act A = make_act(m, ws, L, b, h, w);
  const int am = attn_mode(m->D, precision);
  if (am && nvrec::embed_tc_supported(m->D) && m->W.tc.embf && !precise_simt() &&
      !f32_embed_simt()) {
    // tcgen05 embedding of the float stack (+ block-0 LN/QKV), k_embed_tc.cu F32
    nvrec::EmbedTcArgs ea{};
    ea.f32 = 1;
    ea.x3 = am == 2;
    ea.D = m->D;
    ea.tcw = &m->W.tc;
    ea.emb_wmsum = m->W.emb_wmsum; ea.emb_b = m->W.emb_b; ea.time_pos = m->W.time_pos;
    ea.ln_w = m->W.blk[0].ln_s_w; ea.ln_b = m->W.blk[0].ln_s_b; ea.qkv_b = m->W.blk[0].qkv_s_b;
    ea.stack = stack; ea.f_in = f; ea.pmask = mask;
    ea.x = A.x; ea.qh = A.qh; ea.kh = A.kh; ea.vth = A.vth;
    ea.b = b; ea.h = h; ea.w = w; ea.nh = A.nh; ea.nw = A.nw; ea.ns = A.ns; ea.ns_pad = A.ns_pad;
    cudaError_t e2;
    {
      ProfScope ps(NVREC_STAGE_EMBED, s);
      e2 = nvrec::launch_embed_tc(ea, s);
    }
    if (e2 != cudaSuccess) return cuda_fail(e2, "embed_tc (f32) launch");
  } else {
    rc = embed_and_qkv0(m, A, false, stack, f, mask, nullptr, nullptr, h, w, false, precision, s);
    if (rc) return rc;
  }
  return run_blocks(m, A, L, am, false, h, w, out, nullptr, s);
}

// u8 planes (nvrec_recover_u8) or u16 depth planes (nvrec_recover_u16)
static int recover_planes(const nvrec_model* m, int32_t b, int32_t h, int32_t w,
                          const uint8_t* frames, int32_t n_slots, const int32_t* frame_index,
                          const uint8_t* mask_bits, uint8_t* out, void* ws, int64_t ws_bytes,
                          int32_t precision, void* stream, bool u16) {
  WorkspaceLayout L;
  int rc = common_checks(m, b, h, w, ws, ws_bytes, precision, &L);
  if (rc) return rc;
  if (m->D.p != 16)
    return fail(NVREC_E_UNSUPPORTED, "u8 recover path needs patch == mask block (16)");
  if (!frames || !frame_index || !mask_bits)
    return fail(NVREC_E_INVALID, "null pointer");
  if (n_slots < 1) return fail(NVREC_E_INVALID, "n_slots must be >= 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  nvrec::Act A = make_act(m, ws, L, b, h, w);
  const int am = attn_mode(m->D, precision);
  if (u16 && (m->D.c != 1 || am == 0 || !nvrec::embed_tc_supported(m->D) ||
              !m->W.tc.emb16 || !m->W.tc.emb16_3 || !m->W.tc.last3 || precise_simt() ||
              last_simt() || !nvrec::last_tc_supported(m->D, b)))
    return fail(NVREC_E_UNSUPPORTED, "u16 depth path needs a channels == 1 model inside the "
                "tensor-core envelope (dim 64, 2 heads, patch 16, <= 3 time slices)");
  const bool fast = am == 1;
  const int nbytes = (A.ns + 7) / 8;
  cudaError_t e;
  {
    ProfScope ps(NVREC_STAGE_MASKLIST, s);
    e = nvrec::launch_masklist(mask_bits, b, nbytes, A.ns, A.list, A.rank, A.count, s);
  }
  if (e != cudaSuccess) return cuda_fail(e, "masklist launch");
  if (am && nvrec::embed_tc_supported(m->D) && (am == 1 || !precise_simt())) {
    nvrec::EmbedTcArgs ea{};
    ea.x3 = am == 2;
    ea.u16 = u16;
    ea.D = m->D;
    ea.tcw = &m->W.tc;
    ea.emb_wmsum = m->W.emb_wmsum; ea.emb_b = m->W.emb_b; ea.time_pos = m->W.time_pos;
    ea.ln_w = m->W.blk[0].ln_s_w; ea.ln_b = m->W.blk[0].ln_s_b; ea.qkv_b = m->W.blk[0].qkv_s_b;
    ea.frames = frames; ea.frame_index = frame_index;
    ea.n_slots = n_slots;
    ea.rank = A.rank;
    ea.qrank = m->D.layers == 1 ? A.rank : nullptr;
    ea.x = A.x; ea.qh = A.qh; ea.kh = A.kh; ea.vth = A.vth;
    // the embedding output goes to block 0's tensor-core tail in fp16 (half
    // the traffic of that one hand-off; the tail keeps the residual in fp32)
    A.x_half = fast && !u16 && A.xh && m->D.layers > 1 && nvrec::token_tc_supported(m->D) &&
               m->W.tc.blk[0];
    ea.xh = A.x_half ? A.xh : nullptr;
    ea.b = b; ea.h = h; ea.w = w; ea.nh = A.nh; ea.nw = A.nw; ea.ns = A.ns; ea.ns_pad = A.ns_pad;
    cudaError_t e2;
    {
      ProfScope ps(NVREC_STAGE_EMBED, s);
      e2 = nvrec::launch_embed_tc(ea, s);
    }
    if (e2 != cudaSuccess) return cuda_fail(e2, "embed_tc launch");
  } else {
    rc = embed_and_qkv0(m, A, true, nullptr, 0, nullptr, frames, frame_index, h, w, true,
                        precision, s);
    if (rc) return rc;
  }
  const size_t frame_bytes = size_t(h) * w * m->D.c * (u16 ? 2 : 1);
  if (!out) {
    // in place: the corrupted plane already holds every trusted pixel; only
    // the masked patches are written (after the embedding read the stack)
    InPlace ip;
    ip.frames = const_cast<uint8_t*>(frames);
    ip.frame_index = frame_index;
    return run_blocks(m, A, L, am, true, h, w, nullptr, nullptr, s, ip, u16);
  }
  // the merge base (corrupted plane) is copied only after the embedding has
  // read every stacked frame, so `out` may alias a reference slot (a ring
  // that takes the recovered plane in place of its oldest reference)
  {
    ProfScope ps(NVREC_STAGE_COPY, s);
    e = nvrec::launch_copy_plane(frames, frame_index, m->D.F, frame_bytes, out, b, s);
  }
  if (e != cudaSuccess) return cuda_fail(e, "copy launch");
  return run_blocks(m, A, L, am, true, h, w, nullptr, out, s, {}, u16);
}

int nvrec_recover_u8(const nvrec_model* m, int32_t b, int32_t h, int32_t w,
                     const uint8_t* frames, int32_t n_slots, const int32_t* frame_index,
                     const uint8_t* mask_bits, uint8_t* out, void* ws, int64_t ws_bytes,
                     int32_t precision, void* stream) {
  return recover_planes(m, b, h, w, frames, n_slots, frame_index, mask_bits, out, ws, ws_bytes,
                        precision, stream, false);
}

int nvrec_recover_u16(const nvrec_model* m, int32_t b, int32_t h, int32_t w,
                      const uint16_t* frames, int32_t n_slots, const int32_t* frame_index,
                      const uint8_t* mask_bits, uint16_t* out, void* ws, int64_t ws_bytes,
                      int32_t precision, void* stream) {
  return recover_planes(m, b, h, w, reinterpret_cast<const uint8_t*>(frames), n_slots,
                        frame_index, mask_bits, reinterpret_cast<uint8_t*>(out), ws, ws_bytes,
                        precision, stream, true);
}

int nvrec_loss_mask(const nvrec_lossmask_job* jobs, int32_t n_jobs, void* stream) {
  if (n_jobs < 0 || (n_jobs > 0 && !jobs)) return fail(NVREC_E_INVALID, "bad job array");
  cudaError_t e;
  {
    ProfScope ps(NVREC_STAGE_LOSSMASK, static_cast<cudaStream_t>(stream));
    e = nvrec::launch_lossmask(jobs, n_jobs, static_cast<cudaStream_t>(stream));
  }
  if (e != cudaSuccess) return cuda_fail(e, "loss-mask launch");
  return 0;
}

int nvrec_decode(const nvrec_decode_job* jobs, int32_t n_jobs, int32_t max_blocks, void* stream) {
  if (n_jobs < 0 || (n_jobs > 0 && !jobs)) return fail(NVREC_E_INVALID, "bad job array");
  if (max_blocks < 1) return fail(NVREC_E_INVALID, "max_blocks must be >= 1");
  cudaError_t e;
  {
    ProfScope ps(NVREC_STAGE_DECODE, static_cast<cudaStream_t>(stream));
    ps.kernels(4);
    e = nvrec::launch_decode(jobs, n_jobs, max_blocks, static_cast<cudaStream_t>(stream));
  }
  if (e != cudaSuccess) return cuda_fail(e, "decode launch");
  return 0;
}

int nvrec_rs_plan(int32_t n, int32_t r, const uint8_t* present, uint8_t* coef,
                  int32_t* sources, int32_t* missing, int32_t* m_out) {
  if (n < 1 || r < 0 || n + r > 255) return fail(NVREC_E_INVALID, "need n >= 1, r >= 0, n+r <= 255");
  if (!present || !coef || !sources || !missing || !m_out)
    return fail(NVREC_E_INVALID, "null pointer");
  int have = 0;
  for (int i = 0; i < n + r; ++i) have += present[i] != 0;
  if (have < n) return fail(NVREC_E_INVALID, "only %d of %d required shards present", have, n);
  const int rc = nvrec::rs_plan_host(n, r, present, coef, sources, missing, m_out);
  if (rc == -2) return fail(NVREC_E_INVALID, "singular matrix");
  if (rc) return fail(NVREC_E_INVALID, "rs plan failed");
  return 0;
}

int nvrec_rs_reconstruct(const nvrec_rs_job* jobs, int32_t n_jobs, int32_t max_shard_len,
                         int32_t max_coef, int32_t aligned4, void* stream) {
  if (n_jobs < 0 || (n_jobs > 0 && !jobs)) return fail(NVREC_E_INVALID, "bad job array");
  if (max_shard_len < 1 || max_coef < 0 || max_coef > 255 * 255)
    return fail(NVREC_E_INVALID, "bad shard_len / coefficient bound");
  cudaError_t e;
  {
    ProfScope ps(NVREC_STAGE_RS, static_cast<cudaStream_t>(stream));
    e = nvrec::launch_rs(jobs, n_jobs, max_shard_len, max_coef, aligned4 != 0,
                         static_cast<cudaStream_t>(stream));
  }
  if (e != cudaSuccess) return cuda_fail(e, "rs launch");
  return 0;
}

int64_t nvrec_baseline_workspace_bytes(int32_t b, int32_t h, int32_t w, int32_t c) {
  if (b < 1 || h < 16 || w < 16 || h % 16 || w % 16 || (c != 1 && c != 3))
    return fail(NVREC_E_INVALID, "bad baseline shape");
  const size_t ns = size_t(h / 16) * (w / 16);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  return int64_t(al(b * ns * 4) * 2 + al(b * 4) + al(b * 16) + al(size_t(b) * h * w * c));
}

int nvrec_baseline_u8(int32_t depth, int32_t b, int32_t h, int32_t w, int32_t c,
                      const uint8_t* planes, const uint8_t* refs, const uint8_t* mask_bits,
                      uint8_t* out, void* ws, int64_t ws_bytes, void* stream) {
  const int64_t need = nvrec_baseline_workspace_bytes(b, h, w, c);
  if (need < 0) return int(need);
  if (depth && c != 1) return fail(NVREC_E_INVALID, "depth baseline needs c == 1");
  if (!planes || !refs || !mask_bits || !out) return fail(NVREC_E_INVALID, "null pointer");
  if (!ws || ws_bytes < need) return fail(NVREC_E_WORKSPACE, "baseline workspace too small");
  const size_t ns = size_t(h / 16) * (w / 16);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  char* p = static_cast<char*>(ws);
  int* list = reinterpret_cast<int*>(p); p += al(b * ns * 4);
  int* rank = reinterpret_cast<int*>(p); p += al(b * ns * 4);
  int* count = reinterpret_cast<int*>(p); p += al(b * 4);
  int* bbox = reinterpret_cast<int*>(p); p += al(b * 16);
  uint8_t* base = reinterpret_cast<uint8_t*>(p);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  {
    ProfScope ps(NVREC_STAGE_BASELINE, s);
    ps.kernels(depth ? 3 : 1);
    e = nvrec::launch_baseline(depth, b, h, w, c, planes, refs, mask_bits, out, base, list,
                               rank, count, bbox, s);
  }
  if (e != cudaSuccess) return cuda_fail(e, "baseline launch");
  return 0;
}

#ifdef NVREC_TRACE
// trace build only (not in include/nvrec_b200.h): phase timestamps of one CTA
int nvrec_debug_attn_trace(unsigned long long* host, int n) { return nvrec::attn_trace(host, n); }
int nvrec_debug_last_trace(unsigned long long* host, int n) { return nvrec::last_trace(host, n); }
int nvrec_debug_token_x3_trace(unsigned long long* host, int n) { return nvrec::token_x3_trace(host, n); }
int nvrec_debug_embed_trace(unsigned long long* host, int n) { return nvrec::embed_trace(host, n); }
int nvrec_debug_token_tc_trace(unsigned long long* host, int n) { return nvrec::token_tc_trace(host, n); }
#endif

int64_t nvrec_attn_fixup_items(void) {
  const int64_t n = nvrec::attn_fixup_items();
  if (n < 0) return fail(NVREC_E_CUDA, "reading the fix-up counter failed");
  return n;
}

int nvrec_profile_begin(void) {
  if (g_prof_pool.empty()) {
    g_prof_pool.resize(kProfMax);
    for (auto& r : g_prof_pool) {
      CK(cudaEventCreate(&r.a), "cudaEventCreate");
      CK(cudaEventCreate(&r.b), "cudaEventCreate");
    }
  }
  g_prof_n = 0;
  g_prof = true;
  return 0;
}

int nvrec_profile_end(float* ms_per_stage, int32_t* launches_per_stage, int32_t n_stages) {
  g_prof = false;
  for (int i = 0; i < n_stages; ++i) { ms_per_stage[i] = 0.f; launches_per_stage[i] = 0; }
  for (int i = 0; i < g_prof_n; ++i) {
    ProfRec& r = g_prof_pool[i];
    CK(cudaEventSynchronize(r.b), "cudaEventSynchronize");
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, r.a, r.b), "cudaEventElapsedTime");
    if (r.kind >= 0 && r.kind < n_stages) {
      ms_per_stage[r.kind] += ms;
      launches_per_stage[r.kind] += r.kernels;
    }
  }
  int n = 0;
  for (int i = 0; i < g_prof_n; ++i) n += g_prof_pool[i].kernels;
  g_prof_n = 0;
  return n;
}

}  // extern "C"
