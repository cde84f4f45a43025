// k_rs.cu -- Reed-Solomon erasure reconstruction of I-frames over GF(2^8)
// (SURVEY.md 8(f) rank 4), bit-exact with rgbdstream fec.rs_reconstruct
// (fec.py:144-163): field polynomial 0x11D (fec.py:19-41), systematic
// generator G = V * inv(V[:n]) with V the (n+r) x n Vandermonde matrix on
// the points 0..n+r-1 (fec.py:78-88).
//
// The reference inverts the n x n submatrix G[idx] of the first n present
// shards and multiplies all n rows.  The data rows of G[idx] are unit
// vectors, so the system reduces to the m missing data shards M and the m
// parity rows P in idx:  G[P,M] x_M = y_P ^ G[P,D] x_D.  The solution is
// unique (G is MDS), so x_M = A (y_P ^ G[P,D] x_D), A = inv(G[P,M]), gives
// the same bytes as the reference for any received shards.
//
// Host (nvrec_rs_plan, C++): inv(V[:n]) by Lagrange interpolation (O(n^2),
// cached per n), the m rows G[P,:], the m x m Gauss-Jordan inverse and the
// m x n decode coefficients over the n source shards.
// Device (rs_kernel): HBM-bound byte work.  One thread per 4-byte column of
// the shards; per source word the eight multiples x^k * w are formed once
// (packed xtime on 4 bytes) and every missing row XORs the multiples its
// coefficient selects (coefficients in shared memory, uniform branches).
#include <map>
#include <mutex>
#include <vector>

#include "launch.cuh"

namespace nvrec {

namespace {

// ---- GF(2^8) host arithmetic ------------------------------------------------------
struct Gf {
  uint8_t exp[512];
  int log[256];
  Gf() {
    int x = 1;
    for (int i = 0; i < 255; ++i) {
      exp[i] = uint8_t(x);
      log[x] = i;
      x <<= 1;
      if (x & 0x100) x ^= 0x11D;
    }
    for (int i = 255; i < 512; ++i) exp[i] = exp[i - 255];
    log[0] = 0;
  }
  uint8_t mul(uint8_t a, uint8_t b) const {
    return (a && b) ? exp[log[a] + log[b]] : 0;
  }
  uint8_t inv(uint8_t a) const { return exp[255 - log[a]]; }
};
const Gf& gf() {
  static Gf g;
  return g;
}

// inv(V[:n]) with V[i][j] = i^j (0^0 = 1): column i holds the coefficients
// of the Lagrange basis polynomial L_i(x) = prod_{k != i} (x - k) / (i - k).
std::vector<uint8_t> vandermonde_inverse(int n) {
  const Gf& g = gf();
  // master polynomial M(x) = prod_k (x + k), coefficients low -> high
  std::vector<uint8_t> M(n + 1, 0);
  M[0] = 1;
  for (int k = 0; k < n; ++k) {
    for (int d = k + 1; d >= 1; --d) M[d] = M[d - 1] ^ g.mul(M[d], uint8_t(k));
    M[0] = g.mul(M[0], uint8_t(k));
  }
  std::vector<uint8_t> inv(size_t(n) * n);
  std::vector<uint8_t> q(n);
  for (int i = 0; i < n; ++i) {
    // q(x) = M(x) / (x + i) (synthetic division), denominator = q(i)
    uint8_t carry = 0;
    for (int d = n; d >= 1; --d) {
      carry = M[d] ^ g.mul(carry, uint8_t(i));
      q[d - 1] = carry;
    }
    uint8_t den = 0, pw = 1;
    for (int d = 0; d < n; ++d) {
      den ^= g.mul(q[d], pw);
      pw = g.mul(pw, uint8_t(i));
    }
    const uint8_t s = g.inv(den);
    for (int d = 0; d < n; ++d) inv[size_t(d) * n + i] = g.mul(q[d], s);
  }
  return inv;
}

const std::vector<uint8_t>& cached_vinv(int n) {
  static std::mutex mu;
  static std::map<int, std::vector<uint8_t>> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(n);
  if (it == cache.end()) it = cache.emplace(n, vandermonde_inverse(n)).first;
  return it->second;
}

// Gauss-Jordan over GF(2^8); false if singular.
bool gf_invert(std::vector<uint8_t>& a, int m, std::vector<uint8_t>& out) {
  const Gf& g = gf();
  out.assign(size_t(m) * m, 0);
  for (int i = 0; i < m; ++i) out[size_t(i) * m + i] = 1;
  for (int col = 0; col < m; ++col) {
    int piv = col;
    while (piv < m && a[size_t(piv) * m + col] == 0) ++piv;
    if (piv == m) return false;
    if (piv != col)
      for (int k = 0; k < m; ++k) {
        std::swap(a[size_t(piv) * m + k], a[size_t(col) * m + k]);
        std::swap(out[size_t(piv) * m + k], out[size_t(col) * m + k]);
      }
    const uint8_t s = g.inv(a[size_t(col) * m + col]);
    for (int k = 0; k < m; ++k) {
      a[size_t(col) * m + k] = g.mul(a[size_t(col) * m + k], s);
      out[size_t(col) * m + k] = g.mul(out[size_t(col) * m + k], s);
    }
    for (int row = 0; row < m; ++row) {
      const uint8_t f = a[size_t(row) * m + col];
      if (row == col || !f) continue;
      for (int k = 0; k < m; ++k) {
        a[size_t(row) * m + k] ^= g.mul(f, a[size_t(col) * m + k]);
        out[size_t(row) * m + k] ^= g.mul(f, out[size_t(col) * m + k]);
      }
    }
  }
  return true;
}

// ---- device -------------------------------------------------------------------------
constexpr int kThreads = 128;
constexpr int kRowsPerPass = 16;
constexpr int kMaxCoef = 255 * 255;        // m x n coefficients (m <= r, n + r <= 255)

__device__ __forceinline__ uint32_t xtime4(uint32_t w) {
  return ((w & 0x7f7f7f7fu) << 1) ^ (((w >> 7) & 0x01010101u) * 0x1du);
}

template <bool kWord>
__global__ void __launch_bounds__(kThreads)
rs_kernel(const nvrec_rs_job* __restrict__ jobs) {
  pdl_entry();
  extern __shared__ uint8_t sh_coef[];
  const nvrec_rs_job& jb = jobs[blockIdx.y];
  const int n = jb.n, m = jb.m, L = jb.shard_len;
  if (m <= 0) return;
  const int units = kWord ? L / 4 : L;
  const int u = blockIdx.x * kThreads + threadIdx.x;
  if (blockIdx.x * kThreads >= units) return;
  for (int i = threadIdx.x; i < m * n; i += kThreads) sh_coef[i] = jb.coef[i];
  __syncthreads();
  if (u >= units) return;
  for (int r0 = 0; r0 < m; r0 += kRowsPerPass) {
    uint32_t acc[kRowsPerPass];
#pragma unroll
    for (int i = 0; i < kRowsPerPass; ++i) acc[i] = 0;
    for (int sidx = 0; sidx < n; ++sidx) {
      const int src = jb.sources[sidx];
      const uint8_t* row = src < n ? jb.data + size_t(src) * L
                                   : jb.parity + size_t(src - n) * L;
      uint32_t p[8];
      p[0] = kWord ? __ldg(reinterpret_cast<const uint32_t*>(row) + u) : uint32_t(row[u]);
#pragma unroll
      for (int k = 1; k < 8; ++k) p[k] = xtime4(p[k - 1]);
#pragma unroll
      for (int i = 0; i < kRowsPerPass; ++i) {
        if (r0 + i >= m) break;
        const uint32_t c = sh_coef[(r0 + i) * n + sidx];
        uint32_t a = acc[i];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (c & (1u << k)) a ^= p[k];
        acc[i] = a;
      }
    }
#pragma unroll
    for (int i = 0; i < kRowsPerPass; ++i) {
      if (r0 + i >= m) break;
      uint8_t* dst = jb.data + size_t(jb.missing[r0 + i]) * L;
      if (kWord) reinterpret_cast<uint32_t*>(dst)[u] = acc[i];
      else dst[u] = uint8_t(acc[i]);
    }
  }
}

}  // namespace

int rs_plan_host(int n, int r, const uint8_t* present, uint8_t* coef, int32_t* sources,
                 int32_t* missing, int32_t* m_out) {
  // first n present shards (fec.py:153)
  std::vector<int> idx;
  for (int i = 0; i < n + r && int(idx.size()) < n; ++i)
    if (present[i]) idx.push_back(i);
  if (int(idx.size()) < n) return -1;                         // UnrecoverableError
  std::vector<int> P, M;
  for (int i : idx)
    if (i >= n) P.push_back(i);
  for (int i = 0; i < n; ++i)
    if (!present[i]) M.push_back(i);
  const int m = int(M.size());
  *m_out = m;
  for (int s = 0; s < n; ++s) sources[s] = idx[s];
  for (int i = 0; i < m; ++i) missing[i] = M[i];
  if (m == 0) return 0;                                       // systematic fast path
  const Gf& g = gf();
  const std::vector<uint8_t>& vinv = cached_vinv(n);
  // G[p, :] = V[p, :] * inv(V[:n]) for the m parity rows in idx
  std::vector<uint8_t> GP(size_t(m) * n, 0), vrow(n);
  for (int a = 0; a < m; ++a) {
    uint8_t pw = 1;
    for (int j = 0; j < n; ++j) {
      vrow[j] = pw;
      pw = g.mul(pw, uint8_t(P[a]));
    }
    for (int k = 0; k < n; ++k) {
      if (!vrow[k]) continue;
      const uint8_t* vr = &vinv[size_t(k) * n];
      for (int j = 0; j < n; ++j) GP[size_t(a) * n + j] ^= g.mul(vrow[k], vr[j]);
    }
  }
  std::vector<uint8_t> sub(size_t(m) * m), A;
  for (int a = 0; a < m; ++a)
    for (int b = 0; b < m; ++b) sub[size_t(a) * m + b] = GP[size_t(a) * n + M[b]];
  if (!gf_invert(sub, m, A)) return -2;                       // "singular matrix"
  // coefficient of source s for missing row i:
  //   parity source P[a]: A[i][a];  data source d: sum_a A[i][a] G[P[a]][d]
  for (int i = 0; i < m; ++i)
    for (int s = 0; s < n; ++s) {
      const int src = idx[s];
      uint8_t c = 0;
      if (src >= n) {
        int a = 0;
        while (P[a] != src) ++a;
        c = A[size_t(i) * m + a];
      } else {
        for (int a = 0; a < m; ++a) c ^= g.mul(A[size_t(i) * m + a], GP[size_t(a) * n + src]);
      }
      coef[size_t(i) * n + s] = c;
    }
  return 0;
}

cudaError_t launch_rs(const nvrec_rs_job* jobs, int n_jobs, int max_shard_len, int max_coef,
                      bool word, cudaStream_t s) {
  if (n_jobs <= 0 || max_coef <= 0) return cudaSuccess;
  if (max_coef > kMaxCoef) return cudaErrorInvalidValue;
  const int units = word ? (max_shard_len + 3) / 4 : max_shard_len;
  dim3 grid((units + kThreads - 1) / kThreads, n_jobs);
  const size_t smem = (size_t(max_coef) + 15) & ~size_t(15);
  if (cudaError_t e = smem_optin(rs_kernel<true>, kMaxCoef + 16)) return e;
  if (cudaError_t e = smem_optin(rs_kernel<false>, kMaxCoef + 16)) return e;
  if (word) launch_pdl(rs_kernel<true>, grid, kThreads, smem, s, jobs);
  else launch_pdl(rs_kernel<false>, grid, kThreads, smem, s, jobs);
  return cudaGetLastError();
}

}  // namespace nvrec
