// k_lossmask.cu -- integer loss-mask construction and masked-patch lists.
//
// lossmask_kernel: one CTA per P-frame job runs lm::lossmask_job
// (lossmask.cuh), the bit-exact restatement of the reference receiver +
// codec mask path (receiver.py:224-237, codec.py:172-201,250-281,318-320,
// recovery.py:221).
//
// masklist_kernel turns a wire bitset into the ascending list of masked
// patches of one stream (+ inverse rank table), which the pruned last block
// and the head consume (server.py:196 discards every unmasked prediction).
#include "launch.cuh"
#include "lossmask.cuh"

namespace nvrec {

namespace {
constexpr int kMaskThreads = 1024;   // one bitmap byte per thread up to 8192 blocks (1080p)
using lm::block_exclusive_scan;
}  // namespace

constexpr int kStage = 40 * 1024;   // header + received flags staged in smem

__global__ void __launch_bounds__(kMaskThreads)
lossmask_kernel(const nvrec_lossmask_job* __restrict__ jobs) {
  pdl_entry();
  __shared__ int sh_scan[32];
  __shared__ int sh_flagged;
  extern __shared__ uint8_t stage[];
  const nvrec_lossmask_job job = jobs[blockIdx.x];
  lm::lossmask_job(job, nullptr, nullptr, sh_scan, &sh_flagged, stage, kStage);
}

// Wire bitset (b, nbytes) -> ascending masked-patch list, rank table, count.
__global__ void __launch_bounds__(kMaskThreads)
masklist_kernel(const uint8_t* __restrict__ bits, int nbytes, int ns,
                int* __restrict__ list, int* __restrict__ rank, int* __restrict__ count) {
  pdl_entry();
  __shared__ int sh_scan[32];
  const int b = blockIdx.x;
  const uint8_t* mb = bits + size_t(b) * nbytes;
  int* lst = list + size_t(b) * ns;
  int* rk = rank + size_t(b) * ns;
  int base = 0;
  for (int byte0 = 0; byte0 < nbytes; byte0 += blockDim.x) {
    int t = byte0 + threadIdx.x;
    uint32_t v = 0;
    if (t < nbytes) {
      v = mb[t];
      int valid = ns - 8 * t;
      if (valid < 8) v &= valid > 0 ? (0xFFu << (8 - valid)) & 0xFFu : 0u;
    }
    int tot;
    int r = base + block_exclusive_scan(__popc(v), &tot, sh_scan);
    base += tot;
    for (int bit = 0; bit < 8; ++bit) {
      int s = 8 * t + bit;
      if (t >= nbytes || s >= ns) break;
      if (v & (0x80u >> bit)) { lst[r] = s; rk[s] = r; ++r; }
      else rk[s] = -1;
    }
  }
  if (threadIdx.x == 0) count[b] = base;
}

// ---------------------------------------------------------------------------
cudaError_t launch_lossmask(const nvrec_lossmask_job* jobs, int n_jobs, cudaStream_t s) {
  if (n_jobs <= 0) return cudaSuccess;
  launch_pdl(lossmask_kernel, n_jobs, kMaskThreads, kStage, s, jobs);
  return cudaGetLastError();
}

cudaError_t launch_masklist(const uint8_t* bits, int b, int nbytes, int ns, int* list,
                            int* rank, int* count, cudaStream_t s) {
  launch_pdl(masklist_kernel, b, kMaskThreads, 0, s, bits, nbytes, ns, list, rank, count);
  return cudaGetLastError();
}

}  // namespace nvrec
