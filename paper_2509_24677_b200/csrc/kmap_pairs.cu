// (2) Per-offset pair lists of a kernel map (SURVEY.md §8(a) row KM).
//
// From a neighbour table nbr[i][j] (row index or -1; K offsets), the pair
// list of offset j is every (in = nbr[i][j], out = i) with in >= 0, sorted
// by out, and pair_off is the exclusive prefix of the list lengths over j —
// the canonical form SURVEY.md pins for the gather-GEMM-scatter formulation
// (the reference builds the same pairs implicitly in the 27 slice copies of
// neural.py:187-199).  The convs of this library read the table directly
// (output-stationary tiles); the lists are for callers that want the
// scatter form (spconv-style per-offset GEMMs) and for the kernel-map tests.
//
// Three launches, deterministic: (1) per (1024-row block, offset) counts,
// (2) one CTA scans them into per-block bases and pair_off, (3) per (block,
// offset) an ordered compaction (warp ballots + a CTA scan over 4 x 256 rows)
// writes the pairs.
#include "common.cuh"

namespace fpvs {
namespace kp {

constexpr int ROWS = 1024;
constexpr int THREADS = 256;

__global__ void __launch_bounds__(THREADS) count_kernel(const int32_t* __restrict__ nbr, int K,
                                                        const int32_t* n_dev, int cap, int32_t* __restrict__ counts) {
  const int b = blockIdx.x, j = blockIdx.y;
  const int n = min(*n_dev, cap);
  int c = 0;
  for (int k = 0; k < ROWS / THREADS; ++k) {
    const int r = b * ROWS + k * THREADS + threadIdx.x;
    c += __syncthreads_count(r < n && __ldg(nbr + (long long)r * K + j) >= 0);
  }
  if (threadIdx.x == 0) counts[(long long)b * K + j] = c;
}

// base[b][j] = pair_off[j] + sum_{b' < b} counts[b'][j]; pair_off[K] = total
__global__ void __launch_bounds__(1024) scan_kernel(const int32_t* __restrict__ counts, int nb, int K,
                                                    long long* __restrict__ base, int64_t* __restrict__ pair_off) {
  __shared__ long long tot[32];
  // per offset: serial over blocks in chunks, one warp per offset
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = w; j < K; j += 32) {
    long long run = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int b = b0 + lane;
      const long long v = b < nb ? counts[(long long)b * K + j] : 0;
      long long incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (b < nb) base[(long long)b * K + j] = run + incl - v;  // offset-local for now
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) tot[j] = run;
  }
  __syncthreads();
  __shared__ long long off[33];
  if (threadIdx.x == 0) {
    long long o = 0;
    for (int j = 0; j < K; ++j) {
      off[j] = o;
      pair_off[j] = o;
      o += tot[j];
    }
    pair_off[K] = o;
  }
  __syncthreads();
  for (long long t = threadIdx.x; t < (long long)nb * K; t += blockDim.x) base[t] += off[t % K];
}

__global__ void __launch_bounds__(THREADS) write_kernel(const int32_t* __restrict__ nbr, int K, const int32_t* n_dev,
                                                        int cap, const long long* __restrict__ base,
                                                        int32_t* __restrict__ pin, int32_t* __restrict__ pout,
                                                        long long cap_pairs) {
  __shared__ int wsum[THREADS / 32];
  const int b = blockIdx.x, j = blockIdx.y;
  const int n = min(*n_dev, cap);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long pos = base[(long long)b * K + j];
  for (int k = 0; k < ROWS / THREADS; ++k) {
    const int r = b * ROWS + k * THREADS + threadIdx.x;
    const int v = r < n ? __ldg(nbr + (long long)r * K + j) : -1;
    const unsigned m = __ballot_sync(0xffffffffu, v >= 0);
    if (lane == 0) wsum[w] = __popc(m);
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int i = 0; i < THREADS / 32; ++i) {
      before += i < w ? wsum[i] : 0;
      total += wsum[i];
    }
    const long long at = pos + before + __popc(m & ((1u << lane) - 1u));
    if (v >= 0 && at < cap_pairs) {
      pin[at] = v;
      pout[at] = r;
    }
    pos += total;
    __syncthreads();
  }
}

inline size_t up256(size_t v) { return (v + 255) & ~(size_t)255; }

}  // namespace kp
}  // namespace fpvs

using namespace fpvs;

extern "C" size_t fpvs_kmap_pairs_workspace_size(int K, int cap) {
  if (K < 1 || K > 32 || cap < 1) return 0;
  const long long nb = (cap + kp::ROWS - 1) / kp::ROWS;
  return kp::up256((size_t)nb * K * 4) + kp::up256((size_t)nb * K * 8);
}

extern "C" int fpvs_kmap_pairs(const int32_t* nbr, int K, const int32_t* n_dev, int cap, int32_t* pair_in,
                               int32_t* pair_out, int64_t* pair_off, long long cap_pairs, void* workspace,
                               size_t workspace_bytes, void* stream) {
  FPVS_CHECK_ARG(nbr && n_dev && pair_off && workspace, "null pointer");
  FPVS_CHECK_ARG(K >= 1 && K <= 32, "K must lie in [1, 32]");
  FPVS_CHECK_ARG(cap_pairs >= 0 && (cap_pairs == 0 || (pair_in && pair_out)), "bad pair buffers");
  const size_t need = fpvs_kmap_pairs_workspace_size(K, cap);
  FPVS_CHECK_ARG(workspace_bytes >= need, "workspace too small: need %zu bytes", need);
  cudaStream_t s = as_stream(stream);
  const int nb = (cap + kp::ROWS - 1) / kp::ROWS;
  int32_t* counts = static_cast<int32_t*>(workspace);
  long long* base = reinterpret_cast<long long*>(static_cast<uint8_t*>(workspace) + kp::up256((size_t)nb * K * 4));
  kp::count_kernel<<<dim3(nb, K), kp::THREADS, 0, s>>>(nbr, K, n_dev, cap, counts);
  kp::scan_kernel<<<1, 1024, 0, s>>>(counts, nb, K, base, pair_off);
  kp::write_kernel<<<dim3(nb, K), kp::THREADS, 0, s>>>(nbr, K, n_dev, cap, base, pair_in, pair_out, cap_pairs);
  FPVS_CHECK_LAUNCH("fpvs_kmap_pairs");
  return FPVS_OK;
}
