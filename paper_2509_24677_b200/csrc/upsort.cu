// k2s2 transposed (up) conv rows grouped by parity class.
//
// In the up table (kmap_up_kernel) every fine row has exactly ONE valid tap:
// its own parity j = 4(x&1) + 2(y&1) + (z&1), pointing at the parent.  A
// 128-row tile of fine rows in C-order mixes all 8 parities, so a gather-GEMM
// over it runs all 8 weight slices on mostly-zero rows (8x the useful MMA
// work).  Here the fine rows are stably sorted by parity class, each class
// padded to a multiple of 128 rows, so every tile has a single class: the
// conv (fpvs_spconv_tc_scatter) runs one weight slice per tile and scatters
// the rows back to their C-order positions (perm).  Deterministic: positions
// come from exact prefix counts, not atomics.
#include "common.cuh"

namespace fpvs {
namespace upsort {

constexpr int CH = 256;  // rows per chunk = threads per block
constexpr int kMaxJobs = 4;

struct Job {
  const int* up;
  const int* n;
  int cap;
  int* table;
  int* perm;
  uint32_t* masks;
  int* n_pad;
  int* counts;  // [ceil(cap / CH)][8] per-chunk class counts (workspace)
};
struct Jobs {
  Job j[kMaxJobs];
  int count;
};

__device__ __forceinline__ int chunks_of(const Job& q) { return (min(*q.n, q.cap) + CH - 1) / CH; }

// class (valid tap) and parent of fine row r
__device__ __forceinline__ int row_class(const int* up, long long r, int& parent) {
  const int4 a = __ldg(reinterpret_cast<const int4*>(up + r * 8));
  const int4 b = __ldg(reinterpret_cast<const int4*>(up + r * 8) + 1);
  const int v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  int c = -1;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (v[i] >= 0 && c < 0) {
      c = i;
      parent = v[i];
    }
  return c;
}

__global__ void __launch_bounds__(CH) count_kernel(const Jobs J) {
  __shared__ int s_cnt[8];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int l = 0; l < J.count; ++l) {
    const Job q = J.j[l];
    const int n = min(*q.n, q.cap);
    const int nch = (n + CH - 1) / CH;
    for (int ch = blockIdx.x; ch < nch; ch += gridDim.x) {
      if (tid < 8) s_cnt[tid] = 0;
      __syncthreads();
      const long long r = (long long)ch * CH + tid;
      int parent = -1;
      const int c = r < n ? row_class(q.up, r, parent) : -1;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t m = __ballot_sync(~0u, c == k);
        if (lane == 0 && m) atomicAdd(&s_cnt[k], __popc(m));
      }
      __syncthreads();
      if (tid < 8) q.counts[ch * 8 + tid] = s_cnt[tid];
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(CH) place_kernel(const Jobs J) {
  __shared__ int s_tot[8], s_pre[8], s_base[9];
  __shared__ int s_red[8][8];
  __shared__ int s_warp[8][8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int l = 0; l < J.count; ++l) {
    const Job q = J.j[l];
    const int n = min(*q.n, q.cap);
    const int nch = (n + CH - 1) / CH;
    // class totals and padded class bases (every block, identical)
    {
      int acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int ch = tid; ch < nch; ch += CH)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] += q.counts[ch * 8 + k];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        for (int o = 16; o; o >>= 1) acc[k] += __shfl_xor_sync(~0u, acc[k], o);
        if (lane == 0) s_red[warp][k] = acc[k];
      }
      __syncthreads();
      if (tid < 8) {
        int t = 0;
        for (int w = 0; w < 8; ++w) t += s_red[w][tid];
        s_tot[tid] = t;
      }
      __syncthreads();
      if (tid == 0) {
        int b = 0;
        for (int k = 0; k < 8; ++k) {
          s_base[k] = b;
          b += (s_tot[k] + 127) / 128 * 128;
        }
        s_base[8] = b;
      }
      __syncthreads();
    }
    const int npad = s_base[8];
    if (blockIdx.x == 0) {
      // tile classes, padding slots, padded count
      for (int t = tid; t < npad / 128; t += CH) {
        int k = 0;
        while (t * 128 >= s_base[k + 1]) ++k;
        q.masks[t] = 1u << k;
      }
      for (int k = 0; k < 8; ++k) {
        for (int s = s_base[k] + s_tot[k] + tid; s < s_base[k + 1]; s += CH) {
          q.perm[s] = -1;
          reinterpret_cast<int4*>(q.table + (long long)s * 8)[0] = make_int4(-1, -1, -1, -1);
          reinterpret_cast<int4*>(q.table + (long long)s * 8)[1] = make_int4(-1, -1, -1, -1);
        }
      }
      if (tid == 0) *q.n_pad = npad;
    }
    for (int ch = blockIdx.x; ch < nch; ch += gridDim.x) {
      // rows of this class in earlier chunks
      {
        int acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int c2 = tid; c2 < ch; c2 += CH)
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[k] += q.counts[c2 * 8 + k];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          for (int o = 16; o; o >>= 1) acc[k] += __shfl_xor_sync(~0u, acc[k], o);
          if (lane == 0) s_red[warp][k] = acc[k];
        }
      }
      const long long r = (long long)ch * CH + tid;
      int parent = -1;
      const int c = r < n ? row_class(q.up, r, parent) : -1;
      int rank = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t m = __ballot_sync(~0u, c == k);
        if (c == k) rank = __popc(m & ((1u << lane) - 1u));
        if (lane == 0) s_warp[warp][k] = __popc(m);
      }
      __syncthreads();
      if (tid < 8) {
        int t = 0;
        for (int w = 0; w < 8; ++w) t += s_red[w][tid];
        s_pre[tid] = t;
      }
      __syncthreads();
      if (c >= 0) {
        int before = 0;
        for (int w = 0; w < warp; ++w) before += s_warp[w][c];
        const int pos = s_base[c] + s_pre[c] + before + rank;
        q.perm[pos] = (int)r;
        int v[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k == c) v[k] = parent;
        reinterpret_cast<int4*>(q.table + (long long)pos * 8)[0] = make_int4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<int4*>(q.table + (long long)pos * 8)[1] = make_int4(v[4], v[5], v[6], v[7]);
      }
      __syncthreads();
    }
    __syncthreads();
  }
}

}  // namespace upsort
}  // namespace fpvs

using namespace fpvs;

extern "C" int fpvs_up_sort_cap(int cap_fine) {
  if (cap_fine < 0) return -1;
  return (cap_fine + 8 * 127 + 127) / 128 * 128;
}

extern "C" size_t fpvs_up_sort_workspace_size(int cap_fine) {
  if (cap_fine < 1) return 256;
  return (size_t)((cap_fine + upsort::CH - 1) / upsort::CH) * 8 * sizeof(int) + 256;
}

extern "C" int fpvs_up_sort_multi(const fpvs_up_sort_job* jobs, int njobs, void* stream) {
  FPVS_CHECK_ARG(jobs && njobs >= 1 && njobs <= upsort::kMaxJobs, "1..4 up-sort jobs");
  upsort::Jobs J{};
  J.count = njobs;
  long long chunks = 0;
  for (int i = 0; i < njobs; ++i) {
    const fpvs_up_sort_job& q = jobs[i];
    FPVS_CHECK_ARG(q.up && q.n_fine_dev && q.sorted_table && q.perm && q.masks && q.n_pad_dev && q.workspace,
                   "null pointer in up-sort job %d", i);
    FPVS_CHECK_ARG(q.cap_fine >= 0, "negative capacity");
    FPVS_CHECK_ARG(q.workspace_bytes >= fpvs_up_sort_workspace_size(q.cap_fine), "up-sort workspace too small");
    J.j[i] = upsort::Job{q.up, q.n_fine_dev, q.cap_fine, q.sorted_table, q.perm, q.masks, q.n_pad_dev,
                         (int*)q.workspace};
    const long long c = (q.cap_fine + upsort::CH - 1) / upsort::CH;
    if (c > chunks) chunks = c;
  }
  const int grid = (int)(chunks < 2 * kNumSMs ? (chunks > 0 ? chunks : 1) : 2 * kNumSMs);
  cudaStream_t s = as_stream(stream);
  upsort::count_kernel<<<grid, upsort::CH, 0, s>>>(J);
  upsort::place_kernel<<<grid, upsort::CH, 0, s>>>(J);
  FPVS_CHECK_LAUNCH("fpvs_up_sort");
  return FPVS_OK;
}

extern "C" int fpvs_up_sort(const int32_t* up, const int32_t* n_fine_dev, int cap_fine, int32_t* sorted_table,
                            int32_t* perm, uint32_t* masks, int32_t* n_pad_dev, void* workspace,
                            size_t workspace_bytes, void* stream) {
  fpvs_up_sort_job j{up, n_fine_dev, cap_fine, sorted_table, perm, masks, n_pad_dev, workspace, workspace_bytes};
  return fpvs_up_sort_multi(&j, 1, stream);
}
