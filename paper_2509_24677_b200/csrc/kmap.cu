// (2) Sparse-convolution kernel maps: active-set compaction, submanifold
// 3x3x3 neighbour tables, k2s2 down/up maps, and an open-addressing GPU hash.
//
// Canonical form (SURVEY.md §8(a) row KM, pinned bit-exact by the oracle):
// active cells in C-order of (b, x, y, z) (= np.nonzero order), row = rank,
// nbr[i][j] = row(coords[i] + o_j) or -1 with o_j = (a-1, b-1, c-1),
// j = 9a + 3b + c — the tap order of the reference im2col
// (pkg/src/froxelpvs/neural.py:187-199).
//
// Two lookups produce the same tables: a direct-mapped int32 index volume
// (the perfect hash for bounded froxel grids: 1 MB at 64^3 cells) and an
// open-addressing hash with 8-lane cooperative probing for unbounded grids.
// All kernels are integer/HBM-bound, persistent grid-stride loops that read
// the active count from device memory (no host round trip).
#include "common.cuh"

namespace fpvs {

constexpr int kScanThreads = 256;
constexpr int kScanPer = 16;                              // cells per thread (one 16-byte load)
constexpr int kScanCells = kScanThreads * kScanPer;       // cells per tile
constexpr unsigned kFlagAgg = 1u << 30, kFlagPrefix = 2u << 30, kValMask = (1u << 30) - 1u;

__device__ __forceinline__ long long lin4(int b, int x, int y, int z, int X, int Y, int Z) {
  return (((long long)b * X + x) * Y + y) * Z + z;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Single-pass stream compaction (decoupled look-back): each tile of 4096
// cells takes a dynamic tile id, block-scans its 16-cells-per-thread counts,
// publishes its aggregate, resolves its exclusive prefix from predecessors,
// then writes index_vol (rank or -1, 64 B per thread, coalesced) and the
// C-order coordinates of its active cells.
__global__ void __launch_bounds__(kScanThreads) compact_kernel(
    const uint8_t* __restrict__ act, long long ncell, int X, int Y, int Z, int4* __restrict__ coords,
    int* __restrict__ index_vol, int cap, unsigned* __restrict__ status, int* __restrict__ tile_ctr,
    int* __restrict__ n_out, int ntiles) {
  __shared__ int s_tile, s_prefix;
  __shared__ int s_warp[kScanThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1);
  __syncthreads();
  const int tile = s_tile;
  const long long base = (long long)tile * kScanCells + (long long)tid * kScanPer;
  uint32_t f = 0;
  if (base + kScanPer <= ncell && ((reinterpret_cast<uintptr_t>(act + base) & 15) == 0)) {
    uint4 v = *reinterpret_cast<const uint4*>(act + base);
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 16; ++i) f |= (((w[i >> 2] >> ((i & 3) * 8)) & 0xffu) ? 1u : 0u) << i;
  } else {
    for (int i = 0; i < kScanPer; ++i)
      if (base + i < ncell && act[base + i]) f |= 1u << i;
  }
  const int cnt = __popc(f);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int w = lane < kScanThreads / 32 ? s_warp[lane] : 0, wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < kScanThreads / 32) s_warp[lane] = wi - w;
    if (lane == kScanThreads / 32 - 1) {
      const unsigned agg = (unsigned)wi;
      unsigned prefix = 0;
      if (tile == 0) {
        st_release(status, kFlagPrefix | agg);
      } else {
        st_release(status + tile, kFlagAgg | agg);
        for (int t = tile - 1; t >= 0;) {
          unsigned v = ld_acquire(status + t);
          if (!(v & (kFlagAgg | kFlagPrefix))) continue;  // predecessor not published yet
          prefix += v & kValMask;
          if (v & kFlagPrefix) break;
          --t;
        }
        st_release(status + tile, kFlagPrefix | (prefix + agg));
      }
      s_prefix = (int)prefix;
      if (tile == ntiles - 1) *n_out = (int)(prefix + agg);
    }
  }
  __syncthreads();
  int rank = s_prefix + s_warp[wid] + incl - cnt;
  int rows[kScanPer];
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    const bool a = (f >> i) & 1u;
    rows[i] = (a && rank < cap) ? rank : -1;
    rank += a ? 1 : 0;
  }
  if (base + kScanPer <= ncell && ((reinterpret_cast<uintptr_t>(index_vol + base) & 15) == 0)) {
    int4* dst = reinterpret_cast<int4*>(index_vol + base);
#pragma unroll
    for (int q = 0; q < 4; ++q) dst[q] = make_int4(rows[4 * q], rows[4 * q + 1], rows[4 * q + 2], rows[4 * q + 3]);
  } else {
    for (int i = 0; i < kScanPer; ++i)
      if (base + i < ncell) index_vol[base + i] = rows[i];
  }
  if (f) {
#pragma unroll
    for (int i = 0; i < kScanPer; ++i) {
      if (rows[i] < 0) continue;
      long long r = base + i;
      int z = r % Z; r /= Z;
      int y = r % Y; r /= Y;
      int x = r % X;
      coords[rows[i]] = make_int4((int)(r / X), x, y, z);
    }
  }
}

__global__ void kmap_subm_kernel(const int4* __restrict__ coords, const int* __restrict__ n_dev, int cap,
                                 const int* __restrict__ index_vol, int X, int Y, int Z,
                                 int* __restrict__ nbr) {
  const int n = min(*n_dev, cap);
  const long long total = (long long)n * 27;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int j = t % 27;
    int4 c = coords[t / 27];
    int x = c.y + j / 9 - 1, y = c.z + (j / 3) % 3 - 1, z = c.w + j % 3 - 1;
    int r = -1;
    if (x >= 0 && x < X && y >= 0 && y < Y && z >= 0 && z < Z) r = __ldg(index_vol + lin4(c.x, x, y, z, X, Y, Z));
    nbr[t] = r;
  }
}

// general odd kernel size k (neural.py:187-199 with k^3 taps): offset
// j = (a*k + b)*k + c reads (x + a - p, y + b - p, z + c - p), p = k/2
__global__ void kmap_subm_k_kernel(const int4* __restrict__ coords, const int* __restrict__ n_dev, int cap,
                                   const int* __restrict__ index_vol, int X, int Y, int Z, int k,
                                   int* __restrict__ nbr) {
  const int n = min(*n_dev, cap);
  const int K = k * k * k, pad = k / 2;
  const long long total = (long long)n * K;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(t % K);
    const int4 c = coords[t / K];
    const int x = c.y + j / (k * k) - pad, y = c.z + (j / k) % k - pad, z = c.w + j % k - pad;
    int r = -1;
    if (x >= 0 && x < X && y >= 0 && y < Y && z >= 0 && z < Z) r = __ldg(index_vol + lin4(c.x, x, y, z, X, Y, Z));
    nbr[t] = r;
  }
}

__global__ void kmap_coarsen_kernel(const int4* __restrict__ coords, const int* __restrict__ n_dev, int cap,
                                    int X, int Y, int Z, uint8_t* __restrict__ coarse) {
  const int n = min(*n_dev, cap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int4 c = coords[i];
    coarse[lin4(c.x, c.y >> 1, c.z >> 1, c.w >> 1, X >> 1, Y >> 1, Z >> 1)] = 1;
  }
}

__global__ void kmap_down_kernel(const int4* __restrict__ cc, const int* __restrict__ n_dev, int cap,
                                 const int* __restrict__ fine_vol, int X, int Y, int Z, int* __restrict__ down) {
  const int n = min(*n_dev, cap);
  const long long total = (long long)n * 8;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int j = t & 7;
    int4 c = cc[t >> 3];
    down[t] = __ldg(fine_vol + lin4(c.x, 2 * c.y + (j >> 2), 2 * c.z + ((j >> 1) & 1), 2 * c.w + (j & 1), X, Y, Z));
  }
}

__global__ void kmap_up_kernel(const int4* __restrict__ fc, const int* __restrict__ n_dev, int cap,
                               const int* __restrict__ coarse_vol, int X, int Y, int Z, int* __restrict__ up) {
  const int n = min(*n_dev, cap);
  const long long total = (long long)n * 8;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int j = t & 7;
    int4 c = fc[t >> 3];
    int par = ((c.y & 1) << 2) | ((c.z & 1) << 1) | (c.w & 1);
    up[t] = (j == par) ? __ldg(coarse_vol + lin4(c.x, c.y >> 1, c.z >> 1, c.w >> 1, X >> 1, Y >> 1, Z >> 1)) : -1;
  }
}

// masks[t] = OR over rows [128t, 128t+128) (< n) of (1 << j) for every present
// table entry j: which kernel offsets a 128-row conv tile needs at all.
__global__ void __launch_bounds__(128) tile_masks_kernel(const int* __restrict__ table, int K,
                                                         const int* __restrict__ n_dev, int cap,
                                                         uint32_t* __restrict__ masks) {
  __shared__ uint32_t wm[4];
  const int n = min(*n_dev, cap);
  const int ntiles = (n + 127) / 128;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int row = t * 128 + threadIdx.x;
    uint32_t m = 0;
    if (row < n)
      for (int j = 0; j < K; ++j) m |= (__ldg(table + (long long)row * K + j) >= 0 ? 1u : 0u) << j;
    m = __reduce_or_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) masks[t] = wm[0] | wm[1] | wm[2] | wm[3];
    __syncthreads();
  }
}

// ---------------- open-addressing hash, 8-lane cooperative probing --------
constexpr int kGroup = 8;

__device__ __forceinline__ unsigned long long mix64(unsigned long long k) {
  k ^= k >> 33; k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

// Each query is owned by an 8-lane group; the group inspects 8 consecutive
// slots per step (one 64-byte run of keys), ballots for a hit or an empty slot.
__global__ void hash_build_kernel(const int4* __restrict__ coords, const int* __restrict__ n_dev, int cap,
                                  int X, int Y, int Z, unsigned long long* __restrict__ keys,
                                  int* __restrict__ vals, int hcap) {
  const int n = min(*n_dev, cap);
  const int lane = threadIdx.x & 31, g = lane / kGroup, gl = lane % kGroup;
  const unsigned gmask = 0xffu << (g * kGroup);
  const int groups_total = (gridDim.x * blockDim.x) / kGroup;
  int gid = (blockIdx.x * blockDim.x + threadIdx.x) / kGroup;
  const int iters = (n + groups_total - 1) / groups_total;
  for (int it = 0; it < iters; ++it, gid += groups_total) {
    bool live = gid < n;
    unsigned long long key = 0;
    if (live) {
      int4 c = coords[gid];
      key = (unsigned long long)lin4(c.x, c.y, c.z, c.w, X, Y, Z);
    }
    unsigned long long slot = live ? (mix64(key) & (unsigned long long)(hcap - 1)) & ~(unsigned long long)(kGroup - 1) : 0;
    bool done = !live;
    while (true) {
      if (!__any_sync(0xffffffffu, !done)) break;
      if (!done) {  // uniform across the 8-lane group
        unsigned long long s = (slot + gl) & (unsigned long long)(hcap - 1);
        unsigned long long cur = keys[s];
        unsigned empt = __ballot_sync(gmask, cur == ~0ULL) & gmask;
        bool placed = false;
        while (empt && !placed) {
          int leader = __ffs(empt) - 1;
          unsigned long long prev = 0;
          if (lane == leader) prev = atomicCAS(keys + s, ~0ULL, key);
          prev = __shfl_sync(gmask, prev, leader);
          if (prev == ~0ULL) {
            if (lane == leader) vals[s] = gid;
            placed = true;
          } else {
            empt &= ~(1u << leader);
          }
        }
        if (placed) done = true;
        else slot += kGroup;
      }
    }
  }
}

__device__ __forceinline__ int hash_find(const unsigned long long* __restrict__ keys, const int* __restrict__ vals,
                                         int hcap, unsigned long long key) {
  // same probe sequence as the build: linear from the 8-aligned home slot
  unsigned long long s = mix64(key) & (unsigned long long)(hcap - 1) & ~(unsigned long long)(kGroup - 1);
  for (int p = 0; p < hcap; ++p) {
    unsigned long long k = __ldg(keys + s);
    if (k == key) return __ldg(vals + s);
    if (k == ~0ULL) return -1;
    s = (s + 1) & (unsigned long long)(hcap - 1);
  }
  return -1;
}

// probe: one thread per (row, offset)
__global__ void kmap_subm_hash_kernel(const int4* __restrict__ coords, const int* __restrict__ n_dev, int cap,
                                      const unsigned long long* __restrict__ keys, const int* __restrict__ vals,
                                      int hcap, int X, int Y, int Z, int* __restrict__ nbr) {
  const int n = min(*n_dev, cap);
  const long long total = (long long)n * 27;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int j = t % 27;
    int4 c = coords[t / 27];
    int x = c.y + j / 9 - 1, y = c.z + (j / 3) % 3 - 1, z = c.w + j % 3 - 1;
    int r = -1;
    if (x >= 0 && x < X && y >= 0 && y < Y && z >= 0 && z < Z)
      r = hash_find(keys, vals, hcap, (unsigned long long)lin4(c.x, x, y, z, X, Y, Z));
    nbr[t] = r;
  }
}

}  // namespace fpvs

using namespace fpvs;

static long long ncells(int B, int X, int Y, int Z) { return (long long)B * X * Y * Z; }

extern "C" size_t fpvs_kmap_workspace_size(int B, int X, int Y, int Z) {
  long long nblk = (ncells(B, X, Y, Z) + kScanCells - 1) / kScanCells;
  return (size_t)(nblk + 1) * sizeof(unsigned);
}

extern "C" int fpvs_kmap_compact(const uint8_t* cell_active, int B, int X, int Y, int Z, int32_t* coords,
                                 int32_t* index_vol, int32_t* n_active_dev, int cap, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  FPVS_CHECK_ARG(B >= 1 && X >= 1 && Y >= 1 && Z >= 1, "bad cell grid");
  FPVS_CHECK_ARG(cell_active && coords && index_vol && n_active_dev && workspace, "null pointer");
  FPVS_CHECK_ARG(workspace_bytes >= fpvs_kmap_workspace_size(B, X, Y, Z), "workspace too small");
  const long long nc = ncells(B, X, Y, Z);
  FPVS_CHECK_ARG(nc < (1LL << 30), "cell grid too large for one compaction (%lld cells)", nc);
  const int nblk = (int)((nc + kScanCells - 1) / kScanCells);
  unsigned* status = (unsigned*)workspace;
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(status, 0, (size_t)(nblk + 1) * sizeof(unsigned), s);
  compact_kernel<<<nblk, kScanThreads, 0, s>>>(cell_active, nc, X, Y, Z, (int4*)coords, index_vol, cap, status,
                                               (int*)(status + nblk), n_active_dev, nblk);
  FPVS_CHECK_LAUNCH("fpvs_kmap_compact");
  return FPVS_OK;
}

extern "C" int fpvs_kmap_subm(const int32_t* coords, const int32_t* n_active_dev, int cap, const int32_t* index_vol,
                              int B, int X, int Y, int Z, int32_t* nbr, void* stream) {
  FPVS_CHECK_ARG(coords && n_active_dev && index_vol && nbr, "null pointer");
  (void)B;
  kmap_subm_kernel<<<grid_for((long long)cap * 27, 256), 256, 0, as_stream(stream)>>>(
      (const int4*)coords, n_active_dev, cap, index_vol, X, Y, Z, nbr);
  FPVS_CHECK_LAUNCH("fpvs_kmap_subm");
  return FPVS_OK;
}

extern "C" int fpvs_kmap_subm_k(const int32_t* coords, const int32_t* n_active_dev, int cap, const int32_t* index_vol,
                                int B, int X, int Y, int Z, int k, int32_t* nbr, void* stream) {
  FPVS_CHECK_ARG(coords && n_active_dev && index_vol && nbr, "null pointer");
  FPVS_CHECK_ARG(k >= 1 && k % 2 == 1 && k <= 15, "kernel size must be odd (1..15), got %d", k);
  (void)B;
  if (cap <= 0) return FPVS_OK;
  const long long K = (long long)k * k * k;
  kmap_subm_k_kernel<<<grid_for((long long)cap * K, 256), 256, 0, as_stream(stream)>>>(
      (const int4*)coords, n_active_dev, cap, index_vol, X, Y, Z, k, nbr);
  FPVS_CHECK_LAUNCH("fpvs_kmap_subm_k");
  return FPVS_OK;
}

extern "C" int fpvs_kmap_coarsen(const int32_t* coords, const int32_t* n_active_dev, int cap, int B, int X, int Y,
                                 int Z, uint8_t* coarse_active, void* stream) {
  FPVS_CHECK_ARG((X % 2 == 0) && (Y % 2 == 0) && (Z % 2 == 0), "k2s2 needs even dims (%d, %d, %d)", X, Y, Z);
  (void)B;
  kmap_coarsen_kernel<<<grid_for(cap, 256), 256, 0, as_stream(stream)>>>((const int4*)coords, n_active_dev, cap,
                                                                        X, Y, Z, coarse_active);
  FPVS_CHECK_LAUNCH("fpvs_kmap_coarsen");
  return FPVS_OK;
}

extern "C" int fpvs_kmap_down(const int32_t* coarse_coords, const int32_t* n_coarse_dev, int cap_coarse,
                              const int32_t* fine_index_vol, int B, int X, int Y, int Z, int32_t* down,
                              void* stream) {
  FPVS_CHECK_ARG((X % 2 == 0) && (Y % 2 == 0) && (Z % 2 == 0), "k2s2 needs even dims");
  (void)B;
  kmap_down_kernel<<<grid_for((long long)cap_coarse * 8, 256), 256, 0, as_stream(stream)>>>(
      (const int4*)coarse_coords, n_coarse_dev, cap_coarse, fine_index_vol, X, Y, Z, down);
  FPVS_CHECK_LAUNCH("fpvs_kmap_down");
  return FPVS_OK;
}

extern "C" int fpvs_kmap_up(const int32_t* fine_coords, const int32_t* n_fine_dev, int cap_fine,
                            const int32_t* coarse_index_vol, int B, int X, int Y, int Z, int32_t* up, void* stream) {
  FPVS_CHECK_ARG((X % 2 == 0) && (Y % 2 == 0) && (Z % 2 == 0), "k2s2 needs even dims");
  (void)B;
  kmap_up_kernel<<<grid_for((long long)cap_fine * 8, 256), 256, 0, as_stream(stream)>>>(
      (const int4*)fine_coords, n_fine_dev, cap_fine, coarse_index_vol, X, Y, Z, up);
  FPVS_CHECK_LAUNCH("fpvs_kmap_up");
  return FPVS_OK;
}

extern "C" int fpvs_kmap_tile_masks(const int32_t* table, int K, const int32_t* n_dev, int cap, uint32_t* masks,
                                    void* stream) {
  FPVS_CHECK_ARG(table && n_dev && masks, "null pointer");
  FPVS_CHECK_ARG(K >= 1 && K <= 32, "K must lie in [1, 32]");
  int tiles = (cap + 127) / 128;
  tile_masks_kernel<<<tiles < 4 * kNumSMs ? (tiles > 0 ? tiles : 1) : 4 * kNumSMs, 128, 0, as_stream(stream)>>>(
      table, K, n_dev, cap, masks);
  FPVS_CHECK_LAUNCH("fpvs_kmap_tile_masks");
  return FPVS_OK;
}

extern "C" int fpvs_hash_build(const int32_t* coords, const int32_t* n_active_dev, int cap, int B, int X, int Y,
                               int Z, int64_t* keys, int32_t* vals, int hash_capacity, void* stream) {
  FPVS_CHECK_ARG(hash_capacity >= 2 * kGroup && (hash_capacity & (hash_capacity - 1)) == 0,
                 "hash capacity must be a power of two >= 16");
  FPVS_CHECK_ARG(hash_capacity >= cap, "hash capacity %d < row capacity %d", hash_capacity, cap);
  (void)B;
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(keys, 0xff, sizeof(int64_t) * (size_t)hash_capacity, s);
  hash_build_kernel<<<grid_for((long long)cap * kGroup, 256), 256, 0, s>>>(
      (const int4*)coords, n_active_dev, cap, X, Y, Z, (unsigned long long*)keys, vals, hash_capacity);
  FPVS_CHECK_LAUNCH("fpvs_hash_build");
  return FPVS_OK;
}

extern "C" int fpvs_kmap_subm_hash(const int32_t* coords, const int32_t* n_active_dev, int cap, const int64_t* keys,
                                   const int32_t* vals, int hash_capacity, int B, int X, int Y, int Z, int32_t* nbr,
                                   void* stream) {
  FPVS_CHECK_ARG((hash_capacity & (hash_capacity - 1)) == 0, "hash capacity must be a power of two");
  (void)B;
  kmap_subm_hash_kernel<<<grid_for((long long)cap * 27, 256), 256, 0, as_stream(stream)>>>(
      (const int4*)coords, n_active_dev, cap, (const unsigned long long*)keys, vals, hash_capacity, X, Y, Z, nbr);
  FPVS_CHECK_LAUNCH("fpvs_kmap_subm_hash");
  return FPVS_OK;
}
