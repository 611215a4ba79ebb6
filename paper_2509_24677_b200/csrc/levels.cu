// (2b) One frame's kernel maps in three launches.
//
// The granular kmap entry points (kmap.cu) mirror the reference's per-step
// structure: active flags, compaction, then one table per launch.  For a
// U-Net frame that is ~20 launches, each a few microseconds of mostly idle
// GPU.  fpvs_levels_from_bits builds the same tables (bit-exact: same
// canonical C-order rows, same offset order) for an nlev-level hierarchy in
// three launches:
//
//   K1  level-0 active flags from the packed bits (one block per
//       (b, cell-row y, kZC = 16 cells of z): lanes read contiguous bytes of a voxel
//       row, the d^2 rows of a cell are loaded back to back (d is a template
//       parameter, so the loads are independent and in flight together));
//   K2  single-pass compaction of EVERY level (decoupled look-back with a
//       32-wide warp window); level l > 0 flags are ORs over 2^l boxes of the
//       level-0 flags, computed in the scan's load phase (no coarsen pass);
//   K3  every table in one persistent launch: submanifold 3x3x3 tables, k2s2
//       down/up tables, their per-128-row offset masks (block OR, no extra
//       pass), the level-0 feature gather from the bits, the clear of the
//       output grid, and the reset of K2's look-back state for the next frame.
//
// Everything is sized from device counters: the three launches are
// graph-capturable and never synchronise.
#include <cooperative_groups.h>
#include <type_traits>

#include "common.cuh"
#include "halo_build.cuh"

namespace fpvs {
namespace lv {

constexpr int kMaxLev = 4;
constexpr int kThreads = 256;
constexpr int kPer = 16;                    // cells per scan thread
#ifndef FPVS_K2_THREADS
#define FPVS_K2_THREADS 256  // measured 64 / 128 / 256 / 512 / 1024: 317 / 310 / 307 / 309 / 311 us per frame
#endif
constexpr int kThreads2 = FPVS_K2_THREADS;   // K2 block size (scan tile = kThreads2 * kPer cells)
constexpr int kTileCells = kThreads2 * kPer;
constexpr int kRows = 128;                  // table rows per K3 unit (one conv tile)
#ifndef FPVS_K1_ZC
#define FPVS_K1_ZC 16  // measured 32 / 16 / 8: 309-311 / 307 / 307 us per frame (more blocks in flight)
#endif
constexpr int kZC = FPVS_K1_ZC;             // K1: level-0 z cells per block
constexpr unsigned kFlagAgg = 1u << 30, kFlagPrefix = 2u << 30, kValMask = (1u << 30) - 1u;

struct LevelDev {
  int4* coords;
  int* index_vol;
  int* n;
  int cap;
  int* nbr;
  uint32_t* nbr_masks;
  int* down;
  uint32_t* down_masks;
  int* up;
  uint32_t* up_masks;
  int* halo_rows;     // nullable: per-tile halo tables (halo_build.cuh) of the 3^3 map
  int* halo_n;
  int16_t* halo_lnbr;
  int X, Y, Z;
  int ntiles;         // K2 scan tiles
  unsigned* status;   // [ntiles] look-back flags, then 1 tile counter
};

struct Args {
  const uint8_t* bits;
  int B, Nx, Ny, Nz, d, nlev;
  uint8_t* act[kMaxLev];  // per-level active flags, one byte per cell (workspace)
  long long act_bytes[kMaxLev];
  LevelDev L[kMaxLev];
  int tile_base[kMaxLev + 1];  // K2 block ranges per level
  void* feat;
  int feat_bf16, ldf;
  uint8_t* clear;
  long long clear_bytes;
  unsigned* status_all;
  int status_words;
  int reset_only;  // profiling (FPVS_LV_STOP = 2): K3 runs only the look-back reset
  int k2_abl;      // profiling builds (FPVS_K2_ABL, wrong results): 1 no look-back, 2 no index_vol
                   // stores, 4 no coords stores, 8 no flag loads, 16 no ticket atomic
};

#ifdef FPVS_PROFILE
#define K2ABL(bit) (a.k2_abl & (bit))
#else
#define K2ABL(bit) 0
#endif

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ------------------------------------------------------------------ K1
// Block (b, cy, cz0..cz0+31): thread unit (cz, word xw of the voxel row; a
// word is W bytes) ORs the d x d voxel rows of that cell column (all d^2
// loads in flight), then splits the word into its 8W/d cells.  Flags are
// transposed through shared memory so the C-order (z-fastest) level-0 rows
// go out in 32-byte runs; coarser levels get a 1 for every parent with an
// active child (their arrays are cleared by K3 of the previous frame).
template <int D, int W>
__device__ __forceinline__ void l0_flags_body(const Args& a, int blk, uint8_t* s_flag) {  // s_flag: [X][kZC + 1]
  using T = typename std::conditional<W == 4, uint32_t, uint8_t>::type;
  const int X = a.L[0].X, Y = a.L[0].Y, Z = a.L[0].Z;
  const int nzc = (Z + kZC - 1) / kZC;
  const int zc = blk % nzc;
  blk /= nzc;
  const int cy = blk % Y;
  const int b = blk / Y;
  const int cz0 = zc * kZC, nz = min(kZC, Z - cz0);
  const int roww = a.Nx / (8 * W);  // words per voxel row
  const long long plane = (long long)(a.Nx >> 3) * a.Ny * a.Nz;
  const T* gb = reinterpret_cast<const T*>(a.bits + b * plane);
  const int units = roww * nz;
  constexpr int CPW = 8 * W / D;  // cells per word
  for (int u = threadIdx.x; u < units; u += kThreads) {
    const int xw = u % roww, czl = u / roww;
    const int cz = cz0 + czl;
    T v[D * D];
#pragma unroll
    for (int lz = 0; lz < D; ++lz)
#pragma unroll
      for (int ly = 0; ly < D; ++ly)
        v[lz * D + ly] = __ldg(gb + xw + (long long)roww * ((cy * D + ly) + (long long)a.Ny * (cz * D + lz)));
    uint32_t o = 0;
#pragma unroll
    for (int i = 0; i < D * D; ++i) o |= (uint32_t)v[i];
    constexpr uint32_t M = D >= 32 ? 0xffffffffu : (1u << D) - 1u;
#pragma unroll
    for (int i = 0; i < CPW; ++i) s_flag[(xw * CPW + i) * (kZC + 1) + czl] = ((o >> (i * D)) & M) ? 1 : 0;
  }
  __syncthreads();
  const long long rowbase = ((long long)b * X) * Y * Z;
  for (int u = threadIdx.x; u < X * nz; u += kThreads) {
    const int cx = u / nz, zl = u - cx * nz;
    a.act[0][rowbase + ((long long)cx * Y + cy) * Z + cz0 + zl] = s_flag[cx * (kZC + 1) + zl];
  }
  for (int l = 1; l < a.nlev; ++l) {
    const int F = 1 << l, Xl = X >> l, Yl = Y >> l, Zl = Z >> l, nzl = nz >> l;
    for (int u = threadIdx.x; u < Xl * nzl; u += kThreads) {
      const int cx = u / nzl, zl = u - cx * nzl;
      uint32_t any = 0;
      for (int dx = 0; dx < F; ++dx)
        for (int dz = 0; dz < F; ++dz) any |= s_flag[(cx * F + dx) * (kZC + 1) + zl * F + dz];
      if (any) a.act[l][(((long long)b * Xl + cx) * Yl + (cy >> l)) * Zl + (cz0 >> l) + zl] = 1;
    }
  }
}

template <int D, int W>
__global__ void __launch_bounds__(kThreads) l0_flags_kernel(const Args a) {
  // K2 is launched programmatically: let it take its tile tickets while we run
  if (threadIdx.x == 0) pdl_trigger();
  extern __shared__ uint8_t s_flag[];
  l0_flags_body<D, W>(a, blockIdx.x, s_flag);
}

// ------------------------------------------------------------------ K2
// flags of 16 consecutive C-order cells of level l (base linear index r0)
__device__ __forceinline__ uint32_t level_flags16(const Args& a, int l, int r0, int ncell) {
  const uint8_t* act = a.act[l];
  uint32_t f = 0;
  if (r0 + kPer <= ncell) {
    const uint4 v = *reinterpret_cast<const uint4*>(act + r0);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 16; ++i) f |= (((w[i >> 2] >> ((i & 3) * 8)) & 0xffu) ? 1u : 0u) << i;
  } else {
    for (int i = 0; i < kPer; ++i)
      if (r0 + i < ncell && act[r0 + i]) f |= 1u << i;
  }
  return f;
}

// pdl: launched programmatically after K1 (false inside the cooperative
// single-launch build, where a grid barrier orders the phases)
template <bool PDL>
__device__ __forceinline__ void compact_body(const Args& a, int blk) {
  __shared__ int s_tile, s_prefix;
  __shared__ int s_warp[kThreads2 / 32];
  int l = 0;
  while (l + 1 < a.nlev && blk >= a.tile_base[l + 1]) ++l;
  const LevelDev& L = a.L[l];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // the tile ticket counter was re-armed by K3 of the previous frame (complete
  // before K1 started); the flags below are K1's output: wait for it
  if (tid == 0) s_tile = K2ABL(16) ? blk - a.tile_base[l] : (int)atomicAdd(L.status + L.ntiles, 1u);
  if constexpr (PDL) {
    pdl_wait();
    if (tid == 0) pdl_trigger();
  }
  __syncthreads();
  const int tile = s_tile;
  const int X = L.X, Y = L.Y, Z = L.Z;
  const int ncell = a.B * X * Y * Z;
  const int r0 = tile * kTileCells + tid * kPer;
  const uint32_t f = r0 < ncell ? (K2ABL(8) ? 0x1111u : level_flags16(a, l, r0, ncell)) : 0u;
  const int cnt = __popc(f);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int w = lane < kThreads2 / 32 ? s_warp[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < kThreads2 / 32) s_warp[lane] = wi - w;
    const unsigned agg = (unsigned)__shfl_sync(0xffffffffu, wi, 31);
    unsigned prefix = 0;
    if (tile == 0 || K2ABL(1)) {
      if (lane == 0) st_release(L.status + tile, kFlagPrefix | agg);
    } else {
      if (lane == 0) st_release(L.status + tile, kFlagAgg | agg);
      // look back 32 predecessors at a time
      for (int t = tile - 1;; t -= 32) {
        const int idx = t - lane;
        unsigned v = idx >= 0 ? ld_acquire(L.status + idx) : kFlagPrefix;
        while (__any_sync(0xffffffffu, !(v & (kFlagAgg | kFlagPrefix))))
          if (!(v & (kFlagAgg | kFlagPrefix))) v = ld_acquire(L.status + idx);
        const unsigned pm = __ballot_sync(0xffffffffu, (v & kFlagPrefix) != 0);
        const int stop = pm ? __ffs(pm) - 1 : 31;  // nearest predecessor holding an inclusive prefix
        prefix += __reduce_add_sync(0xffffffffu, lane <= stop ? (v & kValMask) : 0u);
        if (pm) break;
      }
      if (lane == 0) st_release(L.status + tile, kFlagPrefix | (prefix + agg));
    }
    if (lane == 0) {
      s_prefix = (int)prefix;
      if (tile == L.ntiles - 1) *L.n = (int)(prefix + agg);
    }
  }
  __syncthreads();
  if (r0 >= ncell) return;
  int rank = s_prefix + s_warp[wid] + incl - cnt;
  int rows[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const bool on = (f >> i) & 1u;
    rows[i] = (on && rank < L.cap) ? rank : -1;
    rank += on ? 1 : 0;
  }
  if (K2ABL(2)) {
  } else if (r0 + kPer <= ncell) {
    int4* dst = reinterpret_cast<int4*>(L.index_vol + r0);
#pragma unroll
    for (int q = 0; q < 4; ++q) dst[q] = make_int4(rows[4 * q], rows[4 * q + 1], rows[4 * q + 2], rows[4 * q + 3]);
  } else {
    for (int i = 0; i < kPer && r0 + i < ncell; ++i) L.index_vol[r0 + i] = rows[i];
  }
  if (f && !K2ABL(4)) {
    int r = r0;
    int z = r % Z; r /= Z;
    int y = r % Y; r /= Y;
    int x = r % X;
    int b = r / X;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      if (rows[i] >= 0) L.coords[rows[i]] = make_int4(b, x, y, z);
      if (++z == Z) { z = 0; if (++y == Y) { y = 0; if (++x == X) { x = 0; ++b; } } }
    }
  }
}

__global__ void __launch_bounds__(kThreads2) compact_levels_kernel(const Args a) { compact_body<true>(a, blockIdx.x); }

// ------------------------------------------------------------------ K3
enum Task { T_SUBM = 0, T_DOWN, T_UP, T_GATHER, T_CLEAR, T_RESET, T_COUNT };

__device__ __forceinline__ int nrows(const LevelDev& L) { return min(*L.n, L.cap); }

__device__ __forceinline__ void block_or_store(uint32_t m, uint32_t* s_red, uint32_t* dst) {
  m = __reduce_or_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) t |= s_red[w];
    *dst = t;
  }
  __syncthreads();
}

// offsets j in [J0, J0 + NJ) of one row: lookups straight off the row's own
// index-volume position (compile-time offset pattern, runtime strides)
template <int J0, int NJ>
__device__ __forceinline__ uint32_t subm_row(const LevelDev& L, const int4 c, int* dst) {
  const int X = L.X, Y = L.Y, Z = L.Z;
  const int* vol = L.index_vol + ((c.x * X + c.y) * Y + c.z) * Z + c.w;
  int v[NJ];
#pragma unroll
  for (int q = 0; q < NJ; ++q) {
    const int j = J0 + q, da = j / 9 - 1, db = (j / 3) % 3 - 1, dc = j % 3 - 1;
    const bool ok = (da < 0 ? c.y > 0 : da > 0 ? c.y < X - 1 : true) &&
                    (db < 0 ? c.z > 0 : db > 0 ? c.z < Y - 1 : true) &&
                    (dc < 0 ? c.w > 0 : dc > 0 ? c.w < Z - 1 : true);
    v[q] = ok ? __ldg(vol + (da * Y + db) * Z + dc) : -1;
  }
  uint32_t m = 0;
#pragma unroll
  for (int q = 0; q < NJ; ++q) {
    dst[J0 + q] = v[q];
    m |= (v[q] >= 0 ? 1u : 0u) << (J0 + q);
  }
  return m;
}

// 128 rows x 27: thread t handles row t%128, offsets [0,14) or [14,27); the
// tile is staged in shared memory and leaves as coalesced 16-byte stores
__device__ void subm_unit(const LevelDev& L, int n, int tile, int* s_tab, uint32_t* s_red, halob::Smem* s_halo) {
  const int r0 = tile * kRows;
  const int rows = min(kRows, n - r0);
  const int row = threadIdx.x & (kRows - 1);
  uint32_t m = 0;
  if (row < rows) {
    const int4 c = L.coords[r0 + row];
    m = threadIdx.x < kRows ? subm_row<0, 14>(L, c, s_tab + row * 27) : subm_row<14, 13>(L, c, s_tab + row * 27);
  }
  __syncthreads();
  int* out = L.nbr + (long long)r0 * 27;
  if (rows == kRows) {
    const uint4* src = reinterpret_cast<const uint4*>(s_tab);
    uint4* dst = reinterpret_cast<uint4*>(out);
    for (int i = threadIdx.x; i < kRows * 27 / 4; i += kThreads) dst[i] = src[i];
  } else {
    for (int i = threadIdx.x; i < rows * 27; i += kThreads) out[i] = s_tab[i];
  }
  if (L.nbr_masks) block_or_store(m, s_red, L.nbr_masks + tile);
  else __syncthreads();  // s_tab is reused by the next unit
  if (L.halo_rows) {
    // the tile's halo list and local table straight from the staged rows
    halob::build_tile([&](int e) { return e / 27 < rows ? s_tab[e] : -1; }, *s_halo,
                      L.halo_rows + (long long)tile * halob::kHmax, L.halo_n + tile,
                      L.halo_lnbr + (long long)tile * kRows * 27);
  }
}

// down table of level l (rows of l) into level l-1
__device__ void down_unit(const LevelDev& C, const LevelDev& Fn, int n, int tile, uint32_t* s_red) {
  const int r0 = tile * kRows;
  const int nent = min(kRows, n - r0) * 8;
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < kRows * 8 / kThreads; ++k) {
    const int e = threadIdx.x + k * kThreads;
    if (e < nent) {
      const int row = e >> 3, j = e & 7;
      const int4 c = C.coords[r0 + row];
      const int v = __ldg(Fn.index_vol + ((c.x * Fn.X + 2 * c.y + (j >> 2)) * Fn.Y + 2 * c.z + ((j >> 1) & 1)) * Fn.Z +
                          2 * c.w + (j & 1));
      C.down[(long long)r0 * 8 + e] = v;
      m |= (v >= 0 ? 1u : 0u) << j;
    }
  }
  if (C.down_masks) block_or_store(m, s_red, C.down_masks + tile);
}

// up table of level l: rows of level l-1 -> their parent in l (own parity slot)
__device__ void up_unit(const LevelDev& C, const LevelDev& Fn, int n, int tile, uint32_t* s_red) {
  const int r0 = tile * kRows;
  const int nent = min(kRows, n - r0) * 8;
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < kRows * 8 / kThreads; ++k) {
    const int e = threadIdx.x + k * kThreads;
    if (e < nent) {
      const int row = e >> 3, j = e & 7;
      const int4 c = Fn.coords[r0 + row];
      const int par = ((c.y & 1) << 2) | ((c.z & 1) << 1) | (c.w & 1);
      int v = -1;
      if (j == par) v = __ldg(C.index_vol + ((c.x * C.X + (c.y >> 1)) * C.Y + (c.z >> 1)) * C.Z + (c.w >> 1));
      C.up[(long long)r0 * 8 + e] = v;
      m |= (v >= 0 ? 1u : 0u) << j;
    }
  }
  if (C.up_masks) block_or_store(m, s_red, C.up_masks + tile);
}

// level-0 features: channel k = lx + d*(ly + d*lz) of row i = bit of froxel
// (b, x*d + lx, y*d + ly, z*d + lz).  A thread owns 8 channels = 8/d voxel
// rows of d bits (d in {1, 2, 4, 8}): 8/d byte loads, one 16-byte store.
__device__ void gather_unit(const Args& a, int n, int tile) {
  const LevelDev& L = a.L[0];
  const int d = a.d, dl = __ffs(d) - 1, d3 = d * d * d, groups = (d3 + 7) >> 3;
  const int rpg = 8 >> dl;  // voxel rows per 8-channel group
  const int r0 = tile * kRows;
  const int nent = min(kRows, n - r0) * groups;
  const int rowb = a.Nx >> 3;
  const bool vec = (d3 % 8 == 0) && (a.ldf % 8 == 0);
  const uint32_t dm = (1u << d) - 1u;
  constexpr int NB = 4;  // entries per thread per batch: all their loads in flight together
  for (int e0 = 0; e0 < nent; e0 += NB * kThreads) {
    int4 c[NB];
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int e = e0 + threadIdx.x + q * kThreads;
      c[q] = e < nent ? L.coords[r0 + e / groups] : make_int4(0, 0, 0, 0);
    }
    uint32_t bits8[NB];
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int e = e0 + threadIdx.x + q * kThreads;
      const int g = e % groups;
      const int fx = c[q].y * d;
      const uint8_t* gb = a.bits + (long long)c[q].x * rowb * a.Ny * a.Nz + (fx >> 3);
      bits8[q] = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = ((g * 8) >> dl) + i;  // voxel row (ly, lz) = (r % d, r / d)
        if (i < rpg && e < nent && r < d * d) {
          const uint32_t byte =
              __ldg(gb + (long long)rowb * ((c[q].z * d + (r & (d - 1))) + (long long)a.Ny * (c[q].w * d + (r >> dl))));
          bits8[q] |= ((byte >> (fx & 7)) & dm) << (i * d);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int e = e0 + threadIdx.x + q * kThreads;
      if (e >= nent) continue;
      const int row = e / groups, g = e - row * groups;
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = (float)((bits8[q] >> i) & 1u);
      const long long off = (long long)(r0 + row) * a.ldf + g * 8;
      if (a.feat_bf16) {
        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(a.feat) + off;
        if (vec) {
          __nv_bfloat162 h[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
          *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<uint4*>(h);
        } else {
          for (int i = 0; i < 8 && g * 8 + i < d3; ++i) dst[i] = __float2bfloat16_rn(v[i]);
        }
      } else {
        float* dst = reinterpret_cast<float*>(a.feat) + off;
        if (vec) {
          reinterpret_cast<float4*>(dst)[0] = make_float4(v[0], v[1], v[2], v[3]);
          reinterpret_cast<float4*>(dst)[1] = make_float4(v[4], v[5], v[6], v[7]);
        } else {
          for (int i = 0; i < 8 && g * 8 + i < d3; ++i) dst[i] = v[i];
        }
      }
    }
  }
}

constexpr int kClearChunk = kThreads * 64;  // bytes per clear unit

#ifndef FPVS_K3_MINB
#define FPVS_K3_MINB 4  // >= 4 resident blocks per SM (without it ptxas takes 109 registers: 2 blocks, +6 us per frame)
#endif
template <bool PDL>
__device__ __forceinline__ void tables_body(const Args& a) {
  // programmatic launch: everything here reads K2's output.  No early trigger:
  // the first conv's prologue reads the tile masks written here
  if constexpr (PDL) pdl_wait();
  __shared__ uint32_t s_red[kThreads / 32];
  __shared__ __align__(16) int s_tab[kRows * 27];
  __shared__ __align__(16) halob::Smem s_halo;
  __shared__ int s_pre[T_COUNT * kMaxLev + 1];  // unit prefix per (task, level)
  __shared__ int s_nl[kMaxLev];
  if (threadIdx.x < kMaxLev) s_nl[threadIdx.x] = (int)threadIdx.x < a.nlev ? nrows(a.L[threadIdx.x]) : 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    int total = 0;
    for (int t = 0; t < T_COUNT; ++t)
      for (int l = 0; l < kMaxLev; ++l) {
        int c = 0;
        if (l < a.nlev && (!a.reset_only || t == T_RESET)) {
          const LevelDev& L = a.L[l];
          if (t == T_SUBM && L.nbr) c = (s_nl[l] + kRows - 1) / kRows;
          if (t == T_DOWN && l > 0 && L.down) c = (s_nl[l] + kRows - 1) / kRows;
          if (t == T_UP && l > 0 && L.up) c = (s_nl[l - 1] + kRows - 1) / kRows;
          if (t == T_GATHER && l == 0 && a.feat) c = (s_nl[0] + kRows - 1) / kRows;
          if (t == T_CLEAR && l == 0 && a.clear) c = (int)((a.clear_bytes + kClearChunk - 1) / kClearChunk);
          if (t == T_RESET) c = 1;
        }
        s_pre[t * kMaxLev + l] = total;
        total += c;
      }
    s_pre[T_COUNT * kMaxLev] = total;
  }
  __syncthreads();
  const int total = s_pre[T_COUNT * kMaxLev];
  const int lane = threadIdx.x & 31;
  int nl[kMaxLev];
#pragma unroll
  for (int l = 0; l < kMaxLev; ++l) nl[l] = s_nl[l];
  // persistent: the grid is exactly one resident wave, blocks stride the units
  for (int u = blockIdx.x; u < total; u += gridDim.x) {
    // (task, level) = number of prefix entries <= u, minus one
    const bool le = lane < T_COUNT * kMaxLev && s_pre[lane] <= u;
    const int idx = __popc(__ballot_sync(0xffffffffu, le)) - 1;
    const int t = idx / kMaxLev, l = idx % kMaxLev, k = u - s_pre[idx];
    switch (t) {
      case T_SUBM: subm_unit(a.L[l], nl[l], k, s_tab, s_red, &s_halo); break;
      case T_DOWN: down_unit(a.L[l], a.L[l - 1], nl[l], k, s_red); break;
      case T_UP: up_unit(a.L[l], a.L[l - 1], nl[l - 1], k, s_red); break;
      case T_GATHER: gather_unit(a, nl[0], k); break;
      case T_CLEAR: {
        const long long base = (long long)k * kClearChunk;
        const long long nb = min((long long)kClearChunk, a.clear_bytes - base);
        if (nb == kClearChunk && ((reinterpret_cast<uintptr_t>(a.clear + base) & 15) == 0)) {
          uint4* dst = reinterpret_cast<uint4*>(a.clear + base);
#pragma unroll
          for (int q = 0; q < kClearChunk / 16 / kThreads; ++q) dst[threadIdx.x + q * kThreads] = make_uint4(0, 0, 0, 0);
        } else {
          for (long long i = threadIdx.x; i < nb; i += kThreads) a.clear[base + i] = 0;
        }
        break;
      }
      case T_RESET:
        // K2 has finished (stream order): re-arm its look-back state and
        // clear the coarse-level flags K1 of the next frame ORs into
        if (l == 0) {
          for (int i = threadIdx.x; i < a.status_words; i += kThreads) a.status_all[i] = 0;
        } else {
          uint4* p = reinterpret_cast<uint4*>(a.act[l]);
          for (long long i = threadIdx.x; i < a.act_bytes[l] / 16; i += kThreads) p[i] = make_uint4(0, 0, 0, 0);
        }
        break;
    }
  }
}

__global__ void __launch_bounds__(kThreads, FPVS_K3_MINB) tables_kernel(const Args a) { tables_body<true>(a); }

// All three as ONE cooperative launch (grid = every resident block; phases
// ordered by grid barriers instead of kernel boundaries): K1's units, K2's
// tiles, then K3's persistent loop.  Co-residency is guaranteed by the
// cooperative launch, so the barriers cannot deadlock against other work.
template <int D, int W>
__global__ void __launch_bounds__(kThreads, FPVS_K3_MINB) maps_fused_kernel(const Args a, int k1_blocks, int k2_blocks) {
  extern __shared__ uint8_t s_flag[];
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  for (int blk = blockIdx.x; blk < k1_blocks; blk += gridDim.x) {
    l0_flags_body<D, W>(a, blk, s_flag);
    __syncthreads();
  }
  grid.sync();
  for (int blk = blockIdx.x; blk < k2_blocks; blk += gridDim.x) {
    compact_body<false>(a, blk);
    __syncthreads();
  }
  grid.sync();
  tables_body<false>(a);
}

// the cooperative single launch measured 8 us SLOWER per frame than the three
// launches (308 -> 317 us: two grid barriers and a 592-block grid for phases
// that use 256 and 73 blocks cost more than the launch gaps they remove), so it
// is off unless FPVS_MAPS_FUSED=1
#ifndef FPVS_MAPS_FUSED
#define FPVS_MAPS_FUSED 0
#endif
inline bool maps_fused_enabled() {
  static const bool on = [] {
    const char* e = getenv("FPVS_MAPS_FUSED");  // read once: A/B switch (0 = three launches)
    return e ? atoi(e) != 0 : FPVS_MAPS_FUSED != 0;
  }();
  return on;
}

template <int D, int W>
inline cudaError_t launch_fused(const Args& a, int k1_blocks, int k2_blocks, size_t smem1, cudaStream_t s) {
  static const int per_sm = [smem1] {
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, maps_fused_kernel<D, W>, kThreads, smem1) != cudaSuccess)
      v = 0;
    return v;
  }();
  if (per_sm < 1) return cudaErrorNotSupported;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kNumSMs * per_sm);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem1;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, maps_fused_kernel<D, W>, a, k1_blocks, k2_blocks);
}

}  // namespace lv
}  // namespace fpvs

using namespace fpvs;

static long long lv_status_words(int B, int X, int Y, int Z, int nlev) {
  long long w = 0;
  for (int l = 0; l < nlev; ++l) {
    const long long nc = (long long)B * (X >> l) * (Y >> l) * (Z >> l);
    w += (nc + lv::kTileCells - 1) / lv::kTileCells + 1;
  }
  return w;
}

static long long lv_act_bytes(int B, int X, int Y, int Z, int l) {
  const long long nc = (long long)B * (X >> l) * (Y >> l) * (Z >> l);
  return (nc + 255) / 256 * 256;
}

extern "C" size_t fpvs_levels_workspace_size(int B, int Nx, int Ny, int Nz, int d, int nlev) {
  if (B < 1 || d < 1 || nlev < 1 || nlev > lv::kMaxLev || Nx % d || Ny % d || Nz % d) return 0;
  const int X = Nx / d, Y = Ny / d, Z = Nz / d;
  long long act = 0;
  for (int l = 0; l < nlev; ++l) act += lv_act_bytes(B, X, Y, Z, l);
  return (size_t)(act + 4 * lv_status_words(B, X, Y, Z, nlev));
}

extern "C" int fpvs_levels_from_bits(const uint8_t* bits, int B, int Nx, int Ny, int Nz, int d, int nlev,
                                     const fpvs_level* levels, void* workspace, size_t workspace_bytes, void* feat,
                                     int feat_dtype, int ldf, uint8_t* clear_bits, size_t clear_bytes,
                                     void* stream) {
  FPVS_CHECK_ARG(bits && levels && workspace, "null pointer");
  FPVS_CHECK_ARG(B >= 1 && Nx >= 8 && Ny >= 1 && Nz >= 1, "bad grid");
  FPVS_CHECK_ARG(Nx % 8 == 0, "N_x must be divisible by 8, got %d", Nx);
  FPVS_CHECK_ARG(d == 1 || d == 2 || d == 4 || d == 8, "fused level build needs d in {1, 2, 4, 8}, got %d", d);
  FPVS_CHECK_ARG(nlev >= 1 && nlev <= lv::kMaxLev, "nlev must lie in [1, %d]", lv::kMaxLev);
  if (Nx % d || Ny % d || Nz % d)
    return set_error(FPVS_ESHAPE, "interleave factor %d must divide grid dims (%d, %d, %d)", d, Nx, Ny, Nz);
  const int X = Nx / d, Y = Ny / d, Z = Nz / d;
  const int f = 1 << (nlev - 1);
  if (X % f || Y % f || Z % f)
    return set_error(FPVS_ESHAPE, "%d levels need cell dims (%d, %d, %d) divisible by %d", nlev, X, Y, Z, f);
  const long long nc0 = (long long)B * X * Y * Z;
  FPVS_CHECK_ARG(nc0 < (1LL << 30), "cell grid too large (%lld cells)", nc0);
  FPVS_CHECK_ARG(workspace_bytes >= fpvs_levels_workspace_size(B, Nx, Ny, Nz, d, nlev), "workspace too small");
  FPVS_CHECK_ARG((X * (lv::kZC + 1)) <= 48 * 1024, "N_x / d too large for the flag transpose");
  FPVS_CHECK_ARG(!feat || (feat_dtype == FPVS_F32 || feat_dtype == FPVS_BF16), "bad feature dtype");
  FPVS_CHECK_ARG(!feat || ldf >= d * d * d, "feature ld %d < d^3", ldf);
  lv::Args a{};
  a.bits = bits;
  a.B = B; a.Nx = Nx; a.Ny = Ny; a.Nz = Nz; a.d = d; a.nlev = nlev;
  uint8_t* ws = (uint8_t*)workspace;
  for (int l = 0; l < nlev; ++l) {
    a.act[l] = ws;
    a.act_bytes[l] = lv_act_bytes(B, X, Y, Z, l);
    ws += a.act_bytes[l];
  }
  unsigned* st = (unsigned*)ws;
  a.status_all = st;
  a.status_words = (int)lv_status_words(B, X, Y, Z, nlev);
  int tb = 0;
  for (int l = 0; l < nlev; ++l) {
    const fpvs_level& h = levels[l];
    FPVS_CHECK_ARG(h.coords && h.index_vol && h.n, "level %d: null coords/index_vol/n", l);
    FPVS_CHECK_ARG(l > 0 || (!h.down && !h.up), "level 0 has no down/up tables");
    lv::LevelDev& L = a.L[l];
    L.coords = (int4*)h.coords;
    L.index_vol = h.index_vol;
    L.n = h.n;
    L.cap = h.cap;
    L.nbr = h.nbr;
    L.nbr_masks = h.nbr_masks;
    L.down = h.down;
    L.down_masks = h.down_masks;
    L.up = h.up;
    L.up_masks = h.up_masks;
    FPVS_CHECK_ARG(!h.halo_rows || (h.halo_n && h.halo_lnbr && h.nbr), "level %d: halo tables need nbr, n, lnbr", l);
    L.halo_rows = h.halo_rows;
    L.halo_n = h.halo_n;
    L.halo_lnbr = h.halo_lnbr;
    L.X = X >> l; L.Y = Y >> l; L.Z = Z >> l;
    const long long nc = (long long)B * L.X * L.Y * L.Z;
    L.ntiles = (int)((nc + lv::kTileCells - 1) / lv::kTileCells);
    L.status = st;
    st += L.ntiles + 1;
    a.tile_base[l] = tb;
    tb += L.ntiles;
  }
  a.tile_base[nlev] = tb;
  a.feat = feat;
  a.feat_bf16 = feat_dtype == FPVS_BF16;
  a.ldf = ldf;
  a.clear = clear_bits;
  a.clear_bytes = clear_bits ? (long long)clear_bytes : 0;
  cudaStream_t s = as_stream(stream);
  const unsigned k1 = (unsigned)((long long)B * Y * ((Z + lv::kZC - 1) / lv::kZC));
  const size_t smem1 = (size_t)X * (lv::kZC + 1);
  if (lv::maps_fused_enabled() && debug_knob("FPVS_LV_STOP") == 0) {
    // one cooperative launch for K1 + K2 + K3 (falls through to three
    // launches when the device cannot hold the whole grid at once)
    cudaError_t e = cudaErrorNotSupported;
#define FPVS_KF(D)                                                                              \
  e = Nx % 32 == 0 ? lv::launch_fused<D, 4>(a, (int)k1, tb, smem1, s) : lv::launch_fused<D, 1>(a, (int)k1, tb, smem1, s);
    switch (d) {
      case 1: FPVS_KF(1); break;
      case 2: FPVS_KF(2); break;
      case 4: FPVS_KF(4); break;
      default: FPVS_KF(8); break;
    }
#undef FPVS_KF
    if (e == cudaSuccess) {
      FPVS_CHECK_LAUNCH("fpvs_levels_from_bits(fused)");
      return FPVS_OK;
    }
    (void)cudaGetLastError();  // a failed cooperative launch leaves no sticky error
  }
#define FPVS_K1(D)                                                                      \
  if (Nx % 32 == 0) lv::l0_flags_kernel<D, 4><<<k1, lv::kThreads, smem1, s>>>(a);        \
  else lv::l0_flags_kernel<D, 1><<<k1, lv::kThreads, smem1, s>>>(a);
  switch (d) {
    case 1: FPVS_K1(1); break;
    case 2: FPVS_K1(2); break;
    case 4: FPVS_K1(4); break;
    default: FPVS_K1(8); break;
  }
#undef FPVS_K1
  FPVS_CHECK_LAUNCH("fpvs_levels_from_bits(flags)");
  const int stop = debug_knob("FPVS_LV_STOP");  // profiling builds: launch K1 (1) or K1 + K2 (2) only
  if (stop == 1) return FPVS_OK;
  a.k2_abl = debug_knob("FPVS_K2_ABL");
  cudaError_t e = launch_kernel(lv::compact_levels_kernel, dim3(tb), dim3(lv::kThreads2), 0, s, a);
  if (e != cudaSuccess) return set_error(FPVS_ECUDA, "fpvs_levels_from_bits(compact): %s", cudaGetErrorString(e));
  FPVS_CHECK_LAUNCH("fpvs_levels_from_bits(compact)");
  a.reset_only = stop == 2;
  // K3: one resident wave (a second wave of persistent blocks would serialise)
  static const int k3_per_sm = [] {  // thread-safe one-time occupancy query
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, lv::tables_kernel, lv::kThreads, 0) != cudaSuccess || v < 1)
      v = 1;
    return v;
  }();
  e = launch_kernel(lv::tables_kernel, dim3(kNumSMs * k3_per_sm), dim3(lv::kThreads), 0, s, a);
  if (e != cudaSuccess) return set_error(FPVS_ECUDA, "fpvs_levels_from_bits(tables): %s", cudaGetErrorString(e));
  FPVS_CHECK_LAUNCH("fpvs_levels_from_bits(tables)");
  return FPVS_OK;
}
