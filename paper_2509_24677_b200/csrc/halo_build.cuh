// Per-tile halo table of a 27-tap neighbour table (the halo-cached conv,
// spconv_halo.cu, reads it): for one 128-row tile, the sorted distinct
// neighbour rows (<= FPVS_HALO_MAX) and the tile-local table
// lnbr[r][j] = slot of nbr[r][j] in that list (-1 = no neighbour, -2 = not
// cached -> the conv reads the row from HBM, so results never depend on the
// cache).  Shared by the stand-alone build (fpvs_kmap_halo_multi) and the fused
// level build (levels.cu K3, which runs it on the tile it has just written).
#pragma once

#include <limits.h>

#include "common.cuh"

namespace fpvs {
namespace halob {

constexpr int kRows = 128;
constexpr int kOff = 27;
constexpr int kHmax = FPVS_HALO_MAX;
constexpr int kWinWords = 512;  // 16384-row window (wider tiles read directly)
constexpr int kPer = (kRows * kOff + 255) / 256;

struct Smem {
  uint8_t flag[kWinWords * 32];
  uint32_t bits[kWinWords];
  int pre[kWinWords];
  int red[2][8];
  int wsum[8];
};

// 256 threads; vals(e) = neighbour row of entry e = row * 27 + j of the tile
// (-1 none / past the row count).  Writes halo_rows[0..H), *halo_n, lnbr[128*27].
template <typename F>
__device__ __forceinline__ void build_tile(F vals_of, Smem& s, int* __restrict__ hr, int* __restrict__ hn,
                                           int16_t* __restrict__ ln) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int vals[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int e = tid + 256 * k;
    vals[k] = e < kRows * kOff ? vals_of(e) : -1;
  }
  int lo = INT_MAX, hi = -1;
#pragma unroll
  for (int k = 0; k < kPer; ++k)
    if (vals[k] >= 0) {
      lo = min(lo, vals[k]);
      hi = max(hi, vals[k]);
    }
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(~0u, lo, o));
    hi = max(hi, __shfl_xor_sync(~0u, hi, o));
  }
  if (lane == 0) {
    s.red[0][warp] = lo;
    s.red[1][warp] = hi;
  }
  __syncthreads();
  lo = INT_MAX;
  hi = -1;
  for (int w = 0; w < 8; ++w) {
    lo = min(lo, s.red[0][w]);
    hi = max(hi, s.red[1][w]);
  }
  const bool win = hi >= 0 && hi - lo < kWinWords * 32;
  const int nw = win ? ((hi - lo) >> 5) + 1 : 0;
  // mark the window rows with plain byte stores (equal values, no atomics),
  // then fold 32 flags into one bitmap word per thread
  for (int i = tid; i < nw * 2; i += 256) reinterpret_cast<uint4*>(s.flag)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  if (win) {
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if (vals[k] >= 0) s.flag[vals[k] - lo] = 1;
  }
  __syncthreads();
  for (int w = tid; w < nw; w += 256) {
    const uint4 a = reinterpret_cast<const uint4*>(s.flag)[2 * w];
    const uint4 b = reinterpret_cast<const uint4*>(s.flag)[2 * w + 1];
    const uint32_t q[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t v = q[i];  // bytes are 0/1: gather bit 0 of each byte
      m |= ((v & 1u) | ((v >> 7) & 2u) | ((v >> 14) & 4u) | ((v >> 21) & 8u)) << (4 * i);
    }
    s.bits[w] = m;
  }
  __syncthreads();
  // exclusive scan of the word popcounts and the sorted halo list: word w's
  // set bits are rows lo + 32 w + b
  int H = 0;
  for (int base = 0; base < nw; base += 256) {
    const int w = base + tid;
    const uint32_t bw = w < nw ? s.bits[w] : 0u;
    const int c = __popc(bw);
    int incl = c;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(~0u, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s.wsum[warp] = incl;
    __syncthreads();
    int woff = 0, rtot = 0;
    for (int i = 0; i < 8; ++i) {
      if (i < warp) woff += s.wsum[i];
      rtot += s.wsum[i];
    }
    int rk = H + woff + incl - c;
    if (w < nw) s.pre[w] = rk;
    uint32_t bits = bw;
    while (bits && rk < kHmax) {
      hr[rk++] = lo + w * 32 + (__ffs(bits) - 1);
      bits &= bits - 1;
    }
    H += rtot;
    __syncthreads();
  }
  if (tid == 0) *hn = win ? min(H, kHmax) : 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int e = tid + 256 * k;
    if (e >= kRows * kOff) break;
    const int v = vals[k];
    int o = -1;
    if (v >= 0) {
      o = -2;
      if (win) {
        const int dd = v - lo;
        const int rk = s.pre[dd >> 5] + __popc(s.bits[dd >> 5] & ((1u << (dd & 31)) - 1u));
        if (rk < kHmax) o = rk;
      }
    }
    ln[e] = (int16_t)o;
  }
  __syncthreads();
}

}  // namespace halob
}  // namespace fpvs
