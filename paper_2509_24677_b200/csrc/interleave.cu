// (1) 3-D volume-preserving interleave / deinterleave (space-to-depth and
// depth-to-space), replacing pkg/src/froxelpvs/interleave.py:54-85.
//
// Dense grids are (B, Nx, Ny, Nz) C-order (z fastest); cells are
// (B, X, Y, Z, d^3) with channel k = lx + d*(ly + d*lz).  For dense input a
// CTA stages the d*d z-rows of one (bx, by) column slab in shared memory so
// both the global read (runs of Nz along z) and the global write (runs of
// Z*d^3 along (bz, k)) are coalesced; the cast to f32/bf16 is fused.  Packed
// input (FPVS bits, x-fastest) is read byte-wise through L1: at 1 bit per
// froxel it is 1/32 of the f32 output bytes.
#include "common.cuh"
#include "tc_ptx.cuh"

namespace fpvs {

constexpr int kIlSmemElems = 12288;  // 48 KB of f32 staging

// element conversion of the fused cast; same type = exact raw permutation
// (any 1/2/4/8-byte element, e.g. float64 or int64 grids, moves unchanged)
template <typename To, typename Ti> __device__ __forceinline__ To cvt(Ti v) { return from_f32<To>(to_f32<Ti>(v)); }
template <> __device__ __forceinline__ uint8_t cvt<uint8_t, uint8_t>(uint8_t v) { return v; }
template <> __device__ __forceinline__ uint16_t cvt<uint16_t, uint16_t>(uint16_t v) { return v; }
template <> __device__ __forceinline__ uint32_t cvt<uint32_t, uint32_t>(uint32_t v) { return v; }
template <> __device__ __forceinline__ unsigned long long cvt<unsigned long long, unsigned long long>(
    unsigned long long v) { return v; }
template <> __device__ __forceinline__ float cvt<float, float>(float v) { return v; }
template <> __device__ __forceinline__ double cvt<double, double>(double v) { return v; }
template <typename T> __device__ __forceinline__ bool nonzero(T v) { return v != T(0); }
template <> __device__ __forceinline__ bool nonzero<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v) != 0.f;
}
template <> __device__ __forceinline__ bool nonzero<float>(float v) { return v != 0.f; }
template <> __device__ __forceinline__ bool nonzero<double>(double v) { return v != 0.0; }

template <typename Tin, typename Tout>
__global__ void interleave_dense_kernel(const Tin* __restrict__ in, int B, int Nx, int Ny, int Nz,
                                        int d, int zc, Tout* __restrict__ out,
                                        uint8_t* __restrict__ cell_active) {
  extern __shared__ unsigned char smem_raw[];
  Tin* tile = reinterpret_cast<Tin*>(smem_raw);
  const int X = Nx / d, Y = Ny / d, Z = Nz / d;
  const int nzc = (Z + zc - 1) / zc;
  const int d3 = d * d * d;
  long long blk = blockIdx.x;
  const int zi = blk % nzc; blk /= nzc;
  const int by = blk % Y; blk /= Y;
  const int bx = blk % X; blk /= X;
  const int b = (int)blk;
  const int bz0 = zi * zc;
  const int nbz = min(zc, Z - bz0);
  const int zlen = nbz * d;
  // stage d*d rows of zlen froxels: tile[(lx*d + ly)*zlen + zz]
  for (int t = threadIdx.x; t < d * d * zlen; t += blockDim.x) {
    int zz = t % zlen, r = t / zlen;
    int ly = r % d, lx = r / d;
    long long src = (((long long)b * Nx + bx * d + lx) * Ny + by * d + ly) * Nz + bz0 * d + zz;
    tile[t] = in[src];
  }
  __syncthreads();
  long long obase = ((((long long)b * X + bx) * Y + by) * Z + bz0) * d3;
  for (int t = threadIdx.x; t < nbz * d3; t += blockDim.x) {
    int k = t % d3, bzl = t / d3;
    int lx = k % d, ly = (k / d) % d, lz = k / (d * d);
    out[obase + t] = cvt<Tout, Tin>(tile[(lx * d + ly) * zlen + bzl * d + lz]);
  }
  if (cell_active) {
    for (int bzl = threadIdx.x; bzl < nbz; bzl += blockDim.x) {
      uint8_t any = 0;
      for (int lx = 0; lx < d && !any; ++lx)
        for (int ly = 0; ly < d && !any; ++ly)
          for (int lz = 0; lz < d; ++lz)
            if (nonzero<Tin>(tile[(lx * d + ly) * zlen + bzl * d + lz])) { any = 1; break; }
      cell_active[(((long long)b * X + bx) * Y + by) * Z + bz0 + bzl] = any;
    }
  }
}

__device__ __forceinline__ int read_bit(const uint8_t* __restrict__ bits, int b, int x, int y, int z,
                                        int Nx, int Ny, int Nz) {
  return (__ldg(bits + bit_byte(b, x, y, z, Nx, Ny, Nz)) >> (x & 7)) & 1;
}

template <typename Tout>
__global__ void interleave_bits_kernel(const uint8_t* __restrict__ bits, int B, int Nx, int Ny, int Nz,
                                       int d, Tout* __restrict__ out) {
  const int X = Nx / d, Y = Ny / d, Z = Nz / d, d3 = d * d * d;
  const long long total = (long long)B * X * Y * Z * d3;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int k = t % d3;
    long long c = t / d3;
    int bz = c % Z; c /= Z;
    int by = c % Y; c /= Y;
    int bx = c % X;
    int b = (int)(c / X);
    int lx = k % d, ly = (k / d) % d, lz = k / (d * d);
    out[t] = from_f32<Tout>((float)read_bit(bits, b, bx * d + lx, by * d + ly, bz * d + lz, Nx, Ny, Nz));
  }
}

// any bit of the d^3 block of cell (b, bx, by, bz) set?  (all d*d row loads
// issued before the test, no early exit, for memory-level parallelism)
__device__ __forceinline__ uint8_t block_any(const uint8_t* __restrict__ bits, int b, int bx, int by, int bz, int d,
                                             int Nx, int Ny, int Nz) {
  const int x0 = bx * d;
  uint32_t acc = 0;
  for (int lz = 0; lz < d; ++lz)
    for (int ly = 0; ly < d; ++ly) {
      const uint8_t* row = bits + bit_byte(b, 0, by * d + ly, bz * d + lz, Nx, Ny, Nz);
      int x = x0;
      while (x < x0 + d) {
        int sh = x & 7;
        int nb = min(8 - sh, x0 + d - x);
        uint32_t m = ((1u << nb) - 1u) << sh;
        acc |= __ldg(row + (x >> 3)) & m;
        x += nb;
      }
    }
  return acc ? 1 : 0;
}

// Active flags of cells from packed bits.  A block covers 32 (bx) x 32 (bz)
// cells of one (b, by) slab: lanes walk x so the bytes a warp reads per
// froxel row are contiguous, then the flags are transposed through shared
// memory so the C-order (z-fastest) output is written in 32-byte runs.
__global__ void __launch_bounds__(256) cell_active_bits_kernel(const uint8_t* __restrict__ bits, int B, int Nx, int Ny,
                                                               int Nz, int d, uint8_t* __restrict__ cell_active) {
  __shared__ uint8_t flag[32][33];
  const int X = Nx / d, Y = Ny / d, Z = Nz / d;
  const int nxt = (X + 31) / 32, nzt = (Z + 31) / 32;
  long long blk = blockIdx.x;
  const int zt = blk % nzt; blk /= nzt;
  const int xt = blk % nxt; blk /= nxt;
  const int by = blk % Y;
  const int b = (int)(blk / Y);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int bx = xt * 32 + lane;
  for (int i = 0; i < 4; ++i) {
    const int bzl = w + 8 * i, bz = zt * 32 + bzl;
    uint8_t f = 0;
    if (bx < X && bz < Z) f = block_any(bits, b, bx, by, bz, d, Nx, Ny, Nz);
    flag[lane][bzl] = f;
  }
  __syncthreads();
  const int bxl = threadIdx.x >> 3, zq = (threadIdx.x & 7) * 4;
  const int ox = xt * 32 + bxl;
  if (ox < X) {
    const long long row = (((long long)b * X + ox) * Y + by) * Z;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int oz = zt * 32 + zq + q;
      if (oz < Z) cell_active[row + oz] = flag[bxl][zq + q];
    }
  }
}

template <typename Tin, typename Tout>
__global__ void deinterleave_dense_kernel(const Tin* __restrict__ in, int B, int X, int Y, int Z, int d,
                                          Tout* __restrict__ out) {
  const int Nx = X * d, Ny = Y * d, Nz = Z * d, d3 = d * d * d;
  const long long total = (long long)B * Nx * Ny * Nz;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long r = t;
    int z = r % Nz; r /= Nz;
    int y = r % Ny; r /= Ny;
    int x = r % Nx;
    int b = (int)(r / Nx);
    long long cell = (((long long)b * X + x / d) * Y + y / d) * Z + z / d;
    int k = x % d + d * (y % d + d * (z % d));
    out[t] = cvt<Tout, Tin>(in[cell * d3 + k]);
  }
}

// threshold comparison in the input's own precision (numpy's `values >= tau`
// under NEP 50: a float32 array compares in float32, float64 in float64)
template <typename Tin, typename Tc> __device__ __forceinline__ Tc cmp_val(Tin v) { return (Tc)to_f32<Tin>(v); }
template <> __device__ __forceinline__ double cmp_val<double, double>(double v) { return v; }

// one output byte = 8 x-consecutive froxels of one (b, y, z) row
template <typename Tin, typename Tc>
__global__ void deinterleave_thresh_kernel(const Tin* __restrict__ in, int B, int X, int Y, int Z, int d,
                                           Tc tau, uint8_t* __restrict__ out) {
  const int Nx = X * d, Ny = Y * d, Nz = Z * d, d3 = d * d * d;
  const int rb = Nx >> 3;
  const long long total = (long long)B * Nz * Ny * rb;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long r = t;
    int xb = r % rb; r /= rb;
    int y = r % Ny; r /= Ny;
    int z = r % Nz;
    int b = (int)(r / Nz);
    uint32_t byte = 0;
    for (int i = 0; i < 8; ++i) {
      int x = xb * 8 + i;
      long long cell = (((long long)b * X + x / d) * Y + y / d) * Z + z / d;
      int k = x % d + d * (y % d + d * (z % d));
      if (cmp_val<Tin, Tc>(in[cell * d3 + k]) >= tau) byte |= 1u << i;
    }
    out[t] = (uint8_t)byte;
  }
}

template <typename Tout>
__device__ __forceinline__ void store8(Tout* dst, const float (&v)[8]);
template <>
__device__ __forceinline__ void store8<__nv_bfloat16>(__nv_bfloat16* dst, const float (&v)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
}
template <>
__device__ __forceinline__ void store8<float>(float* dst, const float (&v)[8]) {
  reinterpret_cast<float4*>(dst)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(dst)[1] = make_float4(v[4], v[5], v[6], v[7]);
}

// Sparse interleave: one thread per (active row, group of 8 channels); the
// group's bits come from a few L1-cached bytes and leave as one 16-byte
// (bf16) / 32-byte (f32) store.
template <typename Tout>
__global__ void gather_cells_bits_kernel(const uint8_t* __restrict__ bits, int Nx, int Ny, int Nz, int d,
                                         const int4* __restrict__ coords, const int* __restrict__ n_dev,
                                         int cap, Tout* __restrict__ x, int ldx) {
  const int n = min(*n_dev, cap);
  const int d3 = d * d * d;
  const int groups = (d3 + 7) / 8;
  const bool vec = (d3 % 8 == 0) && (ldx % 8 == 0);
  const long long total = (long long)n * groups;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int g = t % groups;
    const long long i = t / groups;
    const int4 c = coords[i];
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = g * 8 + q;
      v[q] = 0.f;
      if (k < d3) {
        const int lx = k % d, ly = (k / d) % d, lz = k / (d * d);
        v[q] = (float)read_bit(bits, c.x, c.y * d + lx, c.z * d + ly, c.w * d + lz, Nx, Ny, Nz);
      }
    }
    Tout* dst = x + i * ldx + g * 8;
    if (vec) {
      store8<Tout>(dst, v);
    } else {
      for (int q = 0; q < 8 && g * 8 + q < d3; ++q) dst[q] = from_f32<Tout>(v[q]);
    }
  }
}

// ===========================================================================
// Tiled, 128-bit vectorised interleave / deinterleave for d in {1, 2, 4, 8}
// (north_star (1); replaces interleave.py:54-85).
//
// For one (b, bx, by) column slab the interleaved output is the contiguous
// run [z][m] of Nz * d^2 elements (m = lx + d * ly, z = bz * d + lz, so
// k = m + d^2 * lz), and the dense input is the d^2 rows (lx, ly) of Nz
// z-contiguous elements: interleave is a [d^2][Nz] -> [Nz][d^2] transpose
// per slab.  A CTA stages a [d^2][zt] tile in shared memory with 16-byte
// loads along z and writes the output with 16-byte stores along m (the cast
// to the output type fused on the way); deinterleave runs the same tile the
// other way round.  Every HBM byte moves once in full 32-byte sectors.
// ===========================================================================
constexpr int kTileBytes = 16384;  // staging per CTA (several CTAs per SM)
constexpr int kTileThreads = 256;

template <int BYTES> struct VecT;
template <> struct VecT<16> { using T = uint4; };
template <> struct VecT<8> { using T = uint2; };
template <> struct VecT<4> { using T = uint32_t; };
template <> struct VecT<2> { using T = uint16_t; };
template <> struct VecT<1> { using T = uint8_t; };

// N elements as one vector access (N * sizeof(T) <= 16) or 16-byte pieces
template <typename T, int N>
__device__ __forceinline__ void vload(const T* src, T (&v)[N]) {
  constexpr int BYTES = N * (int)sizeof(T);
  if constexpr (BYTES <= 16) {
    using V = typename VecT<BYTES>::T;
    const V w = *reinterpret_cast<const V*>(src);
    memcpy(v, &w, sizeof(V));
  } else {
    constexpr int P = 16 / sizeof(T);
#pragma unroll
    for (int i = 0; i < N / P; ++i) {
      const uint4 w = reinterpret_cast<const uint4*>(src)[i];
      memcpy(v + i * P, &w, 16);
    }
  }
}
template <typename T, int N>
__device__ __forceinline__ void vstore(T* dst, const T (&v)[N]) {
  constexpr int BYTES = N * (int)sizeof(T);
  if constexpr (BYTES <= 16) {
    using V = typename VecT<BYTES>::T;
    V w;
    memcpy(&w, v, sizeof(V));
    *reinterpret_cast<V*>(dst) = w;
  } else {
    constexpr int P = 16 / sizeof(T);
#pragma unroll
    for (int i = 0; i < N / P; ++i) {
      uint4 w;
      memcpy(&w, v + i * P, 16);
      reinterpret_cast<uint4*>(dst)[i] = w;
    }
  }
}

constexpr int cmin(int a, int b) { return a < b ? a : b; }

// CTA = (slab b*X*Y + bx*Y + by, z chunk); tile[r][zt + pad], r = lx * D + ly
template <typename Tin, typename Tout, int D>
__global__ void __launch_bounds__(kTileThreads) il_tile_kernel(const Tin* __restrict__ in, int Nx, int Ny, int Nz,
                                                               int zt, Tout* __restrict__ out,
                                                               uint8_t* __restrict__ cell_active) {
  constexpr int R = D * D, M = D * D;
  constexpr int VI = 16 / sizeof(Tin);                  // input elements per 16-byte load
  constexpr int VO = cmin(M, (int)(16 / sizeof(Tout)));  // output elements per store
  extern __shared__ __align__(128) unsigned char il_smem[];
  Tin* tile = reinterpret_cast<Tin*>(il_smem);
  const int X = Nx / D, Y = Ny / D, Z = Nz / D;
  const int ld = zt + VI;  // padded row (keeps 16-byte alignment, shifts banks)
  const int nzc = (Nz + zt - 1) / zt;
  const long long slab = blockIdx.x / nzc;
  const int z0 = (int)(blockIdx.x % nzc) * zt;
  const int zl = min(zt, Nz - z0);
  const int by = (int)(slab % Y);
  const long long bxb = slab / Y;  // b * X + bx
  const int bx = (int)(bxb % X);
  const long long b = bxb / X;
  // ---- load: d^2 rows x zl, 16-byte vectors along z
  const int nv = zl / VI;
  for (int t = threadIdx.x; t < R * nv; t += kTileThreads) {
    const int r = t / nv, zv = t - r * nv;
    const int lx = r / D, ly = r - lx * D;
    const Tin* src = in + ((b * Nx + bx * D + lx) * Ny + by * D + ly) * (long long)Nz + z0 + zv * VI;
    Tin v[VI];
    vload<Tin, VI>(src, v);
    vstore<Tin, VI>(tile + r * ld + zv * VI, v);
  }
  __syncthreads();
  // ---- store: output run [z][m] of this slab chunk, VO elements per thread
  constexpr int MV = M / VO;
  Tout* obase = out + (((b * X + bx) * (long long)Y + by) * Z) * (long long)(D * D * D) + (long long)z0 * M;
  for (int t = threadIdx.x; t < zl * MV; t += kTileThreads) {
    const int z = t / MV, m0 = (t - z * MV) * VO;
    Tout v[VO];
#pragma unroll
    for (int q = 0; q < VO; ++q) {
      const int m = m0 + q, lx = m % D, ly = m / D;
      v[q] = cvt<Tout, Tin>(tile[(lx * D + ly) * ld + z]);
    }
    vstore<Tout, VO>(obase + (long long)z * M + m0, v);
  }
  if (cell_active) {
    const int nbz = zl / D;
    for (int c = threadIdx.x; c < nbz; c += kTileThreads) {
      bool any = false;
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int lz = 0; lz < D; ++lz) any |= nonzero<Tin>(tile[r * ld + c * D + lz]);
      cell_active[((b * X + bx) * (long long)Y + by) * Z + z0 / D + c] = any ? 1 : 0;
    }
  }
}

// packed bits -> interleaved cells: thread = VO consecutive channels m of one
// (slab, z); the bits come from L1-cached bytes (1/32 of the f32 output)
template <typename Tout, int D>
__global__ void __launch_bounds__(kTileThreads) il_bits_kernel(const uint8_t* __restrict__ bits, int B, int Nx, int Ny,
                                                               int Nz, Tout* __restrict__ out) {
  constexpr int M = D * D;
  constexpr int VO = cmin(M, (int)(16 / sizeof(Tout)));
  constexpr int MV = M / VO;
  const int X = Nx / D, Y = Ny / D;
  const long long rowb = Nx >> 3;
  const long long total = (long long)B * X * Y * Nz * MV;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int mv = (int)(t % MV);
    long long r = t / MV;
    const int z = (int)(r % Nz);
    r /= Nz;
    const int by = (int)(r % Y);
    r /= Y;
    const int bx = (int)(r % X);
    const long long b = r / X;
    Tout v[VO];
#pragma unroll
    for (int q = 0; q < VO; ++q) {
      const int m = mv * VO + q, lx = m % D, ly = m / D;
      const int x = bx * D + lx;
      const uint8_t byte = __ldg(bits + ((b * Nz + z) * Ny + by * D + ly) * rowb + (x >> 3));
      v[q] = from_f32<Tout>((float)((byte >> (x & 7)) & 1));
    }
    // output index of (b, bx, by, z, m) = (slab * Nz + z) * M + m
    vstore<Tout, VO>(out + (((b * X + bx) * (long long)Y + by) * Nz + z) * M + mv * VO, v);
  }
}

// deinterleave (dense): [z][m] runs in -> d^2 z-rows out, 16-byte both ways
template <typename Tin, typename Tout, int D>
__global__ void __launch_bounds__(kTileThreads) deil_tile_kernel(const Tin* __restrict__ in, int X, int Y, int Z,
                                                                 int zt, Tout* __restrict__ out) {
  constexpr int R = D * D, M = D * D;
  constexpr int VI = cmin(M, (int)(16 / sizeof(Tin)));
  constexpr int VO = 16 / sizeof(Tout);
  extern __shared__ __align__(128) unsigned char il_smem[];
  Tout* tile = reinterpret_cast<Tout*>(il_smem);
  const int Nx = X * D, Ny = Y * D, Nz = Z * D;
  const int ld = zt + VO;
  const int nzc = (Nz + zt - 1) / zt;
  const long long slab = blockIdx.x / nzc;
  const int z0 = (int)(blockIdx.x % nzc) * zt;
  const int zl = min(zt, Nz - z0);
  const int by = (int)(slab % Y);
  const long long bxb = slab / Y;
  const int bx = (int)(bxb % X);
  const long long b = bxb / X;
  constexpr int MV = M / VI;
  const Tin* ibase = in + slab * (long long)Z * (D * D * D) + (long long)z0 * M;
  for (int t = threadIdx.x; t < zl * MV; t += kTileThreads) {
    const int z = t / MV, m0 = (t - z * MV) * VI;
    Tin v[VI];
    vload<Tin, VI>(ibase + (long long)z * M + m0, v);
#pragma unroll
    for (int q = 0; q < VI; ++q) {
      const int m = m0 + q, lx = m % D, ly = m / D;
      tile[(lx * D + ly) * ld + z] = cvt<Tout, Tin>(v[q]);
    }
  }
  __syncthreads();
  const int nv = zl / VO;
  for (int t = threadIdx.x; t < R * nv; t += kTileThreads) {
    const int r = t / nv, zv = t - r * nv;
    const int lx = r / D, ly = r - lx * D;
    Tout v[VO];
    vload<Tout, VO>(tile + r * ld + zv * VO, v);
    vstore<Tout, VO>(out + ((b * Nx + bx * D + lx) * Ny + by * D + ly) * (long long)Nz + z0 + zv * VO, v);
  }
}

// deinterleave + [value >= tau] -> packed bits: thread = one 32-bit word of
// a (b, z, y) row (32 consecutive x); per cell it loads the d consecutive
// channels lx = 0..d-1 (k = lx + d (ly + d lz)) as one vector
template <typename Tin, typename Tc, int D>
__global__ void __launch_bounds__(kTileThreads) deil_bits_kernel(const Tin* __restrict__ in, int B, int X, int Y,
                                                                 int Z, Tc tau, uint32_t* __restrict__ out) {
  constexpr int D3 = D * D * D;
  const int Nx = X * D, Ny = Y * D, Nz = Z * D;
  const int words = Nx >> 5;
  const long long total = (long long)B * Nz * Ny * words;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int w = (int)(t % words);
    long long r = t / words;
    const int y = (int)(r % Ny);
    r /= Ny;
    const int z = (int)(r % Nz);
    const long long b = r / Nz;
    const int by = y / D, ly = y - by * D, bz = z / D, lz = z - bz * D;
    const int k0 = D * (ly + D * lz);
    uint32_t word = 0;
#pragma unroll
    for (int c = 0; c < 32 / D; ++c) {
      const int bx = (w * 32) / D + c;
      Tin v[D];
      vload<Tin, D>(in + (((b * X + bx) * (long long)Y + by) * Z + bz) * D3 + k0, v);
#pragma unroll
      for (int lx = 0; lx < D; ++lx)
        if (cmp_val<Tin, Tc>(v[lx]) >= tau) word |= 1u << (c * D + lx);
    }
    out[t] = word;
  }
}

// ---- persistent, TMA-fed versions (the ones the entry points launch) -------
// A CTA loops over (slab, z chunk) tiles with two shared-memory buffers: one
// thread issues the next tile's bulk copies (cp.async.bulk, one per
// contiguous run) while all threads transpose + cast + store the current one,
// so HBM reads stay in flight across the store phase.
template <int PAD_BYTES, typename T> constexpr int pad_elems() { return PAD_BYTES / (int)sizeof(T); }

template <typename Tin, typename Tout, int D>
__global__ void __launch_bounds__(kTileThreads) il_tma_kernel(const Tin* __restrict__ in, int Nx, int Ny, int Nz,
                                                              int zt, long long ntiles, Tout* __restrict__ out,
                                                              uint8_t* __restrict__ cell_active) {
  using namespace tc;
  constexpr int R = D * D, M = D * D;
  constexpr int VO = cmin(M, (int)(16 / sizeof(Tout)));
  constexpr int MV = M / VO;
  extern __shared__ __align__(128) unsigned char il_smem[];
  __shared__ __align__(8) uint64_t bars[2];
  // rows padded by 32 bytes: the two m halves a warp reads sit 16 banks apart
  const int ld = zt + pad_elems<32, Tin>();
  Tin* buf0 = reinterpret_cast<Tin*>(il_smem);
  const int X = Nx / D, Y = Ny / D, Z = Nz / D;
  const int nzc = (Nz + zt - 1) / zt;
  auto issue = [&](long long t, int bi) {
    const long long slab = t / nzc;
    const int z0 = (int)(t % nzc) * zt, zl = min(zt, Nz - z0);
    const int by = (int)(slab % Y);
    const long long bxb = slab / Y;
    const int bx = (int)(bxb % X);
    const long long b = bxb / X;
    const uint32_t bar = smem_u32(&bars[bi]);
    mbar_arrive_expect_tx(bar, (uint32_t)(R * zl * sizeof(Tin)));
    Tin* dst = buf0 + (size_t)bi * R * ld;
    for (int r = 0; r < R; ++r) {
      const int lx = r / D, ly = r - lx * D;
      bulk_g2s(smem_u32(dst + r * ld), in + ((b * Nx + bx * D + lx) * Ny + by * D + ly) * (long long)Nz + z0,
               (uint32_t)(zl * sizeof(Tin)), bar);
    }
  };
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bars[0]), 1);
    mbar_init(smem_u32(&bars[1]), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if ((long long)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    if ((long long)blockIdx.x + gridDim.x < ntiles) issue(blockIdx.x + gridDim.x, 1);
  }
  int it = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int bi = it & 1;
    mbar_wait(smem_u32(&bars[bi]), (it >> 1) & 1);
    const Tin* tile = buf0 + (size_t)bi * R * ld;
    const long long slab = t / nzc;
    const int z0 = (int)(t % nzc) * zt, zl = min(zt, Nz - z0);
    Tout* obase = out + slab * (long long)Z * (D * D * D) + (long long)z0 * M;
    for (int u = threadIdx.x; u < zl * MV; u += kTileThreads) {
      const int z = u / MV, m0 = (u - z * MV) * VO;
      Tout v[VO];
#pragma unroll
      for (int q = 0; q < VO; ++q) {
        const int m = m0 + q, lx = m % D, ly = m / D;
        v[q] = cvt<Tout, Tin>(tile[(lx * D + ly) * ld + z]);
      }
      vstore<Tout, VO>(obase + (long long)z * M + m0, v);
    }
    if (cell_active) {
      for (int c = threadIdx.x; c < zl / D; c += kTileThreads) {
        bool any = false;
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int lz = 0; lz < D; ++lz) any |= nonzero<Tin>(tile[r * ld + c * D + lz]);
        cell_active[slab * Z + z0 / D + c] = any ? 1 : 0;
      }
    }
    __syncthreads();  // every thread is done with this buffer
    if (threadIdx.x == 0 && t + 2LL * gridDim.x < ntiles) issue(t + 2LL * gridDim.x, bi);
  }
}

// deinterleave: the slab chunk's [z][m] run lands with ONE bulk copy, is
// transposed to [r][z] in shared memory, and leaves as 16-byte row stores
template <typename Tin, typename Tout, int D>
__global__ void __launch_bounds__(kTileThreads) deil_tma_kernel(const Tin* __restrict__ in, int X, int Y, int Z,
                                                                int zt, long long ntiles, Tout* __restrict__ out) {
  using namespace tc;
  constexpr int R = D * D, M = D * D;
  constexpr int VI = cmin(M, (int)(16 / sizeof(Tin)));
  constexpr int MV = M / VI;
  constexpr int VO = 16 / sizeof(Tout);
  extern __shared__ __align__(128) unsigned char il_smem[];
  __shared__ __align__(8) uint64_t bars[2];
  const int Nx = X * D, Ny = Y * D, Nz = Z * D;
  const int ldo = zt + pad_elems<32, Tout>();
  Tin* in0 = reinterpret_cast<Tin*>(il_smem);                        // 2 x [zt][M]
  Tout* tr = reinterpret_cast<Tout*>(il_smem + 2 * (size_t)zt * M * sizeof(Tin));  // [R][ldo]
  const int nzc = (Nz + zt - 1) / zt;
  auto issue = [&](long long t, int bi) {
    const long long slab = t / nzc;
    const int z0 = (int)(t % nzc) * zt, zl = min(zt, Nz - z0);
    const uint32_t bar = smem_u32(&bars[bi]);
    const uint32_t bytes = (uint32_t)((size_t)zl * M * sizeof(Tin));
    mbar_arrive_expect_tx(bar, bytes);
    bulk_g2s(smem_u32(in0 + (size_t)bi * zt * M), in + slab * (long long)Z * (D * D * D) + (long long)z0 * M, bytes,
             bar);
  };
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bars[0]), 1);
    mbar_init(smem_u32(&bars[1]), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if ((long long)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    if ((long long)blockIdx.x + gridDim.x < ntiles) issue(blockIdx.x + gridDim.x, 1);
  }
  int it = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int bi = it & 1;
    mbar_wait(smem_u32(&bars[bi]), (it >> 1) & 1);
    const Tin* src = in0 + (size_t)bi * zt * M;
    const long long slab = t / nzc;
    const int z0 = (int)(t % nzc) * zt, zl = min(zt, Nz - z0);
    for (int u = threadIdx.x; u < zl * MV; u += kTileThreads) {
      const int z = u / MV, m0 = (u - z * MV) * VI;
      Tin v[VI];
      vload<Tin, VI>(src + z * M + m0, v);
#pragma unroll
      for (int q = 0; q < VI; ++q) {
        const int m = m0 + q, lx = m % D, ly = m / D;
        tr[(lx * D + ly) * ldo + z] = cvt<Tout, Tin>(v[q]);
      }
    }
    __syncthreads();  // the transpose is complete; the input buffer is free
    if (threadIdx.x == 0 && t + 2LL * gridDim.x < ntiles) issue(t + 2LL * gridDim.x, bi);
    const int by = (int)(slab % Y);
    const long long bxb = slab / Y;
    const int bx = (int)(bxb % X);
    const long long b = bxb / X;
    const int nv = zl / VO;
    for (int u = threadIdx.x; u < R * nv; u += kTileThreads) {
      const int r = u / nv, zv = u - r * nv;
      const int lx = r / D, ly = r - lx * D;
      Tout v[VO];
      vload<Tout, VO>(tr + r * ldo + zv * VO, v);
      vstore<Tout, VO>(out + ((b * Nx + bx * D + lx) * Ny + by * D + ly) * (long long)Nz + z0 + zv * VO, v);
    }
    __syncthreads();  // the transpose buffer is read out
  }
}

// packed bits -> cells: CTA = (b, by, z chunk) over every bx: the d rows x zt
// bit-rows (N_x / 8 bytes each) are staged in shared memory with 16-byte
// loads, then every slab's [z][m] run is written with 16-byte stores
template <typename Tout, int D>
__global__ void __launch_bounds__(kTileThreads) il_bits_tile_kernel(const uint8_t* __restrict__ bits, int Nx, int Ny,
                                                                    int Nz, int zt, Tout* __restrict__ out) {
  constexpr int M = D * D;
  constexpr int VO = cmin(M, (int)(16 / sizeof(Tout)));
  constexpr int MV = M / VO;
  extern __shared__ __align__(128) unsigned char il_smem[];
  const int X = Nx / D, Y = Ny / D, Z = Nz / D;
  const int rowb = Nx >> 3;
  const int nzc = (Nz + zt - 1) / zt;
  long long blk = blockIdx.x;
  const int zi = (int)(blk % nzc);
  blk /= nzc;
  const int by = (int)(blk % Y);
  const long long b = blk / Y;
  const int z0 = zi * zt, zl = min(zt, Nz - z0);
  // stage rows (ly, z): bytes of bit-row (b, z0 + z, by * D + ly), rows
  // 4 bytes apart beyond N_x / 8 so a warp's byte reads at consecutive z hit
  // distinct banks
  const int nv = rowb / 16, rs = rowb + 4;
  for (int u = threadIdx.x; u < D * zl * nv; u += kTileThreads) {
    const int v = u % nv, rz = u / nv;
    const int z = rz % zl, ly = rz / zl;
    const uint4 w = reinterpret_cast<const uint4*>(bits + ((b * Nz + z0 + z) * (long long)Ny + by * D + ly) * rowb)[v];
    uint32_t* d32 = reinterpret_cast<uint32_t*>(il_smem + (ly * zt + z) * rs + 16 * v);
    d32[0] = w.x; d32[1] = w.y; d32[2] = w.z; d32[3] = w.w;
  }
  __syncthreads();
  for (int u = threadIdx.x; u < X * zl * MV; u += kTileThreads) {
    const int mv = u % MV;
    const int z = (u / MV) % zl;
    const int bx = u / (MV * zl);
    Tout v[VO];
#pragma unroll
    for (int q = 0; q < VO; ++q) {
      const int m = mv * VO + q, lx = m % D, ly = m / D;
      const int x = bx * D + lx;
      v[q] = from_f32<Tout>((float)((il_smem[(ly * zt + z) * rs + (x >> 3)] >> (x & 7)) & 1));
    }
    vstore<Tout, VO>(out + (((b * X + bx) * (long long)Y + by) * Z) * (D * D * D) + (long long)(z0 + z) * M + mv * VO,
                     v);
  }
}

template <typename Tin, typename Tout, int D>
int launch_il_tile(const void* in, int B, int Nx, int Ny, int Nz, void* out, uint8_t* cell_active, cudaStream_t s) {
  constexpr int VI = 16 / sizeof(Tin);
  int zt = kTileBytes / (D * D * (int)sizeof(Tin));
  zt -= zt % (VI > D ? VI : D);
  if (zt > Nz) zt = Nz;
  const int nzc = (Nz + zt - 1) / zt;
  const long long ntiles = (long long)B * (Nx / D) * (Ny / D) * nzc;
  const size_t smem = 2 * (size_t)D * D * (zt + pad_elems<32, Tin>()) * sizeof(Tin);
  set_smem_once<il_tma_kernel<Tin, Tout, D>>(64 * 1024);
  const long long grid = ntiles < (long long)kNumSMs * 6 ? ntiles : (long long)kNumSMs * 6;
  il_tma_kernel<Tin, Tout, D><<<(unsigned)grid, kTileThreads, smem, s>>>((const Tin*)in, Nx, Ny, Nz, zt, ntiles,
                                                                         (Tout*)out, cell_active);
  return FPVS_OK;
}

// z granularity of a deinterleave tile: whole 16-byte output vectors along z
// and 16-byte aligned bulk copies of the [z][m] input run
template <typename Tin, typename Tout, int D>
constexpr int deil_zalign() {
  constexpr int vo = 16 / sizeof(Tout);
  constexpr int run = D * D * (int)sizeof(Tin);  // bytes per z in the input run
  constexpr int need = run >= 16 ? 1 : 16 / run;
  constexpr int a = vo > D ? vo : D;
  return a > need ? a : need;
}

template <typename Tin, typename Tout, int D>
int launch_deil_tile(const void* in, int B, int X, int Y, int Z, void* out, cudaStream_t s) {
  const int Nz = Z * D;
  const int za = deil_zalign<Tin, Tout, D>();
  int zt = kTileBytes / (D * D * (int)sizeof(Tout));
  zt -= zt % za;
  if (zt > Nz) zt = Nz;
  const int nzc = (Nz + zt - 1) / zt;
  const long long ntiles = (long long)B * X * Y * nzc;
  const size_t smem = 2 * (size_t)zt * D * D * sizeof(Tin) + (size_t)D * D * (zt + pad_elems<32, Tout>()) * sizeof(Tout);
  set_smem_once<deil_tma_kernel<Tin, Tout, D>>(96 * 1024);
  const long long grid = ntiles < (long long)kNumSMs * 4 ? ntiles : (long long)kNumSMs * 4;
  deil_tma_kernel<Tin, Tout, D><<<(unsigned)grid, kTileThreads, smem, s>>>((const Tin*)in, X, Y, Z, zt, ntiles,
                                                                           (Tout*)out);
  return FPVS_OK;
}

// the tiled kernels need d in {1,2,4,8}, 16-byte aligned buffers and z runs
// that are whole 16-byte vectors of the dense side's element; anything else
// takes the generic kernels above
static bool tile_ok(int d, int Nz, size_t esz_dense, const void* a, const void* b) {
  if (d != 1 && d != 2 && d != 4 && d != 8) return false;
  if (((uintptr_t)a | (uintptr_t)b) & 15) return false;
  return Nz % (int)(16 / esz_dense) == 0;
}

static int check_grid(int B, int Nx, int Ny, int Nz, int d) {
  FPVS_CHECK_ARG(B >= 1 && Nx >= 1 && Ny >= 1 && Nz >= 1, "grid dims must be positive");
  FPVS_CHECK_ARG(d >= 1, "interleave factor must be >= 1");
  if (Nx % d || Ny % d || Nz % d)
    return set_error(FPVS_ESHAPE, "interleave factor %d must divide grid dims (%d, %d, %d)", d, Nx, Ny, Nz);
  return FPVS_OK;
}

}  // namespace fpvs

using namespace fpvs;

template <typename Tin, typename Tout>
static int il_dense(const void* in, int B, int Nx, int Ny, int Nz, int d, void* out, uint8_t* cell_active,
                    cudaStream_t s) {
  if (tile_ok(d, Nz, sizeof(Tin), in, out)) {
    switch (d) {
      case 1: return launch_il_tile<Tin, Tout, 1>(in, B, Nx, Ny, Nz, out, cell_active, s);
      case 2: return launch_il_tile<Tin, Tout, 2>(in, B, Nx, Ny, Nz, out, cell_active, s);
      case 4: return launch_il_tile<Tin, Tout, 4>(in, B, Nx, Ny, Nz, out, cell_active, s);
      default: return launch_il_tile<Tin, Tout, 8>(in, B, Nx, Ny, Nz, out, cell_active, s);
    }
  }
  const int Z = Nz / d;
  const int elems = kIlSmemElems * 4 / (int)sizeof(Tin);  // 48 KB of staging
  int zc = elems / (d * d * d);
  if (zc < 1) zc = 1;
  if (zc > Z) zc = Z;
  FPVS_CHECK_ARG(d * d * zc * d <= elems, "interleave factor %d too large", d);
  const int nzc = (Z + zc - 1) / zc;
  const long long nblk = (long long)B * (Nx / d) * (Ny / d) * nzc;
  const size_t smem = (size_t)d * d * zc * d * sizeof(Tin);
  interleave_dense_kernel<Tin, Tout><<<(unsigned)nblk, 256, smem, s>>>((const Tin*)in, B, Nx, Ny, Nz, d, zc,
                                                                       (Tout*)out, cell_active);
  return FPVS_OK;
}

template <typename Tout>
static int il_bits(const uint8_t* in, int B, int Nx, int Ny, int Nz, int d, void* out, cudaStream_t s) {
  const long long X = Nx / d, Y = Ny / d;
  if ((d == 1 || d == 2 || d == 4 || d == 8) && !((uintptr_t)out & 15) && !((uintptr_t)in & 15) && Nx % 128 == 0) {
    const int rowb = Nx / 8;
    // ~4 CTAs per SM: z chunks of 16 (or fewer rows when the grid is small)
    int zt = 16;
    while (zt > 1 && (long long)B * Y * ((Nz + zt - 1) / zt) < 4LL * kNumSMs) zt >>= 1;
    if (zt > Nz) zt = Nz;
    const long long grid = (long long)B * Y * ((Nz + zt - 1) / zt);
    const size_t smem = (size_t)d * zt * (rowb + 4);
    switch (d) {
      case 1: il_bits_tile_kernel<Tout, 1><<<(unsigned)grid, kTileThreads, smem, s>>>(in, Nx, Ny, Nz, zt, (Tout*)out); break;
      case 2: il_bits_tile_kernel<Tout, 2><<<(unsigned)grid, kTileThreads, smem, s>>>(in, Nx, Ny, Nz, zt, (Tout*)out); break;
      case 4: il_bits_tile_kernel<Tout, 4><<<(unsigned)grid, kTileThreads, smem, s>>>(in, Nx, Ny, Nz, zt, (Tout*)out); break;
      default: il_bits_tile_kernel<Tout, 8><<<(unsigned)grid, kTileThreads, smem, s>>>(in, Nx, Ny, Nz, zt, (Tout*)out); break;
    }
    return FPVS_OK;
  }
  if ((d == 1 || d == 2 || d == 4 || d == 8) && !((uintptr_t)out & 15)) {
    const int m = d * d, vo = m < (int)(16 / sizeof(Tout)) ? m : (int)(16 / sizeof(Tout));
    const int g = grid_for((long long)B * X * Y * Nz * (m / vo), kTileThreads, 16);
    switch (d) {
      case 1: il_bits_kernel<Tout, 1><<<g, kTileThreads, 0, s>>>(in, B, Nx, Ny, Nz, (Tout*)out); break;
      case 2: il_bits_kernel<Tout, 2><<<g, kTileThreads, 0, s>>>(in, B, Nx, Ny, Nz, (Tout*)out); break;
      case 4: il_bits_kernel<Tout, 4><<<g, kTileThreads, 0, s>>>(in, B, Nx, Ny, Nz, (Tout*)out); break;
      default: il_bits_kernel<Tout, 8><<<g, kTileThreads, 0, s>>>(in, B, Nx, Ny, Nz, (Tout*)out); break;
    }
    return FPVS_OK;
  }
  const long long total = (long long)B * X * Y * (Nz / d) * d * d * d;
  interleave_bits_kernel<Tout><<<grid_for(total, 256), 256, 0, s>>>(in, B, Nx, Ny, Nz, d, (Tout*)out);
  return FPVS_OK;
}

extern "C" int fpvs_interleave(const void* in, int in_fmt, int B, int Nx, int Ny, int Nz, int d,
                               void* out, int out_dtype, uint8_t* cell_active, void* stream) {
  int rc = check_grid(B, Nx, Ny, Nz, d);
  if (rc) return rc;
  FPVS_CHECK_ARG(in && out, "null pointer");
  FPVS_CHECK_ARG(out_dtype == FPVS_F32 || out_dtype == FPVS_BF16 || out_dtype == FPVS_F64, "bad out dtype");
  FPVS_CHECK_ARG((in_fmt == FPVS_IN_F64) == (out_dtype == FPVS_F64),
                 "float64 grids interleave to float64 cells (an exact permutation) and only they do");
  cudaStream_t s = as_stream(stream);
  const int X = Nx / d, Y = Ny / d, Z = Nz / d;
  if (in_fmt == FPVS_IN_PACKED) {
    FPVS_CHECK_ARG(Nx % 8 == 0, "packed grids need N_x divisible by 8, got %d", Nx);
    rc = out_dtype == FPVS_F32 ? il_bits<float>((const uint8_t*)in, B, Nx, Ny, Nz, d, out, s)
                               : il_bits<__nv_bfloat16>((const uint8_t*)in, B, Nx, Ny, Nz, d, out, s);
    if (rc) return rc;
    if (cell_active) {
      long long nblk = (long long)B * Y * ((X + 31) / 32) * ((Z + 31) / 32);
      cell_active_bits_kernel<<<(unsigned)nblk, 256, 0, s>>>((const uint8_t*)in, B, Nx, Ny, Nz, d, cell_active);
    }
    FPVS_CHECK_LAUNCH("fpvs_interleave(packed)");
    return FPVS_OK;
  }
  FPVS_CHECK_ARG(in_fmt == FPVS_IN_U8 || in_fmt == FPVS_IN_F32 || in_fmt == FPVS_IN_F64, "bad input format %d",
                 in_fmt);
  if (in_fmt == FPVS_IN_F64) rc = il_dense<double, double>(in, B, Nx, Ny, Nz, d, out, cell_active, s);
  else if (in_fmt == FPVS_IN_U8)
    rc = out_dtype == FPVS_F32 ? il_dense<uint8_t, float>(in, B, Nx, Ny, Nz, d, out, cell_active, s)
                               : il_dense<uint8_t, __nv_bfloat16>(in, B, Nx, Ny, Nz, d, out, cell_active, s);
  else
    rc = out_dtype == FPVS_F32 ? il_dense<float, float>(in, B, Nx, Ny, Nz, d, out, cell_active, s)
                               : il_dense<float, __nv_bfloat16>(in, B, Nx, Ny, Nz, d, out, cell_active, s);
  if (rc) return rc;
  FPVS_CHECK_LAUNCH("fpvs_interleave(dense)");
  return FPVS_OK;
}

template <typename Tin, typename Tout>
static int deil_zalign_rt(int d) {
  switch (d) {
    case 1: return deil_zalign<Tin, Tout, 1>();
    case 2: return deil_zalign<Tin, Tout, 2>();
    case 4: return deil_zalign<Tin, Tout, 4>();
    default: return deil_zalign<Tin, Tout, 8>();
  }
}

template <typename Tin, typename Tout>
static int deil_dense(const void* in, int B, int X, int Y, int Z, int d, void* out, cudaStream_t s) {
  if (tile_ok(d, Z * d, sizeof(Tout), in, out) && (Z * d) % deil_zalign_rt<Tin, Tout>(d) == 0) {
    switch (d) {
      case 1: return launch_deil_tile<Tin, Tout, 1>(in, B, X, Y, Z, out, s);
      case 2: return launch_deil_tile<Tin, Tout, 2>(in, B, X, Y, Z, out, s);
      case 4: return launch_deil_tile<Tin, Tout, 4>(in, B, X, Y, Z, out, s);
      default: return launch_deil_tile<Tin, Tout, 8>(in, B, X, Y, Z, out, s);
    }
  }
  const long long total = (long long)B * X * Y * Z * d * d * d;
  deinterleave_dense_kernel<Tin, Tout><<<grid_for(total, 256), 256, 0, s>>>((const Tin*)in, B, X, Y, Z, d,
                                                                           (Tout*)out);
  return FPVS_OK;
}

template <typename Tin, typename Tc>
static int deil_bits(const void* in, int B, int X, int Y, int Z, int d, Tc tau, void* out, cudaStream_t s) {
  const int Nx = X * d;
  if ((d == 1 || d == 2 || d == 4 || d == 8) && Nx % 32 == 0 && !((uintptr_t)out & 3) &&
      !((uintptr_t)in & (d * sizeof(Tin) < 16 ? d * sizeof(Tin) - 1 : 15))) {
    const long long words = (long long)B * Z * d * Y * d * (Nx / 32);
    const int g = grid_for(words, kTileThreads, 16);
    switch (d) {
      case 1: deil_bits_kernel<Tin, Tc, 1><<<g, kTileThreads, 0, s>>>((const Tin*)in, B, X, Y, Z, tau, (uint32_t*)out); break;
      case 2: deil_bits_kernel<Tin, Tc, 2><<<g, kTileThreads, 0, s>>>((const Tin*)in, B, X, Y, Z, tau, (uint32_t*)out); break;
      case 4: deil_bits_kernel<Tin, Tc, 4><<<g, kTileThreads, 0, s>>>((const Tin*)in, B, X, Y, Z, tau, (uint32_t*)out); break;
      default: deil_bits_kernel<Tin, Tc, 8><<<g, kTileThreads, 0, s>>>((const Tin*)in, B, X, Y, Z, tau, (uint32_t*)out); break;
    }
    return FPVS_OK;
  }
  const long long total = (long long)B * Z * d * Y * d * (Nx / 8);
  deinterleave_thresh_kernel<Tin, Tc><<<grid_for(total, 256), 256, 0, s>>>((const Tin*)in, B, X, Y, Z, d, tau,
                                                                          (uint8_t*)out);
  return FPVS_OK;
}

extern "C" int fpvs_deinterleave(const void* in, int in_dtype, int B, int X, int Y, int Z, int d,
                                 double tau, void* out, void* stream) {
  FPVS_CHECK_ARG(in && out, "null pointer");
  FPVS_CHECK_ARG(B >= 1 && X >= 1 && Y >= 1 && Z >= 1 && d >= 1, "bad shape");
  FPVS_CHECK_ARG(in_dtype == FPVS_F32 || in_dtype == FPVS_BF16 || in_dtype == FPVS_F64, "bad dtype");
  cudaStream_t s = as_stream(stream);
  int rc;
  if (tau != tau) {  // NaN: dense real-valued output (f64 for f64 cells, else f32)
    if (in_dtype == FPVS_F64) rc = deil_dense<double, double>(in, B, X, Y, Z, d, out, s);
    else if (in_dtype == FPVS_F32) rc = deil_dense<float, float>(in, B, X, Y, Z, d, out, s);
    else rc = deil_dense<__nv_bfloat16, float>(in, B, X, Y, Z, d, out, s);
  } else {
    if ((X * d) % 8) return set_error(FPVS_ESHAPE, "N_x must be divisible by 8, got %d", X * d);
    if (in_dtype == FPVS_F64) rc = deil_bits<double, double>(in, B, X, Y, Z, d, tau, out, s);
    else if (in_dtype == FPVS_F32) rc = deil_bits<float, float>(in, B, X, Y, Z, d, (float)tau, out, s);
    else rc = deil_bits<__nv_bfloat16, float>(in, B, X, Y, Z, d, (float)tau, out, s);
  }
  if (rc) return rc;
  FPVS_CHECK_LAUNCH("fpvs_deinterleave");
  return FPVS_OK;
}

extern "C" int fpvs_cell_active_from_bits(const uint8_t* bits, int B, int Nx, int Ny, int Nz, int d,
                                          uint8_t* cell_active, void* stream) {
  int rc = check_grid(B, Nx, Ny, Nz, d);
  if (rc) return rc;
  FPVS_CHECK_ARG(Nx % 8 == 0, "packed grids need N_x divisible by 8, got %d", Nx);
  const int X = Nx / d, Y = Ny / d, Z = Nz / d;
  long long nblk = (long long)B * Y * ((X + 31) / 32) * ((Z + 31) / 32);
  cell_active_bits_kernel<<<(unsigned)nblk, 256, 0, as_stream(stream)>>>(bits, B, Nx, Ny, Nz, d, cell_active);
  FPVS_CHECK_LAUNCH("fpvs_cell_active_from_bits");
  return FPVS_OK;
}

extern "C" int fpvs_gather_cells_bits(const uint8_t* bits, int B, int Nx, int Ny, int Nz, int d,
                                      const int32_t* coords, const int32_t* n_active_dev, int cap,
                                      void* x, int ldx, int dtype, void* stream) {
  int rc = check_grid(B, Nx, Ny, Nz, d);
  if (rc) return rc;
  FPVS_CHECK_ARG(ldx >= d * d * d, "ldx %d < d^3", ldx);
  cudaStream_t s = as_stream(stream);
  int g = grid_for((long long)cap * ((d * d * d + 7) / 8), 256);
  if (dtype == FPVS_F32)
    gather_cells_bits_kernel<float><<<g, 256, 0, s>>>(bits, Nx, Ny, Nz, d, (const int4*)coords,
                                                       n_active_dev, cap, (float*)x, ldx);
  else
    gather_cells_bits_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(bits, Nx, Ny, Nz, d, (const int4*)coords,
                                                               n_active_dev, cap, (__nv_bfloat16*)x, ldx);
  FPVS_CHECK_LAUNCH("fpvs_gather_cells_bits");
  return FPVS_OK;
}
