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

namespace fpvs {

constexpr int kIlSmemElems = 12288;  // 48 KB of f32 staging

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
    out[obase + t] = from_f32<Tout>(to_f32<Tin>(tile[(lx * d + ly) * zlen + bzl * d + lz]));
  }
  if (cell_active) {
    for (int bzl = threadIdx.x; bzl < nbz; bzl += blockDim.x) {
      uint8_t any = 0;
      for (int lx = 0; lx < d && !any; ++lx)
        for (int ly = 0; ly < d && !any; ++ly)
          for (int lz = 0; lz < d; ++lz)
            if (to_f32<Tin>(tile[(lx * d + ly) * zlen + bzl * d + lz]) != 0.f) { any = 1; break; }
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

template <typename Tin>
__global__ void deinterleave_dense_kernel(const Tin* __restrict__ in, int B, int X, int Y, int Z, int d,
                                          float* __restrict__ out) {
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
    out[t] = to_f32<Tin>(in[cell * d3 + k]);
  }
}

// one output byte = 8 x-consecutive froxels of one (b, y, z) row
template <typename Tin>
__global__ void deinterleave_thresh_kernel(const Tin* __restrict__ in, int B, int X, int Y, int Z, int d,
                                           float tau, uint8_t* __restrict__ out) {
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
      if (to_f32<Tin>(in[cell * d3 + k]) >= tau) byte |= 1u << i;
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

static int check_grid(int B, int Nx, int Ny, int Nz, int d) {
  FPVS_CHECK_ARG(B >= 1 && Nx >= 1 && Ny >= 1 && Nz >= 1, "grid dims must be positive");
  FPVS_CHECK_ARG(d >= 1, "interleave factor must be >= 1");
  if (Nx % d || Ny % d || Nz % d)
    return set_error(FPVS_ESHAPE, "interleave factor %d must divide grid dims (%d, %d, %d)", d, Nx, Ny, Nz);
  return FPVS_OK;
}

}  // namespace fpvs

using namespace fpvs;

extern "C" int fpvs_interleave(const void* in, int in_fmt, int B, int Nx, int Ny, int Nz, int d,
                               void* out, int out_dtype, uint8_t* cell_active, void* stream) {
  int rc = check_grid(B, Nx, Ny, Nz, d);
  if (rc) return rc;
  FPVS_CHECK_ARG(in && out, "null pointer");
  FPVS_CHECK_ARG(out_dtype == FPVS_F32 || out_dtype == FPVS_BF16, "bad out dtype");
  cudaStream_t s = as_stream(stream);
  const int X = Nx / d, Y = Ny / d, Z = Nz / d, d3 = d * d * d;
  if (in_fmt == FPVS_IN_PACKED) {
    FPVS_CHECK_ARG(Nx % 8 == 0, "packed grids need N_x divisible by 8, got %d", Nx);
    long long total = (long long)B * X * Y * Z * d3;
    int g = grid_for(total, 256);
    if (out_dtype == FPVS_F32)
      interleave_bits_kernel<float><<<g, 256, 0, s>>>((const uint8_t*)in, B, Nx, Ny, Nz, d, (float*)out);
    else
      interleave_bits_kernel<__nv_bfloat16><<<g, 256, 0, s>>>((const uint8_t*)in, B, Nx, Ny, Nz, d,
                                                              (__nv_bfloat16*)out);
    if (cell_active) {
      long long nblk = (long long)B * Y * ((X + 31) / 32) * ((Z + 31) / 32);
      cell_active_bits_kernel<<<(unsigned)nblk, 256, 0, s>>>((const uint8_t*)in, B, Nx, Ny, Nz, d, cell_active);
    }
    FPVS_CHECK_LAUNCH("fpvs_interleave(packed)");
    return FPVS_OK;
  }
  FPVS_CHECK_ARG(in_fmt == FPVS_IN_U8 || in_fmt == FPVS_IN_F32, "bad input format %d", in_fmt);
  int zc = kIlSmemElems / (d * d * d);
  if (zc < 1) zc = 1;
  if (zc > Z) zc = Z;
  FPVS_CHECK_ARG(d * d * zc * d <= kIlSmemElems, "interleave factor %d too large", d);
  const int nzc = (Z + zc - 1) / zc;
  long long nblk = (long long)B * X * Y * nzc;
  size_t esz = in_fmt == FPVS_IN_U8 ? 1 : 4;
  size_t smem = (size_t)d * d * zc * d * esz;
#define FPVS_IL_LAUNCH(TIN, TOUT)                                                              \
  interleave_dense_kernel<TIN, TOUT><<<(unsigned)nblk, 256, smem, s>>>(                        \
      (const TIN*)in, B, Nx, Ny, Nz, d, zc, (TOUT*)out, cell_active)
  if (in_fmt == FPVS_IN_U8) {
    if (out_dtype == FPVS_F32) FPVS_IL_LAUNCH(uint8_t, float);
    else FPVS_IL_LAUNCH(uint8_t, __nv_bfloat16);
  } else {
    if (out_dtype == FPVS_F32) FPVS_IL_LAUNCH(float, float);
    else FPVS_IL_LAUNCH(float, __nv_bfloat16);
  }
#undef FPVS_IL_LAUNCH
  FPVS_CHECK_LAUNCH("fpvs_interleave(dense)");
  return FPVS_OK;
}

extern "C" int fpvs_deinterleave(const void* in, int in_dtype, int B, int X, int Y, int Z, int d,
                                 float tau, void* out, void* stream) {
  FPVS_CHECK_ARG(in && out, "null pointer");
  FPVS_CHECK_ARG(B >= 1 && X >= 1 && Y >= 1 && Z >= 1 && d >= 1, "bad shape");
  FPVS_CHECK_ARG(in_dtype == FPVS_F32 || in_dtype == FPVS_BF16, "bad dtype");
  cudaStream_t s = as_stream(stream);
  if (tau != tau) {  // NaN: dense real-valued output
    long long total = (long long)B * X * Y * Z * d * d * d;
    int g = grid_for(total, 256);
    if (in_dtype == FPVS_F32)
      deinterleave_dense_kernel<float><<<g, 256, 0, s>>>((const float*)in, B, X, Y, Z, d, (float*)out);
    else
      deinterleave_dense_kernel<__nv_bfloat16><<<g, 256, 0, s>>>((const __nv_bfloat16*)in, B, X, Y, Z, d,
                                                                (float*)out);
  } else {
    if ((X * d) % 8) return set_error(FPVS_ESHAPE, "N_x must be divisible by 8, got %d", X * d);
    long long total = (long long)B * Z * d * Y * d * (X * d / 8);
    int g = grid_for(total, 256);
    if (in_dtype == FPVS_F32)
      deinterleave_thresh_kernel<float><<<g, 256, 0, s>>>((const float*)in, B, X, Y, Z, d, tau,
                                                          (uint8_t*)out);
    else
      deinterleave_thresh_kernel<__nv_bfloat16><<<g, 256, 0, s>>>((const __nv_bfloat16*)in, B, X, Y, Z, d,
                                                                  tau, (uint8_t*)out);
  }
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
