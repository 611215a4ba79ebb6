// (3)/(4) SIMT (FFMA) sparse convolution: the fp32 mode and correctness
// anchor of the implicit gather-GEMM, its fused head, and the training
// kernels (dgrad, deterministic wgrad, repulsive-visibility / Dice loss).
//
// Algebra restated from pkg/src/froxelpvs/neural.py:
//   forward   z[i] = b + sum_j x[nbr[i][j]] @ W_j          (neural.py:187-219)
//   relu'     z > 0                                         (neural.py:227-228)
//   dgrad     dx = col2im(dz W^T)                           (neural.py:240-248)
//   wgrad     dW = cols^T dz, db = sum dz                   (neural.py:238-239)
//   losses    ConfusionCounts / dice / rvl / combined       (neural.py:130-144, 353-399)
// The fp32 mode must not use TF32 tensor cores: its
// logits are checked to 1e-4 against the float64 oracle.
#include "common.cuh"
#include <stdlib.h>

namespace fpvs {

constexpr int kTM = 64, kTN = 64, kTK = 32;

// wmode 0: W is (K*Cin, Cout) row-major (reference layout)
// wmode 1: dgrad view of a forward weight W_f (K*Cout_f, Cin_f): the
//          effective (K*Cin, Cout) matrix with Cin = Cout_f, Cout = Cin_f and
//          W_eff[j][ci][co] = W_f[K-1-j][co][ci] (mirrored offset, transposed)
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(256) spconv_simt_kernel(
    const Tin* __restrict__ x, int ldx, const int* __restrict__ nbr, int K, const int* __restrict__ n_dev, int cap,
    const float* __restrict__ w, int wmode, const float* __restrict__ bias, int cin, int cout, int act,
    const void* __restrict__ ymask, int mask_bf16, int ldm, Tout* __restrict__ y, int ldy, int col_off) {
  __shared__ float As[kTK][kTM + 4];
  __shared__ float Bs[kTK][kTN];
  const int n = min(*n_dev, cap);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int mt = (n + kTM - 1) / kTM, nt = (cout + kTN - 1) / kTN;
  const int Ktot = K * cin;
  for (int tile = blockIdx.x; tile < mt * nt; tile += gridDim.x) {
    const int m0 = (tile / nt) * kTM, n0 = (tile % nt) * kTN;
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
    for (int k0 = 0; k0 < Ktot; k0 += kTK) {
      for (int e = threadIdx.x; e < kTM * kTK; e += 256) {
        int kk = e % kTK, r = e / kTK;
        int row = m0 + r, k = k0 + kk;
        float v = 0.f;
        if (row < n && k < Ktot) {
          int j = k / cin, ci = k % cin;
          int src = nbr ? __ldg(nbr + (long long)row * K + j) : row;
          if (src >= 0) v = to_f32<Tin>(x[(long long)src * ldx + ci]);
        }
        As[kk][r] = v;
      }
      for (int e = threadIdx.x; e < kTK * kTN; e += 256) {
        int c = e % kTN, kk = e / kTN;
        int k = k0 + kk, co = n0 + c;
        float v = 0.f;
        if (k < Ktot && co < cout) {
          if (wmode == 0) {
            v = __ldg(w + (long long)k * cout + co);
          } else {
            // W_f[(j_f*Cin_f + ci_f)*Cout_f + co_f] with Cin_f = cout, Cout_f = cin
            int j = k / cin, ci = k % cin;
            v = __ldg(w + ((long long)(K - 1 - j) * cout + co) * cin + ci);
          }
        }
        Bs[kk][c] = v;
      }
      __syncthreads();
#pragma unroll 8
      for (int kk = 0; kk < kTK; ++kk) {
        float a[4], b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) a[q] = As[kk][ty * 4 + q];
#pragma unroll
        for (int q = 0; q < 4; ++q) b[q] = Bs[kk][tx * 4 + q];
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[p][q] = fmaf(a[p], b[q], acc[p][q]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      int row = m0 + ty * 4 + p;
      if (row >= n) continue;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int co = n0 + tx * 4 + q;
        if (co >= cout) continue;
        float z = acc[p][q] + (bias ? __ldg(bias + co) : 0.f);
        z = apply_act(z, act);
        if (ymask) {
          const long long mi = (long long)row * ldm + co;
          const float mv = mask_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(ymask)[mi])
                                     : reinterpret_cast<const float*>(ymask)[mi];
          if (!(mv > 0.f)) z = 0.f;
        }
        y[(long long)row * ldy + col_off + co] = from_f32<Tout>(z);
      }
    }
  }
}

// fp32 forward for the chain nets (config 1's precision): a 64-row x Cout
// tile per CTA (Cout 32 or 64, Cin <= 64 and a multiple of 4).  The tile's
// neighbour rows are staged in shared memory first and give the offsets
// present anywhere in the tile; only those offsets are gathered (float4 rows)
// and multiplied, two offsets in flight (the next offset's gather is issued
// into registers before the current one's FMAs).  4 x 4 outputs per thread,
// fp32 FMA in offset order (deterministic).
constexpr int kT2M = 64;
constexpr int kT2CinMax = 64;

template <int TN>
__global__ void __launch_bounds__(kT2M * TN / 16) spconv_simt_tap_kernel(
    const float* __restrict__ x, int ldx, const int* __restrict__ nbr, int K, const int* __restrict__ n_dev, int cap,
    const float* __restrict__ w, const float* __restrict__ bias, int cin, int cout, int act, float* __restrict__ y,
    int ldy, int col_off) {
  constexpr int NT = kT2M * TN / 16;
  extern __shared__ __align__(16) float sm2[];
  float* As = sm2;                                   // [2][cin][kT2M + 4]
  float* Bs = As + 2 * kT2CinMax * (kT2M + 4);       // [2][cin][TN]
  int* snb = reinterpret_cast<int*>(Bs + 2 * kT2CinMax * TN);  // [kT2M][K]
  __shared__ unsigned s_mask;
  const int n = min(*n_dev, cap);
  const int tx = threadIdx.x % (TN / 4), ty = threadIdx.x / (TN / 4);
  const int c4n = cin / 4;
  const int mt = (n + kT2M - 1) / kT2M;
  for (int tile = blockIdx.x; tile < mt; tile += gridDim.x) {
    const int m0 = tile * kT2M;
    if (threadIdx.x == 0) s_mask = 0u;
    __syncthreads();
    unsigned mloc = 0u;
    for (int e = threadIdx.x; e < kT2M * K; e += NT) {
      const int r = e / K, j = e - r * K;
      const int row = m0 + r;
      int v = -1;
      if (row < n) v = nbr ? __ldg(nbr + (long long)row * K + j) : row;
      snb[e] = v;
      if (v >= 0) mloc |= 1u << j;
    }
    atomicOr(&s_mask, mloc);
    __syncthreads();
    unsigned mask = s_mask;
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
    // register staging of one offset: A pieces (row, 4 channels) and B pieces
    constexpr int AMAX = kT2M * kT2CinMax / 4 / NT + 1;
    constexpr int BMAX = kT2CinMax * TN / 4 / NT + 1;
    float4 ra[AMAX], rb[BMAX];
    auto fetch = [&](int j) {
#pragma unroll
      for (int i = 0; i < AMAX; ++i) {
        const int e = threadIdx.x + i * NT;
        ra[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (e < kT2M * c4n) {
          const int r = e % kT2M, c4 = e / kT2M;
          const int src = snb[r * K + j];
          if (src >= 0) ra[i] = __ldg(reinterpret_cast<const float4*>(x + (long long)src * ldx) + c4);
        }
      }
#pragma unroll
      for (int i = 0; i < BMAX; ++i) {
        const int e = threadIdx.x + i * NT;
        rb[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (e < cin * (TN / 4)) {
          const int k = e / (TN / 4), c4 = e - k * (TN / 4);
          if (c4 * 4 < cout) rb[i] = __ldg(reinterpret_cast<const float4*>(w + ((long long)j * cin + k) * cout) + c4);
        }
      }
    };
    auto stash = [&](int buf) {
      float* a = As + buf * kT2CinMax * (kT2M + 4);
      float* b = Bs + buf * kT2CinMax * TN;
#pragma unroll
      for (int i = 0; i < AMAX; ++i) {
        const int e = threadIdx.x + i * NT;
        if (e < kT2M * c4n) {
          const int r = e % kT2M, c4 = e / kT2M;
          a[(c4 * 4 + 0) * (kT2M + 4) + r] = ra[i].x;
          a[(c4 * 4 + 1) * (kT2M + 4) + r] = ra[i].y;
          a[(c4 * 4 + 2) * (kT2M + 4) + r] = ra[i].z;
          a[(c4 * 4 + 3) * (kT2M + 4) + r] = ra[i].w;
        }
      }
#pragma unroll
      for (int i = 0; i < BMAX; ++i) {
        const int e = threadIdx.x + i * NT;
        if (e < cin * (TN / 4)) reinterpret_cast<float4*>(b)[e] = rb[i];
      }
    };
    int j = mask ? __ffs(mask) - 1 : -1;
    if (j >= 0) {
      fetch(j);
      stash(0);
    }
    __syncthreads();
    int buf = 0;
    while (j >= 0) {
      const int jn = __ffs(mask & ~((2u << j) - 1u)) - 1;
      if (jn >= 0) fetch(jn);  // in flight during the FMAs below
      const float* a = As + buf * kT2CinMax * (kT2M + 4);
      const float* b = Bs + buf * kT2CinMax * TN;
#pragma unroll 4
      for (int k = 0; k < cin; ++k) {
        const float4 av = *reinterpret_cast<const float4*>(a + k * (kT2M + 4) + ty * 4);
        const float4 bv = *reinterpret_cast<const float4*>(b + k * TN + tx * 4);
        const float aa[4] = {av.x, av.y, av.z, av.w}, bb[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[p][q] = fmaf(aa[p], bb[q], acc[p][q]);
      }
      if (jn >= 0) stash(buf ^ 1);
      __syncthreads();
      buf ^= 1;
      j = jn;
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int row = m0 + ty * 4 + p;
      if (row >= n) continue;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int co = tx * 4 + q;
        if (co >= cout) continue;
        float z = acc[p][q] + (bias ? __ldg(bias + co) : 0.f);
        y[(long long)row * ldy + col_off + co] = apply_act(z, act);
      }
    }
    __syncthreads();
  }
}

// Fused head: 1x1x1 conv (Cin -> d^3) + sigmoid + [p >= tau] + packed-bit scatter.
// One thread per (active cell, output channel k); W staged in smem.
template <typename Tin>
__global__ void head_simt_kernel(const Tin* __restrict__ x, int ldx, const int4* __restrict__ coords,
                                 const int* __restrict__ n_dev, int cap, const float* __restrict__ w,
                                 const float* __restrict__ bias, int cin, int d, int Nx, int Ny, int Nz, float tau,
                                 uint8_t* __restrict__ out_bits, float* __restrict__ probs, float* __restrict__ logits) {
  extern __shared__ float wsm[];  // cin * d3 + d3
  const int d3 = d * d * d;
  for (int e = threadIdx.x; e < cin * d3; e += blockDim.x) wsm[e] = w[e];
  for (int e = threadIdx.x; e < d3; e += blockDim.x) wsm[cin * d3 + e] = bias ? bias[e] : 0.f;
  __syncthreads();
  const int n = min(*n_dev, cap);
  const long long total = (long long)n * d3;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int k = t % d3;
    long long i = t / d3;
    const Tin* xr = x + i * ldx;
    float z = wsm[cin * d3 + k];
    for (int ci = 0; ci < cin; ++ci) z = fmaf(to_f32<Tin>(xr[ci]), wsm[ci * d3 + k], z);
    float p = sigmoidf_stable(z);
    if (logits) logits[t] = z;
    if (probs) probs[t] = p;
    if (p >= tau && out_bits) {
      int4 c = coords[i];
      int lx = k % d, ly = (k / d) % d, lz = k / (d * d);
      int fx = c.y * d + lx;
      atomic_or_bit(out_bits, bit_byte(c.x, fx, c.z * d + ly, c.w * d + lz, Nx, Ny, Nz), fx & 7);
    }
  }
}

// Head epilogue over precomputed logits rows (a head layer with k > 1 runs as
// an ordinary conv with no activation first): sigmoid + [p >= tau] +
// packed-bit scatter, probabilities optional (neural.py:513-526, 151-157).
__global__ void head_rows_kernel(const float* __restrict__ logits, int ld, const int4* __restrict__ coords,
                                 const int* __restrict__ n_dev, int cap, int d, int Nx, int Ny, int Nz, float tau,
                                 uint8_t* __restrict__ out_bits, float* __restrict__ probs) {
  const int d3 = d * d * d;
  const int n = min(*n_dev, cap);
  const long long total = (long long)n * d3;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t % d3);
    const long long i = t / d3;
    const float p = sigmoidf_stable(logits[i * ld + k]);
    if (probs) probs[t] = p;
    if (p >= tau && out_bits) {
      const int4 c = coords[i];
      const int lx = k % d, ly = (k / d) % d, lz = k / (d * d);
      const int fx = c.y * d + lx;
      atomic_or_bit(out_bits, bit_byte(c.x, fx, c.z * d + ly, c.w * d + lz, Nx, Ny, Nz), fx & 7);
    }
  }
}

// dz = dy * act'(.) from the layer's kept output y (neural.py:225-232):
// relu z > 0 <=> y > 0, sigmoid y (1 - y), none 1
template <typename Ty>
__global__ void act_backward_kernel(const float* __restrict__ dy, int lddy, const Ty* __restrict__ y, int ldy,
                                    const int* __restrict__ n_dev, int cap, int C, int act, float* __restrict__ dz,
                                    int lddz) {
  const int n = min(*n_dev, cap);
  const long long total = (long long)n * C;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / C;
    const int c = (int)(t % C);
    const float g = dy[i * lddy + c];
    const float v = to_f32<Ty>(y[i * ldy + c]);
    dz[i * lddz + c] = act == FPVS_ACT_RELU ? (v > 0.f ? g : 0.f) : act == FPVS_ACT_SIGMOID ? g * v * (1.f - v) : g;
  }
}

// ---- wgrad: deterministic split over rows, fixed-order reduction ---------
constexpr int kWgSplits = 64;
constexpr int kWgRows = 32;

// partial[s][j][ci][co] = sum over rows of split s of x[nbr[i][j]][ci] * dz[i][co]
template <typename Tx>
__global__ void __launch_bounds__(256) wgrad_partial_kernel(
    const Tx* __restrict__ x, int ldx, const float* __restrict__ dz, int lddz, const int* __restrict__ nbr, int K,
    const int* __restrict__ n_dev, int cap, int cin, int cout, float* __restrict__ part) {
  extern __shared__ float sm[];
  float* xs = sm;                      // kWgRows * cin
  float* ds = sm + kWgRows * cin;      // kWgRows * cout
  const int n = min(*n_dev, cap);
  const int j = blockIdx.x % K, s = blockIdx.x / K;
  const int per = (n + kWgSplits - 1) / kWgSplits;
  const int r0 = s * per, r1 = min(n, r0 + per);
  const int nout = cin * cout;
  const int mine = (nout + 255) / 256;  // outputs per thread (<= 16 for 64x64)
  float acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.f;
  for (int rb = r0; rb < r1; rb += kWgRows) {
    for (int e = threadIdx.x; e < kWgRows * cin; e += 256) {
      int r = e / cin, ci = e % cin, row = rb + r;
      float v = 0.f;
      if (row < r1) {
        int src = nbr ? __ldg(nbr + (long long)row * K + j) : row;
        if (src >= 0) v = to_f32<Tx>(x[(long long)src * ldx + ci]);
      }
      xs[e] = v;
    }
    for (int e = threadIdx.x; e < kWgRows * cout; e += 256) {
      int r = e / cout, co = e % cout, row = rb + r;
      ds[e] = row < r1 ? dz[(long long)row * lddz + co] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      int o = threadIdx.x + q * 256;
      if (q < mine && o < nout) {
        int ci = o / cout, co = o % cout;
        float a = acc[q];
        for (int r = 0; r < kWgRows; ++r) a = fmaf(xs[r * cin + ci], ds[r * cout + co], a);
        acc[q] = a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    int o = threadIdx.x + q * 256;
    if (q < mine && o < nout) part[((long long)s * K + j) * nout + o] = acc[q];
  }
}

__global__ void wgrad_reduce_kernel(const float* __restrict__ part, long long per_split, float* __restrict__ dw) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < per_split;
       e += (long long)gridDim.x * blockDim.x) {
    float a = 0.f;
    for (int s = 0; s < kWgSplits; ++s) a += part[s * per_split + e];
    dw[e] = a;
  }
}

// db[co] = sum_i dz[i][co], one block per column chunk, fixed order
__global__ void bias_grad_kernel(const float* __restrict__ dz, int lddz, const int* __restrict__ n_dev, int cap,
                                 int cout, float* __restrict__ db) {
  __shared__ float red[256];
  const int n = min(*n_dev, cap);
  for (int co = blockIdx.x; co < cout; co += gridDim.x) {
    float a = 0.f;
    for (int i = threadIdx.x; i < n; i += 256) a += dz[(long long)i * lddz + co];
    red[threadIdx.x] = a;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) db[co] = red[0];
    __syncthreads();
  }
}

// ---- loss (neural.py:130-144, 353-399) -----------------------------------
__device__ __forceinline__ int label_bit(const uint8_t* gt, int4 c, int k, int d, int Nx, int Ny, int Nz) {
  int lx = k % d, ly = (k / d) % d, lz = k / (d * d);
  int fx = c.y * d + lx;
  return (__ldg(gt + bit_byte(c.x, fx, c.z * d + ly, c.w * d + lz, Nx, Ny, Nz)) >> (fx & 7)) & 1;
}

// per-row (sum p*g, sum p) in f64
__global__ void loss_rows_kernel(const float* __restrict__ probs, int C, const int4* __restrict__ coords,
                                 const int* __restrict__ n_dev, int cap, const uint8_t* __restrict__ gt, int d, int Nx,
                                 int Ny, int Nz, double2* __restrict__ rows) {
  const int n = min(*n_dev, cap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int4 c = coords[i];
    double pg = 0.0, ps = 0.0;
    for (int k = 0; k < C; ++k) {
      double p = probs[(long long)i * C + k];
      ps += p;
      if (label_bit(gt, c, k, d, Nx, Ny, Nz)) pg += p;
    }
    rows[i] = make_double2(pg, ps);
  }
}

__device__ __forceinline__ int first_row_of(const int4* coords, int n, int b) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int m = (lo + hi) >> 1;
    if (coords[m].x < b) lo = m + 1; else hi = m;
  }
  return lo;
}

// sums[b] = (TP, sum p, GTP): LOSS_G blocks per sample each reduce a slice of
// the sample's rows and of its packed labels (16-byte popcounts) with a
// fixed-order tree, then one warp adds the slices in order (deterministic)
constexpr int LOSS_G = 16;
__global__ void __launch_bounds__(256) loss_sums_part_kernel(const double2* __restrict__ rows,
                                                             const int4* __restrict__ coords,
                                                             const int* __restrict__ n_dev, int cap,
                                                             const uint8_t* __restrict__ gt, long long grid_bytes,
                                                             double* __restrict__ part) {
  __shared__ double r0[256], r1[256], r2[256];
  const int n = min(*n_dev, cap);
  const int g = blockIdx.x, b = blockIdx.y;
  const int i0 = first_row_of(coords, n, b), i1 = first_row_of(coords, n, b + 1);
  const int a0 = i0 + (int)((long long)(i1 - i0) * g / LOSS_G), a1 = i0 + (int)((long long)(i1 - i0) * (g + 1) / LOSS_G);
  double a = 0.0, s = 0.0, c = 0.0;
  for (int i = a0 + threadIdx.x; i < a1; i += 256) {
    const double2 v = rows[i];
    a += v.x;
    s += v.y;
  }
  const uint8_t* gb = gt + (long long)b * grid_bytes;
  const long long nv = grid_bytes / 16;  // whole 16-byte vectors, the tail bytes by block 0
  const long long v0 = nv * g / LOSS_G, v1 = nv * (g + 1) / LOSS_G;
  const bool aligned = (((uintptr_t)gb) & 15) == 0;
  unsigned cnt = 0;
  if (aligned) {
    const uint4* gv = reinterpret_cast<const uint4*>(gb);
    for (long long e = v0 + threadIdx.x; e < v1; e += 256) {
      const uint4 w = __ldg(gv + e);
      cnt += __popc(w.x) + __popc(w.y) + __popc(w.z) + __popc(w.w);
    }
    if (g == 0)
      for (long long e = nv * 16 + threadIdx.x; e < grid_bytes; e += 256) cnt += __popc((unsigned)gb[e]);
  } else {
    const long long e0 = grid_bytes * g / LOSS_G, e1 = grid_bytes * (g + 1) / LOSS_G;
    for (long long e = e0 + threadIdx.x; e < e1; e += 256) cnt += __popc((unsigned)gb[e]);
  }
  c = (double)cnt;
  r0[threadIdx.x] = a; r1[threadIdx.x] = s; r2[threadIdx.x] = c;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      r0[threadIdx.x] += r0[threadIdx.x + o];
      r1[threadIdx.x] += r1[threadIdx.x + o];
      r2[threadIdx.x] += r2[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double* o = part + ((long long)b * LOSS_G + g) * 3;
    o[0] = r0[0]; o[1] = r1[0]; o[2] = r2[0];
  }
}

__global__ void loss_sums_final_kernel(const double* __restrict__ part, int B, double* __restrict__ sums) {
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    for (int g = 0; g < LOSS_G; ++g) {
      const double* o = part + ((long long)b * LOSS_G + g) * 3;
      t0 += o[0]; t1 += o[1]; t2 += o[2];
    }
    sums[3 * b] = t0; sums[3 * b + 1] = t1; sums[3 * b + 2] = t2;
  }
}

struct LossCoef { double g1, g0, loss; };

__device__ __forceinline__ LossCoef loss_coef(const double* sums, int b, double alpha, double lam) {
  const double tp = sums[3 * b], ps = sums[3 * b + 1], gtp = sums[3 * b + 2];
  const double fp = ps - tp, fn = gtp - tp;
  LossCoef c{0.0, 0.0, 0.0};
  const double num = 2.0 * tp, den = 2.0 * tp + alpha * fp + (1.0 - alpha) * fn;
  if (den != 0.0) {  // dice (neural.py:353-373)
    const double den2 = den * den;
    c.g1 += lam * (-(2.0 * den - num * (2.0 - (1.0 - alpha))) / den2);
    c.g0 += lam * (num * alpha / den2);
    c.loss += lam * ((den - num) / den);
  }
  if (gtp != 0.0) {  // rvl (neural.py:376-392)
    c.g1 += (1.0 - lam) * (-1.0 / gtp);
    c.g0 += (1.0 - lam) * (1.0 / gtp);
    c.loss += (1.0 - lam) * ((1.0 - tp / gtp) + fp / gtp);
  }
  return c;
}

__global__ void loss_grad_kernel(const float* __restrict__ probs, int C, const int4* __restrict__ coords,
                                 const int* __restrict__ n_dev, int cap, const uint8_t* __restrict__ gt, int d, int Nx,
                                 int Ny, int Nz, const double* __restrict__ sums, int B, double alpha, double lam,
                                 float* __restrict__ dlogits) {
  // per-sample coefficients once per block (B <= kMaxB), else per element
  constexpr int kMaxB = 256;
  __shared__ double s_g1[kMaxB], s_g0[kMaxB];
  const bool cached = B <= kMaxB;
  if (cached)
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
      const LossCoef lc = loss_coef(sums, b, alpha, lam);
      s_g1[b] = lc.g1;
      s_g0[b] = lc.g0;
    }
  __syncthreads();
  const int n = min(*n_dev, cap);
  const long long total = (long long)n * C;
  const int lc2 = (C & (C - 1)) == 0 ? __ffs(C) - 1 : -1;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = lc2 >= 0 ? (t >> lc2) : t / C;
    const int k = (int)(t - i * C);
    int4 c = coords[i];
    double g1, g0;
    if (cached) {
      g1 = s_g1[c.x];
      g0 = s_g0[c.x];
    } else {
      const LossCoef lc = loss_coef(sums, c.x, alpha, lam);
      g1 = lc.g1;
      g0 = lc.g0;
    }
    double gp = label_bit(gt, c, k, d, Nx, Ny, Nz) ? g1 : g0;
    double p = probs[t];
    dlogits[t] = (float)(gp * p * (1.0 - p) / B);  // sigmoid' = y(1-y) (neural.py:229-230)
  }
}

__global__ void loss_value_kernel(const double* __restrict__ sums, int B, double alpha, double lam,
                                  double* __restrict__ loss_out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double l = 0.0;
    for (int b = 0; b < B; ++b) l += loss_coef(sums, b, alpha, lam).loss;
    loss_out[0] = l / B;
  }
}

// ---- synthetic labels (row LBL) -------------------------------------------
// zfirst[b][x][y] = min{z : occ} or Nz
__global__ void zfirst_kernel(const uint8_t* __restrict__ bits, int B, int Nx, int Ny, int Nz, int* __restrict__ zf) {
  const long long total = (long long)B * Nx * Ny;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int y = t % Ny;
    long long r = t / Ny;
    int x = r % Nx;
    int b = (int)(r / Nx);
    int z = 0;
    for (; z < Nz; ++z)
      if ((__ldg(bits + bit_byte(b, x, y, z, Nx, Ny, Nz)) >> (x & 7)) & 1) break;
    zf[t] = z;
  }
}

__global__ void first_hit_kernel(const uint8_t* __restrict__ bits, int B, int Nx, int Ny, int Nz, int radius,
                                 const int* __restrict__ zf, uint8_t* __restrict__ out) {
  const int rb = Nx >> 3;
  const long long total = (long long)B * Nz * Ny * rb;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long r = t;
    int xb = r % rb; r /= rb;
    int y = r % Ny; r /= Ny;
    int z = r % Nz;
    int b = (int)(r / Nz);
    uint32_t occ = bits[t], v = 0;
    for (int i = 0; i < 8; ++i) {
      if (!((occ >> i) & 1)) continue;
      int x = xb * 8 + i;
      bool hit = false;
      for (int dx = -radius; dx <= radius && !hit; ++dx) {
        int xx = x + dx;
        if (xx < 0 || xx >= Nx) continue;
        for (int dy = -radius; dy <= radius; ++dy) {
          int yy = y + dy;
          if (yy < 0 || yy >= Ny) continue;
          if (zf[((long long)b * Nx + xx) * Ny + yy] == z) { hit = true; break; }
        }
      }
      if (hit) v |= 1u << i;
    }
    out[t] = (uint8_t)v;
  }
}

}  // namespace fpvs

using namespace fpvs;

// FPVS_SIMT_TAP=0 keeps the fp32 forward on the dense-K tile kernel (A/B checks)
static bool simt_tap_enabled() {
  static const bool on = [] {
    const char* e = getenv("FPVS_SIMT_TAP");
    return !(e && e[0] == '0');
  }();
  return on;
}

static int launch_simt(const void* x, int ldx, int in_dtype, const int32_t* nbr, int K, const int32_t* n_dev, int cap,
                       const float* w, int wmode, const float* bias, int cin, int cout, int act, const void* ymask,
                       int mask_bf16, int ldm, void* y, int ldy, int col_off, int out_dtype, cudaStream_t s) {
  if (in_dtype == FPVS_F32 && out_dtype == FPVS_F32 && wmode == 0 && !ymask && (cout == 32 || cout == 64) &&
      cin % 4 == 0 && cin <= kT2CinMax && K <= 32 && ldx % 4 == 0 && simt_tap_enabled()) {
    const int g2 = grid_for((cap + kT2M - 1) / kT2M, 1, 8);
    const size_t sh = sizeof(float) * (2 * kT2CinMax * (kT2M + 4) + 2 * kT2CinMax * cout) + sizeof(int) * kT2M * K;
    if (cout == 32) {
      set_smem_once<spconv_simt_tap_kernel<32>>(96 * 1024);
      spconv_simt_tap_kernel<32><<<g2, kT2M * 32 / 16, sh, s>>>((const float*)x, ldx, nbr, K, n_dev, cap, w, bias, cin,
                                                              cout, act, (float*)y, ldy, col_off);
    } else {
      set_smem_once<spconv_simt_tap_kernel<64>>(96 * 1024);
      spconv_simt_tap_kernel<64><<<g2, kT2M * 64 / 16, sh, s>>>((const float*)x, ldx, nbr, K, n_dev, cap, w, bias, cin,
                                                              cout, act, (float*)y, ldy, col_off);
    }
    FPVS_CHECK_LAUNCH("spconv_simt_tap");
    return FPVS_OK;
  }
  const long long tiles = (long long)((cap + kTM - 1) / kTM) * ((cout + kTN - 1) / kTN);
  const int g = grid_for(tiles, 1, 4);
#define FPVS_SIMT(TI, TO)                                                                                  \
  spconv_simt_kernel<TI, TO><<<g, 256, 0, s>>>((const TI*)x, ldx, nbr, K, n_dev, cap, w, wmode, bias, cin, \
                                              cout, act, ymask, mask_bf16, ldm, (TO*)y, ldy, col_off)
  if (in_dtype == FPVS_F32 && out_dtype == FPVS_F32) FPVS_SIMT(float, float);
  else if (in_dtype == FPVS_F32) FPVS_SIMT(float, __nv_bfloat16);
  else if (out_dtype == FPVS_F32) FPVS_SIMT(__nv_bfloat16, float);
  else FPVS_SIMT(__nv_bfloat16, __nv_bfloat16);
#undef FPVS_SIMT
  FPVS_CHECK_LAUNCH("spconv_simt");
  return FPVS_OK;
}

extern "C" int fpvs_spconv_simt(const void* x, int ldx, int in_dtype, const int32_t* nbr, int K,
                                const int32_t* n_out_dev, int cap_out, const float* w, const float* bias, int cin,
                                int cout, int act, void* y, int ldy, int col_off, int out_dtype, void* stream) {
  FPVS_CHECK_ARG(x && w && y && n_out_dev, "null pointer");
  FPVS_CHECK_ARG(K >= 1 && cin >= 1 && cout >= 1, "bad conv shape");
  FPVS_CHECK_ARG(nbr || K == 1, "nbr may be NULL only for K == 1");
  FPVS_CHECK_ARG(ldx >= cin && ldy >= col_off + cout, "bad leading dimension");
  if (cap_out <= 0) return FPVS_OK;
  return launch_simt(x, ldx, in_dtype, nbr, K, n_out_dev, cap_out, w, 0, bias, cin, cout, act, nullptr, 0, 0, y, ldy,
                     col_off, out_dtype, as_stream(stream));
}

extern "C" int fpvs_head_simt(const void* x, int ldx, int in_dtype, const int32_t* coords, const int32_t* n_dev,
                              int cap, const float* w, const float* bias, int cin, int d, int B, int Nx, int Ny,
                              int Nz, float tau, uint8_t* out_bits, float* probs, float* logits, void* stream) {
  FPVS_CHECK_ARG(x && coords && n_dev && w, "null pointer");
  FPVS_CHECK_ARG(Nx % 8 == 0, "N_x must be divisible by 8");
  (void)B;
  const int d3 = d * d * d;
  size_t smem = sizeof(float) * (size_t)(cin * d3 + d3);
  FPVS_CHECK_ARG(smem <= 48 * 1024, "head weights too large for the SIMT head");
  if (cap <= 0) return FPVS_OK;
  cudaStream_t s = as_stream(stream);
  int g = grid_for((long long)cap * d3, 256);
  if (in_dtype == FPVS_F32)
    head_simt_kernel<float><<<g, 256, smem, s>>>((const float*)x, ldx, (const int4*)coords, n_dev, cap, w, bias,
                                                 cin, d, Nx, Ny, Nz, tau, out_bits, probs, logits);
  else
    head_simt_kernel<__nv_bfloat16><<<g, 256, smem, s>>>((const __nv_bfloat16*)x, ldx, (const int4*)coords, n_dev,
                                                         cap, w, bias, cin, d, Nx, Ny, Nz, tau, out_bits, probs,
                                                         logits);
  FPVS_CHECK_LAUNCH("fpvs_head_simt");
  return FPVS_OK;
}

extern "C" int fpvs_spconv_dgrad_simt(const float* dz, int lddz, const int32_t* nbr, int K, const int32_t* n_dev,
                                      int cap, const float* w, int cin, int cout, const void* ymask, int mask_dtype,
                                      int ldm, float* dx, int lddx, void* stream) {
  FPVS_CHECK_ARG(dz && w && dx && n_dev, "null pointer");
  // the mirrored gather needs a symmetric map: K = k^3 submanifold taps, k odd
  int kk = 1;
  while (kk * kk * kk < K) kk += 2;
  FPVS_CHECK_ARG(kk * kk * kk == K, "dgrad supports symmetric subm maps (K = k^3, k odd), got K = %d", K);
  FPVS_CHECK_ARG(nbr || K == 1, "nbr may be NULL only for K == 1");
  if (cap <= 0) return FPVS_OK;
  // effective conv: input dz (Cin_eff = cout), output dx (Cout_eff = cin)
  FPVS_CHECK_ARG(mask_dtype == FPVS_F32 || mask_dtype == FPVS_BF16, "bad mask dtype");
  return launch_simt(dz, lddz, FPVS_F32, nbr, K, n_dev, cap, w, 1, nullptr, cout, cin, FPVS_ACT_NONE, ymask,
                     mask_dtype == FPVS_BF16, ldm, dx, lddx, 0, FPVS_F32, as_stream(stream));
}

extern "C" size_t fpvs_wgrad_workspace_size(int K, int cin, int cout, int cap) {
  (void)cap;
  return sizeof(float) * (size_t)kWgSplits * K * cin * cout;
}

extern "C" int fpvs_spconv_wgrad_simt(const void* x, int ldx, int x_dtype, const float* dz, int lddz,
                                      const int32_t* nbr, int K,
                                      const int32_t* n_dev, int cap, int cin, int cout, float* dw, float* db,
                                      void* workspace, size_t workspace_bytes, void* stream) {
  FPVS_CHECK_ARG(x && dz && dw && n_dev && workspace, "null pointer");
  FPVS_CHECK_ARG(nbr || K == 1, "nbr may be NULL only for K == 1");
  FPVS_CHECK_ARG(cin * cout <= 16 * 256, "wgrad SIMT supports Cin*Cout <= 4096");
  FPVS_CHECK_ARG(workspace_bytes >= fpvs_wgrad_workspace_size(K, cin, cout, cap), "workspace too small");
  cudaStream_t s = as_stream(stream);
  size_t smem = sizeof(float) * kWgRows * (cin + cout);
  FPVS_CHECK_ARG(x_dtype == FPVS_F32 || x_dtype == FPVS_BF16, "bad x dtype");
  if (x_dtype == FPVS_F32)
    wgrad_partial_kernel<float><<<K * kWgSplits, 256, smem, s>>>((const float*)x, ldx, dz, lddz, nbr, K, n_dev, cap,
                                                                 cin, cout, (float*)workspace);
  else
    wgrad_partial_kernel<__nv_bfloat16><<<K * kWgSplits, 256, smem, s>>>((const __nv_bfloat16*)x, ldx, dz, lddz, nbr,
                                                                         K, n_dev, cap, cin, cout, (float*)workspace);
  long long per = (long long)K * cin * cout;
  wgrad_reduce_kernel<<<grid_for(per, 256), 256, 0, s>>>((const float*)workspace, per, dw);
  if (db) bias_grad_kernel<<<cout < 148 ? cout : 148, 256, 0, s>>>(dz, lddz, n_dev, cap, cout, db);
  FPVS_CHECK_LAUNCH("fpvs_spconv_wgrad_simt");
  return FPVS_OK;
}

extern "C" size_t fpvs_loss_sums_size(int B, int cap) {
  // [B][3] results, cap double2 row partials, [B][LOSS_G][3] slice partials
  return sizeof(double) * (3 * (size_t)B + ((3 * (size_t)B) & 1) + 2 * (size_t)cap + 3 * (size_t)B * fpvs::LOSS_G);
}

extern "C" int fpvs_loss_counts(const float* probs, int C, const int32_t* coords, const int32_t* n_dev, int cap,
                                const uint8_t* gt_bits, int d, int B, int Nx, int Ny, int Nz, double* sums,
                                void* stream) {
  FPVS_CHECK_ARG(probs && coords && n_dev && gt_bits && sums, "null pointer");
  FPVS_CHECK_ARG(C == d * d * d, "C must equal d^3");
  FPVS_CHECK_ARG(Nx % 8 == 0, "N_x must be divisible by 8");
  cudaStream_t s = as_stream(stream);
  // sums layout: [B][3] results followed by cap double2 row partials
  double2* rows = reinterpret_cast<double2*>(sums + 3 * (size_t)B + ((3 * (size_t)B) & 1));
  loss_rows_kernel<<<grid_for(cap, 256), 256, 0, s>>>(probs, C, (const int4*)coords, n_dev, cap, gt_bits, d, Nx, Ny,
                                                      Nz, rows);
  double* part = reinterpret_cast<double*>(rows + cap);
  loss_sums_part_kernel<<<dim3(LOSS_G, B), 256, 0, s>>>(rows, (const int4*)coords, n_dev, cap, gt_bits,
                                                        (long long)(Nx / 8) * Ny * Nz, part);
  loss_sums_final_kernel<<<1, 32, 0, s>>>(part, B, sums);
  FPVS_CHECK_LAUNCH("fpvs_loss_counts");
  return FPVS_OK;
}

extern "C" int fpvs_loss_grad(const float* probs, int C, const int32_t* coords, const int32_t* n_dev, int cap,
                              const uint8_t* gt_bits, int d, int B, int Nx, int Ny, int Nz, const double* sums,
                              double alpha, double lam, float* dlogits, double* loss_out, void* stream) {
  FPVS_CHECK_ARG(probs && coords && n_dev && gt_bits && sums, "null pointer");
  cudaStream_t s = as_stream(stream);
  if (dlogits)
    loss_grad_kernel<<<grid_for((long long)cap * C, 256), 256, 0, s>>>(probs, C, (const int4*)coords, n_dev, cap,
                                                                       gt_bits, d, Nx, Ny, Nz, sums, B, alpha, lam,
                                                                       dlogits);
  if (loss_out) loss_value_kernel<<<1, 32, 0, s>>>(sums, B, alpha, lam, loss_out);
  FPVS_CHECK_LAUNCH("fpvs_loss_grad");
  return FPVS_OK;
}

extern "C" int fpvs_first_hit_labels(const uint8_t* bits, int B, int Nx, int Ny, int Nz, int radius,
                                     uint8_t* out_bits, int32_t* zfirst_ws, void* stream) {
  FPVS_CHECK_ARG(bits && out_bits && zfirst_ws, "null pointer");
  FPVS_CHECK_ARG(Nx % 8 == 0, "N_x must be divisible by 8");
  cudaStream_t s = as_stream(stream);
  zfirst_kernel<<<grid_for((long long)B * Nx * Ny, 256), 256, 0, s>>>(bits, B, Nx, Ny, Nz, zfirst_ws);
  first_hit_kernel<<<grid_for((long long)B * Nz * Ny * (Nx / 8), 256), 256, 0, s>>>(bits, B, Nx, Ny, Nz, radius,
                                                                                     zfirst_ws, out_bits);
  FPVS_CHECK_LAUNCH("fpvs_first_hit_labels");
  return FPVS_OK;
}

extern "C" int fpvs_head_rows(const float* logits, int ld, const int32_t* coords, const int32_t* n_dev, int cap, int d,
                              int B, int Nx, int Ny, int Nz, float tau, uint8_t* out_bits, float* probs,
                              void* stream) {
  FPVS_CHECK_ARG(logits && coords && n_dev, "null pointer");
  FPVS_CHECK_ARG(Nx % 8 == 0, "N_x must be divisible by 8");
  FPVS_CHECK_ARG(d >= 1 && ld >= d * d * d, "bad logits leading dimension");
  (void)B;
  if (cap <= 0) return FPVS_OK;
  const int d3 = d * d * d;
  head_rows_kernel<<<grid_for((long long)cap * d3, 256), 256, 0, as_stream(stream)>>>(
      logits, ld, (const int4*)coords, n_dev, cap, d, Nx, Ny, Nz, tau, out_bits, probs);
  FPVS_CHECK_LAUNCH("fpvs_head_rows");
  return FPVS_OK;
}

extern "C" int fpvs_act_backward(const float* dy, int lddy, const void* y, int y_dtype, int ldy, const int32_t* n_dev,
                                 int cap, int C, int act, float* dz, int lddz, void* stream) {
  FPVS_CHECK_ARG(dy && y && dz && n_dev, "null pointer");
  FPVS_CHECK_ARG(C >= 1 && lddy >= C && ldy >= C && lddz >= C, "bad leading dimension");
  FPVS_CHECK_ARG(act == FPVS_ACT_NONE || act == FPVS_ACT_RELU || act == FPVS_ACT_SIGMOID, "bad activation");
  FPVS_CHECK_ARG(y_dtype == FPVS_F32 || y_dtype == FPVS_BF16, "bad y dtype");
  if (cap <= 0) return FPVS_OK;
  const int g = grid_for((long long)cap * C, 256);
  cudaStream_t s = as_stream(stream);
  if (y_dtype == FPVS_F32)
    act_backward_kernel<float><<<g, 256, 0, s>>>(dy, lddy, (const float*)y, ldy, n_dev, cap, C, act, dz, lddz);
  else
    act_backward_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(dy, lddy, (const __nv_bfloat16*)y, ldy, n_dev, cap, C, act,
                                                         dz, lddz);
  FPVS_CHECK_LAUNCH("fpvs_act_backward");
  return FPVS_OK;
}
