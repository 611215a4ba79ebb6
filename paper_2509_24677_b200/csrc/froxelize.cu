// Perspective froxelization on sm_100a.
//
// Replaces froxel.py:387-394 froxelize() in "perspective" mode: every scene
// triangle is moved to camera space, culled and clipped against the near
// plane (froxel.py:292-325, Sutherland-Hodgman 203-219), projected to the
// supersampled screen, rasterized at pixel centres with inclusive edge tests
// (froxel.py:229-285), its perspective-correct depth quantized into a froxel
// (froxel.py:28-42, 328-348) whose bit is OR-ed into the packed grid.
//
// Bit parity.  The reference computes in float64 with numpy, one rounding
// per operation; every expression below uses the explicit-rounding
// intrinsics (__dadd_rn, __dmul_rn, __ddiv_rn ...) in the reference's
// evaluation order, so the compiler can neither contract nor reassociate.
// The one place numpy fuses is the camera transform: (v - o) @ basis.T goes
// through the BLAS dgemm kernel, which accumulates the k = 3 dot product as
// fma(d2, b2, fma(d1, b1, d0 * b0)); cam_xyz() restates that order.
//
// Kernels (one stream, three launches after the output memset; the span
// raster below replaced the whole-bounding-box raster as the default, which
// stays selectable with FPVS_FROX_SPANS=0 for A/B checks):
//  1. setup: one thread per scene triangle -> up to two clipped screen
//     triangles (slots 2t, 2t+1) with their edge/depth constants and pixel
//     bounding box; each CTA also scans its 512 slots' sample counts
//     (bbox area) into a block-local inclusive prefix + the block total.
//  2. scan: one CTA turns the block totals into exclusive block offsets and
//     the grand total of candidate samples.
//  3. span raster (span_kernel): work items are bounding-box rows cut into
//     16-column segments (64 for the GT z-buffer); a warp bounds its 32
//     items' candidate columns by the three edge functions (row_span,
//     conservative) and expands them into samples 32 at a time, so samples
//     outside the triangle are never evaluated.
//     Whole-box raster (raster_kernel): persistent CTAs walk the flat sample space in 2048-sample
//     chunks; each thread finds its slot by a two-level binary search
//     (block offsets, then the block-local prefix), caches the slot's
//     constants while consecutive samples stay inside it, evaluates the
//     coverage/depth test and atomically ORs the froxel's bit into the
//     32-bit word that holds it.  Work per chunk is uniform no matter how
//     large or small the triangles are (a floor quad of 10^6 samples and
//     10^4 slivers of one sample cost the same per sample).
#include "common.cuh"

namespace fpvs {
namespace frox {

constexpr int kSetupThreads = 64;
constexpr int kSlotsPerBlock = 2 * kSetupThreads;
constexpr int kRasterThreads = 256;
constexpr int kPerThread = 8;
constexpr int kChunk = kRasterThreads * kPerThread;
constexpr double kDegenEps = 1e-12;  // froxel.py:23

struct __align__(16) Slot {
  double v0x, v0y, e1x, e1y, e2x, e2y, den;
  double iz0, iz1, iz2;  // 1/z per vertex
  double wv0, wv1, wv2;  // per-vertex depth coordinate
  double rden;           // 1/den, for the filtered fast path only
  double wtol;           // relative depth tolerance of the fast path (scales with zmax/zmin)
  int x0, y0, w, h;
  unsigned int wmagic;  // ceil(2^32 / w): row = umulhi(r, wmagic) +-1
  int pad;
};
static_assert(sizeof(Slot) == 144, "slot record");

struct Params {
  double o[3], b[9];
  double h, nearz, farz;
  double sx, sy;   // supersampled screen size (as float64, as the reference multiplies)
  int isx, isy;
  int nx, ny, nz;
  int depth_log;
  int rows_mode;  // 1: the flat work space counts bounding-box row segments (span raster), 0: samples
  int seg;        // span raster: columns per work item
};

struct Work {
  Slot* slots;
  unsigned long long* lp;    // [2T] block-local inclusive prefix of slot sample counts
  unsigned long long* bsum;  // [nb]
  unsigned long long* bpre;  // [nb] exclusive block offsets
  unsigned long long* total;
  unsigned long long* nsamples;  // candidate samples (bbox areas), next to total
  unsigned int* out_words;
  int* tabx;  // froxel column of supersampled pixel column px (quantize of (px+0.5)/sx)
  int* taby;
  const unsigned int* pvs_words;  // kMode 1: the PVS grid whose froxels keep their primitives
  uint8_t* kept;                  // kMode 1: per scene triangle, 1 = touches a PVS froxel
  long long* pairs;               // kMode 2: (froxel * T + triangle) per fragment
  unsigned long long* npairs;
  long long pair_cap;
  double* oframe;  // ortho mode: lo[3], spacing of the frustum's world AABB (written by the setup)
  double* ufx;  // GT mode: 2 (px + 0.5) / W - 1 per pixel column (core.py:441), nullptr otherwise
  double* ufy;
  long long ntris;
  int nb;
};

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

struct V3 {
  double x, y, z;
};

// (v - o) @ basis.T, with dgemm's k = 3 accumulation order (froxel.py:288-289).
__device__ __forceinline__ V3 cam_xyz(const Params& p, const double* v) {
  const double d0 = dsub(v[0], p.o[0]), d1 = dsub(v[1], p.o[1]), d2 = dsub(v[2], p.o[2]);
  V3 c;
  c.x = __fma_rn(d2, p.b[2], __fma_rn(d1, p.b[1], dmul(d0, p.b[0])));
  c.y = __fma_rn(d2, p.b[5], __fma_rn(d1, p.b[4], dmul(d0, p.b[3])));
  c.z = __fma_rn(d2, p.b[8], __fma_rn(d1, p.b[7], dmul(d0, p.b[6])));
  return c;
}

// p + t * (q - p) per component (froxel.py:218).
__device__ __forceinline__ V3 lerp(const V3& p, const V3& q, double t) {
  return V3{dadd(p.x, dmul(t, dsub(q.x, p.x))), dadd(p.y, dmul(t, dsub(q.y, p.y))),
            dadd(p.z, dmul(t, dsub(q.z, p.z)))};
}

// Screen triangle (a, b, c) in camera space -> slot constants; returns the
// sample count (0 when culled as degenerate or off-screen).
__device__ unsigned long long make_slot(const Params& p, const V3& a, const V3& b, const V3& c, Slot& s) {
  const V3 v[3] = {a, b, c};
  double u[3], vv[3], iz[3], wv[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    // u = (0.5 + 0.5 * x / (z * h)) * W   (froxel.py:322-323)
    const double zh = dmul(v[k].z, p.h);
    u[k] = dmul(dadd(0.5, ddiv(dmul(0.5, v[k].x), zh)), p.sx);
    vv[k] = dmul(dadd(0.5, ddiv(dmul(0.5, v[k].y), zh)), p.sy);
    iz[k] = ddiv(1.0, v[k].z);
    // froxel.py:335-338
    if (p.depth_log)
      wv[k] = ddiv(log(ddiv(1.0, dmul(iz[k], p.nearz))), log(ddiv(p.farz, p.nearz)));
    else
      wv[k] = ddiv(dsub(ddiv(1.0, iz[k]), p.nearz), dsub(p.farz, p.nearz));
  }
  // froxel.py:243-259
  s.v0x = u[0];
  s.v0y = vv[0];
  s.e1x = dsub(u[1], u[0]);
  s.e1y = dsub(vv[1], vv[0]);
  s.e2x = dsub(u[2], u[0]);
  s.e2y = dsub(vv[2], vv[0]);
  s.den = dsub(dmul(s.e1x, s.e2y), dmul(s.e2x, s.e1y));
  s.iz0 = iz[0];
  s.iz1 = iz[1];
  s.iz2 = iz[2];
  s.wv0 = wv[0];
  s.wv1 = wv[1];
  s.wv2 = wv[2];
  s.rden = 1.0 / s.den;
  {
    const double izmax = fmax(fmax(iz[0], iz[1]), iz[2]), izmin = fmin(fmin(iz[0], iz[1]), iz[2]);
    s.wtol = 1e-12 * (izmax / izmin);
  }
  const double minx = fmin(fmin(u[0], u[1]), u[2]), maxx = fmax(fmax(u[0], u[1]), u[2]);
  const double miny = fmin(fmin(vv[0], vv[1]), vv[2]), maxy = fmax(fmax(vv[0], vv[1]), vv[2]);
  const double x0 = fmin(fmax(ceil(dsub(minx, 0.5)), 0.0), p.sx);
  const double x1 = fmin(fmax(dadd(floor(dsub(maxx, 0.5)), 1.0), 0.0), p.sx);
  const double y0 = fmin(fmax(ceil(dsub(miny, 0.5)), 0.0), p.sy);
  const double y1 = fmin(fmax(dadd(floor(dsub(maxy, 0.5)), 1.0), 0.0), p.sy);
  const int ix0 = (int)x0, ix1 = (int)x1, iy0 = (int)y0, iy1 = (int)y1;
  s.x0 = ix0;
  s.y0 = iy0;
  s.w = max(ix1 - ix0, 0);
  s.h = max(iy1 - iy0, 0);
  const bool live = fabs(s.den) > kDegenEps && s.w > 0 && s.h > 0;
  if (!live) s.w = s.h = 0;
  s.wmagic = s.w > 1 ? (unsigned int)((0x100000000ull + (unsigned long long)s.w - 1) / (unsigned long long)s.w)
                     : 0xffffffffu;
  return (unsigned long long)s.w * (unsigned long long)s.h;
}

// Store a thread's two slots, count its work items and scan the block's
// counts into the block-local prefix (shared by every setup kernel).
__device__ __forceinline__ void finish_setup(const Params& p, const Work& wk, long long t, unsigned long long c0,
                                             unsigned long long c1, Slot& s0, Slot& s1) {
  if (t < wk.ntris) {
    if (c0) wk.slots[2 * t] = s0;
    if (c1) wk.slots[2 * t + 1] = s1;
  }
  {
    // candidate samples (bbox areas) for the statistics counter
    unsigned long long smp = c0 + c1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) smp += __shfl_xor_sync(0xffffffffu, smp, o);
    if ((threadIdx.x & 31) == 0 && smp) atomicAdd(wk.nsamples, smp);
  }
  if (p.rows_mode) {
    // the span raster's work items: bounding-box rows cut into p.seg-column
    // segments (h * ceil(w / seg) per slot); wmagic becomes the segment
    // count's reciprocal for the item -> (row, segment) split
    if (c0) {
      const unsigned int ns = (unsigned int)(s0.w + p.seg - 1) / (unsigned int)p.seg;
      c0 = (unsigned long long)s0.h * ns;
      s0.wmagic = ns > 1 ? (unsigned int)((0x100000000ull + ns - 1) / ns) : 0xffffffffu;
      if (t < wk.ntris) wk.slots[2 * t].wmagic = s0.wmagic;
    }
    if (c1) {
      const unsigned int ns = (unsigned int)(s1.w + p.seg - 1) / (unsigned int)p.seg;
      c1 = (unsigned long long)s1.h * ns;
      s1.wmagic = ns > 1 ? (unsigned int)((0x100000000ull + ns - 1) / ns) : 0xffffffffu;
      if (t < wk.ntris) wk.slots[2 * t + 1].wmagic = s1.wmagic;
    }
  }
  // block scan of (c0 + c1)
  __shared__ unsigned long long warp_tot[kSetupThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long incl = c0 + c1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  unsigned long long base = 0, btot = 0;
#pragma unroll
  for (int i = 0; i < kSetupThreads / 32; ++i) {
    if (i < wid) base += warp_tot[i];
    btot += warp_tot[i];
  }
  const unsigned long long excl = base + incl - (c0 + c1);
  if (t < wk.ntris) {
    wk.lp[2 * t] = excl + c0;
    wk.lp[2 * t + 1] = excl + c0 + c1;
  }
  if (threadIdx.x == 0) wk.bsum[blockIdx.x] = btot;
}

// One thread per (view, scene triangle); flat index f = view * T + tri, slots
// 2f and 2f+1.  kMulti: the view's frustum comes from views[f / T] (GT-PVS
// cameras); else from p (froxelize).  Slot.pad records the view.
template <bool kMulti>
__global__ void __launch_bounds__(kSetupThreads) setup_kernel(Params p, const fpvs_frustum* __restrict__ views,
                                                              const double* __restrict__ verts, long long nverts,
                                                              const int64_t* __restrict__ tris, long long T, Work wk) {
  const long long t = (long long)blockIdx.x * kSetupThreads + threadIdx.x;
  Slot s0, s1;
  unsigned long long c0 = 0, c1 = 0;
  int view = 0;
  if (t < wk.ntris) {
    long long tri = t;
    if (kMulti) {
      view = (int)(t / T);
      tri = t - (long long)view * T;
      const fpvs_frustum& f = views[view];
#pragma unroll
      for (int i = 0; i < 3; ++i) p.o[i] = f.origin[i];
#pragma unroll
      for (int i = 0; i < 9; ++i) p.b[i] = f.basis[i];
      p.h = f.half_extent;
      p.nearz = f.near_z;
      p.farz = f.far_z;
    }
    long long id[3];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      id[k] = tris[tri * 3 + k];
      ok &= id[k] >= 0 && id[k] < nverts;
    }
    if (ok) {
      V3 c[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) c[k] = cam_xyz(p, verts + id[k] * 3);
      const double zmin = fmin(fmin(c[0].z, c[1].z), c[2].z);
      const double zmax = fmax(fmax(c[0].z, c[1].z), c[2].z);
      if (zmax > p.nearz && zmin < p.farz) {  // froxel.py:307
        if (zmin >= p.nearz) {
          c0 = make_slot(p, c[0], c[1], c[2], s0);
        } else {
          // Sutherland-Hodgman against z - near >= 0 (froxel.py:203-219), fan (p0, pk, pk+1)
          V3 poly[4];
          int n = 0;
          double d[3];
#pragma unroll
          for (int k = 0; k < 3; ++k) d[k] = dsub(c[k].z, p.nearz);
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const int j = (i + 1) % 3;
            if (d[i] >= 0) poly[n++] = c[i];
            if ((d[i] >= 0) != (d[j] >= 0)) poly[n++] = lerp(c[i], c[j], ddiv(d[i], dsub(d[i], d[j])));
          }
          if (n >= 3) c0 = make_slot(p, poly[0], poly[1], poly[2], s0);
          if (n >= 4) c1 = make_slot(p, poly[0], poly[2], poly[3], s1);
        }
      }
    }
    s0.pad = s1.pad = view;
  }
  finish_setup(p, wk, t, c0, c1, s0, s1);
}

__global__ void __launch_bounds__(1024) scan_kernel(Params p, Work wk) {
  // pixel column/row -> froxel index, exactly quantize((px + 0.5) / sx) (froxel.py:28-42, 345-346)
  if (wk.ufx) {
    for (int i = threadIdx.x; i < (int)p.sx; i += 1024)
      wk.ufx[i] = dsub(ddiv(dmul(2.0, dadd((double)i, 0.5)), p.sx), 1.0);
    for (int i = threadIdx.x; i < (int)p.sy; i += 1024)
      wk.ufy[i] = dsub(ddiv(dmul(2.0, dadd((double)i, 0.5)), p.sy), 1.0);
  }
  for (int i = threadIdx.x; i < p.isx; i += 1024)
    wk.tabx[i] = min(max((int)floor(dmul(ddiv(dadd((double)i, 0.5), p.sx), (double)p.nx)), 0), p.nx - 1);
  for (int i = threadIdx.x; i < p.isy; i += 1024)
    wk.taby[i] = min(max((int)floor(dmul(ddiv(dadd((double)i, 0.5), p.sy), (double)p.ny)), 0), p.ny - 1);
  __shared__ unsigned long long warp_tot[32];
  __shared__ unsigned long long carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < wk.nb; b0 += 1024) {
    const int b = b0 + threadIdx.x;
    const unsigned long long v = b < wk.nb ? wk.bsum[b] : 0;
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    unsigned long long base = carry, tot = 0;
    for (int i = 0; i < 32; ++i) {
      if (i < wid) base += warp_tot[i];
      tot += warp_tot[i];
    }
    if (b < wk.nb) wk.bpre[b] = base + incl - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *wk.total = carry;
}

// Slot holding flat sample g (g < total): largest block b with bpre[b] <= g,
// then the first slot of that block whose inclusive local prefix exceeds
// g - bpre[b].  Returns the slot and its exclusive global start.
__device__ __forceinline__ long long find_slot(const Work& wk, unsigned long long g, unsigned long long& start) {
  int lo = 0, hi = wk.nb - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(wk.bpre + mid) <= g) lo = mid;
    else hi = mid - 1;
  }
  const unsigned long long bp = __ldg(wk.bpre + lo);
  const unsigned long long local = g - bp;
  long long a = (long long)lo * kSlotsPerBlock;
  long long z = min(a + kSlotsPerBlock, 2 * wk.ntris) - 1;  // ntris = views x scene triangles
  const long long first = a;
  while (a < z) {
    const long long mid = (a + z) >> 1;
    if (__ldg(wk.lp + mid) > local) z = mid;
    else a = mid + 1;
  }
  start = bp + (a > first ? __ldg(wk.lp + a - 1) : 0ull);
  return a;
}

// The reference's own expression sequence for one sample (froxel.py:272-279,
// 340-344; quantize 28-42).  Returns the depth layer, or -1 when the sample
// is outside the triangle or the depth range.
__device__ __forceinline__ int sample_exact(const Slot& s, double cx, double cy, int nz) {
  const double dx = dsub(cx, s.v0x), dy = dsub(cy, s.v0y);
  const double b1 = ddiv(dsub(dmul(dx, s.e2y), dmul(s.e2x, dy)), s.den);
  const double b2 = ddiv(dsub(dmul(s.e1x, dy), dmul(dx, s.e1y)), s.den);
  const double b0 = dsub(dsub(1.0, b1), b2);
  if (!(b0 >= 0 && b1 >= 0 && b2 >= 0)) return -1;
  const double inv = dadd(dadd(s.iz0, dmul(b1, dsub(s.iz1, s.iz0))), dmul(b2, dsub(s.iz2, s.iz0)));
  const double w1 = ddiv(dmul(b1, s.iz1), inv), w2 = ddiv(dmul(b2, s.iz2), inv);
  const double w = dadd(dadd(s.wv0, dmul(w1, dsub(s.wv1, s.wv0))), dmul(w2, dsub(s.wv2, s.wv0)));
  if (!(w >= 0 && w <= 1)) return -1;
  return min(max((int)floor(dmul(w, (double)nz)), 0), nz - 1);
}

__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = __fma_rn(-x, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-x, r, 1.0);
  return __fma_rn(r, e, r);
}

// Filtered evaluation: decides with no division whenever the decision is
// provably the one sample_exact makes, else defers to it.  Returns the depth
// layer, -1 for a dropped sample.
//  * b1 >= 0 / b2 >= 0: the sign of the rounded numerator (computed exactly
//    as the reference does) is the sign of the rounded quotient, barring
//    underflow (|n| tiny -> exact path);
//  * b0 and the depth w from q = n * (1/den) and an approximate 1/inv: their
//    error is ~1e-15 relative (w: times zmax/zmin, folded into s.wtol), so a
//    decision more than 1e-13 / wtol away from its boundary (b0 = 0, w = 0,
//    w = 1, w * nz integral) cannot flip; closer samples take the exact path.
__device__ __forceinline__ int sample_fast(const Slot& s, double cx, double cy, int nz) {
  const double dx = dsub(cx, s.v0x), dy = dsub(cy, s.v0y);
  const double n1 = dsub(dmul(dx, s.e2y), dmul(s.e2x, dy));
  const double n2 = dsub(dmul(s.e1x, dy), dmul(dx, s.e1y));
  const bool dneg = s.den < 0;
  const double a1 = fabs(n1), a2 = fabs(n2);
  constexpr double kTiny = 1e-250;
  if ((a1 != 0 && a1 < kTiny) || (a2 != 0 && a2 < kTiny)) return sample_exact(s, cx, cy, nz);
  if ((n1 != 0 && ((n1 < 0) != dneg)) || (n2 != 0 && ((n2 < 0) != dneg))) return -1;
  const double q1 = n1 * s.rden, q2 = n2 * s.rden;  // >= 0 here
  const double a0 = (1.0 - q1) - q2;
  const double m0 = 1e-13 * (1.0 + q1 + q2);
  if (a0 < -m0) return -1;
  if (a0 <= m0) return sample_exact(s, cx, cy, nz);
  const double inv = __fma_rn(q2, s.iz2 - s.iz0, __fma_rn(q1, s.iz1 - s.iz0, s.iz0));
  const double r = rcp_nr(inv);
  const double w1 = q1 * s.iz1 * r, w2 = q2 * s.iz2 * r;
  const double d1 = s.wv1 - s.wv0, d2 = s.wv2 - s.wv0;
  const double w = __fma_rn(w2, d2, __fma_rn(w1, d1, s.wv0));
  const double mw = s.wtol * (1.0 + fabs(s.wv0) + w1 * fabs(d1) + w2 * fabs(d2));
  if (w < -mw || w > 1.0 + mw) return -1;
  const double t = w * (double)nz, f = floor(t);
  const double mt = mw * (double)nz + 1e-15 * t;
  if (w <= mw || w >= 1.0 - mw || t - f <= mt || f + 1.0 - t <= mt) return sample_exact(s, cx, cy, nz);
  return min(max((int)f, 0), nz - 1);
}

// OR bits into a grid word, skipping the atomic when a (possibly stale, L1)
// read already shows them: bits are only ever set during a pass, so a set
// bit in any copy is set in memory, and a miss just costs the atomic.  Most
// fragments hit froxels other fragments already marked; the contended
// same-address atomics at L2 were the cost.
__device__ __forceinline__ void or_bits(unsigned int* w, unsigned int bits) {
  if ((*reinterpret_cast<volatile unsigned int*>(w) & bits) != bits) atomicOr(w, bits);
}

// (double)px + 0.5 without the int->fp64 converter: 2^52 + px from the bit
// pattern, minus (2^52 - 0.5); both steps are exact for 0 <= px < 2^31.
__device__ __forceinline__ double centre(int px) {
  return __dsub_rn(__hiloint2double(0x43300000, px), 4503599627370495.5);
}

// Global inclusive end of slot sl's sample range.
__device__ __forceinline__ unsigned long long slot_end(const Work& wk, long long sl) {
  return __ldg(wk.bpre + sl / kSlotsPerBlock) + __ldg(wk.lp + sl);
}

// Each warp rasterizes 32 * kPerThread consecutive samples, 32 at a time
// (lane = sample), so the lanes of one step share a slot or walk forward to
// the next few; only the warp's first sample needs the binary search.
// kMode 0: OR fragment bits into the grid (froxelize); 1: mark the triangles
// with a fragment in a PVS froxel (cull, evalrt.py:62-68); 2: emit (froxel,
// triangle) fragment pairs (froxel_id_map, froxel.py:397-417).
template <bool kFilter, int kMode>
__global__ void __launch_bounds__(kRasterThreads, 4) raster_kernel(Params p, Work wk) {
  constexpr int kWarpSpan = 32 * kPerThread;
  const unsigned long long total = *wk.total;
  const unsigned int row = (unsigned int)(p.nx >> 3);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long have = -1;  // slot whose constants are in s
  Slot s;
  for (unsigned long long c0 = (unsigned long long)blockIdx.x * kChunk; c0 < total;
       c0 += (unsigned long long)gridDim.x * kChunk) {
    const unsigned long long wbase = c0 + (unsigned long long)warp * kWarpSpan;
    if (wbase >= total) break;  // warp-uniform
    unsigned long long cs = 0;
    long long cur = 0;
    if (lane == 0) cur = find_slot(wk, wbase, cs);
    cur = __shfl_sync(0xffffffffu, cur, 0);
    cs = __shfl_sync(0xffffffffu, cs, 0);
    unsigned long long ce = slot_end(wk, cur);
#pragma unroll 1
    for (int k = 0; k < kPerThread; ++k) {
      const unsigned long long g = wbase + (unsigned long long)(k * 32 + lane);
      bool valid = g < total;
      unsigned int word = 0, bit = 0;
      long long mine = cur, flat = 0;
      if (valid) {
        unsigned long long ms = cs, me = ce;
        // walk a few slots forward (odd slots of unclipped triangles are
        // empty), then fall back to the search (long zero-count runs)
        int steps = 0;
        while (g >= me && steps < 4) {
          ms = me;
          me = slot_end(wk, ++mine);
          ++steps;
        }
        if (g >= me) {
          mine = find_slot(wk, g, ms);
          me = slot_end(wk, mine);
        }
        if (mine != have) {
          s = wk.slots[mine];
          have = mine;
        }
        const unsigned int r = (unsigned int)(g - ms);
        unsigned int ry = __umulhi(r, s.wmagic);
        const int rem = (int)(r - ry * (unsigned int)s.w);
        if (rem < 0) --ry;
        else if (rem >= s.w) ++ry;
        const int px = s.x0 + (int)(r - ry * (unsigned int)s.w);
        const int py = s.y0 + (int)ry;
        const double cx = centre(px), cy = centre(py);
        const int iz = kFilter ? sample_fast(s, cx, cy, p.nz) : sample_exact(s, cx, cy, p.nz);
        valid = iz >= 0;
        if (valid) {
          const int ix = __ldg(wk.tabx + px), iy = __ldg(wk.taby + py);
          const unsigned long long byte = (unsigned long long)(ix >> 3) +
                                          (unsigned long long)row * ((unsigned long long)iy + (unsigned long long)p.ny * iz);
          word = (unsigned int)(byte >> 2);
          bit = 1u << ((((unsigned int)byte & 3u) << 3) | ((unsigned int)ix & 7u));
          if (kMode == 2) flat = ix + (long long)p.nx * (iy + (long long)p.ny * iz);  // froxel.py:411
        }
      }
      // the warp's next step starts from the last lane's slot
      const long long nxt = __shfl_sync(0xffffffffu, mine, 31);
      if (nxt != cur) {
        cur = nxt;
        cs = (cur % kSlotsPerBlock ? slot_end(wk, cur - 1) : __ldg(wk.bpre + cur / kSlotsPerBlock));
        ce = slot_end(wk, cur);
      }
      if (kMode == 0) {
        // warp-combined OR: one atomic when every covered lane hits the same word
        const unsigned int vm = __ballot_sync(0xffffffffu, valid);
        if (vm) {
          const int leader = __ffs(vm) - 1;
          const unsigned int w0 = __shfl_sync(0xffffffffu, word, leader);
          if (__all_sync(0xffffffffu, !valid || word == w0)) {
            const unsigned int bits = __reduce_or_sync(0xffffffffu, valid ? bit : 0u);
            if (lane == leader) atomicOr(wk.out_words + w0, bits);
          } else if (valid) {
            atomicOr(wk.out_words + word, bit);
          }
        }
      } else if (kMode == 1) {
        if (valid && (__ldg(wk.pvs_words + word) & bit)) wk.kept[mine >> 1] = 1;
      } else {
        // one pair per distinct (froxel, triangle) among the warp's lanes
        const long long key = valid ? flat * wk.ntris + (mine >> 1) : -1 - lane;
        const unsigned int peers = __match_any_sync(0xffffffffu, key);
        if (valid && (__ffs(peers) - 1) == lane) {
          const unsigned long long slot = atomicAdd(wk.npairs, 1ull);
          if ((long long)slot < wk.pair_cap) wk.pairs[slot] = key;
        }
      }
    }
  }
}

struct GtParams {
  double fo[3], fb[9];
  double fh, fnear, ffar, flogr;  // flogr = log(far / near), computed like math.log on the host
  double W, H;
  int iw, ih;
  int nx, ny, nz, depth_log;
  long long T;     // scene triangles (per camera)
  long long npix;  // W * H
};

// Coverage and the reference barycentrics (froxel.py:272-279): false when
// the sample is outside; samples provably outside skip the divisions.
__device__ __forceinline__ bool bary_filtered(const Slot& s, double cx, double cy, double& b1, double& b2) {
  const double dx = dsub(cx, s.v0x), dy = dsub(cy, s.v0y);
  const double n1 = dsub(dmul(dx, s.e2y), dmul(s.e2x, dy));
  const double n2 = dsub(dmul(s.e1x, dy), dmul(dx, s.e1y));
  const bool dneg = s.den < 0;
  const double a1 = fabs(n1), a2 = fabs(n2);
  constexpr double kTiny = 1e-250;
  if (!((a1 != 0 && a1 < kTiny) || (a2 != 0 && a2 < kTiny))) {
    if ((n1 != 0 && ((n1 < 0) != dneg)) || (n2 != 0 && ((n2 < 0) != dneg))) return false;
    const double q1 = n1 * s.rden, q2 = n2 * s.rden;
    if ((1.0 - q1) - q2 < -1e-13 * (1.0 + q1 + q2)) return false;
  }
  b1 = ddiv(n1, s.den);
  b2 = ddiv(n2, s.den);
  const double b0 = dsub(dsub(1.0, b1), b2);
  return b0 >= 0 && b1 >= 0 && b2 >= 0;
}

// The orthographic frame of froxel.py:355-358: the frustum's world AABB
// (core.py:349-354, unproject_ndc of the 8 NDC corners in linear depth, the
// corner product in dgemm k = 3 order), the sample spacing and the per-axis
// sample counts.
__device__ __forceinline__ void ortho_frame(const GtParams& g, int supersample, double lo[3], double hi[3],
                                            double& spacing, int counts[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    lo[k] = __longlong_as_double(0x7ff0000000000000LL);
    hi[k] = -lo[k];
  }
  for (int c = 0; c < 8; ++c) {
    const double u = (double)((c >> 2) & 1), v = (double)((c >> 1) & 1), w = (double)(c & 1);
    const double z = dadd(g.fnear, dmul(w, dsub(g.ffar, g.fnear)));
    const double x = dmul(dmul(dsub(dmul(2.0, u), 1.0), g.fh), z);
    const double y = dmul(dmul(dsub(dmul(2.0, v), 1.0), g.fh), z);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double wk = dadd(g.fo[k], __fma_rn(z, g.fb[6 + k], __fma_rn(y, g.fb[3 + k], dmul(x, g.fb[k]))));
      lo[k] = fmin(lo[k], wk);
      hi[k] = fmax(hi[k], wk);
    }
  }
  const double e0 = dsub(hi[0], lo[0]), e1 = dsub(hi[1], lo[1]), e2 = dsub(hi[2], lo[2]);
  const int dmax = max(g.nx, max(g.ny, g.nz));
  spacing = ddiv(fmax(e0, fmax(e1, e2)), (double)(supersample * dmax));
  const double e[3] = {e0, e1, e2};
#pragma unroll
  for (int k = 0; k < 3; ++k) counts[k] = max((int)ceil(ddiv(e[k], spacing)), 1);
}

__device__ __forceinline__ int quant_fast(double a, int n, double m);
__device__ __forceinline__ int quant_exact(double a, int n);

// project_points (core.py:380-405) of a world point into the frustum, then
// quantize (froxel.py:28-42): froxel (ix, iy, iz) or false when outside.
// Same filtered divisions as resolve_kernel.
__device__ __forceinline__ bool project_quantize(const GtParams& g, double wx, double wy, double wz, int& ix,
                                                 int& iy, int& iz) {
  constexpr double kM = 1e-12;
  const double d0 = dsub(wx, g.fo[0]), d1 = dsub(wy, g.fo[1]), d2 = dsub(wz, g.fo[2]);
  const double lx = __fma_rn(d2, g.fb[2], __fma_rn(d1, g.fb[1], dmul(d0, g.fb[0])));
  const double ly = __fma_rn(d2, g.fb[5], __fma_rn(d1, g.fb[4], dmul(d0, g.fb[3])));
  const double lz = __fma_rn(d2, g.fb[8], __fma_rn(d1, g.fb[7], dmul(d0, g.fb[6])));
  if (!(lz > 0)) return false;
  const double zh = dmul(lz, g.fh);
  const double r = rcp_nr(zh);
  const double rfn = 1.0 / dsub(g.ffar, g.fnear);
  ix = quant_fast(0.5 + (0.5 * lx) * r, g.nx, kM);
  iy = ix == -1 ? -1 : quant_fast(0.5 + (0.5 * ly) * r, g.ny, kM);
  iz = (ix == -1 || iy == -1 || g.depth_log) ? -2 : quant_fast((lz - g.fnear) * rfn, g.nz, kM);
  if (ix == -2) ix = quant_exact(dadd(0.5, ddiv(dmul(0.5, lx), zh)), g.nx);
  if (iy == -2) iy = quant_exact(dadd(0.5, ddiv(dmul(0.5, ly), zh)), g.ny);
  if (iz == -2 && ix >= 0 && iy >= 0)
    iz = quant_exact(g.depth_log ? ddiv(log(ddiv(lz, g.fnear)), g.flogr)
                                 : ddiv(dsub(lz, g.fnear), dsub(g.ffar, g.fnear)), g.nz);
  return ix >= 0 && iy >= 0 && iz >= 0;
}

// Orthographic passes (froxel.py:351-376): one thread per (pass, scene
// triangle), flat index f = pass * T + tri, slot 2f (2f + 1 stays empty).
// Pass 0/1/2 rasterizes axes (1,2)/(2,0)/(0,1) of the world AABB at the
// sample spacing and interpolates axis 0/1/2; triangles whose AABB misses the
// frustum's are skipped (froxel.py:363-364).  Block 0 publishes the frame.
__global__ void __launch_bounds__(kSetupThreads) ortho_setup_kernel(Params p, GtParams g, int supersample,
                                                                    const double* __restrict__ verts,
                                                                    long long nverts,
                                                                    const int64_t* __restrict__ tris, long long T,
                                                                    Work wk) {
  double lo[3], hi[3], spacing;
  int counts[3];
  ortho_frame(g, supersample, lo, hi, spacing, counts);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    wk.oframe[0] = lo[0];
    wk.oframe[1] = lo[1];
    wk.oframe[2] = lo[2];
    wk.oframe[3] = spacing;
  }
  const long long t = (long long)blockIdx.x * kSetupThreads + threadIdx.x;
  Slot s0, s1;
  unsigned long long c0 = 0, c1 = 0;
  if (t < wk.ntris) {
    const int pass = (int)(t / T);
    const long long tri = t - (long long)pass * T;
    const int a0 = pass == 0 ? 1 : pass == 1 ? 2 : 0, a1 = pass == 0 ? 2 : pass == 1 ? 0 : 1;
    const int ar = 3 - a0 - a1;
    long long id[3];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      id[k] = tris[tri * 3 + k];
      ok &= id[k] >= 0 && id[k] < nverts;
    }
    if (ok) {
      const double* v[3] = {verts + id[0] * 3, verts + id[1] * 3, verts + id[2] * 3};
      bool live = true;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double mn = fmin(fmin(v[0][k], v[1][k]), v[2][k]), mx = fmax(fmax(v[0][k], v[1][k]), v[2][k]);
        live &= mx >= lo[k] && mn <= hi[k];
      }
      if (live) {
        double u[3], w[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          u[k] = ddiv(dsub(v[k][a0], lo[a0]), spacing);
          w[k] = ddiv(dsub(v[k][a1], lo[a1]), spacing);
        }
        Slot& sl = s0;
        sl.v0x = u[0];
        sl.v0y = w[0];
        sl.e1x = dsub(u[1], u[0]);
        sl.e1y = dsub(w[1], w[0]);
        sl.e2x = dsub(u[2], u[0]);
        sl.e2y = dsub(w[2], w[0]);
        sl.den = dsub(dmul(sl.e1x, sl.e2y), dmul(sl.e2x, sl.e1y));
        sl.iz0 = v[0][ar];  // the interpolated world coordinate
        sl.iz1 = v[1][ar];
        sl.iz2 = v[2][ar];
        sl.wv0 = sl.wv1 = sl.wv2 = 0.0;
        sl.rden = 1.0 / sl.den;
        sl.wtol = 0.0;
        const double W = (double)counts[a0], H = (double)counts[a1];
        const double minx = fmin(fmin(u[0], u[1]), u[2]), maxx = fmax(fmax(u[0], u[1]), u[2]);
        const double miny = fmin(fmin(w[0], w[1]), w[2]), maxy = fmax(fmax(w[0], w[1]), w[2]);
        const int ix0 = (int)fmin(fmax(ceil(dsub(minx, 0.5)), 0.0), W);
        const int ix1 = (int)fmin(fmax(dadd(floor(dsub(maxx, 0.5)), 1.0), 0.0), W);
        const int iy0 = (int)fmin(fmax(ceil(dsub(miny, 0.5)), 0.0), H);
        const int iy1 = (int)fmin(fmax(dadd(floor(dsub(maxy, 0.5)), 1.0), 0.0), H);
        sl.x0 = ix0;
        sl.y0 = iy0;
        sl.w = max(ix1 - ix0, 0);
        sl.h = max(iy1 - iy0, 0);
        if (!(fabs(sl.den) > kDegenEps && sl.w > 0 && sl.h > 0)) sl.w = sl.h = 0;
        sl.wmagic = sl.w > 1 ? (unsigned int)((0x100000000ull + (unsigned long long)sl.w - 1) / (unsigned long long)sl.w)
                             : 0xffffffffu;
        c0 = (unsigned long long)sl.w * (unsigned long long)sl.h;
      }
    }
    s0.pad = s1.pad = pass;
  }
  finish_setup(p, wk, t, c0, c1, s0, s1);
}

// Reference depth of one sample (froxel.py:272-279 coverage; oracle.py:127
// depth = 1 / interp_affine(invz, b1, b2)); < 0 when not covered.
__device__ __forceinline__ double depth_exact(const Slot& s, double cx, double cy) {
  const double dx = dsub(cx, s.v0x), dy = dsub(cy, s.v0y);
  const double b1 = ddiv(dsub(dmul(dx, s.e2y), dmul(s.e2x, dy)), s.den);
  const double b2 = ddiv(dsub(dmul(s.e1x, dy), dmul(dx, s.e1y)), s.den);
  const double b0 = dsub(dsub(1.0, b1), b2);
  if (!(b0 >= 0 && b1 >= 0 && b2 >= 0)) return -1.0;
  return ddiv(1.0, dadd(dadd(s.iz0, dmul(b1, dsub(s.iz1, s.iz0))), dmul(b2, dsub(s.iz2, s.iz0))));
}

// Coverage filter before the exact evaluation: samples provably outside
// (exact numerator signs, or b0 < 0 by more than the approximation error)
// skip the three divisions.
__device__ __forceinline__ double depth_filtered(const Slot& s, double cx, double cy) {
  const double dx = dsub(cx, s.v0x), dy = dsub(cy, s.v0y);
  const double n1 = dsub(dmul(dx, s.e2y), dmul(s.e2x, dy));
  const double n2 = dsub(dmul(s.e1x, dy), dmul(dx, s.e1y));
  const bool dneg = s.den < 0;
  const double a1 = fabs(n1), a2 = fabs(n2);
  constexpr double kTiny = 1e-250;
  if (!((a1 != 0 && a1 < kTiny) || (a2 != 0 && a2 < kTiny))) {
    if ((n1 != 0 && ((n1 < 0) != dneg)) || (n2 != 0 && ((n2 < 0) != dneg))) return -1.0;
    const double q1 = n1 * s.rden, q2 = n2 * s.rden;
    if ((1.0 - q1) - q2 < -1e-13 * (1.0 + q1 + q2)) return -1.0;
  }
  return depth_exact(s, cx, cy);
}

// ---------------------------------------------------------------------------
// Span raster.  The flat work space counts bounding-box ROWS; a warp takes
// 32 rows at a time (lane = row), bounds each row's candidate columns with
// row_span, and expands the rows' spans into samples 32 at a time (lane =
// sample, its row found by a 5-step search over the warp's span prefix).
// Only samples inside the spans are evaluated (by the same exact / filtered
// per-sample code), so the outside half of every bounding box costs nothing.
// ---------------------------------------------------------------------------

// Conservative candidate columns [xa, xb) of bounding-box row py: each edge's
// sign condition is linear in the pixel centre cx (f = a cx + b >= 0, sign-
// normalised by den); columns are dropped only where an edge value is below
// -tol, with tol ~1e-9 of the magnitudes (its rounding error is ~1e-16 of
// them), and one pixel of margin is kept on either side.
__device__ __forceinline__ void row_span(const Slot& s, int py, int& xa, int& xb) {
  const double dy = centre(py) - s.v0y;
  const double sg = s.den < 0 ? -1.0 : 1.0;
  double lo = s.x0 + 0.5, hi = s.x0 + s.w - 0.5;
  const double M = fmax(fabs(lo), fabs(hi)) + 1.0;
  const double a1 = sg * s.e2y, b1 = -sg * (s.e2y * s.v0x + s.e2x * dy);
  const double a2 = -sg * s.e1y, b2 = sg * (s.e1x * dy + s.e1y * s.v0x);
  const double a0 = -(a1 + a2), b0 = fabs(s.den) - b1 - b2;
  const double t1 = 1e-9 * (fabs(a1) * M + fabs(b1)), t2 = 1e-9 * (fabs(a2) * M + fabs(b2));
  const double t0 = t1 + t2 + 1e-9 * fabs(s.den);
  const double a[3] = {a0, a1, a2}, b[3] = {b0, b1, b2}, tl[3] = {t0, t1, t2};
  bool empty = false;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (a[k] > 0) lo = fmax(lo, (-tl[k] - b[k]) / a[k]);
    else if (a[k] < 0) hi = fmin(hi, (-tl[k] - b[k]) / a[k]);
    else empty |= b[k] < -tl[k];
  }
  xa = s.x0;
  xb = s.x0 + s.w;
  if (empty || lo > hi + 2.0) {
    xb = xa;
    return;
  }
  if (isfinite(lo)) xa = max(xa, (int)fmax(ceil(lo - 1.5), (double)s.x0));
  if (isfinite(hi)) xb = min(xb, (int)fmin(floor(hi + 0.5) + 1.0, (double)(s.x0 + s.w)));
  if (xb < xa) xb = xa;
}

constexpr int kSpanRowsPerThread = 2;
constexpr int kSpanChunk = kRasterThreads * kSpanRowsPerThread;

// kKind 0: OR bits (froxelize), 1: cull marks, 2: (froxel, triangle) pairs,
// 3: z-buffer min (GT), 4: smallest primitive id among z-ties (GT).
template <bool kFilter, int kKind>
__global__ void __launch_bounds__(kRasterThreads, kKind >= 5 ? 4 : 3)
    span_kernel(Params p, GtParams g, const fpvs_frustum* __restrict__ views, const int64_t* __restrict__ prim_ids,
                Work wk, unsigned long long* __restrict__ zbuf, long long* __restrict__ pidbuf) {
  constexpr int kWarpRows = 32 * kSpanRowsPerThread;
  constexpr bool kDepth = kKind == 3 || kKind == 4;
  constexpr bool kOrtho = kKind >= 5;                // kinds 5/6/7: orthographic bits / cull / pairs
  constexpr int kAct = kOrtho ? kKind - 5 : kKind;  // 0 bits, 1 cull, 2 pairs, 3/4 depth
  __shared__ double s_lo[3], s_spacing;
  if (kOrtho) {
    if (threadIdx.x < 3) s_lo[threadIdx.x] = wk.oframe[threadIdx.x];
    if (threadIdx.x == 3) s_spacing = wk.oframe[3];
    __syncthreads();
  }
  const unsigned long long total = *wk.total;  // rows
  const unsigned int row = (unsigned int)(p.nx >> 3);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long have = -1;  // slot whose constants are in s
  Slot s;
  double farz = 0;
  long long zoff = 0;
  for (unsigned long long c0 = (unsigned long long)blockIdx.x * kSpanChunk; c0 < total;
       c0 += (unsigned long long)gridDim.x * kSpanChunk) {
    const unsigned long long wbase = c0 + (unsigned long long)warp * kWarpRows;
    if (wbase >= total) break;  // warp-uniform
    unsigned long long cs = 0;
    long long cur = 0;
    if (lane == 0) cur = find_slot(wk, wbase, cs);
    cur = __shfl_sync(0xffffffffu, cur, 0);
    cs = __shfl_sync(0xffffffffu, cs, 0);
    unsigned long long ce = slot_end(wk, cur);
#pragma unroll 1
    for (int k = 0; k < kSpanRowsPerThread; ++k) {
      // ---- lane = row: its slot, pixel row and candidate span
      const unsigned long long r = wbase + (unsigned long long)(k * 32 + lane);
      long long mine = cur;
      int py = 0, xa = 0, len = 0;
      if (r < total) {
        unsigned long long ms = cs, me = ce;
        int steps = 0;
        while (r >= me && steps < 4) {
          ms = me;
          me = slot_end(wk, ++mine);
          ++steps;
        }
        if (r >= me) {
          mine = find_slot(wk, r, ms);
          me = slot_end(wk, mine);
        }
        if (mine != have) {
          s = wk.slots[mine];
          have = mine;
          if (kDepth) {
            farz = views[s.pad].far_z;
            zoff = (long long)s.pad * g.npix;
          }
        }
        // item -> (bounding-box row, p.seg-column segment)
        const unsigned int it = (unsigned int)(r - ms);
        const unsigned int ns = (unsigned int)(s.w + p.seg - 1) / (unsigned int)p.seg;
        unsigned int ry = __umulhi(it, s.wmagic);
        const int rem = (int)(it - ry * ns);
        if (rem < 0) --ry;
        else if (rem >= (int)ns) ++ry;
        const int seg = (int)(it - ry * ns);
        py = s.y0 + (int)ry;
        int xb;
        row_span(s, py, xa, xb);
        xa = max(xa, s.x0 + seg * p.seg);
        xb = min(xb, s.x0 + seg * p.seg + p.seg);
        len = max(xb - xa, 0);
      }
      const long long nxt = __shfl_sync(0xffffffffu, mine, 31);
      // ---- warp prefix of span lengths
      int incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      // ---- lane = sample
      for (int t0 = 0; t0 < tot; t0 += 32) {
        const int t = t0 + lane;
        int kr = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const int v = __shfl_sync(0xffffffffu, incl, kr + step - 1);
          if (v <= t) kr += step;
        }
        const long long sl = __shfl_sync(0xffffffffu, mine, kr);
        const int spy = __shfl_sync(0xffffffffu, py, kr);
        const int sxa = __shfl_sync(0xffffffffu, xa, kr);
        const int sex = __shfl_sync(0xffffffffu, incl, kr) - __shfl_sync(0xffffffffu, len, kr);
        bool valid = t < tot;
        unsigned int word = 0, bit = 0;
        long long flat = 0;
        if (valid) {
          if (sl != have) {
            s = wk.slots[sl];
            have = sl;
            if (kDepth) {
              farz = views[s.pad].far_z;
              zoff = (long long)s.pad * g.npix;
            }
          }
          const int px = sxa + (t - sex);
          const double cx = centre(px), cy = centre(spy);
          if (kOrtho) {
            // orthographic pass s.pad: axes (a0, a1) on screen, ar interpolated
            // (froxel.py:366-374)
            double b1, b2;
            valid = false;
            if (bary_filtered(s, cx, cy, b1, b2)) {
              const int pass = s.pad;
              const int a0 = pass == 0 ? 1 : pass == 1 ? 2 : 0, a1 = pass == 0 ? 2 : pass == 1 ? 0 : 1;
              double wv[3];
              wv[a0] = dadd(s_lo[a0], dmul(cx, s_spacing));
              wv[a1] = dadd(s_lo[a1], dmul(cy, s_spacing));
              wv[3 - a0 - a1] = dadd(dadd(s.iz0, dmul(b1, dsub(s.iz1, s.iz0))), dmul(b2, dsub(s.iz2, s.iz0)));
              int ix, iy, iz;
              if (project_quantize(g, wv[0], wv[1], wv[2], ix, iy, iz)) {
                const unsigned long long byte = (unsigned long long)(ix >> 3) +
                                                (unsigned long long)row * ((unsigned long long)iy + (unsigned long long)p.ny * iz);
                word = (unsigned int)(byte >> 2);
                bit = 1u << ((((unsigned int)byte & 3u) << 3) | ((unsigned int)ix & 7u));
                if (kAct == 2) flat = ix + (long long)p.nx * (iy + (long long)p.ny * iz);
                valid = true;
              }
            }
          } else if (kDepth) {
            const double depth = depth_filtered(s, cx, cy);
            valid = false;
            if (depth >= 0 && depth <= farz) {  // oracle.py:128
              const long long pix = zoff + (long long)spy * g.iw + px;
              const unsigned long long bits = (unsigned long long)__double_as_longlong(depth);
              if (kKind == 3) {
                atomicMin(zbuf + pix, bits);
              } else if (bits == zbuf[pix]) {
                const long long tri = (sl >> 1) - (long long)s.pad * g.T;
                atomicMin(pidbuf + pix, prim_ids ? prim_ids[tri] : tri);
              }
            }
          } else {
            const int iz = kFilter ? sample_fast(s, cx, cy, p.nz) : sample_exact(s, cx, cy, p.nz);
            valid = iz >= 0;
            if (valid) {
              const int ix = __ldg(wk.tabx + px), iy = __ldg(wk.taby + spy);
              const unsigned long long byte = (unsigned long long)(ix >> 3) +
                                              (unsigned long long)row * ((unsigned long long)iy + (unsigned long long)p.ny * iz);
              word = (unsigned int)(byte >> 2);
              bit = 1u << ((((unsigned int)byte & 3u) << 3) | ((unsigned int)ix & 7u));
              if (kKind == 2) flat = ix + (long long)p.nx * (iy + (long long)p.ny * iz);  // froxel.py:411
            }
          }
        }
        // scene triangle of the sample (ortho slots are numbered pass * T + tri)
        const long long tri = kOrtho ? (sl >> 1) - (long long)s.pad * g.T : (sl >> 1);
        if (kAct == 0) {
          const unsigned int vm = __ballot_sync(0xffffffffu, valid);
          if (vm) {
            const int leader = __ffs(vm) - 1;
            const unsigned int w0 = __shfl_sync(0xffffffffu, word, leader);
            if (__all_sync(0xffffffffu, !valid || word == w0)) {
              const unsigned int bits = __reduce_or_sync(0xffffffffu, valid ? bit : 0u);
              if (lane == leader) atomicOr(wk.out_words + w0, bits);
            } else if (valid) {
              atomicOr(wk.out_words + word, bit);
            }
          }
        } else if (kAct == 1) {
          if (valid && (__ldg(wk.pvs_words + word) & bit)) wk.kept[tri] = 1;
        } else if (kAct == 2) {
          const long long key = valid ? flat * (kOrtho ? g.T : wk.ntris) + tri : -1 - lane;
          const unsigned int peers = __match_any_sync(0xffffffffu, key);
          if (valid && (__ffs(peers) - 1) == lane) {
            const unsigned long long slot = atomicAdd(wk.npairs, 1ull);
            if ((long long)slot < wk.pair_cap) wk.pairs[slot] = key;
          }
        }
      }
      // the warp's next rows start from the last lane's slot
      if (nxt != cur) {
        cur = nxt;
        cs = (cur % kSlotsPerBlock ? slot_end(wk, cur - 1) : __ldg(wk.bpre + cur / kSlotsPerBlock));
        ce = slot_end(wk, cur);
      }
    }
  }
}

struct Layout {
  size_t slots, lp, bsum, bpre, total, tabx, taby, words, bytes;
};

inline size_t up256(size_t v) { return (v + 255) & ~(size_t)255; }

inline Layout layout(long long ntris, long long grid_bytes, long long sx, long long sy) {
  Layout L;
  const long long nslot = 2 * (ntris > 0 ? ntris : 1);
  const long long nb = (nslot + kSlotsPerBlock - 1) / kSlotsPerBlock;
  size_t o = 0;
  L.total = o; o = up256(o + 8);  // first, so fpvs_froxelize_samples finds it without the sizes
  L.slots = o; o = up256(o + (size_t)nslot * sizeof(Slot));
  L.lp = o;    o = up256(o + (size_t)nslot * 8);
  L.bsum = o;  o = up256(o + (size_t)nb * 8);
  L.bpre = o;  o = up256(o + (size_t)nb * 8);
  L.tabx = o;  o = up256(o + (size_t)sx * 4);
  L.taby = o;  o = up256(o + (size_t)sy * 4);
  L.words = o; o = up256(o + (size_t)((grid_bytes + 3) & ~3LL));  // used only for unaligned outputs
  L.bytes = o;
  return L;
}

// raster segment widths: FPVS_FROX_SEG / FPVS_GT_SEG (tuning knobs, read once per process)
inline int env_seg(const char* name, int dflt) {
  const char* e = getenv(name);
  const int v = e ? atoi(e) : dflt;
  return v >= 8 && v <= 1024 ? v : dflt;
}
inline int frox_seg() {
  static const int v = env_seg("FPVS_FROX_SEG", 16);
  return v;
}
inline int gt_seg() {
  static const int v = env_seg("FPVS_GT_SEG", 64);
  return v;
}

// FPVS_FROX_SPANS=0 rasterizes whole bounding boxes instead of row spans (A/B check)
inline bool spans() {
  static const bool f = [] {
    const char* e = getenv("FPVS_FROX_SPANS");
    return !(e && e[0] == '0');
  }();
  return f;
}

// FPVS_FROX_EXACT=1 evaluates every sample with the reference sequence (A/B check)
inline bool filtered() {
  static const bool f = [] {
    const char* e = getenv("FPVS_FROX_EXACT");
    return !(e && e[0] == '1');
  }();
  return f;
}

}  // namespace frox
}  // namespace fpvs

using namespace fpvs;
using namespace fpvs::frox;

extern "C" size_t fpvs_froxelize_workspace_size(long long ntris, int Nx, int Ny, int Nz, int supersample) {
  if (ntris < 0 || Nx <= 0 || Ny <= 0 || Nz <= 0 || supersample < 1) return 0;
  return layout(ntris, (long long)Nx * Ny * Nz / 8, (long long)supersample * Nx, (long long)supersample * Ny).bytes;
}

namespace fpvs {
namespace frox {

template <typename K>
int occupancy_grid(K kernel) {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, kRasterThreads, 0);
  return kNumSMs * (n > 0 ? n : 1);
}

template <int kMode>
int launch_raster(const Params& p, const Work& wk, cudaStream_t s) {
  const GtParams g = {};
  if (spans()) {
    static const int grid[2] = {occupancy_grid(span_kernel<false, kMode>), occupancy_grid(span_kernel<true, kMode>)};
    if (filtered())
      span_kernel<true, kMode><<<grid[1], kRasterThreads, 0, s>>>(p, g, nullptr, nullptr, wk, nullptr, nullptr);
    else
      span_kernel<false, kMode><<<grid[0], kRasterThreads, 0, s>>>(p, g, nullptr, nullptr, wk, nullptr, nullptr);
  } else {
    static const int grid[2] = {occupancy_grid(raster_kernel<false, kMode>), occupancy_grid(raster_kernel<true, kMode>)};
    if (filtered())
      raster_kernel<true, kMode><<<grid[1], kRasterThreads, 0, s>>>(p, wk);
    else
      raster_kernel<false, kMode><<<grid[0], kRasterThreads, 0, s>>>(p, wk);
  }
  FPVS_CHECK_LAUNCH("froxelize raster");
  return FPVS_OK;
}

// Argument checks, workspace carve-up, setup + scan, then the raster of the
// requested mode.  out_words: the (aligned) grid for mode 0.
template <int kMode>
int froxel_pass(const double* verts, long long nverts, const int64_t* tris, long long ntris, const fpvs_frustum* fr,
                int Nx, int Ny, int Nz, int supersample, int depth_mode, void* workspace, size_t workspace_bytes,
                cudaStream_t s, Work& wk, Layout& L) {
  FPVS_CHECK_ARG(fr != nullptr, "froxelize: null frustum");
  FPVS_CHECK_ARG(Nx > 0 && Ny > 0 && Nz > 0 && Nx % 8 == 0, "N_x must be divisible by 8, got %d", Nx);
  FPVS_CHECK_ARG(supersample >= 1, "supersample factor must be >= 1");
  FPVS_CHECK_ARG(depth_mode == FPVS_DEPTH_LINEAR || depth_mode == FPVS_DEPTH_LOG, "bad depth mode %d", depth_mode);
  FPVS_CHECK_ARG(ntris >= 0 && nverts >= 0 && (ntris == 0 || (verts && tris)), "froxelize: bad scene arrays");
  FPVS_CHECK_ARG(fr->near_z > 0 && fr->near_z < fr->far_z && fr->half_extent > 0, "need 0 < near < far");
  const long long sx = (long long)supersample * Nx, sy = (long long)supersample * Ny;
  FPVS_CHECK_ARG(sx * sy < (1LL << 32) && sx < (1LL << 30) && sy < (1LL << 30),
                 "froxelize: supersampled screen %lld x %lld too large", sx, sy);
  const long long grid_bytes = (long long)Nx * Ny * Nz / 8;
  L = layout(ntris, grid_bytes, sx, sy);
  FPVS_CHECK_ARG(workspace != nullptr && workspace_bytes >= L.bytes, "froxelize: workspace too small (%zu < %zu)",
                 workspace_bytes, L.bytes);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  wk.slots = reinterpret_cast<Slot*>(ws + L.slots);
  wk.lp = reinterpret_cast<unsigned long long*>(ws + L.lp);
  wk.bsum = reinterpret_cast<unsigned long long*>(ws + L.bsum);
  wk.bpre = reinterpret_cast<unsigned long long*>(ws + L.bpre);
  wk.total = reinterpret_cast<unsigned long long*>(ws + L.total);
  wk.nsamples = wk.total + 1;
  wk.tabx = reinterpret_cast<int*>(ws + L.tabx);
  wk.taby = reinterpret_cast<int*>(ws + L.taby);
  wk.ntris = ntris;
  wk.nb = (int)((2 * (ntris > 0 ? ntris : 1) + kSlotsPerBlock - 1) / kSlotsPerBlock);
  Params p;
  for (int i = 0; i < 3; ++i) p.o[i] = fr->origin[i];
  for (int i = 0; i < 9; ++i) p.b[i] = fr->basis[i];
  p.h = fr->half_extent;
  p.nearz = fr->near_z;
  p.farz = fr->far_z;
  p.isx = (int)sx;
  p.isy = (int)sy;
  p.sx = (double)sx;
  p.sy = (double)sy;
  p.nx = Nx;
  p.ny = Ny;
  p.nz = Nz;
  p.depth_log = depth_mode == FPVS_DEPTH_LOG;
  p.rows_mode = spans() ? 1 : 0;
  p.seg = frox_seg();
  if (cudaMemsetAsync(wk.total, 0, 16, s) != cudaSuccess) FPVS_CHECK_LAUNCH("memset");  // total + nsamples
  if (ntris == 0) return FPVS_OK;
  setup_kernel<false><<<wk.nb, kSetupThreads, 0, s>>>(p, nullptr, verts, nverts, tris, ntris, wk);
  FPVS_CHECK_LAUNCH("froxelize setup");
  scan_kernel<<<1, 1024, 0, s>>>(p, wk);
  FPVS_CHECK_LAUNCH("froxelize scan");
  return launch_raster<kMode>(p, wk, s);
}

}  // namespace frox
}  // namespace fpvs

extern "C" int fpvs_froxelize(const double* verts, long long nverts, const int64_t* tris, long long ntris,
                              const fpvs_frustum* fr, int Nx, int Ny, int Nz, int supersample, int depth_mode,
                              uint8_t* out_bits, void* workspace, size_t workspace_bytes, void* stream) {
  FPVS_CHECK_ARG(out_bits != nullptr, "froxelize: null output");
  FPVS_CHECK_ARG(Nx > 0 && Ny > 0 && Nz > 0, "froxelize: bad dims");
  cudaStream_t s = as_stream(stream);
  const long long grid_bytes = (long long)Nx * Ny * Nz / 8;
  const bool direct = ((uintptr_t)out_bits & 3) == 0 && grid_bytes % 4 == 0;
  Work wk = {};
  Layout L = {};
  // the scratch grid offset is needed before the pass: compute the layout first
  {
    const long long sx = (long long)supersample * Nx, sy = (long long)supersample * Ny;
    L = layout(ntris, grid_bytes, sx, sy);
  }
  unsigned int* words = direct ? reinterpret_cast<unsigned int*>(out_bits)
                               : reinterpret_cast<unsigned int*>(static_cast<uint8_t*>(workspace) + L.words);
  if (workspace == nullptr || workspace_bytes < L.bytes)
    return set_error(FPVS_EINVAL, "froxelize: workspace too small (%zu < %zu)", workspace_bytes, L.bytes);
  if (cudaMemsetAsync(words, 0, (size_t)((grid_bytes + 3) & ~3LL), s) != cudaSuccess) FPVS_CHECK_LAUNCH("memset");
  wk.out_words = words;
  const int rc = froxel_pass<0>(verts, nverts, tris, ntris, fr, Nx, Ny, Nz, supersample, depth_mode, workspace,
                                workspace_bytes, s, wk, L);
  if (rc) return rc;
  if (!direct && cudaMemcpyAsync(out_bits, words, (size_t)grid_bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    FPVS_CHECK_LAUNCH("froxelize copy");
  return FPVS_OK;
}

extern "C" int fpvs_froxel_cull(const double* verts, long long nverts, const int64_t* tris, long long ntris,
                                const fpvs_frustum* fr, int Nx, int Ny, int Nz, int supersample, int depth_mode,
                                const uint8_t* pvs_bits, uint8_t* kept, void* workspace, size_t workspace_bytes,
                                void* stream) {
  const long long grid_bytes = (long long)Nx * Ny * Nz / 8;
  FPVS_CHECK_ARG(pvs_bits != nullptr && (ntris == 0 || kept != nullptr), "froxel_cull: null pvs or output");
  FPVS_CHECK_ARG(((uintptr_t)pvs_bits & 3) == 0 && grid_bytes % 4 == 0,
                 "froxel_cull: pvs grid must be 4-byte aligned with Nx*Ny*Nz/8 a multiple of 4");
  cudaStream_t s = as_stream(stream);
  if (ntris > 0 && cudaMemsetAsync(kept, 0, (size_t)ntris, s) != cudaSuccess) FPVS_CHECK_LAUNCH("memset");
  Work wk = {};
  Layout L = {};
  wk.pvs_words = reinterpret_cast<const unsigned int*>(pvs_bits);
  wk.kept = kept;
  return froxel_pass<1>(verts, nverts, tris, ntris, fr, Nx, Ny, Nz, supersample, depth_mode, workspace,
                        workspace_bytes, s, wk, L);
}

extern "C" int fpvs_froxel_pairs(const double* verts, long long nverts, const int64_t* tris, long long ntris,
                                 const fpvs_frustum* fr, int Nx, int Ny, int Nz, int supersample, int depth_mode,
                                 long long* pairs, long long cap, unsigned long long* npairs_dev, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  FPVS_CHECK_ARG(npairs_dev != nullptr && cap >= 0 && (cap == 0 || pairs != nullptr), "froxel_pairs: bad output");
  cudaStream_t s = as_stream(stream);
  if (cudaMemsetAsync(npairs_dev, 0, 8, s) != cudaSuccess) FPVS_CHECK_LAUNCH("memset");
  Work wk = {};
  Layout L = {};
  wk.pairs = pairs;
  wk.npairs = npairs_dev;
  wk.pair_cap = cap;
  return froxel_pass<2>(verts, nverts, tris, ntris, fr, Nx, Ny, Nz, supersample, depth_mode, workspace,
                        workspace_bytes, s, wk, L);
}

extern "C" long long fpvs_froxelize_samples(const void* workspace, void* stream) {
  if (workspace == nullptr) return -1;
  unsigned long long v = 0;
  cudaStream_t s = as_stream(stream);
  if (cudaMemcpyAsync(&v, static_cast<const uint8_t*>(workspace) + 8, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return -1;
  if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
  return (long long)v;
}

// Orthographic three-view froxelization (froxel.py:351-376, the dataset
// generator's default mode): one setup over (pass, triangle), the shared
// scan, then span_kernel<5> rasterizes each pass's triangles on the world
// AABB's sample lattice, reconstructs the world point of every covered sample
// and ORs its froxel (project_points + quantize) into the grid.  The 32-byte
// AABB frame (lo, spacing) lives where the perspective path keeps its
// pixel->froxel table.
extern "C" size_t fpvs_froxelize_ortho_workspace_size(long long ntris, int Nx, int Ny, int Nz, int supersample) {
  if (ntris < 0 || Nx <= 0 || Ny <= 0 || Nz <= 0 || supersample < 1) return 0;
  return frox::layout(3 * ntris, (long long)Nx * Ny * Nz / 8, 8, 0).bytes;
}

namespace fpvs {
namespace frox {

// kKind 5: grid bits into out_bits; 6: cull flags (wk.pvs_words / wk.kept);
// 7: fragment pairs (wk.pairs / npairs / pair_cap).  out_bits only for 5.
template <int kKind>
int ortho_pass(const double* verts, long long nverts, const int64_t* tris, long long ntris, const fpvs_frustum* fr,
               int Nx, int Ny, int Nz, int supersample, int depth_mode, uint8_t* out_bits, void* workspace,
               size_t workspace_bytes, cudaStream_t s, Work wk) {
  FPVS_CHECK_ARG(fr != nullptr && (kKind != 5 || out_bits != nullptr), "froxelize_ortho: null output or frustum");
  FPVS_CHECK_ARG(Nx > 0 && Ny > 0 && Nz > 0 && Nx % 8 == 0, "N_x must be divisible by 8, got %d", Nx);
  FPVS_CHECK_ARG(supersample >= 1, "supersample factor must be >= 1");
  FPVS_CHECK_ARG(depth_mode == FPVS_DEPTH_LINEAR || depth_mode == FPVS_DEPTH_LOG, "bad depth mode %d", depth_mode);
  FPVS_CHECK_ARG(ntris >= 0 && nverts >= 0 && (ntris == 0 || (verts && tris)), "froxelize_ortho: bad scene arrays");
  FPVS_CHECK_ARG(fr->near_z > 0 && fr->near_z < fr->far_z && fr->half_extent > 0, "need 0 < near < far");
  const long long dmax = Nx > Ny ? (Nx > Nz ? Nx : Nz) : (Ny > Nz ? Ny : Nz);
  FPVS_CHECK_ARG((long long)supersample * dmax < (1LL << 20), "froxelize_ortho: sample lattice too large");
  const long long grid_bytes = (long long)Nx * Ny * Nz / 8;
  const Layout L = layout(3 * ntris, grid_bytes, 8, 0);
  FPVS_CHECK_ARG(workspace != nullptr && workspace_bytes >= L.bytes, "froxelize_ortho: workspace too small (%zu < %zu)",
                 workspace_bytes, L.bytes);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const bool direct = kKind != 5 || (((uintptr_t)out_bits & 3) == 0 && grid_bytes % 4 == 0);
  unsigned int* words = kKind != 5 ? nullptr
                        : direct   ? reinterpret_cast<unsigned int*>(out_bits)
                                   : reinterpret_cast<unsigned int*>(ws + L.words);
  if (kKind == 5 && cudaMemsetAsync(words, 0, (size_t)((grid_bytes + 3) & ~3LL), s) != cudaSuccess)
    FPVS_CHECK_LAUNCH("memset");
  if (cudaMemsetAsync(ws + L.total, 0, 16, s) != cudaSuccess) FPVS_CHECK_LAUNCH("memset");
  if (ntris > 0) {
    wk.slots = reinterpret_cast<Slot*>(ws + L.slots);
    wk.lp = reinterpret_cast<unsigned long long*>(ws + L.lp);
    wk.bsum = reinterpret_cast<unsigned long long*>(ws + L.bsum);
    wk.bpre = reinterpret_cast<unsigned long long*>(ws + L.bpre);
    wk.total = reinterpret_cast<unsigned long long*>(ws + L.total);
    wk.nsamples = wk.total + 1;
    wk.oframe = reinterpret_cast<double*>(ws + L.tabx);
    wk.out_words = words;
    wk.ntris = 3 * ntris;
    wk.nb = (int)((2 * wk.ntris + kSlotsPerBlock - 1) / kSlotsPerBlock);
    Params p = {};
    p.nx = Nx;
    p.ny = Ny;
    p.nz = Nz;
    p.depth_log = depth_mode == FPVS_DEPTH_LOG;
    p.rows_mode = 1;
    p.seg = frox_seg();
    GtParams g = {};
    for (int i = 0; i < 3; ++i) g.fo[i] = fr->origin[i];
    for (int i = 0; i < 9; ++i) g.fb[i] = fr->basis[i];
    g.fh = fr->half_extent;
    g.fnear = fr->near_z;
    g.ffar = fr->far_z;
    g.flogr = log(fr->far_z / fr->near_z);
    g.nx = Nx;
    g.ny = Ny;
    g.nz = Nz;
    g.depth_log = p.depth_log;
    g.T = ntris;
    ortho_setup_kernel<<<wk.nb, kSetupThreads, 0, s>>>(p, g, supersample, verts, nverts, tris, ntris, wk);
    FPVS_CHECK_LAUNCH("froxelize_ortho setup");
    scan_kernel<<<1, 1024, 0, s>>>(p, wk);
    FPVS_CHECK_LAUNCH("froxelize_ortho scan");
    static const int grid = occupancy_grid(span_kernel<true, kKind>);
    span_kernel<true, kKind><<<grid, kRasterThreads, 0, s>>>(p, g, nullptr, nullptr, wk, nullptr, nullptr);
    FPVS_CHECK_LAUNCH("froxelize_ortho raster");
  }
  if (!direct && cudaMemcpyAsync(out_bits, words, (size_t)grid_bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    FPVS_CHECK_LAUNCH("froxelize_ortho copy");
  return FPVS_OK;
}

}  // namespace frox
}  // namespace fpvs

extern "C" int fpvs_froxelize_ortho(const double* verts, long long nverts, const int64_t* tris, long long ntris,
                                    const fpvs_frustum* fr, int Nx, int Ny, int Nz, int supersample, int depth_mode,
                                    uint8_t* out_bits, void* workspace, size_t workspace_bytes, void* stream) {
  return frox::ortho_pass<5>(verts, nverts, tris, ntris, fr, Nx, Ny, Nz, supersample, depth_mode, out_bits, workspace,
                             workspace_bytes, as_stream(stream), frox::Work{});
}

extern "C" int fpvs_froxel_cull_ortho(const double* verts, long long nverts, const int64_t* tris, long long ntris,
                                      const fpvs_frustum* fr, int Nx, int Ny, int Nz, int supersample, int depth_mode,
                                      const uint8_t* pvs_bits, uint8_t* kept, void* workspace, size_t workspace_bytes,
                                      void* stream) {
  const long long grid_bytes = (long long)Nx * Ny * Nz / 8;
  FPVS_CHECK_ARG(pvs_bits != nullptr && (ntris == 0 || kept != nullptr), "froxel_cull_ortho: null pvs or output");
  FPVS_CHECK_ARG(((uintptr_t)pvs_bits & 3) == 0 && grid_bytes % 4 == 0,
                 "froxel_cull_ortho: pvs grid must be 4-byte aligned with Nx*Ny*Nz/8 a multiple of 4");
  cudaStream_t s = as_stream(stream);
  if (ntris > 0 && cudaMemsetAsync(kept, 0, (size_t)ntris, s) != cudaSuccess) FPVS_CHECK_LAUNCH("memset");
  frox::Work wk = {};
  wk.pvs_words = reinterpret_cast<const unsigned int*>(pvs_bits);
  wk.kept = kept;
  return frox::ortho_pass<6>(verts, nverts, tris, ntris, fr, Nx, Ny, Nz, supersample, depth_mode, nullptr, workspace,
                             workspace_bytes, s, wk);
}

extern "C" int fpvs_froxel_pairs_ortho(const double* verts, long long nverts, const int64_t* tris, long long ntris,
                                       const fpvs_frustum* fr, int Nx, int Ny, int Nz, int supersample, int depth_mode,
                                       long long* pairs, long long cap, unsigned long long* npairs_dev, void* workspace,
                                       size_t workspace_bytes, void* stream) {
  FPVS_CHECK_ARG(npairs_dev != nullptr && cap >= 0 && (cap == 0 || pairs != nullptr), "froxel_pairs_ortho: bad output");
  cudaStream_t s = as_stream(stream);
  if (cudaMemsetAsync(npairs_dev, 0, 8, s) != cudaSuccess) FPVS_CHECK_LAUNCH("memset");
  frox::Work wk = {};
  wk.pairs = pairs;
  wk.npairs = npairs_dev;
  wk.pair_cap = cap;
  return frox::ortho_pass<7>(verts, nverts, tris, ntris, fr, Nx, Ny, Nz, supersample, depth_mode, nullptr, workspace,
                             workspace_bytes, s, wk);
}

// ===========================================================================
// GT PVS: oracle.py:107-172 on the device.
//
// All cameras at once: setup<true> builds slots for every (camera, scene
// triangle) against that camera's frustum at the depth-buffer resolution;
// depth_kernel<0> rasterizes every candidate sample, computes the reference's
// depth 1 / interp(1/z) exactly and keeps the minimum per pixel with a 64-bit
// atomicMin on the (positive) double's bits; with primitive ids,
// depth_kernel<1> re-rasterizes and keeps the smallest id among the samples
// whose depth equals the pixel's minimum (oracle.py:130-136); resolve_kernel
// unprojects every covered pixel from its camera (core.py:431-446), projects
// it into the viewcell frustum (core.py:380-405), quantizes and ORs its bit
// into the GT grid and optionally the geometry grid.
// ===========================================================================
namespace fpvs {
namespace frox {

template <int kPass>
__global__ void __launch_bounds__(kRasterThreads, 4)
    depth_kernel(GtParams g, const fpvs_frustum* __restrict__ views, const int64_t* __restrict__ prim_ids, Work wk,
                 unsigned long long* __restrict__ zbuf, long long* __restrict__ pidbuf) {
  constexpr int kWarpSpan = 32 * kPerThread;
  const unsigned long long total = *wk.total;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long have = -1;
  Slot s;
  double farz = 0;
  long long zoff = 0, pid = 0;
  for (unsigned long long c0 = (unsigned long long)blockIdx.x * kChunk; c0 < total;
       c0 += (unsigned long long)gridDim.x * kChunk) {
    const unsigned long long wbase = c0 + (unsigned long long)warp * kWarpSpan;
    if (wbase >= total) break;
    unsigned long long cs = 0;
    long long cur = 0;
    if (lane == 0) cur = find_slot(wk, wbase, cs);
    cur = __shfl_sync(0xffffffffu, cur, 0);
    cs = __shfl_sync(0xffffffffu, cs, 0);
    unsigned long long ce = slot_end(wk, cur);
#pragma unroll 1
    for (int k = 0; k < kPerThread; ++k) {
      const unsigned long long gi = wbase + (unsigned long long)(k * 32 + lane);
      long long mine = cur;
      if (gi < total) {
        unsigned long long ms = cs, me = ce;
        int steps = 0;
        while (gi >= me && steps < 4) {
          ms = me;
          me = slot_end(wk, ++mine);
          ++steps;
        }
        if (gi >= me) {
          mine = find_slot(wk, gi, ms);
          me = slot_end(wk, mine);
        }
        if (mine != have) {
          s = wk.slots[mine];
          have = mine;
          farz = views[s.pad].far_z;
          zoff = (long long)s.pad * g.npix;
          if (kPass == 1) {
            const long long tri = (mine >> 1) - (long long)s.pad * g.T;
            pid = prim_ids ? prim_ids[tri] : tri;
          }
        }
        const unsigned int r = (unsigned int)(gi - ms);
        unsigned int ry = __umulhi(r, s.wmagic);
        const int rem = (int)(r - ry * (unsigned int)s.w);
        if (rem < 0) --ry;
        else if (rem >= s.w) ++ry;
        const int px = s.x0 + (int)(r - ry * (unsigned int)s.w);
        const int py = s.y0 + (int)ry;
        const double depth = depth_filtered(s, centre(px), centre(py));
        if (depth >= 0 && depth <= farz) {  // oracle.py:128
          const long long pix = zoff + (long long)py * g.iw + px;
          const unsigned long long bits = (unsigned long long)__double_as_longlong(depth);
          if (kPass == 0) {
            atomicMin(zbuf + pix, bits);
          } else if (bits == zbuf[pix]) {
            atomicMin(pidbuf + pix, pid);
          }
        }
      }
      const long long nxt = __shfl_sync(0xffffffffu, mine, 31);
      if (nxt != cur) {
        cur = nxt;
        cs = (cur % kSlotsPerBlock ? slot_end(wk, cur - 1) : __ldg(wk.bpre + cur / kSlotsPerBlock));
        ce = slot_end(wk, cur);
      }
    }
  }
}

// quantize (froxel.py:28-42) of an in-range test on an approximate NDC value
// a whose error is far below m: -1 = certainly outside [0, 1], index = certain
// froxel, -2 = within m of a decision boundary (0, 1, k/n): evaluate exactly.
__device__ __forceinline__ int quant_fast(double a, int n, double m) {
  if (!(a >= -m && a <= 1.0 + m)) return -1;
  if (a <= m || a >= 1.0 - m) return -2;
  const double t = a * (double)n, f = floor(t);
  const double mt = m * (double)n;
  if (t - f <= mt || f + 1.0 - t <= mt) return -2;
  return min(max((int)f, 0), n - 1);
}

__device__ __forceinline__ int quant_exact(double a, int n) {
  if (!(a >= 0 && a <= 1)) return -1;
  return min(max((int)floor(dmul(a, (double)n)), 0), n - 1);
}

// Covered pixel -> world -> viewcell frustum -> froxel bit (core.py:380-452).
// The world point is the reference's exact float64 sequence; the three NDC
// divisions go through one approximate reciprocal and are redone exactly
// only for points within 1e-12 of an inside/outside or froxel boundary.
__global__ void __launch_bounds__(256) resolve_kernel(GtParams g, const fpvs_frustum* __restrict__ views,
                                                      int nviews, const unsigned long long* __restrict__ zbuf,
                                                      const long long* __restrict__ pidbuf,
                                                      const double* __restrict__ ufx, const double* __restrict__ ufy,
                                                      unsigned int* __restrict__ gt_words,
                                                      unsigned int* __restrict__ geo_words) {
  const unsigned int npix = (unsigned int)g.npix, iw = (unsigned int)g.iw;
  const unsigned int wmag = iw > 1 ? (unsigned int)((0x100000000ull + iw - 1) / iw) : 0xffffffffu;
  const unsigned int row = (unsigned int)(g.nx >> 3);
  const int lane = threadIdx.x & 31;
  const double rfn = 1.0 / dsub(g.ffar, g.fnear);
  constexpr double kM = 1e-12;
  // (view, pixel) walk in 32-bit pixel arithmetic; the warp-uniform bound keeps
  // every lane in the ballot below
  const unsigned int per_view_steps = (npix + blockDim.x - 1) / blockDim.x;
  const unsigned int nsteps = (unsigned int)nviews * per_view_steps;  // < 2^32 (checked by the entry)
  for (unsigned int stp = blockIdx.x; stp < nsteps; stp += gridDim.x) {
    const int v = (int)(stp / per_view_steps);
    const unsigned int p = (stp - (unsigned int)v * per_view_steps) * blockDim.x + threadIdx.x;
    const long long i = (long long)v * g.npix + p;
    bool valid = false;
    unsigned int word = 0, bit = 0;
    if (p < npix) {
      const unsigned long long zb = zbuf[i];
      valid = zb != ~0ull && (pidbuf == nullptr || pidbuf[i] >= 0);
      if (valid) {
        unsigned int py = __umulhi(p, wmag);
        const int rem = (int)(p - py * iw);
        if (rem < 0) --py;
        else if (rem >= (int)iw) ++py;
        const int px = (int)(p - py * iw);
        const fpvs_frustum& c = views[v];
        const double z = __longlong_as_double((long long)zb);
        // x = (2 (px + 0.5) / W - 1) h z   (core.py:441-442)
        const double x = dmul(dmul(__ldg(ufx + px), c.half_extent), z);
        const double y = dmul(dmul(__ldg(ufy + py), c.half_extent), z);
        // world = position + [x y z] @ basis (dgemm k = 3 order), core.py:443-446
        double wv[3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
          wv[k] = dadd(c.origin[k], __fma_rn(z, c.basis[6 + k], __fma_rn(y, c.basis[3 + k], dmul(x, c.basis[k]))));
        const double d0 = dsub(wv[0], g.fo[0]), d1 = dsub(wv[1], g.fo[1]), d2 = dsub(wv[2], g.fo[2]);
        const double lx = __fma_rn(d2, g.fb[2], __fma_rn(d1, g.fb[1], dmul(d0, g.fb[0])));
        const double ly = __fma_rn(d2, g.fb[5], __fma_rn(d1, g.fb[4], dmul(d0, g.fb[3])));
        const double lz = __fma_rn(d2, g.fb[8], __fma_rn(d1, g.fb[7], dmul(d0, g.fb[6])));
        valid = lz > 0;
        if (valid) {
          const double zh = dmul(lz, g.fh);
          const double r = rcp_nr(zh);
          int ix = quant_fast(0.5 + (0.5 * lx) * r, g.nx, kM);
          int iy = ix == -1 ? -1 : quant_fast(0.5 + (0.5 * ly) * r, g.ny, kM);
          int iz = (ix == -1 || iy == -1 || g.depth_log) ? -2 : quant_fast((lz - g.fnear) * rfn, g.nz, kM);
          if (ix == -2) ix = quant_exact(dadd(0.5, ddiv(dmul(0.5, lx), zh)), g.nx);
          if (iy == -2) iy = quant_exact(dadd(0.5, ddiv(dmul(0.5, ly), zh)), g.ny);
          if (iz == -2 && ix >= 0 && iy >= 0)
            iz = quant_exact(g.depth_log ? ddiv(log(ddiv(lz, g.fnear)), g.flogr)
                                         : ddiv(dsub(lz, g.fnear), dsub(g.ffar, g.fnear)), g.nz);
          valid = ix >= 0 && iy >= 0 && iz >= 0;
          if (valid) {
            const unsigned long long byte = (unsigned long long)(ix >> 3) +
                                            (unsigned long long)row * ((unsigned long long)iy + (unsigned long long)g.ny * iz);
            word = (unsigned int)(byte >> 2);
            bit = 1u << ((((unsigned int)byte & 3u) << 3) | ((unsigned int)ix & 7u));
          }
        }
      }
    }
    const unsigned int vm = __ballot_sync(0xffffffffu, valid);
    if (vm) {
      const int leader = __ffs(vm) - 1;
      const unsigned int w0 = __shfl_sync(0xffffffffu, word, leader);
      if (__all_sync(0xffffffffu, !valid || word == w0)) {
        const unsigned int bits = __reduce_or_sync(0xffffffffu, valid ? bit : 0u);
        if (lane == leader) {
          or_bits(gt_words + w0, bits);
          if (geo_words) or_bits(geo_words + w0, bits);
        }
      } else if (valid) {
        or_bits(gt_words + word, bit);
        if (geo_words) or_bits(geo_words + word, bit);
      }
    }
  }
}

// DepthBuffer of oracle.py:48-62: depth (+inf where empty), prim (-1 where empty).
__global__ void depth_out_kernel(long long n, const unsigned long long* __restrict__ zbuf,
                                 const long long* __restrict__ pidbuf, double* __restrict__ depth,
                                 long long* __restrict__ prim) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long zb = zbuf[i];
    const bool hit = zb != ~0ull;
    if (depth) depth[i] = hit ? __longlong_as_double((long long)zb) : __longlong_as_double(0x7ff0000000000000LL);
    if (prim) prim[i] = hit ? pidbuf[i] : -1;
  }
}

// z pass (+ the primitive-id tie pass) over every camera's candidate samples
inline int launch_depth(const Params& p, const GtParams& g, const fpvs_frustum* cams, const int64_t* prim_ids,
                        const Work& wk, unsigned long long* zbuf, long long* pidbuf, bool id_pass, cudaStream_t s) {
  if (spans()) {
    static const int grid[2] = {occupancy_grid(span_kernel<true, 3>), occupancy_grid(span_kernel<true, 4>)};
    span_kernel<true, 3><<<grid[0], kRasterThreads, 0, s>>>(p, g, cams, prim_ids, wk, zbuf, pidbuf);
    FPVS_CHECK_LAUNCH("depth (spans)");
    if (id_pass) {
      span_kernel<true, 4><<<grid[1], kRasterThreads, 0, s>>>(p, g, cams, prim_ids, wk, zbuf, pidbuf);
      FPVS_CHECK_LAUNCH("primitive ids (spans)");
    }
  } else {
    static const int grid = occupancy_grid(depth_kernel<0>);
    depth_kernel<0><<<grid, kRasterThreads, 0, s>>>(g, cams, prim_ids, wk, zbuf, pidbuf);
    FPVS_CHECK_LAUNCH("depth");
    if (id_pass) {
      depth_kernel<1><<<grid, kRasterThreads, 0, s>>>(g, cams, prim_ids, wk, zbuf, pidbuf);
      FPVS_CHECK_LAUNCH("primitive ids");
    }
  }
  return FPVS_OK;
}

struct GtLayout {
  size_t total, slots, lp, bsum, bpre, zbuf, pid, ufx, ufy, bytes;
};

constexpr int kMaxRes = 1 << 15;  // depth-buffer width / height bound of the pixel tables

inline GtLayout gt_layout(long long ntris, int nviews, long long npix, bool with_pids) {
  GtLayout L;
  const long long flat = (ntris > 0 ? ntris : 1) * (long long)(nviews > 0 ? nviews : 1);
  const long long nslot = 2 * flat;
  const long long nb = (nslot + kSlotsPerBlock - 1) / kSlotsPerBlock;
  size_t o = 0;
  L.total = o; o = up256(o + 8);
  L.slots = o; o = up256(o + (size_t)nslot * sizeof(Slot));
  L.lp = o;    o = up256(o + (size_t)nslot * 8);
  L.bsum = o;  o = up256(o + (size_t)nb * 8);
  L.bpre = o;  o = up256(o + (size_t)nb * 8);
  L.zbuf = o;  o = up256(o + (size_t)nviews * (size_t)npix * 8);
  L.pid = o;   o = up256(o + (with_pids ? (size_t)nviews * (size_t)npix * 8 : 0));
  L.ufx = o;   o = up256(o + (size_t)npix * 0 + 8 * (size_t)kMaxRes);
  L.ufy = o;   o = up256(o + 8 * (size_t)kMaxRes);
  L.bytes = o;
  return L;
}

}  // namespace frox
}  // namespace fpvs

extern "C" size_t fpvs_gt_pvs_workspace_size(long long ntris, int ncams, int res_w, int res_h, int with_prim_ids) {
  if (ntris < 0 || ncams < 0 || res_w <= 0 || res_h <= 0) return 0;
  return gt_layout(ntris, ncams, (long long)res_w * res_h, with_prim_ids != 0).bytes;
}

extern "C" int fpvs_gt_pvs(const double* verts, long long nverts, const int64_t* tris, long long ntris,
                           const int64_t* prim_ids, const fpvs_frustum* cams, int ncams, int res_w, int res_h,
                           const fpvs_frustum* fr, int Nx, int Ny, int Nz, int depth_mode, int accumulate,
                           uint8_t* gt_bits, uint8_t* geometry_bits, void* workspace, size_t workspace_bytes,
                           void* stream) {
  FPVS_CHECK_ARG(fr != nullptr && gt_bits != nullptr, "gt_pvs: null frustum or output");
  FPVS_CHECK_ARG(Nx > 0 && Ny > 0 && Nz > 0 && Nx % 8 == 0, "N_x must be divisible by 8, got %d", Nx);
  FPVS_CHECK_ARG(res_w >= Nx && res_h >= Ny, "depth buffer must be at least the grid cross-section");
  FPVS_CHECK_ARG((long long)res_w * res_h < (1LL << 32) && res_w <= kMaxRes && res_h <= kMaxRes,
                 "gt_pvs: depth buffer %d x %d too large", res_w, res_h);
  FPVS_CHECK_ARG(depth_mode == FPVS_DEPTH_LINEAR || depth_mode == FPVS_DEPTH_LOG, "bad depth mode %d", depth_mode);
  FPVS_CHECK_ARG(ncams >= 0 && (ncams == 0 || cams != nullptr), "gt_pvs: bad camera array");
  FPVS_CHECK_ARG((long long)ncams * (((long long)res_w * res_h + 255) / 256) < (1LL << 32),
                 "gt_pvs: too many cameras for one call (%d)", ncams);
  FPVS_CHECK_ARG(ntris >= 0 && nverts >= 0 && (ntris == 0 || (verts && tris)), "gt_pvs: bad scene arrays");
  FPVS_CHECK_ARG(fr->near_z > 0 && fr->near_z < fr->far_z && fr->half_extent > 0, "need 0 < near < far");
  const long long grid_bytes = (long long)Nx * Ny * Nz / 8;
  FPVS_CHECK_ARG(grid_bytes % 4 == 0 && ((uintptr_t)gt_bits & 3) == 0 && ((uintptr_t)geometry_bits & 3) == 0,
                 "gt_pvs: grids must be 4-byte aligned with Nx*Ny*Nz/8 a multiple of 4");
  const long long npix = (long long)res_w * res_h;
  const GtLayout L = gt_layout(ntris, ncams, npix, prim_ids != nullptr);
  FPVS_CHECK_ARG(workspace != nullptr && workspace_bytes >= L.bytes, "gt_pvs: workspace too small (%zu < %zu)",
                 workspace_bytes, L.bytes);
  cudaStream_t s = as_stream(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  if (!accumulate && cudaMemsetAsync(gt_bits, 0, (size_t)grid_bytes, s) != cudaSuccess) FPVS_CHECK_LAUNCH("memset");
  if (ntris == 0 || ncams == 0) return FPVS_OK;
  Work wk = {};
  wk.slots = reinterpret_cast<Slot*>(ws + L.slots);
  wk.lp = reinterpret_cast<unsigned long long*>(ws + L.lp);
  wk.bsum = reinterpret_cast<unsigned long long*>(ws + L.bsum);
  wk.bpre = reinterpret_cast<unsigned long long*>(ws + L.bpre);
  wk.total = reinterpret_cast<unsigned long long*>(ws + L.total);
  wk.nsamples = wk.total + 1;
  if (cudaMemsetAsync(wk.total, 0, 16, s) != cudaSuccess) FPVS_CHECK_LAUNCH("memset");
  wk.out_words = nullptr;
  wk.tabx = wk.taby = nullptr;
  wk.ufx = reinterpret_cast<double*>(ws + L.ufx);
  wk.ufy = reinterpret_cast<double*>(ws + L.ufy);
  wk.ntris = ntris * ncams;
  wk.nb = (int)((2 * wk.ntris + kSlotsPerBlock - 1) / kSlotsPerBlock);
  unsigned long long* zbuf = reinterpret_cast<unsigned long long*>(ws + L.zbuf);
  long long* pidbuf = prim_ids ? reinterpret_cast<long long*>(ws + L.pid) : nullptr;
  if (cudaMemsetAsync(zbuf, 0xff, (size_t)ncams * npix * 8, s) != cudaSuccess) FPVS_CHECK_LAUNCH("memset");
  if (pidbuf && cudaMemsetAsync(pidbuf, 0x7f, (size_t)ncams * npix * 8, s) != cudaSuccess) FPVS_CHECK_LAUNCH("memset");
  Params p = {};
  p.sx = (double)res_w;
  p.sy = (double)res_h;
  p.isx = 0;  // no pixel->froxel tables in this mode
  p.isy = 0;
  p.nx = Nx;
  p.ny = Ny;
  p.nz = Nz;
  p.depth_log = 0;
  p.rows_mode = spans() ? 1 : 0;
  p.seg = gt_seg();
  GtParams g;
  for (int i = 0; i < 3; ++i) g.fo[i] = fr->origin[i];
  for (int i = 0; i < 9; ++i) g.fb[i] = fr->basis[i];
  g.fh = fr->half_extent;
  g.fnear = fr->near_z;
  g.ffar = fr->far_z;
  g.flogr = log(fr->far_z / fr->near_z);
  g.W = (double)res_w;
  g.H = (double)res_h;
  g.iw = res_w;
  g.ih = res_h;
  g.nx = Nx;
  g.ny = Ny;
  g.nz = Nz;
  g.depth_log = depth_mode == FPVS_DEPTH_LOG;
  g.T = ntris;
  g.npix = npix;
  setup_kernel<true><<<wk.nb, kSetupThreads, 0, s>>>(p, cams, verts, nverts, tris, ntris, wk);
  FPVS_CHECK_LAUNCH("gt_pvs setup");
  scan_kernel<<<1, 1024, 0, s>>>(p, wk);
  FPVS_CHECK_LAUNCH("gt_pvs scan");
  {
    const int rc = launch_depth(p, g, cams, prim_ids, wk, zbuf, pidbuf, pidbuf != nullptr, s);
    if (rc) return rc;
  }
  resolve_kernel<<<kNumSMs * 8, 256, 0, s>>>(g, cams, ncams, zbuf, pidbuf, wk.ufx, wk.ufy,
                                             reinterpret_cast<unsigned int*>(gt_bits),
                                             reinterpret_cast<unsigned int*>(geometry_bits));
  FPVS_CHECK_LAUNCH("gt_pvs resolve");
  return FPVS_OK;
}

extern "C" int fpvs_render_depth(const double* verts, long long nverts, const int64_t* tris, long long ntris,
                                 const int64_t* prim_ids, const fpvs_frustum* cams, int ncams, int res_w, int res_h,
                                 double* depth_out, int64_t* prim_out, void* workspace, size_t workspace_bytes,
                                 void* stream) {
  FPVS_CHECK_ARG(res_w > 0 && res_h > 0 && (long long)res_w * res_h < (1LL << 32), "render_depth: bad resolution");
  FPVS_CHECK_ARG(ncams >= 0 && (ncams == 0 || cams != nullptr), "render_depth: bad camera array");
  FPVS_CHECK_ARG(ntris >= 0 && nverts >= 0 && (ntris == 0 || (verts && tris)), "render_depth: bad scene arrays");
  const long long npix = (long long)res_w * res_h;
  const GtLayout L = gt_layout(ntris, ncams, npix, true);
  FPVS_CHECK_ARG(workspace != nullptr && workspace_bytes >= L.bytes, "render_depth: workspace too small (%zu < %zu)",
                 workspace_bytes, L.bytes);
  if (ncams == 0) return FPVS_OK;
  cudaStream_t s = as_stream(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  unsigned long long* zbuf = reinterpret_cast<unsigned long long*>(ws + L.zbuf);
  long long* pidbuf = reinterpret_cast<long long*>(ws + L.pid);
  if (cudaMemsetAsync(zbuf, 0xff, (size_t)ncams * npix * 8, s) != cudaSuccess) FPVS_CHECK_LAUNCH("memset");
  if (cudaMemsetAsync(pidbuf, 0x7f, (size_t)ncams * npix * 8, s) != cudaSuccess) FPVS_CHECK_LAUNCH("memset");
  if (ntris > 0) {
    Work wk = {};
    wk.slots = reinterpret_cast<Slot*>(ws + L.slots);
    wk.lp = reinterpret_cast<unsigned long long*>(ws + L.lp);
    wk.bsum = reinterpret_cast<unsigned long long*>(ws + L.bsum);
    wk.bpre = reinterpret_cast<unsigned long long*>(ws + L.bpre);
    wk.total = reinterpret_cast<unsigned long long*>(ws + L.total);
    wk.nsamples = wk.total + 1;
    if (cudaMemsetAsync(wk.total, 0, 16, s) != cudaSuccess) FPVS_CHECK_LAUNCH("memset");
    wk.ntris = ntris * ncams;
    wk.nb = (int)((2 * wk.ntris + kSlotsPerBlock - 1) / kSlotsPerBlock);
    Params p = {};
    p.sx = (double)res_w;
    p.sy = (double)res_h;
    p.rows_mode = spans() ? 1 : 0;
    p.seg = gt_seg();
    GtParams g = {};
    g.iw = res_w;
    g.ih = res_h;
    g.W = (double)res_w;
    g.H = (double)res_h;
    g.T = ntris;
    g.npix = npix;
    setup_kernel<true><<<wk.nb, kSetupThreads, 0, s>>>(p, cams, verts, nverts, tris, ntris, wk);
    FPVS_CHECK_LAUNCH("render_depth setup");
    scan_kernel<<<1, 1024, 0, s>>>(p, wk);
    FPVS_CHECK_LAUNCH("render_depth scan");
    const int rc = launch_depth(p, g, cams, prim_ids, wk, zbuf, pidbuf, true, s);
    if (rc) return rc;
  }
  depth_out_kernel<<<kNumSMs * 8, 256, 0, s>>>((long long)ncams * npix, zbuf, pidbuf, depth_out, reinterpret_cast<long long*>(prim_out));
  FPVS_CHECK_LAUNCH("render_depth out");
  return FPVS_OK;
}
