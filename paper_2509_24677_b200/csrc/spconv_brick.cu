// (3d) Submanifold 3x3x3 sparse convolution over DENSE BRICKS of a
// well-filled level (tcgen05, both operands straight from shared memory, no
// A builders).  Same result as fpvs_spconv_halo / Conv3d.forward on the
// active set (pkg/src/froxelpvs/neural.py:187-219) for Cin, Cout multiples
// of 64: inactive cells read as zero rows, only active rows are written.
//
// Why: the sparse-tile kernels gather every tap's A operand row by row (the
// halo kernel's builder warps), and at levels 1-2 the per-chunk hand-off
// between builders and the MMA issuer paces the conv.  On a
// level that is mostly active (config 2's level 2: 90 % of the 16^3 cells)
// a brick of 1 x 16 x 8 cells is an M = 128 tile whose 27 tap operands are
// all SHIFTED VIEWS of one dense halo brick (3 x 18 x 10 cells) in shared
// memory: with the 128-byte swizzle written by absolute address, a K-major
// SS descriptor may start at any 128-byte row and use a 10-row stride
// between its 8-row groups (tools/micro_desc.cu), so tap (a, b, c) reads
// rows a*180 + b*10 + c + (y*10 + z) directly.  Per (brick, 64-channel
// chunk) the kernel:
//   * 4 loader warps: per halo cell, its row from the level's index volume
//     (-1 / outside the grid -> zeros) and a cp.async (zero-fill) of its 128
//     bytes into a double-buffered halo brick;
//   * 1 warp: bulk copy of the pre-swizzled weight chunk of each tap;
//   * 1 thread: 27 taps x 4 tcgen05.mma (M = 128, N = BN, K = 16) with A and
//     B descriptors into a double-buffered fp32 TMEM accumulator;
//   * 4 epilogue warps: tcgen05.ld, bias + ReLU, bf16 rows of the active
//     cells; or a K split over channel chunks with fp32 partials and the
//     fixed-order reduction by the tile's last CTA (as spconv_halo).
// The MMA runs the channel chunks outer, taps inner (the halo kernel's
// order); taps absent from a row read zeros.
#include <stdlib.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace fpvs {
namespace brick {

using namespace tc;

constexpr int BY = 16, BZ = 8;                 // brick = 1 x BY x BZ cells = the 128 tile rows
constexpr int HY = BY + 2, HZ = BZ + 2;        // halo brick: 3 x HY x HZ cells
constexpr int HPLANE = HY * HZ;                // 180 cells per x plane
constexpr int HROWS = 3 * HPLANE;              // 540
constexpr int HBUF = (HROWS * 128 + 1023) / 1024 * 1024;  // one 64-channel chunk (1024-aligned)
constexpr int KOFF = 27;
constexpr int LOADERS = 192;                   // warps 0-3 and 6-7
constexpr int W_B = 4, W_MMA = 5, W_EPI = 8;   // epilogue warps quadrant-aligned
constexpr int THREADS = 384;

#ifndef FPVS_BRICK_NS
#define FPVS_BRICK_NS 4
#endif
// CL > 1: the K split is a thread-block cluster of CL CTAs (one unit each)
// whose fp32 partials meet in distributed shared memory (see the kernel)
template <int BN, int CL = 1>
struct Cfg {
  static constexpr int NACC = BN == 256 || CL > 1 ? 1 : 2;
  static constexpr int NHB = 2;  // the next channel chunk's halo loads while this one's taps run
  static constexpr int B_SUB = BN * 128;
  // weight stages (one tap's chunk each, a power of two)
  static constexpr int NS = BN == 256 ? 2 : BN == 128 ? FPVS_BRICK_NS : 8;
  static constexpr int B_OFF = NHB * HBUF;
  static constexpr int BAR_OFF = B_OFF + NS * B_SUB;
  static constexpr int NBARS = 2 * NS + 2 * NACC + 2 * NHB;
  static constexpr int CTRL_OFF = BAR_OFF + 8 * NBARS;
  static constexpr int BIAS_OFF = CTRL_OFF + 64;
  static constexpr int SMEM = 1024 + BIAS_OFF + 4 * 1024;
  static constexpr int TMEM_COLS = 256;
  static constexpr int SPITCH = BN + 4;  // cluster mode: staged partial row pitch (floats)
  static_assert(NACC * BN <= TMEM_COLS, "TMEM columns");
  static_assert(SMEM <= 232448, "shared memory budget");
  static_assert(CL == 1 || 128 * SPITCH * 4 <= BAR_OFF, "staged partial fits the halo + weight space");
};

struct Params {
  const __nv_bfloat16* x;
  int ldx;
  const int* index_vol;  // level cell (C order) -> row, -1 inactive
  int B, X, Y, Z, nby, nbz;
  const uint8_t* wpk;    // fpvs_pack_weights_tc image (K = 27, bn)
  int nchunks, nblk, split, cpo;
  const float* bias;
  int cout, act;
  __nv_bfloat16* y;
  int ldy, col_off;
  float* part;           // [items][split][128][BN] fp32 partials (split > 1)
  int* counters;         // [items], zero between launches
  int settled;           // index_vol is two or more launches old: read before the PDL wait
  int abl;               // profiling builds (FPVS_BRICK_ABL, wrong results): 1 weights only for the first stages
  int slot;              // profiling builds: timestamp slot of this launch
};

struct Unit {
  int b, x, y0, z0, nb, s, item, c0, c1;
};

__device__ __forceinline__ void unit_of(const Params& p, int u, Unit& U) {
  U.item = u / p.split;
  U.s = u - U.item * p.split;
  int t = U.item / p.nblk;
  U.nb = U.item - t * p.nblk;
  const int bz = t % p.nbz;
  t /= p.nbz;
  const int by = t % p.nby;
  t /= p.nby;
  U.x = t % p.X;
  U.b = t / p.X;
  U.y0 = by * BY;
  U.z0 = bz * BZ;
  U.c0 = U.s * p.cpo / p.split;
  U.c1 = (U.s + 1) * p.cpo / p.split;
}

// K-major SW128 descriptor with an arbitrary 8-row-group stride (bytes)
__device__ __forceinline__ uint64_t sw128_desc_sbo(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(sbo >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// profiling builds: per-CTA globaltimer stamps (start, after the PDL wait,
// first halo landed, first MMA issued, last MMA committed, epilogue start /
// end of its last unit) — tools/brick_timeline.py
#ifdef FPVS_PROFILE
__device__ unsigned long long g_bts[2][160][8];  // [launch slot][CTA][event]
__device__ long long g_bclk[2][160][8];
static int g_bslot = 0;  // host: launch counter (slot = parity, so two consecutive launches keep their stamps)
#define BTS(i)                                                                      \
  do {                                                                              \
    if (blockIdx.x < 160) {                                                         \
      unsigned long long t_;                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                        \
      g_bts[p.slot][blockIdx.x][i] = t_;                                            \
      g_bclk[p.slot][blockIdx.x][i] = clock64();                                    \
    }                                                                               \
  } while (0)
#else
#define BTS(i) \
  do {         \
  } while (0)
#endif

// One channel chunk's 27 taps: a loop over the 9 (a, b) tap rows with the 3
// taps of a row unrolled.  tcgen05.mma issue is effectively synchronous, so
// the issuing thread's work between MMAs adds to their cost
// (tools/micro_sbo.cu: the brick-view MMAs at the 64-cycle compute floor
// with all 27 taps unrolled, 81 with divisions in the loop); but a fully
// unrolled chunk is ~6 KB of straight-line code run once per chunk, and in
// the frame (the kernel's code cold in the instruction caches after the
// previous kernel) its fetch latency doubled the MMA phase.  Here the
// per-tap work is a few adds and shifts: the stage index and its phase come
// from a running counter (NS is a power of two), the descriptors advance by
// constants.
template <class C>
__device__ __forceinline__ uint32_t chunk_taps(uint32_t st, uint32_t full0, uint32_t empty0, uint64_t a0,
                                               uint64_t b0, uint32_t dtm, uint32_t idesc, uint32_t accum) {
  static_assert((C::NS & (C::NS - 1)) == 0, "power-of-two weight ring");
  constexpr int LOG_NS = C::NS == 2 ? 1 : C::NS == 4 ? 2 : C::NS == 8 ? 3 : 4;
#pragma unroll 1
  for (int ab = 0; ab < 9; ++ab) {
    const int a = ab / 3, b = ab - 3 * (ab / 3);
    // tap (a, b, cc) of output row (y, z) reads halo row a*180 + (y+b)*10 + z+cc
    const uint64_t arow = a0 + (uint64_t)(((a * HPLANE + b * HZ) * 128) >> 4);
#pragma unroll
    for (int cc = 0; cc < 3; ++cc, ++st) {
      const uint32_t stage = st & (C::NS - 1);
      mbar_wait(full0 + 8 * stage, (st >> LOG_NS) & 1u);
      tc_fence_after();
      const uint64_t ad = arow + (uint64_t)((cc * 128) >> 4);
      const uint64_t bd = b0 + (uint64_t)(stage * (C::B_SUB >> 4));
#pragma unroll
      for (int k = 0; k < BK / 16; ++k) umma_bf16(dtm, ad + 2 * k, bd + 2 * k, idesc, (ab | cc | k) ? 1u : accum);
      umma_commit(empty0 + 8 * stage);
    }
  }
  return st;
}

__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int BN, int CL>
__global__ void __launch_bounds__(THREADS, 1) spconv_brick_kernel(const Params p) {
  using C = Cfg<BN, CL>;
  constexpr int NHB = C::NHB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* sB = smem + C::B_OFF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* full = bars;
  uint64_t* empty = full + C::NS;
  uint64_t* tfull = empty + C::NS;
  uint64_t* tempty = tfull + C::NACC;
  uint64_t* hfull = tempty + C::NACC;
  uint64_t* hempty = hfull + NHB;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + C::CTRL_OFF);
  volatile int* s_last = reinterpret_cast<volatile int*>(smem + C::CTRL_OFF + 16);
  float* s_bias = reinterpret_cast<float*>(smem + C::BIAS_OFF);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nunits = p.B * p.X * p.nby * p.nbz * p.nblk * p.split;
  if (tid == 0) BTS(0);
  if (tid == 0) {
    for (int s = 0; s < C::NS; ++s) {
      mbar_init(smem_u32(full + s), 1);
      mbar_init(smem_u32(empty + s), 1);
    }
    for (int a = 0; a < C::NACC; ++a) {
      mbar_init(smem_u32(tfull + a), 1);
      mbar_init(smem_u32(tempty + a), 4);
    }
    for (int h = 0; h < NHB; ++h) {
      mbar_init(smem_u32(hfull + h), LOADERS / 32);
      mbar_init(smem_u32(hempty + h), 1);
    }
    fence_mbar_init();
  }
  for (int c = tid; c < p.cout; c += THREADS) s_bias[c] = p.bias ? p.bias[c] : 0.f;
  if (warp == W_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "n"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *s_tmem;
  // x (and the packed weights, in training) may be the previous launch's
  // output: every role waits before touching them; the index volume is the
  // map build's, read before the wait only when the caller says it is two or
  // more launches old (FPVS_TABLES_SETTLED)
  if (!p.settled) pdl_wait();

  if (warp < 4 || warp == 6 || warp == 7) {
    // ===================== halo-brick loaders =====================
    // a thread's halo rows (h = lt + k * 192): their feature rows are looked
    // up once per unit, all loads in flight together (a dependent lookup per
    // row serialised ~5 L2 round trips per chunk), and reused for every
    // channel chunk of the unit
    constexpr int RPT = (HROWS + LOADERS - 1) / LOADERS;
    const int lt = warp < 4 ? tid : tid - 64;  // loader thread 0..191
    const uint32_t ldx2 = (uint32_t)p.ldx * 2u;
    const long long plane = (long long)p.Y * p.Z;
    auto lookup = [&](const Unit& U, int (&rows)[RPT]) {
      const long long vol0 = (long long)U.b * p.X * plane;
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        const int h = lt + k * LOADERS;
        const int i = h / HPLANE, rem = h - i * HPLANE, jy = rem / HZ, jz = rem - jy * HZ;
        const int cx = U.x - 1 + i, cy = U.y0 - 1 + jy, cz = U.z0 - 1 + jz;
        rows[k] = (h < HROWS && cx >= 0 && cx < p.X && cy >= 0 && cy < p.Y && cz >= 0 && cz < p.Z)
                      ? __ldg(p.index_vol + vol0 + ((long long)cx * p.Y + cy) * p.Z + cz)
                      : -1;
      }
    };
    int rows[RPT];
    if ((int)blockIdx.x < nunits) {
      Unit U;
      unit_of(p, blockIdx.x, U);
      lookup(U, rows);
    }
    pdl_wait();
    if (lt == 0) pdl_trigger();
    if (lt == 0) BTS(1);
    uint32_t gc = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      unit_of(p, u, U);
      if (u != (int)blockIdx.x) lookup(U, rows);
      for (int c = U.c0; c < U.c1; ++c, ++gc) {
        const int hb = gc % NHB;
        mbar_wait_sleep(smem_u32(hempty + hb), ((gc / NHB) & 1) ^ 1, 64);
        const uint32_t hs = smem_u32(smem + hb * HBUF);
        const char* xc = reinterpret_cast<const char*>(p.x) + c * 128;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const int h = lt + k * LOADERS;
          if (h >= HROWS) break;
          const char* src = xc + (long long)(rows[k] >= 0 ? rows[k] : 0) * ldx2;
#pragma unroll
          for (int pc = 0; pc < 8; ++pc)
            cp_async16_zfill(hs + h * 128 + ((pc ^ (h & 7)) << 4), src + pc * 16, rows[k] < 0);
        }
        cp_async_commit();
        cp_async_wait<0>();
        fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tensor-core (async proxy) reads
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(hfull + hb));
        if (lt == 0 && gc == 0) BTS(2);
      }
    }
  } else if (warp == W_B) {
    // ===================== weight loader =====================
    pdl_wait();
    if (lane == 0) {
      uint32_t st = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        Unit U;
        unit_of(p, u, U);
        const uint8_t* wblk = p.wpk + (size_t)U.nb * p.nchunks * C::B_SUB;
        for (int c = U.c0; c < U.c1; ++c)
          for (int j = 0; j < KOFF; ++j, ++st) {
            const int stage = (int)(st % C::NS);
            mbar_wait(smem_u32(empty + stage), ((st / C::NS) & 1) ^ 1);
            const uint32_t fb = smem_u32(full + stage);
#ifdef FPVS_PROFILE
            if ((p.abl & 1) && st >= (uint32_t)C::NS) {
              mbar_arrive(fb);
              continue;
            }
#endif
            mbar_arrive_expect_tx(fb, C::B_SUB);
            bulk_g2s(smem_u32(sB + stage * C::B_SUB), wblk + (size_t)(j * p.cpo + c) * C::B_SUB, C::B_SUB, fb);
          }
      }
    }
  } else if (warp == W_MMA) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16<BN>();
      const uint64_t b_desc0 = sw128_desc(smem_u32(sB));
      uint32_t st = 0, gc = 0;
      int it = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
        Unit U;
        unit_of(p, u, U);
        const int acc = it % C::NACC;
        mbar_wait(smem_u32(tempty + acc), ((it / C::NACC) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dtm = tmem_base + acc * BN;
        for (int c = U.c0; c < U.c1; ++c, ++gc) {
          const int hb = gc % NHB;
          mbar_wait(smem_u32(hfull + hb), (gc / NHB) & 1);
          tc_fence_after();
          // 8-row groups (one y of the brick) are HZ = 10 halo rows apart
          const uint64_t a_desc0 = sw128_desc_sbo(smem_u32(smem + hb * HBUF), HZ * 128);
          if (st == 0) BTS(3);
          st = chunk_taps<C>(st, smem_u32(full), smem_u32(empty), a_desc0, b_desc0, dtm, idesc, c == U.c0 ? 0u : 1u);
          if (st == KOFF) BTS(7);
          umma_commit(smem_u32(hempty + hb));  // the halo brick is free once these MMAs are done
        }
        umma_commit(smem_u32(tfull + acc));
        BTS(4);
      }
    }
  } else if (warp >= W_EPI) {
    // ===================== epilogue (4 warps) =====================
    pdl_wait();  // y may still be read by the previous launch
    const int q4 = warp & 3, r = q4 * 32 + lane;
    const uint32_t tlane = (uint32_t)(q4 * 32) << 16;
    const int yl = r / BZ, zl = r - yl * BZ;
    int it = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
      Unit U;
      unit_of(p, u, U);
      const int cy = U.y0 + yl, cz = U.z0 + zl;
      int row = -1;
      if (cy < p.Y && cz < p.Z)
        row = __ldg(p.index_vol + (((long long)U.b * p.X + U.x) * p.Y + cy) * p.Z + cz);
      const bool valid = row >= 0;
      const int acc = it % C::NACC;
      mbar_wait_sleep(smem_u32(tfull + acc), (it / C::NACC) & 1, 128);
      tc_fence_after();
      if (warp == W_EPI && lane == 0) BTS(5);
      const int col0 = U.nb * BN;
      if constexpr (CL > 1) {
        // cluster split: this CTA's fp32 partial into its own shared memory
        // (the halo + weight space, idle once the MMAs are done), row r at
        // r * SPITCH floats; the cluster sums the partials below
        float* stg = reinterpret_cast<float*>(smem) + r * C::SPITCH;
#pragma unroll 1
        for (int cb = 0; cb < BN; cb += 32) {
          float v[32];
          tmem_ldn<32>(tmem_base + tlane + acc * BN + cb, v);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            *reinterpret_cast<float4*>(stg + cb + 4 * i) = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
      } else if (p.split == 1) {
#pragma unroll 1
        for (int cb = 0; cb < BN; cb += 32) {
          float v[32];
          tmem_ldn<32>(tmem_base + tlane + acc * BN + cb, v);
          if (!valid) continue;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float z = v[i] + s_bias[col0 + cb + i];
            v[i] = p.act == FPVS_ACT_RELU ? fmaxf(z, 0.f) : z;
          }
          uint4* dst = reinterpret_cast<uint4*>(p.y + (long long)row * p.ldy + p.col_off + col0 + cb);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(pack_bf16x2(v[8 * i + 0], v[8 * i + 1]), pack_bf16x2(v[8 * i + 2], v[8 * i + 3]),
                                pack_bf16x2(v[8 * i + 4], v[8 * i + 5]), pack_bf16x2(v[8 * i + 6], v[8 * i + 7]));
        }
      } else {
        // channel-chunk split: fp32 partial [col][128 rows] per split (coalesced);
        // the last CTA of the (brick, column block) sums them in split order
        float* mine = p.part + ((long long)U.item * p.split + U.s) * BM * BN + r;
#pragma unroll 1
        for (int cb = 0; cb < BN; cb += 32) {
          float v[32];
          tmem_ldn<32>(tmem_base + tlane + acc * BN + cb, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) __stcg(mine + (cb + i) * BM, v[i]);
        }
        named_bar(1, 128);
        if (warp == W_EPI && lane == 0) {
          __threadfence();  // release this CTA's partial before the count
          const int last = atomicAdd(p.counters + U.item, 1) == p.split - 1;
          if (last) __threadfence();  // acquire the other splits' partials
          *s_last = last;
        }
        named_bar(1, 128);
        if (*s_last) {
          const float* base = p.part + (long long)U.item * p.split * BM * BN + r;
#pragma unroll 1
          for (int cb = 0; cb < BN; cb += 32) {
            float own[32], v[32];
            tmem_ldn<32>(tmem_base + tlane + acc * BN + cb, own);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
            for (int ss = 0; ss < p.split; ++ss) {
              if (ss == U.s) {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] += own[i];
              } else {
                const float* src = base + (long long)ss * BM * BN + cb * BM;
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] += __ldcg(src + i * BM);
              }
            }
            if (!valid) continue;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float z = v[i] + s_bias[col0 + cb + i];
              v[i] = p.act == FPVS_ACT_RELU ? fmaxf(z, 0.f) : z;
            }
            uint4* dst = reinterpret_cast<uint4*>(p.y + (long long)row * p.ldy + p.col_off + col0 + cb);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              dst[i] = make_uint4(pack_bf16x2(v[8 * i + 0], v[8 * i + 1]), pack_bf16x2(v[8 * i + 2], v[8 * i + 3]),
                                  pack_bf16x2(v[8 * i + 4], v[8 * i + 5]), pack_bf16x2(v[8 * i + 6], v[8 * i + 7]));
          }
          if (warp == W_EPI && lane == 0) p.counters[U.item] = 0;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(tempty + acc));
      if (warp == W_EPI && lane == 0) BTS(6);
    }
  }
  if constexpr (CL > 1) {
    // The CL CTAs of a cluster hold the CL channel-chunk partials of one
    // (brick, column block); CTA q sums rows [q R, (q + 1) R) over the
    // cluster's shared memories in split order (the fixed order of the
    // partial-buffer path, so both give the same bits) and writes them.
    cluster_sync_all();  // every partial staged
    if (warp >= W_EPI) {
      constexpr int R = 128 / CL, TPR = 128 / R, CPT = BN / TPR;  // rows per CTA, threads per row, columns per thread
      const int t = tid - W_EPI * 32;
      const int q = (int)(blockIdx.x % CL);
      Unit U;
      unit_of(p, blockIdx.x, U);
      const int rr = q * R + t / TPR, c0 = (t % TPR) * CPT;
      const int cy = U.y0 + rr / BZ, cz = U.z0 + rr % BZ;
      const int row = (cy < p.Y && cz < p.Z)
                          ? __ldg(p.index_vol + (((long long)U.b * p.X + U.x) * p.Y + cy) * p.Z + cz) : -1;
      if (row >= 0) {
        const uint32_t local = smem_u32(smem) + (uint32_t)((rr * C::SPITCH + c0) * 4);
        const int col0 = U.nb * BN + c0;
#pragma unroll 1
        for (int cb = 0; cb < CPT; cb += 8) {
          float v[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) v[i] = 0.f;
#pragma unroll
          for (int src = 0; src < CL; ++src) {
            const uint32_t a = mapa_shared(local + cb * 4, (uint32_t)src);
            const float4 x0 = ld_dsmem_f4(a), x1 = ld_dsmem_f4(a + 16);
            v[0] += x0.x; v[1] += x0.y; v[2] += x0.z; v[3] += x0.w;
            v[4] += x1.x; v[5] += x1.y; v[6] += x1.z; v[7] += x1.w;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float z = v[i] + s_bias[col0 + cb + i];
            v[i] = p.act == FPVS_ACT_RELU ? fmaxf(z, 0.f) : z;
          }
          *reinterpret_cast<uint4*>(p.y + (long long)row * p.ldy + p.col_off + col0 + cb) =
              make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                         pack_bf16x2(v[6], v[7]));
        }
      }
    }
    cluster_sync_all();  // the peers are done reading this CTA's partial
  }
  tc_fence_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(C::TMEM_COLS)
                 : "memory");
  }
}

template <int BN, int CL>
int launch(const Params& p, long long units, cudaStream_t s) {
  using C = Cfg<BN, CL>;
  const cudaError_t ea = set_smem_once<spconv_brick_kernel<BN, CL>>(C::SMEM);
  if (ea != cudaSuccess) return set_error(FPVS_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(ea));
  cudaError_t e;
  if constexpr (CL == 1) {
    const int grid = (int)(units < kNumSMs ? units : kNumSMs);
    e = launch_kernel(spconv_brick_kernel<BN, 1>, dim3(grid), dim3(THREADS), C::SMEM, s, p);
  } else {
    // one unit per CTA, the CL splits of an item = one cluster
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)units);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    e = cudaLaunchKernelEx(&cfg, spconv_brick_kernel<BN, CL>, p);
  }
  if (e != cudaSuccess) return set_error(FPVS_ECUDA, "spconv_brick: %s", cudaGetErrorString(e));
  FPVS_CHECK_LAUNCH("spconv_brick");
  return FPVS_OK;
}

inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// FPVS_BRICK_CLUSTER=0 keeps K splits on the partial-buffer path (A/B checks; read once)
inline bool cluster_enabled() {
  static const bool on = [] {
    const char* e = getenv("FPVS_BRICK_CLUSTER");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace brick
}  // namespace fpvs

using namespace fpvs;

#ifdef FPVS_PROFILE
extern "C" int fpvs_debug_brick_times(unsigned long long* host) {  // [2][160][8]
  return cudaMemcpyFromSymbol(host, brick::g_bts, sizeof(unsigned long long) * 2 * 160 * 8) == cudaSuccess ? 0 : 3;
}
extern "C" int fpvs_debug_brick_clocks(long long* host) {
  return cudaMemcpyFromSymbol(host, brick::g_bclk, sizeof(long long) * 2 * 160 * 8) == cudaSuccess ? 0 : 3;
}
extern "C" void fpvs_debug_brick_reset_slot(void) { brick::g_bslot = 0; }
#endif

extern "C" size_t fpvs_spconv_brick_workspace_size(int B, int X, int Y, int Z, int cout, int bn, int split) {
  if (B < 1 || X < 1 || Y < 1 || Z < 1 || (bn != 64 && bn != 128 && bn != 256) || split < 1 || cout % bn)
    return 0;
  const size_t bricks = (size_t)B * X * ((Y + brick::BY - 1) / brick::BY) * ((Z + brick::BZ - 1) / brick::BZ);
  const size_t items = bricks * (cout / bn);
  size_t b = brick::align256(items * 4);
  if (split > 1) b += items * split * tc::BM * bn * 4;
  return b;
}

extern "C" int fpvs_spconv_brick(const void* x, int ldx, int x_rows, const int32_t* index_vol, int B, int X, int Y,
                                 int Z, const void* w_packed, int bn, int split, const float* bias, int cin, int cout,
                                 int act, void* y, int ldy, int col_off, void* ws, size_t ws_bytes, void* stream) {
  FPVS_CHECK_ARG(x && index_vol && w_packed && y, "null pointer");
  const int settled = (act & FPVS_TABLES_SETTLED) != 0;
  act &= ~FPVS_TABLES_SETTLED;
  FPVS_CHECK_ARG(B >= 1 && X >= 1 && Y >= 1 && Z >= 1, "level dims must be positive");
  FPVS_CHECK_ARG(bn == 64 || bn == 128 || bn == 256, "brick conv tile width must be 64, 128 or 256");
  FPVS_CHECK_ARG(cin % 64 == 0 && cin >= 64, "brick conv needs Cin %% 64 == 0, got %d", cin);
  FPVS_CHECK_ARG(cout % bn == 0 && cout <= 1024, "brick conv needs Cout %% %d == 0 (<= 1024), got %d", bn, cout);
  FPVS_CHECK_ARG(split >= 1 && (cin / 64) % split == 0, "split must divide Cin / 64");
  FPVS_CHECK_ARG(ldx % 8 == 0 && ldx >= cin, "bad input leading dimension");
  FPVS_CHECK_ARG((long long)x_rows * ldx * 2 < (1LL << 31), "feature buffer too large for 32-bit row offsets");
  FPVS_CHECK_ARG(ldy % 8 == 0 && col_off % 8 == 0 && ldy >= col_off + cout, "bad output leading dimension");
  FPVS_CHECK_ARG(act == FPVS_ACT_NONE || act == FPVS_ACT_RELU, "brick conv epilogue supports none/relu");
  const size_t need = fpvs_spconv_brick_workspace_size(B, X, Y, Z, cout, bn, split);
  FPVS_CHECK_ARG(split == 1 || (ws && ws_bytes >= need), "workspace too small: need %zu bytes", need);
  brick::Params p{};
  p.x = (const __nv_bfloat16*)x;
  p.ldx = ldx;
  p.index_vol = index_vol;
  p.B = B;
  p.X = X;
  p.Y = Y;
  p.Z = Z;
  p.nby = (Y + brick::BY - 1) / brick::BY;
  p.nbz = (Z + brick::BZ - 1) / brick::BZ;
  p.wpk = (const uint8_t*)w_packed;
  p.nchunks = 27 * cin / 64;
  p.nblk = cout / bn;
  p.split = split;
  p.cpo = cin / 64;
  p.bias = bias;
  p.cout = cout;
  p.act = act;
  p.y = (__nv_bfloat16*)y;
  p.ldy = ldy;
  p.col_off = col_off;
  const long long items = (long long)B * X * p.nby * p.nbz * p.nblk;
  p.settled = settled;
  p.abl = debug_knob("FPVS_BRICK_ABL");
#ifdef FPVS_PROFILE
  p.slot = brick::g_bslot++ & 1;
#endif
  p.counters = (int*)ws;
  p.part = ws ? (float*)((uint8_t*)ws + brick::align256((size_t)items * 4)) : nullptr;
  const long long units = items * split;
  const cudaStream_t st = as_stream(stream);
  // a split of 2 or 4 with at most one wave of units runs as clusters (the
  // partials meet in distributed shared memory, no workspace round trip);
  // same bits as the partial-buffer path (same summation order)
  if (units <= kNumSMs && (split == 2 || split == 4) && brick::cluster_enabled()) {
#define FPVS_BRICK_CL(BNV)                                            \
  if (bn == BNV) {                                                    \
    if (split == 2) return brick::launch<BNV, 2>(p, units, st);       \
    return brick::launch<BNV, 4>(p, units, st);                       \
  }
    FPVS_BRICK_CL(64)
    FPVS_BRICK_CL(128)
    FPVS_BRICK_CL(256)
#undef FPVS_BRICK_CL
  }
  if (bn == 64) return brick::launch<64, 1>(p, units, st);
  if (bn == 128) return brick::launch<128, 1>(p, units, st);
  return brick::launch<256, 1>(p, units, st);
}
