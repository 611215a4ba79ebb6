// (3b) Submanifold 3x3x3 sparse convolution with a per-tile halo cache
// (tcgen05, A operand in TMEM).  Replaces Conv3d.forward on the active set
// (pkg/src/froxelpvs/neural.py:187-219) for Cin, Cout multiples of 64.
//
// Why: in the plain gather-GEMM (spconv_tc.cu) every 128-row output tile
// fetches 27 x 128 neighbour rows from L2, but those rows are only ~370-450
// distinct cells (rows are in C-order, so a tile is a compact slab): the
// same feature rows are fetched ~8x, and the L2 -> SM path is the limiter.
// Here each tile's DISTINCT neighbour rows (its halo, <= 512, listed by
// fpvs_kmap_halo) are copied once per 64-channel chunk into shared memory,
// and the per-offset A operand (128 rows x 64 bf16) is assembled from
// shared memory straight into tensor memory:
//   * 2 loader warps: cp.async the halo rows of (tile, channel chunk) into
//     a double-buffered smem halo (16-byte pieces XOR-swizzled by row so the
//     builders' row reads do not bank-conflict) + a bulk copy of the tile's
//     local neighbour table (int16 halo slot per (row, offset));
//   * 8 builder warps (two groups of 4, one warp per TMEM lane quadrant,
//     alternating chunks): thread = tile row; 8 x 16-byte smem loads of the
//     neighbour's row, one tcgen05.st (32x32b.x32) into an A slot in TMEM;
//   * 1 warp: bulk copy (TMA engine) of the pre-swizzled weight chunk;
//   * 1 thread issues tcgen05.mma kind::f16 with A from TMEM, B from smem
//     (M=128, N=BN, K=16, bf16 -> fp32 TMEM), commits stages back;
//   * 4 epilogue warps: tcgen05.ld, bias + ReLU + bf16 store; or, when the
//     K range is split across CTAs (split > 1, for levels with few tiles),
//     an fp32 partial per split and a deterministic fixed-order reduction by
//     the last-arriving CTA of the tile.
// Halo slots past 512 (pathological tiles) fall back to a direct global read
// of that neighbour row, so the result never depends on the cache.
#include <limits.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "halo_build.cuh"

namespace fpvs {
namespace halo {

using namespace tc;

constexpr int HMAX = FPVS_HALO_MAX;         // halo rows cached per tile
constexpr int KOFF = 27;
constexpr int LNBR_BYTES = BM * KOFF * 2;   // int16 [128][27]
constexpr int HALO_BYTES = HMAX * 128;      // one 64-channel chunk of every halo row
constexpr int ROWS_OFF = HALO_BYTES + LNBR_BYTES;   // the tile's halo row list (int32 [HMAX])
constexpr int HBUF = (ROWS_OFF + HMAX * 4 + 1023) / 1024 * 1024;

// ------------------------------------------------------------------------
// Halo build: per 128-row tile, the sorted distinct neighbour rows and the
// local table lnbr[r][j] = slot of nbr[r][j] in that list (-1 = no
// neighbour, -2 = not cached -> direct read).
// ------------------------------------------------------------------------
struct HaloJob {
  const int* nbr;
  const int* n;
  int cap;
  int* rows;
  int* hn;
  int16_t* lnbr;
};
constexpr int kMaxHaloJobs = 4;
struct HaloJobs {
  HaloJob j[kMaxHaloJobs];
  int count;
};

// One launch for every level's table: CTA b takes active tiles b, b + grid, ...
// of the concatenated (level, tile) space (counts read on the device).
__global__ void __launch_bounds__(256) halo_build_kernel(const HaloJobs J) {
  __shared__ __align__(16) halob::Smem s;
  __shared__ int s_base[kMaxHaloJobs + 1];
  pdl_wait();  // the neighbour tables are the previous launch's output
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int l = 0; l < J.count; ++l) {
      s_base[l] = acc;
      acc += (min(*J.j[l].n, J.j[l].cap) + BM - 1) / BM;
    }
    s_base[J.count] = acc;
  }
  __syncthreads();
  const int total = s_base[J.count];
  for (int tt = blockIdx.x; tt < total; tt += gridDim.x) {
    int l = 0;
    while (tt >= s_base[l + 1]) ++l;
    const int t = tt - s_base[l];
    const int* __restrict__ nbr = J.j[l].nbr;
    const int n = min(*J.j[l].n, J.j[l].cap);
    const long long row0 = (long long)t * BM;
    halob::build_tile([&](int e) { return row0 + e / KOFF < n ? __ldg(nbr + row0 * KOFF + e) : -1; }, s,
                      J.j[l].rows + (long long)t * HMAX, J.j[l].hn + t, J.j[l].lnbr + (long long)t * BM * KOFF);
  }
}

// ------------------------------------------------------------------------
// Conv kernel
// ------------------------------------------------------------------------
struct Params {
  const __nv_bfloat16* x;
  int ldx;
  const int* nbr;
  const int16_t* lnbr;
  const int* halo_rows;
  const int* halo_n;
  const uint32_t* tile_masks;
  const int* n_dev;
  int cap;
  const uint8_t* wpk;
  int nchunks, nblk, split;  // split > 0: K ranges per item; < 0: tail balancing (see num_units)
  int smax;                   // partial slots per item in the workspace (|split|)
  const float* bias;
  int cin, cout, act;
  __nv_bfloat16* y;
  int ldy, col_off;
  float* part;    // [tiles][nblk][split][128][BN] fp32 partials (split > 1)
  int* counters;  // [tiles][nblk] arrival counters, zero between launches
  int dbg;        // profiling builds: FPVS_HALO_DEBUG (timestamps)
  int hslot;      // profiling builds: per-CTA span slot of this launch
  int abl;        // profiling builds: FPVS_HALO_ABL (ablations)
  int settled;    // tables / tile masks are two or more launches old: decode units before the PDL wait
  // tile-level dataflow between two convs of one level (fpvs_spconv_halo_flow):
  // done_out[t] reaches 4 (one release add per epilogue warp) once this launch's rows of tile t are stored
  // (zeroed by the owning CTA at its start); with done_in the launch waits for
  // the producer tiles its halo reads instead of the whole producer grid
  int* done_out;
  const int* done_in;
  // fused 1x1x1 head (dec0b of the U-Net, BN = Cout = d^3 = 64, no split):
  // the tile's bf16 activations become the A operand of 4 TS MMAs against the
  // head weights, then the row's 64 [z >= logit(tau)] bits go to row_bits
  int head;
  const uint8_t* head_wpk;   // packed head weights, 64 x 64 bf16 (one SW128 chunk)
  const float* head_bias;
  float zt;
  unsigned long long* row_bits;
};

// ---------------- profiling (profiling builds only) ----------------
// FPVS_HALO_DEBUG = 1 + 256 k: per-role timestamps of CTAs k, k + 1;
// FPVS_HALO_ABL: ablation switches for bound analysis (tools/halo_ablate.py;
// results are wrong by construction): bit 16 weight chunks only for the first
// NS stages, 17 builders skip the smem halo reads, 18 builders skip
// tcgen05.st, 19 loaders skip the halo row copies, 20 no MMAs.
#ifdef FPVS_PROFILE
__device__ unsigned long long g_hts[2][8192];   // CTAs (dbg >> 8) and (dbg >> 8) + 1
constexpr int kSpanSlots = 32;
__device__ unsigned long long g_hcta[kSpanSlots][3][160];  // [launch slot][start / end / loaders' wait done][CTA]
static int g_hslot = 0;                                    // host: halo launch counter (slot = count mod 32)
__device__ unsigned g_hsm[160];
__device__ long long g_hclk[2][160];
#define HTS(slot)                                                                        \
  do {                                                                                   \
    if (p.dbg && blockIdx.x - (unsigned)(p.dbg >> 8) < 2u && (slot) < 8192) {          \
      unsigned long long t_;                                                             \
      if (p.dbg & 128) t_ = clock64();                                                   \
      else asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                        \
      g_hts[blockIdx.x - (p.dbg >> 8)][(slot)] = t_;                                     \
    }                                                                                    \
  } while (0)
#define ABL(bit) (p.abl & (1 << (bit)))
#else
#define HTS(slot) \
  do {            \
  } while (0)
#define ABL(bit) 0
#endif

// Per-CTA unit table: the tile mask and halo size of this CTA's k-th unit,
// loaded once in the prologue so no role pays a global-memory round trip at a
// unit boundary (the MMA thread would stall ~1 us on it).
constexpr int kUnitCache = 64;
constexpr int kNumSMsForCache = 148;  // persistent grid size the unit-cache bound assumes

constexpr int LOADERS = 64;

// Warp roles for NBG builder groups of 4 warps (one warp per TMEM lane
// quadrant): warps [0, 4 NBG) build A, then 2 halo loaders, the weight loader,
// the MMA issuer (TMEM owner) and 4 epilogue warps (first one quadrant-aligned).
template <int NBG>
struct Roles {
  static constexpr int W_LOAD = 4 * NBG;   // two loader warps
  static constexpr int W_B = W_LOAD + 2;   // weight loader
  static constexpr int W_MMA = W_B + 1;    // MMA issuer, TMEM owner
  static constexpr int W_EPI = W_MMA + 1;  // epilogue warps W_EPI .. W_EPI + 3
  static constexpr int THREADS = (W_EPI + 4) * 32;
  static constexpr int NBT = 128 * NBG;  // builder threads
  static_assert(W_EPI % 4 == 0, "epilogue warps must cover the four lane quadrants in order");
};

// Pipeline stage = G = 2 K-chunks: two TMEM A slots (one per builder group)
// + two weight chunks in smem; one full/empty barrier pair and one commit per
// stage (tcgen05 commits measured ~70-150 cycles each at N <= 128).
// BN = 256 keeps a single accumulator (256 TMEM columns) and a single halo
// buffer (its smem goes to the 32 KB weight chunks).
struct Unit {
  int mt, nb, s, ns, npres, q0, q1;  // ns: how many units share this (tile, column block)
  int slot;                          // split items: partial / counter slot (tail-relative when split < 0)
  uint32_t mask;
};

#ifndef FPVS_HALO_NS128
#define FPVS_HALO_NS128 4  // stages at BN 128 (one chunk each; tools/build_variant.py A/B)
#endif
template <int BN, int NBG = 2, int MINB = 1>
struct Cfg {
  // chunks per stage: BN 64 runs 4 chunks (16 MMAs) per stage and commit, two
  // stages deep; BN >= 128: one chunk per stage, deeper weight prefetch; with
  // four builder groups BN 128 runs two chunks (8 MMAs) x two stages.
  // MINB = 2 (BN 64): two CTAs per SM, each with half the tensor memory, one
  // halo buffer and two-chunk stages; one CTA's tile-boundary and halo-load
  // gaps are filled by the other's MMAs.
  static_assert(MINB == 1 || (MINB == 2 && BN == 64 && NBG == 2), "two CTAs per SM: BN 64, two builder groups");
  static constexpr bool W2 = BN == 128 && NBG == 4;
  static constexpr int G = BN == 64 ? (MINB == 2 ? 2 : 4) : BN < 64 ? 2 : W2 ? 2 : 1;
  static constexpr int NACC = BN == 256 ? 1 : 2;
  static constexpr int NHB = BN == 256 || MINB == 2 ? 1 : 2;
  static constexpr int NS = BN == 64 || W2 ? 2 : BN == 128 ? FPVS_HALO_NS128 : 4;
  static constexpr int TMEM_COLS = MINB == 2 ? 256 : 512;
  static constexpr int BIAS_N = MINB == 2 ? 128 : 1024;  // floats (MINB 2: Cout <= 128, no head)
  static constexpr int B_SUB = BN * 128;
  static constexpr int STAGE_B = G * B_SUB;
  static constexpr int ACOL = NACC * BN;  // TMEM: [accumulators | A slots]
  static constexpr int B_OFF = NHB * HBUF;
  static constexpr int BAR_OFF = B_OFF + NS * STAGE_B;
  static constexpr int NBARS = 2 * NS + 2 * NACC + 3 * NHB + 3;  // + fused head: weights landed, head MMA done; dataflow
  static constexpr int CTRL_OFF = BAR_OFF + 8 * NBARS;
  static constexpr int BIAS_OFF = CTRL_OFF + 64;
  static constexpr int UC_OFF = BIAS_OFF + 4 * BIAS_N;  // unit cache: Unit [64] + halo sizes [64]
  static constexpr int UC_END = UC_OFF + kUnitCache * (int)sizeof(Unit) + kUnitCache * 4;
  // fused head (BN = 64 only): 8 KB of packed head weights, 1024-aligned
  static constexpr bool HEAD = BN == 64 && MINB == 1;
  static constexpr int HW_OFF = (UC_END + 1023) / 1024 * 1024;
  static constexpr int SMEM = 1024 + (HEAD ? HW_OFF + 64 * 128 : UC_END);
  static constexpr int HEAD_A = ACOL + NS * G * 32;  // TMEM: head A operand (32 cols), head accumulator (64 cols)
  static constexpr int HEAD_D = HEAD_A + 32;
  static_assert(ACOL + NS * G * 32 <= TMEM_COLS, "TMEM columns");
  static_assert(!HEAD || HEAD_D + 64 <= TMEM_COLS, "TMEM columns (fused head)");
  static_assert(SMEM <= 232448 && MINB * (SMEM + 1024) <= 233472, "shared memory budget");
};


// Work items are (tile, column block) pairs.  split > 0: every item is cut
// into `split` K ranges.  split < 0 (tail balancing): the whole waves of items
// (multiples of the grid) stay whole and only the items of the last partial
// wave are cut, into up to -split K ranges, so no CTA carries a whole extra
// item while others idle.
__device__ __forceinline__ int num_units(const Params& p, int mtiles) {
  const int items = mtiles * p.nblk;
  if (p.split > 0) return items * p.split;
  const int full = items / gridDim.x * gridDim.x, rem = items - full;
  const int ts = rem ? max(1, min(-p.split, (int)gridDim.x / rem)) : 1;
  return full + rem * ts;
}

__device__ __forceinline__ void unit_of(const Params& p, int u, int cpo, int mtiles, Unit& U) {
  int item;
  if (p.split > 0) {
    item = u / p.split;
    U.s = u - item * p.split;
    U.ns = p.split;
    U.slot = item;
  } else {
    const int items = mtiles * p.nblk;
    const int full = items / gridDim.x * gridDim.x, rem = items - full;
    const int ts = rem ? max(1, min(-p.split, (int)gridDim.x / rem)) : 1;
    if (u < full) {
      item = u;
      U.s = 0;
      U.ns = 1;
      U.slot = 0;
    } else {
      const int v = u - full;
      item = full + v / ts;
      U.s = v - (item - full) * ts;
      U.ns = ts;
      U.slot = item - full;  // < grid: the workspace holds only the tail
    }
  }
  U.mt = item / p.nblk;
  U.nb = item - U.mt * p.nblk;
  U.mask = __ldg(p.tile_masks + U.mt);
  if (p.cin == 32) {
    // Cin = 32: a 64-wide K chunk is an offset PAIR (2t, 2t + 1) x 32 channels,
    // the chunk order of the flattened (j, ci) weights; the walk runs over pairs
    uint32_t pm = 0;
#pragma unroll
    for (int t = 0; t < 14; ++t) pm |= ((U.mask >> (2 * t)) & 3u) ? (1u << t) : 0u;
    U.mask = pm ? pm : 1u << 6;
  } else if (!U.mask) {
    U.mask = 1u << 13;
  }
  U.npres = __popc(U.mask);
  // 32-bit: L <= 27 * Cin / 64 (a 64-bit divide is a long software sequence on
  // the MMA thread's critical path at every unit boundary)
  const int L = cpo * U.npres;
  if (U.ns == 1) {
    U.q0 = 0;
    U.q1 = L;
  } else {
    U.q0 = U.s * L / U.ns;
    U.q1 = (U.s + 1) * L / U.ns;
  }
}

__device__ __forceinline__ void get_unit(const Params& p, int u, int cpo, int mtiles, Unit& U, const Unit* s_units) {
  const int k = (u - (int)blockIdx.x) / (int)gridDim.x;
  if (k < kUnitCache) U = s_units[k];
  else unit_of(p, u, cpo, mtiles, U);
}

// offset of the q-th chunk inside channel chunk c: the (q - c*npres)-th set bit
__device__ __forceinline__ int first_offset(uint32_t mask, int rank) { return (int)__fns(mask, 0, rank + 1); }
__device__ __forceinline__ int next_offset(uint32_t mask, int j) { return __ffs(mask & ~((2u << j) - 1u)) - 1; }

// chunk iterator over a unit's K range: q -> (channel chunk c, offset j)
struct ChunkWalk {
  uint32_t mask;
  int npres, c, j;
  __device__ __forceinline__ void start(const Unit& U) {
    mask = U.mask;
    npres = U.npres;
    c = U.q0 / npres;
    j = first_offset(mask, U.q0 - c * npres);
  }
  __device__ __forceinline__ void next() {
    j = next_offset(mask, j);
    if (j < 0) {
      ++c;
      j = __ffs(mask) - 1;
    }
  }
};

template <int BN, bool PAIR, int NBG, int MINB>
__global__ void __launch_bounds__(Roles<NBG>::THREADS, MINB) spconv_halo_kernel(const Params p) {
  using C = Cfg<BN, NBG, MINB>;
  using R = Roles<NBG>;
  constexpr int W_LOAD = R::W_LOAD, W_B = R::W_B, W_MMA = R::W_MMA, W_EPI = R::W_EPI, THREADS = R::THREADS;
  static_assert(C::G == 1 || C::G % NBG == 0 || NBG % C::G == 0,
                "a stage's chunk slots split evenly over the builder groups (or groups over stages)");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* sB = smem + C::B_OFF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::NS;
  uint64_t* tfull = bars + 2 * C::NS;
  uint64_t* tempty = tfull + C::NACC;
  uint64_t* hfull = tempty + C::NACC;
  uint64_t* hempty = hfull + C::NHB;
  uint64_t* hmeta = hempty + C::NHB;  // the tile's local table + halo row list landed (bulk copy)
  uint64_t* hwbar = hmeta + C::NHB;   // fused head: weights landed
  uint64_t* hdbar = hwbar + 1;        // fused head: the tile's head MMAs done
  uint64_t* hdep = hdbar + 1;         // dataflow: the first unit's producer tiles are done
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + C::CTRL_OFF);
  volatile int* s_last = reinterpret_cast<volatile int*>(smem + C::CTRL_OFF + 16);
  float* s_bias = reinterpret_cast<float*>(smem + C::BIAS_OFF);
  Unit* s_units = reinterpret_cast<Unit*>(smem + C::UC_OFF);
  int* s_uhn = reinterpret_cast<int*>(smem + C::UC_OFF + kUnitCache * sizeof(Unit));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) HTS(0);
#ifdef FPVS_PROFILE
  if (p.dbg && tid == 0 && blockIdx.x < 160) {
    unsigned long long t_;
    unsigned sm_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));
    g_hcta[p.hslot][0][blockIdx.x] = t_;
    g_hsm[blockIdx.x] = sm_;
    g_hclk[0][blockIdx.x] = clock64();
  }
#endif
  const int n = min(*p.n_dev, p.cap);
  const int mtiles = (n + BM - 1) / BM;
  const int nunits = num_units(p, mtiles);
  // Cin 32 (PAIR): one 64-wide chunk per offset pair; the 64k-channel kernels
  // are compiled without the pair paths
  const int cpo = PAIR ? 1 : p.cin / BK;
  constexpr bool pair = PAIR;

  if (tid == 0) {
    for (int s = 0; s < C::NS; ++s) {
      mbar_init(smem_u32(full + s), 4 * C::G + 1);  // builder warps (4 per chunk) + the weight loader
      mbar_init(smem_u32(empty + s), 1);
    }
    for (int a = 0; a < C::NACC; ++a) {
      mbar_init(smem_u32(tfull + a), 1);
      mbar_init(smem_u32(tempty + a), 4);
    }
    for (int a = 0; a < C::NHB; ++a) {
      mbar_init(smem_u32(hfull + a), LOADERS + R::NBT);  // loaders + every builder thread (see below)
      mbar_init(smem_u32(hempty + a), 4 * NBG);
      mbar_init(smem_u32(hmeta + a), 1);
    }
    mbar_init(smem_u32(hwbar), 1);
    mbar_init(smem_u32(hdbar), 1);
    mbar_init(smem_u32(hdep), 1);
    fence_mbar_init();
  }
  for (int c = tid; c < p.cout; c += THREADS) s_bias[c] = p.bias ? p.bias[c] : 0.f;
  if (C::HEAD && p.head)
    for (int c = tid; c < 64; c += THREADS) s_bias[512 + c] = p.head_bias ? p.head_bias[c] : 0.f;
  if (tid < kUnitCache) {
    // this CTA's units decoded in parallel.  The tile masks are read before
    // the programmatic-launch wait only when the caller says they are two or
    // more launches old (FPVS_TABLES_SETTLED: every U-Net conv after the
    // first); directly after the table build (the first conv of a frame) the
    // decode waits, since only griddepcontrol.wait makes the immediately
    // preceding kernel's writes visible.  The halo sizes are read by the
    // loader warps after their wait.
    if (!p.settled) pdl_wait();
    const int u = blockIdx.x + tid * gridDim.x;
    Unit U{};
    if (u < nunits) unit_of(p, u, cpo, mtiles, U);
    s_units[tid] = U;
    // dataflow producer: this CTA's tiles are not done yet (the consumer
    // launches only after every CTA of this grid has passed its trigger, which
    // comes after this store and the fence below)
    if (p.done_out && u < nunits) p.done_out[U.mt] = 0;
  }
  if (p.done_out) __threadfence();
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
  if (tid == 0) HTS(1);

  if (warp < W_LOAD) {
    // ===================== A builders =====================
    // group bg builds half of every stage's chunk slots: with G >= 2 the
    // group owns slots [bg G/2, (bg + 1) G/2) and builds its (up to) two
    // chunks of a stage together — both chunks' halo reads in flight at once,
    // one empty-wait, two TMEM stores, one store-wait and one counted arrival
    // (measured: a builder's per-chunk sync, not its shared-memory traffic,
    // paced the N = 64 layers); with G = 1 the groups alternate stages.
    // the direct-read path reads x (the previous launch's output); in dataflow
    // mode every such read follows the loaders' wait on the producer tiles
    if (!p.done_in) pdl_wait();
    const int bg = warp >> 2, q4 = warp & 3, r = q4 * 32 + lane;
    auto grp = [](int i) { return C::G >= NBG ? (i % C::G) / (C::G / NBG) : i % NBG; };
    const uint32_t t_a = tmem_base + ((uint32_t)(q4 * 32) << 16) + C::ACOL;
    const uint32_t ldx2 = (uint32_t)p.ldx * 2u;
    uint32_t sc0 = 0, gc = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      if (lane == 0 && q4 == 0 && bg == 0) HTS(7800 + 2 * gc);
      Unit U;
      get_unit(p, u, cpo, mtiles, U, s_units);
      if (lane == 0 && q4 == 0 && bg == 0) HTS(7801 + 2 * gc);
      const int nq = U.q1 - U.q0;
      for (int c = U.q0 / U.npres; nq > 0 && c * U.npres < U.q1; ++c) {
        const int qs = max(U.q0, c * U.npres), qe = min(U.q1, (c + 1) * U.npres);
        const int hb = gc % C::NHB;
        const uint32_t hph = (gc / C::NHB) & 1;
        if (lane == 0 && q4 == 0 && bg == 0) HTS(6000 + 4 * gc);
        mbar_wait(smem_u32(hmeta + hb), hph);
        if (lane == 0 && q4 == 0 && bg == 0) HTS(6001 + 4 * gc);
        if (gc == 0) {
          // the CTA's first halo: nothing to overlap it with, so the 8 builder
          // warps copy it together with the 2 loader warps (10 warps instead of 2)
          if (p.done_in) mbar_wait(smem_u32(hdep), 0);  // its producer tiles are done
          const int ku = (u - (int)blockIdx.x) / (int)gridDim.x;
          const int H = ku < kUnitCache ? s_uhn[ku] : __ldg(p.halo_n + U.mt);
          const int pt = LOADERS + tid, pc = pt & 7;
          const int* hr = reinterpret_cast<const int*>(smem + hb * HBUF + ROWS_OFF);
          const char* xb = reinterpret_cast<const char*>(p.x) + c * 128 + pc * 16;
          const uint32_t hs = smem_u32(smem + hb * HBUF);
          if (!pair || pc < 4) {
#pragma unroll 4
            for (int i = pt >> 3; i < H; i += (LOADERS + R::NBT) / 8)
              cp_async16(hs + i * 128 + ((pc ^ (i & 7)) << 4), xb + (long long)hr[i] * ldx2, 16);
          }
          cp_async_mbar_arrive_noinc(smem_u32(hfull + hb));
        } else {
          // builders add no copies to later halos: one counted arrival per warp
          // (measured ~4 us per frame faster than 512 single-thread arrivals)
          __syncwarp();
          if (lane == 0) mbar_arrive_cnt(smem_u32(hfull + hb), 32u);
        }
        if (lane == 0 && q4 == 0 && bg < 2) HTS(257 + 4 * gc + 2 * bg);
        mbar_wait(smem_u32(hfull + hb), hph);
        if (lane == 0 && q4 == 0 && bg < 2) HTS(256 + 4 * gc + 2 * bg);
        const uint8_t* hbuf = smem + hb * HBUF;
        const int16_t* ln = reinterpret_cast<const int16_t*>(hbuf + HALO_BYTES) + r * KOFF;
        // one chunk (q = unit chunk index, j = its offset); returns 1 when the
        // group's partner chunk of the stage was built with it
        auto chunk = [&](const int q, const int j) -> int {
          const int i = q - U.q0;
          const uint32_t st = sc0 + i / C::G;
          const int stage = (int)(st % C::NS);
          uint32_t v[32];
          if (pair) {
            // columns 0-31: offset 2j's neighbour (32 channels), 32-63: offset 2j+1's
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int jj = 2 * j + h;
              const int li = jj < KOFF ? ln[jj] : -1;
              if (li >= 0) {
                const uint8_t* src = hbuf + li * 128;
                const int sw = li & 7;
#pragma unroll
                for (int pc = 0; pc < 4; ++pc) {
                  const uint4 t4 = *reinterpret_cast<const uint4*>(src + ((pc ^ sw) << 4));
                  v[16 * h + 4 * pc] = t4.x; v[16 * h + 4 * pc + 1] = t4.y;
                  v[16 * h + 4 * pc + 2] = t4.z; v[16 * h + 4 * pc + 3] = t4.w;
                }
              } else {
                const int g = li == -2 ? __ldg(p.nbr + ((long long)U.mt * BM + r) * KOFF + jj) : -1;
                const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(p.x) +
                                                                  (long long)(g >= 0 ? g : 0) * ldx2);
#pragma unroll
                for (int pc = 0; pc < 4; ++pc) {
                  const uint4 t4 = g >= 0 ? __ldg(src + pc) : make_uint4(0u, 0u, 0u, 0u);
                  v[16 * h + 4 * pc] = t4.x; v[16 * h + 4 * pc + 1] = t4.y;
                  v[16 * h + 4 * pc + 2] = t4.z; v[16 * h + 4 * pc + 3] = t4.w;
                }
              }
            }
          } else {
            if (lane == 0 && q4 == 0 && bg < 2 && st < 300) HTS(5400 + 2 * st + bg);
            auto load = [&](int jj, uint32_t (&vv)[32]) {
              const int li = ABL(17) ? -1 : ln[jj];
              if (li >= 0) {
                const uint8_t* src = hbuf + li * 128;
                const int sw = li & 7;
#pragma unroll
                for (int pc = 0; pc < 8; ++pc) {
                  const uint4 t4 = *reinterpret_cast<const uint4*>(src + ((pc ^ sw) << 4));
                  vv[4 * pc] = t4.x; vv[4 * pc + 1] = t4.y; vv[4 * pc + 2] = t4.z; vv[4 * pc + 3] = t4.w;
                }
              } else if (li == -1) {
#pragma unroll
                for (int k = 0; k < 32; ++k) vv[k] = 0u;
              } else {
                const int g = __ldg(p.nbr + ((long long)U.mt * BM + r) * KOFF + jj);
                const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(p.x) +
                                                                  (long long)g * ldx2 + c * 128);
#pragma unroll
                for (int pc = 0; pc < 8; ++pc) {
                  const uint4 t4 = __ldg(src + pc);
                  vv[4 * pc] = t4.x; vv[4 * pc + 1] = t4.y; vv[4 * pc + 2] = t4.z; vv[4 * pc + 3] = t4.w;
                }
              }
            };
            const int slot = i % C::G;
            // the group's second chunk of this stage, when it is in this range
            constexpr bool kTwo = C::G / NBG >= 2;  // a group owns two slots of a stage
            const bool two = kTwo && q + 1 < qe && slot + 1 < C::G && grp(i + 1) == bg;
            uint32_t w[kTwo ? 32 : 1];
            const int j2 = two ? next_offset(U.mask, j) : j;
            load(j, v);
            if constexpr (kTwo)
              if (two) load(j2, w);
            if (lane == 0 && q4 == 0 && bg < 2 && st < 400) HTS(2000 + 2 * st + bg);
            mbar_wait(smem_u32(empty + stage), ((st / C::NS) & 1) ^ 1);
            if (lane == 0 && q4 == 0 && bg < 2 && st < 400) HTS(2800 + 2 * st + bg);
            tc_fence_after();
            if (!ABL(18)) {
              tmem_st32(t_a + (stage * C::G + slot) * 32, v);
              if constexpr (kTwo)
                if (two) tmem_st32(t_a + (stage * C::G + slot + 1) * 32, w);
              tmem_st_wait();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cnt(smem_u32(full + stage), two ? 2u : 1u);
            if (lane == 0 && q4 == 0 && bg < 2 && st < 1400) HTS(1024 + 2 * st + bg);
            return two ? 1 : 0;  // the partner chunk is done too
          }
          if (lane == 0 && q4 == 0 && bg < 2 && st < 400) HTS(2000 + 2 * st + bg);
          mbar_wait(smem_u32(empty + stage), ((st / C::NS) & 1) ^ 1);
          if (lane == 0 && q4 == 0 && bg < 2 && st < 400) HTS(2800 + 2 * st + bg);
          tc_fence_after();
          if (!ABL(18)) {
            tmem_st32(t_a + (stage * C::G + i % C::G) * 32, v);
            tmem_st_wait();
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(full + stage));
          if (lane == 0 && q4 == 0 && bg < 2 && st < 1400) HTS(1024 + 2 * st + bg);
                  return 0;
        };
        constexpr bool kTwoG = C::G / NBG >= 2;
        if constexpr (!kTwoG) {
          // chunk i goes to group i % NBG: this group's chunks of channel
          // chunk c are every NBG-th present offset, picked out of the tile
          // mask once here (walking all chunks and skipping the other groups'
          // was a dependent bit-scan chain per chunk on every builder warp)
          const int r0 = (bg - (qs - U.q0)) & (NBG - 1);
          uint32_t rem = U.mask, own = 0;
          for (int k = qs - c * U.npres + r0; k > 0; --k) rem &= rem - 1u;  // ranks before this group's first
          for (int q = qs + r0; q < qe && rem; q += NBG) {
            own |= rem & (0u - rem);
#pragma unroll
            for (int k = 0; k < NBG; ++k) rem &= rem - 1u;
          }
          for (int q = qs + r0; own; q += NBG, own &= own - 1u) chunk(q, __ffs(own) - 1);
        } else {
          int j = first_offset(U.mask, qs - c * U.npres);
          for (int q = qs; q < qe; ++q, j = next_offset(U.mask, j)) {
            if (grp(q - U.q0) != bg) continue;
            if (chunk(q, j)) {
              ++q;  // the partner chunk is done; the loop increment moves past it
              j = next_offset(U.mask, j);
            }
          }
        }
        if (lane == 0 && q4 == 0 && bg == 0) HTS(6002 + 4 * gc);
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(hempty + hb));
        if (lane == 0 && q4 == 0 && bg == 0) HTS(6003 + 4 * gc);
        ++gc;
      }
      const uint32_t nst = (nq + C::G - 1) / C::G;
      if (C::G > 1 && nq % C::G) {
        // the unit's last stage is short: its missing slots (owned by group
        // grp(slot)) still arrive
        const uint32_t st = sc0 + nst - 1;
        bool waited = false;
        for (int sl = nq % C::G; sl < C::G; ++sl) {
          if (grp((int)(nst - 1) * C::G + sl) != bg) continue;
          if (!waited) {
            mbar_wait(smem_u32(empty + st % C::NS), ((st / C::NS) & 1) ^ 1);
            waited = true;
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(full + st % C::NS));
        }
      }
      sc0 += nst;
    }
  } else if (warp < W_B) {
    // ===================== halo loaders =====================
    // halo sizes, local tables and row lists come from the table build: with
    // settled tables (two or more launches old) they are read, and the first
    // halo's table + row list copied, before the wait; the halo ROWS are the
    // previous launch's output and always wait
    const bool early = p.settled != 0;
    const bool flow = p.done_in != nullptr;  // dataflow: no grid-wide wait (flow implies settled)
    if (!early) {
      pdl_wait();
      if (tid == W_LOAD * 32) pdl_trigger();
    }
    const int tl = tid - W_LOAD * 32;
    // the unit cache's halo sizes; the builders read them only after the first
    // hmeta barrier, which loader thread 0 arrives on after this named barrier
    for (int k = tl; k < kUnitCache; k += LOADERS) {
      const int u = blockIdx.x + k * gridDim.x;
      s_uhn[k] = u < nunits ? __ldg(p.halo_n + s_units[k].mt) : 0;
    }
    named_bar(2, LOADERS);
    const int pc = tl & 7;
    const uint32_t ldx2 = (uint32_t)p.ldx * 2u;
    // the tile's local table and its halo row list, one bulk copy each
    auto issue_meta = [&](const Unit& U, int hb, int H) {
      const uint32_t rb = (uint32_t)((H * 4 + 15) & ~15);
      const uint32_t mb = smem_u32(hmeta + hb);
      uint8_t* hbuf = smem + hb * HBUF;
      mbar_arrive_expect_tx(mb, LNBR_BYTES + rb);
      bulk_g2s(smem_u32(hbuf + HALO_BYTES), p.lnbr + (long long)U.mt * BM * KOFF, LNBR_BYTES, mb);
      if (rb) bulk_g2s(smem_u32(hbuf + ROWS_OFF), p.halo_rows + (long long)U.mt * HMAX, rb, mb);
    };
    bool pre = false;  // the first halo's meta copy is already in flight
    if (early) {
      if ((int)blockIdx.x < nunits) {
        Unit U;
        get_unit(p, blockIdx.x, cpo, mtiles, U, s_units);
        if (U.q1 > U.q0) {
          pre = true;
          if (tl == 0) issue_meta(U, 0, s_uhn[0]);  // buffer 0 is free: nothing has used it yet
        }
      }
      if (!flow) {
        pdl_wait();
        if (tid == W_LOAD * 32) pdl_trigger();
      }
    }
#ifdef FPVS_PROFILE
    if (p.dbg && tid == W_LOAD * 32 && blockIdx.x < 160) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      g_hcta[p.hslot][2][blockIdx.x] = t_;
    }
#endif
    uint32_t gc = 0;
    int dep_mt = -1;  // dataflow: the tile whose producer tiles were last waited for
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      get_unit(p, u, cpo, mtiles, U, s_units);
      for (int c = U.q0 / U.npres; U.q1 > U.q0 && c * U.npres < U.q1; ++c) {
        const int hb = gc % C::NHB;
        const uint32_t hph = (gc / C::NHB) & 1;
        mbar_wait_sleep(smem_u32(hempty + hb), hph ^ 1, 64);
        if (tl == 0) HTS(16 + 3 * gc);
        uint8_t* hbuf = smem + hb * HBUF;
        const int ku = (u - (int)blockIdx.x) / (int)gridDim.x;
        const int H = ku < kUnitCache ? s_uhn[ku] : __ldg(p.halo_n + U.mt);
        if (pre) {
          pre = false;  // gc == 0: issued before the wait
        } else if (tl == 0) {
          issue_meta(U, hb, H);
        }
        mbar_wait(smem_u32(hmeta + hb), hph);
        if (tl == 0) HTS(17 + 3 * gc);
        const int* hr = reinterpret_cast<const int*>(hbuf + ROWS_OFF);
        if (flow && U.mt != dep_mt) {
          // the producer tiles holding this tile's halo rows (the sorted row
          // list's first and last); a capped or windowless halo (rows read
          // straight from global memory) waits for every producer tile
          int lo = 0, hi = mtiles - 1;
          if (H > 0 && H < HMAX) {
            lo = hr[0] / BM;
            hi = hr[H - 1] / BM;
          }
          for (int t = lo + tl; t <= hi; t += LOADERS) {
            long long spins = 0;
            while (ld_acquire_gpu(p.done_in + t) < 4) {
              __nanosleep(32);
              if (++spins > (1LL << 26)) __trap();  // a producer that never finishes: fail, do not hang
            }
          }
          named_bar(2, LOADERS);
          if (gc == 0 && tl == 0) {
            mbar_arrive(smem_u32(hdep));  // the builders may copy the first halo
            pdl_trigger();                // dependents launch once every CTA got here
          }
          dep_mt = U.mt;
        }
        const char* xb = reinterpret_cast<const char*>(p.x) + c * 128 + pc * 16;
        const uint32_t hs = smem_u32(hbuf);
        // the first halo is shared with the builders: loader thread tl takes rows
        // tl/8 + 40k of the 320-thread split; later halos rows tl/8 + 8k
        const int rstep = gc == 0 ? (LOADERS + R::NBT) / 8 : LOADERS / 8;
        if ((!pair || pc < 4) && !ABL(19)) {  // 32-channel rows: four 16-byte pieces
#pragma unroll 4
          for (int i = tl >> 3; i < H; i += rstep) {
            const int g = hr[i];
            cp_async16(hs + i * 128 + ((pc ^ (i & 7)) << 4), xb + (long long)g * ldx2, 16);
          }
        }
        cp_async_mbar_arrive_noinc(smem_u32(hfull + hb));
        if (tl == 0) HTS(18 + 3 * gc);
        ++gc;
      }
    }
  } else if (warp == W_B) {
    // ===================== weight loader =====================
    // the packed weights may be the previous launch's output (lazy / per-step
    // re-pack); a dataflow consumer's weights are packed before the frame
    if (!p.done_in) pdl_wait();
    if (lane == 0) {
      uint32_t st = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        Unit U;
        get_unit(p, u, cpo, mtiles, U, s_units);
        const int nq = U.q1 - U.q0;
        const uint8_t* wblk = p.wpk + (size_t)U.nb * p.nchunks * C::B_SUB;
        ChunkWalk w;
        w.start(U);
        for (int i = 0; i < nq; i += C::G, ++st) {
          const int stage = (int)(st % C::NS);
          const int nv = min(C::G, nq - i);
          mbar_wait(smem_u32(empty + stage), ((st / C::NS) & 1) ^ 1);
          if (st < 1000) HTS(5000 + st);
          const uint32_t fb = smem_u32(full + stage);
          if (ABL(16) && st >= (uint32_t)C::NS) {
            mbar_arrive(fb);
            continue;
          }
          mbar_arrive_expect_tx(fb, nv * C::B_SUB);
          for (int g = 0; g < nv; ++g, w.next())
            bulk_g2s(smem_u32(sB + stage * C::STAGE_B + g * C::B_SUB), wblk + (size_t)(w.j * cpo + w.c) * C::B_SUB,
                     C::B_SUB, fb);
        }
      }
    }
  } else if (warp == W_MMA) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16<BN>();
      const uint32_t a_base = tmem_base + C::ACOL;
      const uint64_t b_desc0 = sw128_desc(smem_u32(sB));
      uint32_t st = 0;
      int it = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
        HTS(7600 + 2 * it);
        Unit U;
        get_unit(p, u, cpo, mtiles, U, s_units);
        const int nq = U.q1 - U.q0;
        const int acc = it % C::NACC;
        HTS(7601 + 2 * it);
        mbar_wait(smem_u32(tempty + acc), ((it / C::NACC) & 1) ^ 1);
        HTS(7000 + 2 * it);
        tc_fence_after();
        const uint32_t dtm = tmem_base + acc * BN;
        // The issue loop is on the critical path of every MMA (tcgen05.mma
        // issue is effectively synchronous at N <= 128): any dependent scalar
        // work between two MMAs adds straight to their cost (measured
        // tools/micro_commit2.cu: 47 -> 89 cycles per N = 64 MMA with one
        // division in the loop).  So a stage's A / B addresses are affine in
        // the stage index (bases hoisted out of all loops) and a full stage is
        // one fully unrolled run of G x 4 MMAs with immediate offsets; only the
        // unit's first MMA clears the accumulator.
        for (int i = 0; i < nq; i += C::G, ++st) {
          const int stage = (int)(st % C::NS);
          const int nv = min(C::G, nq - i);
          if (st < 400) HTS(3600 + st);
          mbar_wait(smem_u32(full + stage), (st / C::NS) & 1);
          if (st < 450) HTS(4096 + 2 * st);
          tc_fence_after();
          const uint32_t ta0 = a_base + (uint32_t)stage * (C::G * 32);
          const uint64_t bd0 = b_desc0 + (uint64_t)((uint32_t)stage * (C::STAGE_B >> 4));
          if (!ABL(20)) {
            if (nv == C::G) {
#pragma unroll
              for (int g = 0; g < C::G; ++g)
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                  umma_bf16_ts(dtm, ta0 + g * 32 + 8 * k, bd0 + (uint64_t)(g * (C::B_SUB >> 4) + 2 * k), idesc,
                               (g == 0 && k == 0) ? (i != 0 ? 1u : 0u) : 1u);
            } else {
              for (int g = 0; g < nv; ++g)
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                  umma_bf16_ts(dtm, ta0 + g * 32 + 8 * k, bd0 + (uint64_t)(g * (C::B_SUB >> 4) + 2 * k), idesc,
                               (i == 0 && g == 0 && k == 0) ? 0u : 1u);
            }
          }
          umma_commit(smem_u32(empty + stage));
          if (st < 450) HTS(4097 + 2 * st);
        }
        umma_commit(smem_u32(tfull + acc));
        HTS(7001 + 2 * it);
      }
    }
  } else {
    // ===================== epilogue (4 warps) =====================
    // y, partials and counters may be in use by the previous launch (a
    // dataflow consumer writes a buffer its producer never touches)
    if (!p.done_in) pdl_wait();
    const int q4 = warp & 3, r = q4 * 32 + lane;
    const uint32_t tlane = (uint32_t)(q4 * 32) << 16;
    const bool fuse_head = C::HEAD && p.head;
    constexpr int EC = NBG == 4 || MINB == 2 ? 16 : 32;  // 16 where registers are short (768 threads, or 2 CTAs per SM)
    uint32_t head_phase = 0;
    if (fuse_head && warp == W_EPI && lane == 0) {
      // the packed head weights (one 64 x 64 bf16 SW128 chunk), once per CTA
      mbar_arrive_expect_tx(smem_u32(hwbar), 64 * 128);
      bulk_g2s(smem_u32(smem + C::HW_OFF), p.head_wpk, 64 * 128, smem_u32(hwbar));
    }
    int it = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
      Unit U;
      get_unit(p, u, cpo, mtiles, U, s_units);
      const int acc = it % C::NACC;
      mbar_wait_sleep(smem_u32(tfull + acc), (it / C::NACC) & 1, 128);
      if (q4 == 0 && lane == 0) HTS(7200 + 2 * it);
      tc_fence_after();
      const long long row = (long long)U.mt * BM + r;
      const bool valid = row < n;
      const int col0 = U.nb * BN;
      if (U.ns == 1) {
        uint32_t ha[32];  // fused head: this row's bf16 activations as the head's A operand
        // EC columns per TMEM load (16 in the 768-thread variant: 80 registers)
#pragma unroll(BN == 64 ? 64 / EC : 1)
        for (int cb = 0; cb < BN; cb += EC) {
          float v[EC];
          tmem_ldn<EC>(tmem_base + tlane + acc * BN + cb, v);
#pragma unroll
          for (int i = 0; i < EC; ++i) {
            const float z = v[i] + s_bias[col0 + cb + i];
            v[i] = p.act == FPVS_ACT_RELU ? fmaxf(z, 0.f) : z;
          }
          if (fuse_head) {
            if constexpr (BN == 64) {
#pragma unroll
              for (int i = 0; i < EC / 2; ++i) ha[cb / 2 + i] = valid ? pack_bf16x2(v[2 * i], v[2 * i + 1]) : 0u;
            }
            continue;
          }
          if (!valid) continue;
          uint4* dst = reinterpret_cast<uint4*>(p.y + row * p.ldy + p.col_off + col0 + cb);
#pragma unroll
          for (int i = 0; i < EC / 8; ++i)
            dst[i] = make_uint4(pack_bf16x2(v[8 * i + 0], v[8 * i + 1]), pack_bf16x2(v[8 * i + 2], v[8 * i + 3]),
                                pack_bf16x2(v[8 * i + 4], v[8 * i + 5]), pack_bf16x2(v[8 * i + 6], v[8 * i + 7]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(tempty + acc));
        if (p.done_out && !fuse_head) {
          // dataflow producer: each epilogue warp publishes its 32 rows with a
          // release add once they are stored (__syncwarp orders the lanes'
          // stores before lane 0's cumulative release); 4 = the tile is done
          // (with the fused head: once its row masks are stored, below)
          __syncwarp();
          if (lane == 0) red_add_release_gpu(p.done_out + U.mt, 1);
        }
        if constexpr (C::HEAD) {
          if (fuse_head) {
            // head = 1x1x1 conv of the bf16 activations (exactly what the
            // stand-alone head reads back from HBM): A rows into tensor memory,
            // 4 TS MMAs (K = 64) by one epilogue thread, then the threshold
            // bit-pack of head_tc's fast path ([z >= logit(tau)], one RED.OR
            // per (ly, lz) voxel row of the cell)
            tmem_st32(tmem_base + tlane + C::HEAD_A, ha);
            tmem_st_wait();
            tc_fence_before();
            named_bar(3, 128);
            if (warp == W_EPI && lane == 0 && !ABL(22)) {
              if (it == 0) mbar_wait(smem_u32(hwbar), 0);
              tc_fence_after();
              const uint64_t hb = sw128_desc(smem_u32(smem + C::HW_OFF));
              const uint32_t hidesc = idesc_bf16<64>();
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                umma_bf16_ts(tmem_base + C::HEAD_D, tmem_base + C::HEAD_A + 8 * k, hb + 2 * k, hidesc, k ? 1u : 0u);
              umma_commit(smem_u32(hdbar));
            }
            if (!ABL(22)) mbar_wait(smem_u32(hdbar), head_phase);
            head_phase ^= 1;
            tc_fence_after();
            // the row's 64 head outputs as one word (bit k = channel k =
            // lx + 4 ly + 16 lz); rowbits_grid_kernel writes the froxel grid
            unsigned long long rb = 0;
#pragma unroll
            for (int cb = 0; cb < 64; cb += 8) {
              float v[8];
              tmem_ld8(tmem_base + tlane + C::HEAD_D + cb, v);
#pragma unroll
              for (int i = 0; i < 8; ++i)
                rb |= (unsigned long long)(v[i] + s_bias[512 + cb + i] >= p.zt ? 1u : 0u) << (cb + i);
            }
            if (valid && !ABL(21)) p.row_bits[row] = rb;
            if (p.done_out) {  // the grid writer's dataflow: this warp's row masks are stored
              __syncwarp();
              if (lane == 0) red_add_release_gpu(p.done_out + U.mt, 1);
            }
            tc_fence_before();  // the next tile's head A store / MMA come after these reads
            named_bar(3, 128);
          }
        }
      } else {
        // split K: fp32 partial per split, column-major [col][128 rows] so a
        // warp's stores and loads are 128-byte coalesced; the last CTA of the
        // tile to arrive sums the splits in a fixed order (deterministic),
        // taking its own split from TMEM
        const long long slot = U.slot;
        const bool has = U.q1 > U.q0;
        float* mine = p.part + (slot * p.smax + U.s) * BM * BN + r;
#pragma unroll 1
        for (int cb = 0; cb < BN; cb += EC) {
          float v[EC];
          tmem_ldn<EC>(tmem_base + tlane + acc * BN + cb, v);
#pragma unroll
          for (int i = 0; i < EC; ++i) __stcg(mine + (cb + i) * BM, has ? v[i] : 0.f);
        }
        named_bar(1, 128);
        if (q4 == 0 && lane == 0) HTS(7400 + 4 * it);
        if (warp == W_EPI && lane == 0) {
          __threadfence();  // release the CTA's partial (ordered after the barrier) before the count
          const int last = atomicAdd(p.counters + slot, 1) == U.ns - 1;
          if (last) __threadfence();  // acquire the other splits' partials
          *s_last = last;
        }
        named_bar(1, 128);
        if (q4 == 0 && lane == 0) HTS(7402 + 4 * it);
        if (*s_last) {
          const float* base = p.part + slot * p.smax * BM * BN + r;
#pragma unroll 1
          for (int cb = 0; cb < BN; cb += EC) {
            float own[EC], v[EC];
            tmem_ldn<EC>(tmem_base + tlane + acc * BN + cb, own);
#pragma unroll
            for (int i = 0; i < EC; ++i) v[i] = 0.f;
            for (int ss = 0; ss < U.ns; ++ss) {
              const float* src = base + (long long)ss * BM * BN + cb * BM;
              if (ss == U.s) {
#pragma unroll
                for (int i = 0; i < EC; ++i) v[i] += has ? own[i] : 0.f;
              } else {
#pragma unroll
                for (int i = 0; i < EC; ++i) v[i] += __ldcg(src + i * BM);
              }
            }
            if (!valid) continue;
#pragma unroll
            for (int i = 0; i < EC; ++i) {
              const float z = v[i] + s_bias[col0 + cb + i];
              v[i] = p.act == FPVS_ACT_RELU ? fmaxf(z, 0.f) : z;
            }
            uint4* dst = reinterpret_cast<uint4*>(p.y + row * p.ldy + p.col_off + col0 + cb);
#pragma unroll
            for (int i = 0; i < EC / 8; ++i)
              dst[i] = make_uint4(pack_bf16x2(v[8 * i + 0], v[8 * i + 1]), pack_bf16x2(v[8 * i + 2], v[8 * i + 3]),
                                  pack_bf16x2(v[8 * i + 4], v[8 * i + 5]), pack_bf16x2(v[8 * i + 6], v[8 * i + 7]));
          }
          if (warp == W_EPI && lane == 0) p.counters[slot] = 0;
          if (q4 == 0 && lane == 0) HTS(7403 + 4 * it);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(tempty + acc));
      }
    }
  }

  if (tid == 0) HTS(2);
  tc_fence_before();
  __syncthreads();
  if (tid == 0) HTS(3);
#ifdef FPVS_PROFILE
  if (p.dbg && tid == 0 && blockIdx.x < 160) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    g_hcta[p.hslot][1][blockIdx.x] = t_;
    g_hclk[1][blockIdx.x] = clock64();
  }
#endif
  if (warp == W_MMA) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(C::TMEM_COLS)
                 : "memory");
  }
}

template <int BN, bool PAIR, int NBG, int MINB = 1>
int launch(const Params& p, cudaStream_t s) {
  using C = Cfg<BN, NBG, MINB>;
  {
    const cudaError_t e = set_smem_once<spconv_halo_kernel<BN, PAIR, NBG, MINB>>(C::SMEM);
    if (e != cudaSuccess) return set_error(FPVS_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  const long long units = (long long)((p.cap + BM - 1) / BM) * p.nblk * p.smax;
  if (p.cout > C::BIAS_N) return set_error(FPVS_EINVAL, "spconv_halo: Cout %d > %d", p.cout, C::BIAS_N);
  const long long slots = (long long)kNumSMs * MINB;
  const int grid = (int)(units < slots ? (units < 1 ? 1 : units) : slots);
  cudaError_t e = launch_kernel(spconv_halo_kernel<BN, PAIR, NBG, MINB>, dim3(grid), dim3(Roles<NBG>::THREADS), C::SMEM,
                                s, p);
  if (e != cudaSuccess) return set_error(FPVS_ECUDA, "spconv_halo: %s", cudaGetErrorString(e));
  FPVS_CHECK_LAUNCH("spconv_halo");
  return FPVS_OK;
}

// 4 builder groups at N = 64 (level 0: the A build paces the MMA issue) and
// at N = 128 with two-chunk stages (levels 1 / 2: 8 MMAs per barrier round
// instead of 4); measured in-frame with tools/halo_variant.py
#ifndef FPVS_HALO_2CTA
#define FPVS_HALO_2CTA 0
#endif
#ifndef FPVS_HALO_NBG4_MASK
#define FPVS_HALO_NBG4_MASK 1  // bit 0: BN 64, bit 1: BN 128 (tools/build_variant.py A/B builds)
#endif
inline bool default_nbg4(int bn) {
  return (bn == 64 && (FPVS_HALO_NBG4_MASK & 1)) || (bn == 128 && (FPVS_HALO_NBG4_MASK & 2));
}

inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

}  // namespace halo
}  // namespace fpvs

using namespace fpvs;

#ifdef FPVS_PROFILE
// profiling builds only (not part of the ABI): CTA timestamps, SM ids, clocks
extern "C" int fpvs_debug_halo_timestamps(unsigned long long* host, int n) {
  if (n > 2 * 8192) n = 2 * 8192;
  return cudaMemcpyFromSymbol(host, halo::g_hts, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 3;
}
extern "C" int fpvs_debug_halo_cta_times(unsigned long long* host) {  // [32][3][160]
  return cudaMemcpyFromSymbol(host, halo::g_hcta, sizeof(halo::g_hcta)) == cudaSuccess ? 0 : 3;
}
// resets the launch counter (returns the launches counted since the last reset) and clears the spans
extern "C" int fpvs_debug_halo_reset_slot(void) {
  const int n = halo::g_hslot;
  halo::g_hslot = 0;
  static const unsigned long long zeros[halo::kSpanSlots * 3 * 160] = {};
  cudaMemcpyToSymbol(halo::g_hcta, zeros, sizeof(zeros));
  return n;
}
extern "C" int fpvs_debug_halo_slot_count(void) { return halo::g_hslot; }
extern "C" int fpvs_debug_halo_clk(long long* host) {
  return cudaMemcpyFromSymbol(host, halo::g_hclk, sizeof(long long) * 320) == cudaSuccess ? 0 : 3;
}
extern "C" int fpvs_debug_halo_smid(unsigned* host) {
  return cudaMemcpyFromSymbol(host, halo::g_hsm, sizeof(unsigned) * 160) == cudaSuccess ? 0 : 3;
}
#endif

extern "C" size_t fpvs_kmap_halo_size(int cap) {
  if (cap < 1) return 0;
  const size_t tiles = (cap + tc::BM - 1) / tc::BM;
  return halo::align256(tiles * halo::HMAX * 4) + halo::align256(tiles * 4) +
         halo::align256(tiles * tc::BM * halo::KOFF * 2);
}

extern "C" int fpvs_kmap_halo_multi(const fpvs_halo_job* jobs, int njobs, void* stream) {
  FPVS_CHECK_ARG(jobs && njobs >= 1 && njobs <= halo::kMaxHaloJobs, "1..4 halo jobs");
  halo::HaloJobs J{};
  J.count = njobs;
  long long tiles = 0;
  for (int i = 0; i < njobs; ++i) {
    const fpvs_halo_job& q = jobs[i];
    FPVS_CHECK_ARG(q.nbr && q.n_dev && q.halo_rows && q.halo_n && q.lnbr, "null pointer in halo job %d", i);
    FPVS_CHECK_ARG(q.cap >= 0, "negative capacity");
    J.j[i] = halo::HaloJob{q.nbr, q.n_dev, q.cap, q.halo_rows, q.halo_n, q.lnbr};
    tiles += (q.cap + tc::BM - 1) / tc::BM;
  }
  if (tiles == 0) return FPVS_OK;
  const int grid = (int)(tiles < 4 * kNumSMs ? tiles : 4 * kNumSMs);
  cudaError_t e = launch_kernel(halo::halo_build_kernel, dim3(grid), dim3(256), 0, as_stream(stream), J);
  if (e != cudaSuccess) return set_error(FPVS_ECUDA, "fpvs_kmap_halo: %s", cudaGetErrorString(e));
  FPVS_CHECK_LAUNCH("fpvs_kmap_halo");
  return FPVS_OK;
}

extern "C" int fpvs_kmap_halo(const int32_t* nbr, const int32_t* n_dev, int cap, int32_t* halo_rows,
                              int32_t* halo_n, int16_t* lnbr, void* stream) {
  fpvs_halo_job j{nbr, n_dev, cap, halo_rows, halo_n, lnbr};
  return fpvs_kmap_halo_multi(&j, 1, stream);
}

extern "C" size_t fpvs_spconv_halo_workspace_size(int cap, int cout, int bn, int split) {
  if (cap < 1 || (bn != 32 && bn != 64 && bn != 128 && bn != 256) || split == 0) return 0;
  if (cout % bn) return 0;
  const size_t tiles = (cap + tc::BM - 1) / tc::BM, nblk = cout / bn;
  // split < 0: only the last partial wave (< one grid of items) is split
  const size_t items = split < 0 ? (size_t)kNumSMs : tiles * nblk;
  const size_t sm = split < 0 ? (size_t)-split : (size_t)split;
  size_t b = halo::align256(items * 4);
  if (sm > 1) b += items * sm * tc::BM * bn * 4;
  return b;
}

struct HeadArgs {
  const void* wpk;
  const float* bias;
  float tau;
  unsigned long long* row_bits;
};

static int halo_conv(const void* x, int ldx, int x_rows, const int32_t* nbr, const int16_t* lnbr,
                     const int32_t* halo_rows, const int32_t* halo_n, const uint32_t* tile_masks, const int32_t* n_dev,
                     int cap, const void* w_packed, int bn, int split, const float* bias, int cin, int cout, int act,
                     void* y, int ldy, int col_off, void* ws, size_t ws_bytes, void* stream, const HeadArgs* head,
                     int32_t* done_out = nullptr, const int32_t* done_in = nullptr) {
  FPVS_CHECK_ARG(x && nbr && lnbr && halo_rows && halo_n && tile_masks && n_dev && w_packed && y,
                 "null pointer");
  const int settled = (act & FPVS_TABLES_SETTLED) != 0;
  act &= ~FPVS_TABLES_SETTLED;
  if (bn == 0) bn = cout % 256 == 0 ? 256 : cout % 128 == 0 ? 128 : cout % 64 == 0 ? 64 : 32;
  if (split == 0) split = 1;
  FPVS_CHECK_ARG(bn == 32 || bn == 64 || bn == 128 || bn == 256, "halo conv tile width must be 32, 64, 128 or 256");
  FPVS_CHECK_ARG((cin % 64 == 0 && cin >= 64) || cin == 32, "halo conv needs Cin %% 64 == 0 or Cin = 32, got %d",
                 cin);
  FPVS_CHECK_ARG(cout % bn == 0 && cout <= 1024, "halo conv needs Cout %% %d == 0, got %d", bn, cout);
  FPVS_CHECK_ARG(ldx % 8 == 0 && ldx >= cin, "bad input leading dimension");
  FPVS_CHECK_ARG((long long)x_rows * ldx * 2 < (1LL << 31), "feature buffer too large for 32-bit row offsets");
  FPVS_CHECK_ARG(ldy % 8 == 0 && col_off % 8 == 0 && ldy >= col_off + cout, "bad output leading dimension");
  FPVS_CHECK_ARG(act == FPVS_ACT_NONE || act == FPVS_ACT_RELU, "halo conv epilogue supports none/relu");
  FPVS_CHECK_ARG(split != 0 && (split < 0 ? -split : split) <= (27 * cin + 63) / 64,
                 "|split| must lie in [1, ceil(27 * Cin / 64)]");
  const size_t need = fpvs_spconv_halo_workspace_size(cap, cout, bn, split);
  FPVS_CHECK_ARG(ws && ws_bytes >= need, "workspace too small: need %zu bytes", need);
  if (cap <= 0) return FPVS_OK;
  halo::Params p{};
  p.x = (const __nv_bfloat16*)x;
  p.ldx = ldx;
  p.nbr = nbr;
  p.lnbr = lnbr;
  p.halo_rows = halo_rows;
  p.halo_n = halo_n;
  p.tile_masks = tile_masks;
  p.n_dev = n_dev;
  p.cap = cap;
  p.wpk = (const uint8_t*)w_packed;
  p.nchunks = (27 * cin + 63) / 64;
  p.nblk = cout / bn;
  p.split = split;
  p.smax = split < 0 ? -split : split;
  p.bias = bias;
  p.cin = cin;
  p.cout = cout;
  p.act = act;
  p.y = (__nv_bfloat16*)y;
  p.ldy = ldy;
  p.col_off = col_off;
  const size_t tiles = (cap + tc::BM - 1) / tc::BM;
  const size_t items = split < 0 ? (size_t)kNumSMs : tiles * p.nblk;
  p.counters = (int*)ws;
  p.part = (float*)((uint8_t*)ws + halo::align256(items * 4));
  p.dbg = debug_knob("FPVS_HALO_DEBUG");
#ifdef FPVS_PROFILE
  p.hslot = halo::g_hslot++ % halo::kSpanSlots;
#endif
  p.abl = debug_knob("FPVS_HALO_ABL");
  p.settled = settled;
  if (done_out || done_in) {
    // dataflow needs settled tables (the unit decode precedes any wait), one
    // unit per tile for a producer, and every CTA's units in the unit cache
    FPVS_CHECK_ARG(settled || !done_in, "a dataflow consumer needs FPVS_TABLES_SETTLED");
    FPVS_CHECK_ARG(!done_out || split == 1, "a dataflow producer runs unsplit (split = 1)");
    FPVS_CHECK_ARG((tiles * p.nblk * (split < 0 ? -split : split) + halo::kNumSMsForCache - 1) /
                           halo::kNumSMsForCache <= halo::kUnitCache,
                   "dataflow: more units per CTA than the unit cache holds");
    FPVS_CHECK_ARG(!done_out || p.nblk == 1, "a dataflow producer writes whole rows per unit (Cout = bn)");
  }
  p.done_out = done_out;
  p.done_in = done_in;
  if (head) {
    FPVS_CHECK_ARG(bn == 64 && cout == 64 && split == 1 && cin % 64 == 0,
                   "fused head needs a Cout = 64 layer with 64-wide tiles, no K split and Cin %% 64 == 0");
    FPVS_CHECK_ARG(head->wpk && head->row_bits, "fused head: null pointer");
    p.head = 1;
    p.head_wpk = (const uint8_t*)head->wpk;
    p.head_bias = head->bias;
    // [sigmoid(z) >= tau] as [z >= logit(tau)] (head_tc's fast path)
    p.zt = head->tau <= 0.f ? -INFINITY : head->tau >= 1.f ? INFINITY
                                        : (float)log((double)head->tau / (1.0 - (double)head->tau));
    p.row_bits = head->row_bits;
  }
  const cudaStream_t st = as_stream(stream);
  if (cin == 32) {
    if (bn == 32) return halo::launch<32, true, 2>(p, st);
    if (bn == 64) return halo::launch<64, true, 2>(p, st);
    if (bn == 128) return halo::launch<128, true, 2>(p, st);
    return halo::launch<256, true, 2>(p, st);
  }
  // builder groups: 4 (16 builder warps) where the A build paces the MMA
  const int nbg_knob = debug_knob("FPVS_HALO_NBG");
  // (profiling knob: 2 / 4 for every width, 8 + m: bit 0/1/2 of m = 4 groups at BN 64/128/256)
  const int bnbit = bn == 64 ? 1 : bn == 128 ? 2 : 4;
  const bool nbg4 = nbg_knob >= 8 ? ((nbg_knob - 8) & bnbit) != 0 : nbg_knob ? nbg_knob == 4 : halo::default_nbg4(bn);
  if (bn == 32) return halo::launch<32, false, 2>(p, st);
  if (bn == 64) {
#if FPVS_HALO_2CTA
    // two CTAs per SM (Cfg MINB = 2) for the plain 64-wide layers: measured
    // (tools/build_variant.py) equal to one 4-group CTA per SM at Cin 64 and
    // 4 us slower at Cin 128, so the product build leaves it out
    if (!head && split == 1 && cout <= 128) return halo::launch<64, false, 2, 2>(p, st);
#endif
    return nbg4 ? halo::launch<64, false, 4>(p, st) : halo::launch<64, false, 2>(p, st);
  }
  if (bn == 128) return nbg4 ? halo::launch<128, false, 4>(p, st) : halo::launch<128, false, 2>(p, st);
  return nbg4 ? halo::launch<256, false, 4>(p, st) : halo::launch<256, false, 2>(p, st);
}

extern "C" int fpvs_spconv_halo(const void* x, int ldx, int x_rows, const int32_t* nbr, const int16_t* lnbr,
                                const int32_t* halo_rows, const int32_t* halo_n, const uint32_t* tile_masks,
                                const int32_t* n_dev, int cap, const void* w_packed, int bn, int split,
                                const float* bias, int cin, int cout, int act, void* y, int ldy, int col_off,
                                void* ws, size_t ws_bytes, void* stream) {
  return halo_conv(x, ldx, x_rows, nbr, lnbr, halo_rows, halo_n, tile_masks, n_dev, cap, w_packed, bn, split, bias, cin,
                   cout, act, y, ldy, col_off, ws, ws_bytes, stream, nullptr);
}

extern "C" int fpvs_spconv_halo_flow(const void* x, int ldx, int x_rows, const int32_t* nbr, const int16_t* lnbr,
                                     const int32_t* halo_rows, const int32_t* halo_n, const uint32_t* tile_masks,
                                     const int32_t* n_dev, int cap, const void* w_packed, int bn, int split,
                                     const float* bias, int cin, int cout, int act, void* y, int ldy, int col_off,
                                     void* ws, size_t ws_bytes, int32_t* tile_done_out, const int32_t* tile_done_in,
                                     void* stream) {
  return halo_conv(x, ldx, x_rows, nbr, lnbr, halo_rows, halo_n, tile_masks, n_dev, cap, w_packed, bn, split, bias, cin,
                   cout, act, y, ldy, col_off, ws, ws_bytes, stream, nullptr, tile_done_out, tile_done_in);
}

extern "C" int fpvs_spconv_halo_head_flow(const void* x, int ldx, int x_rows, const int32_t* nbr,
                                          const int16_t* lnbr, const int32_t* halo_rows, const int32_t* halo_n,
                                          const uint32_t* tile_masks, const int32_t* n_dev, int cap,
                                          const void* w_packed, const float* bias, int cin, void* ws, size_t ws_bytes,
                                          const void* head_w_packed, const float* head_bias, float tau,
                                          uint64_t* row_bits, int flags, const int32_t* done_in, int32_t* done_out,
                                          void* stream) {
  const HeadArgs h{head_w_packed, head_bias, tau, reinterpret_cast<unsigned long long*>(row_bits)};
  return halo_conv(x, ldx, x_rows, nbr, lnbr, halo_rows, halo_n, tile_masks, n_dev, cap, w_packed, 64, 1, bias, cin, 64,
                   FPVS_ACT_RELU | (flags & FPVS_TABLES_SETTLED), row_bits, 64, 0, ws, ws_bytes, stream, &h, done_out,
                   done_in);
}

extern "C" int fpvs_spconv_halo_head(const void* x, int ldx, int x_rows, const int32_t* nbr, const int16_t* lnbr,
                                     const int32_t* halo_rows, const int32_t* halo_n, const uint32_t* tile_masks,
                                     const int32_t* n_dev, int cap, const void* w_packed, const float* bias, int cin,
                                     void* ws, size_t ws_bytes, const void* head_w_packed, const float* head_bias,
                                     float tau, uint64_t* row_bits, int flags, const int32_t* done_in,
                                     void* stream) {
  const HeadArgs h{head_w_packed, head_bias, tau, reinterpret_cast<unsigned long long*>(row_bits)};
  // the conv's own output is consumed in the epilogue: y is never written
  return halo_conv(x, ldx, x_rows, nbr, lnbr, halo_rows, halo_n, tile_masks, n_dev, cap, w_packed, 64, 1, bias, cin, 64,
                   FPVS_ACT_RELU | (flags & FPVS_TABLES_SETTLED), row_bits, 64, 0, ws, ws_bytes, stream, &h, nullptr,
                   done_in);
}

namespace fpvs {
namespace halo {
// Per-row head bits -> the packed froxel grid (d = 4).  Block = (b, cell row
// cy, RZ = 4 cells of z: 1024 small blocks keep more gathers in flight than
// fewer, larger ones); its cells' 64-bit masks are staged in shared memory
// (level-0 index volume, coalesced along z, read before the PDL wait: it is
// the map kernels' output), then thread (z cell, 32-froxel word w) assembles
// the 16 words of its 8 cells' (ly, lz) voxel rows: every word of the grid is
// written exactly once, no atomics and no clear.
#ifndef FPVS_ROWBITS_RZ
#define FPVS_ROWBITS_RZ 4  // measured 16 / 8 / 4 / 2 / 1: 313.3 / 311.3 / 309.3 / 311.3 / 313.3 us per frame
#endif
constexpr int RZ = FPVS_ROWBITS_RZ;  // z cells per grid-writer block
__device__ __forceinline__ unsigned long long ld_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
struct RowBitsArgs {
  const unsigned long long* row_bits;
  const int* index_vol;
  int B, X, Y, Z, Nx, Ny, Nz;
  uint32_t* out;
};

__global__ void __launch_bounds__(128) rowbits_grid_kernel(const RowBitsArgs a) {
  extern __shared__ unsigned long long s_rb[];  // [RZ][X + 1]
  const int nzc = (a.Z + RZ - 1) / RZ;
  int blk = blockIdx.x;
  const int zc = blk % nzc;
  blk /= nzc;
  const int cy = blk % a.Y, b = blk / a.Y;
  const int cz0 = zc * RZ, nz = min(RZ, a.Z - cz0);
  const int ld = a.X + 1;
  const int cells = a.X * RZ;
  constexpr int kPre = 8;
  int idx[kPre];
#pragma unroll
  for (int k = 0; k < kPre; ++k) {
    const int c = threadIdx.x + k * 128, cx = c / RZ, czl = c % RZ;
    idx[k] = (c < cells && czl < nz) ? __ldg(a.index_vol + (((long long)b * a.X + cx) * a.Y + cy) * a.Z + cz0 + czl) : -1;
  }
  pdl_wait();  // row_bits: the previous launch's output
  if (threadIdx.x == 0) pdl_trigger();
  for (int c0 = 0; c0 < cells; c0 += kPre * 128) {
    if (c0) {
#pragma unroll
      for (int k = 0; k < kPre; ++k) {
        const int c = c0 + threadIdx.x + k * 128, cx = c / RZ, czl = c % RZ;
        idx[k] = (c < cells && czl < nz)
                     ? __ldg(a.index_vol + (((long long)b * a.X + cx) * a.Y + cy) * a.Z + cz0 + czl) : -1;
      }
    }
    // all gathers in flight before the first shared-memory store
    unsigned long long m[kPre];
#pragma unroll
    for (int k = 0; k < kPre; ++k) m[k] = idx[k] >= 0 ? ld_u64(a.row_bits + idx[k]) : 0ull;
#pragma unroll
    for (int k = 0; k < kPre; ++k) {
      const int c = c0 + threadIdx.x + k * 128;
      if (c < cells) s_rb[(c % RZ) * ld + c / RZ] = m[k];
    }
  }
  __syncthreads();
  const int wpr = a.Nx >> 5;  // 32-froxel words per voxel row
  const long long plane = (long long)wpr * a.Ny * a.Nz;
  for (int t = threadIdx.x; t < nz * wpr; t += 128) {
    const int w = t % wpr, czl = t / wpr;
    unsigned long long m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = s_rb[czl * ld + 8 * w + i];
    uint32_t* dst = a.out + b * plane + w + (long long)wpr * (4 * cy + (long long)a.Ny * 4 * (cz0 + czl));
#pragma unroll
    for (int lz = 0; lz < 4; ++lz)
#pragma unroll
      for (int ly = 0; ly < 4; ++ly) {
        const int sh = 4 * (ly + 4 * lz);
        uint32_t word = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) word |= (uint32_t)((m[i] >> sh) & 0xFull) << (4 * i);
        dst[(long long)wpr * (ly + (long long)a.Ny * lz)] = word;
      }
  }
}
// The grid writer as a dataflow consumer of the fused-head conv: block =
// (b, x octet w = the 8 cells of one 32-froxel word column, cell row cy),
// all z; its cells' rows lie in 8 consecutive x slabs, i.e. a contiguous
// range of 128-row tiles, so it waits (acquire polling) only for those
// tiles' done flags instead of the whole conv grid, and the blocks of the
// low x octets run in the conv's last wave.  Words are the plain writer's.
constexpr int kFlowMaxZ = 256;  // cells along z per block (Nz <= 1024)
__global__ void __launch_bounds__(256) rowbits_grid_flow_kernel(const RowBitsArgs a, const int* done_in) {
  __shared__ unsigned long long s_rb[8][kFlowMaxZ];
  __shared__ int s_lo, s_hi;
  const int nw = a.X / 8;
  int blk = blockIdx.x;
  const int w = blk % nw;
  blk /= nw;
  const int cy = blk % a.Y, b = blk / a.Y;
  if (threadIdx.x == 0) {
    s_lo = INT_MAX;
    s_hi = -1;
  }
  __syncthreads();
  // the cells' rows (the map build's index volume: two or more launches old)
  int lo = INT_MAX, hi = -1;
  for (int c = threadIdx.x; c < 8 * a.Z; c += blockDim.x) {
    const int i = c / a.Z, cz = c - i * a.Z;
    const int r = __ldg(a.index_vol + (((long long)b * a.X + 8 * w + i) * a.Y + cy) * a.Z + cz);
    s_rb[i][cz] = (unsigned long long)(long long)r;  // row index for now
    if (r >= 0) {
      lo = min(lo, r);
      hi = max(hi, r);
    }
  }
  if (lo <= hi) {
    atomicMin(&s_lo, lo);
    atomicMax(&s_hi, hi);
  }
  __syncthreads();
  // wait for the producer tiles holding those rows (bounded spin: a producer
  // that never finishes fails the launch instead of hanging it)
  if (s_hi >= 0)
    for (int t = s_lo / 128 + (int)threadIdx.x; t <= s_hi / 128; t += blockDim.x) {
      long long spins = 0;
      while (ld_acquire_gpu(done_in + t) < 4) {
        __nanosleep(32);
        if (++spins > (1LL << 26)) __trap();
      }
    }
  __syncthreads();
  if (threadIdx.x == 0) pdl_trigger();  // after this block's waits, as every kernel here
  for (int c = threadIdx.x; c < 8 * a.Z; c += blockDim.x) {
    const int i = c / a.Z, cz = c - i * a.Z;
    const long long r = (long long)s_rb[i][cz];
    s_rb[i][cz] = r >= 0 ? ld_u64(a.row_bits + r) : 0ull;
  }
  __syncthreads();
  const int wpr = a.Nx >> 5;
  const long long plane = (long long)wpr * a.Ny * a.Nz;
  // 16 words per z cell: (ly, lz) voxel rows of the 8 cells' 4-bit x runs
  for (int t = threadIdx.x; t < 16 * a.Z; t += blockDim.x) {
    const int cz = t >> 4, ly = t & 3, lz = (t >> 2) & 3;
    const int sh = 4 * (ly + 4 * lz);
    uint32_t word = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) word |= (uint32_t)((s_rb[i][cz] >> sh) & 0xFull) << (4 * i);
    a.out[b * plane + w + (long long)wpr * ((4 * cy + ly) + (long long)a.Ny * (4 * cz + lz))] = word;
  }
}

}  // namespace halo
}  // namespace fpvs

extern "C" int fpvs_rowbits_to_grid_flow(const uint64_t* row_bits, const int32_t* index_vol, int B, int Nx, int Ny,
                                         int Nz, int d, uint8_t* out_bits, const int32_t* tile_done_in,
                                         void* stream) {
  FPVS_CHECK_ARG(row_bits && index_vol && out_bits && tile_done_in, "null pointer");
  FPVS_CHECK_ARG(d == 4, "fpvs_rowbits_to_grid_flow: d = 4 (64 bits per cell), got %d", d);
  FPVS_CHECK_ARG(B >= 1 && Nx > 0 && Ny > 0 && Nz > 0 && Nx % 32 == 0 && Ny % 4 == 0 && Nz % 4 == 0,
                 "grid must be B x Nx x Ny x Nz with N_x %% 32 == 0 and N_y, N_z %% 4 == 0");
  FPVS_CHECK_ARG(Nz / 4 <= halo::kFlowMaxZ, "N_z <= %d", 4 * halo::kFlowMaxZ);
  FPVS_CHECK_ARG(((uintptr_t)out_bits & 3) == 0, "out_bits must be 4-byte aligned");
  halo::RowBitsArgs a{reinterpret_cast<const unsigned long long*>(row_bits), index_vol, B, Nx / 4, Ny / 4, Nz / 4,
                      Nx, Ny, Nz, reinterpret_cast<uint32_t*>(out_bits)};
  const long long blocks = (long long)B * (a.X / 8) * a.Y;
  FPVS_CHECK_ARG(blocks < (1LL << 31), "grid too large");
  cudaError_t e = launch_kernel(halo::rowbits_grid_flow_kernel, dim3((unsigned)blocks), dim3(256), 0,
                                as_stream(stream), a, tile_done_in);
  if (e != cudaSuccess) return set_error(FPVS_ECUDA, "fpvs_rowbits_to_grid_flow: %s", cudaGetErrorString(e));
  FPVS_CHECK_LAUNCH("fpvs_rowbits_to_grid_flow");
  return FPVS_OK;
}

extern "C" int fpvs_rowbits_to_grid(const uint64_t* row_bits, const int32_t* index_vol, int B, int Nx, int Ny, int Nz,
                                    int d, uint8_t* out_bits, void* stream) {
  FPVS_CHECK_ARG(row_bits && index_vol && out_bits, "null pointer");
  FPVS_CHECK_ARG(d == 4, "fpvs_rowbits_to_grid: d = 4 (64 bits per cell), got %d", d);
  FPVS_CHECK_ARG(B >= 1 && Nx > 0 && Ny > 0 && Nz > 0 && Nx % 32 == 0 && Ny % 4 == 0 && Nz % 4 == 0,
                 "grid must be B x Nx x Ny x Nz with N_x %% 32 == 0 and N_y, N_z %% 4 == 0");
  FPVS_CHECK_ARG(((uintptr_t)out_bits & 3) == 0, "out_bits must be 4-byte aligned");
  halo::RowBitsArgs a{reinterpret_cast<const unsigned long long*>(row_bits), index_vol, B, Nx / 4, Ny / 4, Nz / 4,
                      Nx, Ny, Nz, reinterpret_cast<uint32_t*>(out_bits)};
  const int nzc = (a.Z + halo::RZ - 1) / halo::RZ;
  const long long blocks = (long long)B * a.Y * nzc;
  const size_t smem = (size_t)halo::RZ * (a.X + 1) * 8;
  FPVS_CHECK_ARG(blocks < (1LL << 31) && smem <= 48 * 1024, "grid too large (N_x <= 1024)");
  cudaError_t e = launch_kernel(halo::rowbits_grid_kernel, dim3((unsigned)blocks), dim3(128), smem, as_stream(stream), a);
  if (e != cudaSuccess) return set_error(FPVS_ECUDA, "fpvs_rowbits_to_grid: %s", cudaGetErrorString(e));
  FPVS_CHECK_LAUNCH("fpvs_rowbits_to_grid");
  return FPVS_OK;
}
