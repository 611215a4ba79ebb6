// (3) Sparse convolution on 5th-generation tensor cores (tcgen05, sm_100a).
//
// Implicit gather-GEMM-scatter.  An output tile is BM = 128 active cells x BN
// output channels.  K is the flattened (offset j, channel ci) index
// k = j*Cin + ci of the reference weight rows (neural.py:163-166), cut into
// 64-element (128-byte) chunks; a pipeline stage holds G chunks.  Per chunk:
//   * A (128 x 64 bf16) is GATHERED: row i of the tile is x[nbr[i][j]].  Eight
//     producer warps issue 16-byte cp.async pieces straight into the
//     128B-swizzled K-major layout the UMMA descriptor reads; a missing
//     neighbour (-1) is a zero-fill.  For Cin < 64 one chunk spans 64/Cin
//     offsets.  (A TMA tile::gather4 producer was measured slower on B200:
//     ~130 cycles per 512-byte gather per SM.)
//   * B (BN x 64 bf16): one bulk copy (cp.async.bulk, TMA engine) of the
//     pre-swizzled weight image from fpvs_pack_weights_tc.
//   * one elected thread issues 4 x tcgen05.mma per chunk (M=128, N=BN, K=16,
//     bf16 -> fp32) into a TMEM accumulator; tcgen05.commit frees the stage.
//     Offsets with no neighbour anywhere in the tile are skipped.
//   * 4 epilogue warps drain TMEM (tcgen05.ld) from a double-buffered
//     accumulator (2 x BN columns) so the epilogue of tile t overlaps the
//     mainloop of tile t+1, and fuse bias + ReLU + bf16 cast, or for the
//     head sigmoid-threshold + the deinterleave bit-pack.
// Stage arrivals are per warp and lag the copies (cp.async.wait_group), so a
// stage costs 9 mbarrier arrivals instead of one per thread.  Each tile's
// neighbour rows are prefetched one tile ahead (double-buffered).  Layers
// with very few row tiles can split N across CTAs (BN < Cout).  The grid is
// persistent (<= 148 CTAs) and reads the active row count from device memory
// (graph-capturable).
#include <math.h>
#include <string.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace fpvs {
namespace tc {

constexpr int A_BYTES = BM * 128;  // 16 KB
constexpr int kMaxK = 27;

struct Params {
  const __nv_bfloat16* x;
  int ldx, x_rows;
  const int* nbr;
  int K;
  const uint32_t* tile_masks;  // per 128-row tile: offsets present (fpvs_kmap_tile_masks)
  const int* n_dev;
  int cap;
  const uint8_t* wpk;
  int nchunks, nblk;
  const float* bias;
  int cin, cout, act;
  __nv_bfloat16* y;
  int ldy, col_off;
  const int* out_rows;  // tile row -> output row (-1 = skip); NULL = identity
  // column-block scatter (k2s2 up conv as one dense GEMM over the coarse rows):
  // columns [j blk_w, (j + 1) blk_w) of row r go to output row blk_rows[8 r + j]
  // (the coarse level's down table: its child in parity class j; -1 = skip)
  const int* blk_rows;
  int blk_w;
  const __nv_bfloat16* mask;  // act == FPVS_ACT_MASK: out = z * (mask[row][col] > 0) (relu' of the layer below)
  int ldm;
  // head epilogue
  int head;
  const int4* coords;
  int d, dlog, Nx, Ny, Nz;
  float tau, zt;
  uint8_t* out_bits;
  float* probs;
  float* logits;
  int dbg;  // profiling knob (FPVS_TC_DEBUG): 1 = no MMA, 2 = no A gather, 4 = no B copy, 16 = timestamps
  // tile-level dataflow consumer (fpvs_spconv_tc_flow): x is the output of the
  // launch just before, which publishes done_in[t] = 4 per 128-row tile of
  // its level (done_n: that level's row count); each tile waits only for the
  // producer tiles its gathered rows lie in, instead of the whole grid
  const int* done_in;
  const int* done_n;
};

template <int BN, int G, int PW = 8, int MINB = 1>
struct Cfg {
  static constexpr int P = PW;                  // A-gather warps
  static constexpr int BW_WARP = P;             // B loader + stage flags
  static constexpr int NB_WARP = P + 1;         // neighbour-row loader
  static constexpr int MMA_WARP = P + 2;
  static constexpr int THREADS = (P + 7) * 32;  // + 4 epilogue warps
  static constexpr int PROD = P * 32;
  static constexpr int B_SUB = BN * 128;        // one 64-wide K chunk of B
  static constexpr int STAGE_A = G * A_BYTES;   // G K-chunks per pipeline stage
  static constexpr int STAGE_B = G * B_SUB;
  static constexpr int STAGE_BYTES = STAGE_A + STAGE_B;
  static constexpr int NBR_BYTES = 2 * BM * kMaxK * 4;  // double-buffered neighbour tile
  static constexpr int kStageBudget = 232448 / MINB - 1024 - NBR_BYTES - 6144;
  static constexpr int STAGES = kStageBudget / STAGE_BYTES > 8 ? 8 : kStageBudget / STAGE_BYTES;
  static constexpr int TMEM_COLS = (2 * BN) <= 32 ? 32 : (2 * BN) <= 64 ? 64 : (2 * BN) <= 128 ? 128
                                 : (2 * BN) <= 256 ? 256 : 512;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES + NBR_BYTES;
  static constexpr int CTRL_OFF = BAR_OFF + 8 * (2 * STAGES + 8);  // tmem addr, stage info
  static constexpr int BIAS_OFF = CTRL_OFF + 128;
  static constexpr int SMEM = 1024 + BIAS_OFF + 4 * 1024 + 16;
  static_assert(STAGES >= 2, "pipeline needs two stages");
  static_assert(STAGES <= 16, "stage info slots");
  static_assert(SMEM * MINB <= 232448, "shared memory budget");
};

// ---------------- profiling timestamps (profiling builds, FPVS_TC_DEBUG & 16) ----------------
#ifdef FPVS_PROFILE
__device__ unsigned long long g_dbg_ts[2][4096];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TS(slot)                                                              \
  do {                                                                        \
    if ((FPVS_KNOB(p) & 16) && blockIdx.x < 2 && (slot) < 4096) g_dbg_ts[blockIdx.x][(slot)] = gtimer(); \
  } while (0)
#else
#define TS(slot) \
  do {           \
  } while (0)
#endif

// Walks the K-chunks a tile needs, in order, from its offset mask: for
// Cin >= 64 every ci-chunk (cpo per offset) of each present offset j; for
// Cin < 64 every chunk (opc offsets wide) holding a present offset.
struct ChunkIter {
  uint32_t mask, rem;
  int cpo, opc, j, cc, cg;
  __device__ void init(uint32_t m, int cpo_, int opc_) {
    mask = m ? m : 1u;
    rem = mask;
    cpo = cpo_;
    opc = opc_;
    j = -1;
    cc = cpo_;
    cg = -1;
  }
  __device__ int count(int nchunks) const {
    if (opc == 1) return __popc(mask) * cpo;
    const uint32_t gm = (1u << opc) - 1u;
    int k = 0;
    for (int c = 0; c < nchunks; ++c) k += ((mask >> (c * opc)) & gm) ? 1 : 0;
    return k;
  }
  // next chunk: jbase (first offset of the chunk), cibase (first channel), chunk id
  __device__ void next(int& jb, int& cib, int& c) {
    if (opc == 1) {
      if (++cc >= cpo) { cc = 0; j = __ffs(rem) - 1; rem &= rem - 1; }
      jb = j; cib = cc * BK; c = j * cpo + cc;
    } else {
      const uint32_t gm = (1u << opc) - 1u;
      do { ++cg; } while (!((mask >> (cg * opc)) & gm));
      jb = cg * opc; cib = 0; c = cg;
    }
  }
};

// Copy neighbour rows [row0, row0 + BM) of a K-wide int32 table into shared
// memory with 16-byte cp.async pieces (zero-filled past the table end), then
// arrive (noinc) on `bar` once this thread's copies have landed.
__device__ __forceinline__ void prefetch_nbr(const Params& p, int row0, uint32_t dst, uint32_t bar, int t, int nt) {
  const long long tab_bytes = (long long)p.cap * p.K * 4;
  const long long base = (long long)row0 * p.K * 4;
  const int bytes = BM * p.K * 4;
  const char* src = reinterpret_cast<const char*>(p.nbr);
  for (int o = t * 16; o < bytes; o += nt * 16) {
    long long rem = tab_bytes - (base + o);
    uint32_t n = rem >= 16 ? 16u : (rem > 0 ? (uint32_t)rem : 0u);
    cp_async16(dst + o, src + (n ? base + o : 0), n);
  }
  cp_async_mbar_arrive_noinc(bar);
}

template <int BN, int G, int PW, int MINB>
__global__ void __launch_bounds__(Cfg<BN, G, PW, MINB>::THREADS, MINB) spconv_tc_kernel(const Params p) {
  using C = Cfg<BN, G, PW, MINB>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // pointers stay derived from the __shared__ array (LDS/STS, not generic)
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* sA = smem;                              // [STAGES][G][16 KB]
  uint8_t* sB = smem + C::STAGES * C::STAGE_A;     // [STAGES][G][B_SUB]
  int* s_nbr = reinterpret_cast<int*>(smem + C::STAGES * C::STAGE_BYTES);  // 2 x BM*K
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* nfull = tempty + 2;   // neighbour tile landed (bulk copy)
  uint64_t* nempty = nfull + 2;   // every A warp is done with the neighbour tile
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + C::CTRL_OFF);
  uint32_t* s_info = s_tmem + 8;  // per stage: bit0 first, bit1 last of the tile, bits 2+ chunks in the stage
  float* s_bias = reinterpret_cast<float*>(smem + C::BIAS_OFF);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) TS(0);
  const int n = min(*p.n_dev, p.cap);
  const int mtiles = (n + BM - 1) / BM;
  const int ntiles = mtiles * p.nblk;

  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(smem_u32(full + s), C::PROD + 1);  // async arrival per A thread + the B loader's expect_tx
      mbar_init(smem_u32(empty + s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(tfull + a), 1);
      mbar_init(smem_u32(tempty + a), 4);  // one arrival per epilogue warp
      mbar_init(smem_u32(nfull + a), 1);
      mbar_init(smem_u32(nempty + a), C::P);
    }
    fence_mbar_init();
  }
  for (int c = tid; c < p.cout; c += C::THREADS) s_bias[c] = p.bias ? p.bias[c] : 0.f;
  if (warp == C::MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "n"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *s_tmem;
  if (tid == 0) TS(1);

  const int cpo = p.cin >= BK ? p.cin / BK : 1;  // chunks per offset (Cin >= 64)
  const int opc = p.cin >= BK ? 1 : BK / p.cin;  // offsets per chunk (Cin < 64)
  const bool ident = p.nbr == nullptr;
  const int nbr_elems = BM * p.K;

  if (warp < C::P) {
    // ===================== A-gather warps =====================
    const bool flow = p.done_in != nullptr;
    if (!flow) {
      pdl_wait();  // x is the previous launch's output
      if (tid == 0) pdl_trigger();
    }
    __shared__ int s_dep[2][C::P];
    bool triggered = false;
    // All PROD threads gather every chunk: thread t owns column slot t%8 and
    // rows t/8 + RSTEP*i of the 128B-swizzled A chunk; a stage's full barrier
    // completes when every thread's cp.async pieces have landed (noinc arrival).
    constexpr int RSTEP = C::PROD / 8;
    constexpr int NPT = BM / RSTEP;  // cp.async ops per thread per chunk
    const int ppo = p.cin >> 3;
    const uint32_t ldx2 = (uint32_t)p.ldx * 2u;  // row pitch in bytes (host checks x < 2^31 B)
    const int piece = tid & 7, rbase = tid >> 3;
    const int tj = opc == 1 ? 0 : piece / ppo;                     // offset delta of my column slot
    const int tci = opc == 1 ? piece * 8 : (piece - tj * ppo) * 8;  // channel of my column slot
    int rowk[NPT];
    uint32_t dsto[NPT];
#pragma unroll
    for (int i = 0; i < NPT; ++i) {
      const int r = rbase + i * RSTEP;
      rowk[i] = r * p.K;
      dsto[i] = r * 128 + ((piece ^ (r & 7)) << 4);
    }
    int stage = 0, gst = 0;
    uint32_t phase = 0;
    int cur_m = -1, mi = -1;
    bool live[NPT];
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int mt = tile / p.nblk;
      const int row0 = mt * BM;
      if (mt != cur_m) {
        if (mi >= 0 && !ident && lane == 0) mbar_arrive(smem_u32(nempty + (mi & 1)));  // done with the old rows
        cur_m = mt;
        ++mi;
        if (!ident) mbar_wait(smem_u32(nfull + (mi & 1)), (mi >> 1) & 1);
#pragma unroll
        for (int i = 0; i < NPT; ++i) live[i] = row0 + rbase + i * RSTEP < n;
        if (flow) {
          // the producer tiles this tile's gathered rows lie in: min / max over
          // the valid rows' table entries (rows past n hold stale entries)
          const int* nbn = s_nbr + (mi & 1) * nbr_elems;
          const int nvalid = ident ? 0 : min(BM, n - row0) * p.K;
          int lo = 0x7fffffff, hi = -1;
          if (ident) {
            lo = row0;
            hi = min(row0 + BM, n) - 1;
          } else {
            for (int e = tid; e < nvalid; e += C::PROD) {
              const int v = nbn[e];
              if (v >= 0) {
                lo = min(lo, v);
                hi = max(hi, v);
              }
            }
          }
#pragma unroll
          for (int o = 16; o; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
          }
          if (lane == 0) {
            s_dep[0][warp] = lo;
            s_dep[1][warp] = hi;
          }
          named_bar(1, C::PROD);
          lo = 0x7fffffff;
          hi = -1;
#pragma unroll
          for (int w = 0; w < C::P; ++w) {
            lo = min(lo, s_dep[0][w]);
            hi = max(hi, s_dep[1][w]);
          }
          const int ptiles = (min(*p.done_n, p.x_rows) + BM - 1) / BM;
          if (hi >= 0) {
            const int t1 = min(hi / BM, ptiles - 1);
            for (int t = lo / BM + tid; t <= t1; t += C::PROD) {
              long long spins = 0;
              while (ld_acquire_gpu(p.done_in + t) < 4) {  // four epilogue warps per producer tile
                __nanosleep(32);
                if (++spins > (1LL << 26)) __trap();  // a producer that never finishes: fail, do not hang
              }
            }
          }
          named_bar(1, C::PROD);  // also: every warp read s_dep before the next tile rewrites it
          if (!triggered) {
            triggered = true;
            if (tid == 0) pdl_trigger();
          }
        }
      }
      const int* nb_s = s_nbr + (mi & 1) * nbr_elems;
      ChunkIter itr;
      itr.init(ident ? 1u : __ldg(p.tile_masks + mt), cpo, opc);
      const int nissue = itr.count(p.nchunks);
      const int nst = (nissue + G - 1) / G;
      for (int st = 0; st < nst; ++st) {
        const int nvalid = min(G, nissue - st * G);
        mbar_wait_sleep(smem_u32(empty + stage), phase ^ 1, 32);
        if (tid == 0) TS(200 + gst);
        const uint32_t a_stage = smem_u32(sA + stage * C::STAGE_A);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          if (g >= nvalid) break;
          int jb, cib, c;
          itr.next(jb, cib, c);
          const int jj = jb + tj;
          const bool jk = jj < p.K;
          const char* base = reinterpret_cast<const char*>(p.x) + (uint32_t)(cib + tci) * 2u;
          const uint32_t a_sub = a_stage + g * A_BYTES;
          uint32_t off[NPT];
          bool skip[NPT];
#pragma unroll
          for (int i = 0; i < NPT; ++i) {
            const int v = !(live[i] && jk) ? -1 : ident ? row0 + rbase + i * RSTEP : nb_s[rowk[i] + jj];
            skip[i] = v < 0;
            off[i] = skip[i] ? 0u : (uint32_t)v * ldx2;
          }
          if (!(FPVS_KNOB(p) & 2)) {
#pragma unroll
            for (int i = 0; i < NPT; ++i) cp_async16_zfill(a_sub + dsto[i], base + off[i], skip[i]);
          }
        }
        // asynchronous arrival once this thread's copies of the stage land
        // (the MMA issuer fences the generic->async proxy after its wait)
        cp_async_mbar_arrive_noinc(smem_u32(full + stage));
        if (tid == 0) TS(600 + gst);
        ++gst;
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
    if (mi >= 0 && !ident && lane == 0) mbar_arrive(smem_u32(nempty + (mi & 1)));
  } else if (warp == C::BW_WARP) {
    // ===================== B loader (one elected lane) =====================
    // Streams each stage's weight chunks with bulk copies (TMA engine) and
    // writes the stage flags the MMA issuer reads.  Waits for the previous
    // launch first: the packed weights may be its output (a lazy or per-step
    // re-pack enqueued right before this conv); a dataflow consumer's weights
    // are packed before its producer launched.
    if (!p.done_in) pdl_wait();
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int mt = tile / p.nblk, nb = tile - mt * p.nblk;
        const uint8_t* wblk = p.wpk + (size_t)nb * p.nchunks * C::B_SUB;
        ChunkIter itr;
        itr.init(ident ? 1u : __ldg(p.tile_masks + mt), cpo, opc);
        const int nissue = itr.count(p.nchunks);
        const int nst = (nissue + G - 1) / G;
        for (int st = 0; st < nst; ++st) {
          const int nvalid = min(G, nissue - st * G);
          mbar_wait(smem_u32(empty + stage), phase ^ 1);
          const uint32_t fb = smem_u32(full + stage);
          const uint32_t b_stage = smem_u32(sB + stage * C::STAGE_B);
          s_info[stage] = (st == 0 ? 1u : 0u) | (st == nst - 1 ? 2u : 0u) | ((uint32_t)nvalid << 2);
          if (FPVS_KNOB(p) & 4) {
            mbar_arrive(fb);
          } else {
            mbar_arrive_expect_tx(fb, nvalid * C::B_SUB);
            for (int g = 0; g < nvalid; ++g) {
              int jb, cib, c;
              itr.next(jb, cib, c);
              bulk_g2s(b_stage + g * C::B_SUB, wblk + (size_t)c * C::B_SUB, C::B_SUB, fb);
            }
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == C::NB_WARP) {
    // ===================== neighbour-row loader =====================
    // Bulk-copies (TMA engine) the neighbour rows of each m-tile into a double
    // buffer one m-tile ahead of the gather warps.
    auto load_rows = [&](int mt2, int b2) {
      const long long row0 = (long long)mt2 * BM;
      long long rows = p.cap - row0;
      if (rows > BM) rows = BM;
      const long long bytes = rows * p.K * 4;
      const long long bulk = bytes & ~15LL;
      const uint32_t dst = smem_u32(s_nbr + b2 * nbr_elems);
      const int* src = p.nbr + row0 * p.K;
      // the < 16-byte tail of the table (if any) goes through registers
      for (long long o = bulk / 4; o < bytes / 4; ++o) s_nbr[b2 * nbr_elems + o] = __ldg(src + o);
      mbar_arrive_expect_tx(smem_u32(nfull + b2), (uint32_t)bulk);
      if (bulk) bulk_g2s(dst, src, (uint32_t)bulk, smem_u32(nfull + b2));
    };
    if (!ident && lane == 0) {
      int cur_m = -1, mi = -1;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int mt = tile / p.nblk;
        if (mt == cur_m) continue;
        cur_m = mt;
        ++mi;
        if (mi == 0) load_rows(mt, 0);
        int nt = tile + gridDim.x;
        while (nt < ntiles && nt / p.nblk == mt) nt += gridDim.x;
        if (nt < ntiles) {
          // buffer (mi+1)&1 held m-tile mi-1: wait until every A warp released it
          if (mi >= 1) mbar_wait(smem_u32(nempty + ((mi + 1) & 1)), ((mi - 1) >> 1) & 1);
          load_rows(nt / p.nblk, (mi + 1) & 1);
        }
      }
    }
  } else if (warp == C::MMA_WARP) {
    // ===================== MMA issuer =====================
    // one thread runs the issue loop (a whole-warp loop measured ~25% slower
    // per chunk: 32-lane barrier polls and fences); lanes 1-31 go straight to
    // the final barrier.
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16<BN>();
      const uint64_t a_desc0 = sw128_desc(smem_u32(sA));
      const uint64_t b_desc0 = sw128_desc(smem_u32(sB));
      int stage = 0;
      uint32_t phase = 0;
      int it = 0, kst = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        mbar_wait(smem_u32(tempty + acc), ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dtm = tmem_base + acc * BN;
        bool firstc = true;
        while (true) {
          mbar_wait(smem_u32(full + stage), phase);
          TS(1000 + kst);
          if (firstc) TS(11 + 8 * it);
          firstc = false;
          tc_fence_after();
          if (!(FPVS_KNOB(p) & 128)) fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tcgen05 (async proxy) reads
          const uint32_t info = s_info[stage];
          if (!(FPVS_KNOB(p) & 1)) {
            // descriptors affine in the stage index, hoisted; a full stage is one
            // unrolled run of MMAs with immediate offsets (no dependent scalar
            // work between MMAs: it adds straight to their issue cost)
            const uint64_t ad0 = a_desc0 + (uint64_t)((uint32_t)stage * (C::STAGE_A >> 4));
            const uint64_t bd0 = b_desc0 + (uint64_t)((uint32_t)stage * (C::STAGE_B >> 4));
            const int nvalid = (int)(info >> 2);
            const uint32_t acc0 = (info & 1u) ? 0u : 1u;
            if (nvalid == G) {
#pragma unroll
              for (int g = 0; g < G; ++g)
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                  umma_bf16(dtm, ad0 + (uint64_t)(g * (A_BYTES >> 4) + 2 * k), bd0 + (uint64_t)(g * (C::B_SUB >> 4) + 2 * k),
                            idesc, (g == 0 && k == 0) ? acc0 : 1u);
            } else {
              for (int g = 0; g < nvalid; ++g)
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                  umma_bf16(dtm, ad0 + (uint64_t)(g * (A_BYTES >> 4) + 2 * k),
                            bd0 + (uint64_t)(g * (C::B_SUB >> 4) + 2 * k), idesc, (g == 0 && k == 0) ? acc0 : 1u);
            }
          }
          umma_commit(smem_u32(empty + stage));
          if (info & 2u) { umma_commit(smem_u32(tfull + acc)); TS(12 + 8 * it); }
          TS(1400 + kst);
          ++kst;
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          if (info & 2u) break;
        }
      }
    }
  } else {
    // ===================== epilogue (4 warps) =====================
    if (!p.done_in) pdl_wait();  // y may alias a buffer the previous launch reads (not so for a dataflow consumer)
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int r = q * 32 + lane;
    const uint32_t tlane = (uint32_t)(q * 32) << 16;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int mt = tile / p.nblk, nb = tile - mt * p.nblk;
      const int acc = it & 1;
      mbar_wait_sleep(smem_u32(tfull + acc), (it >> 1) & 1, 256);
      if (q == 0 && lane == 0) TS(13 + 8 * it);
      tc_fence_after();
      const int row = mt * BM + r;
      const bool valid = row < n;
      const int col0 = nb * BN;
      const long long orow0 = !valid ? -1 : p.out_rows ? (long long)__ldg(p.out_rows + row) : (long long)row;
      if (!p.head) {
#pragma unroll 1
        for (int cb = 0; cb < BN; cb += 32) {
          float v[32];
          tmem_ld32(tmem_base + tlane + acc * BN + cb, v);
          if (!valid || col0 + cb >= p.cout) continue;
          long long orow = orow0;
          int ocol = col0 + cb;
          if (p.blk_rows) {
            const int j = ocol / p.blk_w;
            ocol -= j * p.blk_w;
            orow = __ldg(p.blk_rows + (long long)row * 8 + j);
          }
          if (orow < 0) continue;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float z = v[i] + s_bias[col0 + cb + i];
            v[i] = p.act == FPVS_ACT_RELU ? fmaxf(z, 0.f) : z;
          }
          if (p.act == FPVS_ACT_MASK) {
            const uint4* mk = reinterpret_cast<const uint4*>(p.mask + orow * p.ldm + ocol);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint4 m4 = __ldg(mk + i);
              const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const uint32_t h = (mw[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu;  // bf16 bits; > 0 iff sign 0 and nonzero
                if (!(h != 0u && h < 0x8000u)) v[8 * i + e] = 0.f;
              }
            }
          }
          uint4* dst = reinterpret_cast<uint4*>(p.y + orow * p.ldy + p.col_off + ocol);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(pack_bf16x2(v[8 * i + 0], v[8 * i + 1]), pack_bf16x2(v[8 * i + 2], v[8 * i + 3]),
                                pack_bf16x2(v[8 * i + 4], v[8 * i + 5]), pack_bf16x2(v[8 * i + 6], v[8 * i + 7]));
        }
      } else {
        // [p >= tau] as [z >= logit(tau)] (sigmoid is monotone; the two differ
        // only within fp32 rounding of tau, inside the parity band).  When d is
        // a power of two <= 8, the d bits of one (ly, lz) row of a cell share a
        // byte of the packed grid: build them in a register, one RED.OR per row.
        int4 cc = make_int4(0, 0, 0, 0);
        if (valid) cc = p.coords[row];
        const int d = p.d, dl = p.dlog;
        const bool fast = dl >= 0 && d <= 8 && !p.probs && !p.logits && p.out_bits && p.zt < INFINITY;
#pragma unroll 1
        for (int cb = 0; cb < BN; cb += 8) {
          float v[8];
          tmem_ld8(tmem_base + tlane + acc * BN + cb, v);
          if (!valid || cb >= p.cout) continue;
          if (fast) {
            uint32_t bits8 = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) bits8 |= (v[i] + s_bias[cb + i] >= p.zt ? 1u : 0u) << i;
            if (!bits8) continue;
            const uint32_t dm = (1u << d) - 1u;
            for (int q = 0; q < (8 >> dl); ++q) {
              const uint32_t rb = (bits8 >> (q * d)) & dm;
              if (!rb) continue;
              const int rr = (cb >> dl) + q;  // rr = ly + d*lz
              const int ly = rr & (d - 1), lz = rr >> dl;
              const int fx = cc.y * d;
              const long long byte = bit_byte(cc.x, fx, cc.z * d + ly, cc.w * d + lz, p.Nx, p.Ny, p.Nz);
              uint32_t* word = reinterpret_cast<uint32_t*>(p.out_bits + (byte & ~3LL));
              atomicOr(word, rb << ((int)(byte & 3) * 8 + (fx & 7)));
            }
          } else if (d <= 8 && (d & (d - 1)) == 0 && cb + 8 <= p.cout && (p.cout & 7) == 0) {
            // probabilities / logits requested (training): vector stores, and the
            // [p >= tau] bits one RED.OR per (ly, lz) row of the cell as above
            const int dl2 = __ffs(d) - 1;
            float z8[8], p8[8];
            uint32_t bits8 = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              z8[i] = v[i] + s_bias[cb + i];
              p8[i] = sigmoidf_stable(z8[i]);
              bits8 |= (p8[i] >= p.tau ? 1u : 0u) << i;
            }
            if (p.logits) {
              float4* lg = reinterpret_cast<float4*>(p.logits + (long long)row * p.cout + cb);
              lg[0] = make_float4(z8[0], z8[1], z8[2], z8[3]);
              lg[1] = make_float4(z8[4], z8[5], z8[6], z8[7]);
            }
            if (p.probs) {
              float4* pp = reinterpret_cast<float4*>(p.probs + (long long)row * p.cout + cb);
              pp[0] = make_float4(p8[0], p8[1], p8[2], p8[3]);
              pp[1] = make_float4(p8[4], p8[5], p8[6], p8[7]);
            }
            if (bits8 && p.out_bits) {
              const uint32_t dm = (1u << d) - 1u;
              for (int q = 0; q < (8 >> dl2); ++q) {
                const uint32_t rb = (bits8 >> (q * d)) & dm;
                if (!rb) continue;
                const int rr = (cb >> dl2) + q;  // rr = ly + d*lz
                const int ly = rr & (d - 1), lz = rr >> dl2;
                const int fx = cc.y * d;
                const long long byte = bit_byte(cc.x, fx, cc.z * d + ly, cc.w * d + lz, p.Nx, p.Ny, p.Nz);
                uint32_t* word = reinterpret_cast<uint32_t*>(p.out_bits + (byte & ~3LL));
                atomicOr(word, rb << ((int)(byte & 3) * 8 + (fx & 7)));
              }
            }
          } else {
#pragma unroll 1
            for (int i = 0; i < 8; ++i) {
              const int k = cb + i;
              if (k >= p.cout) break;
              const float z = v[i] + s_bias[k];
              const float pr = sigmoidf_stable(z);
              if (p.logits) p.logits[(long long)row * p.cout + k] = z;
              if (p.probs) p.probs[(long long)row * p.cout + k] = pr;
              if (pr >= p.tau && p.out_bits) {
                const int lx = k % d, rr = k / d;
                const int fx = cc.y * d + lx;
                atomic_or_bit(p.out_bits, bit_byte(cc.x, fx, cc.z * d + rr % d, cc.w * d + rr / d, p.Nx, p.Ny, p.Nz),
                              fx & 7);
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(tempty + acc));
      if (q == 0 && lane == 0) TS(14 + 8 * it);
    }
  }

  if (tid == 0) TS(2);
  tc_fence_before();
  __syncthreads();
  if (tid == 0) TS(3);
  if (warp == C::MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(C::TMEM_COLS)
                 : "memory");
  }
}

// packed[nb][c][n][128 B] for n < BN: element kk of chunk c at
// n*128 + ((kk/8) ^ (n%8))*16 + (kk%8)*2 (Swizzle<3,4,3>), value W[c*64+kk][nb*BN + n]
// dgrad (taps > 0): the packed matrix is W'[(j*cout_src + co)][ci] = W[((taps-1-j)*cin_src + ci)][co]
// (mirrored offsets, transposed per offset), the forward weight of dx = conv(dz).
__device__ __forceinline__ void pack_weight_elem(long long t, const float* __restrict__ w, int Ktot, int cout, int BN,
                                                 int nchunks, __nv_bfloat16* __restrict__ out, int taps, int cin_src,
                                                 int cout_src) {
  int kk = t % BK;
  long long r = t / BK;
  int nn = r % BN;
  r /= BN;
  int c = r % nchunks;
  int nb = (int)(r / nchunks);
  int k = c * BK + kk, col = nb * BN + nn;
  float v = 0.f;
  if (k < Ktot && col < cout) {
    if (taps) {
      const int j = k / cout_src, co = k - j * cout_src;
      v = w[((long long)(taps - 1 - j) * cin_src + col) * cout_src + co];
    } else {
      v = w[(long long)k * cout + col];
    }
  }
  long long byte = (((long long)nb * nchunks + c) * BN + nn) * 128 + (((kk >> 3) ^ (nn & 7)) << 4) + (kk & 7) * 2;
  out[byte / 2] = __float2bfloat16_rn(v);
}

__global__ void pack_weights_kernel(const float* __restrict__ w, int Ktot, int cout, int BN, int nchunks, int nblk,
                                    __nv_bfloat16* __restrict__ out, int taps = 0, int cin_src = 0,
                                    int cout_src = 0) {
  const long long total = (long long)nblk * nchunks * BN * BK;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x)
    pack_weight_elem(t, w, Ktot, cout, BN, nchunks, out, taps, cin_src, cout_src);
}

// every layer's images in one launch (after an optimizer step)
constexpr int kMaxPackJobs = 32;
struct PackJob {
  const float* w;
  __nv_bfloat16* out;
  int Ktot, cout, BN, nchunks, taps, cin_src, cout_src;
  long long base;  // first element of this job in the concatenated space
};
struct PackJobs {
  PackJob j[kMaxPackJobs];
  int count;
  long long total;
};

__global__ void pack_weights_multi_kernel(const PackJobs J) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < J.total;
       t += (long long)gridDim.x * blockDim.x) {
    int q = 0;
    while (q + 1 < J.count && t >= J.j[q + 1].base) ++q;
    const PackJob& b = J.j[q];
    pack_weight_elem(t - b.base, b.w, b.Ktot, b.cout, b.BN, b.nchunks, b.out, b.taps, b.cin_src, b.cout_src);
  }
}

inline int pick_bn(int cout) {
  if (cout <= 32) return 32;
  if (cout <= 64) return 64;
  if (cout <= 128) return 128;
  return 256;
}

inline bool valid_bn(int bn) { return bn == 32 || bn == 64 || bn == 128 || bn == 256; }

template <int BN, int G, int PW, int MINB>
int launch_cfg(const Params& p, cudaStream_t s) {
  using C = Cfg<BN, G, PW, MINB>;
  {
    const cudaError_t e = set_smem_once<spconv_tc_kernel<BN, G, PW, MINB>>(C::SMEM);
    if (e != cudaSuccess) return set_error(FPVS_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  long long tiles = (long long)((p.cap + BM - 1) / BM) * p.nblk;
  long long slots = (long long)kNumSMs * MINB;
  int grid = (int)(tiles < slots ? tiles : slots);
  if (grid < 1) grid = 1;
  cudaError_t e = launch_kernel(spconv_tc_kernel<BN, G, PW, MINB>, dim3(grid), dim3(C::THREADS), C::SMEM, s, p);
  if (e != cudaSuccess) return set_error(FPVS_ECUDA, "spconv_tc: %s", cudaGetErrorString(e));
  FPVS_CHECK_LAUNCH("spconv_tc");
  return FPVS_OK;
}

#ifndef FPVS_TC_MINB2_BN
#define FPVS_TC_MINB2_BN 32  // 32-wide tiles (the chain nets) run two CTAs per SM: config-5 step 692 -> 652 us; wider ones measured slower (U-Net +8 us)
#endif
template <int BN>
int launch(const Params& p, cudaStream_t s) {
  // two K chunks per stage halve the per-stage barrier/commit overhead where
  // the stage still fits >= 4 times in shared memory
  constexpr bool two = BN <= FPVS_TC_MINB2_BN;
  return launch_cfg<BN, (two ? 1 : BN <= 128 ? 2 : 1), 8, (two ? 2 : 1)>(p, s);
}

int dispatch(Params& p, int bn, cudaStream_t s) {
  switch (bn) {
    case 32: return launch<32>(p, s);
    case 64: return launch<64>(p, s);
    case 128: return launch<128>(p, s);
    case 256: return launch<256>(p, s);
  }
  return set_error(FPVS_EINVAL, "bad tensor-core tile width %d", bn);
}

}  // namespace tc
}  // namespace fpvs

using namespace fpvs;

static int resolve_bn(int bn, int cout) {
  if (bn == 0) bn = tc::pick_bn(cout);
  return tc::valid_bn(bn) ? bn : -1;
}

#ifdef FPVS_PROFILE
// profiling builds only (not part of the ABI): copy CTA 0/1 timestamps out
extern "C" int fpvs_debug_tc_timestamps(unsigned long long* host, int n) {
  if (n > 2 * 4096) n = 2 * 4096;
  cudaError_t e = cudaMemcpyFromSymbol(host, tc::g_dbg_ts, sizeof(unsigned long long) * n);
  return e == cudaSuccess ? 0 : 3;
}
#endif

extern "C" size_t fpvs_pack_weights_tc_size(int K, int cin, int cout, int bn) {
  bn = resolve_bn(bn, cout);
  if (bn < 0 || K < 1 || cin < 1 || cout < 1) return 0;
  size_t nchunks = ((size_t)K * cin + tc::BK - 1) / tc::BK;
  size_t nblk = ((size_t)cout + bn - 1) / bn;
  return nblk * nchunks * bn * 128;
}

extern "C" int fpvs_pack_weights_tc(const float* w, int K, int cin, int cout, int bn, void* packed, void* stream) {
  FPVS_CHECK_ARG(w && packed, "null pointer");
  bn = resolve_bn(bn, cout);
  FPVS_CHECK_ARG(bn > 0, "tile width must be 0 (auto), 32, 64, 128 or 256");
  FPVS_CHECK_ARG(cin % 8 == 0, "tcgen05 path needs Cin %% 8 == 0, got %d", cin);
  int nchunks = (K * cin + tc::BK - 1) / tc::BK;
  int nblk = (cout + bn - 1) / bn;
  long long total = (long long)nblk * nchunks * bn * tc::BK;
  tc::pack_weights_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(w, K * cin, cout, bn, nchunks, nblk,
                                                                              (__nv_bfloat16*)packed);
  FPVS_CHECK_LAUNCH("fpvs_pack_weights_tc");
  return FPVS_OK;
}

static int tc_common(tc::Params& p, const void* x, int ldx, int x_rows, const int32_t* nbr, int K,
                     const uint32_t* tile_masks, const int32_t* n_dev, int cap, const void* w_packed,
                     const float* bias, int cin, int cout, int bn) {
  FPVS_CHECK_ARG(x && w_packed && n_dev, "null pointer");
  FPVS_CHECK_ARG(K >= 1 && K <= tc::kMaxK, "K must lie in [1, 27]");
  FPVS_CHECK_ARG(nbr || K == 1, "nbr may be NULL only for K == 1");
  FPVS_CHECK_ARG(!nbr || tile_masks, "tile_masks (fpvs_kmap_tile_masks) are required with a neighbour table");
  FPVS_CHECK_ARG(cin % 8 == 0 && ldx % 8 == 0 && ldx >= cin, "tcgen05 path needs Cin and ldx multiples of 8");
  FPVS_CHECK_ARG(cout >= 1 && cout <= 1024, "bad Cout %d", cout);
  FPVS_CHECK_ARG(x_rows >= 1, "x_rows must be positive");
  FPVS_CHECK_ARG((long long)x_rows * ldx * 2 < (1LL << 31), "feature buffer too large for 32-bit row offsets");
  p = tc::Params{};
  p.x = (const __nv_bfloat16*)x;
  p.ldx = ldx;
  p.x_rows = x_rows;
  p.nbr = nbr;
  p.K = K;
  p.tile_masks = tile_masks;
  p.n_dev = n_dev;
  p.cap = cap;
  p.wpk = (const uint8_t*)w_packed;
  p.nchunks = (K * cin + tc::BK - 1) / tc::BK;
  p.nblk = (cout + bn - 1) / bn;
  p.bias = bias;
  p.cin = cin;
  p.cout = cout;
  p.dbg = debug_knob("FPVS_TC_DEBUG");
  return FPVS_OK;
}

extern "C" int fpvs_spconv_tc(const void* x, int ldx, int x_rows, const int32_t* nbr, int K,
                              const uint32_t* tile_masks, const int32_t* n_out_dev, int cap_out, const void* w_packed,
                              int bn, const float* bias, int cin, int cout, int act, void* y, int ldy, int col_off,
                              void* stream) {
  tc::Params p;
  bn = resolve_bn(bn, cout);
  FPVS_CHECK_ARG(bn > 0, "tile width must be 0 (auto), 32, 64, 128 or 256");
  int rc = tc_common(p, x, ldx, x_rows, nbr, K, tile_masks, n_out_dev, cap_out, w_packed, bias, cin, cout, bn);
  if (rc) return rc;
  FPVS_CHECK_ARG(y, "null output");
  FPVS_CHECK_ARG(cout % 32 == 0, "tcgen05 store epilogue needs Cout %% 32 == 0, got %d", cout);
  FPVS_CHECK_ARG(ldy % 8 == 0 && col_off % 8 == 0 && ldy >= col_off + cout, "bad output leading dimension");
  FPVS_CHECK_ARG(act == FPVS_ACT_NONE || act == FPVS_ACT_RELU, "tcgen05 store epilogue supports none/relu");
  if (cap_out <= 0) return FPVS_OK;
  p.act = act;
  p.y = (__nv_bfloat16*)y;
  p.ldy = ldy;
  p.col_off = col_off;
  return tc::dispatch(p, bn, as_stream(stream));
}

extern "C" int fpvs_spconv_tc_flow(const void* x, int ldx, int x_rows, const int32_t* nbr, int K,
                                   const uint32_t* tile_masks, const int32_t* n_out_dev, int cap_out,
                                   const void* w_packed, int bn, const float* bias, int cin, int cout, int act, void* y,
                                   int ldy, int col_off, const int32_t* tile_done_in, const int32_t* done_n_dev,
                                   void* stream) {
  tc::Params p;
  bn = resolve_bn(bn, cout);
  FPVS_CHECK_ARG(bn > 0, "tile width must be 0 (auto), 32, 64, 128 or 256");
  int rc = tc_common(p, x, ldx, x_rows, nbr, K, tile_masks, n_out_dev, cap_out, w_packed, bias, cin, cout, bn);
  if (rc) return rc;
  FPVS_CHECK_ARG(y, "null output");
  FPVS_CHECK_ARG(cout % 32 == 0, "tcgen05 store epilogue needs Cout %% 32 == 0, got %d", cout);
  FPVS_CHECK_ARG(ldy % 8 == 0 && col_off % 8 == 0 && ldy >= col_off + cout, "bad output leading dimension");
  FPVS_CHECK_ARG(act == FPVS_ACT_NONE || act == FPVS_ACT_RELU, "tcgen05 store epilogue supports none/relu");
  FPVS_CHECK_ARG(!tile_done_in || done_n_dev, "tile_done_in needs the producer's row count");
  if (cap_out <= 0) return FPVS_OK;
  p.act = act;
  p.y = (__nv_bfloat16*)y;
  p.ldy = ldy;
  p.col_off = col_off;
  p.done_in = tile_done_in;
  p.done_n = done_n_dev;
  return tc::dispatch(p, bn, as_stream(stream));
}

extern "C" int fpvs_spconv_tc_scatter(const void* x, int ldx, int x_rows, const int32_t* nbr, int K,
                                      const uint32_t* tile_masks, const int32_t* n_out_dev, int cap_out,
                                      const int32_t* out_rows, const void* w_packed, int bn, const float* bias,
                                      int cin, int cout, int act, void* y, int ldy, int col_off, void* stream) {
  tc::Params p;
  bn = resolve_bn(bn, cout);
  FPVS_CHECK_ARG(bn > 0, "tile width must be 0 (auto), 32, 64, 128 or 256");
  FPVS_CHECK_ARG(out_rows, "null out_rows");
  int rc = tc_common(p, x, ldx, x_rows, nbr, K, tile_masks, n_out_dev, cap_out, w_packed, bias, cin, cout, bn);
  if (rc) return rc;
  FPVS_CHECK_ARG(y, "null output");
  FPVS_CHECK_ARG(cout % 32 == 0, "tcgen05 store epilogue needs Cout %% 32 == 0, got %d", cout);
  FPVS_CHECK_ARG(ldy % 8 == 0 && col_off % 8 == 0 && ldy >= col_off + cout, "bad output leading dimension");
  FPVS_CHECK_ARG(act == FPVS_ACT_NONE || act == FPVS_ACT_RELU, "tcgen05 store epilogue supports none/relu");
  if (cap_out <= 0) return FPVS_OK;
  p.act = act;
  p.y = (__nv_bfloat16*)y;
  p.ldy = ldy;
  p.col_off = col_off;
  p.out_rows = out_rows;
  return tc::dispatch(p, bn, as_stream(stream));
}

extern "C" int fpvs_spconv_tc_upblocks(const void* x, int ldx, int x_rows, const int32_t* n_coarse_dev, int cap_coarse,
                                       const void* w_packed, int bn, const float* bias8, int cin, int cout, int act,
                                       const int32_t* child_rows, void* y, int ldy, int col_off, void* stream) {
  tc::Params p;
  const int cout8 = 8 * cout;
  bn = resolve_bn(bn, cout8);
  FPVS_CHECK_ARG(bn > 0, "tile width must be 0 (auto), 32, 64, 128 or 256");
  FPVS_CHECK_ARG(child_rows, "null child_rows");
  FPVS_CHECK_ARG(cout % 32 == 0 && cout8 <= 1024, "up blocks need Cout %% 32 == 0 and 8 Cout <= 1024, got %d", cout);
  int rc = tc_common(p, x, ldx, x_rows, nullptr, 1, nullptr, n_coarse_dev, cap_coarse, w_packed, bias8, cin, cout8, bn);
  if (rc) return rc;
  FPVS_CHECK_ARG(y, "null output");
  FPVS_CHECK_ARG(ldy % 8 == 0 && col_off % 8 == 0 && ldy >= col_off + cout, "bad output leading dimension");
  FPVS_CHECK_ARG(act == FPVS_ACT_NONE || act == FPVS_ACT_RELU, "tcgen05 store epilogue supports none/relu");
  if (cap_coarse <= 0) return FPVS_OK;
  p.act = act;
  p.y = (__nv_bfloat16*)y;
  p.ldy = ldy;
  p.col_off = col_off;
  p.blk_rows = child_rows;
  p.blk_w = cout;
  return tc::dispatch(p, bn, as_stream(stream));
}

extern "C" int fpvs_pack_weights_tc_dgrad(const float* w, int K, int cin, int cout, int bn, void* packed,
                                          void* stream) {
  FPVS_CHECK_ARG(w && packed, "null pointer");
  // the dgrad conv maps cout -> cin channels
  bn = resolve_bn(bn, cin);
  FPVS_CHECK_ARG(bn > 0, "tile width must be 0 (auto), 32, 64, 128 or 256");
  FPVS_CHECK_ARG(cout % 8 == 0, "tcgen05 dgrad needs Cout %% 8 == 0, got %d", cout);
  const int nchunks = (K * cout + tc::BK - 1) / tc::BK;
  const int nblk = (cin + bn - 1) / bn;
  const long long total = (long long)nblk * nchunks * bn * tc::BK;
  tc::pack_weights_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(
      w, K * cout, cin, bn, nchunks, nblk, (__nv_bfloat16*)packed, K, cin, cout);
  FPVS_CHECK_LAUNCH("fpvs_pack_weights_tc_dgrad");
  return FPVS_OK;
}

extern "C" int fpvs_pack_weights_tc_multi(const fpvs_pack_job* jobs, int njobs, void* stream) {
  FPVS_CHECK_ARG(jobs && njobs >= 1 && njobs <= tc::kMaxPackJobs, "1..%d pack jobs", tc::kMaxPackJobs);
  tc::PackJobs J{};
  J.count = njobs;
  long long tot = 0;
  for (int i = 0; i < njobs; ++i) {
    const fpvs_pack_job& q = jobs[i];
    FPVS_CHECK_ARG(q.w && q.packed && q.K >= 1 && q.cin >= 1 && q.cout >= 1, "bad pack job %d", i);
    // a dgrad image is the forward image of the Cout -> Cin conv with mirrored offsets
    const int kin = q.dgrad ? q.cout : q.cin, kout = q.dgrad ? q.cin : q.cout;
    const int bn = resolve_bn(q.bn, kout);
    FPVS_CHECK_ARG(bn > 0, "pack job %d: tile width must be 0 (auto), 32, 64, 128 or 256", i);
    FPVS_CHECK_ARG(kin % 8 == 0, "pack job %d: tcgen05 path needs the K-side channels %% 8 == 0", i);
    const int nchunks = (q.K * kin + tc::BK - 1) / tc::BK, nblk = (kout + bn - 1) / bn;
    J.j[i] = tc::PackJob{q.w, (__nv_bfloat16*)q.packed, q.K * kin, kout, bn, nchunks, q.dgrad ? q.K : 0,
                         q.dgrad ? q.cin : 0, q.dgrad ? q.cout : 0, tot};
    tot += (long long)nblk * nchunks * bn * tc::BK;
  }
  J.total = tot;
  tc::pack_weights_multi_kernel<<<grid_for(tot, 256), 256, 0, as_stream(stream)>>>(J);
  FPVS_CHECK_LAUNCH("fpvs_pack_weights_tc_multi");
  return FPVS_OK;
}

extern "C" int fpvs_spconv_tc_dgrad(const void* dz, int lddz, int dz_rows, const int32_t* nbr, int K,
                                    const uint32_t* tile_masks, const int32_t* n_dev, int cap,
                                    const void* w_packed_dgrad, int bn, int cin, int cout, const void* mask, int ldm,
                                    void* dx, int lddx, void* stream) {
  tc::Params p;
  bn = resolve_bn(bn, cin);
  FPVS_CHECK_ARG(bn > 0, "tile width must be 0 (auto), 32, 64, 128 or 256");
  // the forward kernel with Cin' = cout (dz channels), Cout' = cin
  int rc = tc_common(p, dz, lddz, dz_rows, nbr, K, tile_masks, n_dev, cap, w_packed_dgrad, nullptr, cout, cin, bn);
  if (rc) return rc;
  FPVS_CHECK_ARG(dx, "null output");
  FPVS_CHECK_ARG(cin % 32 == 0, "tcgen05 dgrad epilogue needs Cin %% 32 == 0, got %d", cin);
  FPVS_CHECK_ARG(lddx % 8 == 0 && lddx >= cin, "bad dx leading dimension");
  FPVS_CHECK_ARG(!mask || (ldm % 8 == 0 && ldm >= cin), "bad mask leading dimension");
  if (cap <= 0) return FPVS_OK;
  p.act = mask ? FPVS_ACT_MASK : FPVS_ACT_NONE;
  p.mask = (const __nv_bfloat16*)mask;
  p.ldm = ldm;
  p.y = (__nv_bfloat16*)dx;
  p.ldy = lddx;
  p.col_off = 0;
  return tc::dispatch(p, bn, as_stream(stream));
}

extern "C" int fpvs_head_tc(const void* x, int ldx, int x_rows, const int32_t* coords, const int32_t* n_dev, int cap,
                            const void* w_packed, const float* bias, int cin, int d, int B, int Nx, int Ny, int Nz,
                            float tau, uint8_t* out_bits, float* probs, float* logits, void* stream) {
  tc::Params p;
  const int d3 = d * d * d;
  FPVS_CHECK_ARG(d3 <= 256, "head supports d^3 <= 256");
  const int bn = tc::pick_bn(d3);
  int rc = tc_common(p, x, ldx, x_rows, nullptr, 1, nullptr, n_dev, cap, w_packed, bias, cin, d3, bn);
  if (rc) return rc;
  FPVS_CHECK_ARG(coords, "null coords");
  FPVS_CHECK_ARG(Nx % 8 == 0, "N_x must be divisible by 8");
  (void)B;
  if (cap <= 0) return FPVS_OK;
  p.head = 1;
  p.coords = (const int4*)coords;
  p.d = d;
  p.dlog = (d & (d - 1)) == 0 ? __builtin_ctz(d) : -1;
  // logit(tau) for the fast threshold; tau outside (0, 1) takes the sigmoid path
  // tau <= 0: every p >= tau; tau >= 1: the fast path is not taken for a
  // saturating sigmoid (see below), so only the p >= tau form decides there
  p.zt = tau <= 0.f ? -INFINITY : tau >= 1.f ? INFINITY : (float)log((double)tau / (1.0 - (double)tau));
  if (!(tau > 0.f && tau < 1.f)) p.dlog = -1;
  p.Nx = Nx;
  p.Ny = Ny;
  p.Nz = Nz;
  p.tau = tau;
  p.out_bits = out_bits;
  p.probs = probs;
  p.logits = logits;
  return tc::dispatch(p, bn, as_stream(stream));
}
