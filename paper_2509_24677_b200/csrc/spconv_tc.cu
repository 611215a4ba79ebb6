// (3) Sparse convolution on 5th-generation tensor cores (tcgen05, sm_100a).
//
// Implicit gather-GEMM-scatter: for a tile of BM = 128 output rows (active
// cells), the K dimension is the flattened (offset j, channel ci) index
// k = j*Cin + ci of the reference weight rows (neural.py:163-166), cut into
// 64-element (128-byte) chunks.  Per chunk:
//   * A (128 x 64 bf16): 4 producer warps gather 16-byte pieces of the
//     neighbour rows x[nbr[i][j]] with cp.async straight into the 128B-swizzled
//     K-major shared-memory layout the UMMA descriptor expects; a missing
//     neighbour (-1) is a zero-fill (src-size 0).  Each producer thread signals
//     the stage's mbarrier with cp.async.mbarrier.arrive.noinc, so gathers for
//     up to STAGES chunks are in flight per SM.
//   * B (BN x 64 bf16): one bulk copy (TMA engine, cp.async.bulk) of the
//     pre-swizzled weight image produced by fpvs_pack_weights_tc.
//   * one elected thread of the MMA warp issues 4 x tcgen05.mma (M=128, N=BN,
//     K=16, bf16 -> fp32) into a TMEM accumulator; tcgen05.commit frees the
//     stage.  Chunks whose offsets have no neighbour in the whole tile are
//     skipped (per-tile 27-bit offset mask), so sparse tiles do less MMA work.
//   * 4 epilogue warps drain TMEM (tcgen05.ld 32x32b) with a double-buffered
//     accumulator (2 x BN columns) so the epilogue of tile t overlaps the
//     mainloop of tile t+1, fuse bias + ReLU + bf16 cast (or, for the head,
//     sigmoid + [p >= tau] + deinterleave bit-pack), and store.
// The grid is persistent (<= 148 CTAs, 1 per SM) and reads the active row
// count from device memory, so the launch is graph-capturable.
#include "common.cuh"

namespace fpvs {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;            // bf16 elements per chunk = 128 bytes
constexpr int A_BYTES = BM * 128;  // 16 KB
constexpr int kProd = 128;        // producer threads (warps 0-3)
constexpr int kMmaWarp = 8;
constexpr int kThreads = 288;
constexpr int kMaxK = 27;

struct Params {
  const __nv_bfloat16* x;
  int ldx;
  const int* nbr;
  int K;
  const int* n_dev;
  int cap;
  const uint8_t* wpk;
  int nchunks;
  const float* bias;
  int cin, cout, act;
  __nv_bfloat16* y;
  int ldy, col_off;
  // head epilogue
  int head;
  const int4* coords;
  int d, Nx, Ny, Nz;
  float tau;
  uint8_t* out_bits;
  float* probs;
  float* logits;
};

template <int BN>
struct Cfg {
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (192 * 1024) / STAGE_BYTES > 8 ? 8 : (192 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = (2 * BN) <= 32 ? 32 : (2 * BN) <= 64 ? 64 : (2 * BN) <= 128 ? 128 : (2 * BN) <= 256 ? 256 : 512;
  static constexpr int NBR_BYTES = BM * kMaxK * 4;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES + NBR_BYTES;
  static constexpr int SMEM = 1024 + BAR_OFF + 8 * (2 * STAGES + 4) + 16 + 4 * STAGES + 16;
};

// ---------------- PTX wrappers ----------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// SW128 K-major UMMA shared-memory descriptor (cute::UMMA::SmemDescriptor):
// start>>4 [0,14), LBO>>4 [16,30) (unused for SW128 K-major), SBO>>4 [32,46)
// = 1024 B between 8-row core-matrix groups, version 1 [46,48), layout
// SWIZZLE_128B = 2 [61,64).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, N, M=128.
template <int BN>
__device__ __forceinline__ uint32_t idesc_bf16() {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// offsets j covered by chunk c (flattened k = j*cin + ci, 64 per chunk)
__device__ __forceinline__ uint32_t chunk_offset_bits(int c, int cin, int K) {
  int jlo = (c * BK) / cin, jhi = (c * BK + BK - 1) / cin;
  if (jhi > K - 1) jhi = K - 1;
  if (jlo > K - 1) return 0;
  uint32_t hi = (jhi >= 31) ? 0xffffffffu : ((1u << (jhi + 1)) - 1u);
  return hi & ~((1u << jlo) - 1u);
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1) spconv_tc_kernel(const Params p) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * A_BYTES;
  int* s_nbr = reinterpret_cast<int*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tempty + 2);
  uint32_t* s_mask = s_tmem + 1;   // 4 warp masks
  uint32_t* s_info = s_tmem + 8;   // per-stage flags (bit0 first, bit1 last)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = min(*p.n_dev, p.cap);
  const int ntiles = (n + BM - 1) / BM;

  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(smem_u32(full + s), kProd + 1);
      mbar_init(smem_u32(empty + s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(tfull + a), 1);
      mbar_init(smem_u32(tempty + a), 128);
    }
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "n"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *s_tmem;

  if (warp < 4) {
    // ===================== gather producers =====================
    int stage = 0;
    uint32_t phase = 0;
    const int ppo = p.cin >> 3;  // 16-byte pieces per offset
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int row0 = tile * BM;
      named_bar(1, kProd);  // previous tile's readers of s_nbr are done
      for (int e = tid; e < BM * p.K; e += kProd) {
        int r = e / p.K;
        int v = -1;
        if (row0 + r < n) v = p.nbr ? __ldg(p.nbr + (long long)row0 * p.K + e) : row0 + r;
        s_nbr[e] = v;
      }
      named_bar(1, kProd);
      uint32_t m = 0;
      for (int j = 0; j < p.K; ++j) m |= (s_nbr[tid * p.K + j] >= 0 ? 1u : 0u) << j;
      m = __reduce_or_sync(0xffffffffu, m);
      if (lane == 0) s_mask[warp] = m;
      named_bar(1, kProd);
      const uint32_t tmask = s_mask[0] | s_mask[1] | s_mask[2] | s_mask[3];
      int last = -1, first = -1;
      for (int c = 0; c < p.nchunks; ++c)
        if (chunk_offset_bits(c, p.cin, p.K) & tmask) { last = c; if (first < 0) first = c; }
      if (last < 0) { first = 0; last = 0; }  // keep the pipeline shape: one zero chunk
      for (int c = first; c <= last; ++c) {
        if (c != first && c != last && !(chunk_offset_bits(c, p.cin, p.K) & tmask)) continue;
        mbar_wait(smem_u32(empty + stage), phase ^ 1);
        const uint32_t fb = smem_u32(full + stage);
        if (tid == 0) {
          s_info[stage] = (c == first ? 1u : 0u) | (c == last ? 2u : 0u);
          mbar_arrive_expect_tx(fb, C::B_BYTES);
          bulk_g2s(smem_u32(sB + stage * C::B_BYTES), p.wpk + (size_t)c * C::B_BYTES, C::B_BYTES, fb);
        }
        const uint32_t a_base = smem_u32(sA + stage * A_BYTES);
        const int piece = lane & 7;
        const int g = c * 8 + piece;          // global 16B piece index along K
        const int j = g / ppo, ci = (g % ppo) * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = i * 16 + warp * 4 + (lane >> 3);
          int src = (j < p.K) ? s_nbr[r * p.K + j] : -1;
          const __nv_bfloat16* gp = p.x + (src >= 0 ? (long long)src * p.ldx + ci : 0);
          cp_async16(a_base + r * 128 + ((piece ^ (r & 7)) << 4), gp, src >= 0 ? 16u : 0u);
        }
        cp_async_mbar_arrive_noinc(fb);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp < 8) {
    // ===================== epilogue =====================
    const int q = warp & 3;  // TMEM lane quadrant
    const int r = q * 32 + lane;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      mbar_wait(smem_u32(tfull + acc), (it >> 1) & 1);
      tc_fence_after();
      const int row = tile * BM + r;
      const bool valid = row < n;
      int4 cc = make_int4(0, 0, 0, 0);
      if (p.head && valid) cc = p.coords[row];
#pragma unroll 1
      for (int cb = 0; cb < BN; cb += 32) {
        float v[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + cb, v);
        if (!valid || cb >= p.cout) continue;
        if (!p.head) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float z = v[i] + (p.bias ? __ldg(p.bias + cb + i) : 0.f);
            v[i] = p.act == FPVS_ACT_RELU ? fmaxf(z, 0.f) : z;
          }
          uint4* dst = reinterpret_cast<uint4*>(p.y + (long long)row * p.ldy + p.col_off + cb);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(pack_bf16x2(v[8 * i + 0], v[8 * i + 1]), pack_bf16x2(v[8 * i + 2], v[8 * i + 3]),
                                pack_bf16x2(v[8 * i + 4], v[8 * i + 5]), pack_bf16x2(v[8 * i + 6], v[8 * i + 7]));
        } else {
          const int d = p.d;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int k = cb + i;
            if (k >= p.cout) continue;
            float z = v[i] + (p.bias ? __ldg(p.bias + k) : 0.f);
            float pr = sigmoidf_stable(z);
            if (p.logits) p.logits[(long long)row * p.cout + k] = z;
            if (p.probs) p.probs[(long long)row * p.cout + k] = pr;
            if (pr >= p.tau && p.out_bits) {
              int lx = k % d, ly = (k / d) % d, lz = k / (d * d);
              int fx = cc.y * d + lx;
              atomic_or_bit(p.out_bits, bit_byte(cc.x, fx, cc.z * d + ly, cc.w * d + lz, p.Nx, p.Ny, p.Nz), fx & 7);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(smem_u32(tempty + acc));
    }
  } else {
    // ===================== MMA issuer (warp 8) =====================
    const uint32_t idesc = idesc_bf16<BN>();
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      mbar_wait(smem_u32(tempty + acc), ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dtm = tmem_base + acc * BN;
      while (true) {
        mbar_wait(smem_u32(full + stage), phase);
        tc_fence_after();
        fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tcgen05 (async proxy) reads
        const uint32_t info = s_info[stage];
        if (lane == 0) {
          const uint64_t ad = sw128_desc(smem_u32(sA + stage * A_BYTES));
          const uint64_t bd = sw128_desc(smem_u32(sB + stage * C::B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16(dtm, ad + 2 * k, bd + 2 * k, idesc, ((info & 1u) && k == 0) ? 0u : 1u);
          umma_commit(smem_u32(empty + stage));
          if (info & 2u) umma_commit(smem_u32(tfull + acc));
        }
        __syncwarp();
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        if (info & 2u) break;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(C::TMEM_COLS)
                 : "memory");
  }
}

// packed[c][n][128 B] for n < BN: element kk of chunk c at
// n*128 + ((kk/8) ^ (n%8))*16 + (kk%8)*2 (Swizzle<3,4,3>), value W[c*64+kk][n]
__global__ void pack_weights_kernel(const float* __restrict__ w, int Ktot, int cout, int BN, int nchunks,
                                    __nv_bfloat16* __restrict__ out) {
  const long long total = (long long)nchunks * BN * BK;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int kk = t % BK;
    long long r = t / BK;
    int nn = r % BN;
    int c = (int)(r / BN);
    int k = c * BK + kk;
    float v = (k < Ktot && nn < cout) ? w[(long long)k * cout + nn] : 0.f;
    long long byte = ((long long)c * BN + nn) * 128 + (((kk >> 3) ^ (nn & 7)) << 4) + (kk & 7) * 2;
    out[byte / 2] = __float2bfloat16_rn(v);
  }
}

inline int pick_bn(int cout) {
  if (cout <= 32) return 32;
  if (cout <= 64) return 64;
  if (cout <= 128) return 128;
  if (cout <= 256) return 256;
  return -1;
}

template <int BN>
int launch(const Params& p, cudaStream_t s) {
  using C = Cfg<BN>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(spconv_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return set_error(FPVS_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    configured = true;
  }
  int tiles = (p.cap + BM - 1) / BM;
  int grid = tiles < kNumSMs ? tiles : kNumSMs;
  if (grid < 1) grid = 1;
  spconv_tc_kernel<BN><<<grid, kThreads, C::SMEM, s>>>(p);
  FPVS_CHECK_LAUNCH("spconv_tc");
  return FPVS_OK;
}

int dispatch(Params& p, cudaStream_t s) {
  switch (pick_bn(p.cout)) {
    case 32: return launch<32>(p, s);
    case 64: return launch<64>(p, s);
    case 128: return launch<128>(p, s);
    case 256: return launch<256>(p, s);
  }
  return set_error(FPVS_EINVAL, "Cout %d > 256 not supported by the tcgen05 path", p.cout);
}

}  // namespace tc
}  // namespace fpvs

using namespace fpvs;

extern "C" size_t fpvs_pack_weights_tc_size(int K, int cin, int cout) {
  int bn = tc::pick_bn(cout);
  if (bn < 0 || K < 1 || cin < 1) return 0;
  size_t nchunks = ((size_t)K * cin + tc::BK - 1) / tc::BK;
  return nchunks * bn * 128;
}

extern "C" int fpvs_pack_weights_tc(const float* w, int K, int cin, int cout, void* packed, void* stream) {
  FPVS_CHECK_ARG(w && packed, "null pointer");
  int bn = tc::pick_bn(cout);
  FPVS_CHECK_ARG(bn > 0, "Cout %d > 256 not supported by the tcgen05 path", cout);
  FPVS_CHECK_ARG(cin % 8 == 0, "tcgen05 path needs Cin %% 8 == 0, got %d", cin);
  int nchunks = (K * cin + tc::BK - 1) / tc::BK;
  long long total = (long long)nchunks * bn * tc::BK;
  tc::pack_weights_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(w, K * cin, cout, bn, nchunks,
                                                                              (__nv_bfloat16*)packed);
  FPVS_CHECK_LAUNCH("fpvs_pack_weights_tc");
  return FPVS_OK;
}

static int tc_common(tc::Params& p, const void* x, int ldx, const int32_t* nbr, int K, const int32_t* n_dev, int cap,
                     const void* w_packed, const float* bias, int cin, int cout) {
  FPVS_CHECK_ARG(x && w_packed && n_dev, "null pointer");
  FPVS_CHECK_ARG(K >= 1 && K <= tc::kMaxK, "K must lie in [1, 27]");
  FPVS_CHECK_ARG(nbr || K == 1, "nbr may be NULL only for K == 1");
  FPVS_CHECK_ARG(cin % 8 == 0 && ldx % 8 == 0, "tcgen05 path needs Cin and ldx multiples of 8");
  FPVS_CHECK_ARG(tc::pick_bn(cout) > 0, "Cout %d > 256 not supported", cout);
  p = tc::Params{};
  p.x = (const __nv_bfloat16*)x;
  p.ldx = ldx;
  p.nbr = nbr;
  p.K = K;
  p.n_dev = n_dev;
  p.cap = cap;
  p.wpk = (const uint8_t*)w_packed;
  p.nchunks = (K * cin + tc::BK - 1) / tc::BK;
  p.bias = bias;
  p.cin = cin;
  p.cout = cout;
  return FPVS_OK;
}

extern "C" int fpvs_spconv_tc(const void* x, int ldx, const int32_t* nbr, int K, const int32_t* n_out_dev,
                              int cap_out, const void* w_packed, const float* bias, int cin, int cout, int act, void* y,
                              int ldy, int col_off, void* stream) {
  tc::Params p;
  int rc = tc_common(p, x, ldx, nbr, K, n_out_dev, cap_out, w_packed, bias, cin, cout);
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
  return tc::dispatch(p, as_stream(stream));
}

extern "C" int fpvs_head_tc(const void* x, int ldx, const int32_t* coords, const int32_t* n_dev, int cap,
                            const void* w_packed, const float* bias, int cin, int d, int B, int Nx, int Ny, int Nz,
                            float tau, uint8_t* out_bits, float* probs, float* logits, void* stream) {
  tc::Params p;
  const int d3 = d * d * d;
  int rc = tc_common(p, x, ldx, nullptr, 1, n_dev, cap, w_packed, bias, cin, d3);
  if (rc) return rc;
  FPVS_CHECK_ARG(coords, "null coords");
  FPVS_CHECK_ARG(Nx % 8 == 0, "N_x must be divisible by 8");
  (void)B;
  if (cap <= 0) return FPVS_OK;
  p.head = 1;
  p.coords = (const int4*)coords;
  p.d = d;
  p.Nx = Nx;
  p.Ny = Ny;
  p.Nz = Nz;
  p.tau = tau;
  p.out_bits = out_bits;
  p.probs = probs;
  p.logits = logits;
  return tc::dispatch(p, as_stream(stream));
}
