// (4) Weight gradient of a 27-tap submanifold conv with Cin = 32, halo-cached.
//
// Same GEMM as wgrad_tc.cu (neural.py:238-239 on the active set):
//   dW[j*32 + ci][co] = sum_i x[nbr[i][j]][ci] * dz[i][co],  db[co] = sum_i dz[i][co]
// i.e. D[M = (j, ci)][N = co] = sum_k A[m][k] B[k][n] with the active row
// index as the reduction dimension.  wgrad_tc.cu gathers every (row, offset)
// piece of A from global memory: 27 x 64 B per row through the L1/LSU, which
// is what bounds it.  Here a CTA walks whole 128-row tiles of the level and,
// per tile, copies the tile's HALO once (the distinct neighbour rows,
// fpvs_kmap_halo: ~3-4 x 128 rows instead of 27 x 128) into shared memory;
// the A operands of all 27 offsets are then built from that copy
// (shared -> shared), so global traffic drops ~8x and the LSU stops being
// the bound.  All seven (j, ci) blocks of 128 (offsets 4b..4b+3) accumulate
// in TMEM at once (7 x 32 fp32 columns), and one dz chunk (B) feeds all seven.
//
//   warps 0-7  A producers: per stage (64 rows x one (j, ci) block) 1024
//              16-byte pieces, halo -> no-swizzle MN-major A layout
//   warps 8,10,11 loaders: per tile the local table + halo row list (bulk
//              copies), the halo rows and the tile's dz rows (cp.async)
//   warp 9     MMA issuer (one lane): 4 x kind::f16 M=128 N=32 K=16 per stage
//   warps 8-11 epilogue after the loop: TMEM -> fp32 partial per CTA
// A second kernel sums the CTA partials in a fixed order (deterministic).
// The spare fourth offset of block 6 (m = 864..895) carries an all-ones row
// at m = 864, so D row 864 is db.
#include <stdlib.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace fpvs {
namespace wgh {

using namespace tc;

constexpr int CIN = 32;
constexpr int KOFF = 27;
constexpr int NMB = 7;           // (j, ci) blocks of 128
constexpr int RT = 128;          // rows per tile (the halo table's tile)
constexpr int KC = 128;          // rows per A stage (the whole tile)
constexpr int NS = 3;            // A stages
constexpr int NPAD = 32;         // MMA N
constexpr int HMAX = FPVS_HALO_MAX;
constexpr int SBO = (KC / 8) * 128;          // MN-direction core-matrix stride
constexpr int A_STAGE = 16 * SBO;            // 128 m x 128 rows x 2 B
constexpr int B_CHUNK = (NPAD / 8) * SBO;    // 128 rows x 32 co x 2 B, MN-major
constexpr int HALO_BYTES = HMAX * 64;       // 32 channels per halo row
constexpr int LNBR_BYTES = RT * KOFF * 2;   // int16 [128][27]
constexpr int HB_LNBR = HALO_BYTES;
constexpr int HB_ROWS = HB_LNBR + ((LNBR_BYTES + 127) & ~127);
constexpr int HB_LNT = HB_ROWS + HMAX * 4;               // the local table transposed: int16 [27][128]
constexpr int HB_B = HB_LNT + ((LNBR_BYTES + 127) & ~127);  // the tile's dz rows
constexpr int HBUF = (HB_B + B_CHUNK + 1023) & ~1023;
constexpr int NHB = 2;
constexpr int THREADS = 384;
constexpr int PROD = 256;
constexpr int W_LOAD = 8, W_MMA = 9;  // loaders: warps 8, 10, 11
constexpr int LOADERS = 96;
constexpr int SMEM = 1024 + NS * A_STAGE + NHB * HBUF + 256;
static_assert(SMEM <= 232448, "shared memory budget");

struct Params {
  const __nv_bfloat16* x;
  int ldx;
  const __nv_bfloat16* dz;
  int lddz;
  const int* nbr;
  const int* n_dev;
  int cap;
  const int* halo_rows;
  const int* halo_n;
  const int16_t* lnbr;
  int cout;
  float* part;  // [grid][NMB][128][NPAD]
  int dbg;      // FPVS_WGRAD_DEBUG (profiling only): 1 no A loads, 2 no MMA, 8 no halo / dz copies
};

__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr) {
  // no-swizzle canonical layout: LBO = 128 B (K direction), SBO (MN direction)
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(SBO >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__global__ void __launch_bounds__(THREADS, 1) wgrad_halo_kernel(const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* sA = smem;
  uint8_t* sH = smem + NS * A_STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sH + NHB * HBUF);
  uint64_t* full = bars;             // [NS] producers -> MMA
  uint64_t* empty = bars + NS;       // [NS] MMA commit -> producers
  uint64_t* hmeta = bars + 2 * NS;   // [NHB] table + row list landed
  uint64_t* hfull = hmeta + NHB;     // [NHB] halo rows + dz landed
  uint64_t* hempty = hfull + NHB;    // [NHB] producers + MMA done with the buffer
  uint64_t* tfull = hempty + NHB;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tfull + 1);
  uint32_t* s_const = reinterpret_cast<uint32_t*>(tfull + 4);  // 16 B zeros, 16 B {bf16 1.0, 0...}

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = min(*p.n_dev, p.cap);
  const int tiles = (n + RT - 1) / RT;
  const int t0 = (int)((long long)blockIdx.x * tiles / gridDim.x);
  const int t1 = (int)((long long)(blockIdx.x + 1) * tiles / gridDim.x);

  if (tid < 8) s_const[tid] = tid == 4 ? 0x3F80u : 0u;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(smem_u32(full + s), PROD / 32);
      mbar_init(smem_u32(empty + s), 1);
    }
    for (int b = 0; b < NHB; ++b) {
      mbar_init(smem_u32(hmeta + b), 1);
      mbar_init(smem_u32(hfull + b), LOADERS);
      mbar_init(smem_u32(hempty + b), PROD / 32 + 1);
    }
    mbar_init(smem_u32(tfull), 1);
    fence_mbar_init();
  }
  if (warp == W_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(s_tmem))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp < W_LOAD) {
    // ===================== A producers =====================
    // piece q (8 per thread): 16-byte column mg = 4 * local offset + channel
    // quarter pc, of row kk.  8 consecutive lanes take 8 consecutive rows of
    // one column, so every store fills a whole 128-byte core-matrix row
    // (conflict-free); the halo rows they read are XOR-swizzled by row so the
    // 8 loads of a quarter-warp spread over the banks; the tile's local table
    // is first transposed to [offset][row] so the index loads of consecutive
    // rows are consecutive.  All pieces' loads are issued before any store.
    pdl_wait();
    constexpr int PPT = KC * 16 / PROD;  // pieces per thread per stage
    const int mg = (tid >> 3) & 15;      // the same column for all of a thread's pieces
    const int pc = mg & 3;
    int a_kk[PPT];
    uint32_t a_dst[PPT];
#pragma unroll
    for (int t = 0; t < PPT; ++t) {
      const int q = tid + PROD * t;
      const int kk = ((q >> 7) << 3) | (q & 7);
      a_kk[t] = kk;
      a_dst[t] = mg * SBO + (kk >> 3) * 128 + (kk & 7) * 16;
    }
    const uint32_t ldx2 = (uint32_t)p.ldx * 2u;
    const uint32_t zero_a = smem_u32(s_const), ones_a = zero_a + 16;
    const uint32_t sA_a = smem_u32(sA), sH_a = smem_u32(sH);
    const uint32_t full_a = smem_u32(full), empty_a = smem_u32(empty), hfull_a = smem_u32(hfull),
                   hempty_a = smem_u32(hempty);
    uint32_t st = 0;
    int gc = 0;
    for (int tile = t0; tile < t1; ++tile, ++gc) {
      const int hb = gc % NHB;
      const uint32_t hph = (gc / NHB) & 1;
      mbar_wait(hfull_a + 8 * hb, hph);
      uint8_t* hbuf = sH + hb * HBUF;
      const uint32_t hbuf_a = sH_a + hb * HBUF;
      const int16_t* ln = reinterpret_cast<const int16_t*>(hbuf + HB_LNBR);
      int16_t* lt = reinterpret_cast<int16_t*>(hbuf + HB_LNT);
      const int nt = n - tile * RT;  // valid rows of this tile
      {
        const int r = tid & (RT - 1), jh = tid >> 7;  // two threads per row: offsets 0-13 and 14-26
        const bool ok = r < nt;
#pragma unroll
        for (int jj = 0; jj < 14; ++jj) {
          const int j = jh * 14 + jj;
          if (j < KOFF) lt[j * RT + r] = ok ? ln[r * KOFF + j] : (int16_t)-1;
        }
      }
      named_bar(1, PROD);
      for (int mb = 0; mb < NMB; ++mb, ++st) {
        const int stage = (int)(st % NS);
        const int j = mb * 4 + (mg >> 2);
        // source address per piece: a halo row, the zero block, or the ones block
        // (the db row); -2 = halo overflow, fixed up below from global memory
        int li[PPT];
        if (j < KOFF) {
#pragma unroll
          for (int t = 0; t < PPT; ++t) li[t] = lt[j * RT + a_kk[t]];
        } else {
#pragma unroll
          for (int t = 0; t < PPT; ++t) li[t] = (j == KOFF && pc == 0 && a_kk[t] < nt) ? -3 : -1;
        }
        uint4 v[PPT];
        bool slow = false;
#pragma unroll
        for (int t = 0; t < PPT; ++t) {
          const int l = li[t];
          const uint32_t a = l >= 0 ? hbuf_a + l * 64 + ((pc ^ (l & 3)) << 4) : (l == -3 ? ones_a : zero_a);
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v[t].x), "=r"(v[t].y), "=r"(v[t].z), "=r"(v[t].w)
                       : "r"(a));
          slow |= l == -2;
        }
        if (slow) {
#pragma unroll
          for (int t = 0; t < PPT; ++t) {
            if (li[t] != -2) continue;
            const int g = __ldg(p.nbr + (long long)(tile * RT + a_kk[t]) * KOFF + j);
            v[t] = g >= 0 ? __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(p.x) +
                                                                 (long long)g * ldx2) + pc)
                          : make_uint4(0u, 0u, 0u, 0u);
          }
        }
        if (FPVS_KNOB(p) & 1) {
#pragma unroll
          for (int t = 0; t < PPT; ++t) v[t] = make_uint4(0u, 0u, 0u, 0u);
        }
        mbar_wait(empty_a + 8 * stage, ((st / NS) & 1) ^ 1);
        const uint32_t a_st = sA_a + stage * A_STAGE;
#pragma unroll
        for (int t = 0; t < PPT; ++t)
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a_st + a_dst[t]), "r"(v[t].x), "r"(v[t].y),
                       "r"(v[t].z), "r"(v[t].w)
                       : "memory");
        fence_proxy_async_smem();  // generic-proxy stores -> tensor-core reads
        __syncwarp();
        if (lane == 0) mbar_arrive(full_a + 8 * stage);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(hempty_a + 8 * hb);
    }
    if (tid == 0) pdl_trigger();
  } else if (warp != W_MMA) {
    // ===================== loaders (warps 8, 10, 11) =====================
    pdl_wait();
    const int lt = (warp == W_LOAD ? 0 : warp - W_MMA) * 32 + lane;  // 0..95
    const uint32_t ldx2 = (uint32_t)p.ldx * 2u, lddz2 = (uint32_t)p.lddz * 2u;
    const char* xg = reinterpret_cast<const char*>(p.x);
    const char* dg = reinterpret_cast<const char*>(p.dz);
    int gc = 0;
    for (int tile = t0; tile < t1; ++tile, ++gc) {
      const int hb = gc % NHB;
      const uint32_t hph = (gc / NHB) & 1;
      mbar_wait_sleep(smem_u32(hempty + hb), hph ^ 1, 32);
      uint8_t* hbuf = sH + hb * HBUF;
      const int H = min(__ldg(p.halo_n + tile), HMAX);
      if (lt == 0) {
        const uint32_t rb = (uint32_t)((H * 4 + 15) & ~15);
        const uint32_t mb = smem_u32(hmeta + hb);
        mbar_arrive_expect_tx(mb, LNBR_BYTES + rb);
        bulk_g2s(smem_u32(hbuf + HB_LNBR), p.lnbr + (long long)tile * RT * KOFF, LNBR_BYTES, mb);
        if (rb) bulk_g2s(smem_u32(hbuf + HB_ROWS), p.halo_rows + (long long)tile * HMAX, rb, mb);
      }
      mbar_wait(smem_u32(hmeta + hb), hph);
      const int* hr = reinterpret_cast<const int*>(hbuf + HB_ROWS);
      const uint32_t hs = smem_u32(hbuf);
      for (int q = lt; q < ((FPVS_KNOB(p) & 8) ? 0 : H * 4); q += LOADERS) {
        const int i = q >> 2, pc = q & 3;
        cp_async16(hs + i * 64 + ((pc ^ (i & 3)) << 4), xg + (long long)hr[i] * ldx2 + pc * 16, 16);
      }
      // the tile's dz rows: two 64-row chunks, MN-major (rows past n and
      // channels past Cout are zero-filled)
      const uint32_t bs = smem_u32(hbuf + HB_B);
      for (int q = lt; q < RT * (NPAD / 8); q += LOADERS) {
        const int kk = q / (NPAD / 8), ng = q - kk * (NPAD / 8);
        const int row = tile * RT + kk;
        const bool ok = row < n && ng * 8 < p.cout;
        const uint32_t dst = bs + ng * SBO + (kk >> 3) * 128 + (kk & 7) * 16;
        cp_async16(dst, dg + (ok ? (long long)row * lddz2 + ng * 16 : 0), ok ? 16u : 0u);
      }
      cp_async_mbar_arrive_noinc(smem_u32(hfull + hb));
    }
  } else if (warp == W_MMA) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                             ((uint32_t)(NPAD >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      uint32_t st = 0;
      int gc = 0;
      unsigned started = 0;
      for (int tile = t0; tile < t1; ++tile, ++gc) {
        const int hb = gc % NHB;
        const uint32_t hph = (gc / NHB) & 1;
        mbar_wait(smem_u32(hfull + hb), hph);  // dz chunks (B) of this tile
        const uint32_t bs = smem_u32(sH + hb * HBUF + HB_B);
        for (int mb = 0; mb < NMB; ++mb, ++st) {
          const int stage = (int)(st % NS);
          mbar_wait(smem_u32(full + stage), (st / NS) & 1);
          tc_fence_after();
          fence_proxy_async_smem();  // cp.async (generic proxy) dz writes -> tensor-core reads
          const uint32_t a_st = smem_u32(sA + stage * A_STAGE);
          const uint32_t acc = tmem + mb * NPAD;
#pragma unroll
          for (int kk = 0; kk < KC / 16; ++kk) {
            const uint32_t accumulate = ((started >> mb) & 1u) | (kk ? 1u : 0u);
            if (!(FPVS_KNOB(p) & 2)) umma_bf16(acc, desc_mn(a_st + kk * 256), desc_mn(bs + kk * 256), idesc, accumulate);
          }
          started |= 1u << mb;
          umma_commit(smem_u32(empty + stage));
        }
        umma_commit(smem_u32(hempty + hb));  // the tile's dz chunks are no longer read
      }
      umma_commit(smem_u32(tfull));
    }
  }
  // ===================== epilogue (warps 8-11): TMEM -> fp32 partial =====================
  if (warp >= W_LOAD) {
    pdl_wait();
    const int q4 = warp & 3, r = q4 * 32 + lane;
    mbar_wait_sleep(smem_u32(tfull), 0, 128);
    tc_fence_after();
    const bool has = t1 > t0;
#pragma unroll 1
    for (int mb = 0; mb < NMB; ++mb) {
      float* dst = p.part + (((long long)blockIdx.x * NMB + mb) * BM + r) * NPAD;
#pragma unroll 1
      for (int cb = 0; cb < NPAD; cb += 8) {
        float v[8];
        tmem_ld8(tmem + ((uint32_t)(q4 * 32) << 16) + mb * NPAD + cb, v);
        float4* d4 = reinterpret_cast<float4*>(dst + cb);
        d4[0] = has ? make_float4(v[0], v[1], v[2], v[3]) : make_float4(0.f, 0.f, 0.f, 0.f);
        d4[1] = has ? make_float4(v[4], v[5], v[6], v[7]) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

// dw[f][co] = sum over CTAs of part[c][f / 128][f % 128][co] in a fixed order
// (eight interleaved partial sums, then those in order); row f = 864 is db.
// One block per row f: 32 channels x 8 partial lanes.
__global__ void __launch_bounds__(256) wgrad_halo_reduce_kernel(const float* __restrict__ part, int nparts, int cout,
                                                                float* __restrict__ dw, float* __restrict__ db) {
  __shared__ float acc[8][NPAD];
  const int f = blockIdx.x, co = threadIdx.x & 31, cl = threadIdx.x >> 5;
  const float* src = part + ((long long)(f >> 7) * BM + (f & 127)) * NPAD + co;
  float s = 0.f;
  for (int c = cl; c < nparts; c += 8) s += __ldg(src + (long long)c * NMB * BM * NPAD);
  acc[cl][co] = s;
  __syncthreads();
  if (cl == 0 && co < cout) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += acc[k][co];
    if (f < KOFF * CIN) dw[(long long)f * cout + co] = t;
    else if (db) db[co] = t;
  }
}

}  // namespace wgh
}  // namespace fpvs

using namespace fpvs;

extern "C" size_t fpvs_wgrad_halo_workspace_size(int cap) {
  if (cap < 1) return 0;
  return (size_t)kNumSMs * wgh::NMB * tc::BM * wgh::NPAD * 4;
}

extern "C" int fpvs_spconv_wgrad_halo(const void* x, int ldx, const void* dz, int lddz, const int32_t* nbr,
                                      const int32_t* n_dev, int cap, const int32_t* halo_rows,
                                      const int32_t* halo_n, const int16_t* lnbr, int cin, int cout, float* dw,
                                      float* db, void* workspace, size_t workspace_bytes, void* stream) {
  FPVS_CHECK_ARG(x && dz && nbr && n_dev && halo_rows && halo_n && lnbr && dw && workspace, "null pointer");
  FPVS_CHECK_ARG(cin == wgh::CIN, "halo wgrad takes Cin = 32, got %d", cin);
  FPVS_CHECK_ARG(cout >= 8 && cout <= wgh::NPAD && cout % 8 == 0, "halo wgrad takes Cout in {8..32} step 8");
  FPVS_CHECK_ARG(ldx % 8 == 0 && ldx >= cin && lddz % 8 == 0 && lddz >= cout, "row strides must be multiples of 8");
  FPVS_CHECK_ARG(workspace_bytes >= fpvs_wgrad_halo_workspace_size(cap), "workspace too small");
  if (cap <= 0) return FPVS_OK;
  {
    const cudaError_t e = set_smem_once<wgh::wgrad_halo_kernel>(wgh::SMEM);
    if (e != cudaSuccess) return set_error(FPVS_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  wgh::Params p{};
  p.x = (const __nv_bfloat16*)x;
  p.ldx = ldx;
  p.dz = (const __nv_bfloat16*)dz;
  p.lddz = lddz;
  p.nbr = nbr;
  p.n_dev = n_dev;
  p.cap = cap;
  p.halo_rows = halo_rows;
  p.halo_n = halo_n;
  p.lnbr = lnbr;
  p.cout = cout;
  p.part = (float*)workspace;
  p.dbg = debug_knob("FPVS_WGRAD_DEBUG");
  cudaStream_t s = as_stream(stream);
  const int grid = kNumSMs;
  cudaError_t e = launch_kernel(wgh::wgrad_halo_kernel, dim3(grid), dim3(wgh::THREADS), wgh::SMEM, s, p);
  if (e != cudaSuccess) return set_error(FPVS_ECUDA, "wgrad_halo: %s", cudaGetErrorString(e));
  wgh::wgrad_halo_reduce_kernel<<<wgh::KOFF * wgh::CIN + (db ? 1 : 0), 256, 0, s>>>(p.part, grid, cout, dw, db);
  FPVS_CHECK_LAUNCH("fpvs_spconv_wgrad_halo");
  return FPVS_OK;
}
