// (4) Weight gradient of the sparse convolution on tcgen05 tensor cores.
//
// Replaces Conv3d.backward's dW = colsᵀ·dz and db = Σ dz (neural.py:238-239)
// on the active set: dW[j*Cin + ci][co] = Σ_i x[nbr[i][j]][ci] · dz[i][co].
// As a GEMM the reduction dimension is the active-row index i:
//   D[M = (j, ci)][N = co] = Σ_k A[m][k] · B[k][n],  A[m][k] = x[nbr[k][j]][ci],
//   B[k][n] = dz[k][n].
// Both operands are MN-major: for a fixed row k the 8 consecutive channels of
// one neighbour (A) or of dz (B) are one contiguous 16-byte piece, gathered
// with cp.async into the no-swizzle canonical layout (core matrix = 8 k-rows
// x 16 B; element (mn, k) at (mn/8)*1024 + (k/8)*128 + (k%8)*16 + (mn%8)*2
// for a 64-row K chunk; layout checked on B200 in tools/micro_mn.cu).
// A work unit = one 128-row block of the flattened (j, ci) index x one range
// of 64-row K chunks; each unit accumulates in TMEM and writes an fp32
// partial; a second kernel sums the partials of each block in a fixed order
// (deterministic, no float atomics), and a third the bias gradient.
#include <stdlib.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace fpvs {
namespace wg {

using namespace tc;

constexpr int KC = 64;          // rows of the reduction per pipeline stage
constexpr int NS = 4;           // stages
constexpr int A_STAGE = 16384;  // 128 (j, ci) x 64 rows x 2 B
constexpr int THREADS = 384;    // warps 0-7 producers, warp 8 MMA, warps 8-11 epilogue
constexpr int PROD = 256;
constexpr int W_MMA = PROD / 32;
constexpr int APT = KC * 16 / PROD;  // A pieces per producer thread per chunk

#ifdef FPVS_PROFILE
__device__ unsigned long long g_wts[4096];  // FPVS_WGRAD_DEBUG & 32: CTA 0 timestamps
__device__ __forceinline__ void wts(const int dbg, int slot) {
  if ((dbg & 32) && blockIdx.x == 0 && slot < 4096) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_wts[slot] = t;
  }
}
#else
__device__ __forceinline__ void wts(const int, int) {}
#endif

struct Params {
  const __nv_bfloat16* x;
  int ldx;
  const __nv_bfloat16* dz;
  int lddz;
  const int* nbr;  // NULL: K = 1, row i reads itself
  int K;
  const int* n_dev;
  int cap;
  int cin, cout, npad;  // npad: MMA N (cout rounded up to 16)
  int nmb, nsplit;      // (j, ci) blocks of 128, K-chunk ranges per block
  float* part;          // [nmb][nsplit][128][npad]
  int dbg;              // FPVS_WGRAD_DEBUG (profiling only): 1 no A copies, 2 no MMA, 4 no nbr loads
};

__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr) {
  // no-swizzle canonical layout: LBO = 128 B (K direction), SBO = 1024 B (MN direction)
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

template <int NPAD>
__global__ void __launch_bounds__(THREADS, 1) wgrad_tc_kernel(const Params p) {
  constexpr int B_STAGE = (NPAD / 8) * 1024;
  constexpr int TCOLS = NPAD <= 32 ? 32 : NPAD <= 64 ? 64 : NPAD <= 128 ? 128 : 256;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* sA = smem;
  uint8_t* sB = smem + NS * A_STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + NS * B_STAGE);
  uint64_t* full = bars;
  uint64_t* empty = bars + NS;
  uint64_t* tfull = bars + 2 * NS;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tfull + 1);
  int* s_nb = reinterpret_cast<int*>(smem + NS * (A_STAGE + B_STAGE) + 1024);  // [64][32] chunk neighbour rows

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mb = blockIdx.x / p.nsplit, rs = blockIdx.x - mb * p.nsplit;
  const int n = min(*p.n_dev, p.cap);
  const int nchunks = (n + KC - 1) / KC;
  const int c0 = (int)((long long)rs * nchunks / p.nsplit), c1 = (int)((long long)(rs + 1) * nchunks / p.nsplit);
  const int kcin = p.K * p.cin;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(smem_u32(full + s), PROD);
      mbar_init(smem_u32(empty + s), 1);
    }
    mbar_init(smem_u32(tfull), 1);
    fence_mbar_init();
  }
  if (warp == W_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "n"(TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp < W_MMA) {
    // ===================== producers: gather A pieces, load B pieces =====================
    // The chunk's neighbour indices of this block's offsets are first loaded
    // (independent, coalesced) into smem, so the cp.async gather issues without
    // dependent global latency; 8 consecutive lanes fill one 128-byte core
    // matrix (8 rows of one 16-byte column), so the smem writes do not conflict.
    pdl_wait();
    const uint32_t ldx2 = (uint32_t)p.ldx * 2u, lddz2 = (uint32_t)p.lddz * 2u;
    const int jlo = (mb * 128) / p.cin;
    const int jn = min(p.K, (mb * 128 + 127) / p.cin + 1) - jlo;  // offsets touched by this block
    const int fones = (kcin % 128) ? kcin : -1;  // padding row used for db (sum of dz)
    // Per-thread piece geometry is the same for every chunk: precomputed once.
    // A: pieces q = tid + PROD t (t < APT): core row kk, 16-byte column mg.
    int a_row[APT], a_nb[APT], a_cof[APT];
    uint32_t a_dst[APT];
#pragma unroll
    for (int t = 0; t < APT; ++t) {
      const int q = tid + PROD * t;
      // 4 consecutive lanes read one row's 4 consecutive 16-byte pieces (64 B
      // coalesced); a warp covers 8 rows; its smem writes are 4 x 128 B
      const int mg = ((q >> 5) & 3) * 4 + (q & 3), kk = ((q >> 7) << 3) | ((q >> 2) & 7);
      const int f = mb * 128 + mg * 8;
      a_row[t] = kk;
      a_dst[t] = mg * 1024 + (kk >> 3) * 128 + (kk & 7) * 16;
      a_nb[t] = f == fones ? -2 : f < kcin ? kk * 32 + (f / p.cin - jlo) : -1;  // s_nb slot, -1 zero, -2 ones
      a_cof[t] = (f % p.cin) * 2;
    }
    // B: pieces q = tid + PROD t
    constexpr int NBP = (KC * (NPAD / 8) + PROD - 1) / PROD;
    int b_row[NBP];
    uint32_t b_dst[NBP], b_off[NBP];
    bool b_ok[NBP];
#pragma unroll
    for (int t = 0; t < NBP; ++t) {
      const int q = tid + PROD * t;
      const int ng = q % (NPAD / 8), kk = q / (NPAD / 8);  // a row's pieces on consecutive lanes
      b_row[t] = kk;
      b_dst[t] = ng * 1024 + (kk >> 3) * 128 + (kk & 7) * 16;
      b_off[t] = ng * 16;
      b_ok[t] = q < KC * (NPAD / 8) && ng * 8 < p.cout;
    }
    // neighbour indices of the block's offsets, loaded one chunk ahead (jn <= 16)
    constexpr int NPT = KC * 16 / PROD;
    int n_slot[NPT], n_row[NPT], n_j[NPT];
#pragma unroll
    for (int t = 0; t < NPT; ++t) {
      const int q = tid + PROD * t;
      const int kk = q / jn, jj = q - kk * jn;
      n_slot[t] = q < KC * jn ? kk * 32 + jj : -1;
      n_row[t] = kk;
      n_j[t] = jlo + jj;
    }
    int pre[NPT];
    auto prefetch = [&](int c) {
#pragma unroll
      for (int t = 0; t < NPT; ++t) {
        const int i = c * KC + n_row[t];
        pre[t] = -1;
        if (n_slot[t] >= 0 && i < n) pre[t] = (p.nbr && !(FPVS_KNOB(p) & 4)) ? __ldg(p.nbr + (long long)i * p.K + n_j[t]) : i;
      }
    };
    const char* xg = reinterpret_cast<const char*>(p.x);
    const char* dg = reinterpret_cast<const char*>(p.dz);
    if (c0 < c1) prefetch(c0);
    for (int c = c0; c < c1; ++c) {
      const int k = c - c0, stage = k % NS;
      const int i0 = c * KC;
      if (tid == 0) wts(FPVS_KNOB(p), 8 * k);
      named_bar(2, PROD);  // previous chunk's readers are done with s_nb
#pragma unroll
      for (int t = 0; t < NPT; ++t)
        if (n_slot[t] >= 0) s_nb[n_slot[t]] = pre[t];
      named_bar(2, PROD);
      if (tid == 0) wts(FPVS_KNOB(p), 8 * k + 1);
      if (c + 1 < c1) prefetch(c + 1);  // in flight while this chunk's copies issue
      mbar_wait_sleep(smem_u32(empty + stage), ((k / NS) & 1) ^ 1, 32);
      if (tid == 0) wts(FPVS_KNOB(p), 8 * k + 2);
      const uint32_t a_st = smem_u32(sA + stage * A_STAGE), b_st = smem_u32(sB + stage * B_STAGE);
#pragma unroll
      for (int t = 0; t < APT; ++t) {
        const uint32_t dst = a_st + a_dst[t];
        if (a_nb[t] == -2) {
          // db row: 1.0 in the first element for valid rows
          const uint32_t one = (i0 + a_row[t] < n) ? 0x3F80u : 0u;
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(one), "r"(0u), "r"(0u), "r"(0u)
                       : "memory");
          continue;
        }
        const int src = a_nb[t] >= 0 ? s_nb[a_nb[t]] : -1;
        const char* g = xg + (src >= 0 ? (long long)src * ldx2 + a_cof[t] : 0);
        if (!(FPVS_KNOB(p) & 1)) cp_async16(dst, g, src >= 0 ? 16u : 0u);
      }
#pragma unroll
      for (int t = 0; t < NBP; ++t) {
        const int i = i0 + b_row[t];
        const bool ok = b_ok[t] && i < n;
        const char* g = dg + (ok ? (long long)i * lddz2 + b_off[t] : 0);
        if (tid + PROD * t < KC * (NPAD / 8)) cp_async16(b_st + b_dst[t], g, ok ? 16u : 0u);
      }
      cp_async_mbar_arrive_noinc(smem_u32(full + stage));
      if (tid == 0) wts(FPVS_KNOB(p), 8 * k + 3);
    }
    if (tid == 0) pdl_trigger();
  } else {
    // ===================== MMA issuer (one lane) =====================
    if (warp == W_MMA && lane == 0) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                             ((uint32_t)(NPAD >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      for (int c = c0; c < c1; ++c) {
        const int k = c - c0, stage = k % NS;
        mbar_wait(smem_u32(full + stage), (k / NS) & 1);
        wts(FPVS_KNOB(p), 8 * k + 4);
        tc_fence_after();
        fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tensor core (async proxy) reads
        const uint32_t a_st = smem_u32(sA + stage * A_STAGE), b_st = smem_u32(sB + stage * B_STAGE);
        if (!(FPVS_KNOB(p) & 2)) {
#pragma unroll
          for (int kk = 0; kk < KC / 16; ++kk)
            umma_bf16(tmem, desc_mn(a_st + kk * 256), desc_mn(b_st + kk * 256), idesc, (k | kk) ? 1u : 0u);
        }
        umma_commit(smem_u32(empty + stage));
        wts(FPVS_KNOB(p), 8 * k + 5);
      }
      umma_commit(smem_u32(tfull));
    }
    // ===================== epilogue (warps 8-11): TMEM -> fp32 partial =====================
    pdl_wait();
    const int q4 = warp & 3, r = q4 * 32 + lane;
    mbar_wait_sleep(smem_u32(tfull), 0, 128);
    tc_fence_after();
    float* dst = p.part + (((long long)mb * p.nsplit + rs) * BM + r) * NPAD;
    const bool has = c1 > c0;
#pragma unroll 1
    for (int cb = 0; cb < NPAD; cb += 8) {
      float v[8];
      tmem_ld8(tmem + ((uint32_t)(q4 * 32) << 16) + cb, v);
      float4* d4 = reinterpret_cast<float4*>(dst + cb);
      d4[0] = has ? make_float4(v[0], v[1], v[2], v[3]) : make_float4(0.f, 0.f, 0.f, 0.f);
      d4[1] = has ? make_float4(v[4], v[5], v[6], v[7]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS) : "memory");
  }
}

// dw[f][co] = sum over splits of part[f / 128][s][f % 128][co] in a fixed order
// (eight interleaved partial sums, then those in order); row f = kcin (the
// all-ones A row, when kcin % 128 != 0) is db.  One block per row f:
// 32 channels x 8 split lanes, looping over channel groups of 32.
__global__ void __launch_bounds__(256) wgrad_reduce_tc_kernel(const float* __restrict__ part, int nsplit, int npad,
                                                              int kcin, int cout, float* __restrict__ dw,
                                                              float* __restrict__ db) {
  __shared__ float acc[8][32];
  const int f = blockIdx.x, cl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mb = f >> 7, m = f & 127;
  for (int co0 = 0; co0 < cout; co0 += 32) {
    const int co = co0 + lane;
    float s = 0.f;
    if (co < cout) {
      const float* src = part + ((long long)mb * nsplit * BM + m) * npad + co;
      for (int k = cl; k < nsplit; k += 8) s += __ldg(src + (long long)k * BM * npad);
    }
    acc[cl][lane] = s;
    __syncthreads();
    if (cl == 0 && co < cout) {
      float t = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) t += acc[k][lane];
      if (f < kcin) dw[(long long)f * cout + co] = t;
      else if (db) db[co] = t;
    }
    __syncthreads();
  }
}

// db[co] = sum_i dz[i][co]: per-block column sums in a fixed row order, then a
// fixed-order sum of the block partials
constexpr int DB_ROWS = 1024;
__global__ void __launch_bounds__(256) bias_partial_kernel(const __nv_bfloat16* __restrict__ dz, int lddz,
                                                           const int* n_dev, int cap, int cout,
                                                           float* __restrict__ part) {
  __shared__ float s[8][256];
  const int n = min(*n_dev, cap);
  const int r0 = blockIdx.x * DB_ROWS;
  const int tid = threadIdx.x;
  for (int co0 = 0; co0 < cout; co0 += 32) {
    const int co = co0 + (tid & 31), rw = tid >> 5;  // 8 row lanes x 32 channels
    float acc = 0.f;
    if (co < cout)
      for (int r = r0 + rw; r < min(n, r0 + DB_ROWS); r += 8) acc += __bfloat162float(dz[(long long)r * lddz + co]);
    s[rw][tid & 31] = acc;
    __syncthreads();
    if (tid < 32 && co0 + tid < cout) {
      float t = 0.f;
      for (int k = 0; k < 8; ++k) t += s[k][tid];
      part[(long long)blockIdx.x * cout + co0 + tid] = t;
    }
    __syncthreads();
  }
}

__global__ void bias_reduce_kernel(const float* __restrict__ part, const int* n_dev, int cap, int cout,
                                   float* __restrict__ db) {
  const int n = min(*n_dev, cap);
  const int nb = (n + DB_ROWS - 1) / DB_ROWS;
  for (int co = blockIdx.x * blockDim.x + threadIdx.x; co < cout; co += gridDim.x * blockDim.x) {
    float t = 0.f;
    for (int b = 0; b < nb; ++b) t += part[(long long)b * cout + co];
    db[co] = t;
  }
}

inline int npad_of(int cout) { return cout <= 16 ? 16 : cout <= 32 ? 32 : cout <= 64 ? 64 : cout <= 128 ? 128 : 256; }
inline int splits_for(int nmb, int cap) {
  const int maxc = (cap + KC - 1) / KC;
  int s = (2 * kNumSMs + nmb - 1) / nmb;
  if (s > maxc) s = maxc;
  return s < 1 ? 1 : s;
}
inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

template <int NPAD>
int launch(const Params& p, cudaStream_t s) {
  constexpr int B_STAGE = (NPAD / 8) * 1024;
  constexpr int SMEM = 1024 + NS * (A_STAGE + B_STAGE) + 1024 + KC * 32 * 4;
  {
    const cudaError_t e = set_smem_once<wgrad_tc_kernel<NPAD>>(SMEM);
    if (e != cudaSuccess) return set_error(FPVS_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  cudaError_t e = launch_kernel(wgrad_tc_kernel<NPAD>, dim3(p.nmb * p.nsplit), dim3(THREADS), SMEM, s, p);
  if (e != cudaSuccess) return set_error(FPVS_ECUDA, "wgrad_tc: %s", cudaGetErrorString(e));
  return FPVS_OK;
}

}  // namespace wg
}  // namespace fpvs

using namespace fpvs;

#ifdef FPVS_PROFILE
extern "C" int fpvs_debug_wgrad_timestamps(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, wg::g_wts, sizeof(unsigned long long) * 4096) == cudaSuccess ? 0 : 3;
}
#endif

extern "C" size_t fpvs_wgrad_tc_workspace_size(int K, int cin, int cout, int cap) {
  if (K < 1 || cin < 8 || cin % 8 || cout < 1 || cout > 256 || cap < 1) return 0;
  const int nmb = (K * cin + 127) / 128;
  const int ns = wg::splits_for(nmb, cap);
  const size_t part = (size_t)nmb * ns * tc::BM * wg::npad_of(cout) * 4;
  const size_t bias = (size_t)((cap + wg::DB_ROWS - 1) / wg::DB_ROWS) * cout * 4;
  return wg::align256(part) + wg::align256(bias);
}

extern "C" int fpvs_spconv_wgrad_tc(const void* x, int ldx, const void* dz, int lddz, const int32_t* nbr, int K,
                                    const int32_t* n_dev, int cap, int cin, int cout, float* dw, float* db,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  FPVS_CHECK_ARG(x && dz && n_dev && dw && workspace, "null pointer");
  FPVS_CHECK_ARG(K >= 1 && K <= 27 && (nbr || K == 1), "nbr may be NULL only for K == 1");
  FPVS_CHECK_ARG(cin % 8 == 0 && ldx % 8 == 0 && ldx >= cin, "wgrad needs Cin and ldx multiples of 8");
  FPVS_CHECK_ARG(cout % 8 == 0 && cout <= 256 && lddz % 8 == 0 && lddz >= cout,
                 "wgrad needs Cout (<= 256) and lddz multiples of 8");
  const size_t need = fpvs_wgrad_tc_workspace_size(K, cin, cout, cap);
  FPVS_CHECK_ARG(workspace_bytes >= need, "workspace too small: need %zu bytes", need);
  if (cap <= 0) return FPVS_OK;
  wg::Params p{};
  p.x = (const __nv_bfloat16*)x;
  p.ldx = ldx;
  p.dz = (const __nv_bfloat16*)dz;
  p.lddz = lddz;
  p.nbr = nbr;
  p.K = K;
  p.n_dev = n_dev;
  p.cap = cap;
  p.cin = cin;
  p.cout = cout;
  p.npad = wg::npad_of(cout);
  p.nmb = (K * cin + 127) / 128;
  p.nsplit = wg::splits_for(p.nmb, cap);
  p.part = (float*)workspace;
  p.dbg = debug_knob("FPVS_WGRAD_DEBUG");
  cudaStream_t s = as_stream(stream);
  int rc = p.npad == 16 ? wg::launch<16>(p, s) : p.npad == 32 ? wg::launch<32>(p, s) : p.npad == 64 ? wg::launch<64>(p, s)
         : p.npad == 128 ? wg::launch<128>(p, s) : wg::launch<256>(p, s);
  if (rc) return rc;
  const int rows = K * cin + ((db && (K * cin) % 128) ? 1 : 0);
  wg::wgrad_reduce_tc_kernel<<<rows, 256, 0, s>>>(p.part, p.nsplit, p.npad, K * cin, cout, dw, db);
  if (db && (K * cin) % 128 == 0) {
    float* bpart = (float*)((uint8_t*)workspace + wg::align256((size_t)p.nmb * p.nsplit * tc::BM * p.npad * 4));
    const int nb = (cap + wg::DB_ROWS - 1) / wg::DB_ROWS;
    wg::bias_partial_kernel<<<nb, 256, 0, s>>>((const __nv_bfloat16*)dz, lddz, n_dev, cap, cout, bpart);
    wg::bias_reduce_kernel<<<1, 256, 0, s>>>(bpart, n_dev, cap, cout, db);
  }
  FPVS_CHECK_LAUNCH("fpvs_spconv_wgrad_tc");
  return FPVS_OK;
}
