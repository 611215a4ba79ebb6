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
#include "common.cuh"
#include "tc_ptx.cuh"

namespace fpvs {
namespace wg {

using namespace tc;

constexpr int KC = 64;          // rows of the reduction per pipeline stage
constexpr int NS = 4;           // stages
constexpr int A_STAGE = 16384;  // 128 (j, ci) x 64 rows x 2 B
constexpr int THREADS = 256;    // warps 0-3 producers, warp 4 MMA, warps 4-7 epilogue
constexpr int PROD = 128;

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
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "n"(TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp < 4) {
    // ===================== producers: gather A pieces, load B pieces =====================
    pdl_wait();
    const uint32_t ldx2 = (uint32_t)p.ldx * 2u, lddz2 = (uint32_t)p.lddz * 2u;
    for (int c = c0; c < c1; ++c) {
      const int k = c - c0, stage = k % NS;
      mbar_wait_sleep(smem_u32(empty + stage), ((k / NS) & 1) ^ 1, 32);
      const uint32_t a_st = smem_u32(sA + stage * A_STAGE), b_st = smem_u32(sB + stage * B_STAGE);
      const int i0 = c * KC;
      // A: 64 rows x 16 groups of 8 (j, ci) values
#pragma unroll 2
      for (int q = tid; q < KC * 16; q += PROD) {
        const int kk = q >> 4, mg = q & 15;
        const int f = mb * 128 + mg * 8;  // flattened (j, ci) of the piece
        const int i = i0 + kk;
        int src = -1;
        if (i < n && f < kcin) {
          const int j = f / p.cin;
          src = p.nbr ? __ldg(p.nbr + (long long)i * p.K + j) : i;
        }
        const char* g = reinterpret_cast<const char*>(p.x) + (src >= 0 ? (long long)src * ldx2 + (f % p.cin) * 2 : 0);
        cp_async16(a_st + mg * 1024 + (kk >> 3) * 128 + (kk & 7) * 16, g, src >= 0 ? 16u : 0u);
      }
      // B: 64 rows x NPAD/8 groups of dz
      for (int q = tid; q < KC * (NPAD / 8); q += PROD) {
        const int kk = q / (NPAD / 8), ng = q - kk * (NPAD / 8);
        const int i = i0 + kk;
        const bool ok = i < n && ng * 8 < p.cout;
        const char* g = reinterpret_cast<const char*>(p.dz) + (ok ? (long long)i * lddz2 + ng * 16 : 0);
        cp_async16(b_st + ng * 1024 + (kk >> 3) * 128 + (kk & 7) * 16, g, ok ? 16u : 0u);
      }
      cp_async_mbar_arrive_noinc(smem_u32(full + stage));
    }
    if (tid == 0) pdl_trigger();
  } else {
    // ===================== MMA issuer (warp 4, one lane) =====================
    if (warp == 4 && lane == 0) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                             ((uint32_t)(NPAD >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      for (int c = c0; c < c1; ++c) {
        const int k = c - c0, stage = k % NS;
        mbar_wait(smem_u32(full + stage), (k / NS) & 1);
        tc_fence_after();
        fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tensor core (async proxy) reads
        const uint32_t a_st = smem_u32(sA + stage * A_STAGE), b_st = smem_u32(sB + stage * B_STAGE);
#pragma unroll
        for (int kk = 0; kk < KC / 16; ++kk)
          umma_bf16(tmem, desc_mn(a_st + kk * 256), desc_mn(b_st + kk * 256), idesc, (k | kk) ? 1u : 0u);
        umma_commit(smem_u32(empty + stage));
      }
      umma_commit(smem_u32(tfull));
    }
    // ===================== epilogue (warps 4-7): TMEM -> fp32 partial =====================
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
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS) : "memory");
  }
}

// dw[f][co] = sum over splits (fixed order) of part[f / 128][s][f % 128][co]
__global__ void wgrad_reduce_tc_kernel(const float* __restrict__ part, int nsplit, int npad, int kcin, int cout,
                                       float* __restrict__ dw) {
  const long long total = (long long)kcin * cout;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int f = (int)(t / cout), co = (int)(t - (long long)f * cout);
    const int mb = f >> 7, m = f & 127;
    const float* src = part + ((long long)mb * nsplit * BM + m) * npad + co;
    float s = 0.f;
    for (int k = 0; k < nsplit; ++k) s += src[(long long)k * BM * npad];
    dw[t] = s;
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
  constexpr int SMEM = 1024 + NS * (A_STAGE + B_STAGE) + 8 * (2 * NS + 1) + 16;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(wgrad_tc_kernel<NPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return set_error(FPVS_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    configured = true;
  }
  cudaError_t e = launch_kernel(wgrad_tc_kernel<NPAD>, dim3(p.nmb * p.nsplit), dim3(THREADS), SMEM, s, p);
  if (e != cudaSuccess) return set_error(FPVS_ECUDA, "wgrad_tc: %s", cudaGetErrorString(e));
  return FPVS_OK;
}

}  // namespace wg
}  // namespace fpvs

using namespace fpvs;

extern "C" size_t fpvs_wgrad_tc_workspace_size(int K, int cin, int cout, int cap) {
  if (K < 1 || cin < 8 || cout < 1 || cout > 256 || cap < 1) return 0;
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
  cudaStream_t s = as_stream(stream);
  int rc = p.npad == 16 ? wg::launch<16>(p, s) : p.npad == 32 ? wg::launch<32>(p, s) : p.npad == 64 ? wg::launch<64>(p, s)
         : p.npad == 128 ? wg::launch<128>(p, s) : wg::launch<256>(p, s);
  if (rc) return rc;
  const long long total = (long long)K * cin * cout;
  wg::wgrad_reduce_tc_kernel<<<grid_for(total, 256), 256, 0, s>>>(p.part, p.nsplit, p.npad, K * cin, cout, dw);
  if (db) {
    float* bpart = (float*)((uint8_t*)workspace + wg::align256((size_t)p.nmb * p.nsplit * tc::BM * p.npad * 4));
    const int nb = (cap + wg::DB_ROWS - 1) / wg::DB_ROWS;
    wg::bias_partial_kernel<<<nb, 256, 0, s>>>((const __nv_bfloat16*)dz, lddz, n_dev, cap, cout, bpart);
    wg::bias_reduce_kernel<<<1, 256, 0, s>>>(bpart, n_dev, cap, cout, db);
  }
  FPVS_CHECK_LAUNCH("fpvs_spconv_wgrad_tc");
  return FPVS_OK;
}
