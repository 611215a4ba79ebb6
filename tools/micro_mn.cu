// Layout check for tcgen05.mma kind::f16 with BOTH operands MN-major in the
// no-swizzle ("interleave") canonical layout:
//   core matrix = 8 k-rows x 16 B (8 consecutive M or N elements), 128 B
//   contiguous; element (mn, k) at (mn/8)*SBO + (k/8)*LBO + (k%8)*16 + (mn%8)*2
//   with LBO = 128 B (K-direction core stride), SBO = 8*128 B (MN-direction).
// D[M=128][N] = sum_k A[m][k] * B[k][n], K = 64 (4 MMAs of K = 16).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro_mn.bin tools/micro_mn.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

constexpr int M = 128, N = 32, K = 64;
constexpr int LBO = 128, SBO = 8 * 128;  // K chunk of 64 = 8 core matrices along K

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  // layout type 0 = SWIZZLE_NONE (bits 61-63)
  return d;
}

__global__ void __launch_bounds__(128, 1) k(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  uint8_t* sb = sa + M * K * 2;
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  const int t = threadIdx.x, w = t >> 5;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // A: host layout A[m][k] row-major; B: B[k][n] row-major
  for (int e = t; e < M * K; e += 128) {
    int m = e / K, kk = e % K;
    int off = (m / 8) * SBO + (kk / 8) * LBO + (kk % 8) * 16 + (m % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sa + off) = A[m * K + kk];
  }
  for (int e = t; e < K * N; e += 128) {
    int kk = e / N, n = e % N;
    int off = (n / 8) * SBO + (kk / 8) * LBO + (kk % 8) * 16 + (n % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sb + off) = B[kk * N + n];
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = tm;
  if (t == 0) {
    // D f32 (bit 4), A bf16 (7), B bf16 (10), A MN-major (15), B MN-major (16), N>>3, M>>4
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t lbo = mode ? SBO : LBO, sbo = mode ? LBO : SBO;  // mode 1: swapped roles (diagnostic)
    for (int kk = 0; kk < K / 16; ++kk) {
      uint64_t ad = desc_none(su32(sa) + kk * 2 * LBO, lbo, sbo);
      uint64_t bd = desc_none(su32(sb) + kk * 2 * LBO, lbo, sbo);
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(base),
          "l"(ad), "l"(bd), "r"(idesc), "r"(kk > 0 ? 1 : 0)
          : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
  }
  asm volatile(
      "{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W%=;\n}\n" ::"r"(
          su32(&bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c = 0; c < N; c += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(base + ((uint32_t)(w * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 8; ++i) D[t * N + c + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(base));
}

int main() {
  std::vector<__nv_bfloat16> a(M * K), b(K * N);
  std::vector<float> af(M * K), bf(K * N), d(M * N);
  srand(3);
  for (int i = 0; i < M * K; ++i) { a[i] = __float2bfloat16((rand() % 17 - 8) / 8.f); af[i] = __bfloat162float(a[i]); }
  for (int i = 0; i < K * N; ++i) { b[i] = __float2bfloat16((rand() % 13 - 6) / 4.f); bf[i] = __bfloat162float(b[i]); }
  __nv_bfloat16 *da, *db;
  float* dd;
  cudaMalloc(&da, M * K * 2); cudaMalloc(&db, K * N * 2); cudaMalloc(&dd, M * N * 4);
  cudaMemcpy(da, a.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), K * N * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  int rc = 0;
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dd, 0, M * N * 4);
    k<<<1, 128, 32768>>>(da, db, dd, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(d.data(), dd, M * N * 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int kk = 0; kk < K; ++kk) s += (double)af[m * K + kk] * bf[kk * N + n];
        err = fmax(err, fabs(s - d[m * N + n]));
      }
    printf("mode %d (%s): MN-major interleave max abs err %.3g -> %s\n", mode,
           mode ? "LBO=MN stride, SBO=K stride" : "LBO=K stride, SBO=MN stride", err, err < 1e-3 ? "OK" : "wrong");
    if (mode == 0 && err >= 1e-3) rc = 2;
  }
  return rc;
}
