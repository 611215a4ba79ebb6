// Layout check for tcgen05.mma with the A operand in TMEM (kind::f16, M=128):
// thread r of warp q writes row 32q+r of A (64 bf16 = 32 columns, low half =
// even k) with tcgen05.st.32x32b.x32; B (N x 64, K-major SW128) from smem.
// D = A * B^T is compared against a host reference.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro_ts.bin tools/micro_ts.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

constexpr int M = 128, N = 64, K = 64;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__global__ void __launch_bounds__(128, 1) k(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sb = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  const int t = threadIdx.x, w = t >> 5, l = t & 31;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // B: row n (0..63), 128 B per row, 16-byte piece p at ((p ^ (n & 7)) << 4)
  for (int i = t; i < N * 8; i += 128) {
    int n = i >> 3, p = i & 7;
    *reinterpret_cast<uint4*>(sb + n * 128 + ((p ^ (n & 7)) << 4)) =
        *reinterpret_cast<const uint4*>(B + n * K + p * 8);
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = tm;
  // A row r -> TMEM lane r, columns 64..95
  {
    uint32_t r[32];
    const uint4* src = reinterpret_cast<const uint4*>(A + t * K);
    for (int p = 0; p < 8; ++p) {
      uint4 v = src[p];
      r[4 * p] = v.x; r[4 * p + 1] = v.y; r[4 * p + 2] = v.z; r[4 * p + 3] = v.w;
    }
    const uint32_t ta = base + ((uint32_t)(w * 32) << 16) + 64;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (t == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    uint64_t bd = desc(su32(sb));
    for (int kk = 0; kk < K / 16; ++kk) {
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(base),
          "r"(base + 64 + kk * 8), "l"(bd + 2 * kk), "r"(idesc), "r"(kk > 0 ? 1 : 0)
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
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(base));
}

int main() {
  std::vector<__nv_bfloat16> a(M * K), b(N * K);
  std::vector<float> af(M * K), bf(N * K), d(M * N);
  srand(1);
  for (int i = 0; i < M * K; ++i) { a[i] = __float2bfloat16((rand() % 17 - 8) / 8.f); af[i] = __bfloat162float(a[i]); }
  for (int i = 0; i < N * K; ++i) { b[i] = __float2bfloat16((rand() % 13 - 6) / 4.f); bf[i] = __bfloat162float(b[i]); }
  __nv_bfloat16 *da, *db;
  float* dd;
  cudaMalloc(&da, M * K * 2); cudaMalloc(&db, N * K * 2); cudaMalloc(&dd, M * N * 4);
  cudaMemcpy(da, a.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), N * K * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  k<<<1, 128, 16384>>>(da, db, dd);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(d.data(), dd, M * N * 4, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int kk = 0; kk < K; ++kk) s += (double)af[m * K + kk] * bf[n * K + kk];
      err = fmax(err, fabs(s - d[m * N + n]));
    }
  printf("TS mma max abs err %.3g (%s)\n", err, err < 1e-3 ? "layout OK" : "LAYOUT MISMATCH");
  return err < 1e-3 ? 0 : 2;
}
