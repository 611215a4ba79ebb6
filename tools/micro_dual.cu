// tcgen05.mma (M=128, K=16, bf16, A in TMEM) issued by ONE vs TWO threads of a
// CTA (different warps, separate accumulators and A slots): is the ~45-cycle
// per-MMA floor at N <= 64 a per-issuer or a per-SM limit?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro_dual.bin tools/micro_dual.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

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

template <int N, int ISSUERS>
__global__ void __launch_bounds__(128, 1) k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tm_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tm_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 4 * N * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = (i * 2654435761u) & 0x3f803f80u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tm_s;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64();
  if (lane == 0 && warp < ISSUERS) {
    const uint32_t sb = su32(base);
    const uint32_t dtm = tm + warp * 64;                  // accumulator per issuer
    const uint32_t abase = tm + 128 + warp * 128;        // 4 A slots of 32 columns per issuer
    const int my = iters / ISSUERS;
    for (int i = 0; i < my; i += 16) {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int slot = (q >> 2) & 3, kk = q & 3;
        const uint64_t bd = desc(sb + slot * N * 128) + 2 * kk;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(dtm), "r"(abase + slot * 32 + 8 * kk), "l"(bd), "r"(idesc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[warp])) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar[warp])));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int ISSUERS>
void run(long long* d) {
  const int smem = 4 * N * 128 + 1024;
  cudaFuncSetAttribute(k<N, ISSUERS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int it = 8192;
  long long h = 0;
  k<N, ISSUERS><<<148, 128, smem>>>(d, it);
  k<N, ISSUERS><<<148, 128, smem>>>(d, it);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("N=%3d issuers=%d: %6.1f cycles per MMA (SM total), ideal %3.0f  %s\n", N, ISSUERS, (double)h / it,
         128.0 * N / 256, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<64, 1>(d); run<64, 2>(d); run<32, 1>(d); run<32, 2>(d); run<128, 1>(d); run<128, 2>(d);
  return 0;
}
