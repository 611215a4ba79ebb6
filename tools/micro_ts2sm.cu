// tcgen05.mma.cta_group::2 (CTA pair, M=256) issue rate, A from TMEM or SMEM, commits multicast.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro_ts2sm.bin tools/micro_ts2sm.cu
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
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N, int TS, int CPER>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t bar, bar2[2];
  __shared__ uint32_t tm;
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar2[0])), "r"(1 << 20));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar2[1])), "r"(1 << 20));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  for (int i = threadIdx.x; i < (16384 + N * 64) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(base)[i] = (i * 2654435761u) & 0x3f803f80u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  long long t0 = clock64();
  if (rank == 0 && threadIdx.x == 0) {
    const uint64_t ad = desc(su32(base)), bd = desc(su32(base + 16384));
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (TS)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                       ::"r"(tm), "r"(tm + 256 + 8 * kk), "l"(bd + 2 * kk), "r"(idesc));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tm), "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(idesc));
      }
      if (CPER && (i % CPER) == CPER - 1)
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(su32(&bar2[i & 1])), "h"((uint16_t)3) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(su32(&bar)), "h"((uint16_t)3) : "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int TS, int CPER>
void run(long long* d) {
  int smem = 16384 + N * 64 + 1024;
  cudaFuncSetAttribute(k<N, TS, CPER>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h = 0;
  int it = 4000;
  k<N, TS, CPER><<<148, 128, smem>>>(d, it);
  k<N, TS, CPER><<<148, 128, smem>>>(d, it);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("2SM %s N=%3d commit/%d: %6.1f cyc per 256x%dx16 MMA (ideal %3.0f per pair) %s\n", TS ? "TS" : "SS", N, CPER,
         (double)h / (it * 4), N, 128.0 * N / 256, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<64, 1, 1>(d); run<64, 1, 2>(d); run<64, 1, 4>(d); run<64, 1, 8>(d); run<64, 1, 16>(d);
  run<64, 0, 1>(d); run<64, 0, 4>(d); run<64, 0, 0>(d);
  run<128, 1, 2>(d); run<128, 1, 4>(d); run<128, 0, 4>(d);
  return 0;
}
