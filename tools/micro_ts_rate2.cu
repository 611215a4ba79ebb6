// TS (A in TMEM) tcgen05.mma issue rate variants, 1 CTA per SM, single issuing thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro_ts_rate2.bin tools/micro_ts_rate2.cu
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
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
               ::"r"(d), "r"(a), "l"(b), "r"(idesc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc));
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// V: 0 TS no commit, 1 TS commit/4 (unrolled x4), 2 TS fence/4, 3 TS commit/4 same A, 4 SS commit/4,
//    5 TS commit/4 with 8 stages A rotating (like the conv), 6 TS commit/16
template <int N, int V>
__global__ void __launch_bounds__(128, 1) k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint64_t bar, bar2[2];
  __shared__ uint32_t tm;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar2[0])), "r"(1 << 20));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar2[1])), "r"(1 << 20));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(base)[i] = (i * 2654435761u) & 0x3f803f80u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint64_t ad = desc(su32(base)), bd = desc(su32(base + 16384));
    const uint32_t a0 = tm + 256;
    for (int i = 0; i < iters; i += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t as = V == 5 ? tm + 256 + ((i + u) & 7) * 32 : a0;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (V == 4) mma_ss(tm, ad + 2 * kk, bd + 2 * kk, idesc);
          else mma_ts(tm, V == 3 ? a0 : as + 8 * kk, bd + 2 * kk, idesc);
        }
        if (V == 1 || V == 3 || V == 4 || V == 5) commit(su32(&bar2[u & 1]));
        if (V == 2) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      if (V == 6) commit(su32(&bar2[0]));
    }
    commit(su32(&bar));
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int V>
void run(long long* d) {
  int smem = 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(k<N, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h;
  int it = 4000;
  k<N, V><<<148, 128, smem>>>(d, it);
  k<N, V><<<148, 128, smem>>>(d, it);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const char* names[] = {"TS no commit", "TS commit/4", "TS fence/4", "TS commit/4 same A", "SS commit/4",
                         "TS commit/4 rotating A", "TS commit/16"};
  printf("N=%3d %-24s %6.1f cyc/MMA (ideal %3.0f) %s\n", N, names[V], (double)h / (it * 4), 128.0 * N / 256,
         cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<64, 0>(d); run<64, 1>(d); run<64, 2>(d); run<64, 3>(d); run<64, 4>(d); run<64, 5>(d); run<64, 6>(d);
  run<128, 0>(d); run<128, 1>(d); run<128, 3>(d); run<128, 4>(d); run<128, 5>(d); run<128, 6>(d);
  return 0;
}
