// Latency of the synchronisation hops the halo conv pipeline runs on, measured
// with clock64 on one SM: (a) issuing tcgen05.commit, (b) commit -> a waiting
// warp observing the mbarrier phase, with 0 or 16 MMAs in flight, (c) a plain
// mbarrier.arrive -> observer.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro_commit_lat.bin tools/micro_commit_lat.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_parity(uint32_t bar, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(bar),
               "r"(par) : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int NMMA, int PLAIN>
__global__ void __launch_bounds__(64, 1) k(long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tm_s;
  __shared__ long long t_issue0[64], t_issue1[64], t_seen[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tm_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tm_s;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t b = su32(&bar);
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    if (warp == 0) {
      if (lane == 0) {
        const uint64_t bd = desc(su32(base));
        long long t0 = clock64();
#pragma unroll
        for (int q = 0; q < NMMA; ++q)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                       ::"r"(tm), "r"(tm + 256 + 8 * (q & 3)), "l"(bd + 2 * (q & 3)), "r"(idesc));
        long long t1 = clock64();
        if (PLAIN) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
        else asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b) : "memory");
        long long t2 = clock64();
        if (r < 64) { t_issue0[r] = t1 - t0; t_issue1[r] = t2; }
      }
    } else {
      wait_parity(b, r & 1);
      long long t3 = clock64();
      if (lane == 0 && r < 64) t_seen[r] = t3;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    long long s0 = 0, s1 = 0;
    for (int r = 8; r < 64; ++r) { s0 += t_issue0[r]; s1 += t_seen[r] - t_issue1[r]; }
    out[0] = s0 / 56;
    out[1] = s1 / 56;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int NMMA, int PLAIN>
void run(long long* d) {
  cudaFuncSetAttribute(k<NMMA, PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 1024);
  long long h[2];
  k<NMMA, PLAIN><<<148, 64, 16384 + 1024>>>(d, 64);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%s after %2d MMAs: MMA issue %5lld cyc; arrive->observed (from after the arrive instr) %5lld cyc  %s\n",
         PLAIN ? "mbarrier.arrive" : "tcgen05.commit ", NMMA, h[0], h[1], cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  run<0, 1>(d); run<0, 0>(d); run<1, 0>(d); run<4, 0>(d); run<16, 0>(d); run<16, 1>(d);
  return 0;
}
