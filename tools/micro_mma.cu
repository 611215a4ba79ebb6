// tcgen05.mma issue/throughput microbenchmark (1 CTA per SM, SS operands).
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
template <int N, int NSTAGE, int MODE>
__global__ void __launch_bounds__(128, 1) k(long long* out, int iters) {
  __shared__ uint64_t bar2[2];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar2[0])), "r"((1 << 20) - 1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar2[1])), "r"((1 << 20) - 1));
  }
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < NSTAGE * (16384 + N * 128) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(base)[i] = (i * 2654435761u) & 0x3f803f80u;  // random-ish bf16 pairs
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64();
  if (MODE >= 4 && threadIdx.x < (MODE == 4 ? 32 : 1)) {
    __shared__ uint32_t info[8];
    if (MODE == 4) { if (threadIdx.x < 8) info[threadIdx.x] = 1; __syncwarp(); }
    else { for (int q = 0; q < 8; ++q) info[q] = 1; }
    for (int i = 0; i < iters; ++i) {
      const int st = i % NSTAGE;
      // wait on an already-completed phase (parity 1 of a fresh barrier)
      if (MODE != 7 || (i & 1) == 0) {
      asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 1;\n@!p bra W%=;\n}\n" ::"r"(su32(&bar2[0])) : "memory");
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (MODE != 6) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      const uint32_t inf = info[st & 7];
      if (threadIdx.x == 0) {
        uint64_t ad = desc(su32(base + st * 16384)), bd = desc(su32(base + NSTAGE * 16384 + st * N * 128));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tm), "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(inf));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2[1])) : "memory");
      }
      if (MODE == 4) __syncwarp();
    }
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
      asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W2;\n}\n" ::"r"(su32(&bar)));
    }
  }
  if (MODE < 4 && threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      const int st = i % NSTAGE;
      if (MODE >= 1) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (MODE >= 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      uint64_t ad = desc(su32(base + st * 16384)), bd = desc(su32(base + NSTAGE * 16384 + st * N * 128));
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tm), "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(1));
      }
      if (MODE >= 3) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2[st & 1])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

template <int N, int NS = 1, int MODE = 0>
void run(long long* d, int grid) {
  int smem = NS * (16384 + N * 128) + 1024;
  cudaFuncSetAttribute(k<N, NS, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h;
  int it = 2000;
  k<N, NS, MODE><<<grid, 128, smem>>>(d, it);
  k<N, NS, MODE><<<grid, 128, smem>>>(d, it);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  double per = (double)h / (it * 4);
  double ideal = 128.0 * N / 256.0;
  printf("MODE=%d NS=%d N=%3d grid=%3d: %7.1f cycles per 128x%dx16 MMA (ideal %.0f) -> %5.1f%% of peak  (%s)\n", MODE, NS, N, grid, per, N,
         ideal, 100 * ideal / per, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  for (int g : {148}) {
    run<64, 8, 3>(d, g); run<64, 8, 4>(d, g); run<64, 8, 5>(d, g); run<64, 8, 6>(d, g); run<64, 8, 7>(d, g); run<128, 6, 5>(d, g); run<128, 6, 7>(d, g);
  }
  return 0;
}
