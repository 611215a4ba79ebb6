// Latency of tcgen05.commit -> mbarrier completion, and of mbarrier wake-up.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(bar), "r"(par) : "memory");
}

// MODE 0: thread 0 commit + wait loop;  MODE 1: thread 0 arrive + wait loop (plain)
// MODE 2: ping-pong between warp 0 (arrive A, wait B) and warp 1 (wait A, commit B)
template <int MODE>
__global__ void k(long long* out, int iters) {
  __shared__ __align__(16) uint64_t bar[2];
  __shared__ uint32_t tm;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  long long t0 = clock64();
  if (MODE == 0 && threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[0])) : "memory");
      wait(su32(&bar[0]), i & 1);
    }
  }
  if (MODE == 1 && threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar[0])) : "memory");
      wait(su32(&bar[0]), i & 1);
    }
  }
  if (MODE == 2) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < iters; ++i) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar[0])) : "memory");
        wait(su32(&bar[1]), i & 1);
      }
    } else if (threadIdx.x == 32) {
      for (int i = 0; i < iters; ++i) {
        wait(su32(&bar[0]), i & 1);
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[1])) : "memory");
      }
    }
  }
  if (MODE == 3) {  // same ping-pong but plain arrive instead of commit
    if (threadIdx.x == 0) {
      for (int i = 0; i < iters; ++i) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar[0])) : "memory");
        wait(su32(&bar[1]), i & 1);
      }
    } else if (threadIdx.x == 32) {
      for (int i = 0; i < iters; ++i) {
        wait(su32(&bar[0]), i & 1);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar[1])) : "memory");
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  const char* names[] = {"commit+wait (1 thread)", "arrive+wait (1 thread)", "ping-pong arrive/commit", "ping-pong arrive/arrive"};
  for (int m = 0; m < 4; ++m) {
    long long h = 0;
    int it = 2000;
    for (int rep = 0; rep < 2; ++rep) {
      if (m == 0) k<0><<<1, 64>>>(d, it);
      if (m == 1) k<1><<<1, 64>>>(d, it);
      if (m == 2) k<2><<<1, 64>>>(d, it);
      if (m == 3) k<3><<<1, 64>>>(d, it);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %8.1f cycles/iter (%s)\n", names[m], (double)h / it, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
