// Microbenchmark of pipeline primitives on one SM (cycles per iteration).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void k(long long* out, const int4* g, int iters) {
  __shared__ __align__(16) uint64_t bar[2];
  __shared__ __align__(16) int4 buf[256];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[0])), "r"((1 << 20) - 1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (MODE == 2) { asm volatile("cp.async.commit_group;" ::: "memory"); asm volatile("cp.async.wait_group 0;" ::: "memory"); }
    if (MODE == 3) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar[0])) : "memory");
    if (MODE == 4) asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&bar[0])) : "memory");
    if (MODE == 5) {
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(&buf[threadIdx.x])), "l"(g + threadIdx.x) : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    if (MODE == 6) {
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(&buf[threadIdx.x])), "l"(g + threadIdx.x) : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (MODE == 7) __syncwarp();
    if (MODE == 8) {
      if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar[0])) : "memory");
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}

int main() {
  long long* d; int4* g;
  cudaMalloc(&d, 8); cudaMalloc(&g, 1 << 20); cudaMemset(g, 0, 1 << 20);
  const char* names[] = {"empty", "fence.proxy.async", "commit+wait_group0", "mbar.arrive x256thr", "noinc arrive x256",
                         "cp.async16+wait", "cp.async16+wait+fence", "syncwarp", "mbar.arrive x8 warps"};
  for (int threads : {32, 256}) {
    for (int m = 0; m < 9; ++m) {
      long long h = 0;
      int it = 1000;
      for (int rep = 0; rep < 2; ++rep) {
        switch (m) {
          case 0: k<0><<<1, threads>>>(d, g, it); break;
          case 1: k<1><<<1, threads>>>(d, g, it); break;
          case 2: k<2><<<1, threads>>>(d, g, it); break;
          case 3: k<3><<<1, threads>>>(d, g, it); break;
          case 4: k<4><<<1, threads>>>(d, g, it); break;
          case 5: k<5><<<1, threads>>>(d, g, it); break;
          case 6: k<6><<<1, threads>>>(d, g, it); break;
          case 7: k<7><<<1, threads>>>(d, g, it); break;
          case 8: k<8><<<1, threads>>>(d, g, it); break;
        }
        cudaDeviceSynchronize();
      }
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("%3d thr %-24s %8.1f cycles/iter  (%s)\n", threads, names[m], (double)h / it, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
