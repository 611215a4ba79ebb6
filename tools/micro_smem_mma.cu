// Does tcgen05.mma (SS) smem operand traffic share bandwidth with LDS/STS?
// One thread issues SS MMAs (M=128, N, K=16) back to back while W warps copy
// smem->smem with LDS.128/STS.128; both rates are reported.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro_smem_mma.bin tools/micro_smem_mma.cu
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

template <int N, int MMA, int COPYW>
__global__ void __launch_bounds__(384, 1) k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  __shared__ volatile int stop;
  __shared__ unsigned long long copied;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    stop = 0;
    copied = 0;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tm)));
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
  if (warp == 0) {
    if (threadIdx.x == 0) {
      if (MMA) {
        uint64_t ad = desc(su32(base)), bd = desc(su32(base + 16384));
        for (int i = 0; i < iters; ++i) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tm), "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(1));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
      } else {
        while (clock64() - t0 < 2000000) {}
      }
      long long t1 = clock64();
      if (blockIdx.x == 0) out[0] = t1 - t0;
      stop = 1;
    }
  } else if (warp <= COPYW) {
    // smem -> smem copy of 16-byte pieces: src region 64 KB at +40 KB, dst region at +104 KB
    const uint8_t* src = base + 40960;
    uint8_t* dst = base + 106496;
    const int t = threadIdx.x - 32;
    unsigned long long n = 0;
    while (!stop) {
#pragma unroll 4
      for (int i = 0; i < 16; ++i) {
        const int o = ((i * COPYW * 32 + t) * 16) & 65535;
        uint32_t a, b, c, e;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(e) : "r"(su32(src + o)));
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(su32(dst + o)), "r"(a), "r"(b), "r"(c), "r"(e));
      }
      n += 16;
    }
    atomicAdd(&copied, n * 16);
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = copied;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

template <int N, int MMA, int COPYW>
void run(long long* d) {
  int smem = 106496 + 65536 + 1024;
  cudaFuncSetAttribute(k<N, MMA, COPYW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h[2];
  int it = 4000;
  k<N, MMA, COPYW><<<148, 384, smem>>>(d, it);
  k<N, MMA, COPYW><<<148, 384, smem>>>(d, it);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  double per = MMA ? (double)h[0] / (it * 4) : 0;
  printf("N=%3d mma=%d copy warps=%2d: %6.1f cyc/MMA (ideal %3.0f) | copy %6.1f B/cyc (read+write = %6.1f) %s\n", N, MMA,
         COPYW, per, 128.0 * N / 256, (double)h[1] / h[0], 2.0 * h[1] / h[0], cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  run<128, 0, 8>(d); run<128, 1, 0>(d); run<128, 1, 4>(d); run<128, 1, 8>(d);
  run<64, 1, 0>(d); run<64, 1, 8>(d); run<256, 1, 0>(d); run<256, 1, 8>(d);
  return 0;
}
