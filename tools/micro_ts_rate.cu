// tcgen05.mma issue rate: A from SMEM (SS) vs A from TMEM (TS), 1 CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro_ts_rate.bin tools/micro_ts_rate.cu
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
// TS: 0 = SS, 1 = TS; COMMIT: commit every 4 MMAs; STW: 1 = other warps keep writing TMEM (STTM) concurrently
template <int N, int TS, int COMMIT, int STW>
__global__ void __launch_bounds__(256, 1) k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint64_t bar, bar2[2];
  __shared__ uint32_t tm;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar2[0])), "r"(1 << 20));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar2[1])), "r"(1 << 20));
    asm volatile("fence.mbarrier_init.release.cluster;");
    stop = 0;
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
    uint64_t ad = desc(su32(base)), bd = desc(su32(base + 16384));
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (TS)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                       ::"r"(tm), "r"(tm + 256 + 8 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(1));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tm), "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(1));
      }
      if (COMMIT && (i % COMMIT) == COMMIT - 1) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2[i & 1])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
    stop = 1;
  } else if (STW && threadIdx.x >= 128) {
    // 4 warps keep storing 32 columns each into the TMEM region at column 384
    const int q = (threadIdx.x >> 5) & 3;
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * 7 + i;
    while (!stop) {
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tm + ((q * 32) << 16) + 384),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
          "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
          "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
          "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int TS, int COMMIT, int STW>
void run(long long* d) {
  int smem = 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(k<N, TS, COMMIT, STW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h;
  int it = 4000;
  k<N, TS, COMMIT, STW><<<148, 256, smem>>>(d, it);
  k<N, TS, COMMIT, STW><<<148, 256, smem>>>(d, it);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  double per = (double)h / (it * 4);
  double ideal = 128.0 * N / 256.0;
  printf("%s N=%3d commit/4xMMA-groups=%d sttm=%d: %6.1f cycles per 128x%dx16 MMA (ideal %.0f, %5.1f%%) %s\n", TS ? "TS" : "SS", N,
         COMMIT, STW, per, N, ideal, 100 * ideal / per, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<64, 1, 1, 0>(d); run<64, 1, 2, 0>(d); run<64, 1, 4, 0>(d); run<64, 1, 8, 0>(d);
  run<64, 0, 1, 0>(d); run<64, 0, 2, 0>(d); run<64, 0, 4, 0>(d);
  run<128, 1, 1, 0>(d); run<128, 1, 2, 0>(d); run<128, 1, 4, 0>(d);
  run<128, 0, 1, 0>(d); run<128, 0, 2, 0>(d); run<256, 1, 1, 0>(d); run<256, 1, 2, 0>(d); run<256, 0, 1, 0>(d);
  return 0;
}
