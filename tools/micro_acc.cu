// tcgen05.mma issue cost vs accumulator rotation (one CTA per SM, one issuing thread).
// Question: is the ~80-cycle cost of an M=128, N=64 MMA a dependency on the
// shared accumulator (then rotating 2-4 independent accumulators hides it) or a
// per-instruction issue floor?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro_acc.bin tools/micro_acc.cu
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

// SS: 0 = TS, 1 = SS.  NACC accumulators; ROT 0 = switch accumulator per 4-MMA chunk, 1 = per MMA.
// CPC = MMAs per commit.
template <int N, int SS, int NACC, int ROT, int CPC, int ABASE = -1>
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
  for (int i = threadIdx.x; i < (16384 + 256 * 128) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(base)[i] = (i * 2654435761u) & 0x3f803f80u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint64_t ad = desc(su32(base)), bd = desc(su32(base + 16384));
    const uint32_t a0 = tm + (ABASE < 0 ? NACC * N : ABASE);  // A slots after the accumulators
    int m = 0;
    for (int i = 0; i < iters; i += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk, ++m) {
          const int acc = ROT ? (m % NACC) : ((m >> 2) % NACC);
          const uint32_t dd = tm + acc * N;
          if (SS == 2 ? (m & 1) : SS) mma_ss(dd, ad + 2 * kk, bd + 2 * kk, idesc);
          else mma_ts(dd, a0 + 8 * kk, bd + 2 * kk, idesc);
          if ((m + 1) % CPC == 0) commit(su32(&bar2[(m / CPC) & 1]));
        }
      }
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

template <int N, int SS, int NACC, int ROT, int CPC, int ABASE = -1>
void run(long long* d) {
  int smem = 16384 + 256 * 128 + 1024;
  cudaFuncSetAttribute(k<N, SS, NACC, ROT, CPC, ABASE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h;
  int it = 4000;
  k<N, SS, NACC, ROT, CPC, ABASE><<<148, 128, smem>>>(d, it);
  k<N, SS, NACC, ROT, CPC, ABASE><<<148, 128, smem>>>(d, it);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("abase=%4d N=%3d %s nacc=%d rot=%s commit/%-2d %6.1f cyc/MMA (ideal %3.0f) %s\n", ABASE, N, SS == 2 ? "MX" : SS ? "SS" : "TS", NACC,
         ROT ? "mma  " : "chunk", CPC, (double)h / (it * 4), 128.0 * N / 256, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<64, 0, 1, 0, 16, 64>(d);
  run<64, 0, 1, 0, 16, 128>(d);
  run<64, 0, 1, 0, 16, 224>(d);
  run<64, 0, 1, 0, 16, 256>(d);
  run<64, 0, 1, 0, 16, 384>(d);
  run<64, 0, 1, 0, 4, 256>(d);
  run<64, 0, 2, 1, 16, 256>(d);
  run<64, 0, 1, 0, 16000, 256>(d);
  run<128, 0, 1, 0, 16, 128>(d);
  run<128, 0, 1, 0, 16, 256>(d);
  run<128, 0, 1, 0, 4, 256>(d);
  run<32, 0, 1, 0, 16, 64>(d);
  run<32, 0, 1, 0, 16, 256>(d);
  return 0;
}
