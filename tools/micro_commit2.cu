// tcgen05.mma (M=128, K=16, bf16) cost vs commit spacing with realistic operand
// rotation: A cycles through 8 TMEM slots (TS) or 8 smem slots (SS), B through
// 4 smem stages, one accumulator; every operand address precomputed in
// registers (the issuing thread does no loads between MMAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro_commit2.bin tools/micro_commit2.cu
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

template <int N, int SS, int C, int RND = 0>
__global__ void __launch_bounds__(128, 1) k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint64_t bar, bar2[2];
  __shared__ uint32_t tm_s;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar2[0])), "r"(1 << 20));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar2[1])), "r"(1 << 20));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tm_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // smem: 8 A slots x 16 KB (SS) at 0, 4 B stages x N*128 B after
  constexpr int A_BYTES = SS ? 8 * 16384 : 0;
  for (int i = threadIdx.x; i < (A_BYTES + 4 * N * 128) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(base)[i] = RND ? ((i * 2654435761u) ^ (i >> 3) * 40503u) & 0xbfffbfffu : (i * 2654435761u) & 0x3f803f80u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tm_s;
  if (RND && threadIdx.x < 128) {
    const uint32_t lanebase = tm + ((uint32_t)((threadIdx.x >> 5) * 32) << 16);
    for (int c = 0; c < 512; c += 4) {
      uint32_t v0 = (threadIdx.x * 977u + c * 131u) * 2654435761u & 0xbfffbfffu, v1 = v0 * 3u + 7u, v2 = v1 ^ 0x12345u, v3 = v2 * 5u;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(lanebase + c), "r"(v0 & 0xbfffbfffu), "r"(v1 & 0xbfffbfffu), "r"(v2 & 0xbfffbfffu), "r"(v3 & 0xbfffbfffu));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t sa = su32(base), sb = su32(base + A_BYTES);
    int m = 0;
    for (int i = 0; i < iters; i += 32) {
#pragma unroll
      for (int q = 0; q < 32; ++q, ++m) {
        // chunk = 4 MMAs; A slot (q/4)%8, B stage (q/4)%4
        const int slot = (q >> 2) & 7, stg = (q >> 2) & 3, kk = q & 3;
        const uint64_t bd = desc(sb + stg * N * 128) + 2 * kk;
        if (SS) {
          const uint64_t ad = desc(sa + slot * 16384) + 2 * kk;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tm), "l"(ad), "l"(bd), "r"(idesc));
        } else {
          if (RND == 8 || RND == 9) {
            // 8: D ping-pong + accumulate reset per 128-MMA tile (shift/mask only); 9: same per 108 (division)
            const int tile = RND == 8 ? (m >> 7) : m / 108;
            const bool first = RND == 8 ? ((m & 127) == 0) : (m % 108 == 0);
            const uint32_t dd = tm + (tile & 1) * N;
            const uint32_t ta = tm + 128 + slot * 32 + 8 * kk;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                         ::"r"(dd), "r"(ta), "l"(bd), "r"(idesc), "r"((uint32_t)!first));
          } else if (RND >= 3) {
            // one factor at a time: 3 accumulate predicate from a runtime register, 4 D ping-pong
            // (per 128 MMAs), 5 A slots at column 128
            const uint32_t dd = tm + (RND == 4 ? ((m >> 7) & 1) * N : 0);
            const uint32_t ta = tm + (RND == 5 ? 128 : 256) + slot * 32 + 8 * kk;
            const uint32_t acc = RND == 3 ? (uint32_t)(iters - m > 0) : 1u;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                         ::"r"(dd), "r"(ta), "l"(bd), "r"(idesc), "r"(acc));
          } else if (RND >= 2) {
            // the conv's pattern: D ping-pongs between two accumulators per 108-MMA tile,
            // A slots at 128 + 32 * slot, accumulate flag from a register
            const int tile = m / 108;
            const uint32_t dd = tm + (tile & 1) * N;
            const uint32_t acc = (m % 108) != 0;
            const uint32_t ta = tm + 128 + slot * 32 + 8 * kk;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                         ::"r"(dd), "r"(ta), "l"(bd), "r"(idesc), "r"(acc));
          } else {
          const uint32_t ta = tm + 256 + slot * 32 + 8 * kk;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                       ::"r"(tm), "r"(ta), "l"(bd), "r"(idesc));
          }
        }
        if (C <= 32 && (q + 1) % C == 0)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                       ::"r"(su32(&bar2[(q / C) & 1])) : "memory");
      }
      if (C > 32 && C < 100000 && ((i + 32) % C) == 0)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(su32(&bar2[0])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int SS, int C, int RND = 0>
void run(long long* d) {
  int smem = (SS ? 8 * 16384 : 0) + 4 * N * 128 + 1024;
  cudaFuncSetAttribute(k<N, SS, C, RND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h = 0;
  int it = 8192;
  k<N, SS, C, RND><<<148, 128, smem>>>(d, it);
  k<N, SS, C, RND><<<148, 128, smem>>>(d, it);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("rnd=%d %s N=%3d commit/%-6d %6.1f cyc/MMA (ideal %3.0f) %s\n", RND, SS ? "SS" : "TS", N, C, (double)h / it,
         128.0 * N / 256, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<64, 0, 16, 1>(d); run<64, 0, 16, 8>(d); run<64, 0, 16, 9>(d); run<64, 0, 16, 2>(d);
  return 0;
}
