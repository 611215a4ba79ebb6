// tcgen05.mma (M=128, N=64 or 128, K=16, bf16) issue cost while other warps
// load the same ports the halo conv's builders use: tcgen05.st into TMEM
// (A slots), ld.shared 16-byte reads (the halo), or both.  One CTA per SM,
// 12 warps: warp 0 lane 0 issues MMAs (commit every 16), warps 4..11 are the
// "builders" (a fixed amount of work each), warps 1..3 idle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro_contend.bin tools/micro_contend.cu
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

// MODE bit 0: builders tcgen05.st; bit 1: builders ld.shared; MMA_ON: MMA thread active
template <int N, int MODE, int MMA_ON>
__global__ void __launch_bounds__(384, 1) k(long long* out, int iters, int biters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t bar, bar2[2], spinbar;
  __shared__ uint32_t tm_s;
  __shared__ long long t_mma, t_b[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar2[0])), "r"(1 << 20));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar2[1])), "r"(1 << 20));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&spinbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tm_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // smem: B 4 stages x N*128 at 0; halo 64 KB after
  for (int i = threadIdx.x; i < (4 * N * 128 + 65536) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(base)[i] = (i * 2654435761u) & 0x3f803f80u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tm_s;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (warp == 0 && lane == 0 && MMA_ON) {
    long long t0 = clock64();
    const uint32_t sb = su32(base);
    for (int i = 0; i < iters; i += 16) {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int slot = (q >> 2) & 7, stg = (q >> 2) & 3, kk = q & 3;
        const uint64_t bd = desc(sb + stg * N * 128) + 2 * kk;
        const uint32_t ta = tm + 256 + slot * 32 + 8 * kk;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tm), "r"(ta), "l"(bd), "r"(idesc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   ::"r"(su32(&bar2[(i >> 4) & 1])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
    t_mma = clock64() - t0;
  }
  if (warp >= 4 && MODE == 4) {
    const int bw = warp - 4;
    long long t0 = clock64();
    int n = 0;
    while (clock64() - t0 < (long long)biters) {
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n}\n" ::"r"(su32(&spinbar)) : "memory");
      ++n;
    }
    if (lane == 0) t_b[bw] = n;
  } else if (warp >= 4 && MODE == 5) {
    const int bw = warp - 4;
    long long t0 = clock64();
    int n = 0;
    uint32_t x = lane;
    while (clock64() - t0 < (long long)biters) {
#pragma unroll
      for (int i = 0; i < 16; ++i) x = x * 1664525u + 1013904223u;
      ++n;
    }
    if (lane == 0) t_b[bw] = n + (x == 7);
  } else if (warp >= 4) {
    const int bw = warp - 4, q4 = bw & 3;
    long long t0 = clock64();
    const uint8_t* halo = base + 4 * N * 128;
    uint32_t acc = 0;
    for (int it = 0; it < biters; ++it) {
      uint32_t v[32];
      if (MODE & 2) {
        const int row = (lane * 7 + it * 13 + bw * 3) & 511;
#pragma unroll
        for (int pc = 0; pc < 8; ++pc) {
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[4 * pc]), "=r"(v[4 * pc + 1]), "=r"(v[4 * pc + 2]), "=r"(v[4 * pc + 3])
                       : "r"(su32(halo + row * 128 + ((pc ^ (row & 7)) << 4))));
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = it + i;
      }
      if (MODE & 1) {
        // A slots 256 + 32 * (8 + ...) would collide with the MMA's reads; write
        // the same column range anyway (bandwidth, not correctness)
        const uint32_t taddr = tm + ((uint32_t)(q4 * 32) << 16) + 256 + ((it + bw) & 7) * 32;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
            "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
            "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
            "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += v[i];
      }
    }
    if (lane == 0) t_b[bw] = clock64() - t0;
    if (acc == 0x12345) t_b[bw] = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    out[0] = MMA_ON ? t_mma : 0;
    long long m = 0;
    for (int i = 0; i < 8; ++i) m = t_b[i] > m ? t_b[i] : m;
    out[1] = m;
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int MODE, int MMA_ON>
void run(long long* d, int biters) {
  int smem = 4 * N * 128 + 65536 + 1024;
  cudaFuncSetAttribute(k<N, MODE, MMA_ON>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h[2] = {0, 0};
  int it = 8192;
  k<N, MODE, MMA_ON><<<148, 384, smem>>>(d, it, biters);
  k<N, MODE, MMA_ON><<<148, 384, smem>>>(d, it, biters);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const char* mn[] = {"none", "tmem st", "lds", "lds+tmem st", "try_wait spin", "alu spin"};
  // builders move 4 KB (one 32-lane x 128 B slab) per warp-iteration
  printf("N=%3d builders %-12s mma %s: %6.1f cyc/MMA | builders %6.0f cyc total (%5.1f B/cyc per port-stream)  %s\n", N,
         mn[MODE], MMA_ON ? "on " : "off", MMA_ON ? (double)h[0] / it : 0.0, (double)h[1],
         h[1] ? 8.0 * 4096 * biters / h[1] : 0.0, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  run<64, 0, 1>(d, 1);
  run<64, 4, 1>(d, 400000);
  run<64, 5, 1>(d, 400000);
  run<128, 0, 1>(d, 1);
  run<128, 4, 1>(d, 600000);
  run<128, 5, 1>(d, 600000);
  return 0;
}
