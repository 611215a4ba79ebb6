// The halo conv's producer -> MMA -> producer handoff in isolation: 8 builder
// warps (two groups, alternating chunks; one arrival per warp per chunk), one
// "weight" lane (one arrival per stage), one MMA lane (waits full[stage],
// optionally issues 4 MMAs per chunk, commits empty[stage]).  NS stages of G
// chunks.  Measures cycles per chunk for the pure synchronisation skeleton and
// with MMAs (N = 64, A from TMEM, dummy data).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro_pipe.bin tools/micro_pipe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}\n"
               ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity, int ns) {
  uint32_t ok = 0;
  while (true) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    if (ok) return;
    __nanosleep(ns);
  }
}
__device__ __forceinline__ void mbar_wait_hint(uint32_t bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t@!p bra W_%=;\n}\n"
               ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
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

template <int NS, int G, int MMA, int FENCE, int WAIT = 0>
__global__ void __launch_bounds__(384, 1) k(long long* out, int nchunks) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  __shared__ uint32_t tm_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(su32(&full[s]), 4 * G + 1);
      mbar_init(su32(&empty[s]), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 11) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tm_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 4 * 8192 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3f803f80u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tm_s;
  long long t0 = clock64();
  const int nst = nchunks / G;
  if (warp < 8) {
    const int bg = warp >> 2;
    for (int q = 0; q < nchunks; ++q) {
      if ((q & 1) != bg) continue;
      const int st = q / G, stage = st % NS;
      if (WAIT == 9) { mbar_wait(su32(&empty[stage]), ((st / NS) & 1) ^ 1); continue; }
      if (WAIT == 1) mbar_wait_sleep(su32(&empty[stage]), ((st / NS) & 1) ^ 1, 32);
      else if (WAIT == 2) mbar_wait_hint(su32(&empty[stage]), ((st / NS) & 1) ^ 1);
      else if (WAIT == 3) { if (bg == 1 || (warp & 3) != 0) mbar_wait_sleep(su32(&empty[stage]), ((st / NS) & 1) ^ 1, 64); else mbar_wait(su32(&empty[stage]), ((st / NS) & 1) ^ 1); }
      else mbar_wait(su32(&empty[stage]), ((st / NS) & 1) ^ 1);
      if (FENCE) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (FENCE >= 2) {
        // the builders' TMEM store of one 128-row x 64-channel A chunk (warp = lane quadrant)
        const uint32_t q4 = warp & 3;
        const uint32_t ta = tm + (q4 * 32 << 16) + 128 + ((stage * G + q % G) % 8) * 32;
        uint32_t v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = (q * 977u + i * 131u + lane) * 2654435761u & 0x3fff3fffu;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
            "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
            "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
            "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
        if (FENCE == 2) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      if (FENCE) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(su32(&full[stage]));
    }
  } else if (warp == 10) {
    if (lane == 0)
      for (int st = 0; st < nst; ++st) {
        const int stage = st % NS;
        mbar_wait(su32(&empty[stage]), ((st / NS) & 1) ^ 1);
        if (WAIT != 9) mbar_arrive(su32(&full[stage]));
      }
  } else if (warp == 11) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint64_t bd = desc(su32(base));
      for (int st = 0; st < nst; ++st) {
        const int stage = st % NS;
        if (WAIT != 9) mbar_wait(su32(&full[stage]), (st / NS) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (MMA) {
#pragma unroll
          for (int g = 0; g < G; ++g)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                           ::"r"(tm), "r"(tm + 128 + (stage * G + g) % 8 * 32 + 8 * kk), "l"(bd + 2 * kk), "r"(idesc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(su32(&empty[stage])) : "memory");
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (warp == 11) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int NS, int G, int MMA, int FENCE, int WAIT = 0>
void run(long long* d) {
  const int smem = 4 * 8192 + 1024;
  cudaFuncSetAttribute(k<NS, G, MMA, FENCE, WAIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int nchunks = 27 * 40;
  long long h = 0;
  k<NS, G, MMA, FENCE, WAIT><<<148, 384, smem>>>(d, nchunks);
  k<NS, G, MMA, FENCE, WAIT><<<148, 384, smem>>>(d, nchunks);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("wait=%d NS=%d G=%d mma=%d fence=%d: %7.1f cycles / chunk (4 MMAs ideal 128, floor ~180)  %s\n", WAIT, NS, G, MMA, FENCE,
         (double)h / nchunks, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<2, 4, 1, 1, 0>(d); run<2, 4, 1, 2, 0>(d); run<2, 4, 1, 3, 0>(d); run<2, 4, 0, 2, 0>(d);
  return 0;
}
