// SS-form tcgen05.mma (M = 128, N = 128, K = 16, bf16) issue rate when the A
// operand is a shifted view of a dense halo brick (spconv_brick.cu): start at
// an arbitrary 128-byte row and 8-row groups SBO bytes apart, against the
// canonical 1024-aligned, SBO = 1024 layout.  One issuing thread, 27 x 4 MMAs
// per commit round (a brick's taps), B rotating over 4 stages.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro_sbo.bin tools/micro_sbo.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(sbo >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// mode bit 0: brick view; bit 1: per-tap pipeline overhead as in the kernel
// (wait on a completed mbarrier phase + tcgen05 fence before the tap's MMAs,
// a commit to a stage barrier after them); bit 2: two taps per commit round
template <int mode>
__global__ void __launch_bounds__(128, 1) k(long long* out, int rounds) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint64_t bar, done_bar, stage_bar[4];
  __shared__ uint32_t tm_s;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&done_bar)));
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(su32(&stage_bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&done_bar)));  // phase 0 complete
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tm_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // halo brick 540 rows x 128 B at 0, B: 4 stages x 16 KB after 69632
  for (int i = threadIdx.x; i < (69632 + 4 * 16384) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(base)[i] = ((i * 2654435761u) >> 3) & 0x3f803f80u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tm_s;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t sa = su32(base), sb = su32(base + 69632);
    for (int r = 0; r < rounds; ++r) {
#pragma unroll
      for (int t = 0; t < 27; ++t) {
        const int a = t / 9, b = (t / 3) % 3, c = t % 3;
        // mode 0: canonical (start 1024-aligned rows 0..127 + 8 t, SBO 1024); 1: brick view (SBO 1280)
        const uint32_t row = (mode & 1) ? a * 180 + b * 10 + c : 8 * (t % 4);
        const uint64_t ad = desc(sa + row * 128, (mode & 1) ? 1280 : 1024);
        if ((mode & 2) && (!(mode & 4) || !(t & 1))) {
          asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W2;\n}\n"
                       ::"r"(su32(&done_bar)) : "memory");
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        const uint64_t bd = desc(sb + (t & 3) * 16384, 1024);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tm), "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"((uint32_t)(t | kk)));
        if ((mode & 2) && (!(mode & 4) || (t & 1) || t == 26))
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                       ::"r"(su32(&stage_bar[t & 3])) : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

template <int mode>
void run(long long* d, const char* name) {
  const int smem = 69632 + 4 * 16384 + 1024;
  cudaFuncSetAttribute(k<mode>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h = 0;
  const int rounds = 64;
  k<mode><<<148, 128, smem>>>(d, rounds);
  k<mode><<<148, 128, smem>>>(d, rounds);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-45s: %.1f cycles per N=128 MMA (compute floor 64) %s\n", name, (double)h / (rounds * 27 * 4),
         cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<0>(d, "canonical (SBO 1024)");
  run<1>(d, "brick view (unaligned start, SBO 1280)");
  run<2>(d, "canonical + per-tap wait/fence/commit");
  run<3>(d, "brick view + per-tap wait/fence/commit");
  run<6>(d, "canonical + wait/commit per 2 taps");
  run<7>(d, "brick view + wait/commit per 2 taps");
  return 0;
}
