// Can an SS-form tcgen05.mma read its A operand as 8-row groups that start at
// an arbitrary 128-byte row of a 128B-swizzled buffer (the swizzle written by
// absolute address), with a group stride that is not a multiple of 8 rows?
// A[h][k] = h, B = identity (K = 16 x N = 16): D[r][0] = the row the MMA used
// for output row r; expected h0 + (r / 8) * S + r % 8.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro_desc.bin tools/micro_desc.cu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(int h0, int S, int bofs_mode, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  uint8_t* A = base;               // 512 rows x 128 B
  uint8_t* B = base + 512 * 128;   // 16 rows x 128 B (1024-aligned)
  __shared__ uint64_t bar;
  __shared__ uint32_t tm_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 512 * 64; i += blockDim.x) {  // A: bf16 element (h, kk)
    const int h = i / 64, kk = i % 64, c = kk / 8, e = kk % 8;
    reinterpret_cast<__nv_bfloat16*>(A + h * 128 + ((c ^ (h & 7)) << 4))[e] = __float2bfloat16((float)h);
  }
  for (int i = tid; i < 16 * 64; i += blockDim.x) {
    const int n = i / 64, kk = i % 64, c = kk / 8, e = kk % 8;
    reinterpret_cast<__nv_bfloat16*>(B + n * 128 + ((c ^ (n & 7)) << 4))[e] = __float2bfloat16(kk == n ? 1.f : 0.f);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tm_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tm_s;
  if (tid == 0) {
    const uint32_t sa = su32(A) + h0 * 128;
    uint64_t ad = 0;
    ad |= (uint64_t)((sa & 0x3FFFF) >> 4);
    ad |= (uint64_t)1 << 16;
    ad |= (uint64_t)((S * 128) >> 4) << 32;
    ad |= (uint64_t)1 << 46;
    if (bofs_mode == 1) ad |= (uint64_t)(h0 & 7) << 49;
    ad |= (uint64_t)2 << 61;
    const uint32_t sb = su32(B);
    uint64_t bd = 0;
    bd |= (uint64_t)((sb & 0x3FFFF) >> 4);
    bd |= (uint64_t)1 << 16;
    bd |= (uint64_t)(1024 >> 4) << 32;
    bd |= (uint64_t)1 << 46;
    bd |= (uint64_t)2 << 61;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(tm), "l"(ad), "l"(bd), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    uint32_t v[2];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(v[0]), "=r"(v[1])
                 : "r"(tm + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    out[warp * 32 + lane] = __uint_as_float(v[0]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 4);
  const int smem = 512 * 128 + 16 * 128 + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int cases[][2] = {{0, 8}, {0, 10}, {3, 8}, {3, 10}, {5, 18}, {7, 13}};
  for (auto& c : cases)
    for (int mode = 0; mode < 2; ++mode) {
      k<<<1, 128, smem>>>(c[0], c[1], mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      float h[128];
      cudaMemcpy(h, d, 512, cudaMemcpyDeviceToHost);
      int bad = 0, first = -1;
      for (int r = 0; r < 128; ++r) {
        const int want = c[0] + (r / 8) * c[1] + r % 8;
        if ((int)h[r] != want) { ++bad; if (first < 0) first = r; }
      }
      printf("h0=%d S=%2d base_offset=%s: %3d / 128 rows wrong%s (first r=%d got %.0f want %d) %s\n", c[0], c[1],
             mode ? "h0&7" : "0   ", bad, bad ? "" : " OK", first, first >= 0 ? h[first] : 0.f,
             first >= 0 ? c[0] + (first / 8) * c[1] + first % 8 : 0, cudaGetErrorString(e));
    }
  return 0;
}
