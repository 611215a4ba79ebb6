// Shared helpers for libfpvs (sm_100a).
#pragma once

#include <mutex>

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include <stdlib.h>

#include "../../include/fpvs.h"

namespace fpvs {

constexpr int kNumSMs = 148;

// thread-local error text behind fpvs_last_error()
int set_error(int code, const char* fmt, ...);

#define FPVS_CHECK_ARG(cond, ...)                                   \
  do {                                                              \
    if (!(cond)) return ::fpvs::set_error(FPVS_EINVAL, __VA_ARGS__); \
  } while (0)

#define FPVS_CHECK_LAUNCH(name)                                                      \
  do {                                                                               \
    cudaError_t e_ = cudaGetLastError();                                             \
    if (e_ != cudaSuccess)                                                           \
      return ::fpvs::set_error(FPVS_ECUDA, "%s: %s", name, cudaGetErrorString(e_)); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// -------- programmatic dependent launch (PDL) ------------------------------
// Conv kernels are launched with cudaLaunchAttributeProgrammaticStreamSerialization:
// a kernel may start while its predecessor drains, runs its prologue (barrier
// init, TMEM alloc, weight prefetch: data produced two or more launches back),
// and calls pdl_wait() before touching anything the predecessor writes or
// reads.  Each kernel triggers its dependents only after its own wait, so a
// kernel never overlaps anything older than its immediate predecessor.
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_release_gpu(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();  // FPVS_PDL=0 disables (read once)

template <typename... KArgs, typename... Args>
cudaError_t launch_kernel(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                          Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// -------- profiling builds ----------------------------------------------
// Per-role timestamp buffers and ablation switches exist only in a profiling
// build (-DFPVS_PROFILE; `python -m paper_2509_24677_b200.build --profile`
// writes libfpvs_prof.so).  In the production library a kernel's knob is the
// constant 0, so every debug branch folds away, no launcher reads the
// environment and no __device__ scratch is shared between concurrent launches.
#ifdef FPVS_PROFILE
#define FPVS_KNOB(p) ((p).dbg)
inline int debug_knob(const char* name) {
  const char* e = getenv(name);
  return e ? atoi(e) : 0;
}
#else
#define FPVS_KNOB(p) 0
inline int debug_knob(const char*) { return 0; }
#endif

// The kernel's dynamic shared-memory ceiling, set once per process and kernel
// (thread-safe: the C ABI may be called from several host threads).
template <auto Kernel>
inline cudaError_t set_smem_once(int bytes) {
  static std::once_flag flag;
  static cudaError_t err = cudaSuccess;
  std::call_once(flag, [&] { err = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); });
  return err;
}

inline int grid_for(long long work, int block, int per_sm = 8) {
  long long g = (work + block - 1) / block;
  long long cap = (long long)kNumSMs * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// -------- numeric conversion --------------------------------------------
template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}
template <> __device__ __forceinline__ float to_f32<uint8_t>(uint8_t v) { return (float)v; }

template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// split-branch stable sigmoid, as neural.py:151-157
__device__ __forceinline__ float sigmoidf_stable(float z) {
  if (z >= 0.f) return 1.f / (1.f + expf(-z));
  float e = expf(z);
  return e / (1.f + e);
}

__device__ __forceinline__ float apply_act(float z, int act) {
  if (act == FPVS_ACT_RELU) return fmaxf(z, 0.f);
  if (act == FPVS_ACT_SIGMOID) return sigmoidf_stable(z);
  return z;
}

// bit address of froxel (b, x, y, z) in a batch of packed grids
__device__ __forceinline__ long long bit_byte(int b, int x, int y, int z, int Nx, int Ny, int Nz) {
  return (long long)b * ((long long)(Nx >> 3) * Ny * Nz) + (x >> 3) +
         (long long)(Nx >> 3) * (y + (long long)Ny * z);
}

__device__ __forceinline__ void atomic_or_bit(uint8_t* bits, long long byte, int bit) {
  uint32_t* word = reinterpret_cast<uint32_t*>(bits + (byte & ~3LL));
  atomicOr(word, 1u << (((int)(byte & 3)) * 8 + bit));
}

}  // namespace fpvs
