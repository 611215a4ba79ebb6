// (4b) Optimizer steps on the flat fp32 master parameters, and hard
// confusion counts of packed PVS bits.
//
// The reference's update is plain SGD with a decayed rate
// (pkg/src/froxelpvs/neural.py:293-297, 481); BASELINE config 5 asks for
// AdamW with fp32 master weights.  Both run over ONE flat parameter buffer
// (all layers' weights and biases back to back) so a data-parallel step is
// one NCCL all-reduce of one flat gradient plus one launch here.
//
// fpvs_bits_confusion replaces the hard-count loop of the reference's train /
// evaluate_pairs (neural.py:423-439, 485-490): TP, FP, FN, GTP of a thresholded
// prediction against the label grid, per sample, straight from packed bits
// (HBM-bound popcounts, uint4 loads).
#include "common.cuh"

namespace fpvs {

__global__ void sgd_kernel(float* __restrict__ p, const float* __restrict__ g, long long n, float lr) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] -= lr * g[i];
}

// decoupled weight decay (AdamW): p -= lr * (mhat / (sqrt(vhat) + eps) + wd * p)
__global__ void adamw_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                             float* __restrict__ v, long long n, float lr, float b1, float b2, float eps, float wd,
                             float c1, float c2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const float mh = mi / c1, vh = vi / c2;
    p[i] -= lr * (mh / (sqrtf(vh) + eps) + wd * p[i]);
  }
}

// counts[4b..4b+3] = (TP, FP, FN, GTP) of sample b; one block per (sample, slice)
constexpr int kConfThreads = 256;
constexpr int kConfSlices = 16;

__global__ void __launch_bounds__(kConfThreads) confusion_kernel(const uint8_t* __restrict__ pred,
                                                                 const uint8_t* __restrict__ gt, long long grid_bytes,
                                                                 unsigned long long* __restrict__ part) {
  __shared__ unsigned long long red[4][kConfThreads / 32];
  const int b = blockIdx.y, sl = blockIdx.x;
  const uint8_t* pp = pred + (long long)b * grid_bytes;
  const uint8_t* gg = gt + (long long)b * grid_bytes;
  const long long per = ((grid_bytes + kConfSlices - 1) / kConfSlices + 15) / 16 * 16;
  const long long lo = sl * per, hi = min(grid_bytes, lo + per);
  unsigned long long tp = 0, fp = 0, fn = 0, gp = 0;
  const bool vec = ((reinterpret_cast<uintptr_t>(pp) | reinterpret_cast<uintptr_t>(gg)) & 15) == 0 && (lo & 15) == 0;
  long long i = lo;
  if (vec) {
    for (long long q = lo / 16 + threadIdx.x; q < hi / 16; q += kConfThreads) {
      const uint4 a = reinterpret_cast<const uint4*>(pp)[q];
      const uint4 c = reinterpret_cast<const uint4*>(gg)[q];
      const uint32_t av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        tp += __popc(av[k] & cv[k]);
        fp += __popc(av[k] & ~cv[k]);
        fn += __popc(~av[k] & cv[k]);
        gp += __popc(cv[k]);
      }
    }
    i = hi / 16 * 16;
    if (i < lo) i = lo;
  }
  for (long long e = i + threadIdx.x; e < hi; e += kConfThreads) {
    const uint32_t a = pp[e], c = gg[e];
    tp += __popc(a & c);
    fp += __popc(a & ~c & 0xffu);
    fn += __popc(~a & c & 0xffu);
    gp += __popc(c);
  }
  const unsigned long long vals[4] = {tp, fp, fn, gp};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    unsigned long long x = vals[k];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = x;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    unsigned long long s = 0;
    for (int w = 0; w < kConfThreads / 32; ++w) s += red[threadIdx.x][w];
    part[((long long)b * kConfSlices + sl) * 4 + threadIdx.x] = s;
  }
}

__global__ void confusion_reduce_kernel(const unsigned long long* __restrict__ part, int B,
                                        long long* __restrict__ counts) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 4 * B) return;
  const int b = t / 4, k = t % 4;
  unsigned long long s = 0;
  for (int sl = 0; sl < kConfSlices; ++sl) s += part[((long long)b * kConfSlices + sl) * 4 + k];
  counts[t] = (long long)s;
}

// ---- data-parallel exchange buffer ---------------------------------------
// One NCCL all-reduce per training step moves [gradient (n f32) | tail]: the
// local mean gradient pre-scaled by B_local / B_global (so the sum over ranks
// is the reference's batch mean, neural.py:472-477) and a tail that carries
// the step's loss and hard counts.  Counts are split into 12-bit digits so
// their f32 sums stay exact (< 2^24 per digit for up to 4096 ranks).
//   tail[0] = batch-mean loss x local samples   tail[1] = local samples
//   tail[2 + 2q], tail[3 + 2q] = (count_q >> 12, count_q & 4095), q = TP, FP, FN, GTP
constexpr int kExchTail = FPVS_EXCHANGE_TAIL;

__global__ void exchange_pack_kernel(float* __restrict__ flat, long long n, float weight,
                                     const double* __restrict__ loss, const long long* __restrict__ counts, int B) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    flat[i] *= weight;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    float* t = flat + n;
    long long c[4] = {0, 0, 0, 0};
    for (int b = 0; b < B; ++b)
      for (int q = 0; q < 4; ++q) c[q] += counts[4 * b + q];
    t[0] = B > 0 ? (float)(loss[0] * B) : 0.f;
    t[1] = (float)B;
    for (int q = 0; q < 4; ++q) {
      t[2 + 2 * q] = (float)(c[q] >> 12);
      t[3 + 2 * q] = (float)(c[q] & 4095);
    }
  }
}

// acc: [0] sum of batch-mean loss x batch size, [1] samples, [2..5] TP FP FN GTP,
//      [6] index of the first batch with a non-finite loss (-1 none), [7] that loss
__global__ void exchange_accumulate_kernel(const float* __restrict__ t, double* __restrict__ acc, int batch_index) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double ls = t[0], ns = t[1];
  const double mean = ns > 0 ? ls / ns : 0.0;
  if (!isfinite(mean) && acc[6] < 0) {
    acc[6] = batch_index;
    acc[7] = mean;
  }
  acc[0] += ls;
  acc[1] += ns;
  for (int q = 0; q < 4; ++q) acc[2 + q] += (double)t[2 + 2 * q] * 4096.0 + (double)t[3 + 2 * q];
}

}  // namespace fpvs

using namespace fpvs;

extern "C" int fpvs_exchange_pack(float* flat, size_t n, float weight, const double* loss, const int64_t* counts,
                                  int B, void* stream) {
  FPVS_CHECK_ARG(flat, "null pointer");
  FPVS_CHECK_ARG(B == 0 || (loss && counts), "loss and counts are required with B > 0");
  exchange_pack_kernel<<<grid_for((long long)n, 256), 256, 0, as_stream(stream)>>>(
      flat, (long long)n, weight, loss, (const long long*)counts, B);
  FPVS_CHECK_LAUNCH("fpvs_exchange_pack");
  return FPVS_OK;
}

extern "C" int fpvs_exchange_accumulate(const float* tail, double* acc, int batch_index, void* stream) {
  FPVS_CHECK_ARG(tail && acc, "null pointer");
  exchange_accumulate_kernel<<<1, 32, 0, as_stream(stream)>>>(tail, acc, batch_index);
  FPVS_CHECK_LAUNCH("fpvs_exchange_accumulate");
  return FPVS_OK;
}

extern "C" int fpvs_sgd_step(float* params, const float* grads, size_t n, float lr, void* stream) {
  FPVS_CHECK_ARG(params && grads, "null pointer");
  if (!n) return FPVS_OK;
  sgd_kernel<<<grid_for((long long)n, 256), 256, 0, as_stream(stream)>>>(params, grads, (long long)n, lr);
  FPVS_CHECK_LAUNCH("fpvs_sgd_step");
  return FPVS_OK;
}

extern "C" int fpvs_adamw_step(float* params, const float* grads, float* m, float* v, size_t n, float lr,
                               float beta1, float beta2, float eps, float weight_decay, int step, void* stream) {
  FPVS_CHECK_ARG(params && grads && m && v, "null pointer");
  FPVS_CHECK_ARG(step >= 1, "AdamW step count starts at 1");
  FPVS_CHECK_ARG(beta1 >= 0.f && beta1 < 1.f && beta2 >= 0.f && beta2 < 1.f, "betas must lie in [0, 1)");
  if (!n) return FPVS_OK;
  const float c1 = 1.f - powf(beta1, (float)step), c2 = 1.f - powf(beta2, (float)step);
  adamw_kernel<<<grid_for((long long)n, 256), 256, 0, as_stream(stream)>>>(params, grads, m, v, (long long)n, lr,
                                                                           beta1, beta2, eps, weight_decay, c1, c2);
  FPVS_CHECK_LAUNCH("fpvs_adamw_step");
  return FPVS_OK;
}

extern "C" size_t fpvs_bits_confusion_workspace_size(int B) {
  return sizeof(unsigned long long) * 4 * (size_t)kConfSlices * (size_t)(B > 0 ? B : 0);
}

extern "C" int fpvs_bits_confusion(const uint8_t* pred_bits, const uint8_t* gt_bits, int B, long long grid_bytes,
                                   long long* counts, void* workspace, size_t workspace_bytes, void* stream) {
  FPVS_CHECK_ARG(pred_bits && gt_bits && counts && workspace, "null pointer");
  FPVS_CHECK_ARG(B >= 1 && grid_bytes >= 1, "bad batch");
  FPVS_CHECK_ARG(workspace_bytes >= fpvs_bits_confusion_workspace_size(B), "workspace too small");
  cudaStream_t s = as_stream(stream);
  confusion_kernel<<<dim3(kConfSlices, B), kConfThreads, 0, s>>>(pred_bits, gt_bits, grid_bytes,
                                                                 (unsigned long long*)workspace);
  confusion_reduce_kernel<<<(4 * B + 127) / 128, 128, 0, s>>>((const unsigned long long*)workspace, B, counts);
  FPVS_CHECK_LAUNCH("fpvs_bits_confusion");
  return FPVS_OK;
}

namespace fpvs {
__global__ void cast_bf16_kernel(const float* __restrict__ src, long long n, __nv_bfloat16* __restrict__ dst) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    dst[t] = __float2bfloat16_rn(src[t]);
}
__global__ void cast_bf16_rows_kernel(const float* __restrict__ src, int cols, const int* n_dev, int cap,
                                      __nv_bfloat16* __restrict__ dst) {
  const long long n = (long long)min(*n_dev, cap) * cols;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    dst[t] = __float2bfloat16_rn(src[t]);
}
}  // namespace fpvs

extern "C" int fpvs_cast_bf16_rows(const float* src, int cols, const int32_t* n_dev, int cap, void* dst,
                                   void* stream) {
  FPVS_CHECK_ARG(src && dst && n_dev && cols > 0 && cap >= 0, "bad arguments");
  if (cap == 0) return FPVS_OK;
  fpvs::cast_bf16_rows_kernel<<<fpvs::grid_for((long long)cap * cols, 256, 4), 256, 0, fpvs::as_stream(stream)>>>(
      src, cols, n_dev, cap, (__nv_bfloat16*)dst);
  FPVS_CHECK_LAUNCH("fpvs_cast_bf16_rows");
  return FPVS_OK;
}

extern "C" int fpvs_cast_bf16(const float* src, long long n, void* dst, void* stream) {
  FPVS_CHECK_ARG(src && dst && n >= 0, "bad arguments");
  if (n == 0) return FPVS_OK;
  fpvs::cast_bf16_kernel<<<fpvs::grid_for(n, 256), 256, 0, fpvs::as_stream(stream)>>>(src, n, (__nv_bfloat16*)dst);
  FPVS_CHECK_LAUNCH("fpvs_cast_bf16");
  return FPVS_OK;
}
