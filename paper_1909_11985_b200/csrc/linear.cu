// Linear-model SGD step on the GPU in f64, bit-identical to the reference trainer
// (src/trainer.cpp:14-61) and collective (src/allreduce.cpp:60-148).
//
// Bit-exactness comes from reproducing the reference's operation order and suppressing
// FMA contraction (__dmul_rn / __dadd_rn):
//   local_gradient : z_j = sum_i w_i a_ji (sequential per sample), s_j = z_j - b_j;
//                    g_i  = sum_j s_j a_ji  in draw order (one thread per feature i)
//   batch_loss     : sum_j 0.5*e_j*e_j in draw order
//   sgd_step       : w_i -= (eta/count) * g_i
//   ring allreduce : chunk c = [c*len/n, (c+1)*len/n) folds ranks c, c+1, ... left to right
// The logistic model goes through CUDA's exp/log1p, which agree with glibc to within an
// ulp, so it is checked to 1e-12 relative instead of bit-for-bit.
//
// These are latency-bound at the reference's sizes (dim 64, batch 64); they exist for the
// bit-exact parity gate on the C1 job, not for throughput (BASELINE.json configs[0]).
#include <cuda_runtime.h>

#include <cstdint>

#include "edl_internal.hpp"
#include "kernels.hpp"

namespace edl {
namespace {

// Phase 1: per-sample scale s_j (trainer.cpp:18-26).
__global__ void sample_scale_kernel(int kind, const double* __restrict__ w,
                                    const double* __restrict__ x, const double* __restrict__ y,
                                    int64_t n, int dim, double* __restrict__ scale) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  const double* a = x + j * dim;
  double z = 0.0;
  for (int i = 0; i < dim; ++i) z = __dadd_rn(z, __dmul_rn(w[i], a[i]));
  double s;
  if (kind == EDL_MODEL_LEAST_SQUARES) {
    s = __dsub_rn(z, y[j]);
  } else {
    const double m = __dmul_rn(-y[j], z);
    s = __ddiv_rn(-y[j], __dadd_rn(1.0, exp(-m)));
  }
  scale[j] = s;
}

// Phase 2: g_i = sum_j s_j a_ji in draw order; grad_out[dim] = count.
__global__ void feature_sum_kernel(const double* __restrict__ x, const double* __restrict__ scale,
                                   int64_t n, int dim, double* __restrict__ g) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < dim) {
    double acc = 0.0;
    for (int64_t j = 0; j < n; ++j) acc = __dadd_rn(acc, __dmul_rn(scale[j], x[j * dim + i]));
    g[i] = acc;
  }
  if (i == 0) g[dim] = static_cast<double>(n);
}

__global__ void sample_loss_kernel(int kind, const double* __restrict__ w,
                                   const double* __restrict__ x, const double* __restrict__ y,
                                   int64_t n, int dim, double* __restrict__ out) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  const double* a = x + j * dim;
  double z = 0.0;
  for (int i = 0; i < dim; ++i) z = __dadd_rn(z, __dmul_rn(w[i], a[i]));
  if (kind == EDL_MODEL_LEAST_SQUARES) {
    const double e = __dsub_rn(z, y[j]);
    out[j] = __dmul_rn(__dmul_rn(0.5, e), e);  // 0.5 * e * e, trainer.cpp:48
  } else {
    out[j] = log1p(exp(__dmul_rn(-y[j], z)));
  }
}

__global__ void ordered_total_kernel(const double* __restrict__ v, int64_t n,
                                     double* __restrict__ out) {
  double acc = 0.0;
  for (int64_t j = 0; j < n; ++j) acc = __dadd_rn(acc, v[j]);
  *out = acc;
}

__global__ void sgd_kernel(double* __restrict__ w, const double* __restrict__ g, double scale,
                           int dim, int device_count, double eta) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= dim) return;
  double sc = scale;
  if (device_count) {
    const double c = g[dim];
    if (c == 0.0) return;  // nothing applied (oracle_replay skips count 0)
    sc = __ddiv_rn(eta, c);
  }
  w[i] = __dsub_rn(w[i], __dmul_rn(sc, g[i]));
}

// Workspace-free variants for the C-ABI entry points (edl_local_gradient / edl_batch_loss:
// no allocation on the call path).  Same operation order: per chunk of blockDim samples the
// threads compute s_j (or the loss term) into shared memory, then the features (gradient) or
// thread 0 (loss) fold the chunk in draw order before the next chunk.  Each block of the
// gradient kernel owns blockDim features and recomputes the chunk's s_j.
constexpr int kFusedThreads = 128;

__device__ __forceinline__ double sample_scale(int kind, const double* __restrict__ w,
                                               const double* __restrict__ a, double b, int dim) {
  double z = 0.0;
  for (int i = 0; i < dim; ++i) z = __dadd_rn(z, __dmul_rn(w[i], a[i]));
  if (kind == EDL_MODEL_LEAST_SQUARES) return __dsub_rn(z, b);
  const double m = __dmul_rn(-b, z);
  return __ddiv_rn(-b, __dadd_rn(1.0, exp(-m)));
}

__global__ void __launch_bounds__(kFusedThreads)
local_gradient_fused_kernel(int kind, const double* __restrict__ w, const double* __restrict__ x,
                            const double* __restrict__ y, int64_t n, int dim,
                            double* __restrict__ g) {
  __shared__ double sc[kFusedThreads];
  const int i = blockIdx.x * kFusedThreads + threadIdx.x;
  double acc = 0.0;
  for (int64_t j0 = 0; j0 < n; j0 += kFusedThreads) {
    const int64_t j = j0 + threadIdx.x;
    if (j < n) sc[threadIdx.x] = sample_scale(kind, w, x + j * dim, y[j], dim);
    __syncthreads();
    const int m = n - j0 < kFusedThreads ? static_cast<int>(n - j0) : kFusedThreads;
    if (i < dim)
      for (int k = 0; k < m; ++k) acc = __dadd_rn(acc, __dmul_rn(sc[k], x[(j0 + k) * dim + i]));
    __syncthreads();
  }
  if (i < dim) g[i] = acc;
  if (i == 0) g[dim] = static_cast<double>(n);
}

__global__ void __launch_bounds__(kFusedThreads)
batch_loss_fused_kernel(int kind, const double* __restrict__ w, const double* __restrict__ x,
                        const double* __restrict__ y, int64_t n, int dim,
                        double* __restrict__ out) {
  __shared__ double lv[kFusedThreads];
  double acc = 0.0;
  for (int64_t j0 = 0; j0 < n; j0 += kFusedThreads) {
    const int64_t j = j0 + threadIdx.x;
    if (j < n) {
      const double* a = x + j * dim;
      double z = 0.0;
      for (int i = 0; i < dim; ++i) z = __dadd_rn(z, __dmul_rn(w[i], a[i]));
      if (kind == EDL_MODEL_LEAST_SQUARES) {
        const double e = __dsub_rn(z, y[j]);
        lv[threadIdx.x] = __dmul_rn(__dmul_rn(0.5, e), e);
      } else {
        lv[threadIdx.x] = log1p(exp(__dmul_rn(-y[j], z)));
      }
    }
    __syncthreads();
    const int m = n - j0 < kFusedThreads ? static_cast<int>(n - j0) : kFusedThreads;
    if (threadIdx.x == 0)
      for (int k = 0; k < m; ++k) acc = __dadd_rn(acc, lv[k]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = acc;
}

struct PtrArray {
  const double* p[64];
};

__global__ void ring_allreduce_kernel(PtrArray in, int n, size_t len, int average,
                                      double* __restrict__ out) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < len;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    int c = 0;  // chunk owning element i: lo(c) <= i < lo(c+1)
    while (c + 1 < n && len * static_cast<size_t>(c + 1) / static_cast<size_t>(n) <= i) ++c;
    double acc = in.p[c][i];
    for (int k = 1; k < n; ++k) acc = __dadd_rn(acc, in.p[(c + k) % n][i]);
    if (average) acc = __ddiv_rn(acc, static_cast<double>(n));
    out[i] = acc;
  }
}

__global__ void ordered_sum_kernel(PtrArray in, int n, double* __restrict__ out) {
  double acc = 0.0;
  for (int k = 0; k < n; ++k) acc = __dadd_rn(acc, *in.p[k]);
  *out = acc;
}

}  // namespace

int linear_local_gradient(int kind, const double* w, const double* x, const double* y, int64_t n,
                          int dim, double* grad_out, double* scale_ws, cudaStream_t s) {
  if (!scale_ws) {  // C-ABI call: no workspace, one fused launch
    local_gradient_fused_kernel<<<(dim + kFusedThreads - 1) / kFusedThreads, kFusedThreads, 0,
                                  s>>>(kind, w, x, y, n, dim, grad_out);
    EDL_CUDA_TRY(cudaGetLastError());
    return EDL_OK;
  }
  if (n > 0) {
    sample_scale_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, s>>>(kind, w, x, y, n,
                                                                               dim, scale_ws);
  }
  feature_sum_kernel<<<(dim + 127) / 128, 128, 0, s>>>(x, scale_ws, n, dim, grad_out);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int linear_batch_loss(int kind, const double* w, const double* x, const double* y, int64_t n,
                      int dim, double* loss_out, double* ws, cudaStream_t s) {
  if (!ws) {  // C-ABI call: no workspace, one launch
    batch_loss_fused_kernel<<<1, kFusedThreads, 0, s>>>(kind, w, x, y, n, dim, loss_out);
    EDL_CUDA_TRY(cudaGetLastError());
    return EDL_OK;
  }
  if (n > 0)
    sample_loss_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, s>>>(kind, w, x, y, n,
                                                                              dim, ws);
  ordered_total_kernel<<<1, 1, 0, s>>>(ws, n, loss_out);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int linear_sgd(double* w, const double* g, int64_t count, double eta, int dim, cudaStream_t s) {
  if (count == 0) return fail(EDL_EINVAL, "sgd_step with zero sample count");
  const bool dev = count < 0;
  const double scale = dev ? 0.0 : eta / static_cast<double>(count);
  sgd_kernel<<<(dim + 127) / 128, 128, 0, s>>>(w, g, scale, dim, dev ? 1 : 0, eta);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int ring_allreduce_f64(const double* const* inputs, int n, size_t len, int op, double* out,
                       cudaStream_t s) {
  if (n < 1 || n > 64) return fail(EDL_EINVAL, "ring_allreduce: 1 <= n <= 64");
  PtrArray a{};
  for (int k = 0; k < n; ++k) a.p[k] = inputs[k];
  if (len == 0) return EDL_OK;
  const unsigned blocks = static_cast<unsigned>((len + 255) / 256 < 1024 ? (len + 255) / 256 : 1024);
  ring_allreduce_kernel<<<blocks, 256, 0, s>>>(a, n, len, op == EDL_REDUCE_AVERAGE, out);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int ordered_sum_f64(const double* const* inputs, int n, double* out, cudaStream_t s) {
  if (n < 1 || n > 64) return fail(EDL_EINVAL, "ordered_sum: 1 <= n <= 64");
  PtrArray a{};
  for (int k = 0; k < n; ++k) a.p[k] = inputs[k];
  ordered_sum_kernel<<<1, 1, 0, s>>>(a, n, out);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

}  // namespace edl
