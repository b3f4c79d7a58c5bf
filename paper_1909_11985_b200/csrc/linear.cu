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

#include <atomic>
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

// Job-path variants: the same operation order, with the batch streamed through shared memory
// by asynchronous copies (cp.async, a 4-deep ring) so the dependent f64 adds -- the reference
// folds left to right, trainer.cpp:18-28 -- never wait on memory.  One warp per 32 samples
// stages 32-row x 64-dim tiles and every lane folds its own sample's products in dimension
// order: z_j = sum_i w_i a_ji exactly as the reference.  z is kept for the loss (batch_loss
// uses the same w, trainer.cpp:41-54).
constexpr int kZChunk = 64;
constexpr int kZStages = 4;
constexpr int kZRow = kZChunk + 1;  // padded row: lanes reading their own rows hit distinct banks
constexpr size_t kZSmem = sizeof(double) * kZStages * (32 * kZRow + kZChunk);

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst))),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__global__ void __launch_bounds__(32)
sample_scale_z_kernel(int kind, const double* __restrict__ w, const double* __restrict__ x,
                      const double* __restrict__ y, int64_t n, int dim,
                      double* __restrict__ scale, double* __restrict__ zout) {
  extern __shared__ double zsm[];  // [kZStages][32][kZRow] tiles, then [kZStages][kZChunk] w
  double* wst = zsm + kZStages * 32 * kZRow;
  const int lane = threadIdx.x;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * 32, j = j0 + lane;
  const int rows = n - j0 < 32 ? static_cast<int>(n - j0) : 32;
  const int n_chunks = (dim + kZChunk - 1) / kZChunk;
  auto load = [&](int c) {
    const int c0 = c * kZChunk, cw = dim - c0 < kZChunk ? dim - c0 : kZChunk;
    double* t = zsm + (c % kZStages) * 32 * kZRow;
    if (rows == 32 && cw == kZChunk) {  // full tile: plain strides, no index arithmetic
      const double* src = x + j0 * dim + c0 + lane;
#pragma unroll 8
      for (int r = 0; r < 32; ++r) {
        cp_async8(t + r * kZRow + lane, src + static_cast<int64_t>(r) * dim);
        cp_async8(t + r * kZRow + lane + 32, src + static_cast<int64_t>(r) * dim + 32);
      }
    } else {
      for (int idx = lane; idx < rows * cw; idx += 32) {
        const int r = idx / cw, k = idx - r * cw;
        cp_async8(t + r * kZRow + k, x + (j0 + r) * dim + c0 + k);
      }
    }
    for (int k = lane; k < cw; k += 32) cp_async8(wst + (c % kZStages) * kZChunk + k, w + c0 + k);
  };
  for (int c = 0; c < kZStages - 1; ++c) {
    if (c < n_chunks) load(c);
    cp_async_commit();  // (empty groups keep the wait count uniform)
  }
  double z = 0.0;
  for (int c = 0; c < n_chunks; ++c) {
    if (c + kZStages - 1 < n_chunks) load(c + kZStages - 1);
    cp_async_commit();
    cp_async_wait<kZStages - 1>();  // chunk c has landed (this lane's copies)
    __syncwarp();                   // ... and every lane's
    const int cw = dim - c * kZChunk < kZChunk ? dim - c * kZChunk : kZChunk;
    const double* t = zsm + (c % kZStages) * 32 * kZRow + lane * kZRow;
    const double* ws = wst + (c % kZStages) * kZChunk;
    if (cw == kZChunk) {  // full chunk: constant trip count, the loads run ahead of the adds
      if (lane < rows) {
#pragma unroll
        for (int i = 0; i < kZChunk; ++i) z = __dadd_rn(z, __dmul_rn(ws[i], t[i]));
      }
    } else if (lane < rows) {
      for (int i = 0; i < cw; ++i) z = __dadd_rn(z, __dmul_rn(ws[i], t[i]));
    }
    __syncwarp();  // the stage is refilled next iteration
  }
  if (j >= n) return;
  double s;
  if (kind == EDL_MODEL_LEAST_SQUARES) {
    s = __dsub_rn(z, y[j]);
  } else {
    const double m = __dmul_rn(-y[j], z);
    s = __ddiv_rn(-y[j], __dadd_rn(1.0, exp(-m)));
  }
  scale[j] = s;
  zout[j] = z;
}

// g_i = sum_j s_j a_ji in draw order, 64 features per CTA (64 CTAs at dim 4096): 32-sample x
// 64-feature tiles stream through a 4-deep cp.async ring, each lane folds its feature's column.
constexpr int kFRows = 32;
constexpr size_t kFSmem = sizeof(double) * kZStages * (kFRows * 64 + kFRows);

__global__ void __launch_bounds__(64)
feature_sum_wide_kernel(const double* __restrict__ x, const double* __restrict__ scale,
                        int64_t n, int dim, double* __restrict__ g) {
  extern __shared__ double fsm[];  // [kZStages][kFRows][64] tiles, then [kZStages][kFRows] s
  double* sst = fsm + kZStages * kFRows * 64;
  const int t = threadIdx.x;
  const int f0 = blockIdx.x * 64, i = f0 + t;
  const int fw = dim - f0 < 64 ? dim - f0 : 64;
  const int n_chunks = static_cast<int>((n + kFRows - 1) / kFRows);
  auto load = [&](int c) {
    const int64_t r0 = static_cast<int64_t>(c) * kFRows;
    const int rows = n - r0 < kFRows ? static_cast<int>(n - r0) : kFRows;
    double* tile = fsm + (c % kZStages) * kFRows * 64;
    if (fw == 64) {  // full-width column block: thread t copies column t of every row
      const double* src = x + r0 * dim + f0 + t;
#pragma unroll 8
      for (int r = 0; r < rows; ++r) cp_async8(tile + r * 64 + t, src + static_cast<int64_t>(r) * dim);
    } else {
      for (int idx = t; idx < rows * fw; idx += 64) {
        const int r = idx / fw, k = idx - r * fw;
        cp_async8(tile + r * 64 + k, x + (r0 + r) * dim + f0 + k);
      }
    }
    for (int r = t; r < rows; r += 64) cp_async8(sst + (c % kZStages) * kFRows + r, scale + r0 + r);
  };
  for (int c = 0; c < kZStages - 1; ++c) {
    if (c < n_chunks) load(c);
    cp_async_commit();
  }
  double acc = 0.0;
  for (int c = 0; c < n_chunks; ++c) {
    if (c + kZStages - 1 < n_chunks) load(c + kZStages - 1);
    cp_async_commit();
    cp_async_wait<kZStages - 1>();
    __syncthreads();
    const int64_t r0 = static_cast<int64_t>(c) * kFRows;
    const int rows = n - r0 < kFRows ? static_cast<int>(n - r0) : kFRows;
    const double* tile = fsm + (c % kZStages) * kFRows * 64 + t;
    const double* ss = sst + (c % kZStages) * kFRows;
    if (t < fw && rows == kFRows) {
#pragma unroll
      for (int r = 0; r < kFRows; ++r) acc = __dadd_rn(acc, __dmul_rn(ss[r], tile[r * 64]));
    } else if (t < fw) {
      for (int r = 0; r < rows; ++r) acc = __dadd_rn(acc, __dmul_rn(ss[r], tile[r * 64]));
    }
    __syncthreads();
  }
  if (i < dim && t < fw) g[i] = acc;
  if (i == 0) g[dim] = static_cast<double>(n);
}

// batch_loss from the z of the gradient pass: per-sample terms in parallel, folded in draw
// order by one thread (trainer.cpp:41-54).
__global__ void __launch_bounds__(256)
loss_from_z_kernel(int kind, const double* __restrict__ z, const double* __restrict__ y,
                   int64_t n, double* __restrict__ out) {
  __shared__ double lv[256];
  double acc = 0.0;
  for (int64_t j0 = 0; j0 < n; j0 += 256) {
    const int64_t j = j0 + threadIdx.x;
    if (j < n) {
      if (kind == EDL_MODEL_LEAST_SQUARES) {
        const double e = __dsub_rn(z[j], y[j]);
        lv[threadIdx.x] = __dmul_rn(__dmul_rn(0.5, e), e);
      } else {
        lv[threadIdx.x] = log1p(exp(__dmul_rn(-y[j], z[j])));
      }
    }
    __syncthreads();
    const int m = n - j0 < 256 ? static_cast<int>(n - j0) : 256;
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
  // scale_ws holds [n] per-sample scales then [n] dot products z (linear_batch_loss_from_z)
  static std::atomic<uint64_t> attr_set{0};  // dynamic smem above 48 KB, once per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_set.load() >> dev & 1)) {
    EDL_CUDA_TRY(cudaFuncSetAttribute(sample_scale_z_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kZSmem));
    EDL_CUDA_TRY(cudaFuncSetAttribute(feature_sum_wide_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmem));
    attr_set.fetch_or(1ull << dev);
  }
  if (n > 0) {
    sample_scale_z_kernel<<<static_cast<unsigned>((n + 31) / 32), 32, kZSmem, s>>>(
        kind, w, x, y, n, dim, scale_ws, scale_ws + n);
  }
  feature_sum_wide_kernel<<<(dim + 63) / 64, 64, kFSmem, s>>>(x, scale_ws, n, dim, grad_out);
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

int linear_batch_loss_from_z(int kind, const double* z, const double* y, int64_t n,
                             double* loss_out, cudaStream_t s) {
  loss_from_z_kernel<<<1, 256, 0, s>>>(kind, z, y, n, loss_out);
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
