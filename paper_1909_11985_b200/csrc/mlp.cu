// MLP step kernels around the tcgen05 GEMMs (gemm_sm100.cu):
//   * deterministic weight init (fp32 master + bf16 working copy);
//   * softmax cross-entropy: warp-shuffle row reductions producing per-row loss and
//     dlogits = softmax - onehot (sum semantics: the 1/count of sgd_step is applied in the
//     update, as trainer.cpp:56-61 / 244-271 do for the linear model);
//   * the fused gradient-average + SGD/momentum update: one pass over HBM that reads the
//     bf16 gradient(s), updates the fp32 master and writes the bf16 working weights.
// The update restates sgd_step (trainer.cpp:56-61) in fp32 with explicit round-to-nearest
// multiply/subtract so the CPU oracle (oracle/mlp.py) can reproduce it exactly.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "collective.hpp"
#include "edl_internal.hpp"
#include "kernels.hpp"

namespace edl {
namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__global__ void init_kernel(float* __restrict__ master, __nv_bfloat16* __restrict__ w, size_t n,
                            uint64_t seed, uint64_t offset, double bound) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint64_t idx = offset + i;
    const uint64_t h = splitmix64(seed ^ (idx * 0x9e3779b97f4a7c15ULL + 0x632be59bd9b4e019ULL));
    const double u = static_cast<double>(h >> 11) * 0x1.0p-53;
    const float v = __double2float_rn(__dmul_rn(__dsub_rn(__dmul_rn(2.0, u), 1.0), bound));
    master[i] = v;
    w[i] = __float2bfloat16_rn(v);
  }
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One CTA (256 threads) per row; classes <= 256 * kPer values held in registers
// (kPer = 16: <= 4096 classes, the configs[1] model; kPer = 64: <= 16384, configs[4]).
constexpr int kXentThreads = 256;
constexpr int kXentMaxClasses = kXentThreads * 64;
// Deterministic loss sum of `rows` per-row losses by one CTA: thread t sums rows t, t+256, ...
// in order, a fixed warp-shuffle tree combines the lanes and thread 0 adds the 8 warp
// partials in order (a serial 256-term tail here cost ~4 us per mini-batch).
__device__ void ordered_row_sum(const float* v, int rows, double* out, double* part) {
  double acc = 0.0;
  for (int r = threadIdx.x; r < rows; r += blockDim.x) acc += static_cast<double>(v[r]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x / 32] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < static_cast<int>(blockDim.x / 32); ++k) t += part[k];
    *out += t;
  }
}

template <int kPer>
__global__ void __launch_bounds__(kXentThreads)
    xent_kernel(const float* __restrict__ logits, const int32_t* __restrict__ labels, int classes,
                __nv_bfloat16* __restrict__ dlogits, float* __restrict__ row_loss,
                double* __restrict__ loss_out, unsigned* __restrict__ done) {
  __shared__ float red[kXentThreads / 32];
  __shared__ double part[kXentThreads / 32];
  __shared__ bool last;
  // launched with programmatic serialization after the last forward GEMM: wait for it here
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int row = blockIdx.x;
  const float* x = logits + static_cast<size_t>(row) * classes;
  float v[kPer];
  float m = -INFINITY;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int c = j * kXentThreads + threadIdx.x;
    v[j] = c < classes ? x[c] : -INFINITY;
    m = fmaxf(m, v[j]);
  }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  m = warp_max(m);
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = red[0];
#pragma unroll
  for (int w = 1; w < kXentThreads / 32; ++w) m = fmaxf(m, red[w]);
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    v[j] = (j * kXentThreads + static_cast<int>(threadIdx.x) < classes) ? __expf(v[j] - m) : 0.f;
    s += v[j];
  }
  s = warp_sum(s);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  s = 0.f;
#pragma unroll
  for (int w = 0; w < kXentThreads / 32; ++w) s += red[w];
  const float inv = 1.0f / s;
  const int label = labels[row];
  __nv_bfloat16* d = dlogits + static_cast<size_t>(row) * classes;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int c = j * kXentThreads + threadIdx.x;
    if (c < classes) d[c] = __float2bfloat16_rn(v[j] * inv - (c == label ? 1.0f : 0.0f));
  }
  if (threadIdx.x == 0) row_loss[row] = logf(s) + m - x[label];
  if (!loss_out) return;
  // the last CTA to finish adds the row losses into the worker's loss (fused sum_rows)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  ordered_row_sum(row_loss, gridDim.x, loss_out, part);
  if (threadIdx.x == 0) *done = 0;  // ready for the next mini-batch
}

__global__ void sum_rows_kernel(const float* __restrict__ v, int rows, double* __restrict__ out) {
  __shared__ double part[8];
  ordered_row_sum(v, rows, out, part);
}

}  // namespace

int mlp_init_weights(float* master, __nv_bfloat16* w, size_t n, uint64_t seed, uint64_t offset,
                     double bound, cudaStream_t s) {
  init_kernel<<<148 * 8, 256, 0, s>>>(master, w, n, seed, offset, bound);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int softmax_xent(const float* logits, const int32_t* labels, int rows, int classes,
                 __nv_bfloat16* dlogits, float* row_loss, double* loss_out, unsigned* done,
                 cudaStream_t s) {
  if (classes > kXentMaxClasses) return fail(EDL_EINVAL, "softmax_xent: classes > 16384");
  if (rows <= 0) return EDL_OK;
  if (loss_out && !done) return fail(EDL_EINVAL, "softmax_xent: loss sum needs a counter");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(rows);
  cfg.blockDim = dim3(kXentThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (classes <= kXentThreads * 16)
    EDL_CUDA_TRY(cudaLaunchKernelEx(&cfg, xent_kernel<16>, logits, labels, classes, dlogits,
                                    row_loss, loss_out, done));
  else
    EDL_CUDA_TRY(cudaLaunchKernelEx(&cfg, xent_kernel<64>, logits, labels, classes, dlogits,
                                    row_loss, loss_out, done));
  return EDL_OK;
}

int sum_rows(const float* row_loss, int rows, double* loss_out, cudaStream_t s) {
  sum_rows_kernel<<<1, 256, 0, s>>>(row_loss, rows, loss_out);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int sgd_update_bf16(const __nv_bfloat16* const* grads, int n_src, float* master, float* mom,
                    __nv_bfloat16* const* w_out, int n_dst, size_t n, float scale,
                    float inv_count, float eta, float mu, cudaStream_t s) {
  if (n % 8) return fail(EDL_EINVAL, "sgd_update: n must be a multiple of 8");
  if (n_src < 1 || n_src > kCollMaxSources || n_dst < 0 || n_dst > kCollMaxReplicas)
    return fail(EDL_EINVAL, "sgd_update: fan-in/out");
  CollArgs a;
  for (int k = 0; k < n_src; ++k) a.grads[k] = grads[k];
  for (int k = 0; k < n_dst; ++k) a.w_dst[k] = w_out[k];
  a.n_src = n_src;
  a.n_dst = n_dst;
  a.lo8 = 0;
  a.hi8 = n / 8;
  a.master = master;
  a.mom = mom;
  a.scale = scale;
  a.inv_count = inv_count;
  a.eta = eta;
  a.mu = mu;
  return allreduce_sgd(a, s);
}

}  // namespace edl

namespace edl {
namespace {
__global__ void master_to_bf16_kernel(const float* __restrict__ m, __nv_bfloat16* __restrict__ w,
                                      size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    w[i] = __float2bfloat16_rn(m[i]);
}
// split master (gemm_plan_init_sgd_lo): m <-> (W = RNE(m), lo = low 16 bits of m).  A tie
// that RNE rounds up (lo = 0x8000, odd high half) is stored as lo = 0x8001 (one fp32 ulp
// above m, the same W), so hi = W - (lo > 0x8000) recovers the high half.
__device__ __forceinline__ uint32_t split_lo_bits(uint32_t mb) {
  const uint32_t l = mb & 0xFFFFu;
  return (l == 0x8000u && (mb & 0x10000u)) ? 0x8001u : l;
}
__device__ __forceinline__ float join_lo(uint32_t wb, uint32_t lb) {
  return __uint_as_float(((wb - (lb > 0x8000u ? 1u : 0u)) << 16) | lb);
}
// 8 values per thread per iteration (32 B of master, 16 B of W, 16 B of lo), scalar tail
__global__ void master_split_kernel(const float* __restrict__ m, uint16_t* __restrict__ lo,
                                    __nv_bfloat16* __restrict__ w, size_t n) {
  const size_t n8 = n / 8;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n8; i += stride) {
    const float4 a = reinterpret_cast<const float4*>(m)[2 * i];
    const float4 b = reinterpret_cast<const float4*>(m)[2 * i + 1];
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t wo[4], lw[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
      wo[k] = *reinterpret_cast<uint32_t*>(&h);
      lw[k] = split_lo_bits(__float_as_uint(v[2 * k])) |
              (split_lo_bits(__float_as_uint(v[2 * k + 1])) << 16);
    }
    reinterpret_cast<uint4*>(w)[i] = make_uint4(wo[0], wo[1], wo[2], wo[3]);
    reinterpret_cast<uint4*>(lo)[i] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  }
  if (blockIdx.x == 0)
    for (size_t i = n8 * 8 + threadIdx.x; i < n; i += blockDim.x) {
      w[i] = __float2bfloat16_rn(m[i]);
      lo[i] = static_cast<uint16_t>(split_lo_bits(__float_as_uint(m[i])));
    }
}
__global__ void master_join_kernel(const __nv_bfloat16* __restrict__ w,
                                   const uint16_t* __restrict__ lo, float* __restrict__ m,
                                   size_t n) {
  const size_t n8 = n / 8;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n8; i += stride) {
    const uint4 wv = reinterpret_cast<const uint4*>(w)[i];
    const uint4 lv = reinterpret_cast<const uint4*>(lo)[i];
    const uint32_t wi[4] = {wv.x, wv.y, wv.z, wv.w}, li[4] = {lv.x, lv.y, lv.z, lv.w};
    float v[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[2 * k] = join_lo(wi[k] & 0xFFFFu, li[k] & 0xFFFFu);
      v[2 * k + 1] = join_lo(wi[k] >> 16, li[k] >> 16);
    }
    reinterpret_cast<float4*>(m)[2 * i] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(m)[2 * i + 1] = make_float4(v[4], v[5], v[6], v[7]);
  }
  if (blockIdx.x == 0)
    for (size_t i = n8 * 8 + threadIdx.x; i < n; i += blockDim.x)
      m[i] = join_lo(__bfloat16_as_ushort(w[i]), lo[i]);
}
}  // namespace

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int master_split(const float* master, uint16_t* lo, __nv_bfloat16* w, size_t n, cudaStream_t s) {
  if (n == 0) return EDL_OK;
  if (!aligned16(master) || !aligned16(lo) || !aligned16(w))
    return fail(EDL_EINVAL, "master split: buffers must be 16-byte aligned");
  master_split_kernel<<<148 * 8, 256, 0, s>>>(master, lo, w, n);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int master_join(const __nv_bfloat16* w, const uint16_t* lo, float* master, size_t n,
                cudaStream_t s) {
  if (n == 0) return EDL_OK;
  if (!aligned16(master) || !aligned16(lo) || !aligned16(w))
    return fail(EDL_EINVAL, "master join: buffers must be 16-byte aligned");
  master_join_kernel<<<148 * 8, 256, 0, s>>>(w, lo, master, n);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int mlp_prepare_device() {
  cudaFuncAttributes fa;
  EDL_CUDA_TRY(cudaFuncGetAttributes(&fa, xent_kernel<16>));
  EDL_CUDA_TRY(cudaFuncGetAttributes(&fa, xent_kernel<64>));
  EDL_CUDA_TRY(cudaFuncGetAttributes(&fa, master_to_bf16_kernel));
  EDL_CUDA_TRY(cudaFuncGetAttributes(&fa, master_split_kernel));
  EDL_CUDA_TRY(cudaFuncGetAttributes(&fa, master_join_kernel));
  return EDL_OK;
}

int master_to_bf16(const float* master, __nv_bfloat16* w, size_t n, cudaStream_t s) {
  master_to_bf16_kernel<<<148 * 8, 256, 0, s>>>(master, w, n);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}
}  // namespace edl
