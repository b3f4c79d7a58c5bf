// HBM-resident synthetic dataset + coalesced lease gather.
//
// Replaces edl::SyntheticDataset (include/edl/dataset.hpp:25-50, src/dataset.cpp:11-58).
// Sample i is a pure function of (seed, i):
//   state = splitmix64(seed ^ (i * 0xd1342543de82ef95 + 1));
//   feature k: state = splitmix64(state); f = 2 * ((state >> 11) * 2^-53) - 1   (exact in f64)
//   label     = sum_k w_true[k] * f[k] sequentially with no FMA (+ noise, optional sign)
// F64 datasets are bit-identical to the reference; BF16 datasets (the MLP workload) round
// each f64 feature f64 -> f32 -> bf16 (RNE) and carry int32 class labels.
//
// The dataset is materialised once in HBM (2^20 x 4096 bf16 = 8 GiB for BASELINE.json
// configs[1]); per step the gather kernel copies the leased runs of sample ids into the
// contiguous batch the first GEMM reads.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <vector>

#include "edl_internal.hpp"
#include "kernels.hpp"

namespace edl {

namespace {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ double unit_double(uint64_t bits) {
  return static_cast<double>(bits >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ uint16_t f64_to_bf16_bits(double f) {
  const float x = __double2float_rn(f);
  const __nv_bfloat16 b = __float2bfloat16_rn(x);
  return *reinterpret_cast<const uint16_t*>(&b);
}

// One thread per sample; sequential feature chain (the recurrence is inherently serial
// per sample).  Label: FMA-free sequential dot, dataset.cpp:48-49.
__global__ void gen_f64_kernel(double* __restrict__ x, double* __restrict__ y,
                               const double* __restrict__ w_true, uint64_t size, int dim,
                               uint64_t seed, double noise, int sign_labels) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= size) return;
  uint64_t st = splitmix64(seed ^ (i * 0xd1342543de82ef95ULL + 1));
  double* row = x + i * static_cast<uint64_t>(dim);
  double acc = 0.0;
  for (int k = 0; k < dim; ++k) {
    st = splitmix64(st);
    const double f = 2.0 * unit_double(st) - 1.0;
    row[k] = f;
    acc = __dadd_rn(acc, __dmul_rn(w_true[k], f));
  }
  if (noise > 0.0) {
    st = splitmix64(st);
    acc = __dadd_rn(acc, __dmul_rn(noise, 2.0 * unit_double(st) - 1.0));
  }
  y[i] = sign_labels ? (acc >= 0.0 ? 1.0 : -1.0) : acc;
}

// BF16 generator: a warp owns 32 samples; each lane walks its sample's chain 64 features
// at a time into a [32][64] shared tile, then the warp writes the tile as 32 coalesced
// 128-byte row segments.
constexpr int kGenWarps = 4;
__global__ void __launch_bounds__(kGenWarps * 32)
    gen_bf16_kernel(__nv_bfloat16* __restrict__ x, int32_t* __restrict__ y, uint64_t size,
                    int dim, uint64_t seed, int num_classes) {
  __shared__ __align__(16) uint16_t tile[kGenWarps][32][64];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint64_t base = (blockIdx.x * static_cast<uint64_t>(kGenWarps) + warp) * 32;
  const uint64_t i = base + lane;
  uint64_t st = splitmix64(seed ^ (i * 0xd1342543de82ef95ULL + 1));
  for (int k0 = 0; k0 < dim; k0 += 64) {
    const int width = dim - k0 < 64 ? dim - k0 : 64;
    for (int k = 0; k < width; ++k) {
      st = splitmix64(st);
      tile[warp][lane][k] = f64_to_bf16_bits(2.0 * unit_double(st) - 1.0);
    }
    __syncwarp();
    if ((dim & 7) == 0 && width == 64) {
      // 32 rows x 128 B: each instruction covers 4 rows (8 lanes x 16 B per row)
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int r = it * 4 + lane / 8, part = lane % 8;
        const uint64_t row = base + r;
        if (row < size) {
          const uint4 v = *reinterpret_cast<const uint4*>(&tile[warp][r][part * 8]);
          *reinterpret_cast<uint4*>(x + row * dim + k0 + part * 8) = v;
        }
      }
    } else {
      for (int r = 0; r < 32; ++r) {
        const uint64_t row = base + r;
        if (row >= size) break;
        for (int k = lane; k < width; k += 32)
          reinterpret_cast<uint16_t*>(x)[row * dim + k0 + k] = tile[warp][r][k];
      }
    }
    __syncwarp();
  }
  if (i < size) {
    const uint64_t ls = splitmix64(seed ^ ~(i * 0xd1342543de82ef95ULL + 1));
    y[i] = static_cast<int32_t>(ls % static_cast<uint64_t>(num_classes));
  }
}

// Gather: output row r <- dataset row of the r-th leased sample.  Runs are few (a batch
// spans 1-3 shards); each CTA resolves its row's run by a linear scan, then copies the
// row with 16-byte vector loads/stores.
__global__ void gather_kernel(const uint8_t* __restrict__ src, const void* __restrict__ labels,
                              int label_bytes, const EdlRun* __restrict__ runs, int n_runs,
                              int64_t n_rows, size_t row_bytes, uint8_t* __restrict__ dst,
                              uint8_t* __restrict__ dst_labels) {
  for (int64_t r = blockIdx.x; r < n_rows; r += gridDim.x) {
    int64_t k = r;
    uint64_t id = 0;
    for (int j = 0; j < n_runs; ++j) {
      const int64_t c = static_cast<int64_t>(runs[j].count);
      if (k < c) {
        id = runs[j].first + static_cast<uint64_t>(k);
        break;
      }
      k -= c;
    }
    const uint8_t* s = src + id * row_bytes;
    uint8_t* d = dst + static_cast<size_t>(r) * row_bytes;
    if ((row_bytes & 15) == 0) {
      for (size_t off = threadIdx.x * 16; off < row_bytes; off += blockDim.x * 16)
        *reinterpret_cast<uint4*>(d + off) = __ldg(reinterpret_cast<const uint4*>(s + off));
    } else {
      for (size_t off = threadIdx.x; off < row_bytes; off += blockDim.x) d[off] = s[off];
    }
    if (threadIdx.x == 0 && dst_labels) {
      if (label_bytes == 8)
        reinterpret_cast<uint64_t*>(dst_labels)[r] = reinterpret_cast<const uint64_t*>(labels)[id];
      else
        reinterpret_cast<uint32_t*>(dst_labels)[r] = reinterpret_cast<const uint32_t*>(labels)[id];
    }
  }
}

}  // namespace

std::vector<double> synthetic_true_weights(uint64_t seed, int dim) {
  std::vector<double> w(static_cast<size_t>(dim));
  uint64_t st = splitmix64(seed ^ 0x77ee55aa11cc33ddULL);  // dataset.cpp:29
  for (auto& v : w) {
    st = splitmix64(st);
    v = 2.0 * unit_double(st) - 1.0;
  }
  return w;
}

int dataset_create(const EdlSyntheticSpec& spec, int dtype, int num_classes, Dataset** out) {
  if (spec.size == 0 || spec.dim <= 0) return fail(EDL_EINVAL, "dataset: empty spec");
  if (dtype != EDL_DTYPE_F64 && dtype != EDL_DTYPE_BF16) return fail(EDL_EINVAL, "dataset dtype");
  if (dtype == EDL_DTYPE_BF16 && num_classes <= 0) return fail(EDL_EINVAL, "num_classes");
  auto* ds = new Dataset;
  ds->spec = spec;
  ds->dtype = dtype;
  ds->num_classes = num_classes;
  ds->w_true = synthetic_true_weights(spec.seed, spec.dim);
  const size_t esz = dtype == EDL_DTYPE_F64 ? 8 : 2;
  ds->row_bytes = esz * static_cast<size_t>(spec.dim);
  ds->label_bytes = dtype == EDL_DTYPE_F64 ? 8 : 4;
  cudaError_t e = cudaMalloc(&ds->x, ds->row_bytes * spec.size);
  if (e == cudaSuccess) e = cudaMalloc(&ds->y, ds->label_bytes * spec.size);
  if (e != cudaSuccess) {
    cudaFree(ds->x);
    delete ds;
    return cuda_fail(e, "dataset cudaMalloc");
  }
  if (dtype == EDL_DTYPE_F64) {
    double* wt = nullptr;
    EDL_CUDA_TRY(cudaMalloc(&wt, sizeof(double) * spec.dim));
    EDL_CUDA_TRY(cudaMemcpy(wt, ds->w_true.data(), sizeof(double) * spec.dim,
                            cudaMemcpyHostToDevice));
    const int threads = 256;
    const unsigned blocks = static_cast<unsigned>((spec.size + threads - 1) / threads);
    gen_f64_kernel<<<blocks, threads>>>(static_cast<double*>(ds->x), static_cast<double*>(ds->y),
                                        wt, spec.size, spec.dim, spec.seed, spec.noise,
                                        spec.sign_labels);
    EDL_CUDA_TRY(cudaGetLastError());
    EDL_CUDA_TRY(cudaDeviceSynchronize());
    cudaFree(wt);
  } else {
    const uint64_t per_block = kGenWarps * 32;
    const unsigned blocks = static_cast<unsigned>((spec.size + per_block - 1) / per_block);
    gen_bf16_kernel<<<blocks, kGenWarps * 32>>>(static_cast<__nv_bfloat16*>(ds->x),
                                               static_cast<int32_t*>(ds->y), spec.size, spec.dim,
                                               spec.seed, num_classes);
    EDL_CUDA_TRY(cudaGetLastError());
    EDL_CUDA_TRY(cudaDeviceSynchronize());
  }
  *out = ds;
  return EDL_OK;
}

void dataset_destroy(Dataset* ds) {
  if (!ds) return;
  cudaFree(ds->x);
  cudaFree(ds->y);
  delete ds;
}

int dataset_get(const Dataset* ds, uint64_t index, double* features, double* label) {
  if (index >= ds->spec.size) return fail(EDL_OUT_OF_RANGE, "sample index");
  const int dim = ds->spec.dim;
  if (ds->dtype == EDL_DTYPE_F64) {
    EDL_CUDA_TRY(cudaMemcpy(features, static_cast<const uint8_t*>(ds->x) + index * ds->row_bytes,
                            ds->row_bytes, cudaMemcpyDeviceToHost));
    EDL_CUDA_TRY(cudaMemcpy(label, static_cast<const double*>(ds->y) + index, 8,
                            cudaMemcpyDeviceToHost));
  } else {
    std::vector<__nv_bfloat16> row(static_cast<size_t>(dim));
    int32_t cls = 0;
    EDL_CUDA_TRY(cudaMemcpy(row.data(), static_cast<const uint8_t*>(ds->x) + index * ds->row_bytes,
                            ds->row_bytes, cudaMemcpyDeviceToHost));
    EDL_CUDA_TRY(cudaMemcpy(&cls, static_cast<const int32_t*>(ds->y) + index, 4,
                            cudaMemcpyDeviceToHost));
    for (int k = 0; k < dim; ++k) features[k] = static_cast<double>(__bfloat162float(row[k]));
    *label = static_cast<double>(cls);
  }
  return EDL_OK;
}

// Same gather with the (few) leased runs passed as kernel parameters, and the worker's
// loss accumulator zeroed by the first thread: no H2D copy or memset before the step.
__global__ void gather_inline_kernel(const uint8_t* __restrict__ src,
                                     const void* __restrict__ labels, int label_bytes,
                                     const __grid_constant__ InlineRuns runs, int64_t n_rows,
                                     size_t row_bytes, uint8_t* __restrict__ dst,
                                     uint8_t* __restrict__ dst_labels, double* zero) {
  if (zero && blockIdx.x == 0 && threadIdx.x == 0) *zero = 0.0;
  for (int64_t r = blockIdx.x; r < n_rows; r += gridDim.x) {
    int64_t k = r;
    uint64_t id = 0;
    for (int j = 0; j < runs.n; ++j) {
      const int64_t c = static_cast<int64_t>(runs.r[j].count);
      if (k < c) {
        id = runs.r[j].first + static_cast<uint64_t>(k);
        break;
      }
      k -= c;
    }
    const uint8_t* s = src + id * row_bytes;
    uint8_t* d = dst + static_cast<size_t>(r) * row_bytes;
    if ((row_bytes & 15) == 0) {
      // every load of the row issued before the first store (4 x 16 B in flight per thread)
      const size_t n16 = row_bytes / 16;
      const uint4* s16 = reinterpret_cast<const uint4*>(s);
      uint4* d16 = reinterpret_cast<uint4*>(d);
      for (size_t base = threadIdx.x; base < n16; base += 4 * blockDim.x) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (base + u * blockDim.x < n16) v[u] = __ldg(s16 + base + u * blockDim.x);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (base + u * blockDim.x < n16) d16[base + u * blockDim.x] = v[u];
      }
    } else {
      for (size_t off = threadIdx.x; off < row_bytes; off += blockDim.x) d[off] = s[off];
    }
    if (threadIdx.x == 0 && dst_labels) {
      if (label_bytes == 8)
        reinterpret_cast<uint64_t*>(dst_labels)[r] = reinterpret_cast<const uint64_t*>(labels)[id];
      else
        reinterpret_cast<uint32_t*>(dst_labels)[r] = reinterpret_cast<const uint32_t*>(labels)[id];
    }
  }
}

int gather_inline(const Dataset* ds, const EdlRun* runs, int n_runs, int64_t n_rows, void* x_out,
                  void* y_out, double* zero, cudaStream_t stream) {
  if (n_runs < 0 || n_runs > kInlineRuns) return fail(EDL_EINVAL, "gather_inline: too many runs");
  InlineRuns ir{};
  ir.n = n_runs;
  for (int j = 0; j < n_runs; ++j) ir.r[j] = runs[j];
  const int threads = ds->row_bytes >= 4096 ? 256 : 64;
  int64_t blocks = n_rows < 4 * 148 ? n_rows : 4 * 148;
  if (blocks < 1) blocks = 1;
  gather_inline_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
      static_cast<const uint8_t*>(ds->x), ds->y, ds->label_bytes, ir, n_rows, ds->row_bytes,
      static_cast<uint8_t*>(x_out), static_cast<uint8_t*>(y_out), zero);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int gather(const Dataset* ds, const EdlRun* runs_dev, int n_runs, int64_t n_rows, void* x_out,
           void* y_out, cudaStream_t stream) {
  if (n_rows <= 0) return EDL_OK;
  const int threads = ds->row_bytes >= 4096 ? 256 : 64;
  int64_t blocks = n_rows < 4 * 148 ? n_rows : 4 * 148;
  gather_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
      static_cast<const uint8_t*>(ds->x), ds->y, ds->label_bytes, runs_dev, n_runs, n_rows,
      ds->row_bytes, static_cast<uint8_t*>(x_out), static_cast<uint8_t*>(y_out));
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int dataset_prepare_device() {
  cudaFuncAttributes fa;
  EDL_CUDA_TRY(cudaFuncGetAttributes(&fa, gather_kernel));
  EDL_CUDA_TRY(cudaFuncGetAttributes(&fa, gather_inline_kernel));
  return EDL_OK;
}

}  // namespace edl
