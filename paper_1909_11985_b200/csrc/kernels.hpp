// Launch wrappers for the hot-path kernels (dataset.cu, linear.cu, mlp.cu, collective.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/edl_b200.h"

struct EdlDataset;

namespace edl {

struct Dataset {
  EdlSyntheticSpec spec{};
  int dtype = EDL_DTYPE_F64;
  int num_classes = 0;
  size_t row_bytes = 0;
  int label_bytes = 8;
  void* x = nullptr;  // [size][dim] f64 or bf16
  void* y = nullptr;  // [size] f64 labels or int32 classes
  std::vector<double> w_true;
};

std::vector<double> synthetic_true_weights(uint64_t seed, int dim);
int dataset_create(const EdlSyntheticSpec& spec, int dtype, int num_classes, Dataset** out);
void dataset_destroy(Dataset* ds);
int dataset_get(const Dataset* ds, uint64_t index, double* features, double* label);
int gather(const Dataset* ds, const EdlRun* runs_dev, int n_runs, int64_t n_rows, void* x_out,
           void* y_out, cudaStream_t stream);
constexpr int kInlineRuns = 32;
struct InlineRuns {
  EdlRun r[kInlineRuns];
  int n;
};
// gather with <= kInlineRuns runs as kernel parameters; *zero = 0 (the worker's loss) first.
int gather_inline(const Dataset* ds, const EdlRun* runs, int n_runs, int64_t n_rows, void* x_out,
                  void* y_out, double* zero, cudaStream_t stream);

// ---- linear model, f64, bit-identical to trainer.cpp
// scale_ws: nullptr (C-ABI: one fused launch) or [2n] doubles (job: scales, then z)
int linear_local_gradient(int kind, const double* w, const double* x, const double* y, int64_t n,
                          int dim, double* grad_out, double* scale_ws, cudaStream_t s);
int linear_batch_loss(int kind, const double* w, const double* x, const double* y, int64_t n,
                      int dim, double* loss_out, double* ws, cudaStream_t s);
// batch_loss from the z = w . a_j a preceding linear_local_gradient(..., ws) left in ws + n
// (same w: the loss and the gradient of one mini-batch, trainer.cpp:41-54)
int linear_batch_loss_from_z(int kind, const double* z, const double* y, int64_t n,
                             double* loss_out, cudaStream_t s);
int linear_sgd(double* w, const double* g, int64_t count, double eta, int dim, cudaStream_t s);
// Ring-order allreduce (ring_order_reduce semantics) over n buffers of len doubles.
int ring_allreduce_f64(const double* const* inputs, int n, size_t len, int op, double* out,
                       cudaStream_t s);
// Sum of n scalars in the given order (loss aggregation across ring members).
int ordered_sum_f64(const double* const* inputs, int n, double* out, cudaStream_t s);

// ---- MLP step kernels (mlp.cu)
// Deterministic init: master[i] = float((2u - 1) * bound), u from splitmix64(seed, i).
int mlp_init_weights(float* master, __nv_bfloat16* w, size_t n, uint64_t seed, uint64_t offset,
                     double bound, cudaStream_t s);
// Softmax cross-entropy over rows x classes fp32 logits; dlogits bf16 = softmax - onehot
// (sum semantics, no 1/B); row_loss[r] = logsumexp - logit[label].
int softmax_xent(const float* logits, const int32_t* labels, int rows, int classes,
                 __nv_bfloat16* dlogits, float* row_loss, double* loss_out, unsigned* done,
                 cudaStream_t s);
// loss_out[0] += sum(row_loss[0..rows)) (deterministic, one CTA).
int sum_rows(const float* row_loss, int rows, double* loss_out, cudaStream_t s);
// Fused gradient average + SGD(+momentum) over n params, reading n_src gradient buffers
// (summed in order), updating the fp32 master and writing the bf16 working copy to every
// destination buffer:
//   mu == 0:  master -= scale * sum(g)            (scale = f32(eta_t / count), sgd_step)
//   mu != 0:  v = mu*v + sum(g)*inv_count;  master -= eta * v
// bf16 working copy of an fp32 master (checkpoint restore).
int master_to_bf16(const float* master, __nv_bfloat16* w, size_t n, cudaStream_t s);
// split master: W = RNE(m) and lo = low 16 bits of m (m: fp32 master); join: m from (W, lo)
int master_split(const float* master, uint16_t* lo, __nv_bfloat16* w, size_t n, cudaStream_t s);
int master_join(const __nv_bfloat16* w, const uint16_t* lo, float* master, size_t n,
                cudaStream_t s);
// current device: load the step's kernels now (lazy module loading would otherwise put it on
// the first mini-batch a newly added GPU runs -- the scale-out switch step)
int mlp_prepare_device();
int dataset_prepare_device();
int sgd_update_bf16(const __nv_bfloat16* const* grads, int n_src, float* master, float* mom,
                    __nv_bfloat16* const* w_out, int n_dst, size_t n, float scale,
                    float inv_count, float eta, float mu, cudaStream_t s);

}  // namespace edl
