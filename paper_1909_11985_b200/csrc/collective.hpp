// Fused allreduce + SGD update over NVLink peer memory (collective.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace edl {

constexpr int kCollMaxReplicas = 8;   // GPUs in one NVLink domain
constexpr int kCollMaxSources = 16;   // ring members contributing gradients
constexpr int kCollMaxBlocks = 1024;  // >= coll_blocks()
constexpr int kCollMaxSegs = 64;      // owned parameter segments (one per MLP layer)
// Flag buffer per replica: [2 phases][kCollMaxBlocks][kCollMaxReplicas] uint32.
constexpr size_t kCollFlagBytes = 2ull * kCollMaxBlocks * kCollMaxReplicas * sizeof(uint32_t);

struct CollArgs {
  const __nv_bfloat16* grads[kCollMaxSources];  // ring order; local or peer pointers
  int n_src = 0;
  __nv_bfloat16* w_dst[kCollMaxReplicas];  // bf16 working weights of every replica
  float* m_dst[kCollMaxReplicas];          // fp32 masters of every replica (all-gather)
  int n_dst = 0;
  uint32_t* flags[kCollMaxReplicas];  // flag buffers of every replica (peer-mapped)
  int me = 0, n_rep = 1;
  uint32_t epoch = 0;  // strictly increasing per launch
  size_t lo8 = 0, hi8 = 0;  // owned shard, in units of 8 params (when n_seg == 0)
  // owned shard as a list of [lo, hi) segments in units of 8 params: every replica owns a
  // slice of every layer, so a collective restricted to one layer stays balanced
  int n_seg = 0;
  size_t seg_lo8[kCollMaxSegs], seg_hi8[kCollMaxSegs];
  float* master = nullptr;  // this replica's fp32 master (full size; shard updated)
  float* mom = nullptr;
  float scale = 0.f, inv_count = 0.f, eta = 0.f, mu = 0.f;
  int update = 1;  // 0: barriers + loss only (count == 0 / fused single-replica update)
  int blocks = 0;  // grid size; 0 = coll_blocks() (fewer to co-reside with running GEMMs)
  // ordered sum of the ring members' batch losses (between the barriers, so every peer's
  // loss is final and no peer has started the next mini-batch)
  const double* losses[kCollMaxSources];
  int n_loss = 0;
  double* loss_out = nullptr;
};

// f64 ring allreduce of [grad_sum, count] vectors + sgd_step, over peer pointers
// (allreduce.cpp:60-148, trainer.cpp:56-61), bracketed by the same replica barriers.
struct LinearCollArgs {
  const double* g[kCollMaxSources];  // ring order, each [dim + 1]
  int n_src = 0;
  int dim = 0;
  double* total = nullptr;  // local scratch [dim + 1]
  double* w = nullptr;      // local replica parameters
  double eta = 0.0;
  const double* losses[kCollMaxSources];
  double* loss_out = nullptr;
  uint32_t* flags[kCollMaxReplicas];
  int me = 0, n_rep = 1;
  uint32_t epoch = 0;
};

int coll_blocks();
int allreduce_sgd(const CollArgs& a, cudaStream_t s);
int replica_barrier(const CollArgs& a, cudaStream_t s);
int linear_allreduce_sgd(const LinearCollArgs& a, cudaStream_t s);
// Every replica copies its master shard into every peer's master (checkpoint / scale events).
int master_allgather(const CollArgs& a, cudaStream_t s);
void shard_range(size_t n8, int n_rep, int r, size_t* lo, size_t* hi);

}  // namespace edl
