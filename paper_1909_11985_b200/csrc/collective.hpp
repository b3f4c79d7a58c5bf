// Fused allreduce + SGD update over NVLink peer memory (collective.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace edl {

constexpr int kCollMaxReplicas = 8;   // GPUs in one NVLink domain
constexpr int kCollMaxSources = 16;   // ring members contributing gradients
constexpr int kCollMaxBlocks = 4096;  // >= coll_blocks() and EDL_COLL_BLOCKS
constexpr int kCollMaxSegs = 64;      // owned parameter segments (one per MLP layer)
// Flag buffer per replica: barrier flags [2 phases][kCollMaxBlocks][kCollMaxReplicas], then
// copy-engine overlap flags [2 kinds][kCollMaxSegs layers][kCollMaxReplicas] (uint32 each).
constexpr size_t kCollBarrierWords = 2ull * kCollMaxBlocks * kCollMaxReplicas;
constexpr size_t kCeFlagWords = 2ull * kCollMaxSegs * kCollMaxReplicas;
// Deferred all-gather (push collective overlapped with the next mini-batch's forward): per
// layer, "replica src's updated bf16 weights of layer l are in your W" [kCollMaxSegs][
// kCollMaxReplicas], then this replica's per-layer CTA completion counters [kCollMaxSegs].
constexpr size_t kAgFlagWords = static_cast<size_t>(kCollMaxSegs) * kCollMaxReplicas + kCollMaxSegs;
constexpr size_t kAgFlagOffset = kCollBarrierWords + kCeFlagWords;  // in words
// scale-out across processes: source replica j of the old ring stores [2j] = its collective
// epoch, then [2j+1] = the new topology version, into a joining replica's flags once the
// joiner's model slice is copied (join_words)
// per source replica j: [2j] collective epoch, [2j+1] topology version; [2R + j] 1 when
// source j shipped the low master halves instead of the fp32 master (Job::lo_reshard)
constexpr size_t kJoinFlagWords = 3ull * kCollMaxReplicas;
constexpr size_t kJoinFlagOffset = kCollBarrierWords + kCeFlagWords + kAgFlagWords;
constexpr size_t kCollFlagBytes =
    (kCollBarrierWords + kCeFlagWords + kAgFlagWords + kJoinFlagWords) * sizeof(uint32_t);
// this replica's flags for layer l: one word per source replica
#ifdef __CUDACC__
__host__ __device__
#endif
inline uint32_t* ag_layer_flags(uint32_t* flags, int l) {
  return flags + kAgFlagOffset + static_cast<size_t>(l) * kCollMaxReplicas;
}

struct CollArgs {
  const __nv_bfloat16* grads[kCollMaxSources];  // ring order; local or peer pointers
  int n_src = 0;
  __nv_bfloat16* w_dst[kCollMaxReplicas];  // bf16 working weights of every replica
  float* m_dst[kCollMaxReplicas];          // fp32 masters of every replica (all-gather)
  float* v_dst[kCollMaxReplicas];          // momentum buffers of every replica (all-gather)
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
  // push variant (one ring member per replica): every NVLink byte is a store.  Phase A
  // pushes this replica's gradient slices to their owners' recv, phase B sums its own shard
  // from local memory (own gradient + recv) and pushes the updated bf16 weights.
  int push = 0;
  int skip_push = 0;  // phase A already done by the routed weight-gradient GEMMs
  int n_layer = 0;
  size_t lay_off8[kCollMaxSegs], lay_len8[kCollMaxSegs];  // layer l: [off8, off8 + len8)
  const __nv_bfloat16* own_grad = nullptr;
  __nv_bfloat16* recv_me = nullptr;                     // this replica's recv
  __nv_bfloat16* recv_peer[kCollMaxReplicas];           // replica r's recv (peer-mapped)
  int src_rep[kCollMaxSources];                         // ring member k -> replica index
  // deferred all-gather: after its share of layer l every CTA counts itself; the last one
  // signals "layer l of my shard is in your W" to every replica (ag_layer_flags), so the
  // next mini-batch's forward GEMM of layer l can start while later layers are in flight
  int ag_signal = 0;
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

// Copy-engine overlapped collective (runtime.cpp launch_layer_ce): NVLink transfers are
// cudaMemcpyAsync peer copies (no SM time, so they run under the backward GEMMs); these
// kernels only signal / wait on flags and apply the sharded update.
//   kind 0: "my gradient slices of layer l are in your recv buffer"
//   kind 1: "my updated bf16 weights of layer l are in your W"
struct CeSignal {
  uint32_t* flags[kCollMaxReplicas];  // every replica's flag buffer (peer-mapped)
  int n_rep = 1, me = 0, kind = 0, layer = 0;
  uint32_t epoch = 0;
};
struct CeWait {
  const uint32_t* flags = nullptr;  // this replica's flag buffer
  int n_rep = 1, me = 0, kind = 0, l_lo = 0, l_hi = 0;  // layers [l_lo, l_hi)
  uint32_t epoch = 0;
};
// master[i] -= scale * sum_k src[k][i] (ring order, fp32 adds of bf16 terms; momentum with
// mu != 0), W[i] = bf16(master[i]), for one owned segment of n8 * 8 parameters.
struct ShardUpdateArgs {
  const __nv_bfloat16* src[kCollMaxSources];
  int n_src = 0;
  float* master = nullptr;
  float* mom = nullptr;
  __nv_bfloat16* W = nullptr;
  size_t n8 = 0;
  float scale = 0.f, inv_count = 0.f, eta = 0.f, mu = 0.f;
  int blocks = 0;
};
int ce_signal(const CeSignal& a, cudaStream_t s);
// Copy-engine all-gather (EDL_AG_DEFER=2): after the copies of layer l of replica `me`'s
// shard into the replicas listed here (stream order), store `epoch` into their
// ag_layer_flags(flags[d], layer)[me] -- the word the next forward GEMM of layer l waits on.
struct AgSignal {
  uint32_t* flags[kCollMaxReplicas];  // the target replicas' flag buffers (peer-mapped)
  int n_dst = 0, me = 0, layer = 0;
  uint32_t epoch = 0;
};
int ag_signal(const AgSignal& a, cudaStream_t s);
// Stream-ordered 32-bit store to device memory (local or peer-mapped), preceded by a
// system-wide fence (cuStreamWriteValue32): no SM involved.
int stream_write_u32(uint32_t* addr, uint32_t value, cudaStream_t s);
int ce_wait(const CeWait& a, cudaStream_t s);
int shard_update(const ShardUpdateArgs& a, cudaStream_t s);

// SM-driven copy of up to kMaxCopySegs (dst, src, bytes) segments in one launch (every SM,
// 16-byte vectors, several loads in flight): the model re-sharding of a scale event, where
// dst is mostly peer memory over NVLink (SM stores reach ~690 GB/s per direction, more than
// one copy-engine memcpy of an IPC mapping).  bytes must be multiples of 16.
constexpr int kMaxCopySegs = 64;
struct CopySeg {
  void* dst;
  const void* src;
  size_t bytes;
};
struct MultiCopyArgs {
  CopySeg seg[kMaxCopySegs];
  int n = 0;
};
int multi_copy(const MultiCopyArgs& a, cudaStream_t s);

int coll_blocks();
int coll_prepare_device();  // current device: load the collective kernels
// Debug timeline: one thread writes %globaltimer (ns) to dst (mapped pinned host memory).
int stamp(unsigned long long* dst, cudaStream_t s);
// One thread busy-waits `ns` nanoseconds of %globaltimer (injected straggler delay).
int spin(uint64_t ns, cudaStream_t s);
int allreduce_sgd(const CollArgs& a, cudaStream_t s);
int replica_barrier(const CollArgs& a, cudaStream_t s);
int linear_allreduce_sgd(const LinearCollArgs& a, cudaStream_t s);
// Every replica copies its master shard (and, with a.mom set, its momentum shard) into every
// peer's master / momentum (checkpoint / scale events).
int master_allgather(const CollArgs& a, cudaStream_t s);
void shard_range(size_t n8, int n_rep, int r, size_t* lo, size_t* hi);

}  // namespace edl
