// Gradient allreduce fused with the SGD update, over NVLink peer memory.
//
// Replaces ring_allreduce (src/allreduce.cpp:60-130) followed by sgd_step
// (src/trainer.cpp:56-61, applied as in trainer.cpp:244-271) for the MLP workload.
// One kernel per replica (= per GPU), all replicas launched with the same grid:
//
//   phase 0  barrier: CTA b of every replica signals CTA b of every peer (st.release.sys)
//            and waits for the peers' signals -> every peer's wgrad GEMMs have finished
//   phase 1  reduce-scatter + sharded update: replica r owns params [lo_r, hi_r); it reads
//            the bf16 gradients of ALL ring members for its shard (local HBM or peer HBM
//            over NVLink), sums them in ring order, applies SGD/momentum to its fp32
//            master shard and writes the bf16 weights of the shard into EVERY replica
//            (all-gather by peer stores)
//   phase 2  barrier again -> every shard of every replica's weights has been written
//
// Per replica and step that moves 2P/N + 2P(N-1)/N bytes over NVLink each way (the
// reduce-scatter + all-gather lower bound of a bf16 allreduce) and touches HBM for
// 4P + 8P/N bytes instead of the 12P of "allreduce then full update".  With one
// replica both barriers vanish and the kernel is the plain fused update.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "collective.hpp"
#include "edl_internal.hpp"

namespace edl {
namespace {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// flags[phase][block][source]
__device__ __forceinline__ uint32_t* flag_slot(uint32_t* base, int phase, int block, int src) {
  return base + (static_cast<size_t>(phase) * kCollMaxBlocks + block) * kCollMaxReplicas + src;
}

// CTA b of this replica signals CTA b of every peer, then waits for theirs.  After phase 0
// every peer's earlier kernels (its weight-gradient GEMMs) have completed; after phase 1
// every peer has finished this kernel's reads of our memory and writes into it.
__device__ void cross_replica_barrier(uint32_t* const* flags, int me, int n_rep, uint32_t epoch,
                                      int phase) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int r = 0; r < n_rep; ++r)
      if (r != me) st_release_sys(flag_slot(flags[r], phase, blockIdx.x, me), epoch);
    for (int r = 0; r < n_rep; ++r) {
      if (r == me) continue;
      const uint32_t* f = flag_slot(flags[me], phase, blockIdx.x, r);
      const uint64_t t0 = clock64();
      while (static_cast<int32_t>(ld_acquire_sys(f) - epoch) < 0) {
        __nanosleep(32);
        if (clock64() - t0 > (1ull << 36)) __trap();  // a peer died: fail, don't hang
      }
    }
  }
  __syncthreads();
}
__device__ __forceinline__ void cross_replica_barrier(const CollArgs& a, int phase) {
  cross_replica_barrier(a.flags, a.me, a.n_rep, a.epoch, phase);
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 t = __bfloat1622float2(h[k]);
    f[2 * k] = t.x;
    f[2 * k + 1] = t.y;
  }
}

// SGD / momentum on 8 parameters of this replica's shard + bf16 weights to every replica.
template <bool kMomentum>
__device__ __forceinline__ void apply8(const CollArgs& a, size_t i, const float (&gs)[8]) {
  float4* mp = reinterpret_cast<float4*>(a.master) + 2 * i;
  const float4 m0 = __ldcs(mp), m1 = __ldcs(mp + 1);
  float m[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
  if (kMomentum) {
    float4* vp = reinterpret_cast<float4*>(a.mom) + 2 * i;
    const float4 v0 = __ldcs(vp), v1 = __ldcs(vp + 1);
    float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      v[e] = __fadd_rn(__fmul_rn(a.mu, v[e]), __fmul_rn(gs[e], a.inv_count));
      m[e] = __fsub_rn(m[e], __fmul_rn(a.eta, v[e]));
    }
    __stcs(vp, make_float4(v[0], v[1], v[2], v[3]));
    __stcs(vp + 1, make_float4(v[4], v[5], v[6], v[7]));
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) m[e] = __fsub_rn(m[e], __fmul_rn(a.scale, gs[e]));
  }
  __stcs(mp, make_float4(m[0], m[1], m[2], m[3]));
  __stcs(mp + 1, make_float4(m[4], m[5], m[6], m[7]));
  uint4 o;
  __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
  for (int k = 0; k < 4; ++k) oh[k] = __floats2bfloat162_rn(m[2 * k], m[2 * k + 1]);
  for (int d = 0; d < a.n_dst; ++d) reinterpret_cast<uint4*>(a.w_dst[d])[i] = o;
}

// 8 parameters per thread and unrolled group; kU groups (a grid stride apart) keep kU loads
// of every source in flight at once (the peer loads are NVLink-latency bound).
template <bool kMomentum, int kU>
__global__ void __launch_bounds__(256) allreduce_sgd_kernel(CollArgs a) {
  if (a.n_rep > 1) cross_replica_barrier(a, 0);
  if (a.loss_out && blockIdx.x == 0 && threadIdx.x == 0) {
    double acc = 0.0;
    for (int k = 0; k < a.n_loss; ++k) acc = __dadd_rn(acc, *a.losses[k]);
    *a.loss_out = acc;
  }
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const int n_seg = a.update ? (a.n_seg > 0 ? a.n_seg : 1) : 0;
  for (int sg = 0; sg < n_seg; ++sg) {
    const size_t lo = a.n_seg > 0 ? a.seg_lo8[sg] : a.lo8;
    const size_t hi = a.n_seg > 0 ? a.seg_hi8[sg] : a.hi8;
    for (size_t i0 = lo + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i0 < hi;
         i0 += stride * kU) {
      float gs[kU][8];
      uint4 t[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const size_t i = i0 + u * stride;
        if (i < hi) t[u] = __ldcs(reinterpret_cast<const uint4*>(a.grads[0]) + i);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (i0 + u * stride < hi) bf16x8_to_f32(t[u], gs[u]);
      for (int k = 1; k < a.n_src; ++k) {
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const size_t i = i0 + u * stride;
          if (i < hi) t[u] = __ldcs(reinterpret_cast<const uint4*>(a.grads[k]) + i);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (i0 + u * stride >= hi) continue;
          float f[8];
          bf16x8_to_f32(t[u], f);
#pragma unroll
          for (int e = 0; e < 8; ++e) gs[u][e] = __fadd_rn(gs[u][e], f[e]);
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (i0 + u * stride < hi) apply8<kMomentum>(a, i0 + u * stride, gs[u]);
    }
  }
  if (a.n_rep > 1) cross_replica_barrier(a, 1);
}

// Push variant: replica r owns slice r/n of every layer (shard_range, as own_segments);
// recv of owner o = [n-1 slots (sources in replica order, o skipped)][its shard, layers
// concatenated].
__device__ __forceinline__ void lay_shard(const CollArgs& a, int l, int r, size_t* lo,
                                          size_t* hi) {
  const size_t n8 = a.lay_len8[l];
  *lo = a.lay_off8[l] + n8 * static_cast<size_t>(r) / static_cast<size_t>(a.n_rep);
  *hi = a.lay_off8[l] + n8 * static_cast<size_t>(r + 1) / static_cast<size_t>(a.n_rep);
}
__device__ __forceinline__ size_t shard_prefix8(const CollArgs& a, int r, int l) {
  size_t t = 0;
  for (int k = 0; k < l; ++k) {
    size_t lo, hi;
    lay_shard(a, k, r, &lo, &hi);
    t += hi - lo;
  }
  return t;
}

// Phase B of one layer with a compile-time source count: every source's 16-byte load of a
// thread's 8 parameters is in flight before the first is used (the runtime-count loop issued
// them one at a time).  src[k][i - lo] = ring member k's gradient of parameter group i.
template <bool kMomentum, int kS>
__device__ __forceinline__ void push_phase_b(const CollArgs& a, const uint4* const (&src)[kS],
                                             size_t lo, size_t hi, size_t tid, size_t stride) {
  for (size_t i = lo + tid; i < hi; i += stride) {
    uint4 v[kS];
#pragma unroll
    for (int k = 0; k < kS; ++k) v[k] = __ldcs(src[k] + (i - lo));
    float gs[8];
    bf16x8_to_f32(v[0], gs);
#pragma unroll
    for (int k = 1; k < kS; ++k) {
      float f[8];
      bf16x8_to_f32(v[k], f);
#pragma unroll
      for (int e = 0; e < 8; ++e) gs[e] = __fadd_rn(gs[e], f[e]);
    }
    apply8<kMomentum>(a, i, gs);
  }
}

template <bool kMomentum>
__global__ void __launch_bounds__(256) push_allreduce_sgd_kernel(CollArgs a) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const size_t tid = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  const uint4* own = reinterpret_cast<const uint4*>(a.own_grad);
  if (a.update && !a.skip_push) {
    // phase A: my gradient slices -> their owners' recv (NVLink stores, 2 in flight)
    for (int j = 1; j < a.n_rep; ++j) {
      const int o = (a.me + j) % a.n_rep;  // rotated: every GPU pushes to a different owner
      const size_t total = shard_prefix8(a, o, a.n_layer);
      const size_t slot = static_cast<size_t>(a.me < o ? a.me : a.me - 1);
      uint4* dst_o = reinterpret_cast<uint4*>(a.recv_peer[o]) + slot * total;
      for (int l = 0; l < a.n_layer; ++l) {
        size_t lo, hi;
        lay_shard(a, l, o, &lo, &hi);
        uint4* dst = dst_o + shard_prefix8(a, o, l);
        const size_t len = hi - lo;
        for (size_t i = tid; i < len; i += 2 * stride) {
          uint4 v[2];
#pragma unroll
          for (int u = 0; u < 2; ++u)
            if (i + u * stride < len) v[u] = __ldcs(own + lo + i + u * stride);
#pragma unroll
          for (int u = 0; u < 2; ++u)
            if (i + u * stride < len) dst[i + u * stride] = v[u];
        }
      }
    }
  }
  cross_replica_barrier(a, 0);  // every peer's slices of my shard have landed
  if (a.loss_out && blockIdx.x == 0 && threadIdx.x == 0) {
    double acc = 0.0;
    for (int k = 0; k < a.n_loss; ++k) acc = __dadd_rn(acc, *a.losses[k]);
    *a.loss_out = acc;
  }
  if (a.update) {
    // phase B: ring-order sum of my shard from local memory, SGD, weights to every replica
    const size_t total = shard_prefix8(a, a.me, a.n_layer);
    const uint4* rv = reinterpret_cast<const uint4*>(a.recv_me);
    for (int l = 0; l < a.n_layer; ++l) {
      size_t lo, hi;
      lay_shard(a, l, a.me, &lo, &hi);
      const size_t pre = shard_prefix8(a, a.me, l);
      auto src_of = [&](int k) -> const uint4* {
        const int r = a.src_rep[k];
        return r == a.me ? own + lo : rv + static_cast<size_t>(r < a.me ? r : r - 1) * total + pre;
      };
      if (a.n_src == 2 || a.n_src == 4 || a.n_src == 8) {
        if (a.n_src == 2) {
          const uint4* s[2] = {src_of(0), src_of(1)};
          push_phase_b<kMomentum, 2>(a, s, lo, hi, tid, stride);
        } else if (a.n_src == 4) {
          const uint4* s[4] = {src_of(0), src_of(1), src_of(2), src_of(3)};
          push_phase_b<kMomentum, 4>(a, s, lo, hi, tid, stride);
        } else {
          const uint4* s[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) s[k] = src_of(k);
          push_phase_b<kMomentum, 8>(a, s, lo, hi, tid, stride);
        }
      } else {
      for (size_t i = lo + tid; i < hi; i += stride) {
        float gs[8];
        for (int k = 0; k < a.n_src; ++k) {
          const int r = a.src_rep[k];
          const uint4 v = r == a.me
                              ? __ldcs(own + i)
                              : __ldcs(rv + static_cast<size_t>(r < a.me ? r : r - 1) * total +
                                       pre + (i - lo));
          float f[8];
          bf16x8_to_f32(v, f);
          if (k == 0) {
#pragma unroll
            for (int e = 0; e < 8; ++e) gs[e] = f[e];
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) gs[e] = __fadd_rn(gs[e], f[e]);
          }
        }
        apply8<kMomentum>(a, i, gs);
      }
      }
      if (a.ag_signal) {
        // every thread's weight stores of layer l (local and peer) before the count
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) {
          uint32_t* ctr = a.flags[a.me] + kAgFlagOffset + kCollMaxSegs * kCollMaxReplicas + l;
          if (atomicAdd(ctr, 1u) == gridDim.x - 1) {  // last CTA of this replica for layer l
            __threadfence_system();
            *ctr = 0;  // every CTA has counted: ready for the next mini-batch
            for (int r = 0; r < a.n_rep; ++r)
              st_release_sys(ag_layer_flags(a.flags[r], l) + a.me, a.epoch);
          }
        }
      }
    }
  }
  cross_replica_barrier(a, 1);
}

__global__ void barrier_kernel(CollArgs a) { cross_replica_barrier(a, 0); }

// One CTA: barrier, ring-order f64 reduction of every member's [grad_sum, count] (chunk c =
// [c*len/n, (c+1)*len/n) folds ranks c, c+1, ... left to right, allreduce.cpp:132-148),
// ordered loss sum, barrier, then sgd_step on the local replica (trainer.cpp:56-61).
__global__ void linear_allreduce_sgd_kernel(LinearCollArgs a) {
  // block b owns elements [b*256, (b+1)*256) of [grad_sum, count]; the per-block barrier
  // slots make block b of every replica meet (same grid everywhere)
  if (a.n_rep > 1) cross_replica_barrier(a.flags, a.me, a.n_rep, a.epoch, 0);
  const int n = a.n_src;
  const size_t len = static_cast<size_t>(a.dim) + 1;
  auto ring_sum = [&](size_t i) {  // chunk c = [c*len/n, (c+1)*len/n) folds c, c+1, ...
    int c = 0;
    while (c + 1 < n && len * static_cast<size_t>(c + 1) / static_cast<size_t>(n) <= i) ++c;
    double acc = a.g[c][i];
    for (int k = 1; k < n; ++k) acc = __dadd_rn(acc, a.g[(c + k) % n][i]);
    return acc;
  };
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  double v = 0.0;
  if (i < len) {
    v = ring_sum(i);
    a.total[i] = v;
  }
  // every block needs the global count (element dim): the same ring-order sum, recomputed
  __shared__ double count;
  if (threadIdx.x == 0) count = ring_sum(len - 1);
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.loss_out) {
    double acc = 0.0;
    for (int k = 0; k < n; ++k) acc = __dadd_rn(acc, *a.losses[k]);
    *a.loss_out = acc;
  }
  __syncthreads();
  if (a.n_rep > 1) cross_replica_barrier(a.flags, a.me, a.n_rep, a.epoch, 1);
  if (count == 0.0) return;
  const double sc = __ddiv_rn(a.eta, count);
  if (i < static_cast<size_t>(a.dim)) a.w[i] = __dsub_rn(a.w[i], __dmul_rn(sc, v));
}

__global__ void __launch_bounds__(256) master_allgather_kernel(CollArgs a) {
  cross_replica_barrier(a, 0);
  const float4* src = reinterpret_cast<const float4*>(a.master);
  const int n_seg = a.n_seg > 0 ? a.n_seg : 1;
  for (int sg = 0; sg < n_seg; ++sg) {
    const size_t lo = a.n_seg > 0 ? a.seg_lo8[sg] : a.lo8;
    const size_t hi = a.n_seg > 0 ? a.seg_hi8[sg] : a.hi8;
    for (size_t i = lo * 2 + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
         i < hi * 2; i += static_cast<size_t>(gridDim.x) * blockDim.x) {
      const float4 v = src[i];
      for (int d = 0; d < a.n_dst; ++d)
        if (d != a.me) reinterpret_cast<float4*>(a.m_dst[d])[i] = v;
      if (a.mom) {  // the momentum shard is as current as the master shard, and only there
        const float4 u = reinterpret_cast<const float4*>(a.mom)[i];
        for (int d = 0; d < a.n_dst; ++d)
          if (d != a.me) reinterpret_cast<float4*>(a.v_dst[d])[i] = u;
      }
    }
  }
  cross_replica_barrier(a, 1);
}

__device__ __forceinline__ uint32_t* ce_flag(uint32_t* base, int kind, int layer, int src) {
  return base + kCollBarrierWords +
         (static_cast<size_t>(kind) * kCollMaxSegs + layer) * kCollMaxReplicas + src;
}

__global__ void ce_signal_kernel(CeSignal a) {
  __threadfence_system();  // the copies before this kernel (stream order) are performed
  for (int r = 0; r < a.n_rep; ++r)
    if (r != a.me) st_release_sys(ce_flag(a.flags[r], a.kind, a.layer, a.me), a.epoch);
}

__global__ void ag_signal_kernel(AgSignal a) {
  __threadfence_system();  // the copies before this kernel (stream order) are performed
  for (int d = 0; d < a.n_dst; ++d) st_release_sys(ag_layer_flags(a.flags[d], a.layer) + a.me, a.epoch);
}

__global__ void ce_wait_kernel(CeWait a) {
  uint32_t* base = const_cast<uint32_t*>(a.flags);
  for (int l = a.l_lo; l < a.l_hi; ++l)
    for (int r = 0; r < a.n_rep; ++r) {
      if (r == a.me) continue;
      const uint32_t* f = ce_flag(base, a.kind, l, r);
      const uint64_t t0 = clock64();
      while (static_cast<int32_t>(ld_acquire_sys(f) - a.epoch) < 0) {
        __nanosleep(64);
        if (clock64() - t0 > (1ull << 36)) __trap();  // a peer died: fail, don't hang
      }
    }
  __threadfence_system();
}

template <bool kMomentum>
__global__ void __launch_bounds__(256) shard_update_kernel(ShardUpdateArgs a) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < a.n8;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float gs[8];
    bf16x8_to_f32(__ldcs(reinterpret_cast<const uint4*>(a.src[0]) + i), gs);
    for (int k = 1; k < a.n_src; ++k) {
      float t[8];
      bf16x8_to_f32(__ldcs(reinterpret_cast<const uint4*>(a.src[k]) + i), t);
#pragma unroll
      for (int e = 0; e < 8; ++e) gs[e] = __fadd_rn(gs[e], t[e]);
    }
    float4* mp = reinterpret_cast<float4*>(a.master) + 2 * i;
    const float4 m0 = __ldcs(mp), m1 = __ldcs(mp + 1);
    float m[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
    if (kMomentum) {
      float4* vp = reinterpret_cast<float4*>(a.mom) + 2 * i;
      const float4 v0 = __ldcs(vp), v1 = __ldcs(vp + 1);
      float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        v[e] = __fadd_rn(__fmul_rn(a.mu, v[e]), __fmul_rn(gs[e], a.inv_count));
        m[e] = __fsub_rn(m[e], __fmul_rn(a.eta, v[e]));
      }
      __stcs(vp, make_float4(v[0], v[1], v[2], v[3]));
      __stcs(vp + 1, make_float4(v[4], v[5], v[6], v[7]));
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) m[e] = __fsub_rn(m[e], __fmul_rn(a.scale, gs[e]));
    }
    __stcs(mp, make_float4(m[0], m[1], m[2], m[3]));
    __stcs(mp + 1, make_float4(m[4], m[5], m[6], m[7]));
    uint4 o;
    __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) oh[k] = __floats2bfloat162_rn(m[2 * k], m[2 * k + 1]);
    reinterpret_cast<uint4*>(a.W)[i] = o;
  }
}

__global__ void stamp_kernel(unsigned long long* dst) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *dst = t;
}

__global__ void spin_kernel(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(256);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

}  // namespace

int spin(uint64_t ns, cudaStream_t s) {
  spin_kernel<<<1, 1, 0, s>>>(ns);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int stamp(unsigned long long* dst, cudaStream_t s) {
  stamp_kernel<<<1, 1, 0, s>>>(dst);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int ce_signal(const CeSignal& a, cudaStream_t s) {
  if (a.n_rep <= 1) return EDL_OK;
  ce_signal_kernel<<<1, 1, 0, s>>>(a);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

namespace {
// cuStreamWriteValue32: the flag store is a stream memory operation (front end, preceded by a
// system-wide fence after the copies), so it needs no SM.  A signal kernel would have to find
// a free slot next to the next mini-batch's forward GEMM CTAs (PDL-resident, spinning on
// these very flags); measured, it could starve behind them.
using WriteValue32Fn = int (*)(void*, unsigned long long, unsigned int, unsigned int);
WriteValue32Fn write_value32_fn() {
  static WriteValue32Fn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    const char* e = getenv("EDL_AG_SIGNAL_KERNEL");
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (!(e && *e == '1') &&
        cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WriteValue32Fn>(p);
  }
  return fn;
}
}  // namespace

int stream_write_u32(uint32_t* addr, uint32_t value, cudaStream_t s) {
  static WriteValue32Fn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return fail(EDL_ECUDA, "cuStreamWriteValue32 unavailable");
    fn = reinterpret_cast<WriteValue32Fn>(p);
  }
  const int rc = fn(s, reinterpret_cast<unsigned long long>(addr), value, 0);
  if (rc != 0) return fail(EDL_ECUDA, "cuStreamWriteValue32 failed (" + std::to_string(rc) + ")");
  return EDL_OK;
}

int ag_signal(const AgSignal& a, cudaStream_t s) {
  if (a.n_dst <= 0) return EDL_OK;
  if (WriteValue32Fn fn = write_value32_fn()) {
    for (int d = 0; d < a.n_dst; ++d) {
      const int rc = fn(s, reinterpret_cast<unsigned long long>(
                              ag_layer_flags(a.flags[d], a.layer) + a.me), a.epoch, 0);
      if (rc != 0) return fail(EDL_ECUDA, "cuStreamWriteValue32 failed (" + std::to_string(rc) + ")");
    }
    return EDL_OK;
  }
  ag_signal_kernel<<<1, 1, 0, s>>>(a);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int ce_wait(const CeWait& a, cudaStream_t s) {
  if (a.n_rep <= 1 || a.l_hi <= a.l_lo) return EDL_OK;
  ce_wait_kernel<<<1, 1, 0, s>>>(a);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int shard_update(const ShardUpdateArgs& a, cudaStream_t s) {
  if (a.n8 == 0) return EDL_OK;
  if (a.n_src < 1 || a.n_src > kCollMaxSources) return fail(EDL_EINVAL, "shard_update: sources");
  const int blocks = a.blocks > 0 ? a.blocks : coll_blocks();
  if (a.mu != 0.0f)
    shard_update_kernel<true><<<blocks, 256, 0, s>>>(a);
  else
    shard_update_kernel<false><<<blocks, 256, 0, s>>>(a);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int master_allgather(const CollArgs& a, cudaStream_t s) {
  master_allgather_kernel<<<coll_blocks(), 256, 0, s>>>(a);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

__global__ void __launch_bounds__(256) multi_copy_kernel(const __grid_constant__ MultiCopyArgs a) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (int k = 0; k < a.n; ++k) {
    const uint4* src = static_cast<const uint4*>(a.seg[k].src);
    uint4* dst = static_cast<uint4*>(a.seg[k].dst);
    const size_t n = a.seg[k].bytes / 16;
    size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {  // four loads in flight per thread
      const uint4 v0 = __ldcs(src + i), v1 = __ldcs(src + i + stride);
      const uint4 v2 = __ldcs(src + i + 2 * stride), v3 = __ldcs(src + i + 3 * stride);
      dst[i] = v0;
      dst[i + stride] = v1;
      dst[i + 2 * stride] = v2;
      dst[i + 3 * stride] = v3;
    }
    for (; i < n; i += stride) dst[i] = __ldcs(src + i);
  }
}

int multi_copy(const MultiCopyArgs& a, cudaStream_t s) {
  if (a.n < 0 || a.n > kMaxCopySegs) return fail(EDL_EINVAL, "multi_copy: segments");
  for (int k = 0; k < a.n; ++k)
    if (a.seg[k].bytes % 16) return fail(EDL_EINVAL, "multi_copy: 16-byte multiples");
  if (a.n == 0) return EDL_OK;
  multi_copy_kernel<<<coll_blocks(), 256, 0, s>>>(a);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int coll_blocks() { return 148 * 4; }

// Loads the collective kernels on the current device (cudaFuncGetAttributes forces the lazy
// load), off the switch step of a scale-out.
int coll_prepare_device() {
  cudaFuncAttributes fa;
  EDL_CUDA_TRY(cudaFuncGetAttributes(&fa, push_allreduce_sgd_kernel<false>));
  EDL_CUDA_TRY(cudaFuncGetAttributes(&fa, push_allreduce_sgd_kernel<true>));
  EDL_CUDA_TRY(cudaFuncGetAttributes(&fa, allreduce_sgd_kernel<false, 2>));
  EDL_CUDA_TRY(cudaFuncGetAttributes(&fa, allreduce_sgd_kernel<true, 2>));
  EDL_CUDA_TRY(cudaFuncGetAttributes(&fa, master_allgather_kernel));
  EDL_CUDA_TRY(cudaFuncGetAttributes(&fa, multi_copy_kernel));
  EDL_CUDA_TRY(cudaFuncGetAttributes(&fa, barrier_kernel));
  EDL_CUDA_TRY(cudaFuncGetAttributes(&fa, linear_allreduce_sgd_kernel));
  return EDL_OK;
}

int allreduce_sgd(const CollArgs& a, cudaStream_t s) {
  if (a.n_src < 1 || a.n_src > kCollMaxSources) return fail(EDL_EINVAL, "allreduce_sgd: sources");
  if (a.n_dst < 0 || a.n_dst > kCollMaxReplicas || a.n_rep > kCollMaxReplicas)
    return fail(EDL_EINVAL, "allreduce_sgd: replicas");
  static int env_blocks = -1, unroll = -1;  // tuning knobs (EDL_COLL_BLOCKS / _UNROLL)
  if (env_blocks < 0) {
    const char* e = getenv("EDL_COLL_BLOCKS");
    env_blocks = e ? atoi(e) : 0;
    e = getenv("EDL_COLL_UNROLL");
    unroll = e ? atoi(e) : 2;
  }
  int blocks = a.blocks > 0 ? a.blocks : (env_blocks > 0 ? env_blocks : coll_blocks());
  if (blocks > kCollMaxBlocks) return fail(EDL_EINVAL, "allreduce_sgd: grid");
  if (a.push) {
    if (a.n_src != a.n_rep || a.n_layer < 1 || a.n_layer > kCollMaxSegs)
      return fail(EDL_EINVAL, "allreduce_sgd: push variant needs one member per replica");
    if (a.mu != 0.0f)
      push_allreduce_sgd_kernel<true><<<blocks, 256, 0, s>>>(a);
    else
      push_allreduce_sgd_kernel<false><<<blocks, 256, 0, s>>>(a);
    EDL_CUDA_TRY(cudaGetLastError());
    return EDL_OK;
  }
  if (a.mu != 0.0f) {
    if (unroll >= 2)
      allreduce_sgd_kernel<true, 2><<<blocks, 256, 0, s>>>(a);
    else
      allreduce_sgd_kernel<true, 1><<<blocks, 256, 0, s>>>(a);
  } else {
    if (unroll >= 4)
      allreduce_sgd_kernel<false, 4><<<blocks, 256, 0, s>>>(a);
    else if (unroll >= 2)
      allreduce_sgd_kernel<false, 2><<<blocks, 256, 0, s>>>(a);
    else
      allreduce_sgd_kernel<false, 1><<<blocks, 256, 0, s>>>(a);
  }
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int linear_allreduce_sgd(const LinearCollArgs& a, cudaStream_t s) {
  if (a.n_src < 1 || a.n_src > kCollMaxSources) return fail(EDL_EINVAL, "linear allreduce: sources");
  const unsigned blocks = static_cast<unsigned>((a.dim + 1 + 255) / 256);
  if (blocks > static_cast<unsigned>(kCollMaxBlocks)) return fail(EDL_EINVAL, "linear allreduce: dim");
  linear_allreduce_sgd_kernel<<<blocks, 256, 0, s>>>(a);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

int replica_barrier(const CollArgs& a, cudaStream_t s) {
  if (a.n_rep <= 1) return EDL_OK;
  barrier_kernel<<<1, 32, 0, s>>>(a);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

// Shard boundaries in units of 8 parameters: replica r owns [r*n8/N, (r+1)*n8/N), the
// same rounding as chunk_range (allreduce.cpp:33-37).
void shard_range(size_t n8, int n_rep, int r, size_t* lo, size_t* hi) {
  *lo = n8 * static_cast<size_t>(r) / static_cast<size_t>(n_rep);
  *hi = n8 * static_cast<size_t>(r + 1) / static_cast<size_t>(n_rep);
}

}  // namespace edl
