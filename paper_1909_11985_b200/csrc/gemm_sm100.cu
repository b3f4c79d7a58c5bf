// Dense-layer GEMMs of the MLP SGD step on tcgen05 tensor cores.
//
//   C[M][N] = sum_k A(m,k) * B(n,k)      bf16 x bf16 -> fp32 (TMEM) -> epilogue
//
// A is either K-major (row-major [M][K]) or MN-major (row-major [K][M]); same for B with N.
// That lets the three GEMMs of one Linear layer run with no transposed copies:
//   forward  Y  = X  . W^T : A = X  [b][in]  K-major,  B = W [out][in] K-major
//   dgrad    dX = dY . W   : A = dY [b][out] K-major,  B = W [out][in] MN-major (N = in)
//   wgrad    dW = dY^T . X : A = dY [b][out] MN-major, B = X [b][in]   MN-major (K = batch)
//
// Structure (one CTA per SM, persistent over output tiles):
//   warp 0        TMA producer: A/B tiles -> smem ring (SWIZZLE_128B), mbarrier full/empty
//   warp 1        TMEM allocator + single-thread tcgen05.mma issuer, 128 x BN x 16 per MMA
//   warps 2..5    epilogue: tcgen05.ld TMEM -> registers -> fused op -> global
// TMEM holds two accumulator buffers so the epilogue of tile i overlaps the MMAs of i+1.
//
// This file replaces the inner loops of the reference's per-sample gradient
// (proj/src/trainer.cpp:14-28, local_gradient :30-39) for the MLP workload of
// BASELINE.json configs[1]; the reference itself only has dense-vector f64 loops.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "edl_internal.hpp"
#include "sm100.cuh"

namespace edl {
namespace {

using namespace sm100;

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle row of bf16
constexpr int kThreads = 192;
constexpr uint32_t kMnBlockBytes = 64 * BK * 2;  // one 64(MN) x 64(K) TMA box = 8 KB

template <int BN>
struct Cfg {
  static constexpr uint32_t kABytes = BM * BK * 2;  // 16 KB
  static constexpr uint32_t kBBoxes = (BN + 63) / 64;
  static constexpr uint32_t kBBytesK = BN * BK * 2;              // K-major B tile
  static constexpr uint32_t kBBytesMN = kBBoxes * kMnBlockBytes;  // MN-major B tile
  static constexpr uint32_t kBSlot = (kBBytesK > kBBytesMN ? kBBytesK : kBBytesMN);
  static constexpr uint32_t kStageBytes = kABytes + ((kBSlot + 1023) / 1024) * 1024;
#ifndef EDL_GEMM_SMEM_KB
#define EDL_GEMM_SMEM_KB 200
#endif
#ifndef EDL_GEMM_MAX_STAGES
#define EDL_GEMM_MAX_STAGES 8
#endif
  static constexpr int kFit = (EDL_GEMM_SMEM_KB * 1024) / kStageBytes;
  static constexpr int kStages = kFit > EDL_GEMM_MAX_STAGES ? EDL_GEMM_MAX_STAGES : kFit;
  static constexpr uint32_t kAccCols = BN;  // fp32 columns per accumulator
  static constexpr uint32_t kTmemCols = (2 * BN <= 32)    ? 32
                                        : (2 * BN <= 64)  ? 64
                                        : (2 * BN <= 128) ? 128
                                        : (2 * BN <= 256) ? 256
                                                          : 512;
  static constexpr uint32_t kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*bars*/;
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tmap_a,
                        const __grid_constant__ CUtensorMap tmap_b, int M, int N, int K,
                        EpiParams ep) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty_bar = full_bar + C::kStages;
  uint64_t* tfull_bar = empty_bar + C::kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int m_tiles = (M + BM - 1) / BM;
  const int n_tiles = (N + BN - 1) / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int num_kb = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_a);
    prefetch_tmap(&tmap_b);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue above overlaps the previous kernel's tail (PDL); every CTA of this persistent
  // grid is resident, so dependents may launch now and run their own prologue
  griddep_wait();
  griddep_launch();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t tx = C::kABytes + (B_MN ? C::kBBytesMN : C::kBBytesK);
    if (ep.wait_flags) {  // weights still arriving from the deferred all-gather
      if (lane == 0) wait_flags_acquire(ep.wait_flags, ep.wait_n, ep.wait_epoch);
      __syncwarp();
    }
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m0 = (tile % m_tiles) * BM;
      const int n0 = (tile / m_tiles) * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (elect_one()) {
          uint8_t* sa = smem + stage * C::kStageBytes;
          uint8_t* sb = sa + C::kABytes;
          mbar_arrive_expect_tx(&full_bar[stage], tx);
          if (A_MN) {
            tma_load_2d(sa, &tmap_a, &full_bar[stage], m0, kb * BK);
            tma_load_2d(sa + kMnBlockBytes, &tmap_a, &full_bar[stage], m0 + 64, kb * BK);
          } else {
            tma_load_2d(sa, &tmap_a, &full_bar[stage], kb * BK, m0);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < (int)C::kBBoxes; ++j)
              tma_load_2d(sb + j * kMnBlockBytes, &tmap_b, &full_bar[stage], n0 + 64 * j,
                          kb * BK);
          } else {
            tma_load_2d(sb, &tmap_b, &full_bar[stage], kb * BK, n0);
          }
        }
        __syncwarp();
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, A_MN, B_MN);
    const uint32_t s0 = smem_u32(smem);
    const uint64_t a0 = A_MN ? smem_desc_sw128(s0, kMnBlockBytes, 1024) : smem_desc_sw128(s0, 16, 1024);
    const uint64_t b0 = B_MN ? smem_desc_sw128(s0 + C::kABytes, kMnBlockBytes, 1024)
                             : smem_desc_sw128(s0 + C::kABytes, 16, 1024);
    constexpr uint32_t kStepA = A_MN ? 2048 : 32, kStepB = B_MN ? 2048 : 32;
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    // one fixed issuing lane: tcgen05.commit only tracks the MMAs of the executing thread
    const bool issuer = elect_one();
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * C::kAccCols;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        const uint64_t so = static_cast<uint64_t>(stage * C::kStageBytes) >> 4;
        if (issuer) {
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16(d_tmem, a0 + so + ((k * kStepA) >> 4), b0 + so + ((k * kStepB) >> 4), idesc,
                      (kb | k) != 0 ? 1u : 0u);
          umma_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (issuer) umma_commit(&tfull_bar[acc]);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int local = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      const int m0 = (tile % m_tiles) * BM;
      const int n0 = (tile / m_tiles) * BN;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + q * 32 + lane;
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * C::kAccCols;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(t_row + c, r);
        tmem_ld_wait();
        const int col0 = n0 + c;
        if (row >= M || col0 >= N) continue;
        const int lim = min(min(32, BN - c), N - col0);  // valid columns in this chunk
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if (ep.relu) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.0f);
        }
        const bool full = (lim == 32);
        if (ep.mask) {
          const __nv_bfloat16* mrow = ep.mask + static_cast<size_t>(row) * ep.ldm + col0;
          if (full) {
#pragma unroll
            for (int j8 = 0; j8 < 4; ++j8) {
              uint4 mv = *reinterpret_cast<const uint4*>(mrow + j8 * 8);
              const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&mv);
#pragma unroll
              for (int t = 0; t < 8; ++t)
                if (!(__bfloat162float(mb[t]) > 0.0f)) v[j8 * 8 + t] = 0.0f;
            }
          } else {
            // constant indices only: a runtime-indexed v[] would live in local memory
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < lim && !(__bfloat162float(mrow[j]) > 0.0f)) v[j] = 0.0f;
          }
        }
        if (ep.out_f32) {
          float* crow = static_cast<float*>(ep.C) + static_cast<size_t>(row) * ep.ldc + col0;
          if (full) {
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4)
              *reinterpret_cast<float4*>(crow + j4 * 4) =
                  make_float4(v[j4 * 4], v[j4 * 4 + 1], v[j4 * 4 + 2], v[j4 * 4 + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < lim) crow[j] = v[j];
          }
        } else {
          __nv_bfloat16* crow =
              static_cast<__nv_bfloat16*>(ep.C) + static_cast<size_t>(row) * ep.ldc + col0;
          if (full) {
#pragma unroll
            for (int j8 = 0; j8 < 4; ++j8) {
              uint4 o;
              o.x = pack_bf16(v[j8 * 8 + 0], v[j8 * 8 + 1]);
              o.y = pack_bf16(v[j8 * 8 + 2], v[j8 * 8 + 3]);
              o.z = pack_bf16(v[j8 * 8 + 4], v[j8 * 8 + 5]);
              o.w = pack_bf16(v[j8 * 8 + 6], v[j8 * 8 + 7]);
              *reinterpret_cast<uint4*>(crow + j8 * 8) = o;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < lim) crow[j] = __float2bfloat16_rn(v[j]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
    }
  }

  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

// ------------------------------------------------------------------ CTA-pair kernel
// cta_group::2 variant: a cluster of 2 CTAs (one TPC) computes a 256 x BN tile with
// M=256 UMMAs issued by the pair leader.  Each CTA stages its own 128 rows of A and BN/2
// rows of B, so each SM's shared memory feeds half the operand bytes per MMA that the
// 1-SM kernel needs (the 1-SM kernel is shared-memory-bound at BN=128).  The epilogue
// goes TMEM -> registers -> 128B-swizzled smem -> TMA bulk-tensor store (coalesced,
// asynchronous); the two accumulator buffers let tile i's epilogue overlap tile i+1's MMAs.
//
// kMc = 2: a cluster of 4 CTAs = 2 pairs working on horizontally adjacent N tiles of the
// same 256-row M tile.  Both pairs need the same A rows, so each CTA loads half of its
// 128-row A slice and multicasts it to the matching CTA of the other pair: the L2 -> SM
// operand stream (which bounds the M=512 GEMMs of the step) drops from 3 to 2 units per k
// block.  A stage is refilled only when both pairs' MMAs have consumed it (empty barriers
// count one commit from each pair leader).
constexpr int kEpiChunkBytes = 32 * 128;  // one warp's 32 rows x 128 B staging box

#ifdef EDL_GEMM_TRACE
// [cta][0] mma wait-full cycles, [1] mma wait-tempty, [2] mma loop total, [3] producer
// wait-empty, [4] producer total, [5] epilogue wait-tfull (warp 2), [6] epilogue total
__device__ unsigned long long g_gemm_trace[296][16];
// timeline (globaltimer ns, last write wins): [0] entry, [1] after the setup cluster_sync,
// [2] first full stage seen by MMA, [3] MMA loop end, [4] first tfull seen by epilogue warp 2,
// [5] warp 2 stores drained, [6] producer end, [7] after the final cluster_sync
__device__ unsigned long long g_gemm_tl[296][16];
#define TRACE_T0(v) const unsigned long long v = clock64()
#define TRACE_ADD(slot, t0) \
  if ((threadIdx.x & 31) == 0) atomicAdd(&g_gemm_trace[blockIdx.x][slot], clock64() - (t0))
#define TL(slot) \
  if ((threadIdx.x & 31) == 0) g_gemm_tl[blockIdx.x][slot] = globaltimer_ns()
#else
#define TRACE_T0(v)
#define TRACE_ADD(slot, t0)
#define TL(slot)
#endif

template <int BN, bool kSgd = false, int kLo = 0, bool kAres = false>
struct Cfg2 {
  static_assert(BN % 64 == 0 && BN >= 64 && BN <= 256, "2-SM tiles: BN multiple of 64");
  static constexpr int kHalfN = BN / 2;
  static constexpr uint32_t kABytes = 128 * BK * 2;                      // 16 KB
  static constexpr int kBBoxesMN = (kHalfN + 63) / 64;  // MN-major B: 64-column TMA boxes
  static constexpr uint32_t kBBytesK = static_cast<uint32_t>(kHalfN) * BK * 2;  // per CTA
  static constexpr uint32_t kBBytesMN = kBBoxesMN * kMnBlockBytes;
  static constexpr uint32_t kBSlot = kBBytesK > kBBytesMN ? kBBytesK : kBBytesMN;
  // kAres (A-resident fused SGD): the whole A panel of the current row block (up to K = 512:
  // 8 k-blocks x 16 KB per CTA) stays in shared memory; the stages hold B only
  static constexpr int kAresMaxKb = 8;
  static constexpr uint32_t kAPanel = kAres ? kAresMaxKb * kABytes : 0;
  static constexpr uint32_t kStageBytes =
      (kAres ? 0 : kABytes) + ((kBSlot + 1023) / 1024) * 1024;
  // epilogue warps: 4 (one per TMEM lane quarter); the fused-SGD epilogue is latency-bound
  // (TMEM loads, master loads, smem shared with the mainloop) and runs two warps per quarter,
  // each owning half of the tile's columns
#ifndef EDL_SGD_EPI_WARPS
#define EDL_SGD_EPI_WARPS 8
#endif
  // the split-master epilogue (kLo != 0) runs EDL_SGD_LO_WARPS (16: four per quarter)
#ifndef EDL_SGD_LO_WARPS
#define EDL_SGD_LO_WARPS 16
#endif
  static constexpr int kEpiWarps = kLo ? EDL_SGD_LO_WARPS : (kSgd ? EDL_SGD_EPI_WARPS : 4);
  static constexpr int kThreads2 = 64 + 32 * kEpiWarps;
  // epilogue staging per warp: plain 2 x 4 KB; fused SGD kSgdBufs x (8 KB master + 4 KB W).
  // EDL_SGD_WDIRECT: the bf16 weights go from registers straight to global memory (each lane
  // its row's 128 contiguous bytes), so a buffer is the 8 KB master chunk only and two of them
  // per warp fit: the next tile's master load is issued a whole tile ahead
#ifndef EDL_SGD_WDIRECT
#define EDL_SGD_WDIRECT 0
#endif
  static constexpr bool kWDirect = kSgd && EDL_SGD_WDIRECT;
  // split master (kLo, see the kernel): a warp's 32 x 32 chunk, 4 KB (2 KB low halves +
  // 2 KB weights, or 4 KB of fp32 master in); kLo = 2 writes 4 KB of fp32 master + 2 KB of
  // weights: 6 KB
  static constexpr uint32_t kSgdBufBytes =
      kLo == 2 ? 6144u : kLo ? 4096u : (kWDirect ? 2 : 3) * kEpiChunkBytes;
#ifndef EDL_SGD_LO_BUFS
#define EDL_SGD_LO_BUFS 1
#endif
#ifdef EDL_SGD_BUFS
  static constexpr int kSgdBufs = EDL_SGD_BUFS;
#else
  static constexpr int kSgdBufs = kLo ? EDL_SGD_LO_BUFS : (kEpiWarps == 8 && !kWDirect ? 1 : 2);
#endif
  // master prefetch distance in chunks (1 .. kSgdBufs - 1)
#ifdef EDL_SGD_PFD
  static constexpr int kSgdPfd = EDL_SGD_PFD;
#else
  static constexpr int kSgdPfd = kSgdBufs > 1 ? kSgdBufs - 1 : 0;
#endif
  static constexpr uint32_t kEpiBytes =
      kSgd ? kEpiWarps * kSgdBufs * kSgdBufBytes : 4 * 2 * kEpiChunkBytes;
#ifndef EDL_GEMM2_MAX_STAGES
#define EDL_GEMM2_MAX_STAGES 6
#endif
  static constexpr int kFit = (224 * 1024 - kEpiBytes - kAPanel) / kStageBytes;
#ifndef EDL_SGD_STAGES
#define EDL_SGD_STAGES EDL_GEMM2_MAX_STAGES
#endif
#ifndef EDL_ARES_STAGES
#define EDL_ARES_STAGES 4
#endif
  static constexpr int kMaxStages =
      kAres ? EDL_ARES_STAGES : kSgd ? EDL_SGD_STAGES : EDL_GEMM2_MAX_STAGES;
  static constexpr int kStages = kFit > kMaxStages ? kMaxStages : kFit;
  static constexpr uint32_t kAccCols = BN;
  // TMEM accumulator ring: 2 tiles; the fused-SGD kernel may use EDL_SGD_ACC (up to 512
  // columns) so the MMA can run further ahead of its epilogue
#ifndef EDL_SGD_ACC
#define EDL_SGD_ACC 2
#endif
  static constexpr int kAcc = (kSgd && EDL_SGD_ACC * BN <= 512) ? EDL_SGD_ACC : 2;
  static constexpr uint32_t kTmemCols = (kAcc * kAccCols <= 256) ? 256 : 512;
  static constexpr uint32_t kSmemBytes = kAPanel + kStages * kStageBytes + kEpiBytes + 1024 + 512;
};

// kSk = 2 (split-K): a cluster of 4 CTAs = 2 pairs computes ONE 256 x BN tile, pair p over
// k-blocks [p * nkb/2, ...) of K.  256 x 256 pair tiles halve the shared-memory bytes per MAC
// of 256 x 128 (the M = 512 GEMMs of the step are shared-memory-bound at 256 x 128: measured
// 55% of the MMA rate vs 95% at 256 x 256), and the K split keeps 128 SMs busy.  After the
// mainloop each CTA owns one column half of the tile: it sends the other half of its fp32
// partial to the matching CTA of the other pair through DSMEM (into that CTA's idle stage
// buffers), receives that CTA's partial of its own half, adds, and runs the epilogue.
template <int BN, bool A_MN, bool B_MN, bool kSgd, int kMc, int kSk = 1, bool kX = false,
          int kLo = 0, bool kAres = false>
__global__ void __launch_bounds__(Cfg2<BN, kSgd, kLo, kAres>::kThreads2, 1)
    gemm_bf16_2sm_kernel(const __grid_constant__ CUtensorMap tmap_a,
                         const __grid_constant__ CUtensorMap tmap_b,
                         const __grid_constant__ CUtensorMap tmap_c,
                         const __grid_constant__ CUtensorMap tmap_m, int M, int N, int K,
                         EpiParams ep, const __grid_constant__ PeerMaps pm) {
  using C = Cfg2<BN, kSgd, kLo, kAres>;
  // kAres: A-resident variant of the split-master fused SGD (mode 1 / 3): each CTA pair takes
  // a contiguous range of tiles in row-major order and keeps the A panel of the current row
  // block (dY^T: 256 rows x K) in shared memory, reloading it only when the row block changes;
  // only B streams.  Operand bytes from L2 per tile: 128 KB instead of 384 KB.
  static_assert(!kAres || ((kLo == 1 || kLo == 3) && kMc == 1 && kSk == 1),
                "A-resident: split-master SGD plans");
  // kLo (fused SGD over the split master, tmap_m = the 16-bit low halves lo, pm.m[0] = the
  // fp32 master): 1 = (W, lo) in and out; 2 = (W, lo) in, fp32 master + W out (the last
  // mini-batch before a switch to another update path); 3 = fp32 master in, (W, lo) out
  // (the first fused mini-batch after one)
  static_assert(kLo == 0 || (kSgd && !kX && !C::kWDirect), "split master: fused-SGD plans");
  constexpr bool kLoIn = kLo == 1 || kLo == 2;
  constexpr bool kLoOut = kLo == 1 || kLo == 3;
  static_assert(kSk == 1 || (kSk == 2 && kMc == 1 && !kSgd && BN == 256),
                "split-K: 256-wide plain tiles, no multicast");
  static_assert(!kX || (kSgd && kMc == 1 && kSk == 1), "fused exchange: fused-SGD plans");
  // kMc = 4 (8-CTA clusters, K-major A) compiles and was measured: slower than 2 on B200
  static_assert(kMc == 1 || kMc == 2 || (kMc == 4 && !A_MN), "A multicast: 2 pairs, or 4 (K-major A)");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* a_panel = smem;                // kAres: the resident A panel
  uint8_t* sbase = smem + C::kAPanel;     // the stage ring
  uint8_t* epi = sbase + C::kStages * C::kStageBytes;  // 1024-aligned staging
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(epi + C::kEpiBytes);
  uint64_t* empty_bar = full_bar + C::kStages;
  uint64_t* tfull_bar = empty_bar + C::kStages;
  uint64_t* tempty_bar = tfull_bar + C::kAcc;
  uint64_t* sgd_bar = tempty_bar + C::kAcc;  // fused SGD: master-load barriers per epilogue warp
  uint64_t* a_full = sgd_bar + 32;   // kAres: A panel landed
  uint64_t* a_empty = a_full + 1;    // kAres: the MMAs reading the A panel are done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_empty + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const uint32_t pr = rank & 1;     // rank inside the CTA pair
  const uint32_t pidx = rank >> 1;  // pair inside the cluster (kMc = 2)
  const bool leader = pr == 0;
  const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (2 * pidx));
  const int unit = blockIdx.x / (2 * kMc * kSk), n_units = gridDim.x / (2 * kMc * kSk);
  const int m_tiles = (M + 255) / 256;
  const int n_tiles = (N + BN - 1) / BN;  // the host guarantees n_tiles % kMc == 0
  const int num_work = m_tiles * (n_tiles / kMc);
  const int num_kb = (K + BK - 1) / BK;
  auto tile_m = [&](int w) { return kAres ? w / n_tiles : w % m_tiles; };
  auto tile_n = [&](int w) {
    if (kAres) return w % n_tiles;
    return (w / m_tiles) * kMc + (kMc >= 2 ? static_cast<int>(pidx) : 0);
  };
  // the unit's work sequence: tiles unit, unit + n_units, ...  (Running the fused
  // exchange's routed tiles first was measured slower: it separates the epilogue-heavy own
  // tiles from the mainloop-heavy routed ones instead of overlapping them.)  kAres: the
  // contiguous range [unit * W / U, (unit + 1) * W / U) of the row-major tile order.
  const int ares_lo = static_cast<int>(static_cast<long>(unit) * num_work / n_units);
  const int ares_hi = static_cast<int>(static_cast<long>(unit + 1) * num_work / n_units);
  auto seq_tile = [&](int i) -> int {
    if (kAres) return ares_lo + i < ares_hi ? ares_lo + i : num_work;
    const int t = unit + i * n_units;
    return t < num_work ? t : num_work;
  };
  // split-K: this pair's k-blocks (the host guarantees one tile per cluster)
  const int kb_begin = kSk == 2 ? static_cast<int>(pidx) * (num_kb / 2) : 0;
#ifdef EDL_GEMM_TRACE
  const int kb_end = (ep.dbg & 1) ? kb_begin : (kSk == 2 && pidx == 0 ? num_kb / 2 : num_kb);
  const bool skip_epi = (ep.dbg & 2) != 0;
#else
  const int kb_end = kSk == 2 && pidx == 0 ? num_kb / 2 : num_kb;
  constexpr bool skip_epi = false;
#endif

  if (warp == 0) TL(0);
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_a);
    prefetch_tmap(&tmap_b);
    prefetch_tmap(&tmap_c);
    if (kSgd) prefetch_tmap(&tmap_m);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kMc);
    }
    for (int a = 0; a < C::kAcc; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 2 * C::kEpiWarps);  // lane 0 of every epilogue warp, both CTAs
    }
    for (int a = 0; a < 32; ++a) mbar_init(&sgd_bar[a], kSk == 2 && a < 2 ? 4 : 1);
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_2sm<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (warp == 1) TL(1);
  griddep_wait();  // see gemm_bf16_tn_kernel
  griddep_launch();

  // Producer and MMA loops run warp-uniform (all 32 lanes wait on the barriers; elect.sync
  // picks the issuing lane) so descriptors and coordinates stay in uniform registers and
  // each UTCHMMA / UTMALDG issues without a per-instruction R2UR waterfall.
  if (warp == 0 && kAres) {
    // ------------------------------------------------------------ TMA producer, A resident
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t tx_b = 2 * (B_MN ? C::kBBytesMN : C::kBBytesK);
    const uint32_t tx_a = 2 * static_cast<uint32_t>(num_kb) * C::kABytes;
    int cur_m = -1, panel = 0;
    for (int wi = 0, w = seq_tile(0); w < num_work; w = seq_tile(++wi)) {
      const int m = tile_m(w);
      const int m0 = m * 256 + static_cast<int>(pr) * 128;
      const int n0 = tile_n(w) * BN + static_cast<int>(pr) * C::kHalfN;
      if (m != cur_m) {  // a new row block: its A panel, once the MMAs on the old one are done
        if (panel > 0) mbar_wait(a_empty, (panel - 1) & 1);
        if (elect_one()) {
          if (leader) mbar_arrive_expect_tx(a_full, tx_a);
          for (int kb = 0; kb < num_kb; ++kb) {
            uint8_t* sa = a_panel + kb * C::kABytes;
            if (A_MN) {
              tma_load_2d_2sm(sa, &tmap_a, a_full, m0, kb * BK);
              tma_load_2d_2sm(sa + kMnBlockBytes, &tmap_a, a_full, m0 + 64, kb * BK);
            } else {
              tma_load_2d_2sm(sa, &tmap_a, a_full, kb * BK, m0);
            }
          }
        }
        __syncwarp();
        cur_m = m;
        ++panel;
      }
      for (int kb = kb_begin; kb < kb_end; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (elect_one()) {
          uint8_t* sb = sbase + stage * C::kStageBytes;
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], tx_b);
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < C::kBBoxesMN; ++j)
              tma_load_2d_2sm(sb + j * kMnBlockBytes, &tmap_b, &full_bar[stage], n0 + 64 * j,
                              kb * BK);
          } else {
            tma_load_2d_2sm(sb, &tmap_b, &full_bar[stage], kb * BK, n0);
          }
        }
        __syncwarp();
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1 && kAres) {
    if (leader) {
      // ------------------------------------------------------------ MMA issuer, A resident
      constexpr uint32_t idesc = idesc_bf16_f32(256, BN, A_MN, B_MN);
      const uint32_t sa0 = smem_u32(a_panel), sb0 = smem_u32(sbase);
      const uint64_t a0 = A_MN ? smem_desc_sw128(sa0, kMnBlockBytes, 1024) : smem_desc_sw128(sa0, 16, 1024);
      const uint64_t b0 = B_MN ? smem_desc_sw128(sb0, kMnBlockBytes, 1024) : smem_desc_sw128(sb0, 16, 1024);
      constexpr uint32_t kStepA = A_MN ? 2048 : 32, kStepB = B_MN ? 2048 : 32;
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      int cur_m = -1, panel = 0;
      const bool issuer = elect_one();
      for (int wi = 0, w = seq_tile(0); w < num_work; w = seq_tile(++wi), ++local) {
        const int acc = local % C::kAcc;
        const uint32_t acc_phase = (local / C::kAcc) & 1;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const int m = tile_m(w);
        if (m != cur_m) {
          mbar_wait(a_full, panel & 1);
          tc_fence_after();
          cur_m = m;
          ++panel;
        }
        const uint32_t d_tmem = tmem_base + acc * C::kAccCols;
        for (int kb = kb_begin; kb < kb_end; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t sob = static_cast<uint64_t>(stage * C::kStageBytes) >> 4;
          const uint64_t soa = static_cast<uint64_t>(kb * C::kABytes) >> 4;
          if (issuer) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16_2sm(d_tmem, a0 + soa + ((k * kStepA) >> 4), b0 + sob + ((k * kStepB) >> 4),
                            idesc, (kb != kb_begin || k != 0) ? 1u : 0u);
            umma_commit_2sm(&empty_bar[stage], pair_mask);
          }
          __syncwarp();
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (issuer) umma_commit_2sm(&tfull_bar[acc], pair_mask);
        // the row block ends here: the producer may overwrite the A panel once these MMAs
        // have read it
        const int wn = seq_tile(wi + 1);
        if (wn < num_work && tile_m(wn) != m && issuer) umma_commit_2sm(a_empty, pair_mask);
        __syncwarp();
      }
    }
  } else if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    int stage = 0;
    uint32_t phase = 0;
    // both CTAs' bytes (full boxes, OOB included) are counted on the leader's barrier
    const uint32_t tx = 2 * (C::kABytes + (B_MN ? C::kBBytesMN : C::kBBytesK));
    TRACE_T0(t_prod);
    uint16_t a_mask = 0;  // the CTA with my rank-in-pair in every pair of the cluster
    for (int p2 = 0; p2 < kMc; ++p2) a_mask |= static_cast<uint16_t>(1u << (pr + 2 * p2));
    if (ep.wait_flags) {  // weights still arriving from the deferred all-gather
      if (lane == 0) wait_flags_acquire(ep.wait_flags, ep.wait_n, ep.wait_epoch);
      __syncwarp();
    }
    // ep.l2pf: this CTA's share of the prefetch region, 64 KB per k-block from the first
    size_t pf_lo = 0, pf_hi = 0, pf_step = 65536;
    if (ep.l2pf_bytes) {
      const size_t share = ((ep.l2pf_bytes / gridDim.x) + 15) & ~static_cast<size_t>(15);
      pf_lo = share * blockIdx.x;
      pf_hi = pf_lo + share < ep.l2pf_bytes ? pf_lo + share : ep.l2pf_bytes;
      // spread evenly over this CTA's k-blocks
      int my_kb = 0;
      for (int wi = 0, w = seq_tile(0); w < num_work; w = seq_tile(++wi)) my_kb += kb_end - kb_begin;
      if (my_kb > 0) pf_step = ((share / my_kb) + 1023) & ~static_cast<size_t>(1023);
      if (pf_step == 0) pf_step = 1024;
    }
    for (int wi = 0, w = seq_tile(0); w < num_work; w = seq_tile(++wi)) {
      const int m0 = tile_m(w) * 256 + static_cast<int>(pr) * 128;
      const int n0 = tile_n(w) * BN + static_cast<int>(pr) * C::kHalfN;
      for (int kb = kb_begin; kb < kb_end; ++kb) {
        TRACE_T0(t_w);
        mbar_wait(&empty_bar[stage], phase ^ 1);
        TRACE_ADD(3, t_w);
        if (pf_lo < pf_hi) {  // warp-uniform: every lane advances pf_lo
          const size_t n = pf_hi - pf_lo < pf_step ? pf_hi - pf_lo : pf_step;
          if (elect_one())
            bulk_prefetch_l2(static_cast<const uint8_t*>(ep.l2pf) + pf_lo, static_cast<uint32_t>(n));
          __syncwarp();
          pf_lo += n;
        }
        if (elect_one()) {
          uint8_t* sa = sbase + stage * C::kStageBytes;
          uint8_t* sb = sa + C::kABytes;
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], tx);
          if (kMc >= 2) {  // my 1/kMc of the A slice, to me and my twins in the other pairs
            constexpr int kRows = 128 / kMc;
            if (A_MN)
              tma_load_2d_2sm_mc(sa + pidx * kMnBlockBytes, &tmap_a, &full_bar[stage],
                                 m0 + 64 * static_cast<int>(pidx), kb * BK, a_mask);
            else
              tma_load_2d_2sm_mc(sa + pidx * (kRows * 128), &tmap_a, &full_bar[stage], kb * BK,
                                 m0 + kRows * static_cast<int>(pidx), a_mask);
          } else if (A_MN) {
            tma_load_2d_2sm(sa, &tmap_a, &full_bar[stage], m0, kb * BK);
            tma_load_2d_2sm(sa + kMnBlockBytes, &tmap_a, &full_bar[stage], m0 + 64, kb * BK);
          } else {
            tma_load_2d_2sm(sa, &tmap_a, &full_bar[stage], kb * BK, m0);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < C::kBBoxesMN; ++j)
              tma_load_2d_2sm(sb + j * kMnBlockBytes, &tmap_b, &full_bar[stage], n0 + 64 * j,
                              kb * BK);
          } else {
            tma_load_2d_2sm(sb, &tmap_b, &full_bar[stage], kb * BK, n0);
          }
          // pull k-block kb + pf_kb into L2 now so its TMA load above (kStages later) does
          // not pay the HBM latency the stage ring is too shallow to cover
          const int kp = kb + ep.pf_kb;
          if (ep.pf_kb > 0 && kp < kb_end) {
            if (A_MN) {
              tma_prefetch_2d(&tmap_a, m0, kp * BK);
              tma_prefetch_2d(&tmap_a, m0 + 64, kp * BK);
            } else {
              tma_prefetch_2d(&tmap_a, kp * BK, m0);
            }
            if (B_MN) {
#pragma unroll
              for (int j = 0; j < C::kBBoxesMN; ++j) tma_prefetch_2d(&tmap_b, n0 + 64 * j, kp * BK);
            } else {
              tma_prefetch_2d(&tmap_b, kp * BK, n0);
            }
          }
        }
        __syncwarp();
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    TRACE_ADD(4, t_prod);
    TL(6);
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------------------------ MMA issuer (pair leader)
      constexpr uint32_t idesc = idesc_bf16_f32(256, BN, A_MN, B_MN);
      // descriptors of stage 0 / k = 0; stage s, k-step k add (s*stage + k*step) >> 4 to the
      // 14-bit start-address field (smem offsets < 256 KB never carry out of it)
      const uint32_t s0 = smem_u32(sbase);
      const uint64_t a0 = A_MN ? smem_desc_sw128(s0, kMnBlockBytes, 1024) : smem_desc_sw128(s0, 16, 1024);
      const uint64_t b0 = B_MN ? smem_desc_sw128(s0 + C::kABytes, kMnBlockBytes, 1024)
                               : smem_desc_sw128(s0 + C::kABytes, 16, 1024);
      constexpr uint32_t kStepA = A_MN ? 2048 : 32, kStepB = B_MN ? 2048 : 32;
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      // one fixed issuing lane: tcgen05.commit only tracks the MMAs of the executing thread
      const bool issuer = elect_one();
      TRACE_T0(t_mma);
      for (int wi = 0, w = seq_tile(0); w < num_work; w = seq_tile(++wi), ++local) {
        const int acc = local % C::kAcc;
        const uint32_t acc_phase = (local / C::kAcc) & 1;
        TRACE_T0(t_te);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        TRACE_ADD(1, t_te);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * C::kAccCols;
        for (int kb = kb_begin; kb < kb_end; ++kb) {
          TRACE_T0(t_f);
          mbar_wait(&full_bar[stage], phase);
          TRACE_ADD(0, t_f);
          if (local == 0 && kb == 0) TL(2);
          tc_fence_after();
          const uint64_t so = static_cast<uint64_t>(stage * C::kStageBytes) >> 4;
          if (issuer) {
  #pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16_2sm(d_tmem, a0 + so + ((k * kStepA) >> 4), b0 + so + ((k * kStepB) >> 4),
                            idesc, (kb != kb_begin || k != 0) ? 1u : 0u);
            // kMc = 2: the stage also holds A multicast by the other pair -> free it there too
            umma_commit_2sm(&empty_bar[stage],
                            kMc >= 2 ? static_cast<uint16_t>((1u << (2 * kMc)) - 1) : pair_mask);
          }
          __syncwarp();
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (issuer) umma_commit_2sm(&tfull_bar[acc], pair_mask);
        __syncwarp();
      }
      TRACE_ADD(2, t_mma);
      TL(3);
    }
  } else if constexpr (kSgd && kLo != 0) {
    // ------------------------------------------------------------ fused SGD, split master
    // m = (hi << 16) | lo with hi = W - (lo > 0x8000) and W = RNE(m) (the bf16 weights the
    // GEMMs read); the update is the fp32 one, then W' = RNE(m'), lo' = the low half of m'
    // except a tie RNE rounds up (low half 0x8000, odd high half), stored as 0x8001 (one
    // fp32 ulp) so the decode stays unambiguous.  kLo = 1: (W, lo) in and out; 2: (W, lo) in,
    // fp32 master + W out; 3: fp32 master in, (W, lo) out.  16 epilogue warps, four per TMEM
    // lane quarter, each 32 rows x 32 columns of a tile: twice the warps of the fp32-master
    // epilogue, whose per-warp chain (TMEM load -> staged load -> update -> store) is
    // latency-bound.  Staging rows are 64 B (16-bit) or 128 B (fp32) under the TMA's
    // swizzle (64 B: SWIZZLE_64B): 16-byte unit u of row r sits at sw(row_bytes * r + 16 u).
    const int q = warp & 3;           // TMEM lane quarter
    const int ew = warp - 2;          // epilogue warp index
    constexpr int kQW = C::kEpiWarps / 4;
    const int cq = ew / 4;            // column slot of this warp inside the quarter
    constexpr int kCW = 32;           // columns per chunk
    static_assert(BN % (kCW * kQW) == 0, "split-master SGD: column chunks split across warps");
    constexpr int kCPW = BN / (kCW * kQW);
    constexpr uint32_t kH = 32 * 64;   // 32 rows x 32 16-bit values
    constexpr uint32_t kF = 32 * 128;  // 32 rows x 32 fp32 values
    constexpr int NB = C::kSgdBufs;
    uint8_t* wbase = epi + ew * NB * C::kSgdBufBytes;
    uint64_t* mb = sgd_bar + ew * NB;
    // TMA swizzle of a 1024-aligned staging block: 128-byte rows (fp32) XOR the 16-byte unit
    // with address bits 7-9, 64-byte rows (16-bit, SWIZZLE_64B) with bits 7-8
    auto sw = [](uint32_t a) -> uint32_t { return a ^ (((a >> 7) & 7u) << 4); };
    auto sw64 = [](uint32_t a) -> uint32_t { return a ^ (((a >> 7) & 3u) << 4); };
    auto coords = [&](int j, int* r0, int* c0) -> bool {
      const int t = seq_tile(j / kCPW);
      if (t >= num_work) return false;
      *r0 = tile_m(t) * 256 + static_cast<int>(pr) * 128 + q * 32;
      *c0 = tile_n(t) * BN + (cq * kCPW + j % kCPW) * kCW;
      return true;
    };
    auto load = [&](int j) {  // lane 0
      int r0, c0;
      if (!coords(j, &r0, &c0)) return;
      uint8_t* dst = wbase + (j % NB) * C::kSgdBufBytes;
      if constexpr (kLoIn) {
        mbar_arrive_expect_tx(&mb[j % NB], 2 * kH);
        tma_load_2d(dst, &tmap_m, &mb[j % NB], c0, r0);          // lo
        tma_load_2d(dst + kH, &pm.m[1], &mb[j % NB], c0, r0);    // W
      } else {
        mbar_arrive_expect_tx(&mb[j % NB], kF);
        tma_load_2d(dst, &pm.m[0], &mb[j % NB], c0, r0);         // fp32 master
      }
    };
    // L2 prefetch (ep.pf_tiles tiles ahead, EDL_GEMM_PF_TILES) of this warp's chunk: the
    // staged TMA load then hits L2 instead of paying the HBM latency
    auto l2pf = [&](int jj) {
      int r0, c0;
      if (!coords(jj, &r0, &c0)) return;
      if constexpr (kLoIn) {
        tma_prefetch_2d(&tmap_m, c0, r0);
        tma_prefetch_2d(&pm.m[1], c0, r0);
      } else {
        tma_prefetch_2d(&pm.m[0], c0, r0);
      }
    };
    if (lane == 0 && !skip_epi) {
      for (int p0 = 0; p0 < (NB > 1 ? NB - 1 : 1); ++p0) load(p0);
      for (int p0 = 1; p0 <= ep.pf_tiles * kCPW; ++p0) l2pf(p0);
    }
    int j = 0;
    int local = 0;
    TRACE_T0(t_epi);
    for (int wi = 0, w = seq_tile(0); w < num_work; w = seq_tile(++wi), ++local) {
      const int acc = local % C::kAcc;
      const uint32_t acc_phase = (local / C::kAcc) & 1;
      TRACE_T0(t_tf);
      mbar_wait(&tfull_bar[acc], acc_phase);
      if (warp == 2) TRACE_ADD(5, t_tf);
      tc_fence_after();
      const uint32_t t_row =
          tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * C::kAccCols;
#pragma unroll 1
      for (int cc = 0; cc < (skip_epi ? 0 : kCPW); ++cc, ++j) {
        const int b = j % NB;
        if (NB > 1 && lane == 0) {
          tma_store_wait_read<0>();  // the buffer refilled next was stored from last
          load(j + NB - 1);
        }
        float g[32];
        TRACE_T0(t_ld);
        {
          uint32_t r[32];
          tmem_ld32(t_row + static_cast<uint32_t>((cq * kCPW + cc) * kCW), r);
          tmem_ld_wait();
          // same numerics as the unfused path: the gradient is rounded to bf16 first
#pragma unroll
          for (int e = 0; e < 32; ++e) g[e] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(r[e])));
        }
        if (warp == 2) TRACE_ADD(9, t_ld);
        TRACE_T0(t_ml);
        mbar_wait(&mb[b], (j / NB) & 1);
        if (warp == 2) TRACE_ADD(7, t_ml);
        TRACE_T0(t_cs);
        uint8_t* buf = wbase + b * C::kSgdBufBytes;
        const uint32_t bo = static_cast<uint32_t>(buf - smem);  // 1024-aligned
        (void)bo;
        // read + update: g <- m'
        if constexpr (kLoIn) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint4 lv = *reinterpret_cast<const uint4*>(buf + sw64(64u * lane + 16u * u));
            const uint4 wv = *reinterpret_cast<const uint4*>(buf + kH + sw64(64u * lane + 16u * u));
            const uint32_t li[4] = {lv.x, lv.y, lv.z, lv.w};
            const uint32_t wi[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) {
              uint32_t m0 = __byte_perm(li[q2], wi[q2], 0x5410);  // W0 << 16 | lo0
              uint32_t m1 = __byte_perm(li[q2], wi[q2], 0x7632);  // W1 << 16 | lo1
              m0 -= ((m0 & 0xFFFFu) + 0x7FFFu) & 0x10000u;        // hi -= (lo > 0x8000)
              m1 -= ((m1 & 0xFFFFu) + 0x7FFFu) & 0x10000u;
              float* gg = &g[8 * u + 2 * q2];
              gg[0] = __fsub_rn(__uint_as_float(m0), __fmul_rn(ep.scale, gg[0]));
              gg[1] = __fsub_rn(__uint_as_float(m1), __fmul_rn(ep.scale, gg[1]));
            }
          }
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 m = *reinterpret_cast<const float4*>(buf + sw(128u * lane + 16u * u));
            float* gg = &g[4 * u];
            gg[0] = __fsub_rn(m.x, __fmul_rn(ep.scale, gg[0]));
            gg[1] = __fsub_rn(m.y, __fmul_rn(ep.scale, gg[1]));
            gg[2] = __fsub_rn(m.z, __fmul_rn(ep.scale, gg[2]));
            gg[3] = __fsub_rn(m.w, __fmul_rn(ep.scale, gg[3]));
          }
        }
        if (warp == 2) TRACE_ADD(11, t_cs);
        __syncwarp();  // outputs overwrite other lanes' input rows (kLo 2 / 3)
        if constexpr (kLoOut) {  // lo' -> [0, 2 KB), W' -> [2 KB, 4 KB)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint32_t wo[4], lo[4];
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) {
              const float f0 = g[8 * u + 2 * q2], f1 = g[8 * u + 2 * q2 + 1];
              wo[q2] = pack_bf16(f0, f1);
              uint32_t b0 = __float_as_uint(f0), b1 = __float_as_uint(f1);
              b0 |= (b0 & 0x1FFFFu) == 0x18000u ? 1u : 0u;  // rounded-up tie -> lo 0x8001
              b1 |= (b1 & 0x1FFFFu) == 0x18000u ? 1u : 0u;
              lo[q2] = __byte_perm(b0, b1, 0x5410);
            }
            *reinterpret_cast<uint4*>(buf + sw64(64u * lane + 16u * u)) =
                make_uint4(lo[0], lo[1], lo[2], lo[3]);
            *reinterpret_cast<uint4*>(buf + kH + sw64(64u * lane + 16u * u)) =
                make_uint4(wo[0], wo[1], wo[2], wo[3]);
          }
        } else {  // fp32 master -> [0, 4 KB), W' -> [4 KB, 6 KB)
#pragma unroll
          for (int u = 0; u < 8; ++u)
            *reinterpret_cast<float4*>(buf + sw(128u * lane + 16u * u)) =
                make_float4(g[4 * u], g[4 * u + 1], g[4 * u + 2], g[4 * u + 3]);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint4 o;
            o.x = pack_bf16(g[8 * u + 0], g[8 * u + 1]);
            o.y = pack_bf16(g[8 * u + 2], g[8 * u + 3]);
            o.z = pack_bf16(g[8 * u + 4], g[8 * u + 5]);
            o.w = pack_bf16(g[8 * u + 6], g[8 * u + 7]);
            *reinterpret_cast<uint4*>(buf + kF + sw64(64u * lane + 16u * u)) = o;
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          int r0, c0;
          coords(j, &r0, &c0);
          if constexpr (kLoOut) {
            tma_store_2d(&tmap_m, buf, c0, r0);
            tma_store_2d(&pm.m[1], buf + kH, c0, r0);
          } else {
            tma_store_2d(&pm.m[0], buf, c0, r0);
            tma_store_2d(&pm.m[1], buf + kF, c0, r0);
          }
          tma_store_commit();
          if (NB == 1) {  // single buffer: refill it for this warp's next chunk
            TRACE_T0(t_wr);
            tma_store_wait_read<0>();
            if (warp == 2) TRACE_ADD(6, t_wr);
            load(j + 1);
          }
          if (ep.pf_tiles > 0) l2pf(j + 1 + ep.pf_tiles * kCPW);
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(&tempty_bar[acc], 2 * pidx);
    }
    if (lane == 0) tma_store_wait<0>();
    if (warp == 2) TRACE_ADD(8, t_epi);
  } else if constexpr (kSgd) {
    // ------------------------------------------------------------ fused SGD epilogue
    // Per warp (32 rows of the CTA's 128) and 64-column chunk: TMA-load the fp32 master
    // chunk (prefetched one chunk ahead, across tiles), fold master -= scale * bf16(acc) in
    // place in swizzled smem, then TMA-store master and the bf16 working weights.
    // HBM per parameter: 4 B master read + 4 B master write + 2 B weight write.
    const int q = warp & 3;          // TMEM lane quarter
    const int ew = warp - 2;         // epilogue warp index
    constexpr int kHalves = C::kEpiWarps / 4;
    const int half = ew / 4;         // which column half of the tile (8 warps)
    constexpr int kChunks = BN / 64;
    static_assert(kChunks % kHalves == 0, "fused SGD: column chunks split across warps");
    constexpr int kCPW = kChunks / kHalves;  // 64-column chunks per warp per tile
    constexpr int NB = C::kSgdBufs;
    uint8_t* wbase = epi + ew * NB * C::kSgdBufBytes;
    uint64_t* mb = sgd_bar + ew * NB;
    auto coords = [&](int j, int* r0, int* c0) -> bool {
      const int t = seq_tile(j / kCPW);
      if (t >= num_work) return false;
      *r0 = tile_m(t) * 256 + static_cast<int>(pr) * 128 + q * 32;
      *c0 = tile_n(t) * BN + (half * kCPW + j % kCPW) * 64;
      return true;
    };
    // fused exchange: does this replica own the rows of chunk j's tile?  (the host keeps
    // whole 256-row tiles inside one owner block and NB == 1)
    auto owner_of = [&](int j) -> int {
      const int t = seq_tile(j / kCPW);
      return kX ? (tile_m(t) * 256) / ep.route_rows : ep.route_me;
    };
    auto next_own = [&](int j) -> int {  // first chunk >= j whose master this warp loads
      if (!kX) return j;
      for (;; ++j) {
        if (seq_tile(j / kCPW) >= num_work) return j;  // past the end: no load
        if (owner_of(j) == ep.route_me) return j;
      }
    };
    auto prefetch = [&](int j) {
      int r0, c0;
      if (!coords(j, &r0, &c0)) return;
      uint8_t* dst = wbase + (j % NB) * C::kSgdBufBytes;
      mbar_arrive_expect_tx(&mb[j % NB], 2 * kEpiChunkBytes);
      tma_load_2d(dst, &tmap_m, &mb[j % NB], c0, r0);
      tma_load_2d(dst + kEpiChunkBytes, &tmap_m, &mb[j % NB], c0 + 32, r0);
    };
    // L2 prefetch of this warp's 32 master rows of tile t (BN columns, 32-column boxes): the
    // master stream is the kernel's HBM traffic, and pf_tiles tiles of lead time keep enough
    // of it in flight without spending shared memory on it
    auto l2_prefetch_tile = [&](int t) {
      if (t >= num_work) return;
      const int r0 = tile_m(t) * 256 + static_cast<int>(pr) * 128 + q * 32;
      const int c0 = tile_n(t) * BN + half * (BN / kHalves);
#pragma unroll
      for (int c = 0; c < BN / kHalves; c += 32) tma_prefetch_2d(&tmap_m, c0 + c, r0);
    };
    if (lane == 0) {
      for (int i = 0; i < ep.pf_tiles && !kX; ++i) l2_prefetch_tile(unit + i * n_units);
      if (NB == 1) {
        if (!skip_epi) prefetch(next_own(0));
      } else {
        for (int p0 = 0; p0 < C::kSgdPfd && !skip_epi; ++p0) prefetch(p0);
      }
    }
    int j = 0;
    int n_used = 0;  // master chunks consumed (NB == 1: barrier phase n_used & 1)
    int local = 0;
    TRACE_T0(t_epi);
    for (int wi = 0, w = seq_tile(0); w < num_work; w = seq_tile(++wi), ++local) {
      const int acc = local % C::kAcc;
      const uint32_t acc_phase = (local / C::kAcc) & 1;
      if (lane == 0 && ep.pf_tiles > 0 && !kX) l2_prefetch_tile(w + ep.pf_tiles * n_units);
      TRACE_T0(t_tf);
      mbar_wait(&tfull_bar[acc], acc_phase);
      if (warp == 2) TRACE_ADD(5, t_tf);
      if (warp == 2 && local == 0) TL(4);
      tc_fence_after();
      const uint32_t t_row =
          tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * C::kAccCols;
#pragma unroll 1
      for (int cc = 0; cc < (skip_epi ? 0 : kCPW); ++cc, ++j) {
        const int b = j % NB;
        if (NB > 1 && lane == 0) {
          TRACE_T0(t_wr);
          // the buffer refilled next was last used by chunk j + PD - NB: its stores (and only
          // those older) must have read it
          tma_store_wait_read<(NB > 1 ? NB - C::kSgdPfd - 1 : 0)>();
          if (warp == 2) TRACE_ADD(6, t_wr);
          prefetch(j + C::kSgdPfd);
        }
        TRACE_T0(t_ld);
        float g[64];
        {
          const uint32_t col = static_cast<uint32_t>((half * kCPW + cc) * 64);
          uint32_t r[32], r2[32];
          tmem_ld32(t_row + col, r);
          tmem_ld32(t_row + col + 32, r2);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            g[e] = __uint_as_float(r[e]);
            g[32 + e] = __uint_as_float(r2[e]);
          }
        }
        // same numerics as the unfused path: the gradient is rounded to bf16 first
#pragma unroll
        for (int e = 0; e < 64; ++e) g[e] = __bfloat162float(__float2bfloat16_rn(g[e]));
        if (warp == 2) TRACE_ADD(9, t_ld);
        uint8_t* buf = wbase + b * C::kSgdBufBytes;
        uint8_t* wrow = buf + 2 * kEpiChunkBytes + lane * 128;
        if constexpr (kX) {
          int r0, c0;
          coords(j, &r0, &c0);
          const int owner = owner_of(j);
          const int tile = seq_tile(j / kCPW);
          // the previous chunk's bulk store (a routed one is not waited on) must have read the
          // staging area before it is written again
          if (lane == 0) tma_store_wait_read<0>();
          __syncwarp();
          if (owner != ep.route_me) {
            // reduce-scatter: my bf16 gradient chunk -> the owner's receive slot, then count it
            // on the owner's arrival counter once the bulk store has completed
#pragma unroll
            for (int j8 = 0; j8 < 8; ++j8) {
              uint4 o;
              o.x = pack_bf16(g[8 * j8 + 0], g[8 * j8 + 1]);
              o.y = pack_bf16(g[8 * j8 + 2], g[8 * j8 + 3]);
              o.z = pack_bf16(g[8 * j8 + 4], g[8 * j8 + 5]);
              o.w = pack_bf16(g[8 * j8 + 6], g[8 * j8 + 7]);
              *reinterpret_cast<uint4*>(wrow + ((j8 ^ (lane & 7)) << 4)) = o;
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && !(ep.dbg & 32)) {  // EDL_GEMM_DBG=32: diagnostics only
              tma_store_2d(&pm.m[owner], buf + 2 * kEpiChunkBytes, c0, r0 - owner * ep.route_rows);
              tma_store_commit();
            }
            __syncwarp();
            continue;
          }
          // my rows: the receive slots hold the sentinel 0xFFFF (a NaN no bf16 rounding
          // produces) until a peer's bf16 chunk lands, so the data is its own arrival signal
          // (no per-chunk completion wait or flag round trip on the sender).  Per 32-column
          // half: walk the ring order, taking my own values from g and each peer's from its
          // slot (4 independent 16-byte loads, re-issued until no sentinel is left), then put
          // the sentinel back for the next mini-batch.
          const size_t rrow = static_cast<size_t>(r0 - ep.route_me * ep.route_rows + lane);
#pragma unroll
          for (int h = 0; h < (ep.dbg & 16 ? 0 : 2); ++h) {  // EDL_GEMM_DBG=16: diagnostics
            float s[32];
#pragma unroll 1
            for (int k = 0; k < ep.x_n; ++k) {
              const int r = ep.x_order[k];
              float v[32];
              if (r == ep.route_me) {
#pragma unroll
                for (int e = 0; e < 32; ++e) v[e] = g[32 * h + e];
              } else {
                const uint4* src =
                    reinterpret_cast<const uint4*>(ep.x_recv[r] + rrow * ep.x_ldr + c0 + 32 * h);
                uint4 u[4];
                const bool no_wait = (ep.dbg & 4) != 0;  // diagnostics only: EDL_GEMM_DBG=4
                const uint64_t t_wait = globaltimer_ns();
                for (;;) {
#pragma unroll
                  for (int q4 = 0; q4 < 4; ++q4)
                    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(u[q4].x), "=r"(u[q4].y), "=r"(u[q4].z), "=r"(u[q4].w)
                                 : "l"(src + q4));
                  bool ready = true;
#pragma unroll
                  for (int q4 = 0; q4 < 4; ++q4) {
                    const uint32_t wv[4] = {u[q4].x, u[q4].y, u[q4].z, u[q4].w};
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                      ready = ready && (wv[e] & 0xFFFFu) != 0xFFFFu && (wv[e] >> 16) != 0xFFFFu;
                  }
                  if (ready || no_wait) break;
                  // a peer died before storing its chunk: fail the launch, don't hang the GPU
                  if (globaltimer_ns() - t_wait > 5000000000ull) __trap();
                  __nanosleep(32);
                }
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                  const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u[q4]);
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    const float2 f2 = __bfloat1622float2(h2[e]);
                    v[8 * q4 + 2 * e] = f2.x;
                    v[8 * q4 + 2 * e + 1] = f2.y;
                  }
                }
                uint4* dst = const_cast<uint4*>(src);  // consumed: sentinel back
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) dst[q4] = make_uint4(~0u, ~0u, ~0u, ~0u);
              }
#pragma unroll
              for (int e = 0; e < 32; ++e) s[e] = k == 0 ? v[e] : __fadd_rn(s[e], v[e]);
            }
#pragma unroll
            for (int e = 0; e < 32; ++e) g[32 * h + e] = s[e];
          }
          (void)tile;
        }
        TRACE_T0(t_ml);
        mbar_wait(&mb[b], NB == 1 ? (n_used & 1) : ((j / NB) & 1));
        ++n_used;
        if (warp == 2) TRACE_ADD(7, t_ml);
        TRACE_T0(t_cs);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint8_t* mrow = buf + h * kEpiChunkBytes + lane * 128;
#pragma unroll
          for (int k4 = 0; k4 < 8; ++k4) {
            float4* pm = reinterpret_cast<float4*>(mrow + ((k4 ^ (lane & 7)) << 4));
            float4 m = *pm;
            const float* gg = &g[h * 32 + k4 * 4];
            m.x = __fsub_rn(m.x, __fmul_rn(ep.scale, gg[0]));
            m.y = __fsub_rn(m.y, __fmul_rn(ep.scale, gg[1]));
            m.z = __fsub_rn(m.z, __fmul_rn(ep.scale, gg[2]));
            m.w = __fsub_rn(m.w, __fmul_rn(ep.scale, gg[3]));
            *pm = m;
            g[h * 32 + k4 * 4 + 0] = m.x;  // reuse g for the new weights
            g[h * 32 + k4 * 4 + 1] = m.y;
            g[h * 32 + k4 * 4 + 2] = m.z;
            g[h * 32 + k4 * 4 + 3] = m.w;
          }
        }
        if (warp == 2) TRACE_ADD(11, t_cs);
        TRACE_T0(t_w8);
        if constexpr (C::kWDirect) {
          int r0, c0;
          coords(j, &r0, &c0);
          uint4* wp = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(ep.C) +
                                               static_cast<size_t>(r0 + lane) * ep.ldc + c0);
#pragma unroll
          for (int j8 = 0; j8 < 8; ++j8) {
            uint4 o;
            o.x = pack_bf16(g[8 * j8 + 0], g[8 * j8 + 1]);
            o.y = pack_bf16(g[8 * j8 + 2], g[8 * j8 + 3]);
            o.z = pack_bf16(g[8 * j8 + 4], g[8 * j8 + 5]);
            o.w = pack_bf16(g[8 * j8 + 6], g[8 * j8 + 7]);
            wp[j8] = o;
          }
        } else {
#pragma unroll
        for (int j8 = 0; j8 < 8; ++j8) {
          uint4 o;
          o.x = pack_bf16(g[8 * j8 + 0], g[8 * j8 + 1]);
          o.y = pack_bf16(g[8 * j8 + 2], g[8 * j8 + 3]);
          o.z = pack_bf16(g[8 * j8 + 4], g[8 * j8 + 5]);
          o.w = pack_bf16(g[8 * j8 + 6], g[8 * j8 + 7]);
          *reinterpret_cast<uint4*>(wrow + ((j8 ^ (lane & 7)) << 4)) = o;
        }
        }
        if (warp == 2) TRACE_ADD(12, t_w8);
        TRACE_T0(t_fe);
        fence_proxy_async_smem();
        __syncwarp();
        if (warp == 2) TRACE_ADD(13, t_fe);
        if (lane == 0) {
          int r0, c0;
          coords(j, &r0, &c0);
          tma_store_2d(&tmap_m, buf, c0, r0);
          tma_store_2d(&tmap_m, buf + kEpiChunkBytes, c0 + 32, r0);
          if (!C::kWDirect) tma_store_2d(&tmap_c, buf + 2 * kEpiChunkBytes, c0, r0);
          if (kX) {  // all-gather: the updated weights into every other replica
            for (int o = 0; o < ep.x_n; ++o)
              if (o != ep.route_me && !(ep.dbg & 8))  // EDL_GEMM_DBG=8: diagnostics only
                tma_store_2d(&pm.w[o], buf + 2 * kEpiChunkBytes, c0, r0);
          }
          tma_store_commit();
          if (NB == 1) {  // single buffer: refill it for this warp's next chunk (next tile)
            TRACE_T0(t_wr);
            tma_store_wait_read<0>();
            if (warp == 2) TRACE_ADD(6, t_wr);
            prefetch(next_own(j + 1));
          }
        }
        if (warp == 2) TRACE_ADD(10, t_cs);
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(&tempty_bar[acc], 2 * pidx);
    }
    if (lane == 0) tma_store_wait<0>();
    if (warp == 2) TRACE_ADD(8, t_epi);
    if (warp == 2) TL(5);
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;  // TMEM lane quarter
    uint8_t* stage_buf = epi + q * 2 * kEpiChunkBytes;
    int buf = 0;
    int local = 0;
    for (int w = unit; w < num_work; w += n_units, ++local) {
      const int acc = local % C::kAcc;
      const uint32_t acc_phase = (local / C::kAcc) & 1;
      const int row0 = tile_m(w) * 256 + static_cast<int>(pr) * 128 + q * 32;
      const int n0 = tile_n(w) * BN;
      // the ReLU' mask of this lane's row (dgrad): pull it into L2 while the mainloop runs,
      // so the epilogue's loads do not pay the HBM latency after the accumulator is ready
      // (EDL_MASK_PF=1; off by default: no measurable gain)
      if (ep.mask && ep.mask_pf && row0 + lane < M) {
        const __nv_bfloat16* mrow =
            ep.mask + static_cast<size_t>(row0 + lane) * ep.ldm + n0;
#pragma unroll
        for (int c = 0; c < BN; c += 64)
          if (n0 + c < N) asm volatile("prefetch.global.L2 [%0];" ::"l"(mrow + c));
      }
      mbar_wait(&tfull_bar[acc], acc_phase);
      if (warp == 2 && local == 0) TL(4);
      tc_fence_after();
      const int row = row0 + lane;
      const uint32_t t_row =
          tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * C::kAccCols;
      const int cw = ep.out_f32 ? 32 : 64;  // columns per 128-byte staging row
      int c_lo = 0, c_hi = BN;
      const float* xrow = nullptr;
      if constexpr (kSk == 2) {
        // split-K reduction through DSMEM (see the kernel comment).  xbuf = this CTA's stage
        // buffers, idle once this pair's MMAs have completed: [128 rows][kXs] fp32
        constexpr int kHalf = BN / 2;
        constexpr int kXs = kHalf + 4;  // padded row: 16-byte accesses of a warp hit all banks
        static_assert(128 * kXs * 4 <= C::kStages * C::kStageBytes, "split-K exchange buffer");
        float* xbuf = reinterpret_cast<float*>(smem);
        uint64_t* xready = sgd_bar;     // arrived by the partner: its stage buffers are free
        uint64_t* xfull = sgd_bar + 1;  // arrived by the partner: my half of its partial is in
        const uint32_t partner = rank ^ 2u;
        if (lane == 0) mbar_arrive_remote(xready, partner);
        mbar_wait(xready, 0);
        if (warp == 2) TL(8);
        const int c_send = (1 - static_cast<int>(pidx)) * kHalf;
        const uint32_t xdst = mapa_u32(xbuf, partner) + static_cast<uint32_t>((q * 32 + lane) * kXs * 4);
#pragma unroll 1
        for (int c = 0; c < kHalf; c += 32) {
          uint32_t r[32];
          tmem_ld32(t_row + c_send + c, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            st_cluster_v4(xdst + static_cast<uint32_t>((c + j) * 4), r[j], r[j + 1], r[j + 2],
                          r[j + 3]);
        }
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_remote_release(xfull, partner);
        mbar_wait_cluster(xfull, 0);
        if (warp == 2) TL(15);
        c_lo = static_cast<int>(pidx) * kHalf;
        c_hi = c_lo + kHalf;
        xrow = xbuf + (q * 32 + lane) * kXs - c_lo;
      }
#pragma unroll 1
      for (int c = c_lo; c < c_hi; c += cw) {
        float v[64];
        {
          uint32_t r[32], r2[32];
          tmem_ld32(t_row + c, r);
          if (!ep.out_f32) tmem_ld32(t_row + c + 32, r2);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          if (!ep.out_f32) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[32 + j] = __uint_as_float(r2[j]);
          }
        }
        if constexpr (kSk == 2) {  // + the other pair's partial (fp32 add: commutative)
          const float4* xp = reinterpret_cast<const float4*>(xrow + c);
#pragma unroll
          for (int j4 = 0; j4 < 16; ++j4) {
            if (j4 >= 8 && ep.out_f32) break;
            const float4 x = xp[j4];
            v[4 * j4] += x.x;
            v[4 * j4 + 1] += x.y;
            v[4 * j4 + 2] += x.z;
            v[4 * j4 + 3] += x.w;
          }
        }
        if (ep.relu) {
#pragma unroll
          for (int j = 0; j < 64; ++j) v[j] = fmaxf(v[j], 0.0f);
        }
        if (ep.mask && row < M) {
          const __nv_bfloat16* mrow = ep.mask + static_cast<size_t>(row) * ep.ldm + n0 + c;
          if (n0 + c + 64 <= N) {
#pragma unroll
            for (int j8 = 0; j8 < 8; ++j8) {
              const uint4 mv = __ldg(reinterpret_cast<const uint4*>(mrow + j8 * 8));
              const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&mv);
#pragma unroll
              for (int t = 0; t < 8; ++t)
                if (!(__bfloat162float(mb[t]) > 0.0f)) v[j8 * 8 + t] = 0.0f;
            }
          } else {
            // constant indices only: a runtime-indexed v[] would live in local memory
#pragma unroll
            for (int j = 0; j < 64; ++j)
              if (n0 + c + j < N && !(__bfloat162float(mrow[j]) > 0.0f)) v[j] = 0.0f;
          }
        }
        // staging buffer reuse: the TMA store issued two chunks ago must have read it
        if (lane == 0) tma_store_wait_read<1>();
        __syncwarp();
        uint8_t* sbuf = stage_buf + buf * kEpiChunkBytes + lane * 128;
        if (ep.out_f32) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint4 o = make_uint4(__float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                                       __float_as_uint(v[4 * j + 2]),
                                       __float_as_uint(v[4 * j + 3]));
            *reinterpret_cast<uint4*>(sbuf + ((j ^ (lane & 7)) << 4)) = o;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint4 o;
            o.x = pack_bf16(v[8 * j + 0], v[8 * j + 1]);
            o.y = pack_bf16(v[8 * j + 2], v[8 * j + 3]);
            o.z = pack_bf16(v[8 * j + 4], v[8 * j + 5]);
            o.w = pack_bf16(v[8 * j + 6], v[8 * j + 7]);
            *reinterpret_cast<uint4*>(sbuf + ((j ^ (lane & 7)) << 4)) = o;
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const CUtensorMap* dst = &tmap_c;
          int drow = row0;
          if (ep.route_rows > 0) {  // reduce-scatter: the owner's receive slot, over NVLink
            const int owner = row0 / ep.route_rows;
            if (owner != ep.route_me) {
              dst = &pm.m[owner];
              drow = row0 - owner * ep.route_rows;
            }
          }
          tma_store_2d(dst, stage_buf + buf * kEpiChunkBytes, n0 + c, drow);
          tma_store_commit();
        }
        if (warp == 2 && local == 0) {
          if (c == 0) TL(9);
          else TL(10);
        }
        buf ^= 1;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(&tempty_bar[acc], 2 * pidx);
    }
    if (warp == 2) TL(11);
    if (lane == 0) tma_store_wait<0>();
    if (warp == 2) TL(5);
    if (warp == 5) TL(12);
  }
  if (warp == 0) TL(13);
  if (warp == 1) TL(14);

  tc_fence_before();
  cluster_sync();
  if (warp == 0) TL(7);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm<C::kTmemCols>(tmem_base);
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// Row-major bf16 matrix [rows][cols] with leading dimension ld (elements); box = 64 cols x
// box_rows rows, 128-byte swizzle.
int make_tmap_t(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                uint32_t box_cols, uint32_t box_rows, bool f32) {
  auto fn = encode_fn();
  if (!fn) return EDL_ECUDA;
  const uint64_t esz = f32 ? 4 : 2;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * esz};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  // the swizzle span matches the box row: 128-byte rows SWIZZLE_128B, 64-byte rows 64B
  const CUtensorMapSwizzle swz =
      box_cols * esz >= 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  CUresult r = fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? EDL_OK : EDL_ECUDA;
}

// Row-major bf16 operand [rows][cols]: box = 64 cols (one 128-byte swizzle row) x box_rows.
int make_tmap(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
              uint32_t box_rows) {
  return make_tmap_t(m, base, rows, cols, ld, 64, box_rows, false);
}

// Programmatic dependent launch of the GEMMs (EDL_PDL=0 disables, for comparisons).
static bool gemm_pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("EDL_PDL");
    on = e ? atoi(e) != 0 : 1;
  }
  return on != 0;
}

int num_sms() {
  static int n = 0;  // identical B200s: the first device's count holds for all
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int BN, bool A_MN, bool B_MN>
int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K,
                const EpiParams& ep, cudaStream_t stream) {
  using Cf = Cfg<BN>;
  auto kern = gemm_bf16_tn_kernel<BN, A_MN, B_MN>;
  static uint64_t attr_set = 0;  // per device: the attribute lives in each context
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_set >> dev & 1)) {
    EDL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      Cf::kSmemBytes));
    attr_set |= 1ull << dev;
  }
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cf::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = gemm_pdl_enabled() ? 1 : 0;
  EDL_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ta, tb, M, N, K, ep));
  return EDL_OK;
}

// prepare_only: set the kernel's attributes on the current device and query its cluster
// occupancy (this also loads the function), without launching -- gemm_prepare_device()
template <int BN, bool A_MN, bool B_MN, bool kSgd = false, int kMc = 1, int kSk = 1,
          bool kX = false, int kLo = 0, bool kAres = false>
int launch_gemm_2sm(const GemmPlan& p, cudaStream_t stream, float scale = 0.f,
                    bool prepare_only = false) {
  using Cf = Cfg2<BN, kSgd, kLo, kAres>;
  auto kern = gemm_bf16_2sm_kernel<BN, A_MN, B_MN, kSgd, kMc, kSk, kX, kLo, kAres>;
  constexpr int kCl = 2 * kMc * kSk;  // CTAs per cluster
  // per device: the attribute lives in each context.  Atomic: a newcomer's replica is
  // prepared on a side thread while the step thread launches on the other devices.
  static std::atomic<uint64_t> attr_set{0};
  static int max_units[64];  // co-resident clusters per device (persistent grid size)
  int dev = 0;
  cudaGetDevice(&dev);
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(Cf::kThreads2);
  cfg.dynamicSmemBytes = Cf::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (!(attr_set.load() >> dev & 1)) {
    EDL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      Cf::kSmemBytes));
    // a persistent grid must not exceed what the GPCs can hold at once (4-CTA clusters
    // need two TPCs of one GPC)
    cfg.gridDim = dim3((num_sms() / kCl) * kCl);  // a whole number of clusters
    int n = 0;
    EDL_CUDA_TRY(cudaOccupancyMaxActiveClusters(&n, kern, &cfg));
    max_units[dev] = n > 0 ? n : 1;
    attr_set.fetch_or(1ull << dev);
  }
  if (prepare_only) return EDL_OK;
  const int work = ((p.M + 255) / 256) * ((p.N + BN - 1) / BN / kMc);
  int units = num_sms() / kCl;
  if (units > max_units[dev]) units = max_units[dev];
  // split-K clusters run exactly one tile (the DSMEM exchange reuses the stage buffers)
  if (kSk == 2 && work > units) return fail(EDL_EINVAL, "gemm: split-K needs one tile per cluster");
  EpiParams ep = p.ep;
  ep.scale = scale;
  cfg.numAttrs = gemm_pdl_enabled() ? 2 : 1;
  cfg.gridDim = dim3(kCl * (work < units ? work : units));
  EDL_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p.ta, p.tb, p.tc, p.tm, p.M, p.N, p.K, ep, p.pm));
  return EDL_OK;
}

}  // namespace

// CTA-pair N tile: fill the 74 TPCs evenly, preferring wide tiles (less smem traffic/MAC).
int gemm_pick_bn_2sm(int M, int N) {
  const int pairs = num_sms() / 2;
  int best = 128;
  double best_eff = -1;
  for (int bn : {256, 192, 128}) {
    const long tiles = static_cast<long>((M + 255) / 256) * ((N + bn - 1) / bn);
    const long waves = (tiles + pairs - 1) / pairs;
    const double eff = static_cast<double>(M) * N / (static_cast<double>(waves) * pairs * 256 * bn) *
                       (bn == 256 ? 1.0 : bn == 192 ? 0.97 : 0.93);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = bn;
    }
  }
  return best;
}

// Picks the N tile so the output-tile count fills the 148 SMs as evenly as possible.
int gemm_pick_bn(int M, int N, bool b_mn) {
  const int sms = num_sms();
  const int cands[] = {256, 224, 192, 160, 128, 112, 96, 64};
  int best = 128;
  double best_eff = -1;
  for (int bn : cands) {
    if (b_mn && bn % 64 != 0 && bn != 112 && bn != 224 && bn != 96 && bn != 160) continue;
    const long tiles = static_cast<long>((M + BM - 1) / BM) * ((N + bn - 1) / bn);
    const long waves = (tiles + sms - 1) / sms;
    // useful work / (waves x full-machine tile capacity), penalise narrow tiles a little
    const double useful = static_cast<double>(M) * N;
    const double cap = static_cast<double>(waves) * sms * BM * bn;
    double eff = useful / cap * (bn >= 128 ? 1.0 : 0.9);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = bn;
    }
  }
  return best;
}

// Split-K 256-wide tiles for few-tile GEMMs (EDL_GEMM_SPLITK=1).  Off by default: measured
// on B200 the M = 512 GEMMs keep the same mainloop time at 256 x 256 split over K as at
// 256 x 128 (both read ~8.3 TB/s of operands from L2, which is the bound, not shared memory)
// and the DSMEM exchange of the fp32 partials adds ~4 us.
static bool gemm_splitk_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("EDL_GEMM_SPLITK");
    on = e ? atoi(e) != 0 : 0;
  }
  return on != 0;
}

// A-operand multicast across two CTA pairs (EDL_GEMM_MC=0 disables, for comparisons).
static bool gemm_multicast_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("EDL_GEMM_MC");
    on = e ? atoi(e) : 2;
  }
  return on != 0;
}


// EDL_SGD_ARES: the A-resident split-master fused SGD kernel
static bool sgd_ares_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("EDL_SGD_ARES");
    on = e ? atoi(e) != 0 : 0;
  }
  return on != 0;
}

// L2 prefetch distances; EDL_GEMM_PF_KB / EDL_GEMM_PF_TILES override (tuning runs).
static void gemm_prefetch_defaults(EpiParams* ep) {
  static int kb = -1, tiles = -1;
  if (kb < 0) {
    const char* e = getenv("EDL_GEMM_PF_KB");
    kb = e ? atoi(e) : 8;
    e = getenv("EDL_GEMM_PF_TILES");
    tiles = e ? atoi(e) : 0;  // measured: 38.9 us per fused wgrad+SGD at 0, 40.2 at 1
  }
  ep->pf_kb = kb;
  ep->pf_tiles = tiles;
  static int mask_pf = -1;
  if (mask_pf < 0) {
    const char* e = getenv("EDL_MASK_PF");
    mask_pf = e ? atoi(e) : 0;  // measured: 816-827k vs 815-820k samples/s, within noise
  }
  ep->mask_pf = mask_pf;
  const char* d = getenv("EDL_GEMM_DBG");
  ep->dbg = d ? atoi(d) : 0;
}

int gemm_plan_init(GemmPlan* p, const void* A, int lda, int a_mn, const void* B, int ldb,
                   int b_mn, void* Cout, int ldc, int M, int N, int K, int relu, int out_f32,
                   const void* mask, int ldm, int bn) {
  if (M <= 0 || N <= 0 || K <= 0) return fail(EDL_EINVAL, "gemm: empty shape");
  if ((lda * 2) % 16 || (ldb * 2) % 16) return fail(EDL_EINVAL, "gemm: 16-byte row alignment");
  // bn: 0 = auto, 1..256 = 1-SM kernel with that N tile, 1000 + x = CTA-pair kernel, N tile x,
  // 2256 = CTA-pair kernel with 256-wide tiles split over K between two pairs
  int cg = 1, sk = 1;
  if (bn >= 2000) {
    cg = 2;
    sk = 2;
    bn -= 2000;
    if (bn != 256) return fail(EDL_EINVAL, "gemm: split-K uses 256-wide tiles");
  } else if (bn >= 1000) {
    cg = 2;
    bn -= 1000;
  } else if (bn <= 0) {
    if (M >= 256 && (ldc * (out_f32 ? 4 : 2)) % 16 == 0) {
      cg = 2;
      bn = gemm_pick_bn_2sm(M, N);
      // few output tiles (the M = 512 GEMMs of the step): 256-wide tiles split over K keep
      // 128+ SMs busy at half the shared-memory bytes per MAC of 256 x 128 tiles
      const int t256 = ((M + 255) / 256) * ((N + 255) / 256);
      if (gemm_splitk_enabled() && t256 <= num_sms() / 4 && 4 * t256 >= (num_sms() * 3) / 4 &&
          (K + BK - 1) / BK >= 8) {
        bn = 256;
        sk = 2;
      }
    } else {
      bn = gemm_pick_bn(M, N, b_mn != 0);
    }
  }
  p->cg = cg;
  if (cg == 2) {
    if (bn != 128 && bn != 192 && bn != 256) return fail(EDL_EINVAL, "gemm: 2-SM N tile");
    // pairs of N tiles share A through multicast when the N tiles pair up and the grid is a
    // single wave (persistent multi-wave grids lose more to 4-CTA cluster placement)
    const int n_tiles = (N + bn - 1) / bn, m_tiles = (M + 255) / 256;
    if (sk == 2 && m_tiles * n_tiles > num_sms() / 4)
      return fail(EDL_EINVAL, "gemm: split-K needs one tile per 4-CTA cluster");
    int mc = (sk == 1 && n_tiles % 2 == 0 && m_tiles * n_tiles <= num_sms() / 2 &&
              gemm_multicast_enabled())
                 ? 2
                 : 1;
    p->sk = sk;
    int rc = a_mn ? make_tmap(&p->ta, A, K, M, lda, 64)
                  : make_tmap(&p->ta, A, M, K, lda, static_cast<uint32_t>(128 / mc));
    if (rc) return fail(rc, "gemm: tensor map A");
    p->mc = mc;
    rc = b_mn ? make_tmap(&p->tb, B, K, N, ldb, 64) : make_tmap(&p->tb, B, N, K, ldb, bn / 2);
    if (rc) return fail(rc, "gemm: tensor map B");
    rc = make_tmap_t(&p->tc, Cout, M, N, ldc, out_f32 ? 32 : 64, 32, out_f32 != 0);
    if (rc) return fail(rc, "gemm: tensor map C");
    if (mask && out_f32) return fail(EDL_EINVAL, "gemm: mask needs a bf16 output");
    p->M = M;
    p->N = N;
    p->K = K;
    p->a_mn = a_mn;
    p->b_mn = b_mn;
    p->bn = bn;
    p->ep = EpiParams{Cout, static_cast<const __nv_bfloat16*>(mask), ldc, ldm, relu, out_f32, 0, 0.f};
    gemm_prefetch_defaults(&p->ep);
    p->tm = p->tc;
    return EDL_OK;
  }
  int rc = a_mn ? make_tmap(&p->ta, A, K, M, lda, 64) : make_tmap(&p->ta, A, M, K, lda, BM);
  if (rc) return fail(rc, "gemm: tensor map A");
  rc = b_mn ? make_tmap(&p->tb, B, K, N, ldb, 64) : make_tmap(&p->tb, B, N, K, ldb, bn);
  if (rc) return fail(rc, "gemm: tensor map B");
  p->M = M;
  p->N = N;
  p->K = K;
  p->a_mn = a_mn;
  p->b_mn = b_mn;
  p->bn = bn;
  p->ep = EpiParams{Cout, static_cast<const __nv_bfloat16*>(mask), ldc, ldm, relu, out_f32, 0, 0.f};
  return EDL_OK;
}

int gemm_plan_route(GemmPlan* p, int rows_per_owner, int me, void* const* dst, int n_owner) {
  if (p->cg != 2 || p->ep.out_f32 || p->ep.mask || p->ep.sgd)
    return fail(EDL_EINVAL, "gemm route: needs a plain bf16 CTA-pair plan");
  if (n_owner < 1 || n_owner > kMaxPeerMaps || rows_per_owner <= 0 || rows_per_owner % 32 ||
      rows_per_owner * n_owner != p->M || me < 0 || me >= n_owner)
    return fail(EDL_EINVAL, "gemm route: owner blocks must tile M in 32-row multiples");
  for (int o = 0; o < n_owner; ++o) {
    if (o == me) {
      p->pm.m[o] = p->tc;
      continue;
    }
    const int rc = make_tmap_t(&p->pm.m[o], dst[o], rows_per_owner, p->N, p->N, 64, 32, false);
    if (rc) return fail(rc, "gemm route: tensor map of a peer receive slot");
  }
  p->ep.route_rows = rows_per_owner;
  p->ep.route_me = me;
  return EDL_OK;
}

int gemm_plan_exchange(GemmPlan* p, int rows_per_owner, int me, int n, void* const* recv_dst,
                       __nv_bfloat16* const* w_dst, const __nv_bfloat16* const* recv_src,
                       int ld_recv, const int* order) {
  if (!p->ep.sgd || p->cg != 2 || p->bn != 128 || p->mc != 1)
    return fail(EDL_EINVAL, "gemm exchange: needs a fused-SGD CTA-pair plan (N tile 128)");
  if (Cfg2<128, true>::kSgdBufs != 1)
    return fail(EDL_EINVAL, "gemm exchange: single-buffer fused-SGD epilogue only");
  if (n < 2 || n > kMaxPeerMaps || me < 0 || me >= n || rows_per_owner <= 0 ||
      rows_per_owner % 256 || rows_per_owner * n != p->M || p->N % 128)
    return fail(EDL_EINVAL, "gemm exchange: owner blocks must tile M in 256-row multiples");
  for (int o = 0; o < n; ++o) {
    p->ep.x_recv[o] = recv_src[o];
    p->ep.x_order[o] = order[o];
    if (o == me) {
      p->pm.m[o] = p->tc;
      p->pm.w[o] = p->tc;
      continue;
    }
    int rc = make_tmap_t(&p->pm.m[o], recv_dst[o], rows_per_owner, p->N, p->N, 64, 32, false);
    if (rc) return fail(rc, "gemm exchange: tensor map of a peer receive slot");
    rc = make_tmap_t(&p->pm.w[o], w_dst[o], p->M, p->N, p->N, 64, 32, false);
    if (rc) return fail(rc, "gemm exchange: tensor map of a peer's weights");
  }
  p->ep.route_rows = rows_per_owner;
  p->ep.route_me = me;
  p->ep.xchg = 1;
  p->ep.x_n = n;
  p->ep.x_ldr = ld_recv;
  return EDL_OK;
}

// Loads and configures, on the current device, the GEMM variants a training step launches
// (fwd / dgrad / wgrad / fused wgrad+SGD at the CTA-pair tile), so the first mini-batch on a
// newly added GPU does not pay lazy module loading and attribute setup on the switch step.
int gemm_prepare_device() {
  GemmPlan p;
  int rc = EDL_OK;
  if (!rc) rc = launch_gemm_2sm<128, false, false, false, 2>(p, nullptr, 0.f, true);
  if (!rc) rc = launch_gemm_2sm<128, false, true, false, 2>(p, nullptr, 0.f, true);
  if (!rc) rc = launch_gemm_2sm<128, true, true, false, 1>(p, nullptr, 0.f, true);
  if (!rc) rc = launch_gemm_2sm<128, true, true, true, 1>(p, nullptr, 0.f, true);
  if (!rc) rc = launch_gemm_2sm<128, true, true, true, 1, 1, false, 1>(p, nullptr, 0.f, true);
  if (!rc) rc = launch_gemm_2sm<128, true, true, true, 1, 1, false, 2>(p, nullptr, 0.f, true);
  if (!rc) rc = launch_gemm_2sm<128, true, true, true, 1, 1, false, 3>(p, nullptr, 0.f, true);
  if (!rc && sgd_ares_enabled()) {
    rc = launch_gemm_2sm<128, true, true, true, 1, 1, false, 1, true>(p, nullptr, 0.f, true);
    if (!rc) rc = launch_gemm_2sm<128, true, true, true, 1, 1, false, 3, true>(p, nullptr, 0.f, true);
  }
  if (!rc) rc = launch_gemm_2sm<128, false, false, false, 1>(p, nullptr, 0.f, true);
  if (!rc) rc = launch_gemm_2sm<128, false, true, false, 1>(p, nullptr, 0.f, true);
  if (!rc) rc = gemm_pair_prepare_device(nullptr);
  if (!rc) rc = wgrad_sgd_bres_prepare_device(nullptr);
  return rc;
}

int gemm_plan_run_wait(const GemmPlan& p, cudaStream_t stream, const uint32_t* flags, int n,
                       uint32_t epoch) {
  if (!flags || n <= 0) return gemm_plan_run(p, stream);
  GemmPlan q = p;
  q.ep.wait_flags = flags;
  q.ep.wait_n = n;
  q.ep.wait_epoch = epoch;
  return gemm_plan_run(q, stream);
}

int gemm_plan_init_sgd(GemmPlan* p, const void* A, int lda, int a_mn, const void* B, int ldb,
                       int b_mn, float* master, __nv_bfloat16* W, int ldw, int M, int N, int K) {
  if (!a_mn || !b_mn) return fail(EDL_EINVAL, "fused SGD: weight-gradient layout (MN-major A/B)");
  if (M <= 0 || N <= 0 || K <= 0 || (ldw * 2) % 16) return fail(EDL_EINVAL, "fused SGD: shape");
  // N tile 128 (measured: 256 halves the operand re-reads but is slower in the step);
  // EDL_SGD_BN=256 selects the wide tile
  static int sgd_bn = -1;
  if (sgd_bn < 0) {
    const char* e = getenv("EDL_SGD_BN");
    sgd_bn = e ? atoi(e) : 128;
  }
  const int bn = (sgd_bn == 256 && N >= 256) ? 256 : 128;
  int rc = gemm_plan_init(p, A, lda, a_mn, B, ldb, b_mn, W, ldw, M, N, K, 0, 0, nullptr, 0,
                          1000 + bn);
  if (rc) return rc;
  // EDL_SGD_MC=1: 4-CTA clusters multicast the shared A (dY) slice across two pairs
  static int sgd_mc = -1;
  if (sgd_mc < 0) {
    const char* e = getenv("EDL_SGD_MC");
    sgd_mc = e ? atoi(e) : 0;
  }
  p->mc = (sgd_mc && ((N + bn - 1) / bn) % 2 == 0) ? 2 : 1;
  rc = make_tmap_t(&p->tm, master, M, N, ldw, 32, 32, true);
  if (rc) return fail(rc, "fused SGD: tensor map master");
  p->ep.sgd = 1;
  return EDL_OK;
}

int gemm_plan_init_sgd_lo(GemmPlan* p, const void* A, int lda, const void* B, int ldb,
                          uint16_t* lo, __nv_bfloat16* W, float* master, int ldw, int M, int N,
                          int K) {
  if (M <= 0 || N <= 0 || K <= 0 || (ldw * 2) % 16) return fail(EDL_EINVAL, "split-master SGD: shape");
  int rc = gemm_plan_init(p, A, lda, 1, B, ldb, 1, W, ldw, M, N, K, 0, 0, nullptr, 0, 1128);
  if (rc) return rc;
  p->mc = 1;
  // 32 x 32 boxes (one epilogue warp's chunk): the low halves and the weights (pm.m[1]; the
  // plan's own 64-column weight map tc stays for the fp32-master kernel)
  rc = make_tmap_t(&p->tm, lo, M, N, ldw, 32, 32, false);
  if (rc) return fail(rc, "split-master SGD: tensor map of the low halves");
  rc = make_tmap_t(&p->pm.m[1], W, M, N, ldw, 32, 32, false);
  if (rc) return fail(rc, "split-master SGD: tensor map of the weights");
  if (master) {  // the conversion launches (gemm_plan_lo_mode 2 / 3) read or write it
    rc = make_tmap_t(&p->pm.m[0], master, M, N, ldw, 32, 32, true);
    if (rc) return fail(rc, "split-master SGD: tensor map of the fp32 master");
  }
  p->ep.sgd = 1;
  p->lo = 1;
  p->lo_master = master != nullptr;
  return EDL_OK;
}

int gemm_plan_run(const GemmPlan& p, cudaStream_t stream, float sgd_scale) {
  const int a_mn = p.a_mn, b_mn = p.b_mn;
  if (p.ep.sgd) {
    if (p.cg != 2 || (p.bn != 128 && p.bn != 256) || !a_mn || !b_mn)
      return fail(EDL_EINVAL, "gemm: fused SGD plans are CTA-pair, N tile 128/256, MN-major A/B");
    // opt-in (EDL_SGD_BRES=1): the B-resident kernel (wgrad_sgd.cu) streams ~1/3 fewer
    // operand bytes per parameter; measured slower, the epilogue bounds this GEMM
    if (p.lo) {
      if (p.bn != 128 || p.mc != 1 || p.ep.xchg) return fail(EDL_EINVAL, "gemm: split-master plan shape");
      if (p.lo != 1 && !p.lo_master) return fail(EDL_EINVAL, "gemm: split-master conversion needs the fp32 master");
      if (p.lo == 2) return launch_gemm_2sm<128, true, true, true, 1, 1, false, 2>(p, stream, sgd_scale);
      // A-resident variant (EDL_SGD_ARES, K <= 512 in whole k-blocks)
      const bool ares = sgd_ares_enabled() && p.K % BK == 0 && p.K <= 512;
      if (p.lo == 3) {
        if (ares) return launch_gemm_2sm<128, true, true, true, 1, 1, false, 3, true>(p, stream, sgd_scale);
        return launch_gemm_2sm<128, true, true, true, 1, 1, false, 3>(p, stream, sgd_scale);
      }
      if (ares) return launch_gemm_2sm<128, true, true, true, 1, 1, false, 1, true>(p, stream, sgd_scale);
      return launch_gemm_2sm<128, true, true, true, 1, 1, false, 1>(p, stream, sgd_scale);
    }
    if (wgrad_sgd_bres_eligible(p)) return wgrad_sgd_bres_run(p, stream, sgd_scale);
    if (p.ep.xchg) {
      if (p.bn != 128 || p.mc != 1) return fail(EDL_EINVAL, "gemm: fused-exchange plan shape");
      return launch_gemm_2sm<128, true, true, true, 1, 1, true>(p, stream, sgd_scale);
    }
    if (p.mc == 2 && p.bn == 128) return launch_gemm_2sm<128, true, true, true, 2>(p, stream, sgd_scale);
    if (p.bn == 256) return launch_gemm_2sm<256, true, true, true, 1>(p, stream, sgd_scale);
    return launch_gemm_2sm<128, true, true, true, 1>(p, stream, sgd_scale);
  }
  if (p.cg == 2 && p.sk == 2) {
    if (p.bn != 256 || p.mc != 1) return fail(EDL_EINVAL, "gemm: split-K plan");
    if (!a_mn && !b_mn) return launch_gemm_2sm<256, false, false, false, 1, 2>(p, stream);
    if (!a_mn && b_mn) return launch_gemm_2sm<256, false, true, false, 1, 2>(p, stream);
    if (a_mn && !b_mn) return launch_gemm_2sm<256, true, false, false, 1, 2>(p, stream);
    return launch_gemm_2sm<256, true, true, false, 1, 2>(p, stream);
  }
  if (p.cg == 2) {
#define EDL_GEMM2_MC(BNV, AM, BM_, MC) \
  return launch_gemm_2sm<BNV, AM, BM_, false, MC>(p, stream);
#define EDL_GEMM2_CASE(BNV)                                                          \
  case BNV:                                                                          \
    if (p.mc == 2) {                                                                 \
      if (!a_mn && !b_mn) EDL_GEMM2_MC(BNV, false, false, 2)                         \
      if (!a_mn && b_mn) EDL_GEMM2_MC(BNV, false, true, 2)                           \
      if (a_mn && !b_mn) EDL_GEMM2_MC(BNV, true, false, 2)                           \
      EDL_GEMM2_MC(BNV, true, true, 2)                                               \
    }                                                                                \
    if (!a_mn && !b_mn) EDL_GEMM2_MC(BNV, false, false, 1)                           \
    if (!a_mn && b_mn) EDL_GEMM2_MC(BNV, false, true, 1)                             \
    if (a_mn && !b_mn) EDL_GEMM2_MC(BNV, true, false, 1)                             \
    EDL_GEMM2_MC(BNV, true, true, 1)
    switch (p.bn) {
      EDL_GEMM2_CASE(128)
      EDL_GEMM2_CASE(192)
      EDL_GEMM2_CASE(256)
      default:
        return fail(EDL_EINVAL, "gemm: unsupported 2-SM N tile");
    }
#undef EDL_GEMM2_CASE
#undef EDL_GEMM2_MC
  }
#define EDL_GEMM_CASE(BNV)                                                                  \
  case BNV:                                                                                 \
    if (!a_mn && !b_mn) return launch_gemm<BNV, false, false>(p.ta, p.tb, p.M, p.N, p.K, p.ep, stream); \
    if (!a_mn && b_mn) return launch_gemm<BNV, false, true>(p.ta, p.tb, p.M, p.N, p.K, p.ep, stream);   \
    if (a_mn && !b_mn) return launch_gemm<BNV, true, false>(p.ta, p.tb, p.M, p.N, p.K, p.ep, stream);   \
    return launch_gemm<BNV, true, true>(p.ta, p.tb, p.M, p.N, p.K, p.ep, stream);
  switch (p.bn) {
    EDL_GEMM_CASE(64)
    EDL_GEMM_CASE(96)
    EDL_GEMM_CASE(112)
    EDL_GEMM_CASE(128)
    EDL_GEMM_CASE(160)
    EDL_GEMM_CASE(192)
    EDL_GEMM_CASE(224)
    EDL_GEMM_CASE(256)
    default:
      return fail(EDL_EINVAL, "gemm: unsupported N tile");
  }
#undef EDL_GEMM_CASE
}

int gemm_bf16(const void* A, int lda, int a_mn, const void* B, int ldb, int b_mn, void* Cout,
              int ldc, int M, int N, int K, int relu, int out_f32, const void* mask, int ldm,
              int bn, cudaStream_t stream) {
  GemmPlan p;
  int rc = gemm_plan_init(&p, A, lda, a_mn, B, ldb, b_mn, Cout, ldc, M, N, K, relu, out_f32, mask,
                          ldm, bn);
  if (rc) return rc;
  return gemm_plan_run(p, stream);
}

}  // namespace edl

#ifdef EDL_GEMM_TRACE
extern "C" int edl_debug_gemm_timeline(unsigned long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, edl::g_gemm_tl, sizeof(edl::g_gemm_tl));
  return 0;
}
extern "C" int edl_debug_gemm_trace(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, edl::g_gemm_trace, sizeof(edl::g_gemm_trace));
  if (reset) {
    static unsigned long long zero[296][16];
    cudaMemcpyToSymbol(edl::g_gemm_trace, zero, sizeof(zero));
  }
  return 0;
}
#endif
