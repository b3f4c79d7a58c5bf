// Backward pair kernel (N = 1, fused-update path): the data-gradient GEMM of layer l-1 and
// the weight-gradient GEMM + SGD update of layer l in ONE persistent launch.
//
//   D tiles  dX_{l-1} = relu'(act[l-1]) * (dY_{l-1} . W_{l-1})   tensor-bound (K = out = 4096)
//   W tiles  master_l -= scale * bf16(dY_l^T . X_l); W_l = bf16    HBM-bound (K = batch = 512)
//
// The two are independent (dgrad l-1 reads W_{l-1}, the update writes W_l; dgrad l, which
// reads W_l, finished in the previous launch), and they load different units: the D tiles
// keep the tensor pipe busy for 64 k-blocks while the W tiles' epilogues stream 10 bytes per
// parameter through HBM.  Run back to back (round 1) the dgrad GEMM left HBM idle and the
// fused wgrad+SGD GEMM left the tensor pipe at 24%; here every CTA pair interleaves them: the
// MMA warp alternates one W tile (8 k-blocks) with a slice of its D tile's k-blocks, so the
// epilogue warps always have a finished W accumulator to update while the D accumulator
// grows.  TMEM (512 columns) holds three W accumulators in a ring and one D accumulator.
//
// Roles per CTA (cta_group::2 pairs, 320 threads): warp 0 TMA producer, warp 1 MMA issuer
// (pair leader), warps 2-9 epilogue (two per TMEM lane quarter, each half of the 128-column
// tile).  Both producer and MMA walk the same deterministic segment sequence; the epilogue
// walks it too and acts on the segments that complete a tile.
//
// Measured on B200 (profiles/r02_pair.md): parity-green, but no faster than the two
// kernels back to back (65 vs 23 + 43 us per layer): both halves are bound by the same
// L2 -> SM operand stream (474 MB per launch at ~8 TB/s, ncu l1tex__m_xbar2l1tex_read_bytes;
// the epilogue warps wait on the MMA, the MMA on the loads), so overlapping them gains
// nothing.  Opt-in (EDL_BWD_PAIR=1); the weight-gradient kernel that cuts those bytes is
// wgrad_sgd.cu.
//
// Numerics are exactly those of the two kernels it replaces (gemm_sm100.cu): fp32 TMEM
// accumulation of bf16 products in K order, the gradient rounded to bf16 before the update,
// separate multiply / subtract roundings, RNE to bf16.  This is the per-sample gradient +
// sgd_step of the reference (proj/src/trainer.cpp:14-61) for the MLP workload.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "edl_internal.hpp"
#include "sm100.cuh"

namespace edl {
namespace {

using namespace sm100;

constexpr int kBK = 64;
constexpr uint32_t kMnBox = 64 * kBK * 2;     // 64 (M/N) x 64 (K) bf16 box: 8 KB
constexpr uint32_t kABytes = 128 * kBK * 2;   // per CTA: 128 rows x 64 K
constexpr uint32_t kBBytes = 64 * kBK * 2;    // per CTA: 64 columns (half of N = 128) x 64 K
constexpr uint32_t kStage = kABytes + kBBytes;
constexpr int kStages = 5;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr uint32_t kChunk = 32 * 128;         // one warp's 32 rows x 128 B box
constexpr uint32_t kBuf = 3 * kChunk;         // master 2 x 4 KB (fp32 32 cols each) + W 4 KB
constexpr uint32_t kEpiBytes = kEpiWarps * kBuf;
constexpr int kWAcc = 3;                      // W accumulators in the TMEM ring; D uses #3
constexpr uint32_t kSmemBytes = kStages * kStage + kEpiBytes + 1024 + 512;
constexpr int kMaxUnits = 128;

struct PairArgs {
  CUtensorMap d_a, d_b, d_c;        // dgrad: dY_{l-1} K-major, W_{l-1} MN-major, dX out
  CUtensorMap w_a, w_b, w_m, w_c;   // wgrad: dY_l MN-major, X_l MN-major, master, W_l
  const __nv_bfloat16* mask;        // act[l-1] [M_d][ldm]: relu' of the dgrad output
  int ldm;
  int d_mt, d_nt, d_kb, d_a_boxes;  // D: M/256, N/128, K/64, A boxes per k-block (1 or 2)
  int w_mt, w_nt, w_kb;             // W: M/256, N/128, K/64
  float scale;                      // f32(eta_t / count)
  int pf_kb;                        // L2 prefetch distance of the operand loads (k-blocks)
  uint16_t w_begin[kMaxUnits + 1];  // unit u owns W tiles [w_begin[u], w_begin[u+1])
};

enum { kD = 0, kW = 1 };

// The unit's segment sequence: W tile i, then the i-th slice of the unit's D k-blocks, for
// i = 0 .. nw-1 (D tiles u, u + U, ... concatenated; a slice is cut at D tile boundaries).
// f(kind, tile, kb0, kb1, first, last, acc, acc_phase)
template <class F>
__device__ __forceinline__ void walk(const PairArgs& a, int u, int U, F&& f) {
  const int nD = a.d_mt * a.d_nt;
  const int nd = u < nD ? (nD - 1 - u) / U + 1 : 0;
  const int w0 = a.w_begin[u], nw = a.w_begin[u + 1] - w0;
  const int TD = nd * a.d_kb;
  const int slots = nw > 0 ? nw : 1;
  for (int i = 0; i < slots; ++i) {
    if (i < nw) f(kW, w0 + i, 0, a.w_kb, true, true, i % kWAcc, static_cast<uint32_t>((i / kWAcc) & 1));
    int lo = static_cast<int>(static_cast<long long>(i) * TD / slots);
    const int hi = static_cast<int>(static_cast<long long>(i + 1) * TD / slots);
    while (lo < hi) {
      const int j = lo / a.d_kb, kb0 = lo % a.d_kb;
      const int kb1 = min(a.d_kb, kb0 + (hi - lo));
      f(kD, u + j * U, kb0, kb1, kb0 == 0, kb1 == a.d_kb, kWAcc, static_cast<uint32_t>(j & 1));
      lo += kb1 - kb0;
    }
  }
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

__global__ void __launch_bounds__(kThreads, 1) bwd_pair_kernel(const __grid_constant__ PairArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* epi = smem + kStages * kStage;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(epi + kEpiBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull = empty_bar + kStages;
  uint64_t* tempty = tfull + 4;
  uint64_t* mbar = tempty + 4;  // per epilogue warp: master chunk loaded
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + kEpiWarps);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t pr = cluster_ctarank() & 1;
  const bool leader = pr == 0;
  const int u = blockIdx.x / 2, U = gridDim.x / 2;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&a.d_a);
    prefetch_tmap(&a.d_b);
    prefetch_tmap(&a.d_c);
    prefetch_tmap(&a.w_a);
    prefetch_tmap(&a.w_b);
    prefetch_tmap(&a.w_m);
    prefetch_tmap(&a.w_c);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * kEpiWarps);  // lane 0 of every epilogue warp, both CTAs
    }
    for (int i = 0; i < kEpiWarps; ++i) mbar_init(&mbar[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_2sm<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();
  griddep_launch();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    int stage = 0;
    uint32_t phase = 0;
    walk(a, u, U, [&](int kind, int tile, int kb0, int kb1, bool, bool, int, uint32_t) {
      int m0, n0;
      if (kind == kW) {
        m0 = (tile / a.w_nt) * 256 + static_cast<int>(pr) * 128;
        n0 = (tile % a.w_nt) * 128 + static_cast<int>(pr) * 64;
      } else {
        m0 = (tile % a.d_mt) * 256 + static_cast<int>(pr) * 128;
        n0 = (tile / a.d_mt) * 128 + static_cast<int>(pr) * 64;
      }
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (elect_one()) {
          uint8_t* sa = smem + stage * kStage;
          uint8_t* sb = sa + kABytes;
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * kStage);
          if (kind == kW) {  // dY_l [b][out] MN-major: two 64-wide M boxes
            tma_load_2d_2sm(sa, &a.w_a, &full_bar[stage], m0, kb * kBK);
            tma_load_2d_2sm(sa + kMnBox, &a.w_a, &full_bar[stage], m0 + 64, kb * kBK);
            tma_load_2d_2sm(sb, &a.w_b, &full_bar[stage], n0, kb * kBK);
          } else {  // dY_{l-1} [b][out] K-major (one 128-row box or two 64-row boxes)
            if (a.d_a_boxes == 1) {
              tma_load_2d_2sm(sa, &a.d_a, &full_bar[stage], kb * kBK, m0);
            } else {
              tma_load_2d_2sm(sa, &a.d_a, &full_bar[stage], kb * kBK, m0);
              tma_load_2d_2sm(sa + 64 * 128, &a.d_a, &full_bar[stage], kb * kBK, m0 + 64);
            }
            tma_load_2d_2sm(sb, &a.d_b, &full_bar[stage], n0, kb * kBK);
          }
          // L2 prefetch a few k-blocks ahead (the stage ring alone cannot cover the HBM
          // latency of W_{l-1} / act[l]): D tiles kb + pf of the same tile, W tiles the same
          // k-block of the unit's next W tile (a W tile is only 8 k-blocks long)
          if (kind == kD) {
            const int kp = kb + a.pf_kb;
            if (a.pf_kb > 0 && kp < a.d_kb) {
              tma_prefetch_2d(&a.d_a, kp * kBK, m0);
              if (a.d_a_boxes == 2) tma_prefetch_2d(&a.d_a, kp * kBK, m0 + 64);
              tma_prefetch_2d(&a.d_b, n0, kp * kBK);
            }
          } else if (a.pf_kb > 0 && tile + 1 < a.w_begin[u + 1]) {
            const int m1 = ((tile + 1) / a.w_nt) * 256 + static_cast<int>(pr) * 128;
            const int n1 = ((tile + 1) % a.w_nt) * 128 + static_cast<int>(pr) * 64;
            tma_prefetch_2d(&a.w_a, m1, kb * kBK);
            tma_prefetch_2d(&a.w_a, m1 + 64, kb * kBK);
            tma_prefetch_2d(&a.w_b, n1, kb * kBK);
          }
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    });
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------------------------ MMA issuer (pair leader)
      constexpr uint32_t idesc_w = idesc_bf16_f32(256, 128, true, true);
      constexpr uint32_t idesc_d = idesc_bf16_f32(256, 128, false, true);
      const uint32_t s0 = smem_u32(smem);
      const uint64_t a_mn = smem_desc_sw128(s0, kMnBox, 1024);
      const uint64_t a_k = smem_desc_sw128(s0, 16, 1024);
      const uint64_t b0 = smem_desc_sw128(s0 + kABytes, kMnBox, 1024);
      int stage = 0;
      uint32_t phase = 0;
      const bool issuer = elect_one();
      walk(a, u, U, [&](int kind, int, int kb0, int kb1, bool first, bool last, int acc,
                        uint32_t acc_phase) {
        if (first) {
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
        }
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc) * 128;
        const uint32_t idesc = kind == kW ? idesc_w : idesc_d;
        const uint64_t a0 = kind == kW ? a_mn : a_k;
        const uint32_t step_a = kind == kW ? 2048 : 32;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t so = static_cast<uint64_t>(stage * kStage) >> 4;
          if (issuer) {
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              umma_bf16_2sm(d_tmem, a0 + so + ((k * step_a) >> 4), b0 + so + ((k * 2048) >> 4),
                            idesc, (kb | k) != 0 ? 1u : 0u);
            umma_commit_2sm(&empty_bar[stage], 0x3);
          }
          __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (last) {
          if (issuer) umma_commit_2sm(&tfull[acc], 0x3);
          __syncwarp();
        }
      });
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;      // TMEM lane quarter
    const int ew = warp - 2;     // epilogue warp
    const int half = ew / 4;     // column half of the 128-column tile
    uint8_t* buf = epi + ew * kBuf;
    uint8_t* wrow = buf + 2 * kChunk + lane * 128;
    uint64_t* mb = &mbar[ew];
    const int w0 = a.w_begin[u], nw = a.w_begin[u + 1] - w0;
    auto w_coords = [&](int i, int* r0, int* c0) {
      const int t = w0 + i;
      *r0 = (t / a.w_nt) * 256 + static_cast<int>(pr) * 128 + q * 32;
      *c0 = (t % a.w_nt) * 128 + half * 64;
    };
    auto prefetch = [&](int i) {  // master chunk of this warp's share of W tile i
      if (i >= nw) return;
      int r0, c0;
      w_coords(i, &r0, &c0);
      mbar_arrive_expect_tx(mb, 2 * kChunk);
      tma_load_2d(buf, &a.w_m, mb, c0, r0);
      tma_load_2d(buf + kChunk, &a.w_m, mb, c0 + 32, r0);
    };
    if (lane == 0) prefetch(0);
    int n_used = 0;
    walk(a, u, U, [&](int kind, int tile, int, int, bool, bool last, int acc, uint32_t acc_phase) {
      if (!last) return;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                             static_cast<uint32_t>(acc) * 128 + static_cast<uint32_t>(half) * 64;
      float g[64];
      {
        uint32_t r[32], r2[32];
        tmem_ld32(t_row, r);
        tmem_ld32(t_row + 32, r2);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          g[e] = __uint_as_float(r[e]);
          g[32 + e] = __uint_as_float(r2[e]);
        }
      }
      if (kind == kW) {
        const int i = tile - w0;
        // same numerics as the unfused path: the gradient is rounded to bf16 first
#pragma unroll
        for (int e = 0; e < 64; ++e) g[e] = __bfloat162float(__float2bfloat16_rn(g[e]));
        mbar_wait(mb, n_used & 1);
        ++n_used;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint8_t* mrow = buf + h * kChunk + lane * 128;
#pragma unroll
          for (int k4 = 0; k4 < 8; ++k4) {
            float4* pm = reinterpret_cast<float4*>(mrow + ((k4 ^ (lane & 7)) << 4));
            float4 m = *pm;
            const float* gg = &g[h * 32 + k4 * 4];
            m.x = __fsub_rn(m.x, __fmul_rn(a.scale, gg[0]));
            m.y = __fsub_rn(m.y, __fmul_rn(a.scale, gg[1]));
            m.z = __fsub_rn(m.z, __fmul_rn(a.scale, gg[2]));
            m.w = __fsub_rn(m.w, __fmul_rn(a.scale, gg[3]));
            *pm = m;
            g[h * 32 + k4 * 4 + 0] = m.x;
            g[h * 32 + k4 * 4 + 1] = m.y;
            g[h * 32 + k4 * 4 + 2] = m.z;
            g[h * 32 + k4 * 4 + 3] = m.w;
          }
        }
#pragma unroll
        for (int j8 = 0; j8 < 8; ++j8) {
          uint4 o;
          o.x = pack2(g[8 * j8 + 0], g[8 * j8 + 1]);
          o.y = pack2(g[8 * j8 + 2], g[8 * j8 + 3]);
          o.z = pack2(g[8 * j8 + 4], g[8 * j8 + 5]);
          o.w = pack2(g[8 * j8 + 6], g[8 * j8 + 7]);
          *reinterpret_cast<uint4*>(wrow + ((j8 ^ (lane & 7)) << 4)) = o;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          int r0, c0;
          w_coords(i, &r0, &c0);
          tma_store_2d(&a.w_m, buf, c0, r0);
          tma_store_2d(&a.w_m, buf + kChunk, c0 + 32, r0);
          tma_store_2d(&a.w_c, buf + 2 * kChunk, c0, r0);
          tma_store_commit();
          tma_store_wait_read<0>();  // the buffer is refilled with the next chunk's master
          prefetch(i + 1);
        }
      } else {
        // dgrad tile: relu' mask of act[l-1], bf16, TMA store (staged in the W slot, whose
        // previous store has been read: every chunk waits for its stores' smem reads)
        const int r0 = (tile % a.d_mt) * 256 + static_cast<int>(pr) * 128 + q * 32;
        const int c0 = (tile / a.d_mt) * 128 + half * 64;
        const uint4* mrow = reinterpret_cast<const uint4*>(
            a.mask + static_cast<size_t>(r0 + lane) * a.ldm + c0);
#pragma unroll
        for (int j8 = 0; j8 < 8; ++j8) {
          const uint4 mv = __ldg(mrow + j8);
          const __nv_bfloat16* mk = reinterpret_cast<const __nv_bfloat16*>(&mv);
#pragma unroll
          for (int t = 0; t < 8; ++t)
            if (!(__bfloat162float(mk[t]) > 0.0f)) g[8 * j8 + t] = 0.0f;
        }
#pragma unroll
        for (int j8 = 0; j8 < 8; ++j8) {
          uint4 o;
          o.x = pack2(g[8 * j8 + 0], g[8 * j8 + 1]);
          o.y = pack2(g[8 * j8 + 2], g[8 * j8 + 3]);
          o.z = pack2(g[8 * j8 + 4], g[8 * j8 + 5]);
          o.w = pack2(g[8 * j8 + 6], g[8 * j8 + 7]);
          *reinterpret_cast<uint4*>(wrow + ((j8 ^ (lane & 7)) << 4)) = o;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&a.d_c, buf + 2 * kChunk, c0, r0);
          tma_store_commit();
          tma_store_wait_read<0>();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(&tempty[acc], 0);
    });
    if (lane == 0) tma_store_wait<0>();
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm<512>(tmem_base);
  }
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("EDL_PDL");
    on = e ? atoi(e) != 0 : 1;
  }
  return on != 0;
}

}  // namespace

bool gemm_pair_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("EDL_BWD_PAIR");
    on = e ? atoi(e) != 0 : 0;
  }
  return on != 0;
}

bool gemm_pair_eligible(const GemmPlan& d, const GemmPlan& w) {
  return d.cg == 2 && d.bn == 128 && d.sk == 1 && !d.a_mn && d.b_mn && d.ep.mask &&
         !d.ep.out_f32 && !d.ep.relu && (d.mc == 1 || d.mc == 2) && d.M % 256 == 0 &&
         d.N % 128 == 0 && d.K % kBK == 0 && w.ep.sgd && !w.ep.xchg && !w.lo && w.cg == 2 &&
         w.bn == 128 && w.mc == 1 && w.a_mn && w.b_mn && w.M % 256 == 0 && w.N % 128 == 0 &&
         w.K % kBK == 0;
}

int gemm_pair_prepare_device(int* units_out) {
  static std::atomic<uint64_t> attr_set{0};
  static int max_units[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_set.load() >> dev & 1)) {
    EDL_CUDA_TRY(cudaFuncSetAttribute(bwd_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kSmemBytes));
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.gridDim = dim3((sm_count() / 2) * 2);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    EDL_CUDA_TRY(cudaOccupancyMaxActiveClusters(&n, bwd_pair_kernel, &cfg));
    max_units[dev] = n > 0 ? n : 1;
    attr_set.fetch_or(1ull << dev);
  }
  if (units_out) *units_out = max_units[dev];
  return EDL_OK;
}

int gemm_pair_run(const GemmPlan& d, const GemmPlan& w, cudaStream_t stream, float scale) {
  if (!gemm_pair_eligible(d, w)) return fail(EDL_EINVAL, "gemm pair: plan shapes");
  int max_units = 0;
  const int prc = gemm_pair_prepare_device(&max_units);
  if (prc != EDL_OK) return prc;
  int U = sm_count() / 2;
  if (U > max_units) U = max_units;
  if (U > kMaxUnits) U = kMaxUnits;
  PairArgs a;
  a.d_a = d.ta;
  a.d_b = d.tb;
  a.d_c = d.tc;
  a.w_a = w.ta;
  a.w_b = w.tb;
  a.w_m = w.tm;
  a.w_c = w.tc;
  a.mask = d.ep.mask;
  a.ldm = d.ep.ldm;
  a.d_mt = d.M / 256;
  a.d_nt = d.N / 128;
  a.d_kb = d.K / kBK;
  a.d_a_boxes = d.mc;
  a.w_mt = w.M / 256;
  a.w_nt = w.N / 128;
  a.w_kb = w.K / kBK;
  a.scale = scale;
  a.pf_kb = d.ep.pf_kb;
  // W tiles over the units: greedy to the least loaded unit, where a D tile costs
  // EDL_PAIR_DCOST W tiles (its MMAs overlap the W epilogues, so it is cheap), then
  // contiguous ranges (consecutive W tiles share dY rows: L2 locality of the A operand)
  static double dcost = -1;
  if (dcost < 0) {
    const char* e = getenv("EDL_PAIR_DCOST");
    dcost = e ? atof(e) : 1.0;
  }
  const int nD = a.d_mt * a.d_nt, nW = a.w_mt * a.w_nt;
  if (nW > 65535) return fail(EDL_EINVAL, "gemm pair: too many weight tiles");
  std::vector<double> load(U);
  std::vector<int> cnt(U, 0);
  for (int v = 0; v < U; ++v) load[v] = dcost * (v < nD ? (nD - 1 - v) / U + 1 : 0);
  for (int t = 0; t < nW; ++t) {
    int best = 0;
    for (int v = 1; v < U; ++v)
      if (load[v] < load[best] - 1e-9) best = v;
    load[best] += 1.0;
    ++cnt[best];
  }
  a.w_begin[0] = 0;
  for (int v = 0; v < U; ++v) a.w_begin[v + 1] = static_cast<uint16_t>(a.w_begin[v] + cnt[v]);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * U);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  EDL_CUDA_TRY(cudaLaunchKernelEx(&cfg, bwd_pair_kernel, a));
  return EDL_OK;
}

}  // namespace edl
