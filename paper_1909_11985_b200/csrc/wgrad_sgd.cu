// Weight-gradient GEMM + fused SGD update with the B operand resident in shared memory
// (N = 1 fused-update path, the dominant kernel of the step):
//
//   dW = dY^T . X      dY [b][out] (A, MN-major), X = act[l] [b][in] (B, MN-major), K = b
//   master -= scale * bf16(dW);   W = bf16(master)        (trainer.cpp:56-61, sgd_step)
//
// Why a second kernel: K (the mini-batch, 512) is short, so every 256 x 128 output tile of
// the general CTA-pair kernel (gemm_sm100.cu) re-streams its whole A and B panels from L2 --
// 12 bytes of operands per parameter next to the 4-byte master read, and that L2 -> SM
// stream (~8 TB/s, ncu) is what bounded it, not HBM.  Here each CTA pair walks its tiles
// column-block by column-block and keeps the B panel of the current column block (its 64
// columns x K, 64 KB per CTA at K = 512) in shared memory, loading it once per column block;
// only A (16 KB per k-block) streams through a 4-stage ring.  Operand bytes per parameter
// drop from 12 to ~8, and the kernel moves toward its HBM roofline (10 B/param).
//
// Measured on B200 (profiles/r02_wgrad_sgd.md): parity-green but slower than the general
// kernel (45.3 vs 42.9 us per layer): fewer L2 -> SM bytes did not help because the fused
// epilogue, not the operand stream, bounds this kernel (in-kernel trace of the general one:
// per epilogue warp 6.6 us waiting for master loads, 3.4 us for TMA store reads, 3.3 us of
// TMEM reads at 64 B/clk, 4.6 us of smem read-modify-write, 6.8 us waiting for the MMA).
// Opt-in: EDL_SGD_BRES=1.
//
// Roles per CTA (cta_group::2, 320 threads): warp 0 TMA producer, warp 1 MMA issuer (pair
// leader), warps 2-9 epilogue (two per TMEM lane quarter, 64 columns each).  TMEM holds a
// ring of four 128-column fp32 accumulators.  The epilogue is the fused-SGD epilogue of the
// general kernel: master chunk TMA-loaded into swizzled smem (prefetched a tile ahead),
// updated in place, TMA-stored with the bf16 weights.  Numerics identical to it.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "edl_internal.hpp"
#include "sm100.cuh"

namespace edl {
namespace {

using namespace sm100;

constexpr int kBK = 64;
constexpr int kMaxKb = 8;                      // K <= 512: the resident panel is <= 64 KB
constexpr uint32_t kBox = 64 * kBK * 2;        // 64 x 64 bf16 box (8 KB)
constexpr uint32_t kAStage = 2 * kBox;         // A: 128 rows (two 64-wide boxes) x 64 K
constexpr int kAStages = 4;
constexpr uint32_t kPanel = kMaxKb * kBox;     // B: 64 columns x K
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr uint32_t kChunk = 32 * 128;
constexpr uint32_t kBuf = 3 * kChunk;          // master 2 x 4 KB + W 4 KB per epilogue warp
constexpr uint32_t kEpiBytes = kEpiWarps * kBuf;
constexpr int kAcc = 4;                        // TMEM ring: 4 x 128 fp32 columns
constexpr uint32_t kSmemBytes = kAStages * kAStage + kPanel + kEpiBytes + 1024 + 512;

struct WgradArgs {
  CUtensorMap ta, tb, tm, tc;  // dY (MN-major), X (MN-major), master fp32, W bf16
  int mt, nt, nkb;             // M / 256, N / 128, K / 64
  float scale;
  int pf;                      // L2 prefetch of the next tile's A (0 = off)
};

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

__global__ void __launch_bounds__(kThreads, 1)
    wgrad_sgd_bres_kernel(const __grid_constant__ WgradArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* panel = smem + kAStages * kAStage;
  uint8_t* epi = panel + kPanel;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(epi + kEpiBytes);
  uint64_t* empty_bar = full_bar + kAStages;
  uint64_t* bfull = empty_bar + kAStages;  // the B panel of the current column block landed
  uint64_t* bfree = bfull + 1;             // the MMAs reading the previous panel completed
  uint64_t* tfull = bfree + 1;
  uint64_t* tempty = tfull + kAcc;
  uint64_t* mbar = tempty + kAcc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + kEpiWarps);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t pr = cluster_ctarank() & 1;
  const bool leader = pr == 0;
  const int u = blockIdx.x / 2, U = gridDim.x / 2;
  // tiles in column-block-major order (consecutive tiles share the B panel); unit u owns
  // the contiguous range [t0, t1)
  const int n_tiles = a.mt * a.nt;
  const int t0 = static_cast<int>(static_cast<long long>(u) * n_tiles / U);
  const int t1 = static_cast<int>(static_cast<long long>(u + 1) * n_tiles / U);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&a.ta);
    prefetch_tmap(&a.tb);
    prefetch_tmap(&a.tm);
    prefetch_tmap(&a.tc);
    for (int s = 0; s < kAStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(bfull, 1);
    mbar_init(bfree, 1);
    for (int i = 0; i < kAcc; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * kEpiWarps);
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
    int prev_n = -1, panels = 0;
    for (int t = t0; t < t1; ++t) {
      const int tn = t / a.mt, tm = t % a.mt;
      const int m0 = tm * 256 + static_cast<int>(pr) * 128;
      if (tn != prev_n) {
        // refill the panel once the MMAs of the previous column block are done with it
        if (panels > 0) mbar_wait(bfree, static_cast<uint32_t>((panels - 1) & 1));
        if (elect_one()) {
          const int n0 = tn * 128 + static_cast<int>(pr) * 64;
          if (leader) mbar_arrive_expect_tx(bfull, 2 * a.nkb * kBox);
          for (int kb = 0; kb < a.nkb; ++kb)
            tma_load_2d_2sm(panel + kb * kBox, &a.tb, bfull, n0, kb * kBK);
        }
        __syncwarp();
        prev_n = tn;
        ++panels;
      }
      for (int kb = 0; kb < a.nkb; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (elect_one()) {
          uint8_t* sa = smem + stage * kAStage;
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * kAStage);
          tma_load_2d_2sm(sa, &a.ta, &full_bar[stage], m0, kb * kBK);
          tma_load_2d_2sm(sa + kBox, &a.ta, &full_bar[stage], m0 + 64, kb * kBK);
          if (a.pf && t + 1 < t1) {  // the next tile's A k-block into L2
            const int m1 = ((t + 1) % a.mt) * 256 + static_cast<int>(pr) * 128;
            tma_prefetch_2d(&a.ta, m1, kb * kBK);
            tma_prefetch_2d(&a.ta, m1 + 64, kb * kBK);
          }
        }
        __syncwarp();
        if (++stage == kAStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------------------------ MMA issuer (pair leader)
      constexpr uint32_t idesc = idesc_bf16_f32(256, 128, true, true);
      const uint64_t a0 = smem_desc_sw128(smem_u32(smem), kBox, 1024);
      const uint64_t b0 = smem_desc_sw128(smem_u32(panel), kBox, 1024);
      int stage = 0;
      uint32_t phase = 0;
      int prev_n = -1, panels = 0;
      const bool issuer = elect_one();
      for (int t = t0, i = 0; t < t1; ++t, ++i) {
        const int tn = t / a.mt;
        if (tn != prev_n) {
          if (panels > 0) {  // every MMA on the old panel issued: release it when they finish
            if (issuer) umma_commit_2sm(bfree, 0x3);
            __syncwarp();
          }
          mbar_wait(bfull, static_cast<uint32_t>(panels & 1));
          tc_fence_after();
          prev_n = tn;
          ++panels;
        }
        const int acc = i % kAcc;
        mbar_wait(&tempty[acc], static_cast<uint32_t>(((i / kAcc) & 1) ^ 1));
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc) * 128;
        for (int kb = 0; kb < a.nkb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t so = static_cast<uint64_t>(stage * kAStage) >> 4;
          const uint64_t bo = static_cast<uint64_t>(kb * kBox) >> 4;
          if (issuer) {
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              umma_bf16_2sm(d_tmem, a0 + so + ((k * 2048) >> 4), b0 + bo + ((k * 2048) >> 4),
                            idesc, (kb | k) != 0 ? 1u : 0u);
            umma_commit_2sm(&empty_bar[stage], 0x3);
          }
          __syncwarp();
          if (++stage == kAStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (issuer) umma_commit_2sm(&tfull[acc], 0x3);
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ fused SGD epilogue
    const int q = warp & 3;
    const int ew = warp - 2;
    const int half = ew / 4;
    uint8_t* buf = epi + ew * kBuf;
    uint8_t* wrow = buf + 2 * kChunk + lane * 128;
    uint64_t* mb = &mbar[ew];
    auto coords = [&](int t, int* r0, int* c0) {
      *r0 = (t % a.mt) * 256 + static_cast<int>(pr) * 128 + q * 32;
      *c0 = (t / a.mt) * 128 + half * 64;
    };
    auto prefetch = [&](int t) {  // this warp's master chunk of tile t
      if (t >= t1) return;
      int r0, c0;
      coords(t, &r0, &c0);
      mbar_arrive_expect_tx(mb, 2 * kChunk);
      tma_load_2d(buf, &a.tm, mb, c0, r0);
      tma_load_2d(buf + kChunk, &a.tm, mb, c0 + 32, r0);
    };
    if (lane == 0) prefetch(t0);
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
      const int acc = i % kAcc;
      mbar_wait(&tfull[acc], static_cast<uint32_t>((i / kAcc) & 1));
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
      // the accumulator is in registers: hand it back to the MMA before the HBM part
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(&tempty[acc], 0);
      // same numerics as the unfused path: the gradient is rounded to bf16 first
#pragma unroll
      for (int e = 0; e < 64; ++e) g[e] = __bfloat162float(__float2bfloat16_rn(g[e]));
      mbar_wait(mb, static_cast<uint32_t>(i & 1));
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
        coords(t, &r0, &c0);
        tma_store_2d(&a.tm, buf, c0, r0);
        tma_store_2d(&a.tm, buf + kChunk, c0 + 32, r0);
        tma_store_2d(&a.tc, buf + 2 * kChunk, c0, r0);
        tma_store_commit();
        tma_store_wait_read<0>();  // refill the buffer with the next tile's master
        prefetch(t + 1);
      }
      __syncwarp();
    }
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

}  // namespace

bool wgrad_sgd_bres_eligible(const GemmPlan& p) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("EDL_SGD_BRES");
    on = e ? atoi(e) != 0 : 0;
  }
  return on && p.ep.sgd && !p.ep.xchg && !p.lo && p.cg == 2 && p.bn == 128 && p.mc == 1 && p.a_mn &&
         p.b_mn && p.M % 256 == 0 && p.N % 128 == 0 && p.K % kBK == 0 && p.K <= kMaxKb * kBK;
}

int wgrad_sgd_bres_prepare_device(int* units_out) {
  static std::atomic<uint64_t> attr_set{0};
  static int max_units[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_set.load() >> dev & 1)) {
    EDL_CUDA_TRY(cudaFuncSetAttribute(wgrad_sgd_bres_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
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
    EDL_CUDA_TRY(cudaOccupancyMaxActiveClusters(&n, wgrad_sgd_bres_kernel, &cfg));
    max_units[dev] = n > 0 ? n : 1;
    attr_set.fetch_or(1ull << dev);
  }
  if (units_out) *units_out = max_units[dev];
  return EDL_OK;
}

int wgrad_sgd_bres_run(const GemmPlan& p, cudaStream_t stream, float scale) {
  if (!wgrad_sgd_bres_eligible(p)) return fail(EDL_EINVAL, "wgrad sgd: plan shape");
  int max_units = 0;
  const int rc = wgrad_sgd_bres_prepare_device(&max_units);
  if (rc != EDL_OK) return rc;
  WgradArgs a;
  a.ta = p.ta;
  a.tb = p.tb;
  a.tm = p.tm;
  a.tc = p.tc;
  a.mt = p.M / 256;
  a.nt = p.N / 128;
  a.nkb = p.K / kBK;
  a.scale = scale;
  a.pf = p.ep.pf_kb > 0 ? 1 : 0;
  int U = sm_count() / 2;
  if (U > max_units) U = max_units;
  if (U > a.mt * a.nt) U = a.mt * a.nt;
  static int pdl = -1;
  if (pdl < 0) {
    const char* e = getenv("EDL_PDL");
    pdl = e ? atoi(e) != 0 : 1;
  }
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
  cfg.numAttrs = pdl ? 2 : 1;
  EDL_CUDA_TRY(cudaLaunchKernelEx(&cfg, wgrad_sgd_bres_kernel, a));
  return EDL_OK;
}

}  // namespace edl
