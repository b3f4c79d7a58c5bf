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

#include <cstdint>
#include <cstdio>

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
  static constexpr int kStages = (200 * 1024) / kStageBytes > 8 ? 8 : (200 * 1024) / kStageBytes;
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

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t tx = C::kABytes + (B_MN ? C::kBBytesMN : C::kBBytesK);
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m0 = (tile % m_tiles) * BM;
        const int n0 = (tile / m_tiles) * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
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
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * C::kAccCols;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::kStageBytes);
          const uint32_t sb = sa + C::kABytes;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t da = A_MN ? smem_desc_sw128(sa + k * 2048, kMnBlockBytes, 1024)
                                     : smem_desc_sw128(sa + k * 32, 16, 1024);
            const uint64_t db = B_MN ? smem_desc_sw128(sb + k * 2048, kMnBlockBytes, 1024)
                                     : smem_desc_sw128(sb + k * 32, 16, 1024);
            umma_bf16(d_tmem, da, db, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(&empty_bar[stage]);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull_bar[acc]);
      }
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
            for (int j = 0; j < lim; ++j)
              if (!(__bfloat162float(mrow[j]) > 0.0f)) v[j] = 0.0f;
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
            for (int j = 0; j < lim; ++j) crow[j] = v[j];
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
            for (int j = 0; j < lim; ++j) crow[j] = __float2bfloat16_rn(v[j]);
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
int make_tmap(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
              uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return EDL_ECUDA;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? EDL_OK : EDL_ECUDA;
}

int num_sms() {
  static int n = 0;
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
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cf::kSmemBytes) != cudaSuccess)
      return EDL_ECUDA;
    attr_set = true;
  }
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  kern<<<grid, kThreads, Cf::kSmemBytes, stream>>>(ta, tb, M, N, K, ep);
  EDL_CUDA_TRY(cudaGetLastError());
  return EDL_OK;
}

}  // namespace

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

int gemm_plan_init(GemmPlan* p, const void* A, int lda, int a_mn, const void* B, int ldb,
                   int b_mn, void* Cout, int ldc, int M, int N, int K, int relu, int out_f32,
                   const void* mask, int ldm, int bn) {
  if (M <= 0 || N <= 0 || K <= 0) return fail(EDL_EINVAL, "gemm: empty shape");
  if ((lda * 2) % 16 || (ldb * 2) % 16) return fail(EDL_EINVAL, "gemm: 16-byte row alignment");
  if (bn <= 0) bn = gemm_pick_bn(M, N, b_mn != 0);
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
  p->ep = EpiParams{Cout, static_cast<const __nv_bfloat16*>(mask), ldc, ldm, relu, out_f32};
  return EDL_OK;
}

int gemm_plan_run(const GemmPlan& p, cudaStream_t stream) {
  const int a_mn = p.a_mn, b_mn = p.b_mn;
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
