// Internal declarations shared by the CUDA translation units and the C-ABI layer.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/edl_b200.h"

namespace edl {

// Thread-local last-error string surfaced through edl_last_error().
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define EDL_CUDA_TRY(expr)                                  \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return ::edl::cuda_fail(_e, #expr); \
  } while (0)

// ---- GEMM (gemm_sm100.cu)
constexpr int kMaxPeerMaps = 8;
struct EpiParams {
  void* C;                     // bf16 or fp32 output [M][ldc]
  const __nv_bfloat16* mask;   // optional: zero outputs where mask <= 0 ([M][ldm])
  int ldc;
  int ldm;
  int relu;     // apply max(0, x)
  int out_f32;  // store fp32 instead of bf16
  // fused SGD epilogue (weight-gradient GEMM): master[M][N] -= scale * bf16(acc);
  // C (bf16) <- master.  Set per launch by gemm_plan_run(plan, stream, scale).
  int sgd;
  float scale;
  // L2 prefetch distances (0 = off): operand k-blocks ahead in the producer; master tiles
  // ahead in the fused-SGD epilogue.  Defaults from gemm_prefetch_defaults().
  int pf_kb;
  int pf_tiles;
  int mask_pf;  // L2 prefetch of the ReLU' mask rows before the epilogue waits (dgrad)
  // reduce-scatter routing of a weight-gradient GEMM (N > 1): output rows are owned in
  // blocks of route_rows by replica row / route_rows; blocks owned by another replica are
  // stored through PeerMaps::m[owner] (that replica's receive slot for this one, over NVLink)
  int route_rows;
  int route_me;
  int dbg;  // trace builds only: 1 = skip the K loop, 2 = skip the epilogue work
  // L2 prefetch of an unrelated region while this (tensor-bound) GEMM runs: the producer of
  // every CTA pulls its 1/grid share of [l2pf, l2pf + l2pf_bytes) into L2 over its first
  // k-blocks (the dgrad GEMM of layer l prefetches layer l's fp32 master for the fused
  // wgrad + SGD kernel that follows: HBM is idle during the dgrad mainloop)
  const void* l2pf;
  size_t l2pf_bytes;
  // B operand (the layer's weights) all-gathered by the previous mini-batch's deferred push
  // collective: the producer waits until wait_flags[r] >= wait_epoch for r < wait_n (every
  // replica signalled this layer) before its first load.  nullptr: no wait.
  const uint32_t* wait_flags;
  int wait_n;
  uint32_t wait_epoch;
  // fused exchange (fused-SGD plan, N > 1, one ring member per GPU; gemm_plan_exchange):
  // tiles whose rows replica o != route_me owns are stored as bf16 into o's receive slot
  // (PeerMaps::m[o]); tiles this replica owns wait until every peer's chunk has replaced the
  // sentinel in its slot, sum the members' gradients in ring order (x_order: replica of ring
  // member k), update the fp32 master and store the bf16 weights into every replica
  // (PeerMaps::w[o]).  The reduce-scatter, the update and the all-gather of the weights all
  // happen inside the weight-gradient GEMM.
  int xchg;
  int x_n;
  const __nv_bfloat16* x_recv[kMaxPeerMaps];    // my receive slot of source replica r ([prow][ldr])
  int x_ldr;
  int x_order[kMaxPeerMaps];
};
struct PeerMaps {
  CUtensorMap m[kMaxPeerMaps];  // routed plans: replica o's receive slot for this replica
  CUtensorMap w[kMaxPeerMaps];  // fused-exchange plans: replica o's bf16 weights of the layer
};
// Pre-encoded launch (TMA descriptors built once; launching costs one kernel launch).
struct GemmPlan {
  CUtensorMap ta, tb, tc, tm;  // tm: fp32 master (fused-SGD plans)
  PeerMaps pm;                 // reduce-scatter destinations (routed plans)
  int M = 0, N = 0, K = 0, a_mn = 0, b_mn = 0, bn = 0, cg = 1;
  int mc = 1;  // CTA-pair kernel: pairs per cluster sharing A by TMA multicast (1 or 2)
  int sk = 1;  // CTA-pair kernel: 2 = split-K over two pairs, 256-wide tiles (gemm_sm100.cu)
  // fused-SGD plan over the split master (tm: the 16-bit low halves, pm.m[0]: the fp32
  // master): 1 = split in / out, 2 = split in, fp32 out, 3 = fp32 in, split out
  int lo = 0;
  bool lo_master = false;  // pm.m[0] is set (modes 2 and 3 allowed)
  EpiParams ep{};
};
int gemm_plan_init(GemmPlan* p, const void* A, int lda, int a_mn, const void* B, int ldb,
                   int b_mn, void* C, int ldc, int M, int N, int K, int relu, int out_f32,
                   const void* mask, int ldm, int bn);
int gemm_plan_run(const GemmPlan& p, cudaStream_t stream, float sgd_scale = 0.f);
int gemm_prepare_device();  // current device: load + configure the step's GEMM variants
// gemm_plan_run whose producer first waits for n per-replica flags >= epoch (system-scope
// acquire; the deferred all-gather's "layer l is in your W" signals, collective.hpp)
int gemm_plan_run_wait(const GemmPlan& p, cudaStream_t stream, const uint32_t* flags, int n,
                       uint32_t epoch);
// Weight-gradient GEMM with the SGD step fused into its epilogue (CTA-pair kernel, one
// replica): dW = A^T-major x B^T-major as for wgrad, then master -= scale * bf16(dW) and
// W (bf16) <- master, with no gradient buffer round trip through HBM.
int gemm_plan_init_sgd(GemmPlan* p, const void* A, int lda, int a_mn, const void* B, int ldb,
                       int b_mn, float* master, __nv_bfloat16* W, int ldw, int M, int N, int K);
// The same over the split master: the fp32 master m is kept as its bf16 rounding W (the
// weights the GEMMs read) plus the low 16 bits of m (lo): 8 B per parameter per update
// instead of 10 (gemm_sm100.cu; master_split_lo / master_join_lo convert).
int gemm_plan_init_sgd_lo(GemmPlan* p, const void* A, int lda, const void* B, int ldb,
                          uint16_t* lo, __nv_bfloat16* W, float* master, int ldw, int M, int N,
                          int K);
int gemm_pick_bn(int M, int N, bool b_mn);
// Backward pair (bwd_pair.cu): the dgrad plan of layer l-1 (CTA pair, N tile 128, relu'
// mask, bf16 out) and the fused wgrad + SGD plan of layer l in one persistent launch.
bool gemm_pair_enabled();  // EDL_BWD_PAIR (default 0: measured no faster)
bool gemm_pair_eligible(const GemmPlan& dgrad, const GemmPlan& wgrad_sgd);
int gemm_pair_run(const GemmPlan& dgrad, const GemmPlan& wgrad_sgd, cudaStream_t stream,
                  float scale);
int gemm_pair_prepare_device(int* units_out);
// Fused wgrad + SGD with the B panel resident in shared memory (wgrad_sgd.cu): used by
// gemm_plan_run for fused-SGD plans with K <= 512 when EDL_SGD_BRES=1 (measured slower).
bool wgrad_sgd_bres_eligible(const GemmPlan& p);
int wgrad_sgd_bres_run(const GemmPlan& p, cudaStream_t stream, float scale);
int wgrad_sgd_bres_prepare_device(int* units_out);
// Turns a bf16-output CTA-pair plan into a reduce-scatter producer: rows owned by replica o
// (blocks of rows_per_owner) go to dst[o] ([rows_per_owner][N], ld = N), o != me.
int gemm_plan_route(GemmPlan* p, int rows_per_owner, int me, void* const* dst, int n_owner);
// Turns a fused-SGD plan into the fused exchange (EpiParams::xchg): recv_dst[o] = replica o's
// receive slot for this replica (layer-relative rows), w_dst[o] = replica o's weights of the
// layer, recv_src[r] = this replica's receive slot of source r (ld_recv; filled with 0xFF
// bytes before the first mini-batch), order[k] = replica of ring member k.
int gemm_plan_exchange(GemmPlan* p, int rows_per_owner, int me, int n, void* const* recv_dst,
                       __nv_bfloat16* const* w_dst, const __nv_bfloat16* const* recv_src,
                       int ld_recv, const int* order);
int gemm_bf16(const void* A, int lda, int a_mn, const void* B, int ldb, int b_mn, void* C,
              int ldc, int M, int N, int K, int relu, int out_f32, const void* mask, int ldm,
              int bn, cudaStream_t stream);

}  // namespace edl
