// Error plumbing for the C ABI: reference exceptions become EDL_E* codes plus a
// thread-local message (see include/edl_b200.h).
#include <cuda_runtime.h>

#include <string>

#include "edl_internal.hpp"

namespace edl {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? EDL_ENOMEM : EDL_ECUDA;
}

}  // namespace edl

extern "C" {

const char* edl_last_error(void) { return edl::g_last_error.c_str(); }

const char* edl_version(void) { return "edl-b200 0.1 (sm_100a)"; }

int edl_gemm_bf16(const void* A, int32_t lda, int32_t a_mn, const void* B, int32_t ldb,
                  int32_t b_mn, void* C, int32_t ldc, int32_t M, int32_t N, int32_t K,
                  int32_t relu, int32_t out_f32, const void* mask, int32_t ldm, int32_t bn,
                  void* stream) {
  int rc = edl::gemm_bf16(A, lda, a_mn, B, ldb, b_mn, C, ldc, M, N, K, relu, out_f32, mask, ldm,
                          bn, static_cast<cudaStream_t>(stream));
  if (rc != EDL_OK && edl_last_error()[0] == 0) edl::set_error("edl_gemm_bf16 failed");
  return rc;
}

}  // extern "C"

extern "C" int edl_gemm_wgrad_sgd(const void* dy, int32_t ld_dy, const void* x, int32_t ld_x,
                                  float* master, void* W, int32_t ldw, int32_t M, int32_t N,
                                  int32_t K, float scale, void* stream) {
  edl::GemmPlan p;
  int rc = edl::gemm_plan_init_sgd(&p, dy, ld_dy, 1, x, ld_x, 1, master,
                                   static_cast<__nv_bfloat16*>(W), ldw, M, N, K);
  if (rc) return rc;
  return edl::gemm_plan_run(p, static_cast<cudaStream_t>(stream), scale);
}

extern "C" int edl_gemm_wgrad_sgd_split(const void* dy, int32_t ld_dy, const void* x,
                                        int32_t ld_x, uint16_t* lo, void* W, float* master,
                                        int32_t mode, int32_t ldw, int32_t M, int32_t N,
                                        int32_t K, float scale, void* stream) {
  if (mode < 1 || mode > 3 || (mode != 1 && !master))
    return edl::fail(EDL_EINVAL, "split-master SGD: mode 1..3 (2 and 3 need the fp32 master)");
  edl::GemmPlan p;
  int rc = edl::gemm_plan_init_sgd_lo(&p, dy, ld_dy, x, ld_x, lo, static_cast<__nv_bfloat16*>(W),
                                      master, ldw, M, N, K);
  if (rc) return rc;
  p.lo = mode;
  return edl::gemm_plan_run(p, static_cast<cudaStream_t>(stream), scale);
}
