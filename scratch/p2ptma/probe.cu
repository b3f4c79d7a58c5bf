// Probe: can a TMA bulk-tensor store / load target a peer GPU's memory (peer access enabled)?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void store_kernel(const __grid_constant__ CUtensorMap tm, int rows) {
  __shared__ alignas(1024) float buf[32 * 32];
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) buf[i] = 1000.f * blockIdx.x + i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tm),
                 "r"((uint32_t)__cvta_generic_to_shared(buf)), "r"(0), "r"((int)blockIdx.x * 32) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
int main() {
  int n = 0; cudaGetDeviceCount(&n);
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  int can = 0; cudaDeviceCanAccessPeer(&can, 0, 1);
  printf("can access peer 0->1: %d\n", can);
  cudaSetDevice(1);
  float* peer = nullptr; const int rows = 32 * 64, cols = 32;
  cudaMalloc(&peer, rows * cols * 4); cudaMemset(peer, 0, rows * cols * 4);
  cudaSetDevice(0);
  cudaDeviceEnablePeerAccess(1, 0);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p;
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}; cuuint64_t str[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, peer, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode on peer pointer: %d\n", (int)r);
  store_kernel<<<64, 128>>>(tm, rows);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> h(rows * cols);
  cudaSetDevice(1);
  cudaMemcpy(h.data(), peer, rows * cols * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int b = 0; b < 64; ++b) for (int i = 0; i < 1024; ++i) if (h[b * 1024 + i] != 1000.f * b + i) ++bad;
  printf("TMA store to peer memory: %s (%d mismatches)\n", bad ? "FAIL" : "OK", bad);
  return 0;
}
