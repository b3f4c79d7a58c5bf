#include <cuda_bf16.h>
#include <cstdint>
extern "C" __global__ void ld_reduce_bf16(const void* mc, float* out, size_t n16) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x) {
    uint32_t r0, r1, r2, r3;
    const char* p = static_cast<const char*>(mc) + 16 * i;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "l"(p) : "memory");
    uint32_t r[4] = {r0, r1, r2, r3};
    for (int k = 0; k < 4; ++k) {
      __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&r[k]);
      float2 f = __bfloat1622float2(h);
      out[8 * i + 2 * k] = f.x;
      out[8 * i + 2 * k + 1] = f.y;
    }
  }
}
extern "C" __global__ void mc_store_bf16(void* mc, const uint4* src, size_t n16) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x) {
    uint4 v = src[i];
    char* p = static_cast<char*>(mc) + 16 * i;
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(p),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  }
}
extern "C" int launch_ld_reduce(const void* mc, float* out, size_t n16, void* s) {
  ld_reduce_bf16<<<148, 256, 0, (cudaStream_t)s>>>(mc, out, n16);
  return (int)cudaGetLastError();
}
extern "C" int launch_mc_store(void* mc, const void* src, size_t n16, void* s) {
  mc_store_bf16<<<148, 256, 0, (cudaStream_t)s>>>(mc, (const uint4*)src, n16);
  return (int)cudaGetLastError();
}
