// NVLink P2P bandwidth of SM-driven reads vs writes (both GPUs at once, 2 GPUs, one process).
#include <cuda_runtime.h>
#include <cstdio>
#include <thread>
__global__ void rd(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  size_t s = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += 4 * s) {
    uint4 a = __ldcs(src + i), b = i + s < n ? __ldcs(src + i + s) : uint4{}, c = i + 2 * s < n ? __ldcs(src + i + 2 * s) : uint4{},
          d = i + 3 * s < n ? __ldcs(src + i + 3 * s) : uint4{};
    dst[i] = a; if (i + s < n) dst[i + s] = b; if (i + 2 * s < n) dst[i + 2 * s] = c; if (i + 3 * s < n) dst[i + 3 * s] = d;
  }
}
int main() {
  const size_t bytes = 256ull << 20, n = bytes / 16;
  uint4 *a[2], *b[2];
  for (int d = 0; d < 2; ++d) { cudaSetDevice(d); cudaDeviceEnablePeerAccess(1 - d, 0); cudaMalloc(&a[d], bytes); cudaMalloc(&b[d], bytes); cudaMemset(a[d], 1, bytes); }
  for (int mode = 0; mode < 2; ++mode) for (int blocks : {592, 1184, 2368}) {
    float ms[2];
    auto run = [&](int d) {
      cudaSetDevice(d); cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      // mode 0: pull (read peer a, write local b); mode 1: push (read local a, write peer b)
      const uint4* src = mode == 0 ? a[1 - d] : a[d]; uint4* dst = mode == 0 ? b[d] : b[1 - d];
      for (int it = 0; it < 2; ++it) rd<<<blocks, 256>>>(src, dst, n);
      cudaDeviceSynchronize();
      cudaEventRecord(e0); for (int it = 0; it < 5; ++it) rd<<<blocks, 256>>>(src, dst, n); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms[d], e0, e1);
    };
    std::thread t0(run, 0), t1(run, 1); t0.join(); t1.join();
    printf("%s blocks=%d: GPU0 %.0f GB/s, GPU1 %.0f GB/s per direction\n", mode ? "push (st peer)" : "pull (ld peer)", blocks,
           5 * bytes / (ms[0] * 1e6), 5 * bytes / (ms[1] * 1e6));
  }
  return 0;
}
