# GEMM timing via CUDA graphs (no host encode/launch cost in the measurement)
import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_1909_11985_b200 import _lib
L = _lib.lib()
def timed(fn, it=50):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(it): fn()
    g.replay(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / it
def bench(a_mn, b_mn, M, N, K, bn=0):
    A = (torch.randn(K, M) if a_mn else torch.randn(M, K)).to(torch.bfloat16).cuda()
    B = (torch.randn(K, N) if b_mn else torch.randn(N, K)).to(torch.bfloat16).cuda()
    out = torch.empty(M, N, dtype=torch.bfloat16, device='cuda')
    args = (A.data_ptr(), A.shape[1], a_mn, B.data_ptr(), B.shape[1], b_mn, out.data_ptr(), N, M, N, K, 0, 0, None, 0, bn)
    us = timed(lambda: L.edl_gemm_bf16(*args, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    print(f"a_mn={a_mn} b_mn={b_mn} M={M} N={N} K={K} bn={bn}: {us:.1f} us {2*M*N*K/us/1e6:.0f} TFLOP/s", flush=True)
for bn in [0, 112, 128, 192, 256]:
    bench(0, 0, 512, 4096, 4096, bn)
    bench(0, 1, 512, 4096, 4096, bn)
    bench(1, 1, 4096, 4096, 512, bn)
A = torch.randn(512, 4096, dtype=torch.bfloat16, device='cuda'); B = torch.randn(4096, 4096, dtype=torch.bfloat16, device='cuda')
us = timed(lambda: A @ B.t()); print(f"cuBLAS fwd 512x4096x4096: {us:.1f} us {2*512*4096*4096/us/1e6:.0f} TFLOP/s")
us = timed(lambda: A @ B); print(f"cuBLAS dgrad 512x4096x4096: {us:.1f} us {2*512*4096*4096/us/1e6:.0f} TFLOP/s")
us = timed(lambda: A.t() @ A); print(f"cuBLAS wgrad 4096x4096x512: {us:.1f} us {2*512*4096*4096/us/1e6:.0f} TFLOP/s")
