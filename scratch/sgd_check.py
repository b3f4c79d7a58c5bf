import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_1909_11985_b200 import _lib
L = _lib.lib()
def bf16r(x): return x.to(torch.bfloat16).float()
for (M, N, K) in [(256, 256, 64), (512, 384, 200), (4096, 4096, 512), (4096, 1024, 512)]:
    torch.manual_seed(0)
    dy = torch.randn(K, M).to(torch.bfloat16).cuda(); x = torch.randn(K, N).to(torch.bfloat16).cuda()
    master = (torch.randn(M, N) * 0.05).cuda(); W = master.to(torch.bfloat16)
    scale = 1e-3
    ref_g = bf16r(dy.float().t() @ x.float())
    ref_m = master - (scale * ref_g)
    m2 = master.clone()
    rc = L.edl_gemm_wgrad_sgd(dy.data_ptr(), M, x.data_ptr(), N, m2.data_ptr(), W.data_ptr(), N, M, N, K, scale, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    em = (m2 - ref_m).abs().max().item(); ew = (W.float() - bf16r(m2)).abs().max().item()
    dmax = (ref_m - master).abs().max().item()
    print(f"M={M} N={N} K={K} rc={rc} master err {em:.3e} (update max {dmax:.3e}) W-vs-master err {ew:.3e}", flush=True)
    # timing
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    for _ in range(3): L.edl_gemm_wgrad_sgd(dy.data_ptr(), M, x.data_ptr(), N, m2.data_ptr(), W.data_ptr(), N, M, N, K, scale, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): L.edl_gemm_wgrad_sgd(dy.data_ptr(), M, x.data_ptr(), N, m2.data_ptr(), W.data_ptr(), N, M, N, K, scale, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1)*1e3/20
    print(f"   {us:.1f} us  ({M*N*10/us/1e3:.0f} GB/s of master/W traffic, {2*M*N*K/us/1e6:.0f} TF/s)")
