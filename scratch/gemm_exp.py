import ctypes as C, sys, os, torch
sys.path.insert(0, '.')
from paper_1909_11985_b200 import _lib
L = _lib.lib()
tag = os.environ.get("EDL_LIB_PATH", "default")
def timed(fn, it=40):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(it): fn()
    g.replay(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / it
def bench(a_mn, b_mn, M, N, K, bn):
    A = (torch.randn(K, M) if a_mn else torch.randn(M, K)).to(torch.bfloat16).cuda()
    B = (torch.randn(K, N) if b_mn else torch.randn(N, K)).to(torch.bfloat16).cuda()
    out = torch.empty(M, N, dtype=torch.bfloat16, device='cuda')
    args = (A.data_ptr(), A.shape[1], a_mn, B.data_ptr(), B.shape[1], b_mn, out.data_ptr(), N, M, N, K, 0, 0, None, 0, bn)
    us = timed(lambda: L.edl_gemm_bf16(*args, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    tiles = ((M+127)//128)*((N+bn-1)//bn); ctas = min(tiles, 148)
    mac_clk = M*N*K/(us*1e-6)/ctas/1.965e9
    print(f"[{tag[-24:]}] a{a_mn}b{b_mn} M={M} N={N} K={K} bn={bn} ctas={ctas}: {us:.1f} us {2*M*N*K/us/1e6:.0f} TF/s  per-SM {mac_clk:.0f} MAC/clk ({100*mac_clk/4096:.0f}%)", flush=True)
for bn in (128, 256):
    bench(0, 0, 512, 4096, 4096, bn)
    bench(0, 0, 1024, 4096, 4096, bn)
    bench(0, 0, 512, 4096, 16384, bn)
bench(0, 0, 2048, 4096, 4096, 256)
bench(1, 1, 4096, 4096, 512, 256)
bench(1, 1, 4096, 4096, 2048, 256)
