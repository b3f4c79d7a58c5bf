import ctypes as C, sys, time
import torch
sys.path.insert(0, '.')
from paper_1909_11985_b200 import _lib
L = _lib.lib()
def run(a_mn, b_mn, M, N, K, bn=0):
    torch.manual_seed(0)
    A = (torch.randn(K, M) if a_mn else torch.randn(M, K)).to(torch.bfloat16).cuda()
    B = (torch.randn(K, N) if b_mn else torch.randn(N, K)).to(torch.bfloat16).cuda()
    out = torch.zeros(M, N, dtype=torch.float32, device='cuda')
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    rc = L.edl_gemm_bf16(A.data_ptr(), A.shape[1], a_mn, B.data_ptr(), B.shape[1], b_mn, out.data_ptr(), N, M, N, K, 0, 1, None, 0, bn, s)
    torch.cuda.synchronize()
    a = A.float().t() if a_mn else A.float(); b = B.float() if b_mn else B.float().t()
    ref = a @ b
    err = (out-ref).abs().max().item()
    print(f"a_mn={a_mn} b_mn={b_mn} M={M} N={N} K={K} bn={bn} rc={rc} maxerr={err:.3e} refmax={ref.abs().max().item():.3e}", flush=True)
    if err > 1e-2:
        print("  out[0,:8]", out[0,:8].tolist()); print("  ref[0,:8]", ref[0,:8].tolist())
        bad = ((out-ref).abs() > 1e-2).nonzero()
        print("  nbad", bad.shape[0], "first", bad[:8].tolist())
    # timing bf16 out
    outb = torch.empty(M, N, dtype=torch.bfloat16, device='cuda')
    for _ in range(3):
        L.edl_gemm_bf16(A.data_ptr(), A.shape[1], a_mn, B.data_ptr(), B.shape[1], b_mn, outb.data_ptr(), N, M, N, K, 0, 0, None, 0, bn, s)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    it = 20
    for _ in range(it):
        L.edl_gemm_bf16(A.data_ptr(), A.shape[1], a_mn, B.data_ptr(), B.shape[1], b_mn, outb.data_ptr(), N, M, N, K, 0, 0, None, 0, bn, s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)/it
    print(f"  {ms*1e3:.1f} us  {2*M*N*K/ms/1e9:.1f} TFLOP/s", flush=True)
    return err
for combo in [(0,0),(0,1),(1,0),(1,1)]:
    run(*combo, 128, 128, 64, 128)
for combo in [(0,0),(0,1),(1,0),(1,1)]:
    run(*combo, 512, 4096, 4096)
    run(*combo, 4096, 4096, 512)
for bn in [64, 96, 112, 128, 160, 192, 224, 256]:
    run(0, 0, 512, 4096, 4096, bn)
    run(0, 1, 512, 4096, 4096, bn)
# torch reference speed
A = torch.randn(512, 4096, dtype=torch.bfloat16, device='cuda'); B = torch.randn(4096, 4096, dtype=torch.bfloat16, device='cuda')
for _ in range(3): A @ B.t()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): A @ B.t()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)/20
print(f"cuBLAS 512x4096x4096: {ms*1e3:.1f} us {2*512*4096*4096/ms/1e9:.1f} TFLOP/s")
