import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_1909_11985_b200 import _lib
L = _lib.lib()
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
def run(a_mn, b_mn, M, N, K, bn, f32=0, mask=False, relu=0, t=True):
    torch.manual_seed(0)
    A = (torch.randn(K, M) if a_mn else torch.randn(M, K)).to(torch.bfloat16).cuda()
    B = (torch.randn(K, N) if b_mn else torch.randn(N, K)).to(torch.bfloat16).cuda()
    out = torch.zeros(M, N, dtype=torch.float32 if f32 else torch.bfloat16, device='cuda')
    mk = torch.randn(M, N).to(torch.bfloat16).cuda() if mask else None
    args = (A.data_ptr(), A.shape[1], a_mn, B.data_ptr(), B.shape[1], b_mn, out.data_ptr(), N, M, N, K, relu, f32, mk.data_ptr() if mask else None, N if mask else 0, bn)
    rc = L.edl_gemm_bf16(*args, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    a = A.float().t() if a_mn else A.float(); b = B.float() if b_mn else B.float().t()
    ref = a @ b
    if relu: ref = torch.relu(ref)
    if mask: ref = ref * (mk.float() > 0)
    err = (out.float() - ref).abs().max().item(); scale = ref.abs().max().item()
    ok = err <= (1e-3 if f32 else 1e-2) * scale + 1e-2
    us = timed(lambda: L.edl_gemm_bf16(*args, C.c_void_p(torch.cuda.current_stream().cuda_stream))) if t else 0
    print(f"{'OK ' if ok and rc==0 else 'BAD'} a{a_mn}b{b_mn} M={M} N={N} K={K} bn={bn} f32={f32} mask={mask} rc={rc} err={err:.2e}/{scale:.1e} {us:.1f} us {2*M*N*K/max(us,1e-9)/1e6:.0f} TF/s", flush=True)
    if not ok:
        bad = ((out.float()-ref).abs() > 1e-2*scale).nonzero()
        print("   nbad", bad.shape[0], bad[:6].tolist())
for combo in [(0,0),(0,1),(1,0),(1,1)]:
    run(*combo, 256, 256, 128, 1128, t=False)
    run(*combo, 512, 512, 256, 1256, t=False)
    run(*combo, 384, 320, 200, 1192, t=False)
run(0, 0, 512, 1024, 512, 1128, f32=1, t=False)
run(0, 1, 512, 1024, 512, 1128, mask=True, t=False)
run(0, 0, 512, 1024, 512, 1256, relu=1, t=False)
for bn in (1128, 1192, 1256, 0):
    run(0, 0, 512, 4096, 4096, bn)
    run(0, 1, 512, 4096, 4096, bn)
    run(1, 1, 4096, 4096, 512, bn)
run(0, 0, 512, 4096, 4096, 1128, f32=1)
run(0, 1, 512, 4096, 4096, 1128, mask=True)
