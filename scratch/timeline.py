import ctypes as C, sys, os, torch, numpy as np
sys.path.insert(0, '.')
os.environ["EDL_LIB_PATH"] = os.path.abspath(sys.argv[1])
from paper_1909_11985_b200 import _lib
L = _lib.lib()
L.edl_debug_gemm_timeline.argtypes = [C.c_void_p]
tl = np.zeros((296, 16), dtype=np.uint64)
s = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)
names = ["entry", "setup_done", "mma_first_full", "mma_end", "epi_first_tfull", "epi_drained", "prod_end", "exit", "xready_seen", "w2_chunk0_store", "w2_chunk1_store", "w2_before_wait", "w5_drained", "w0_final", "w1_final", "xfull_seen"]
def show(tag, ctas):
    tl[:] = 0
    L.edl_debug_gemm_timeline(tl.ctypes.data)
    t = tl[:ctas].astype(np.int64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    print(f"{tag}: ctas={ctas}")
    for i, n in enumerate(names):
        col = rel[:, i][t[:, i] > 0]
        if len(col):
            print(f"   {n:16s} min {col.min():7.2f}  med {np.median(col):7.2f}  max {col.max():7.2f} us")
def chain(fn, n=8):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3
Ws = [torch.randn(4096, 4096).to(torch.bfloat16).cuda() for _ in range(8)]
acts = [torch.randn(512, 4096).to(torch.bfloat16).cuda() for _ in range(9)]
for bn in (1128, 1256, 2256):
    def fwd():
        for i in range(8):
            L.edl_gemm_bf16(acts[i].data_ptr(), 4096, 0, Ws[i].data_ptr(), 4096, 0, acts[i + 1].data_ptr(), 4096, 512, 4096, 4096, 1, 0, None, 0, bn, s())
    us = chain(fwd)
    show(f"fwd chain bn={bn}: {us/8:.1f} us per GEMM (graph)", 128 if bn in (1128, 2256) else 64)
    def dgrad():
        for i in range(8):
            L.edl_gemm_bf16(acts[i].data_ptr(), 4096, 0, Ws[i].data_ptr(), 4096, 1, acts[i + 1].data_ptr(), 4096, 512, 4096, 4096, 0, 0, None, 0, bn, s())
    us = chain(dgrad)
    show(f"dgrad chain bn={bn}: {us/8:.1f} us per GEMM (graph)", 128 if bn in (1128, 2256) else 64)
master = [torch.randn(4096, 4096, device='cuda') for _ in range(2)]
def wg():
    for i in range(8):
        L.edl_gemm_wgrad_sgd(acts[i].data_ptr(), 4096, acts[i+1].data_ptr(), 4096, master[i % 2].data_ptr(), Ws[i].data_ptr(), 4096, 4096, 4096, 512, C.c_float(1e-6), s())
us = chain(wg)
show(f"wgrad+sgd chain: {us/8:.1f} us per GEMM (graph)", 148)
g = torch.empty(4096, 4096, dtype=torch.bfloat16, device='cuda')
def wgp():
    for i in range(8):
        L.edl_gemm_bf16(acts[i].data_ptr(), 4096, 1, acts[i+1].data_ptr(), 4096, 1, g.data_ptr(), 4096, 4096, 4096, 512, 0, 0, None, 0, 1128, s())
us = chain(wgp)
show(f"wgrad bf16 chain: {us/8:.1f} us per GEMM (graph)", 148)
