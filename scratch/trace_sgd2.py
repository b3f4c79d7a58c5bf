import ctypes as C, sys, os, torch, numpy as np
sys.path.insert(0, '.')
os.environ["EDL_LIB_PATH"] = os.path.abspath(sys.argv[1] if len(sys.argv) > 1 else "scratch/trace/libedl_b200.so")
from paper_1909_11985_b200 import _lib
L = _lib.lib()
L.edl_debug_gemm_trace.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros((296, 16), dtype=np.uint64)
s = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)
names = {0: "mma_wait_full", 1: "mma_wait_tempty", 2: "mma_total", 3: "prod_wait_empty", 4: "prod_total",
         5: "epi_wait_tfull", 6: "sgd_wait_read", 7: "sgd_wait_master", 8: "epi_total", 9: "tmem_ld", 10: "compute_store", 11: "rmw", 12: "w_sts", 13: "fence"}
acts = [torch.randn(512, 4096).to(torch.bfloat16).cuda() for _ in range(9)]
Ws = [torch.empty(4096, 4096, dtype=torch.bfloat16, device='cuda') for _ in range(8)]
master = [torch.randn(4096, 4096, device='cuda') for _ in range(8)]
def wg():
    for i in range(8):
        L.edl_gemm_wgrad_sgd(acts[i].data_ptr(), 4096, acts[i+1].data_ptr(), 4096, master[i].data_ptr(), Ws[i].data_ptr(), 4096, 4096, 4096, 512, C.c_float(1e-6), s())
for _ in range(2): wg()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    wg()
g.replay(); torch.cuda.synchronize()
L.edl_debug_gemm_trace(buf.ctypes.data, 1)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
L.edl_debug_gemm_trace(buf.ctypes.data, 1)
print(f"wgrad+sgd (8 distinct masters, graph): {e0.elapsed_time(e1)*1e3/8:.1f} us per GEMM")
b = buf.astype(np.float64) / 1.965e3 / 8
for role, sl in (("leader", slice(0, 148, 2)), ("peer", slice(1, 148, 2))):
    print(role, " ".join(f"{n}={b[sl, i].mean():.2f}" for i, n in names.items() if b[sl, i].any()))
