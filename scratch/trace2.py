import ctypes as C, sys, os, torch, numpy as np
sys.path.insert(0, '.')
os.environ["EDL_LIB_PATH"] = os.path.abspath(sys.argv[1] if len(sys.argv) > 1 else "scratch/trace/libedl_b200.so")
from paper_1909_11985_b200 import _lib
L = _lib.lib()
TRACE = hasattr(L, "edl_debug_gemm_trace")
try:
    L.edl_debug_gemm_trace.argtypes = [C.c_void_p, C.c_int]
except AttributeError:
    TRACE = False
buf = np.zeros((296, 8), dtype=np.uint64)
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
s = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)
names = ["mma_wait_full", "mma_wait_tempty", "mma_total", "prod_wait_empty", "prod/epi_total", "epi_wait_tfull", "sgd_wait_read", "sgd_wait_master"]
def timed(fn, cold):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    if TRACE: L.edl_debug_gemm_trace(buf.ctypes.data, 1)
    if cold: flush.fill_(1)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3
    if TRACE: L.edl_debug_gemm_trace(buf.ctypes.data, 1)
    return us
def report(tag, us, ctas):
    line = f"{tag}: {us:.1f} us"
    if TRACE:
        lead = buf[0:ctas:2].astype(np.float64) / 1.965e3; peer = buf[1:ctas:2].astype(np.float64) / 1.965e3
        line += " | leader " + " ".join(f"{n}={lead[:, i].mean():.2f}" for i, n in enumerate(names) if lead[:, i].any())
        line += " | peer " + " ".join(f"{n}={peer[:, i].mean():.2f}" for i, n in enumerate(names) if peer[:, i].any())
    print(line, flush=True)
M, N, K = 512, 4096, 4096
for a_mn, b_mn, tag in ((0, 0, "fwd"), (0, 1, "dgrad")):
    A = (torch.randn(K, M) if a_mn else torch.randn(M, K)).to(torch.bfloat16).cuda()
    B = (torch.randn(K, N) if b_mn else torch.randn(N, K)).to(torch.bfloat16).cuda()
    out = torch.empty(M, N, dtype=torch.bfloat16, device='cuda')
    for bn in (1128, 1256):
        args = (A.data_ptr(), A.shape[1], a_mn, B.data_ptr(), B.shape[1], b_mn, out.data_ptr(), N, M, N, K, 0, 0, None, 0, bn)
        fn = lambda: L.edl_gemm_bf16(*args, s())
        tiles = 2 * ((N + bn - 1000 - 1) // (bn - 1000))
        for cold in (0, 1):
            report(f"{tag} bn={bn} {'cold' if cold else 'hot '}", timed(fn, cold), 2 * min(tiles, 74))
dy = torch.randn(512, 4096).to(torch.bfloat16).cuda(); x = torch.randn(512, 4096).to(torch.bfloat16).cuda()
master = torch.randn(4096, 4096, device='cuda'); W = torch.empty(4096, 4096, dtype=torch.bfloat16, device='cuda')
fn = lambda: L.edl_gemm_wgrad_sgd(dy.data_ptr(), 4096, x.data_ptr(), 4096, master.data_ptr(), W.data_ptr(), 4096, 4096, 4096, 512, C.c_float(1e-6), s())
for cold in (0, 1):
    report(f"wgrad+sgd {'cold' if cold else 'hot '}", timed(fn, cold), 148)
# plain wgrad without sgd (bf16 out)
g = torch.empty(4096, 4096, dtype=torch.bfloat16, device='cuda')
args = (dy.data_ptr(), 4096, 1, x.data_ptr(), 4096, 1, g.data_ptr(), 4096, 4096, 4096, 512, 0, 0, None, 0, 1128)
fn = lambda: L.edl_gemm_bf16(*args, s())
for cold in (0, 1):
    report(f"wgrad bf16 {'cold' if cold else 'hot '}", timed(fn, cold), 148)
# chain of 8 fwd GEMMs over distinct weights (as in the step), graph-captured
Ws = [torch.randn(4096, 4096).to(torch.bfloat16).cuda() for _ in range(8)]
acts = [torch.randn(512, 4096).to(torch.bfloat16).cuda() for _ in range(9)]
def chain():
    for i in range(8):
        L.edl_gemm_bf16(acts[i].data_ptr(), 4096, 0, Ws[i].data_ptr(), 4096, 0, acts[i + 1].data_ptr(), 4096, 512, 4096, 4096, 1, 0, None, 0, 1128, s())
for _ in range(3): chain()
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr):
    chain()
gr.replay(); torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
print(f"chain of 8 fwd (distinct W, graph): {e0.elapsed_time(e1)*1e3/8:.1f} us per GEMM", flush=True)
gr2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr2):
    for i in range(8):
        L.edl_gemm_bf16(acts[0].data_ptr(), 4096, 0, Ws[0].data_ptr(), 4096, 0, acts[1].data_ptr(), 4096, 512, 4096, 4096, 1, 0, None, 0, 1128, s())
gr2.replay(); torch.cuda.synchronize()
e0.record(); gr2.replay(); e1.record(); torch.cuda.synchronize()
print(f"chain of 8 fwd (same W, graph): {e0.elapsed_time(e1)*1e3/8:.1f} us per GEMM", flush=True)
