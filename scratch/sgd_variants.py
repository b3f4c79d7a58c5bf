import ctypes as C, sys, os, torch
sys.path.insert(0, '.')
os.environ["EDL_LIB_PATH"] = os.path.abspath(sys.argv[1])
from paper_1909_11985_b200 import _lib
L = _lib.lib()
s = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)
torch.manual_seed(0)
acts = [torch.randn(512, 4096).to(torch.bfloat16).cuda() for _ in range(9)]
Ws = [torch.empty(4096, 4096, dtype=torch.bfloat16, device='cuda') for _ in range(8)]
master = [torch.randn(4096, 4096, device='cuda') for _ in range(8)]
m0 = master[0].clone()
L.edl_gemm_wgrad_sgd(acts[0].data_ptr(), 4096, acts[1].data_ptr(), 4096, master[0].data_ptr(), Ws[0].data_ptr(), 4096, 4096, 4096, 512, C.c_float(1e-3), s())
torch.cuda.synchronize()
g = (acts[0].float().t() @ acts[1].float()).bfloat16().float()
ref = m0 - 1e-3 * g
err = (master[0] - ref).abs().max().item()
ok = err <= 1e-3 * g.abs().max().item() * 2 ** -7 + 1e-6 and torch.equal(Ws[0], master[0].bfloat16())
def wg():
    for i in range(8):
        L.edl_gemm_wgrad_sgd(acts[i].data_ptr(), 4096, acts[i+1].data_ptr(), 4096, master[i].data_ptr(), Ws[i].data_ptr(), 4096, 4096, 4096, 512, C.c_float(1e-6), s())
for _ in range(2): wg()
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr):
    wg()
gr.replay(); torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(3):
    e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) * 1e3 / 8)
print(f"{sys.argv[1].split('/')[-2]:14s} {best:6.1f} us per wgrad+sgd  numerics {'OK' if ok else 'FAIL'} (err {err:.2e})", flush=True)
