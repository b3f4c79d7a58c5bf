import ctypes as C, sys, os, torch, numpy as np
sys.path.insert(0, '.')
os.environ["EDL_LIB_PATH"] = os.path.abspath("scratch/trace/libedl_b200.so")
from paper_1909_11985_b200 import _lib
L = _lib.lib()
L.edl_debug_gemm_trace.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros((296, 8), dtype=np.uint64)
M=N=4096; K=512
dy = torch.randn(K, M).to(torch.bfloat16).cuda(); x = torch.randn(K, N).to(torch.bfloat16).cuda()
master = (torch.randn(M, N) * 0.05).cuda(); W = master.to(torch.bfloat16)
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
args=(dy.data_ptr(), M, x.data_ptr(), N, master.data_ptr(), W.data_ptr(), N, M, N, K, 1e-3, s)
for _ in range(3): L.edl_gemm_wgrad_sgd(*args)
L.edl_debug_gemm_trace(buf.ctypes.data, 1)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); L.edl_gemm_wgrad_sgd(*args); e1.record(); torch.cuda.synchronize()
L.edl_debug_gemm_trace(buf.ctypes.data, 1)
us = e0.elapsed_time(e1)*1e3
b = buf[:148].astype(np.float64) / 1.965e3  # us
lead = b[0::2]
print(f"fused wgrad+sgd 4096^2 x 512: {us:.1f} us")
print(f"MMA (leader): total {lead[:,2].mean():.1f} wait_full {lead[:,0].mean():.1f} wait_tempty {lead[:,1].mean():.1f}")
print(f"producer wait_empty {b[:,3].mean():.1f}")
print(f"epilogue per CTA summed over 4 warps: total(+producer) {b[:,4].mean():.1f} wait_tfull {b[:,5].mean():.1f} wait_store_read {b[:,6].mean():.1f} wait_master_load {b[:,7].mean():.1f}")
