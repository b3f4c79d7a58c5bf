import ctypes as C, sys, os, torch, numpy as np
sys.path.insert(0, '.')
os.environ["EDL_LIB_PATH"] = os.path.abspath("scratch/trace/libedl_b200.so")
from paper_1909_11985_b200 import _lib
L = _lib.lib()
L.edl_debug_gemm_trace.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros((296, 8), dtype=np.uint64)
def run(a_mn, b_mn, M, N, K, bn):
    A = (torch.randn(K, M) if a_mn else torch.randn(M, K)).to(torch.bfloat16).cuda()
    B = (torch.randn(K, N) if b_mn else torch.randn(N, K)).to(torch.bfloat16).cuda()
    out = torch.empty(M, N, dtype=torch.bfloat16, device='cuda')
    args = (A.data_ptr(), A.shape[1], a_mn, B.data_ptr(), B.shape[1], b_mn, out.data_ptr(), N, M, N, K, 0, 0, None, 0, bn)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(3): L.edl_gemm_bf16(*args, s)
    L.edl_debug_gemm_trace(buf.ctypes.data, 1)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); L.edl_gemm_bf16(*args, s); e1.record(); torch.cuda.synchronize()
    L.edl_debug_gemm_trace(buf.ctypes.data, 1)
    us = e0.elapsed_time(e1)*1e3
    real = bn - 1000
    tiles = ((M+255)//256)*((N+real-1)//real); ctas = 2*min(tiles, 74)
    lead = buf[0:ctas:2].astype(np.float64); peer = buf[1:ctas:2].astype(np.float64)
    f = lambda x: x.mean()/1.965e3
    kb = (K+63)//64 * ((tiles + 73)//74)
    print(f"a{a_mn}b{b_mn} M={M} N={N} K={K} bn={bn}: {us:.1f} us (1 launch)  per leader CTA (us): mma_total {f(lead[:,2]):.2f}  wait_full {f(lead[:,0]):.2f}  wait_tempty {f(lead[:,1]):.2f} | producer total L {f(lead[:,4]):.2f} P {f(peer[:,4]):.2f}  wait_empty L {f(lead[:,3]):.2f} P {f(peer[:,3]):.2f} | kblocks {kb} -> mma-bound time {kb*4*(256*real/512)/1.965e3:.2f} us", flush=True)
for bn in (1128, 1256):
    run(0, 0, 512, 4096, 4096, bn)
    run(0, 0, 512, 4096, 16384, bn)
run(1, 1, 4096, 4096, 512, 1256)
