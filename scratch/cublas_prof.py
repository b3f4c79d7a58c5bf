import torch, sys, ctypes as C
sys.path.insert(0,'.')
from paper_1909_11985_b200 import _lib
L=_lib.lib()
A = torch.randn(512, 4096, dtype=torch.bfloat16, device='cuda'); B = torch.randn(4096, 4096, dtype=torch.bfloat16, device='cuda')
dy = torch.randn(512, 4096, dtype=torch.bfloat16, device='cuda')
out = torch.empty(512, 4096, dtype=torch.bfloat16, device='cuda')
out2 = torch.empty(4096, 4096, dtype=torch.bfloat16, device='cuda')
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    A @ B.t(); A @ B; dy.t() @ A
    L.edl_gemm_bf16(A.data_ptr(), 4096, 0, B.data_ptr(), 4096, 0, out.data_ptr(), 4096, 512, 4096, 4096, 0, 0, None, 0, 1128, s)
    L.edl_gemm_bf16(A.data_ptr(), 4096, 0, B.data_ptr(), 4096, 0, out.data_ptr(), 4096, 512, 4096, 4096, 0, 0, None, 0, 128, s)
    L.edl_gemm_bf16(dy.data_ptr(), 4096, 1, A.data_ptr(), 4096, 1, out2.data_ptr(), 4096, 4096, 4096, 512, 0, 0, None, 0, 1256, s)
torch.cuda.synchronize()
print("done")
