import os, ctypes as C, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
import glob
cudart = None
for cand in glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + glob.glob("/usr/local/cuda/lib64/libcudart.so*"):
    try:
        cudart = C.CDLL(cand); break
    except OSError:
        pass
n = 128 << 20  # bf16 elements = 256 MB
buf = symm.empty(n, dtype=torch.bfloat16, device="cuda")
h = symm.rendezvous(buf, dist.group.WORLD.group_name)
src = torch.ones(n, dtype=torch.bfloat16, device="cuda")
peer = (rank + 1) % world
s = torch.cuda.Stream()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
for nbytes in (32 << 20, 134 << 20, 256 << 20):
    for it in range(3):
        dist.barrier(); torch.cuda.synchronize()
        with torch.cuda.stream(s):
            e0.record(s)
            rc = cudart.cudaMemcpyAsync(C.c_void_p(h.buffer_ptrs[peer]), C.c_void_p(src.data_ptr()), C.c_size_t(nbytes), 3, C.c_void_p(s.cuda_stream))
            e1.record(s)
        torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3
    print(rank, f"CE push {nbytes/1e6:.0f} MB to peer (both ranks at once): {us:.1f} us -> {nbytes/us/1e3:.0f} GB/s rc={rc}", flush=True)
# CE pull
for it in range(3):
    dist.barrier(); torch.cuda.synchronize()
    e0.record(s)
    rc = cudart.cudaMemcpyAsync(C.c_void_p(src.data_ptr()), C.c_void_p(h.buffer_ptrs[peer]), C.c_size_t(134 << 20), 3, C.c_void_p(s.cuda_stream))
    e1.record(s)
    torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3
print(rank, f"CE pull 134 MB from peer: {us:.1f} us -> {(134<<20)/us/1e3:.0f} GB/s", flush=True)
# GEMM slowdown under a concurrent CE push
A = torch.randn(512, 4096, device="cuda").bfloat16(); B = torch.randn(4096, 4096, device="cuda").bfloat16()
def gemms(k=40):
    for _ in range(k): A @ B.t()
for it in range(2):
    torch.cuda.synchronize(); e0.record(); gemms(); e1.record(); torch.cuda.synchronize()
alone = e0.elapsed_time(e1) * 1e3 / 40
dist.barrier(); torch.cuda.synchronize()
with torch.cuda.stream(s):
    for _ in range(4):
        cudart.cudaMemcpyAsync(C.c_void_p(h.buffer_ptrs[peer]), C.c_void_p(src.data_ptr()), C.c_size_t(256 << 20), 3, C.c_void_p(s.cuda_stream))
e0.record(); gemms(); e1.record(); torch.cuda.synchronize()
both = e0.elapsed_time(e1) * 1e3 / 40
print(rank, f"cuBLAS 512x4096x4096: alone {alone:.1f} us, under CE push {both:.1f} us", flush=True)
dist.barrier()
