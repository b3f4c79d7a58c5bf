import os, ctypes as C, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
backend = os.environ.get("PROBE_BACKEND", "nccl")
dist.init_process_group(backend)
n = 1 << 20
t = symm.empty(n, dtype=torch.bfloat16, device="cuda")
h = symm.rendezvous(t, dist.group.WORLD.group_name)
print(rank, "multicast_ptr", h.multicast_ptr, "bufs", len(h.buffer_ptrs), flush=True)
L = C.CDLL(os.path.join(os.path.dirname(__file__), "libnvls_probe.so"))
t.fill_(rank + 1)
torch.cuda.synchronize(); dist.barrier()
if h.multicast_ptr:
    out = torch.empty(n, device="cuda")
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    print(rank, "ld_reduce rc", L.launch_ld_reduce(C.c_void_p(h.multicast_ptr), C.c_void_p(out.data_ptr()), C.c_size_t(n // 8), s), flush=True)
    torch.cuda.synchronize()
    print(rank, "sum", out[:4].tolist(), "expect", sum(range(1, world + 1)), flush=True)
    # timing: ld_reduce bandwidth on 256 MB
    big = symm.empty(128 << 20, dtype=torch.bfloat16, device="cuda")
    hb = symm.rendezvous(big, dist.group.WORLD.group_name)
    outb = torch.empty(128 << 20, device="cuda")
    dist.barrier(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    nb = (128 << 20) // 8 // world  # each rank reduces its 1/world shard
    off = rank * nb * 16
    for it in range(3):
        e0.record()
        L.launch_ld_reduce(C.c_void_p(hb.multicast_ptr + off), C.c_void_p(outb.data_ptr()), C.c_size_t(nb), s)
        e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3
    print(rank, f"ld_reduce shard {nb*16/1e6:.1f} MB bf16 in {us:.1f} us -> {nb*16/us/1e3:.1f} GB/s (shard bytes)", flush=True)
    src = torch.empty(128 << 20, dtype=torch.bfloat16, device="cuda")
    for it in range(3):
        dist.barrier(); torch.cuda.synchronize()
        e0.record()
        L.launch_mc_store(C.c_void_p(hb.multicast_ptr + off), C.c_void_p(src.data_ptr() + off), C.c_size_t(nb), s)
        e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3
    print(rank, f"multimem.st shard {nb*16/1e6:.1f} MB in {us:.1f} us -> {nb*16/us/1e3:.1f} GB/s", flush=True)
dist.barrier()
dist.destroy_process_group()
