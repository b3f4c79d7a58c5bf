T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu --no-nccl"
for s in 1 2 3; do EDL_AG_DEFER=2 EDL_AG_CE_SPLIT=$s $T > gpurun_out/mg_ce$s.log 2>&1; done
$T > gpurun_out/mg_b3.log 2>&1
