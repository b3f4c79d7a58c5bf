python -m pytest tests -m gpu -x -q > gpurun_out/pt4.log 2>&1; echo rc=$? >> gpurun_out/pt4.log
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu"
$T > gpurun_out/b4.log 2>&1
EDL_AG_DEFER=2 $T --no-nccl > gpurun_out/b4ce.log 2>&1
