set -x
python -m pytest tests/test_multigpu_gpu.py -x -q -k "defer" > gpurun_out/mg_pt.log 2>&1; echo rc=$? >> gpurun_out/mg_pt.log
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu --no-nccl"
$T > gpurun_out/mg_b3.log 2>&1
EDL_AG_DEFER=2 $T > gpurun_out/mg_b3ce.log 2>&1
