export PYTHONUNBUFFERED=1
EDL_CE_TRACE=1 EDL_OVERLAP=2 EDL_CE_UPDATE_BLOCKS=296 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/cetrace.log 2>&1
grep "ce-trace rank 0" gpurun_out/cetrace.log | tail -44
