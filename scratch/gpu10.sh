export PYTHONUNBUFFERED=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench2.log 2>&1; echo "rc=$?" >> gpurun_out/bench2.log
tail -c 2500 gpurun_out/bench2.log
