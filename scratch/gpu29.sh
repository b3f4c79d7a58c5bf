export PYTHONUNBUFFERED=1
nvidia-smi topo -m | head -8
for be in nccl gloo; do echo "== backend $be"; PROBE_BACKEND=$be timeout 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 scratch/nvls/probe.py 2>&1 | grep -v Warning | tail -12; done
