export PYTHONUNBUFFERED=1
for dbg in 68 72 80 116; do
EDL_GEMM_DBG=$dbg EDL_OVERLAP=4 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus 2 --no-nccl --steps 30 > gpurun_out/b87_$dbg.log 2>&1; echo "dbg=$dbg rc=$?"
tail -1 gpurun_out/b87_$dbg.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()}, round(d['wgrad_ms_per_step']*1e3,1))" || tail -3 gpurun_out/b87_$dbg.log
done
