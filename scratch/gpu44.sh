export PYTHONUNBUFFERED=1
unset EDL_OVERLAP
for n in 2 4; do for ov in 3 0; do EDL_OVERLAP=$ov timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $n --steps 30 --warmup 5 --no-cpu > gpurun_out/rs${n}_$ov.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/rs${n}_$ov.log').read().strip().splitlines()[-1]); print('N=$n overlap=$ov', round(d['value']), round(d['ms_per_step'],4), {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()})" || tail -5 gpurun_out/rs${n}_$ov.log; done; done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu > gpurun_out/rs4_default.log 2>&1; tail -1 gpurun_out/rs4_default.log | cut -c1-200
