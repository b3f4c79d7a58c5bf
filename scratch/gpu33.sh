export PYTHONUNBUFFERED=1
for n in 4 2; do for ov in 0 2; do EDL_OVERLAP=$ov timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $n --steps 30 --warmup 5 --no-cpu > gpurun_out/ce${n}_$ov.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/ce${n}_$ov.log').read().strip().splitlines()[-1]); print('N=$n overlap', $ov, round(d['value']), d['ms_per_step'], {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()}, d.get('update_roofline'))" || tail -3 gpurun_out/ce${n}_$ov.log; done; done
