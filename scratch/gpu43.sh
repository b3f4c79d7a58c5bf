export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_multigpu_gpu.py -q -x 2>&1 | tail -3
for ov in "" 0; do EDL_OVERLAP=$ov timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu > gpurun_out/rs2_$ov.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/rs2_$ov.log').read().strip().splitlines()[-1]); print('N=2 overlap=[$ov]', round(d['value']), round(d['ms_per_step'],4), {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()})" || tail -5 gpurun_out/rs2_$ov.log; done
