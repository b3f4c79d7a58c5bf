export PYTHONUNBUFFERED=1
EDL_OVERLAP=3 timeout 900 python -m pytest tests/test_multigpu_gpu.py -q -x > gpurun_out/m3_pytest.log 2>&1; tail -1 gpurun_out/m3_pytest.log; grep -E "MP-PARITY|FAILED" gpurun_out/m3_pytest.log | head -3
for n in 2 4; do for ov in 3 0; do EDL_OVERLAP=$ov timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $n --steps 30 --warmup 5 --no-cpu > gpurun_out/m3_${n}_$ov.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/m3_${n}_$ov.log').read().strip().splitlines()[-1]); print('N=$n overlap=$ov', round(d['value']), round(d['ms_per_step'],4), {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()})" || tail -5 gpurun_out/m3_${n}_$ov.log; done; done
