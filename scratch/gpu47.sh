export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_multigpu_gpu.py tests/test_elastic_multigpu_gpu.py -q -x 2>&1 | tail -2
for n in 2 4; do for p in 1 0; do EDL_COLL_PUSH=$p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $n --steps 30 --warmup 5 --no-cpu > gpurun_out/push${n}_$p.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/push${n}_$p.log').read().strip().splitlines()[-1]); print('N=$n push=$p', round(d['value']), round(d['ms_per_step'],4), 'update', round(d['phase_ms_per_step']['update']*1e3,1), 'GB/s', round(d['update_roofline']['achieved']))" || tail -5 gpurun_out/push${n}_$p.log; done; done
