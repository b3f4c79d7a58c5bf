export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_multigpu_gpu.py -q -x -k "4" 2>&1 | tail -2
for n in 2 4; do for ov in 4; do
EDL_OVERLAP=$ov timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n bench.py --gpus $n --no-nccl > gpurun_out/b80_${n}_$ov.log 2>&1; echo "N=$n ov=$ov rc=$?"
tail -1 gpurun_out/b80_${n}_$ov.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); u=d['update_roofline']; print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()}, 'mode', u.get('exchange_mode'))" || tail -5 gpurun_out/b80_${n}_$ov.log
done; done
