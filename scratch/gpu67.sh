export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_multigpu_gpu.py -q -x 2>&1 | tail -2
for n in 2 4; do for d in 0 1; do
EDL_AG_DEFER=$d timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n bench.py --gpus $n > gpurun_out/b67_${n}_$d.log 2>&1; echo "N=$n defer=$d rc=$?"
tail -1 gpurun_out/b67_${n}_$d.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); u=d['update_roofline']; print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()}, round(u['achieved']))" || tail -5 gpurun_out/b67_${n}_$d.log
done; done
