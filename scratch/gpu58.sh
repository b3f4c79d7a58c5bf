export PYTHONUNBUFFERED=1
for wl in wide11264x8 mlp4096x8; do
for n in 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n --workload $wl > gpurun_out/b58_${wl}_$n.log 2>&1; echo "$wl N=$n rc=$?"
done; done
for f in gpurun_out/b58_*.log; do echo $f; tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); u=d['update_roofline']; print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), round(d['gemm_roofline']['frac'],3), {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()}, round(u['achieved']), round(u['exposed_allreduce_bus_gbs']), u['exchange_mode'])" || tail -5 $f; done
