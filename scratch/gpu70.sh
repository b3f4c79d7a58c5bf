export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_multigpu_gpu.py tests/test_elastic_multigpu_gpu.py -q 2>&1 | tail -2
for wl in mlp4096x8 wide11264x8; do for n in 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --gpus $n --workload $wl > gpurun_out/b70_${wl}_$n.log 2>&1; echo "$wl N=$n rc=$?"
tail -1 gpurun_out/b70_${wl}_$n.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); u=d['update_roofline']; print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()}, 'AG', round(u['achieved']), 'nccl', u.get('nccl_allreduce_same_bytes'))" || tail -5 gpurun_out/b70_${wl}_$n.log
done; done
timeout 600 python tools/elastic_bench.py --gpus 4 > gpurun_out/elastic.log 2>&1; echo "elastic rc=$?"; tail -30 gpurun_out/elastic.log
