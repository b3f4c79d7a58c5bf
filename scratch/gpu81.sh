export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_job_gpu.py -q -x 2>&1 | tail -1
timeout 900 python -m pytest tests/test_multigpu_gpu.py -q -x -k "4 or 3" 2>&1 | tail -2
timeout 300 python bench.py --no-cpu > gpurun_out/b81_1.log 2>&1; tail -1 gpurun_out/b81_1.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N=1', round(d['value']), round(d['roofline']['frac'],3))"
for n in 2 4; do for ov in 4 ""; do
EDL_OVERLAP=$ov timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n bench.py --gpus $n --no-nccl > gpurun_out/b81_${n}_$ov.log 2>&1; echo "N=$n ov=$ov rc=$?"
tail -1 gpurun_out/b81_${n}_$ov.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); u=d['update_roofline']; print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()}, 'mode', u.get('exchange_mode'))" || tail -5 gpurun_out/b81_${n}_$ov.log
done; done
