export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/full_pytest4.log 2>&1; echo "rc=$?" >> gpurun_out/full_pytest4.log; tail -3 gpurun_out/full_pytest4.log
python bench.py --no-cpu > gpurun_out/s1.log 2>&1
for n in 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $n > gpurun_out/s$n.log 2>&1; done
for n in 1 2 4; do tail -1 gpurun_out/s$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=%d' % d['n_gpus'], round(d['value']), 'e2e', round(d['e2e']['value']), 'ms', round(d['ms_per_step'],4), 'launches', d['gpu_launches'], 'clocks', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
