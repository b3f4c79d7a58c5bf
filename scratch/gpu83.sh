export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for i in 1 2; do timeout 600 python bench.py > gpurun_out/bench$i.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench$i.log; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 300 python tools/profile_step.py --size 65536 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --size 65536 > gpurun_out/ncu_launch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16|allreduce_sgd|xent|gather" -s 72 -c 24 -o gpurun_out/prof_full python tools/profile_step.py --size 65536 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
for i in 1 2; do tail -2 gpurun_out/bench$i.log | head -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N=1', round(d['value']), round(d['e2e']['value']), round(d['roofline']['frac'],3), round(d['roofline']['launch_ms']*1e3,1), d['clocks'])"; done
tail -1 gpurun_out/bench_ref.log | cut -c1-200
