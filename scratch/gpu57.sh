export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python bench.py --no-cpu > gpurun_out/b57_1.log 2>&1; echo rc=$?
timeout 300 python bench.py --no-cpu --workload wide11264x8 > gpurun_out/b57_w1.log 2>&1; echo rc=$?
for f in gpurun_out/b57_*.log; do echo $f; tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), round(d['roofline']['launch_ms']*1e3,1), round(d['gemm_roofline']['frac'],3), {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()})" || tail -5 $f; done
