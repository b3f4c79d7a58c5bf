export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python bench.py --no-cpu > gpurun_out/b64_1.log 2>&1; echo rc=$?
EDL_GEMM_SPLITK=0 timeout 300 python bench.py --no-cpu > gpurun_out/b64_0.log 2>&1; echo rc=$?
for f in gpurun_out/b64_*.log; do echo $f; tail -1 $f | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), round(d['gemm_roofline']['frac'],3), {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()})" || tail -5 $f; done
