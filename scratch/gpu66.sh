export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -3
for cfg in "EDL_GEMM_MC=4" "EDL_GEMM_MC=2"; do
env $cfg timeout 300 python bench.py --no-cpu > gpurun_out/b66.log 2>&1; echo "$cfg rc=$?"
tail -1 gpurun_out/b66.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), round(d['gemm_roofline']['frac'],3), {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()})" || tail -5 gpurun_out/b66.log
done
