export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_job_gpu.py -q -x 2>&1 | tail -1
python scratch/trace_sgd2.py scratch/trace/libedl_b200.so
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/direct.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/direct.log').read().strip().splitlines()[-1]); print(round(d['value']), d['ms_per_step'], {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()})"
