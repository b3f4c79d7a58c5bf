export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_job_gpu.py -q -x 2>&1 | tail -1
for pdl in 1 0; do EDL_PDL=$pdl python scratch/timeline.py scratch/trace/libedl_b200.so 2>&1 | grep chain; done
for pdl in 1 0; do EDL_PDL=$pdl timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/pdl$pdl.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/pdl$pdl.log').read().strip().splitlines()[-1]); print('pdl', $pdl, round(d['value']), d['ms_per_step'], {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()})"; done
