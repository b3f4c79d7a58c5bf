export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_job_gpu.py -q -x 2>&1 | tail -2
for bn in 128 256; do EDL_SGD_BN=$bn python scratch/timeline.py scratch/trace/libedl_b200.so > gpurun_out/timeline5_$bn.log 2>&1; done
grep chain gpurun_out/timeline5_*.log
for bn in 128 256; do EDL_SGD_BN=$bn timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/sgdbn$bn.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/sgdbn$bn.log').read().strip().splitlines()[-1]); print($bn, round(d['value']), d['ms_per_step'], {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()})"; done
