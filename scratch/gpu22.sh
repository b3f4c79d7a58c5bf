export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_job_gpu.py -q -x 2>&1 | tail -2
python scratch/timeline.py scratch/trace/libedl_b200.so > gpurun_out/timeline4.log 2>&1
EDL_GEMM_MC=0 python scratch/timeline.py scratch/trace/libedl_b200.so > gpurun_out/timeline4_mc0.log 2>&1
grep chain gpurun_out/timeline4.log gpurun_out/timeline4_mc0.log
for mc in 1 0; do EDL_GEMM_MC=$mc timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/mc$mc.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/mc$mc.log').read().strip().splitlines()[-1]); print($mc, round(d['value']), d['ms_per_step'], {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()})"; done
