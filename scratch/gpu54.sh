export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_job_gpu.py tests/test_recovery_gpu.py tests/test_straggler_gpu.py tests/test_elastic_multigpu_gpu.py tests/test_multigpu_gpu.py -q -x 2>&1 | tail -1
timeout 300 python bench.py --no-cpu > gpurun_out/inl.log 2>&1; tail -1 gpurun_out/inl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), d['gpu_launches'], {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()})"
