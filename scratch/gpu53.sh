export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_job_gpu.py tests/test_gemm_gpu.py tests/test_recovery_gpu.py tests/test_straggler_gpu.py -q -x 2>&1 | tail -1
for bn in 128 256; do EDL_SGD_BN=$bn timeout 120 python scratch/sgd_variants.py paper_1909_11985_b200/libedl_b200.so; done
for bn in 128 256; do EDL_SGD_BN=$bn timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/sbn$bn.log 2>&1; tail -1 gpurun_out/sbn$bn.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sgd bn $bn', round(d['value']), d['roofline']['launch_ms'], d['gpu_launches'])"; done
