timeout 300 python scratch/gemm_time.py > gpurun_out/gemm_time.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench.log 2>&1
cat gpurun_out/gemm_time.log; tail -3 gpurun_out/pytest_gpu.log; tail -c 1500 gpurun_out/bench.log
