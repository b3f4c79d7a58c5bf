timeout 120 python scratch/sgd_check.py > gpurun_out/sgd.log 2>&1; cat gpurun_out/sgd.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -c 1500 gpurun_out/bench.log
