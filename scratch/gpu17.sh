export PYTHONUNBUFFERED=1
timeout 900 python tools/elastic_bench.py --gpus 4 > gpurun_out/elastic.log 2>&1; echo "rc=$?" >> gpurun_out/elastic.log
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log; tail -c 600 gpurun_out/elastic.log
