export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_elastic_multigpu_gpu.py -q -x 2>&1 | grep -v "^    " | tail -60
timeout 600 python tools/elastic_bench.py --gpus 4 > gpurun_out/elastic.log 2>&1; echo "elastic rc=$?"; tail -3 gpurun_out/elastic.log | cut -c1-3000
