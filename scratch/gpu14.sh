export PYTHONUNBUFFERED=1
timeout 900 python tools/elastic_bench.py --gpus 4 > gpurun_out/elastic.log 2>&1; echo "rc=$?" >> gpurun_out/elastic.log
tail -c 4000 gpurun_out/elastic.log
