timeout 600 python -m pytest tests/test_elastic_multigpu_gpu.py tests/test_multigpu_gpu.py -q -x > gpurun_out/elastic_test.log 2>&1; echo "rc=$?" >> gpurun_out/elastic_test.log
tail -30 gpurun_out/elastic_test.log
