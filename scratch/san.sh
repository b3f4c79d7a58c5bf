export PYTHONUNBUFFERED=1
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_elastic_multigpu_gpu.py -x -q -k linear > gpurun_out/san.log 2>&1; echo rc=$? >> gpurun_out/san.log
