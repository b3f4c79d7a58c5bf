export PYTHONUNBUFFERED=1
for i in 1 2 3; do timeout 900 python -m pytest tests/test_multigpu_gpu.py tests/test_elastic_multigpu_gpu.py -q > gpurun_out/push_pytest_$i.log 2>&1; tail -1 gpurun_out/push_pytest_$i.log; grep -E "^FAILED|MP-PARITY FAIL|Error" gpurun_out/push_pytest_$i.log | head -5; done
