export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/rec_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rec_pytest.log; tail -15 gpurun_out/rec_pytest.log
