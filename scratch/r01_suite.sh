timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -n 12 gpurun_out/pytest_gpu4.log; cat gpurun_out/smoke.log
