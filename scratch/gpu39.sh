export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/full_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/full_pytest.log; tail -6 gpurun_out/full_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
