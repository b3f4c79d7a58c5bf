export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_elastic_multigpu_gpu.py -q -x 2>&1 | grep -v "^  " | tail -40
