export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_job_gpu.py -q -x -k "wide or mlp" 2>&1 | grep -E "passed|failed|^E " | head -20
