export PYTHONUNBUFFERED=1
for i in 1 2 3; do timeout 900 python -m pytest tests/test_straggler_gpu.py -q -x 2>&1 | grep -E "^E |passed|failed" | head -6; done
