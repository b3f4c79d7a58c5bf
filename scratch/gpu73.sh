export PYTHONUNBUFFERED=1
echo "== session-start build"
(cd scratch/base && timeout 600 python -m pytest tests/test_elastic_multigpu_gpu.py -q -x -k linear 2>&1 | tail -3)
echo "== current under memcheck"
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_elastic_multigpu_gpu.py -q -x -k linear 2>&1 | grep -v "^    " | head -60
