export PYTHONUNBUFFERED=1
for s in 0 1; do echo "== spread=$s"; EDL_BCAST_SPREAD=$s timeout 600 python -m pytest tests/test_elastic_multigpu_gpu.py -q -x 2>&1 | tail -2; done
