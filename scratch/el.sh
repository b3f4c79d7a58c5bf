export PYTHONUNBUFFERED=1
for i in 1 2 3 4; do
timeout 300 python -m pytest tests/test_elastic_multigpu_gpu.py -x -q 2>&1 | tail -n 1 >> gpurun_out/el_new.log
done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pt4d.log 2>&1; echo rc=$? >> gpurun_out/pt4d.log
