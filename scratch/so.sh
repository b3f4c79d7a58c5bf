export PYTHONUNBUFFERED=1
CUDA_VISIBLE_DEVICES=0,1 timeout 300 python -m pytest tests/test_multigpu_gpu.py -x -q -k "scale_out or scale_in" > gpurun_out/so2.log 2>&1; echo rc=$? >> gpurun_out/so2.log
timeout 300 python -m pytest tests/test_multigpu_gpu.py -x -q -k "scale_out or scale_in" > gpurun_out/so4.log 2>&1; echo rc=$? >> gpurun_out/so4.log
