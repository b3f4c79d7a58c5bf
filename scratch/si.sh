python -m pytest tests/test_multigpu_gpu.py -x -q -k scale_in > gpurun_out/si4.log 2>&1; echo rc=$? >> gpurun_out/si4.log
CUDA_VISIBLE_DEVICES=0,1 python -m pytest tests/test_multigpu_gpu.py -x -q -k scale_in > gpurun_out/si2.log 2>&1; echo rc=$? >> gpurun_out/si2.log
