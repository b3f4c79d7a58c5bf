for st in 6 8; do echo "=== stages $st"; python scratch/timeline.py scratch/trace$st/libedl_b200.so; done > gpurun_out/timeline2.log 2>&1
cat gpurun_out/timeline2.log
