timeout 200 python scratch/trace_run.py > gpurun_out/trace.log 2>&1
timeout 200 python scratch/gemm2_check.py > gpurun_out/gemm2.log 2>&1
cat gpurun_out/trace.log; grep -E "BAD|4096" gpurun_out/gemm2.log; grep -c OK gpurun_out/gemm2.log
