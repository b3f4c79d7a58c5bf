export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/mc_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/mc_gemm.log
tail -5 gpurun_out/mc_gemm.log
if grep -q "rc=0" gpurun_out/mc_gemm.log; then
  python scratch/timeline.py scratch/trace/libedl_b200.so > gpurun_out/timeline3.log 2>&1
  EDL_GEMM_MC=0 python scratch/timeline.py scratch/trace/libedl_b200.so > gpurun_out/timeline3_mc0.log 2>&1
  grep chain gpurun_out/timeline3.log gpurun_out/timeline3_mc0.log
  timeout 600 python -m pytest tests/test_job_gpu.py -q -x 2>&1 | tail -2
  for mc in 1 0; do EDL_GEMM_MC=$mc timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/mc$mc.log 2>&1; tail -1 gpurun_out/mc$mc.log | cut -c1-200; done
fi
