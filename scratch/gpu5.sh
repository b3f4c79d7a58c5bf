timeout 120 python scratch/cublas_prof.py > gpurun_out/cublas_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none -s 12 -c 6 -o gpurun_out/cublas_cmp python scratch/cublas_prof.py > gpurun_out/ncu_cublas.log 2>&1
echo rc=$?
tail -3 gpurun_out/ncu_cublas.log
