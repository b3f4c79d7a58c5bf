python scratch/trace2.py scratch/trace/libedl_b200.so > gpurun_out/trace2.log 2>&1
echo ---- >> gpurun_out/trace2.log
python scratch/trace2.py paper_1909_11985_b200/libedl_b200.so >> gpurun_out/trace2.log 2>&1
cat gpurun_out/trace2.log
