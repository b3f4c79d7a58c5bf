export PYTHONUNBUFFERED=1
timeout 300 python scratch/repro_elastic.py > gpurun_out/repro.log 2>&1; echo "rc=$?" >> gpurun_out/repro.log
cat gpurun_out/repro.log | tail -20
