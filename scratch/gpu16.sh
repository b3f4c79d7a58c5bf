export PYTHONUNBUFFERED=1
timeout 200 python scratch/repro2.py sched > gpurun_out/repro2a.log 2>&1
timeout 200 python scratch/repro2.py api > gpurun_out/repro2b.log 2>&1
tail -6 gpurun_out/repro2a.log; tail -6 gpurun_out/repro2b.log
