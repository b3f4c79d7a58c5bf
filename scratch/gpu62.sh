export PYTHONUNBUFFERED=1
timeout 200 python scratch/trace2.py scratch/var/trace/libedl_b200.so 2>&1 | head -12
timeout 200 python scratch/timeline.py scratch/var/trace/libedl_b200.so 2>&1 | head -40
