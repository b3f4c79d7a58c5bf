export PYTHONUNBUFFERED=1
timeout 200 python scratch/timeline.py scratch/var/trace/libedl_b200.so 2>&1 | grep -A16 "chain bn=2256"
