export PYTHONUNBUFFERED=1
for v in paper_1909_11985_b200 scratch/var/wd scratch/var/wd3; do timeout 120 python scratch/sgd_variants.py $v/libedl_b200.so; done
timeout 120 python scratch/trace_sgd2.py scratch/var/wdtr/libedl_b200.so
