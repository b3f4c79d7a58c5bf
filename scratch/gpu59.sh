export PYTHONUNBUFFERED=1
for v in paper_1909_11985_b200 scratch/var/w4b2 scratch/var/w4b3; do timeout 120 python scratch/sgd_variants.py $v/libedl_b200.so; done
for pt in 0 2 3; do EDL_GEMM_PF_TILES=$pt timeout 120 python scratch/sgd_variants.py paper_1909_11985_b200/libedl_b200.so | sed "s/^/pf_tiles=$pt /"; done
EDL_SGD_BN=256 timeout 120 python scratch/sgd_variants.py paper_1909_11985_b200/libedl_b200.so | sed "s/^/bn256 /"
timeout 120 python scratch/trace_sgd2.py scratch/var/trace/libedl_b200.so
