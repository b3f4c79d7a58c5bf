export PYTHONUNBUFFERED=1
for mc in 0 1; do for pt in 0 1; do EDL_SGD_MC=$mc EDL_GEMM_PF_TILES=$pt timeout 120 python scratch/sgd_variants.py paper_1909_11985_b200/libedl_b200.so | sed "s/^/mc=$mc pf_tiles=$pt /"; done; done
EDL_SGD_MC=1 EDL_GEMM_PF_TILES=0 timeout 120 python scratch/trace_sgd2.py scratch/var/trace/libedl_b200.so
EDL_SGD_MC=0 EDL_GEMM_PF_TILES=0 timeout 120 python scratch/trace_sgd2.py scratch/var/trace/libedl_b200.so
