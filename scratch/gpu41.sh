for d in 1 0; do for pf in 0 1 2; do echo "dbg=$d pf_tiles=$pf"; EDL_GEMM_DBG=$d EDL_GEMM_PF_TILES=$pf timeout 120 python scratch/trace_sgd2.py scratch/trace/libedl_b200.so | head -2; done; done
