for d in 0 1 2; do echo "== dbg $d"; EDL_GEMM_DBG=$d timeout 120 python scratch/trace_sgd2.py scratch/trace/libedl_b200.so; done
