for v in scratch/st2 scratch/st3 scratch/st4 paper_1909_11985_b200; do EDL_LIB_PATH=$PWD/$v/libedl_b200.so timeout 200 python scratch/gemm_exp.py; done > gpurun_out/gemm_exp.log 2>&1
cat gpurun_out/gemm_exp.log
