for v in scratch/g2st3 scratch/g2st4 paper_1909_11985_b200 scratch/g2st8; do EDL_LIB_PATH=$PWD/$v/libedl_b200.so timeout 200 python scratch/gemm2_exp.py; done > gpurun_out/gemm2_exp.log 2>&1
cat gpurun_out/gemm2_exp.log
