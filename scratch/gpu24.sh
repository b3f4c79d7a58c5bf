for bn in 128 256; do echo "SGD_BN=$bn"; EDL_SGD_BN=$bn python scratch/trace_sgd2.py; done
