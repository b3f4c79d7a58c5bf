for v in v_lsu v_tma v_lsu_w4b2 v_lsu_w4b3s4 v_lsu_w8b2s3; do timeout 120 python scratch/sgd_variants.py scratch/$v/libedl_b200.so; done
