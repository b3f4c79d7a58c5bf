for v in v_w8b1 v_w4b3s3p1 v_w4b3s3p2 v_w4b2s5 v_w8b1s3; do timeout 120 python scratch/sgd_variants.py scratch/$v/libedl_b200.so; done
