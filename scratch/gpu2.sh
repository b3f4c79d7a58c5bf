timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python tools/profile_step.py --size 65536 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --size 65536 > gpurun_out/ncu_launch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16|allreduce_sgd|xent|gather" -s 78 -c 26 -o gpurun_out/prof_full python tools/profile_step.py --size 65536 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
tail -5 gpurun_out/pytest_gpu.log; tail -c 2500 gpurun_out/bench.log
