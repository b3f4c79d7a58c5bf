export PYTHONUNBUFFERED=1
python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
python tools/profile_step.py --size 65536 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --size 65536 > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16|allreduce_sgd|xent|gather" -s 78 -c 26 -f -o gpurun_out/prof_full python tools/profile_step.py --size 65536 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
tail -2 gpurun_out/bench_full.log | cut -c1-600
