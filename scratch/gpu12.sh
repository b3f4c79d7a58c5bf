export PYTHONUNBUFFERED=1
timeout 300 python tools/profile_step.py --size 65536 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --size 65536 > gpurun_out/ncu_launch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16|allreduce_sgd|xent|gather" -s 78 -c 26 -o gpurun_out/prof_full python tools/profile_step.py --size 65536 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
timeout 400 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 1200 gpurun_out/bench_ref.log
nproc; lscpu | grep -E "Model name|^CPU\(s\)"
