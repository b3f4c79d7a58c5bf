timeout 900 python -m pytest tests/test_multigpu_gpu.py tests/test_elastic_multigpu_gpu.py tests/test_job_gpu.py -x -q > gpurun_out/pytest_mg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mg.log
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
tail -n 3 gpurun_out/pytest_mg.log; cat gpurun_out/bench_n1.json gpurun_out/bench_n2.json gpurun_out/bench_n4.json
