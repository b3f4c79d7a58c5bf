timeout 600 python bench.py --workload wide11264x8 --no-cpu > gpurun_out/wide_n1.json 2> gpurun_out/wide_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 2 --workload wide11264x8 > gpurun_out/wide_n2.json 2> gpurun_out/wide_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29536 bench.py --gpus 4 --workload wide11264x8 > gpurun_out/wide_n4.json 2> gpurun_out/wide_n4.err
tail -n 2 gpurun_out/wide_n*.err
