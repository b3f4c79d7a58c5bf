export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt4b.log 2>&1; echo rc=$? >> gpurun_out/pt4b.log
E="timeout 300 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29571"
$E --nproc-per-node 4 tools/mp_elastic_bench.py > gpurun_out/mpel4.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 $E --nproc-per-node 2 tools/mp_elastic_bench.py > gpurun_out/mpel2.log 2>&1
