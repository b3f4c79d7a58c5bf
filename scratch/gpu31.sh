export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_multigpu_gpu.py tests/test_elastic_multigpu_gpu.py -q -x 2>&1 | tail -1
for cfg in "2 148" "2 296" "2 74" "0 148"; do set -- $cfg; EDL_OVERLAP=$1 EDL_CE_UPDATE_BLOCKS=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu > gpurun_out/ce2_$1_$2.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/ce2_$1_$2.log').read().strip().splitlines()[-1]); print('N=2 overlap', $1, $2, round(d['value']), d['ms_per_step'], {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()})" || tail -5 gpurun_out/ce2_$1_$2.log; done
