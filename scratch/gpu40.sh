export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_multigpu_gpu.py -q -x 2>&1 | tail -1
for cfg in "1 592" "2 592" "4 592" "2 1184" "1 1184" "2 296"; do set -- $cfg; EDL_COLL_UNROLL=$1 EDL_COLL_BLOCKS=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu > gpurun_out/coll_$1_$2.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/coll_$1_$2.log').read().strip().splitlines()[-1]); print('N=2 unroll', $1, 'blocks', $2, round(d['value']), round(d['ms_per_step'],4), 'update', round(d['phase_ms_per_step']['update']*1e3,1), 'GB/s', round(d['update_roofline']['achieved']))" || tail -3 gpurun_out/coll_$1_$2.log; done
