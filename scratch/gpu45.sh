export PYTHONUNBUFFERED=1
unset EDL_OVERLAP
for cfg in "3 592 1" "3 296 1" "3 1184 1" "3 592 0"; do set -- $cfg; EDL_OVERLAP=$1 EDL_COLL_BLOCKS=$2 EDL_PDL=$3 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu > gpurun_out/rsv.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/rsv.log').read().strip().splitlines()[-1]); print('N=2 $cfg', round(d['value']), round(d['ms_per_step'],4), {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()})" || tail -5 gpurun_out/rsv.log; done
