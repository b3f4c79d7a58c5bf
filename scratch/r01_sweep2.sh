run() { env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29537 bench.py --gpus 2 --no-cpu --no-nccl 2>/dev/null | tail -n 1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value']), d['wgrad_ms_per_step'], d['phase_ms_per_step'])"; }
run X=0
run EDL_GEMM_MC=0
run EDL_GEMM_PF_KB=0
run EDL_GEMM_PF_KB=4
run EDL_GEMM_PF_KB=16
run EDL_PDL=0
