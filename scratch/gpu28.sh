export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/seg_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/seg_pytest.log; tail -2 gpurun_out/seg_pytest.log
EDL_OVERLAP=1 timeout 900 python -m pytest tests/test_elastic_multigpu_gpu.py tests/test_multigpu_gpu.py tests/test_job_gpu.py -q -x > gpurun_out/seg_pytest_ov.log 2>&1; echo "rc=$?" >> gpurun_out/seg_pytest_ov.log; tail -2 gpurun_out/seg_pytest_ov.log
for cfg in "0 148" "1 148" "1 296" "1 592"; do set -- $cfg; EDL_OVERLAP=$1 EDL_OVERLAP_BLOCKS=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu > gpurun_out/ov2_$1_$2.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/ov2_$1_$2.log').read().strip().splitlines()[-1]); print('N=2 overlap', $1, $2, round(d['value']), d['ms_per_step'], {k: round(v*1e3,1) for k,v in d['phase_ms_per_step'].items()})"; done
