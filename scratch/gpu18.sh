export PYTHONUNBUFFERED=1
python -m pytest tests/test_gemm_gpu.py tests/test_job_gpu.py -q -x > gpurun_out/pf_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pf_pytest.log
for cfg in "0 0" "8 0" "0 1" "8 1" "4 1" "16 1" "8 2"; do
  set -- $cfg
  EDL_GEMM_PF_KB=$1 EDL_GEMM_PF_TILES=$2 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/pf_$1_$2.log 2>&1
  python - $1 $2 <<'P'
import json,sys
d=json.loads(open(f"gpurun_out/pf_{sys.argv[1]}_{sys.argv[2]}.log").read().strip().splitlines()[-1])
print(sys.argv[1:], round(d["value"]), round(d["ms_per_step"],4), {k: round(v*1e3,1) for k,v in d["phase_ms_per_step"].items()})
P
done
tail -1 gpurun_out/pf_pytest.log
