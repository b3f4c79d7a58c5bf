export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python tools/elastic_bench.py --gpus 4 > gpurun_out/elastic.log 2>&1; echo "elastic rc=$?"; tail -1 gpurun_out/elastic.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for e in d['events']: print(e['kind'], e['ids'], 'stall', round(e['stall_ms'],3), 'before', round(e['step_ms_before'],3), 'after', round(e['step_ms_after'],3), 'switch', round(e['switch_step_ms'],3))
print('stop-resume', d['stop_resume_1_to_2']['stall_ms'], 'coverage', d['coverage_ok'])"
