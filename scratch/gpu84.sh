export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_straggler_gpu.py tests/test_elastic_multigpu_gpu.py -q -x 2>&1 | tail -3
timeout 900 python tools/elastic_bench.py --gpus 4 > gpurun_out/elastic.log 2>&1; echo "elastic rc=$?"; tail -1 gpurun_out/elastic.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for e in d['events']: print(e['kind'], e.get('ids', e.get('straggler')), 'stall', round(e['stall_ms'],3), 'before', round(e['step_ms_before'],3), 'after', round(e['step_ms_after'],3), {k: e[k] for k in ('slow_minibatches_to_detection','ring') if k in e})
print('stop-resume', d['stop_resume_1_to_2']['stall_ms'], 'coverage', d['coverage_ok'], d['ring_final'])" || tail -20 gpurun_out/elastic.log
