mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -rA -k "graded or layer_parity or tensor_core or chi256_blocked or ragged or fullsize or sharded or chi1024" > gpurun_out/r02/pytest_gpu_run5.log 2>&1
echo pytest_rc=$?
grep -E "PASSED|FAILED|ERROR|passed|failed|^E  .*Error|worst" gpurun_out/r02/pytest_gpu_run5.log | tail -60
timeout 300 python tools/dev/spec_dump.py g62 g64 g128 g16
for v in "EAMPS_TC_BATCH=0" ""; do
  env $v timeout 600 python bench.py --chi 256 --count 4096 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-per-chi --config5-depth 0 > gpurun_out/r02/b5.jsonl 2>&1
  python -c "
import json
for l in open('gpurun_out/r02/b5.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print('$v chi256', d['value'], d['ms_per_step'], d['phase_ms_per_step'])
"
done
timeout 600 python bench.py --chi 1024 --count 128 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-per-chi --config5-depth 0 > gpurun_out/r02/b5.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/r02/b5.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print('chi1024', d['value'], d['ms_per_step'], d['phase_ms_per_step'])
"
