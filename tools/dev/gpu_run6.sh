mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -rA -k "graded or layer_parity or tensor_core or chi256_blocked or ragged or chi1024" > gpurun_out/r02/pytest_gpu_run6.log 2>&1
echo pytest_rc=$?
grep -E "PASSED|FAILED|ERROR|passed|failed|^E  .*Error|worst" gpurun_out/r02/pytest_gpu_run6.log | tail -60
timeout 600 python bench.py --chi 1024 --count 128 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-per-chi --config5-depth 0 > gpurun_out/r02/b6.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/r02/b6.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print('chi1024', d['value'], d['ms_per_step'], d['sweeps_mean'], d['phase_ms_per_step'])
"
timeout 600 python bench.py --chi 256 --count 4096 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-per-chi --config5-depth 0 > gpurun_out/r02/b6.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/r02/b6.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print('chi256', d['value'], d['ms_per_step'], d['sweeps_mean'], d['phase_ms_per_step'])
"
