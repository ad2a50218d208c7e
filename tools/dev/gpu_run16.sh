mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
for v in "X=1" "EAMPS_ROT_LEAN=1" "EAMPS_TC_GROUPS_ALL=1" "EAMPS_ROT_LEAN=1 EAMPS_TC_GROUPS_ALL=1"; do
  env $v timeout 600 python bench.py --chi 256 --count 4096 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-per-chi --config5-depth 0 > gpurun_out/r02/b16.jsonl 2>&1
  python -c "
import json
for l in open('gpurun_out/r02/b16.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print('[$v] chi256', round(d['value'],1), round(d['ms_per_step'],1), d['sweeps_mean'])
"
  env $v timeout 600 python bench.py --chi 1024 --count 128 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-per-chi --config5-depth 0 > gpurun_out/r02/b16.jsonl 2>&1
  python -c "
import json
for l in open('gpurun_out/r02/b16.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print('[$v] chi1024', round(d['value'],2), round(d['ms_per_step'],1), d['sweeps_mean'])
"
done
