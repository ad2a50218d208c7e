mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
for c in 1 2 4 8; do
  timeout 600 python bench.py --steps 3 --warmup 3 --e2e-chunks $c --no-cpu-baseline --no-per-chi --config5-depth 0 > gpurun_out/r02/b14.jsonl 2>gpurun_out/r02/b14.err
  python -c "
import json
for l in open('gpurun_out/r02/b14.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print('chunks $c value', round(d['value']), 'e2e', round(d['e2e']['value']))
"
  tail -2 gpurun_out/r02/b14.err
done
