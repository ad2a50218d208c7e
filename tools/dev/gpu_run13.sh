mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -x -rA -k "graded or ragged or fullsize or config2_micro or layer_parity or mixed_wave or multiwave" > gpurun_out/r02/pytest_gpu_run13.log 2>&1
echo pytest_rc=$?
grep -E "FAILED|ERROR|passed|failed|^E  .*Error|^E   " gpurun_out/r02/pytest_gpu_run13.log | head -20
for v in "EAMPS_PC_UNFUSED=1" ""; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-per-chi --config5-depth 0 > gpurun_out/r02/b13.jsonl 2>&1
  python -c "
import json
for l in open('gpurun_out/r02/b13.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); p=d['phase_ms_per_step']; print('[$v]', round(d['value']), round(d['ms_per_step'],2), 'precond', round(p['svd_precond'],2), 'jacobi', round(p['svd_jacobi'],2), 'spec', round(p['svd_spectrum'],2), 'frac', round(d['roofline']['frac'],3))
"
done
