# A/B: scaled (square-root-free-update) rotations in the chi=64 block-recursive Jacobi (EAMPS_QR_SCALED)
mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-per-chi --config5-depth 0 --no-e2e"
for arm in base scaled base scaled; do
  if [ $arm = scaled ]; then export EAMPS_QR_SCALED=1; else unset EAMPS_QR_SCALED; fi
  timeout 300 $B > gpurun_out/r02/ab_scaled_$arm.log 2>&1
  echo "$arm chi64: $(tail -1 gpurun_out/r02/ab_scaled_$arm.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["sweeps_mean"], d["phase_ms_per_step"]["svd_jacobi"])')"
done
export EAMPS_QR_SCALED=1
timeout 900 python -m pytest tests -m gpu -q -x -k "parity or edge or fullsize or layer" > gpurun_out/r02/pytest_scaled.log 2>&1
echo pytest_rc=$?
tail -3 gpurun_out/r02/pytest_scaled.log
