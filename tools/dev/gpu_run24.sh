# A/B: QR-regime Rayleigh from L^H V (default) vs theta V (EAMPS_RAYLEIGH_THETA=1); parity subset
mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-per-chi --config5-depth 0 --no-e2e"
for arm in L theta L theta; do
  if [ $arm = theta ]; then export EAMPS_RAYLEIGH_THETA=1; else unset EAMPS_RAYLEIGH_THETA; fi
  timeout 300 $B > gpurun_out/r02/ab_ray_$arm.log 2>&1
  echo "$arm chi64: $(tail -1 gpurun_out/r02/ab_ray_$arm.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["phase_ms_per_step"]["svd_spectrum"], d["sweeps_mean"], d["k_mean"])')"
done
unset EAMPS_RAYLEIGH_THETA
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02/pytest_gpu_run24.log 2>&1
echo pytest_rc=$?
tail -3 gpurun_out/r02/pytest_gpu_run24.log
