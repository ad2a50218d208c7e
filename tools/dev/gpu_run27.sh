# fused small-gate reabsorb (k_reabsorb_small): chi=16 A/B + full GPU suite
mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
B="python bench.py --chi 16 --steps 10 --warmup 3 --no-cpu-baseline --no-per-chi --config5-depth 0 --no-e2e"
for arm in fused tiled fused tiled; do
  if [ $arm = tiled ]; then export EAMPS_NO_REABSORB_SMALL=1; else unset EAMPS_NO_REABSORB_SMALL; fi
  timeout 300 $B > gpurun_out/r02/ab_rs_$arm.log 2>&1
  echo "$arm chi16: $(tail -1 gpurun_out/r02/ab_rs_$arm.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["phase_ms_per_step"]["reabsorb"], d["k_mean"], d["gpu_launches"])')"
done
unset EAMPS_NO_REABSORB_SMALL
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02/pytest_gpu_run27.log 2>&1
echo pytest_rc=$?
tail -3 gpurun_out/r02/pytest_gpu_run27.log
