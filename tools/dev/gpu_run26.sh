# parallel L_JJ inverse + one-barrier LDL^H diagonal factorisation in the Cholesky kernels
mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-per-chi --config5-depth 0 --no-e2e > gpurun_out/r02/chol2_64.log 2>&1
tail -1 gpurun_out/r02/chol2_64.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["phase_ms_per_step"]["svd_precond"], d["phase_ms_per_step"]["svd_spectrum"], d["sweeps_mean"])'
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02/pytest_gpu_run26.log 2>&1
echo pytest_rc=$?
tail -3 gpurun_out/r02/pytest_gpu_run26.log
