mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
export EAMPS_DEBUG_SYNC=1
timeout 1700 python -m pytest tests -m gpu -q -rA --durations=12 > gpurun_out/r02/pytest_gpu_run9.log 2>&1
echo pytest_rc=$?
grep -E "FAILED|ERROR|passed|failed|^E  .*Error|eamps debug|worst" gpurun_out/r02/pytest_gpu_run9.log | head -40
