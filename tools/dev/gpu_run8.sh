mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
export EAMPS_DEBUG_SYNC=1
timeout 900 python -m pytest tests -m gpu -q -x -rA -k "config3_deep or config4_every or config5_every" > gpurun_out/r02/pytest_gpu_run8.log 2>&1
echo pytest_rc=$?
grep -E "PASSED|FAILED|passed|failed|^E  .*Error|eamps debug" gpurun_out/r02/pytest_gpu_run8.log | head -30
unset EAMPS_DEBUG_SYNC
timeout 600 python tools/dev/c4_gate.py 2>&1 | tail -20
