mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=15 -k "graded or layer_parity or sharded or chi1024 or ragged" > gpurun_out/r02/pytest_gpu_run3.log 2>&1
echo pytest_rc=$?
grep -E "PASSED|FAILED|ERROR|worst|passed|failed" gpurun_out/r02/pytest_gpu_run3.log | tail -60
