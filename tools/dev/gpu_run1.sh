set -x
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./tools/peaks/peaks > gpurun_out/r02/peaks.json 2> gpurun_out/r02/peaks.err
cat gpurun_out/r02/peaks.json
timeout 1500 python -m pytest tests -m gpu -q -x -rA --durations=25 > gpurun_out/r02/pytest_gpu_run1.log 2>&1
echo pytest_rc=$?
tail -40 gpurun_out/r02/pytest_gpu_run1.log
