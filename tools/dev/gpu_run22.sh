mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
bash tools/dev/gpu_run21.sh
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02/pytest_gpu_run22.log 2>&1
echo pytest_rc=$?
tail -3 gpurun_out/r02/pytest_gpu_run22.log
