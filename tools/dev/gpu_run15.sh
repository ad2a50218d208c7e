mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/r02/pytest_gpu_run15.log 2>&1
echo pytest_rc=$?
grep -E "FAILED|ERROR|passed|failed|xfail|^E  .*Error" gpurun_out/r02/pytest_gpu_run15.log | head -20
timeout 1500 python tools/run_sharded.py --depth 23 --progress --slab-gb 160 > gpurun_out/r02/config5_depth23_1gpu.log 2>&1
echo c5_rc=$?
tail -8 gpurun_out/r02/config5_depth23_1gpu.log
