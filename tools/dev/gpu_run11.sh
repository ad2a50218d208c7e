mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -rA -k "observables or canonical or alternating or fixed_chi" > gpurun_out/r02/pytest_gpu_run11.log 2>&1
echo pytest_rc=$?
grep -E "PASSED|FAILED|ERROR|passed|failed|^E  .*Error|^E   |fixed chi" gpurun_out/r02/pytest_gpu_run11.log | head -40
timeout 900 python tools/ea_vs_fixed.py --config 3 > gpurun_out/r02/ea_vs_fixed_c3.json 2>&1; echo c3_rc=$?
tail -c 1500 gpurun_out/r02/ea_vs_fixed_c3.json
timeout 900 python tools/ea_vs_fixed.py --config 5 --depth 14 > gpurun_out/r02/ea_vs_fixed_c5.json 2>&1; echo c5_rc=$?
tail -c 600 gpurun_out/r02/ea_vs_fixed_c5.json
