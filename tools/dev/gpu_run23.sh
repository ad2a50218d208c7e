# pair-planar small-regime kernel: chi=16 bench + full GPU suite
mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
timeout 300 python bench.py --chi 16 --steps 10 --warmup 3 --no-cpu-baseline --no-per-chi --config5-depth 0 --no-e2e > gpurun_out/r02/planar16.log 2>&1
tail -1 gpurun_out/r02/planar16.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["phase_ms_per_step"]["svd_small"], d["roofline"]["frac"], d["sweeps_mean"])'
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02/pytest_gpu_run23.log 2>&1
echo pytest_rc=$?
tail -3 gpurun_out/r02/pytest_gpu_run23.log
