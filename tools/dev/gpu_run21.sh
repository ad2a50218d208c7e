# host-side time of the layer path (EAMPS_HOST_PROF) at chi = 16 and 64
mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1 EAMPS_HOST_PROF=1
for c in 16 64; do
timeout 300 python bench.py --chi $c --steps 10 --warmup 3 --no-cpu-baseline --no-per-chi --config5-depth 0 --no-e2e > gpurun_out/r02/hostprof_$c.log 2>&1
grep "eamps host" gpurun_out/r02/hostprof_$c.log
tail -1 gpurun_out/r02/hostprof_$c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["phase_ms_per_step"], d["gpu_launches"])'
done
