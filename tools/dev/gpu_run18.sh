mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
timeout 600 python tools/dev/e2e_overlap.py > gpurun_out/r02/e2e_overlap2.log 2>&1
echo rc=$?
cat gpurun_out/r02/e2e_overlap2.log | grep "C="
for c in 1 2 4; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-per-chi --config5-depth 0 --e2e-chunks $c > gpurun_out/r02/bench_e2e_c$c.log 2>&1
echo "chunks $c: $(tail -1 gpurun_out/r02/bench_e2e_c$c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"])')"
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02/pytest_gpu_run18.log 2>&1
echo pytest_rc=$?
tail -3 gpurun_out/r02/pytest_gpu_run18.log
