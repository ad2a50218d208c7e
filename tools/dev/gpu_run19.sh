mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
for c in 3 4 5; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-per-chi --config5-depth 0 --e2e-chunks $c > gpurun_out/r02/bench_e2e_g$c.log 2>&1
echo "geo chunks $c: $(tail -1 gpurun_out/r02/bench_e2e_g$c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"])')"
done
