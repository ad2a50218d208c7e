# usage: bash tools/ab_bench.sh "ENV1=.." "ENV2=.." ... ; one chi = 64 bench line per setting
# (value, sweeps, Jacobi ms, roofline frac); sub-records, e2e and the CPU baseline switched off
for e in "$@"; do
  env $e timeout 300 python bench.py --no-per-chi --config5-depth 0 --no-e2e --no-cpu-baseline > gpurun_out/ab.log 2>&1
  echo "$e: $(tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['sweeps_mean'],2), round(d['phase_ms_per_step']['svd_jacobi'],2), round(d['roofline']['frac'],3))")"
done
