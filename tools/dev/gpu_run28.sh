# default bench line (all sub-records) after the r02 late optimisations
mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
timeout 1500 python bench.py > gpurun_out/r02/bench_default_run28.log 2>&1
echo rc=$?
tail -1 gpurun_out/r02/bench_default_run28.log > gpurun_out/r02/bench_default_run28.jsonl
tail -1 gpurun_out/r02/bench_default_run28.jsonl | python -c '
import json,sys; d=json.loads(sys.stdin.read())
print("chi64", d["value"], d["ms_per_step"], d["roofline"]["frac"], "e2e", d["e2e"]["value"], "clocks", d["clocks"])
for k,v in d.get("per_chi",{}).items(): print(k, v.get("value"), v.get("ms_per_step"), v.get("roofline",{}).get("frac"))
print("c5", d.get("config5_slice"))
print("cpu", d.get("cpu_baseline"))'
