mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
timeout 1700 python -m pytest tests -m gpu -q -rA --durations=12 > gpurun_out/r02/pytest_gpu_run10.log 2>&1
echo pytest_rc=$?
grep -E "FAILED|ERROR|passed|failed|xfail|^E  .*Error|worst" gpurun_out/r02/pytest_gpu_run10.log | head -30
timeout 1200 python bench.py > gpurun_out/r02/bench_run10.jsonl 2> gpurun_out/r02/bench_run10.err
echo bench_rc=$?
tail -3 gpurun_out/r02/bench_run10.err
python - <<'PY'
import json
for l in open("gpurun_out/r02/bench_run10.jsonl"):
    if l.startswith("{"):
        d=json.loads(l)
        print("headline", d["value"], d["ms_per_step"], d["roofline"]["frac"], d.get("e2e",{}).get("value"))
        for k,v in d.get("per_chi",{}).items(): print(k, v.get("value"), v.get("ms_per_step"), v.get("roofline",{}).get("frac"), v.get("error"))
        print("c5", json.dumps(d.get("config5_slice"))[:600])
        print("cpu", d.get("cpu_baseline"))
PY
