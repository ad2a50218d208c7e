mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x -rA -k "tensor_core or chi256_blocked or ragged or fullsize or boundary_gates" > gpurun_out/r02/pytest_gpu_run4.log 2>&1
echo pytest_rc=$?
grep -E "PASSED|FAILED|ERROR|passed|failed|^E " gpurun_out/r02/pytest_gpu_run4.log | tail -30
for v in "" "EAMPS_NO_POLISH=1" ; do echo "== variant [$v]"; env $v timeout 300 python tools/dev/spec_dump.py g62 g64 g128 g16 c256; done
echo "== bench fused chi256/1024"
timeout 600 python bench.py --chi 256 --count 4096 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-per-chi --config5-depth 0 > gpurun_out/r02/bench_fused_chi256.jsonl 2>&1; echo rc=$?
timeout 600 python bench.py --chi 1024 --count 128 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-per-chi --config5-depth 0 > gpurun_out/r02/bench_fused_chi1024.jsonl 2>&1; echo rc=$?
EAMPS_TC_UNFUSED=1 timeout 600 python bench.py --chi 256 --count 4096 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-per-chi --config5-depth 0 > gpurun_out/r02/bench_unfused_chi256.jsonl 2>&1; echo rc=$?
python - <<'PY'
import json
for f in ["bench_fused_chi256","bench_fused_chi1024","bench_unfused_chi256"]:
    try:
        for l in open("gpurun_out/r02/%s.jsonl"%f):
            if l.startswith("{"):
                d=json.loads(l); print(f, d["value"], d["ms_per_step"], d["sweeps_mean"], d["phase_ms_per_step"].get("svd_blocked"), d["roofline"]["frac"])
    except Exception as e: print(f, "ERR", e)
PY
tail -5 gpurun_out/r02/bench_fused_chi256.jsonl
