# round-1 evidence run (final state of session 3): bench lines, launch list, top-kernel capture, GPU suite
set -x
D=gpurun_out/r01e
mkdir -p $D
timeout 600 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1
timeout 300 python bench.py > $D/bench_default.jsonl 2> $D/bench_default.err
timeout 200 python bench.py --chi 16 --no-cpu-baseline > $D/bench_chi16.jsonl 2> $D/bench_chi16.err
timeout 600 python bench.py --chi 256 --steps 2 > $D/bench_chi256.jsonl 2> $D/bench_chi256.err
timeout 900 python bench.py --chi 1024 --count 32 --steps 1 --no-cpu-baseline --no-e2e > $D/bench_chi1024.jsonl 2> $D/bench_chi1024.err
EAMPS_TC_PROF=1 ORACLE=0 timeout 600 python tools/large_check.py 256 1 1024 > $D/tcprof_256.log 2>&1
EAMPS_TC_PROF=1 ORACLE=0 timeout 600 python tools/large_check.py 1024 1 16 > $D/tcprof_1024.log 2>&1
timeout 300 python bench.py --chi 64 --count 1024 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $D/plain64.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_chi64.csv python bench.py --chi 64 --count 1024 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_svd_qr|k_rayleigh|k_tc_polish|k_contract|k_reabsorb" -s 5 -c 5 -o $D/prof_chi64 python bench.py --chi 64 --count 1024 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la $D
