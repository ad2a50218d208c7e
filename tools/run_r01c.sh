# round-1 evidence run: bench lines (chi 16/64/256/1024), launch lists, ncu captures of the top kernels
set -x
D=gpurun_out/r01c
mkdir -p $D
python bench.py > $D/bench_default.jsonl 2> $D/bench_default.err
python bench.py --chi 16 --no-cpu-baseline > $D/bench_chi16.jsonl 2> $D/bench_chi16.err
python bench.py --chi 256 --steps 2 > $D/bench_chi256.jsonl 2> $D/bench_chi256.err
timeout 900 python bench.py --chi 1024 --count 32 --steps 1 --no-cpu-baseline --no-e2e > $D/bench_chi1024.jsonl 2> $D/bench_chi1024.err
python bench.py --chi 64 --count 1024 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $D/plain64.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_chi64.csv python bench.py --chi 64 --count 1024 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_svd_theta|k_svd_vrep" -s 6 -c 2 -o $D/prof_chi64 python bench.py --chi 64 --count 1024 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/large_check.py 256 64 > $D/plain_tc.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tc_" -s 60 -c 4 -o $D/prof_tc256 python tools/large_check.py 256 64 > /dev/null 2>&1
ls -la $D
