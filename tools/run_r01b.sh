set -x
mkdir -p gpurun_out/r01b
python bench.py --chi 64 > gpurun_out/r01b/bench_chi64.jsonl 2> gpurun_out/r01b/bench_chi64.err
python bench.py --chi 16 --no-cpu-baseline > gpurun_out/r01b/bench_chi16.jsonl 2> gpurun_out/r01b/bench_chi16.err
python bench.py --chi 256 --steps 2 --no-cpu-baseline > gpurun_out/r01b/bench_chi256.jsonl 2> gpurun_out/r01b/bench_chi256.err
timeout 900 python bench.py --chi 1024 --count 32 --steps 1 --no-cpu-baseline --no-e2e > gpurun_out/r01b/bench_chi1024.jsonl 2> gpurun_out/r01b/bench_chi1024.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01b/launches_chi64.csv python bench.py --chi 64 --count 1024 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_svd_theta|k_svd_vrep" -s 6 -c 2 -o gpurun_out/r01b/prof_chi64 python bench.py --chi 64 --count 1024 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_tc_" -s 60 -c 3 -o gpurun_out/r01b/prof_tc256 python tools/large_check.py 256 64 > /dev/null 2>&1
ls -la gpurun_out/r01b
