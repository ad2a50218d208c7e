set -x
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench_chi64.log 2>&1; tail -1 gpurun_out/bench_chi64.log | cut -c1-200
timeout 400 python bench.py --chi 16 > gpurun_out/bench_chi16.log 2>&1; tail -1 gpurun_out/bench_chi16.log | cut -c1-200
timeout 600 python bench.py --chi 256 --steps 2 > gpurun_out/bench_chi256.log 2>&1; tail -1 gpurun_out/bench_chi256.log | cut -c1-200
timeout 600 python bench.py --chi 1024 --count 32 --steps 1 > gpurun_out/bench_chi1024.log 2>&1; tail -1 gpurun_out/bench_chi1024.log | cut -c1-200
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv --log-file gpurun_out/launches_chi64.csv python bench.py --count 1024 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; tail -c 300 gpurun_out/ncu_l.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_svd_qr -c 1 -o gpurun_out/qr_final python bench.py --count 1024 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_qr.log 2>&1; tail -c 200 gpurun_out/ncu_qr.log
