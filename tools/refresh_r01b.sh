timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench_chi64.log 2>&1; tail -1 gpurun_out/bench_chi64.log | cut -c1-80
timeout 600 python bench.py --chi 256 --steps 2 > gpurun_out/bench_chi256.log 2>&1; tail -1 gpurun_out/bench_chi256.log | cut -c1-80
timeout 600 python bench.py --chi 1024 --count 32 --steps 1 > gpurun_out/bench_chi1024.log 2>&1; tail -1 gpurun_out/bench_chi1024.log | cut -c1-80
