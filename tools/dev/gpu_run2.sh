mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q -x -rA --durations=25 --deselect tests/test_gpu_configs_prefix.py --deselect tests/test_gpu_edge.py --deselect tests/test_gpu_fullsize.py > gpurun_out/r02/pytest_gpu_run2.log 2>&1
echo pytest_rc=$?
tail -30 gpurun_out/r02/pytest_gpu_run2.log
timeout 900 python bench.py > gpurun_out/r02/bench_run2.jsonl 2> gpurun_out/r02/bench_run2.err
echo bench_rc=$?
tail -5 gpurun_out/r02/bench_run2.err
