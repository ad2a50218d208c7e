mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
CMD="python bench.py --chi 16 --steps 1 --warmup 3 --no-cpu-baseline --no-per-chi --config5-depth 0 --no-e2e"
$CMD > gpurun_out/r02/ncu16_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_svd_small" -s 3 -c 1 -o gpurun_out/r02/prof_svd_small16 $CMD > gpurun_out/r02/ncu16_full.log 2>&1
echo rc=$?
tail -c 300 gpurun_out/r02/ncu16_full.log
$CMD > gpurun_out/r02/ncu16_plain2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^k_" --csv --log-file gpurun_out/r02/launches_chi16.csv $CMD > gpurun_out/r02/ncu16_launch.log 2>&1
echo rc2=$?
