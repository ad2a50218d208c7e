# ncu launch list of the default bench command (eamps kernels only), with per-launch DRAM bytes
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"^k_" --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_default.log 2>&1
tail -c 300 gpurun_out/ncu_default.log
