# ncu launch list of the default bench step (chi = 64 x 4096; eamps kernels only), with per-launch DRAM
# bytes. The per-chi sub-records and the config-5 slice are switched off so that the un-profiled
# pre-run gpurun makes of the same command ends inside its 300 s limit.
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"^k_" --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  --no-per-chi --config5-depth 0 --no-e2e > gpurun_out/ncu_default.log 2>&1
tail -c 300 gpurun_out/ncu_default.log
