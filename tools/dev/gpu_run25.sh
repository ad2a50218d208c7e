# ncu --set full on k_pc_chol_cta (chi=64 default bench)
mkdir -p gpurun_out/r02
export PYTHONUNBUFFERED=1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-per-chi --config5-depth 0 --no-e2e"
$CMD > gpurun_out/r02/chol_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pc_chol_cta" -s 3 -c 1 -o gpurun_out/r02/prof_chol $CMD > gpurun_out/r02/chol_ncu.log 2>&1
echo rc=$?
tail -c 300 gpurun_out/r02/chol_ncu.log
