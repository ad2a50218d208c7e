# A/B of large-regime settings: svd_blocked phase per layer (ms) at chi=256 x1024 and chi=1024 x16
for e in "$@"; do
  for cfg in "256 1 1024" "1024 1 16"; do
    env $e ORACLE=0 timeout 300 python tools/large_check.py $cfg > gpurun_out/abl.log 2>&1
    echo "$e chi=${cfg%% *}: $(grep -o "'svd_blocked': ([0-9.]*" gpurun_out/abl.log | tail -1) sweeps $(grep -o 'sweeps mean [0-9.]*' gpurun_out/abl.log | tail -1)"
  done
done
