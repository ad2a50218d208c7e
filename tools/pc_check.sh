timeout 300 python tools/large_check.py 256 2 > gpurun_out/pc256.log 2>&1; tail -4 gpurun_out/pc256.log
timeout 300 python tools/large_check.py 128 2 > gpurun_out/pc128.log 2>&1; tail -3 gpurun_out/pc128.log
EAMPS_TC_PROF=1 ORACLE=0 timeout 300 python tools/large_check.py 256 1 1024 > gpurun_out/pc256t.log 2>&1; grep -v "^ *$" gpurun_out/pc256t.log | tail -4
EAMPS_TC_PROF=1 ORACLE=0 timeout 300 python tools/large_check.py 1024 1 16 > gpurun_out/pc1024t.log 2>&1; tail -4 gpurun_out/pc1024t.log
