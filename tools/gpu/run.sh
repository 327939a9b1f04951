timeout 2400 python tools/fuzz_parity.py 150 5000 > gpurun_out/r2_fuzz1.log 2>&1; echo fuzz1 rc=$?
timeout 1800 python tools/fuzz_parity.py 40 7000 big > gpurun_out/r2_fuzz2.log 2>&1; echo fuzz2 rc=$?
tail -2 gpurun_out/r2_fuzz1.log gpurun_out/r2_fuzz2.log
