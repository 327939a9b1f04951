timeout 3500 python tools/fuzz_parity.py 600 90000 > gpurun_out/r2_fuzz7.log 2>&1; echo fuzz7 rc=$?
timeout 2000 python tools/fuzz_parity.py 100 95000 big > gpurun_out/r2_fuzz8.log 2>&1; echo fuzz8 rc=$?
