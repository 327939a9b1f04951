timeout 3000 python tools/fuzz_parity.py 200 70000 > gpurun_out/r2_fuzz5.log 2>&1; echo fuzz5 rc=$?
timeout 3000 python tools/fuzz_parity.py 60 80000 big > gpurun_out/r2_fuzz6.log 2>&1; echo fuzz6 rc=$?
