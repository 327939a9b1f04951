timeout 3000 python tools/fuzz_parity.py 200 70000 > gpurun_out/r2_fuzz5.log 2>&1; echo fuzz5 rc=$?
