timeout 900 python -m pytest tests/test_gpu_packed.py -q -x 2>&1 | tail -2
timeout 3000 python tools/fuzz_parity.py 250 5000 > gpurun_out/r2_fuzz1.log 2>&1; echo fuzz1 rc=$?
timeout 3000 python tools/fuzz_parity.py 250 30000 > gpurun_out/r2_fuzz4.log 2>&1; echo fuzz4 rc=$?
