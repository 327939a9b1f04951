timeout 1800 python tools/parity_full.py c4 gpurun_out/r2_parity_c4.jsonl > gpurun_out/r2_parity.log 2>&1; echo parity rc=$?
timeout 1800 python tools/sweep_c3.py 100000000 gpurun_out/r2_c3_sweep.jsonl > gpurun_out/r2_c3.log 2>&1; echo c3 rc=$?
