timeout 3000 python tools/fuzz_parity.py 200 5000 > gpurun_out/r2_fuzz1.log 2>&1; echo fuzz1 rc=$?
timeout 1800 python tools/fuzz_parity.py 60 8000 big > gpurun_out/r2_fuzz3.log 2>&1; echo fuzz3 rc=$?
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_alt.json 2> gpurun_out/r2_bench_alt.err; echo bench rc=$?
