timeout 600 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo rc=$?; tail -c 400 gpurun_out/bench_c1.json
