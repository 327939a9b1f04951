timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/r2_bench_final2.json 2> gpurun_out/r2_bench_final2.err; echo bench rc=$?
timeout 900 python bench.py --config c2 > gpurun_out/r2_bench_c2_final.json 2> gpurun_out/r2_bench_c2_final.err; echo bench c2 rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; echo ref rc=$?
