for spec in "c4 trie -1" "c4 packed -1" "c2 trie -1"; do
  set -- $spec
  RB_BUILD_TRACE=1 timeout 600 python tools/build_time.py $1 $2 $3 6 2> gpurun_out/r2_build4_$1_$2.trace | tail -1
done
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_packed.py -q -x 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r2_bench_pin.json 2> gpurun_out/r2_bench_pin.err; echo bench rc=$?
