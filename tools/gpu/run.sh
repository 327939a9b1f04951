timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_packed.py -q -x 2>&1 | tail -3
for spec in "c2 trie -1" "c4 trie -1" "c4 packed -1"; do
  set -- $spec
  RB_BUILD_TRACE=1 timeout 600 python tools/build_time.py $1 $2 $3 5 2> gpurun_out/r2_build3_$1_$2.trace | tail -1
done
