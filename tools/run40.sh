# summary through L1 (global memory) instead of shared memory: frees 32 KB -> 164 KB carveout step
for r in 1 2; do
  echo "== cur $(RASTERBOUND_B200_LIB=build/ab/cur.so timeout 300 python tools/ablate.py 1e8 | grep c2 | tr -s ' ' | tr '\n' '|')"
  echo "== summg S7 $(RASTERBOUND_B200_LIB=build/ab/summg.so timeout 300 python tools/ablate.py 1e8 | grep c2 | tr -s ' ' | tr '\n' '|')"
  echo "== summg S8 $(RB_SUMMARY_LEVEL=8 RASTERBOUND_B200_LIB=build/ab/summg.so timeout 300 python tools/ablate.py 1e8 | grep c2 | tr -s ' ' | tr '\n' '|')"
done
RASTERBOUND_B200_LIB=build/ab/summg.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "city or c1_full" 2>&1 | tail -1
