# warp match_any aggregation of the histogram updates (RB_MATCH_AGG build) vs bank-staggered copies
for r in 1 2; do
  echo "== cur C4 $(RASTERBOUND_B200_LIB=build/ab/cur.so timeout 300 python tools/ablate.py 1e8 | grep c2 | tr -s ' ' | tr '\n' '|')"
  echo "== match C4 $(RASTERBOUND_B200_LIB=build/ab/match.so timeout 300 python tools/ablate.py 1e8 | grep c2 | tr -s ' ' | tr '\n' '|')"
  echo "== match C1 $(RB_HIST_COPIES=1 RASTERBOUND_B200_LIB=build/ab/match.so timeout 300 python tools/ablate.py 1e8 | grep c2 | tr -s ' ' | tr '\n' '|')"
done
RASTERBOUND_B200_LIB=build/ab/match.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "city or single_hot or drains" 2>&1 | tail -1
