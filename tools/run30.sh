RB_WARP_CFG=7 RB_HIST_COPIES=4 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for r in 1 2; do for cfg in 0 1 7 8 9; do for c in 2 4; do
  echo "CFG=$cfg COPIES=$c $(RB_WARP_CFG=$cfg RB_HIST_COPIES=$c timeout 120 python tools/ablate.py 1e8 | grep c2 | tr -s ' ' | tr '\n' '|')"
done; done; done
