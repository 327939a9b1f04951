# fewer consumer warps (smaller tiles -> smaller carveout, more L1)
for r in 1 2; do for cfg in 0 4 5 6 7 8; do for c in 2 4; do
  echo "CFG=$cfg COPIES=$c $(RB_WARP_CFG=$cfg RB_HIST_COPIES=$c timeout 120 python tools/ablate.py 1e8 | grep c2 | tr -s ' ' | tr '\n' '|')"
done; done; done
