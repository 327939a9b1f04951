# ring configuration x histogram copies x summary level (C2); L1 share check via RB_CARVEOUT
for S in 7 6; do for cfg in 0 1 2 3 4 5 6; do for c in 2 4 8; do
  echo "S=$S CFG=$cfg COPIES=$c $(RB_SUMMARY_LEVEL=$S RB_WARP_CFG=$cfg RB_HIST_COPIES=$c timeout 120 python tools/ablate.py 1e8 | grep c2 | tr -s ' ' | tr '\n' '|')"
done; done; done
echo "carveout 100: $(RB_CARVEOUT=100 RB_WARP_CFG=1 RB_HIST_COPIES=4 timeout 120 python tools/ablate.py 1e8 | grep c2 | tr -s ' ' | tr '\n' '|')"
