# ring depth vs histogram copies (C2 SUM)
for cfg in "0 2" "0 1" "1 8" "1 4" "1 2"; do set -- $cfg; echo "CFG=$1 COPIES=$2"; RB_WARP_CFG=$1 RB_HIST_COPIES=$2 timeout 300 python tools/ablate.py 1e8 | grep "c2 *SUM"; done
for cfg in "0 2" "1 8"; do set -- $cfg; echo "CFG=$1 COPIES=$2"; RB_WARP_CFG=$1 RB_HIST_COPIES=$2 timeout 300 python tools/ablate.py 1e8 | grep "c2 *SUM"; done
