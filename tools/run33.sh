# deep kernel: ring depth x hot-slot copies x hot-slot count (C4, 200M points)
run() { echo "CFG=$1 COPIES=$2 HOTK=$3 $(RB_DEEP_CFG=$1 RB_DEEP_COPIES=$2 RB_HOT_K=$3 timeout 240 python tools/profile_pass.py c4 2e8 trie 3 2>&1 | grep Gpts | tail -1)"; }
for hk in 4095 2048 1024; do for cfg in 1 2; do for c in 1 2; do run $cfg $c $hk; done; done; done
run 0 1 4095; run 0 1 2048
