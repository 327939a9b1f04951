# C4 deep kernel: root level x node split (RB_NODE_KS), 200M points
run() { echo "T0=$1 KS=$2 $(RB_NODE_KS=$2 timeout 240 python tools/profile_pass.py c4 2e8 trie 3 $1 8 2>&1 | grep -E 'Gpts|Error' | tail -1)"; }
run 11 3,4; run 11 2,5; run 11 4,3; run 11 1,6
run 12 2,4; run 12 3,3; run 12 1,5
run 10 4,4; run 10 3,5; run 10 2,6
run 13 2,3; run 13 1,4
