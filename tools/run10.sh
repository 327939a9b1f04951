for S in 7 8; do for cfg in 2; do echo S $S cfg $cfg; RB_HIST_COPIES=1 RB_SUMMARY_LEVEL=$S RB_WARP_CFG=$cfg timeout 120 python tools/profile_pass.py c2 1e8 trie 4 2>&1 | grep Gpts | tail -1; done; done
echo S 9 cfg 3; RB_HIST_COPIES=1 RB_SUMMARY_LEVEL=9 RB_WARP_CFG=3 timeout 120 python tools/profile_pass.py c2 1e8 trie 4 2>&1 | grep -E "Gpts|rror" | tail -2
