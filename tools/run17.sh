for cfg in 0 2 3; do echo cfg $cfg; RB_WARP_CFG=$cfg timeout 120 python tools/profile_pass.py c2 1e8 trie 5 2>&1 | grep Gpts | tail -1; done
