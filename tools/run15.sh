for A in 0 1 2 3 6 7; do echo ablate $A; RB_ABLATE=$A RB_WARP_CFG=1 timeout 120 python tools/profile_pass.py c2 1e8 trie 4 2>&1 | grep Gpts | tail -1; done
