for A in 0 1 2 3; do echo ablate $A; RB_ABLATE=$A timeout 600 python tools/profile_pass.py c4 2e8 trie 3 11 8 2>&1 | grep -E "Gpts" | tail -1 | cut -c1-200; done
