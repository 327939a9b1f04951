for T in 9 10 11 12; do echo T0 $T; timeout 120 python tools/profile_pass.py c2 1e8 trie 5 $T 8 2>&1 | grep Gpts | tail -1; done
echo T0 12 rw 4; timeout 120 python tools/profile_pass.py c2 1e8 trie 5 12 4 2>&1 | grep Gpts | tail -1
