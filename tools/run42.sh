# C4: cold-region count and sum REDs in one 16-byte pair (RB_COLD_PAIR timing build) vs separate arrays
for r in 1 2; do for lib in build/ab/cur.so build/ab/pair.so; do echo "== $lib $(RASTERBOUND_B200_LIB=$lib timeout 300 python tools/profile_pass.py c4 2e8 trie 3 2>&1 | grep Gpts | tail -1)"; done; done
