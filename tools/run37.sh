# C4 timing: cold-region sum RED as u64 (integer) instead of f64 (timing build; results wrong by design)
for r in 1 2; do for lib in build/ab/cur.so build/ab/intsum.so; do echo "== $lib $(RASTERBOUND_B200_LIB=$lib timeout 300 python tools/profile_pass.py c4 2e8 trie 3 2>&1 | grep Gpts | tail -1)"; done; done
