# C4: cost of the cold-region global REDs (ablation build) and of the hot-slot count
for lib in build/ab/cur.so build/ab/nocold.so; do for hk in 4095 1024; do echo "== $lib HOTK=$hk $(RB_HOT_K=$hk RASTERBOUND_B200_LIB=$lib timeout 300 python tools/profile_pass.py c4 2e8 trie 3 2>&1 | grep Gpts | tail -1)"; done; done
