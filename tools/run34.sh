# A/B: ld.global.nc vs ld.global.nc.L1::no_allocate for the index lookups (C2 and C4)
bash tools/ab.sh build/ab/cur.so build/ab/noalloc.so
for lib in build/ab/cur.so build/ab/noalloc.so; do echo "== $lib C4"; RASTERBOUND_B200_LIB=$lib timeout 300 python tools/profile_pass.py c4 2e8 trie 3 | grep Gpts | tail -1; done
