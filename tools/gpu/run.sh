for r in 1 2; do
for lib in build/ab/head.so build/ab/reorder.so; do
  RASTERBOUND_B200_LIB=$lib timeout 300 python tools/profile_pass.py c4 200000000 trie 3 12 2>&1 | grep Gpts | tail -1 | sed "s|^|$lib cfg0 |"
done
RB_DEEP_CFG=3 RASTERBOUND_B200_LIB=build/ab/reorder.so timeout 300 python tools/profile_pass.py c4 200000000 trie 3 12 2>&1 | grep Gpts | tail -1 | sed "s|^|reorder cfg3 |"
for lib in build/ab/head.so build/ab/reorder.so; do
  RASTERBOUND_B200_LIB=$lib timeout 300 python tools/profile_pass.py c4 200000000 packed 3 12 2>&1 | grep Gpts | tail -1 | sed "s|^|$lib PKL |"
done
done
