for r in 1 2 3; do
  for lib in build/ab/lib_base.so build/ab/lib_u2.so; do
    RASTERBOUND_B200_LIB=$lib timeout 300 python tools/profile_pass.py c2 100000000 trie 5 2>&1 | grep Gpts | tail -1 | sed "s|^|$lib |"
  done
done
