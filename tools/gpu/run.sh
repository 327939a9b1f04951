for r in 1 2; do
  for ab in 0 1 8; do
    RB_DEEP_ABLATE=$ab timeout 300 python tools/profile_pass.py c4 200000000 trie 3 2>&1 | grep Gpts | tail -1 | sed "s|^|ablate=$ab |"
  done
done
