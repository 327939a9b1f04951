for r in 1 2; do
  for c in 0 4 5; do
    RB_WARP_CFG=$c timeout 300 python tools/profile_pass.py c2 100000000 trie 5 2>&1 | grep Gpts | tail -1 | sed "s|^|cfg=$c |"
  done
done
RB_WARP_CFG=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "city or c1 or ring" 2>&1 | tail -2
