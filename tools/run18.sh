timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t18.log 2>&1; tail -2 gpurun_out/t18.log
timeout 300 python tools/ablate.py 1e8
for cfg in 0 1; do echo cfg $cfg; RB_WARP_CFG=$cfg timeout 120 python tools/profile_pass.py c2 1e8 trie 5 2>&1 | grep Gpts | tail -1; done
echo c4; timeout 600 python tools/profile_pass.py c4 2e8 trie 3 11 8 2>&1 | grep -E "Gpts" | tail -1 | cut -c1-200
