timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t8.log 2>&1; tail -2 gpurun_out/t8.log
timeout 300 python tools/ablate.py 1e8
for cfg in 1 3; do echo cfg $cfg; RB_WARP_CFG=$cfg timeout 120 python tools/profile_pass.py c2 1e8 trie 4 2>&1 | grep Gpts | tail -1; done
