timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t24.log 2>&1; tail -2 gpurun_out/t24.log
echo c4; timeout 600 python tools/profile_pass.py c4 2e8 trie 3 2>&1 | grep -E "Gpts" | tail -1 | cut -c1-200
echo c4 old; RB_KERNEL=3 timeout 600 python tools/profile_pass.py c4 2e8 trie 3 2>&1 | grep -E "Gpts" | tail -1 | cut -c1-200
echo c2; timeout 120 python tools/profile_pass.py c2 1e8 trie 5 2>&1 | grep Gpts | tail -1
