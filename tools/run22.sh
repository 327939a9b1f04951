timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t26.log 2>&1; tail -2 gpurun_out/t26.log
timeout 300 python tools/ablate.py 1e8
for i in 1 2; do timeout 120 python tools/profile_pass.py c2 1e8 trie 5 2>&1 | grep Gpts | tail -1; done
