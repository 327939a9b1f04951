timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t6.log 2>&1; tail -2 gpurun_out/t6.log
timeout 300 python tools/ablate.py 1e8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_point_pass_ring -s 1 -c 1 -o gpurun_out/prof_w6 python tools/profile_pass.py c2 1e8 trie 1 > gpurun_out/ncu_w6.log 2>&1; tail -1 gpurun_out/ncu_w6.log
