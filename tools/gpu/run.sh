timeout 1500 python -m pytest tests/test_gpu_scale.py -q -x 2>&1 | tail -5
for c in 0 1; do for k in 3071 4095 5119; do
RB_DEEP_CFG=$c RB_HOT_K=$k timeout 300 python tools/profile_pass.py c4 200000000 trie 3 12 2>&1 | grep -E "Gpts" | tail -1 | sed "s/^/TRIE12 cfg=$c K=$k /"
done; done
