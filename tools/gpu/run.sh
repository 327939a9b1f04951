timeout 900 python -m pytest tests/test_gpu_packed.py tests/test_gpu_scale.py -q -x -k "not c3" 2>&1 | tail -3
for r in 1 2; do
timeout 300 python tools/profile_pass.py c4 200000000 trie 3 12 2>&1 | grep -E "Gpts" | tail -1 | sed "s/^/TRIE12 /"
RB_PK3_CFG=0 timeout 300 python tools/profile_pass.py c4 200000000 packed 3 12 2>&1 | grep -E "Gpts" | tail -1 | sed "s/^/PKL12 cfg0 /"
RB_PK3_CFG=1 timeout 300 python tools/profile_pass.py c4 200000000 packed 3 12 2>&1 | grep -E "Gpts" | tail -1 | sed "s/^/PKL12 cfg1 /"
timeout 300 python tools/profile_pass.py c4 200000000 packed 3 13 2>&1 | grep -E "Gpts" | tail -1 | sed "s/^/PK2-13 /"
done
