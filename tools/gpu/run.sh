set -x
./tools/microbench/dsmem 2>&1 | tail -15
for abl in 0 1 3 6 7; do RB_DEEP_ABLATE=$abl timeout 300 python tools/profile_pass.py c4 200000000 packed 3 13 2>&1 | grep Gpts | tail -1 | sed "s/^/ABL=$abl /"; done
for rl in 11 12 13; do timeout 300 python tools/profile_pass.py c4 200000000 trie 3 $rl 2>&1 | grep Gpts | tail -1; done
timeout 300 python tools/profile_pass.py c4 200000000 packed 2 13 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_point_pass_deep -s 1 -c 1 -o gpurun_out/prof_c4_packed -f python tools/profile_pass.py c4 200000000 packed 2 13 > gpurun_out/ncu3.log 2>&1
tail -3 gpurun_out/ncu3.log
