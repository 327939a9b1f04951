timeout 300 python tools/profile_pass.py c4 200000000 packed 1 > gpurun_out/plain_pp_c4_packed.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_point_pass -s 1 -c 1 -o gpurun_out/prof_c4_pkl python tools/profile_pass.py c4 200000000 packed 1 > gpurun_out/ncu_full_c4_pkl.log 2>&1; echo rc=$?
