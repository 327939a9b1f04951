#!/bin/bash
# Run on a GPU box (via gpurun): launch lists + one full ncu capture of the
# point-pass kernel for C2 and C4.  Each command first exits 0 without ncu.
set -u
O=gpurun_out
python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu > $O/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_point_pass|k_init_out|k_reduce_fixed|k_attr_scale" \
    --csv --log-file $O/launches_c2.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu > $O/ncu_launch_c2.log 2>&1
python tools/profile_pass.py c2 1e8 trie 1 > $O/plain_pp_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_point_pass -s 1 -c 1 -o $O/prof_c2 \
    python tools/profile_pass.py c2 1e8 trie 1 > $O/ncu_full_c2.log 2>&1
python tools/profile_pass.py c4 2e8 trie 1 > $O/plain_pp_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_point_pass -s 1 -c 1 -o $O/prof_c4 \
    python tools/profile_pass.py c4 2e8 trie 1 > $O/ncu_full_c4.log 2>&1
ls -la $O
