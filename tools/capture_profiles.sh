#!/bin/bash
# Run on a GPU box (via gpurun): bench lines, a launch list of the bench
# command, and one full ncu capture of the point-pass kernel per config.
# Every command first exits 0 without ncu.  Usage: capture_profiles.sh [c2|c4|all]
set -u
O=gpurun_out
W=${1:-c2}
for C in c2 c4; do
  if [ "$W" != all ] && [ "$W" != $C ]; then continue; fi
  N=1e8; [ $C = c4 ] && N=2e8
  timeout 900 python bench.py --config $C > $O/bench_$C.json 2> $O/bench_$C.err
  timeout 900 python bench.py --config $C --steps 3 --warmup 1 --no-e2e --no-cpu --rebuilds 0 > $O/plain_launch_$C.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_point_pass|k_init_out|k_reduce_fixed|k_attr_scale" \
      --csv --log-file $O/launches_$C.csv python bench.py --config $C --steps 3 --warmup 1 --no-e2e --no-cpu --rebuilds 0 > $O/ncu_launch_$C.log 2>&1
  timeout 300 python tools/profile_pass.py $C $N trie 1 > $O/plain_pp_$C.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_point_pass -s 1 -c 1 -o $O/prof_$C \
      python tools/profile_pass.py $C $N trie 1 > $O/ncu_full_$C.log 2>&1
done
ls -la $O
