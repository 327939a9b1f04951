# A/B timing of library builds on one box for C4 (200M points): tools/ab_c4.sh layout root_level lib.so...
layout=$1; rl=$2; shift 2
for r in 1 2 3; do
  for lib in "$@"; do
    RASTERBOUND_B200_LIB=$lib timeout 300 python tools/profile_pass.py c4 200000000 $layout 3 $rl 2>&1 | grep Gpts | tail -1 | sed "s|^|$lib |"
  done
done
