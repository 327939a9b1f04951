# A/B timing of library builds on one box: tools/ab.sh <lib.so>... (ablate.py c2 lines, 3 rounds interleaved)
for r in 1 2 3; do
  for lib in "$@"; do
    echo "== $lib"; RASTERBOUND_B200_LIB=$lib timeout 300 python tools/ablate.py 1e8 | grep c2
  done
done
