# L2 prefetch distance sweep (RB_PREFETCH) on the ring kernel
for pf in 0 1 2 4 8; do echo "PF=$pf"; RB_PREFETCH=$pf timeout 300 python tools/ablate.py 1e8; done
