for pf in 0 1 2 4; do echo "PF=$pf (evict_first)"; RB_PREFETCH=$pf timeout 300 python tools/ablate.py 1e8 | grep c2; done
