# ablations at the current configuration: 1 skip rare path, 2 skip node level, 4 skip root loads
for ab in 0 1 2 4 3 7; do echo "ABLATE=$ab"; RB_ABLATE=$ab timeout 300 python tools/ablate.py 1e8 | grep c2; done
