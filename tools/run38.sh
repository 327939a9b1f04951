# e2e (join_host) with one or two H2D copy streams
for r in 1 2; do for s in 1 2; do echo "streams=$s $(RB_JH_STREAMS=$s timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["e2e"])')"; done; done
