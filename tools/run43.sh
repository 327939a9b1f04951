# KEYS ring instantiation: trie path unchanged (A/B), keys layout parity and timing
bash tools/ab.sh build/ab/cur.so build/ab/new.so 2>&1 | tail -8
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sorted_key or ring_drains or city" 2>&1 | tail -1
for L in keys trie; do timeout 600 python bench.py --layout $L --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$L\", d[\"value\"]/1e9, d[\"roofline\"][\"kernel_ms\"])"; done
