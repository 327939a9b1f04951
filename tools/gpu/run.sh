bash tools/gpu/run_xd.sh
timeout 1200 python -m pytest tests/test_gpu_capacity.py -q -x 2>&1 | tail -3
