timeout 600 python -m pytest tests/test_gpu_integration_stub.py tests/test_gpu_capacity.py -q -x 2>&1 | tail -3
