timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q > gpurun_out/t26.log 2>&1; tail -3 gpurun_out/t26.log
for ab in 0 1 2 4; do echo "ABLATE=$ab"; RB_ABLATE=$ab timeout 300 python tools/ablate.py 1e8 | grep c2; done
