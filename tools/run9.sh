timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t9.log 2>&1; tail -2 gpurun_out/t9.log
timeout 300 python tools/ablate.py 1e8
