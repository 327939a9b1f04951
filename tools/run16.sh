timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t16.log 2>&1; tail -2 gpurun_out/t16.log
timeout 300 python tools/ablate.py 1e8
timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/b16.json 2>&1; cut -c1-300 gpurun_out/b16.json; grep -o '"roofline.*' gpurun_out/b16.json | cut -c1-200
