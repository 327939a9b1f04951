MLP_SWEEP=5 timeout 300 ./tools/microbench/mlp > gpurun_out/r2_mlp5.jsonl 2>&1; echo rc=$?
