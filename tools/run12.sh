timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t12.log 2>&1; tail -3 gpurun_out/t12.log
for cfg in "-1 8" "11 8" "12 4"; do set -- $cfg; echo "T0=$1 rw=$2"; timeout 600 python tools/profile_pass.py c4 2e8 trie 3 $1 $2 2>&1 | grep -E "Gpts|rror" | tail -1 | cut -c1-300; done
