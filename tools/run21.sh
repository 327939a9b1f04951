for cfg in "11 4" "10 4" "11 2" "13 4"; do set -- $cfg; echo "T0=$1 rw=$2"; timeout 600 python tools/profile_pass.py c4 2e8 trie 3 $1 $2 2>&1 | grep -E "Gpts|rror" | tail -1 | cut -c1-200; done
