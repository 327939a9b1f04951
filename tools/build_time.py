"""Approximation build times (warm rebuilds) per config and layout, with the
per-phase trace (RB_BUILD_TRACE=1 prints phases to stderr).
usage: python tools/build_time.py [c2|c4|c1] [layout] [root_level] [reps]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2010_12548_b200 import workloads as W  # noqa: E402
from paper_2010_12548_b200.query import AggregationQuery, PreparedJoin  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
layout = sys.argv[2] if len(sys.argv) > 2 else "trie"
root_level = int(sys.argv[3]) if len(sys.argv) > 3 else -1
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
w = {"c1": lambda: W.c1(n=1000), "c2": lambda: W.c2(n=1000), "c4": lambda: W.c4(n=1000)}[cfg]()
q = AggregationQuery("COUNT" if cfg == "c1" else "SUM:fare", w.epsilon)
runs = []
for k in range(reps):
    t = time.perf_counter()
    p = PreparedJoin(w.regions, q, w.grid, layout=layout, root_level=root_level)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t) * 1e3
    st = p.stats()
    runs.append({"lib_ms": round(st["build_ms"], 1), "wall_ms": round(wall, 1)})
    del p
print(json.dumps({"config": cfg, "layout": layout, "root_level": root_level, "index_bytes": st["index_bytes"],
                  "runs": runs}))
