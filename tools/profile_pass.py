"""Run the point pass of a config a few times (for ncu / quick timing).
usage: python tools/profile_pass.py [c2|c4] [points] [layout] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2010_12548_b200 import workloads as W
from paper_2010_12548_b200.query import AggregationQuery, PreparedJoin

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 20_000_000
layout = sys.argv[3] if len(sys.argv) > 3 else "trie"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
root_level = int(sys.argv[5]) if len(sys.argv) > 5 else -1
radix_width = int(sys.argv[6]) if len(sys.argv) > 6 else 8
if cfg == "c2":
    w = W.c2(n=n)
elif cfg == "c4u":  # C4 regions, uniform points (no hot spots)
    w = W.c4(n=1000)
    w.xy = (np.random.default_rng(0).random((n, 2)) * 100_000.0).astype(np.float32)
    w.attrs = {"fare": W.fares(n, 0)}
else:
    w = W.c4(n=n)
q = AggregationQuery("SUM:fare", w.epsilon)
prep = PreparedJoin(w.regions, q, w.grid, layout=layout, root_level=root_level, radix_width=radix_width)
xy = torch.from_numpy(w.xy).cuda()
at = torch.from_numpy(w.attrs["fare"]).cuda()
r = prep.index.point_pass(xy, at)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(reps):
    e0.record()
    prep.index.point_pass(xy, at, out=r)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    bpp = 20 if cfg == "c2" else 12
    print(f"{cfg} {layout} T0={prep.stats()['root_level']} rw={radix_width} idxMB={prep.stats()['index_bytes']/1e6:.0f} n={n} {ms:.3f} ms  {n / ms / 1e6:.2f} Gpts/s  {n * bpp / ms / 1e6:.1f} GB/s", flush=True)
r.check()
print(prep.stats())
