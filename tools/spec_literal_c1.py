"""the SPEC-literal oracle tier (i) -- pure Python, single thread --
on C1 (100 tiling polygons, eps = 1e-3, L = 11): build time, join rate on a
point prefix, and COUNT parity with tier (ii) (oracle/rb_oracle.c) on that
prefix.  CPU only.  usage: python tools/spec_literal_c1.py [points] [out.json]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

from oracle import oracle as O
from oracle import spec_literal as SL
from paper_2010_12548_b200 import workloads as W
from paper_2010_12548_b200.geometry import pack_regions
from paper_2010_12548_b200.grid import level_for_bound

m = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000
out = sys.argv[2] if len(sys.argv) > 2 else None
w = W.c1()
L = level_for_bound(w.grid, w.epsilon)
regs = [(r.id, [[r.geometry.outer.tolist()] + [h.tolist() for h in r.geometry.holes]]) for r in w.regions]
t = time.perf_counter()
trie, covers = SL.build(regs, (w.grid.origin.x, w.grid.origin.y), w.grid.extent, L)
build_s = time.perf_counter() - t
xy = w.xy[:m]
t = time.perf_counter()
res = SL.join_act(xy.tolist(), trie, (w.grid.origin.x, w.grid.origin.y), w.grid.extent)
join_s = time.perf_counter() - t
p = pack_regions(w.regions)
O.build_lib()
A = O.Approx((w.grid.origin.x, w.grid.origin.y, w.grid.extent, L), p.vx, p.vy, p.ring_off, p.poly_ring_off,
             p.poly_region, p.n_regions, 0)
cnt, _ = A.join(xy, None, nthreads=1)
lit = np.zeros_like(cnt)
for rid, (a, b, _sa, _sb) in res.items():
    lit[rid] = (a, b)
rec = {"config": "C1", "tier": "i (oracle/spec_literal.py, pure Python, 1 thread)", "level": L,
       "build_s": round(build_s, 2), "cells": int(sum(len(c) for _, c in covers)), "points": m,
       "join_s": round(join_s, 2), "points_per_s": round(m / join_s, 1),
       "count_equal_tier_ii": bool(np.array_equal(lit, cnt))}
print(json.dumps(rec))
if out:
    with open(out, "w") as f:
        f.write(json.dumps(rec) + "\n")
