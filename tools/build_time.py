"""Approximation build time (rb_approx_build) for C2 at several levels, 3 builds each.
usage: python tools/build_time.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2010_12548_b200 import workloads as W
from paper_2010_12548_b200.engine import ApproxIndex
from paper_2010_12548_b200.geometry import pack_regions

w = W.c2(n=1000)
p = pack_regions(w.regions)
for L in (13, 14, 16):
    for r in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        idx = ApproxIndex(p, w.grid.with_level(L), 0)
        torch.cuda.synchronize()
        print(f"L={L} build {r}: wall {(time.perf_counter() - t) * 1e3:.1f} ms, internal {idx.stats()['build_ms']:.1f} ms",
              flush=True)
        del idx
