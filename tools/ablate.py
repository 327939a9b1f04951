"""Point-pass ablations on the GPU (timing only): which part of the pass costs what
(RB_ABLATE=1 skips the rare path; RASTERBOUND_B200_LIB picks a library build for A/B).
  c2 SUM / c2 COUNT          the real workload
  square SUM / square COUNT  one square region over the whole domain: every point resolves
                             from the shared-memory summary (no L2 index traffic)
usage: python tools/ablate.py [n]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2010_12548_b200 import workloads as W
from paper_2010_12548_b200.engine import ApproxIndex
from paper_2010_12548_b200.geometry import Polygon, RegionRecord, pack_regions
from paper_2010_12548_b200.grid import level_for_bound

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
w = W.c2(n=n)
grid = w.grid.with_level(level_for_bound(w.grid, w.epsilon))
xy = torch.from_numpy(w.xy).cuda()
at = torch.from_numpy(w.attrs["fare"]).cuda()


def timeit(idx, attr, reps=5):
    r = idx.point_pass(xy, attr)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record()
        idx.point_pass(xy, attr, out=r)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


idx = ApproxIndex(pack_regions(w.regions), grid, 0, layout="trie")
sq = [RegionRecord(0, Polygon([(0.0, 0.0), (40000.0, 0.0), (40000.0, 40000.0), (0.0, 40000.0)]))]
idx_sq = ApproxIndex(pack_regions(sq), grid, 0, layout="trie")
for name, ix in (("c2", idx), ("square", idx_sq)):
    for agg, a in (("SUM", at), ("COUNT", None)):
        ms = timeit(ix, a)
        bpp = 20 if a is not None else 16
        print(f"{name:7s} {agg:5s} {ms:.3f} ms  {n / ms / 1e6:7.2f} Gpts/s  {n * bpp / ms / 1e6:7.1f} GB/s", flush=True)
