import sys, time
sys.path.insert(0, '/root/repo')
import torch, numpy as np
from paper_2010_12548_b200 import workloads as W
from paper_2010_12548_b200.geometry import PointSet, pack_regions
from paper_2010_12548_b200.grid import level_for_bound
from paper_2010_12548_b200.engine import ApproxIndex
from paper_2010_12548_b200.pointindex import lps_build
from paper_2010_12548_b200.query import _region_cells
w = W.c2(n=100_000_000)
pts = PointSet(torch.from_numpy(w.xy).cuda(), {"fare": torch.from_numpy(w.attrs["fare"]).cuda()})
packed = pack_regions(w.regions)
L = level_for_bound(w.grid, w.epsilon); grid = w.grid.with_level(L)
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    lps = lps_build(pts, grid, ("fare",)); torch.cuda.synchronize(); t1 = time.perf_counter()
    idx = ApproxIndex(packed, grid, 0, layout="trie", keep_cells=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    rc = _region_cells(packed, idx, L); t3 = time.perf_counter()
    print(f"lps {1e3*(t1-t):.0f} ms, index {1e3*(t2-t1):.0f} ms, region_cells {1e3*(t3-t2):.0f} ms", flush=True)
