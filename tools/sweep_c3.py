"""C3 accuracy/performance sweep (BASELINE.json configs[2]) on the C2 inputs:
eps in {50, 10, 4.9, 1, 0.5} m x {uniform raster (dense leaf grid), hierarchical
quadtree raster (radix table)}: points/s of the point pass, approximation build
time, cell count, and the fraction of points whose approximate owner set
differs from the exact test (the eps-validator checks every such point lies
within eps of the boundary).  One JSON line per (eps, raster).

usage: python tools/sweep_c3.py [points] [out.jsonl]
(the validator is rb_validate_full: every one of the points, not a sample)"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2010_12548_b200 import workloads as W
from paper_2010_12548_b200.engine import ApproxIndex
from paper_2010_12548_b200.geometry import pack_regions
from paper_2010_12548_b200.grid import level_for_bound
from paper_2010_12548_b200.validate import validate_full

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
out = sys.argv[2] if len(sys.argv) > 2 else None
w = W.c2(n=n)
packed = pack_regions(w.regions)
xy = torch.from_numpy(w.xy).cuda()
at = torch.from_numpy(w.attrs["fare"]).cuda()
DENSE_MAX_BYTES = 20e9  # the dense leaf grid is 4 bytes per leaf cell: L <= 16
lines = []
for eps in (50.0, 10.0, 4.9, 1.0, 0.5):
    grid = w.grid.with_level(level_for_bound(w.grid, eps))
    L = grid.max_level
    ref_cnt = None
    for raster, layout in (("uniform", "dense"), ("hierarchical", "trie"), ("hierarchical", "keys")):
        rec = {"config": "C3", "epsilon_m": eps, "level": L, "raster": raster, "layout": layout, "points": n}
        if layout == "dense" and 4.0 ** L * 4 > DENSE_MAX_BYTES:
            rec["skipped"] = f"dense leaf grid would be {4.0 ** L * 4 / 1e9:.0f} GB"
            lines.append(rec)
            print(json.dumps(rec), flush=True)
            continue
        torch.cuda.synchronize()
        t = time.perf_counter()
        idx = ApproxIndex(packed, grid, 0, layout=layout)
        torch.cuda.synchronize()
        first_ms = (time.perf_counter() - t) * 1e3
        del idx
        t = time.perf_counter()
        idx = ApproxIndex(packed, grid, 0, layout=layout)  # warm rebuild: no first-use costs
        torch.cuda.synchronize()
        build_ms = (time.perf_counter() - t) * 1e3
        st = idx.stats()
        r = idx.point_pass(xy, at)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(5):
            e0.record()
            idx.point_pass(xy, at, out=r)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        r.check()
        cnt = r.cnt.cpu().numpy()
        if ref_cnt is None:
            ref_cnt = cnt
        rep = validate_full(idx, xy, eps)
        cells = (st["n_uniform_interior"] + st["n_partial_leaves"]) if raster == "uniform" else \
            (st["n_interior_cells"] + st["n_boundary_cells"])
        rec.update(points_per_s=n / (best / 1e3), pass_ms=round(best, 4), build_ms=round(build_ms, 1),
                   build_ms_first=round(first_ms, 1),
                   build_ms_internal=round(st["build_ms"], 1), cells=int(cells), index_bytes=int(st["index_bytes"]),
                   alpha_total=int(cnt[:, 0].sum()), beta_total=int(cnt[:, 1].sum()),
                   counts_equal_uniform=bool(np.array_equal(cnt, ref_cnt)),
                   validated_points=rep.points, mismatch_fraction=rep.mismatch_fraction,
                   false_negatives=rep.false_negatives, max_mismatch_distance_m=rep.max_mismatch_distance,
                   violations=rep.violations, eps_ok=rep.ok)
        lines.append(rec)
        print(json.dumps(rec), flush=True)
        del idx
        torch.cuda.empty_cache()
if out:
    with open(out, "w") as f:
        for rec in lines:
            f.write(json.dumps(rec) + "\n")
