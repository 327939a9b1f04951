"""join_pointindex on the C2 inputs: point-index build
(lps_build: leaf codes + stable radix sort + prefix sums; rs_build: RadixSpline),
then repeated polygon queries answered from the index (covering cells -> two
lower-bound lookups + prefix difference each).  Checks COUNT equality with
join_act.  One JSON line.  usage: python tools/bench_pointindex.py [points]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2010_12548_b200 import pointindex as P
from paper_2010_12548_b200 import workloads as W
from paper_2010_12548_b200.geometry import PointSet, pack_regions
from paper_2010_12548_b200.grid import level_for_bound
from paper_2010_12548_b200.query import AggregationQuery, PreparedJoin, PreparedPointIndexJoin, join_pointindex

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
w = W.c2(n=n)
grid = w.grid.with_level(level_for_bound(w.grid, w.epsilon))
pts = PointSet(torch.from_numpy(w.xy).cuda(), {"fare": torch.from_numpy(w.attrs["fare"]).cuda()})
q = AggregationQuery("SUM:fare", w.epsilon)
packed = pack_regions(w.regions)


def timed(fn, reps=1):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t) / reps * 1e3


lps, lps_ms = timed(lambda: P.lps_build(pts, grid, ["fare"]))
rs, rs_ms = timed(lambda: P.rs_build(lps))
pj, cover_ms = timed(lambda: PreparedPointIndexJoin(packed, q, w.grid))
pj.run_device(lps, rs)  # warm
_, join_rs_ms = timed(lambda: pj.run_device(lps, rs), 5)
_, join_bs_ms = timed(lambda: pj.run_device(lps, None), 5)
res_rs = pj.run(lps, rs)
prep = PreparedJoin(packed, q, w.grid)
act = prep.run(pts)
same = all(a.region_id == b.region_id and abs(a.alpha - b.alpha) <= 1e-6 * max(1.0, abs(a.alpha))
           for a, b in zip(act, res_rs))
qc = AggregationQuery("COUNT", w.epsilon)
cnt_same = [(r.alpha, r.boundary_part) for r in PreparedJoin(packed, qc, w.grid).run(pts)] == \
           [(r.alpha, r.boundary_part) for r in join_pointindex(lps, rs, packed, qc)]
st = prep.stats()
print(json.dumps({
    "engine": "join_pointindex", "config": "C2 inputs (100M f64 points + fare, 260 regions, eps 4.9 m)",
    "points": n, "lps_build_ms": round(lps_ms, 1), "rs_build_ms": round(rs_ms, 1),
    "radix_bits": rs.radix_bits, "max_error": rs.max_error, "spline_knots": rs.n_knots,
    "covering_cells": pj.n_cells, "covering_build_ms": round(cover_ms, 1),
    "query_ms_radixspline": round(join_rs_ms, 3), "query_ms_binary_search": round(join_bs_ms, 3),
    "points_per_s_per_query": n / (join_rs_ms / 1e3),
    "note": "query = rb_join_pointindex over the prepared coverings (2 lower-bound lookups + prefix difference per cell)",
    "sum_equal_join_act_rel1e-6": same, "count_alpha_beta_equal_join_act": cnt_same}))
