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
# CPU baseline (oracle/pointindex_oracle.py, numpy, one thread): the same build and the same query
from oracle import pointindex_oracle as PO

L = grid.max_level
t = time.perf_counter()
codes_h, perm_h, pref_h = PO.lps_build(w.xy, (grid.origin.x, grid.origin.y), grid.extent, L, {"fare": w.attrs["fare"]})
cpu_build_ms = (time.perf_counter() - t) * 1e3
lv = pj._level.cpu().numpy().astype(np.int64)
cd = pj._code.cpu().numpy().view(np.uint64)
rg = pj._region.cpu().numpy().astype(np.int64)
sh = (2 * (L - lv)).astype(np.uint64)
t = time.perf_counter()
lo_i, hi_i = PO.bounds_lookup(codes_h, cd << sh, (cd + np.uint64(1)) << sh)
cpu_cnt = np.bincount(rg, weights=(hi_i - lo_i), minlength=packed.n_regions)
cpu_sum = np.bincount(rg, weights=pref_h["fare"][hi_i] - pref_h["fare"][lo_i], minlength=packed.n_regions)
cpu_query_ms = (time.perf_counter() - t) * 1e3
gcnt, gsum = pj.run_device(lps, rs)
gcnt = gcnt.cpu().numpy()
gsum = gsum.cpu().numpy()
cpu_same = bool(np.array_equal(gcnt[:, 0], cpu_cnt.astype(np.int64))) and \
    bool(np.allclose(gsum[:, 0], cpu_sum, rtol=1e-9, atol=1e-6))
print(json.dumps({
    "engine": "join_pointindex", "config": "C2 inputs (100M f64 points + fare, 260 regions, eps 4.9 m)",
    "points": n, "lps_build_ms": round(lps_ms, 1), "rs_build_ms": round(rs_ms, 1),
    "radix_bits": rs.radix_bits, "max_error": rs.max_error, "spline_knots": rs.n_knots,
    "covering_cells": pj.n_cells, "covering_build_ms": round(cover_ms, 1),
    "query_ms_radixspline": round(join_rs_ms, 3), "query_ms_binary_search": round(join_bs_ms, 3),
    "points_per_s_per_query": n / (join_rs_ms / 1e3),
    "note": "query = rb_join_pointindex over the prepared coverings (2 lower-bound lookups + prefix difference per cell)",
    "sum_equal_join_act_rel1e-6": same, "count_alpha_beta_equal_join_act": cnt_same,
    "cpu_baseline": {"impl": "oracle/pointindex_oracle.py (numpy, 1 thread)", "lps_build_ms": round(cpu_build_ms, 1),
                     "query_ms": round(cpu_query_ms, 1), "alpha_equal_gpu": cpu_same}}))
