"""join_canvas (the Bounded Raster Join) on C1 and C2: the fused
dense plan (L <= 13) and the literal canvas-algebra plan (canvas.brj, tiled),
each checked against join_act (COUNT equal, SUM rel 1e-6).  One JSON line per
case.  usage: python tools/bench_canvas.py [c2_points]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2010_12548_b200 import workloads as W
from paper_2010_12548_b200.geometry import PointSet
from paper_2010_12548_b200.query import AggregationQuery, join_act, join_canvas

n2 = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000


def run(name, w, agg, plans):
    q = AggregationQuery(agg, w.epsilon)
    attrs = {"fare": torch.from_numpy(w.attrs["fare"]).cuda()} if "fare" in w.attrs and agg != "COUNT" else {}
    pts = PointSet(torch.from_numpy(w.xy).cuda(), attrs)
    ref = join_act(pts, w.regions, q, w.grid)
    for plan in plans:
        join_canvas(pts, w.regions, q, w.grid, plan=plan)  # warm
        torch.cuda.synchronize()
        t = time.perf_counter()
        res = join_canvas(pts, w.regions, q, w.grid, plan=plan)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) * 1e3
        same_cnt = all(a.region_id == b.region_id for a, b in zip(ref, res))
        if agg == "COUNT":
            same = same_cnt and all(a.alpha == b.alpha and a.boundary_part == b.boundary_part for a, b in zip(ref, res))
        else:
            same = same_cnt and all(abs(a.alpha - b.alpha) <= 1e-6 * max(1.0, abs(a.alpha)) for a, b in zip(ref, res))
        print(json.dumps({"engine": "join_canvas", "plan": plan, "config": name, "points": int(w.n), "agg": agg,
                          "regions": len(w.regions), "wall_ms": round(ms, 1), "points_per_s": w.n / (ms / 1e3),
                          "equal_join_act": bool(same)}), flush=True)


run("C1", W.c1(), "COUNT", ("fused", "algebra"))
w2 = W.c2(n=n2)
run("C2", w2, "SUM:fare", ("algebra",))
