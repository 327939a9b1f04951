"""Full-size parity against the CPU oracle (oracle/rb_oracle.c, all host threads):
every point of C1, of C2 at each C3 epsilon (hierarchical raster, radix table),
and of C4 (1B points).  COUNT must be bit-exact; SUM within rel 1e-6.
One JSON line per case.  usage: python tools/parity_full.py [c1,c3,c4] [out.jsonl]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from oracle import oracle as O
from paper_2010_12548_b200 import workloads as W
from paper_2010_12548_b200.engine import ApproxIndex
from paper_2010_12548_b200.geometry import pack_regions
from paper_2010_12548_b200.grid import level_for_bound

which = (sys.argv[1] if len(sys.argv) > 1 else "c1,c3,c4").split(",")
out = sys.argv[2] if len(sys.argv) > 2 else None
cores = len(os.sched_getaffinity(0))
O.build_lib()
recs = []


def case(name, w, eps, attr, layout="trie"):
    grid = w.grid.with_level(level_for_bound(w.grid, eps))
    p = pack_regions(w.regions)
    t = time.perf_counter()
    A = O.Approx((grid.origin.x, grid.origin.y, grid.extent, grid.max_level), p.vx, p.vy, p.ring_off,
                 p.poly_ring_off, p.poly_region, p.n_regions, 0)
    cnt_o, sum_o = A.join(w.xy, attr, nthreads=cores)
    cpu_s = time.perf_counter() - t
    del A
    idx = ApproxIndex(p, grid, 0, layout=layout)
    r = idx.point_pass(torch.from_numpy(w.xy).cuda(), None if attr is None else torch.from_numpy(attr).cuda()).check()
    cnt = r.cnt.cpu().numpy()
    rec = {"case": name, "epsilon": eps, "level": grid.max_level, "layout": layout, "points": int(w.n),
           "regions": int(p.n_regions), "count_bit_exact": bool(np.array_equal(cnt, cnt_o)),
           "count_abs_diff": int(np.abs(cnt - cnt_o).sum()), "oracle_s": round(cpu_s, 1), "oracle_threads": cores}
    if attr is not None:
        s = r.sum.cpu().numpy()
        rec["sum_max_rel_err"] = float(np.max(np.abs(s - sum_o) / np.maximum(np.abs(sum_o), 1e-30)))
    print(json.dumps(rec), flush=True)
    recs.append(rec)
    del idx
    torch.cuda.empty_cache()


if "c1" in which:
    w = W.c1()
    case("C1", w, w.epsilon, None, "dense")
    case("C1", w, w.epsilon, None, "trie")
if "c3" in which:
    w = W.c2()
    for eps in (50.0, 10.0, 4.9, 1.0, 0.5):
        case("C3/C2", w, eps, w.attrs["fare"])
    del w
if "c4" in which:
    w = W.c4()
    case("C4", w, w.epsilon, w.attrs["fare"])
if out:
    with open(out, "w") as f:
        for r in recs:
            f.write(json.dumps(r) + "\n")
