"""Run the complete epsilon validator (rb_validate_full: every point) on the
bench workloads and print one JSON line per workload/mode.

    python tools/validate_full.py [--configs c1,c2,c4] [--c4-points 200000000]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c4")
    ap.add_argument("--c4-points", type=int, default=200_000_000)
    ap.add_argument("--modes", default="0,1")
    a = ap.parse_args()
    import torch

    from paper_2010_12548_b200 import workloads as W
    from paper_2010_12548_b200.engine import ApproxIndex
    from paper_2010_12548_b200.geometry import pack_regions
    from paper_2010_12548_b200.grid import level_for_bound
    from paper_2010_12548_b200.validate import validate_full

    for cfg in a.configs.split(","):
        w = {"c1": lambda: W.c1(), "c2": lambda: W.c2(), "c4": lambda: W.c4(n=a.c4_points)}[cfg]()
        L = level_for_bound(w.grid, w.epsilon)
        xy = torch.as_tensor(w.xy).cuda()
        packed = pack_regions(w.regions)
        for mode in (int(m) for m in a.modes.split(",")):
            idx = ApproxIndex(packed, w.grid.with_level(L), mode)
            torch.cuda.synchronize()
            t = time.perf_counter()
            rep = validate_full(idx, xy, w.epsilon)
            el = time.perf_counter() - t
            d = rep.as_dict()
            d.update(workload=w.name, mode=["CONSERVATIVE", "CENTER_SAMPLED"][mode], max_level=L, seconds=round(el, 3),
                     grid=w.meta.get("grid", "ingest"), leaf_side=w.grid.extent / (1 << L),
                     polygons=packed.n_polygons, regions=packed.n_regions)
            print(json.dumps(d), flush=True)
            del idx


if __name__ == "__main__":
    main()
