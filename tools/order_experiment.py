"""Design experiment for C4 (B200): how much of the deep point pass's cost is
the random order of the points?  Times the same pass over the same points in
the generator's order and stably grouped by a coarse cell (level 4/5/7 bins,
and full leaf Z order).  Grouping the input is not the benchmark (its input
order is the generator's); this bounds what a partition-then-join design
could gain in its second pass.

usage: python tools/order_experiment.py [points] [levels ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2010_12548_b200 import _native as N  # noqa: E402
from paper_2010_12548_b200 import workloads as W  # noqa: E402
from paper_2010_12548_b200.query import AggregationQuery, PreparedJoin  # noqa: E402


def timed(prep, xy, at, reps=5):
    r = prep.index.point_pass(xy, at)
    torch.cuda.synchronize()
    N.instrument(1)
    for _ in range(reps):
        prep.index.point_pass(xy, at, out=r)
    torch.cuda.synchronize()
    _, nt, kms = N.instrument(0)
    N.instrument(2)
    r.check()
    return kms / max(nt, 1), r.cnt.cpu().numpy()


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 200_000_000
    levels = [int(x) for x in sys.argv[2:]] or [4, 5, 7, 18]
    layout = os.environ.get("LAYOUT", "trie")
    w = W.c4(n=n)
    g = w.grid
    prep = PreparedJoin(w.regions, AggregationQuery("SUM:fare", w.epsilon), g, layout=layout)
    L = prep.stats()["max_level"]
    xy = torch.from_numpy(w.xy).cuda()
    at = torch.from_numpy(w.attrs["fare"]).cuda()
    k0, cnt0 = timed(prep, xy, at)
    print(json.dumps({"order": "generator", "n": n, "layout": layout, "kernel_ms": round(k0, 4),
                      "Gpts_s": round(n / k0 / 1e6, 2)}), flush=True)
    side = g.extent / (1 << L)
    bx = ((xy[:, 0].double() - g.origin.x) / side).floor().clamp(0, (1 << L) - 1).long()
    by = ((xy[:, 1].double() - g.origin.y) / side).floor().clamp(0, (1 << L) - 1).long()
    for lv in levels:
        s = L - lv
        key = ((by >> s) << lv) | (bx >> s) if lv < 18 else None
        if key is None:  # Z order of the leaf
            z = torch.zeros_like(bx)
            for b in range(L):
                z |= ((bx >> b) & 1) << (2 * b) | ((by >> b) & 1) << (2 * b + 1)
            key = z
        perm = torch.sort(key, stable=True).indices
        xs, as_ = xy[perm].contiguous(), at[perm].contiguous()
        del perm, key
        k, cnt = timed(prep, xs, as_)
        print(json.dumps({"order": f"grouped by level-{lv} cell" if lv < 18 else "leaf Z order", "n": n,
                          "layout": layout, "kernel_ms": round(k, 4), "Gpts_s": round(n / k / 1e6, 2),
                          "count_equal": bool(np.array_equal(cnt, cnt0))}), flush=True)
        del xs, as_
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
