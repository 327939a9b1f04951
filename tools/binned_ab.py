"""A/B of the partitioned point pass (RB_BINNED=1) against the one-pass deep
kernel (RB_BINNED=0) on C4: kernel time per pass, COUNT equality, SUM relative
difference.  usage: python tools/binned_ab.py [points] [layout]"""
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


def run(prep, xy, at, reps):
    r = prep.index.point_pass(xy, at)
    torch.cuda.synchronize()
    N.instrument(1)
    for _ in range(reps):
        prep.index.point_pass(xy, at, out=r)
    torch.cuda.synchronize()
    launches, nt, kms = N.instrument(0)
    N.instrument(2)
    r.check()
    return kms / max(nt, 1), r.cnt.cpu().numpy(), r.sum.cpu().numpy() if at is not None else None


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 200_000_000
    layout = sys.argv[2] if len(sys.argv) > 2 else "trie"
    reps = int(os.environ.get("REPS", "5"))
    w = W.c4(n=n)
    prep = PreparedJoin(w.regions, AggregationQuery("SUM:fare", w.epsilon), w.grid, layout=layout)
    xy = torch.from_numpy(w.xy).cuda()
    at = torch.from_numpy(w.attrs["fare"]).cuda()
    out = {}
    for mode in os.environ.get("MODES", "0,1,0,1").split(","):
        os.environ["RB_BINNED"] = mode
        k, c, s = run(prep, xy, at, reps)
        kc, cc, _ = run(prep, xy, None, 2)
        out.setdefault(mode, []).append((k, c, s, kc, cc))
    first = next(iter(out.values()))[0]
    c0, s0 = first[1], first[2]
    for mode, runs in out.items():
        for k, c, s, kc, cc in runs:
            rel = float(np.max(np.abs(s - s0) / np.maximum(np.abs(s0), 1e-30)))
            print(json.dumps({"binned": mode, "n": n, "layout": layout, "kernel_ms": round(k, 4),
                              "Gpts_s": round(n / k / 1e6, 2), "count_ms": round(kc, 4),
                              "count_equal": bool(np.array_equal(c, c0)), "count_only_equal": bool(np.array_equal(cc, c0)),
                              "sum_max_rel_vs_onepass": rel}), flush=True)


if __name__ == "__main__":
    main()
