"""C4 index sweep (B200): one point set, several (grid, layout, root level)
indexes; per index the build time, index bytes, point-pass kernel time and
points/s, COUNT equality against the first index, and the point mix (no owner,
owner list, boundary single, hot / cold interior single) from a lookup sample.

usage: python tools/sweep_c4.py [points] [spec ...]    spec = grid:layout:root_level (e.g. eps:packed:13)
Prints one JSON line per index."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2010_12548_b200 import _native as N  # noqa: E402
from paper_2010_12548_b200 import workloads as W  # noqa: E402
from paper_2010_12548_b200.query import AggregationQuery, PreparedJoin  # noqa: E402


def mix(idx, xy):
    v = idx.lookup(xy[: min(len(xy), 4_000_000)]).to(torch.int64) & 0xFFFFFFFF
    tot = len(v)
    lst = (v & N.VALUE_LIST) != 0
    single = (v != 0) & ~lst
    code = v & N.CODE_MASK
    bnd = single & ((code - 1) & 1).bool()
    ishot = torch.zeros(idx.n_regions + 1, dtype=torch.bool, device=v.device)
    if idx._hot is not None and len(idx._hot):
        ishot[torch.as_tensor(idx._hot, dtype=torch.int64, device=v.device)] = True
    reg = torch.where(single, (code - 1) >> 1, torch.full_like(code, idx.n_regions))
    hot = single & ~bnd & ishot[reg]
    cold = single & ~bnd & ~ishot[reg]
    return {k: round(m.sum().item() / tot, 5) for k, m in
            (("none", v == 0), ("list", lst), ("boundary", bnd), ("hot", hot), ("cold", cold))}


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 200_000_000
    specs = sys.argv[2:] or ["eps:packed:-1", "eps:trie:-1"]
    reps = int(os.environ.get("REPS", "5"))
    t = time.time()
    base = W.c4(n=n)
    print(f"# data {time.time() - t:.1f} s", flush=True)
    xy = torch.from_numpy(base.xy).cuda()
    at = torch.from_numpy(base.attrs["fare"]).cuda()
    ref = None
    for spec in specs:
        gname, layout, rl = spec.split(":")
        grid = base.grid if gname == "eps" else W.ingest_grid(0.0, 0.0, 100_000.0, 100_000.0)
        q = AggregationQuery("SUM:fare", base.epsilon)
        t = time.time()
        prep = PreparedJoin(base.regions, q, grid, layout=layout, root_level=int(rl))
        st = prep.stats()
        build_s = time.time() - t
        r = prep.index.point_pass(xy, at)
        torch.cuda.synchronize()
        N.instrument(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            prep.index.point_pass(xy, at, out=r)
        e1.record()
        torch.cuda.synchronize()
        _, timed, kms = N.instrument(0)
        N.instrument(2)
        step = e0.elapsed_time(e1) / reps
        k = kms / max(timed, 1)
        r.check()
        cnt = r.cnt.cpu().numpy()
        same = None
        if gname == "eps" and ref is not None:
            same = bool(np.array_equal(cnt, ref))
        if gname == "eps" and ref is None:
            ref = cnt
        line = {"spec": spec, "n": n, "L": st["max_level"], "root_level": st["root_level"],
                "index_MB": round(st["index_bytes"] / 1e6, 1), "n_nodes": st["n_nodes"], "build_s": round(build_s, 2),
                "build_ms_lib": round(st["build_ms"], 1), "kernel_ms": round(k, 4), "step_ms": round(step, 4),
                "Gpts_s": round(n / k / 1e6, 2), "GBps": round(n * 12 / k / 1e6, 1),
                "frac": round(n * 12 / k / 1e6 / 6459.9, 4), "count_equal_first_eps": same, "mix": mix(prep.index, xy)}
        print(json.dumps(line), flush=True)
        del prep, r
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
