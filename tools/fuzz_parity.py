"""Randomised parity against the oracle: random (possibly overlapping, holed)
polygons, random grid levels, both modes, every index layout (radix table, sorted keys, dense grid, packed
in both forms) and the opt-in partitioned pass, f64/f32
points drawn uniformly, clustered, on grid lines and on polygon vertices,
attributes spanning many magnitudes (zero, negative, out of the fixed-point
window).  COUNT must be bit-exact, SUM within rel 1e-6.  Prints one line per
case and a summary; exits 1 on any mismatch.
usage: python tools/fuzz_parity.py [cases] [seed] [kind: random|holes|tiling|big]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

from helpers import oracle_approx, random_polygons
from oracle import oracle as O
from paper_2010_12548_b200 import workloads as W
from paper_2010_12548_b200.engine import ApproxIndex
from paper_2010_12548_b200.geometry import Point2D, pack_regions
from paper_2010_12548_b200.grid import GridConfig

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
O.build_lib()
fails = 0
t0 = time.time()
for c in range(cases):
    rng = np.random.default_rng(seed0 + c)
    kind = rng.choice(["random", "holes", "tiling", "big"]) if len(sys.argv) <= 3 else sys.argv[3]
    try:
        if kind == "tiling":
            regions = W.voronoi_tiling(int(rng.integers(20, 400)), 1.0, seed=int(seed0 + c), verts=(6, 20))
            L = int(rng.integers(3, 15))
        elif kind == "big":  # region sets beyond shared memory: deep / global kernels, hot slots
            regions = W.voronoi_tiling(int(rng.integers(2000, 6000)), 1.0, seed=int(seed0 + c), verts=(6, 14))
            L = int(rng.integers(10, 15))
    except RuntimeError as e:  # the tiling generator gave up on this seed (no simple polygons): not a parity case
        print(f"case {c}: {kind} skipped ({e})", flush=True)
        continue
    if kind in ("random", "holes"):
        regions = random_polygons(int(seed0 + c), int(rng.integers(3, 40)), holes=(kind == "holes"))
        L = int(rng.integers(3, 22))  # up to 21: beyond the ring kernels' 2^20 window
    mode = int(rng.integers(0, 2))
    # "binned": the radix table through the opt-in partitioned pass (RB_BINNED=1, csrc/rb_binned.cuh)
    layouts = [("trie", -1), ("binned", -1), ("keys", -1), ("packed", -1)] + \
        ([("packed", L - 3)] if 3 <= L <= 19 else []) + ([("dense", -1)] if L <= 12 else [])
    grid = GridConfig(Point2D(0.0, 0.0), 1.0, L)
    n = int(rng.integers(1, 300_000))
    parts = [rng.random((n, 2))]
    ctr = rng.random((5, 2))
    parts.append(np.clip(ctr[rng.integers(0, 5, n // 2)] + rng.normal(0, 0.02, (n // 2, 2)), 0, 1 - 1e-12))
    side = 1.0 / (1 << L)
    gl = rng.integers(0, 1 << L, (n // 8, 2)) * side  # exactly on grid lines / corners
    parts.append(np.clip(gl, 0, 1 - 1e-12))
    p = pack_regions(regions)
    vv = np.stack([p.vx, p.vy], 1)
    parts.append(np.clip(vv[rng.integers(0, len(vv), min(len(vv), n // 8))], 0, 1 - 1e-12))  # on vertices
    xy = np.concatenate(parts)
    rng.shuffle(xy)
    attr = (rng.lognormal(0, 3, len(xy)) * rng.choice([-1.0, 1.0], len(xy))).astype(np.float32)
    attr[rng.random(len(xy)) < 0.05] = 0.0
    A, _ = oracle_approx(O, regions, grid, mode)
    hot = None
    if kind == "big" and rng.random() < 0.5:  # an explicit hot subset: cold regions take the global REDs
        hot = np.sort(rng.choice(p.n_regions, int(rng.integers(0, min(4095, p.n_regions))), replace=False))
    for layout, rl in layouts:
        idx = ApproxIndex(p, grid, mode, layout="trie" if layout == "binned" else layout, root_level=rl)
        os.environ["RB_BINNED"] = "1" if layout == "binned" else "0"
        if hot is not None:
            idx.set_hot(hot)
        for pts, at in ((xy, attr), (xy.astype(np.float32), None)):
            pts = np.ascontiguousarray(pts)
            try:
                cnt_o, sum_o = A.join(pts, at, nthreads=8)
            except O.OracleError:
                continue  # f32 rounding pushed a point out of the domain: both sides raise, skip
            r = idx.point_pass(pts, at).check()
            cnt = r.cnt.cpu().numpy()
            ok = np.array_equal(cnt, cnt_o)
            if at is not None:
                s = r.sum.cpu().numpy()
                ok = ok and np.allclose(s, sum_o, rtol=1e-6, atol=1e-6 * np.abs(attr).max())
            if not ok:
                fails += 1
                print(f"FAIL case {c} seed {seed0 + c}: {kind} R={p.n_regions} L={L} mode={mode} layout={layout}/{rl} "
                      f"n={len(pts)} f32={pts.dtype == np.float32} count_diff={int(np.abs(cnt - cnt_o).sum())}",
                      flush=True)
        del idx
    os.environ.pop("RB_BINNED", None)
    print(f"case {c}: {kind} R={p.n_regions} L={L} mode={mode} n={len(xy)} layouts={[x for x, _ in layouts]} ok",
          flush=True)
print(f"{cases} cases, {fails} mismatches, {time.time() - t0:.0f} s")
sys.exit(1 if fails else 0)
