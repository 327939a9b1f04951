"""Epsilon validator (north star: "a validator confirms that every point the
approximation assigns differently from the exact test lies within eps of a
polygon boundary").

For a sample of points: the approximate owner set comes from the device
index (rb_lookup); the exact owner set from point_in_polygon (boundary =
inside) evaluated on the GPU (rb_exact_pip) for every candidate
(point, polygon) pair whose MBR contains the point; every mismatching
(point, region) pair gets its exact distance to the region's boundary
(rb_exact_distance).  The candidate filter is a bucket grid over polygon MBRs
built on the host (test-of-the-answer plumbing, not the join path).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .engine import ApproxIndex
from .geometry import DevicePolygons, PackedRegions


@dataclass
class ValidationReport:
    points: int
    mismatched_points: int
    mismatched_pairs: int
    false_positives: int
    false_negatives: int
    max_mismatch_distance: float
    epsilon: float

    @property
    def ok(self) -> bool:
        return self.max_mismatch_distance <= self.epsilon * (1 + 1e-9)

    @property
    def mismatch_fraction(self) -> float:
        return self.mismatched_points / max(self.points, 1)

    def as_dict(self) -> dict:
        d = dict(self.__dict__)
        d.update(ok=self.ok, mismatch_fraction=self.mismatch_fraction)
        return d


def _candidate_pairs(packed: PackedRegions, xy: np.ndarray):
    """(point index, polygon index) pairs whose polygon MBR contains the point."""
    npoly = packed.n_polygons
    vstart = packed.ring_off[packed.poly_ring_off[:-1]]
    vend = packed.ring_off[packed.poly_ring_off[1:]]
    mnx = np.minimum.reduceat(packed.vx, vstart)
    mxx = np.maximum.reduceat(packed.vx, vstart)
    mny = np.minimum.reduceat(packed.vy, vstart)
    mxy = np.maximum.reduceat(packed.vy, vstart)
    x0, y0 = min(mnx.min(), xy[:, 0].min()), min(mny.min(), xy[:, 1].min())
    x1, y1 = max(mxx.max(), xy[:, 0].max()), max(mxy.max(), xy[:, 1].max())
    nb = max(1, int(np.sqrt(4 * npoly)))
    sx, sy = (x1 - x0) / nb or 1.0, (y1 - y0) / nb or 1.0
    bx0 = np.clip(((mnx - x0) / sx).astype(np.int64), 0, nb - 1)
    bx1 = np.clip(((mxx - x0) / sx).astype(np.int64), 0, nb - 1)
    by0 = np.clip(((mny - y0) / sy).astype(np.int64), 0, nb - 1)
    by1 = np.clip(((mxy - y0) / sy).astype(np.int64), 0, nb - 1)
    buckets = [[] for _ in range(nb * nb)]
    for p in range(npoly):
        for by in range(by0[p], by1[p] + 1):
            for bx in range(bx0[p], bx1[p] + 1):
                buckets[by * nb + bx].append(p)
    pb = np.clip(((xy[:, 0] - x0) / sx).astype(np.int64), 0, nb - 1) + nb * np.clip(
        ((xy[:, 1] - y0) / sy).astype(np.int64), 0, nb - 1)
    pts, polys = [], []
    for b in np.unique(pb):
        idx = np.nonzero(pb == b)[0]
        cand = np.asarray(buckets[b], np.int64)
        if len(cand) == 0:
            continue
        inm = ((xy[idx, None, 0] >= mnx[None, cand]) & (xy[idx, None, 0] <= mxx[None, cand]) &
               (xy[idx, None, 1] >= mny[None, cand]) & (xy[idx, None, 1] <= mxy[None, cand]))
        ii, cc = np.nonzero(inm)
        pts.append(idx[ii])
        polys.append(cand[cc])
    if not pts:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    return np.concatenate(pts), np.concatenate(polys)


def _exact(dev: DevicePolygons, xy: np.ndarray, pt: np.ndarray, poly: np.ndarray, fn: str) -> np.ndarray:
    torch = N.require_cuda()
    n = len(pt)
    if n == 0:
        return np.zeros(0, bool if fn == "pip" else np.float64)
    px = torch.as_tensor(np.ascontiguousarray(xy[pt, 0]), device="cuda")
    py = torch.as_tensor(np.ascontiguousarray(xy[pt, 1]), device="cuda")
    pp = torch.as_tensor(poly.astype(np.int32), device="cuda")
    L = N.load()
    if fn == "pip":
        out = torch.empty(n, dtype=torch.uint8, device="cuda")
        N.check(L.rb_exact_pip(C.byref(dev.desc), px.data_ptr(), py.data_ptr(), pp.data_ptr(), n, out.data_ptr(),
                               N.stream_ptr()), "validator pip")
        return out.bool().cpu().numpy()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    N.check(L.rb_exact_distance(C.byref(dev.desc), px.data_ptr(), py.data_ptr(), pp.data_ptr(), n, out.data_ptr(),
                                N.stream_ptr()), "validator distance")
    return out.cpu().numpy()


def validate(index: ApproxIndex, xy, epsilon: float, max_points: int | None = 200_000,
             seed: int = 0) -> ValidationReport:
    """Check the epsilon guarantee on (a seeded sample of) the points."""
    packed = index.packed
    xy = np.asarray(xy.cpu().numpy() if hasattr(xy, "cpu") else xy, dtype=np.float64).reshape(-1, 2)
    if max_points is not None and len(xy) > max_points:
        sel = np.sort(np.random.default_rng(seed).choice(len(xy), max_points, replace=False))
        xy = xy[sel]
    n = len(xy)
    R = packed.n_regions
    owners = index.decode(index.lookup(xy))
    approx = {(k, r) for k, lst in enumerate(owners) for r, _b in lst}
    dev = DevicePolygons(packed)
    pt, poly = _candidate_pairs(packed, xy)
    inside = _exact(dev, xy, pt, poly, "pip")
    exact = {(int(k), int(packed.poly_region[p])) for k, p, i in zip(pt, poly, inside) if i}
    fp = approx - exact
    fn = exact - approx
    mism = sorted(fp | fn)
    maxd = 0.0
    if mism:
        # distance to the region boundary = min over the region's polygons
        reg_polys = [np.nonzero(packed.poly_region == r)[0] for r in range(R)]
        mp_pt, mp_poly, mp_pair = [], [], []
        for j, (k, r) in enumerate(mism):
            for p in reg_polys[r]:
                mp_pt.append(k)
                mp_poly.append(p)
                mp_pair.append(j)
        d = _exact(dev, xy, np.asarray(mp_pt), np.asarray(mp_poly), "dist")
        best = np.full(len(mism), np.inf)
        np.minimum.at(best, np.asarray(mp_pair), d)
        maxd = float(best.max())
    return ValidationReport(n, len({k for k, _ in mism}), len(mism), len(fp), len(fn), maxd, float(epsilon))


__all__ = ["validate", "ValidationReport"]
