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


def _bucket_grid(packed: PackedRegions, epsilon: float, extent_hint):
    """Uniform grid of polygon MBRs expanded by epsilon (CSR), for rb_validate_full."""
    npoly = packed.n_polygons
    vstart = packed.ring_off[packed.poly_ring_off[:-1]]
    vend = packed.ring_off[packed.poly_ring_off[1:]]
    mnx = np.minimum.reduceat(packed.vx, vstart)
    mxx = np.maximum.reduceat(packed.vx, vstart)
    mny = np.minimum.reduceat(packed.vy, vstart)
    mxy = np.maximum.reduceat(packed.vy, vstart)
    del vend
    x0, y0, ext = extent_hint
    nb = int(min(1024, max(1, np.sqrt(4 * npoly))))
    bs = max(ext / nb, 1e-300)
    pad = 2.0 * epsilon
    bx0 = np.clip(np.floor((mnx - pad - x0) / bs), 0, nb - 1).astype(np.int64)
    bx1 = np.clip(np.floor((mxx + pad - x0) / bs), 0, nb - 1).astype(np.int64)
    by0 = np.clip(np.floor((mny - pad - y0) / bs), 0, nb - 1).astype(np.int64)
    by1 = np.clip(np.floor((mxy + pad - y0) / bs), 0, nb - 1).astype(np.int64)
    counts = np.zeros(nb * nb + 1, np.int64)
    pairs_b, pairs_p = [], []
    for p in range(npoly):
        ys = np.arange(by0[p], by1[p] + 1)
        xs = np.arange(bx0[p], bx1[p] + 1)
        b = (ys[:, None] * nb + xs[None, :]).ravel()
        pairs_b.append(b)
        pairs_p.append(np.full(len(b), p, np.int32))
    pb = np.concatenate(pairs_b)
    pp = np.concatenate(pairs_p)
    o = np.argsort(pb, kind="stable")
    pb, pp = pb[o], pp[o]
    off = np.searchsorted(pb, np.arange(nb * nb + 1)).astype(np.int32)
    mbr = np.stack([mnx, mny, mxx, mxy], 1).astype(np.float64)
    return mbr, off, pp.astype(np.int32), nb, x0, y0, bs


@dataclass
class FullValidationReport:
    """Every point checked (not a sample)."""
    points: int
    mismatched_points: int
    false_positives: int
    false_negatives: int
    violations: int
    owner_set_overflows: int
    max_mismatch_distance: float
    epsilon: float

    @property
    def ok(self) -> bool:
        return self.violations == 0 and self.owner_set_overflows == 0

    @property
    def mismatch_fraction(self) -> float:
        return self.mismatched_points / max(self.points, 1)

    def as_dict(self) -> dict:
        d = dict(self.__dict__)
        d.update(ok=self.ok, mismatch_fraction=self.mismatch_fraction)
        return d


def validate_full(index: ApproxIndex, xy, epsilon: float) -> FullValidationReport:
    """The complete validator (rb_validate_full): every point's approximate
    owner regions against its exact owner regions; every mismatch must lie
    within epsilon of the region's boundary."""
    torch = N.require_cuda()
    packed = index.packed
    g = index.grid
    mbr, off, bp, nb, bx0, by0, bs = _bucket_grid(packed, epsilon, (g.origin.x, g.origin.y, g.extent))
    dev = DevicePolygons(packed)
    t_mbr = torch.as_tensor(mbr).cuda()
    t_off = torch.as_tensor(off).cuda()
    t_bp = torch.as_tensor(bp if len(bp) else np.zeros(1, np.int32)).cuda()
    t_xy, dt = index._xy(xy)
    out = (C.c_int64 * 6)()
    md = C.c_double()
    N.check(N.load().rb_validate_full(index._h, C.byref(dev.desc), t_mbr.data_ptr(), t_off.data_ptr(),
                                      t_bp.data_ptr(), nb, bx0, by0, bs, t_xy.data_ptr(), dt, int(t_xy.shape[0]),
                                      float(epsilon), out, C.byref(md), N.stream_ptr()), "validate_full")
    return FullValidationReport(int(out[0]), int(out[1]), int(out[2]), int(out[3]), int(out[4]), int(out[5]),
                                float(md.value), float(epsilon))


__all__ = ["validate", "ValidationReport", "validate_full", "FullValidationReport"]
