"""rasterbound.geometry: types and the exact primitives.

Types mirror SPEC.md:27-46.  The exact tests (point_in_polygon,
distance_to_boundary) run on the GPU through the C-ABI (rb_exact_pip /
rb_exact_distance) -- they are the epsilon validator of the north star, and
the same float64 predicate order as the rasterizer (boundary = inside,
SPEC.md:52,93).  Bulk inputs are columnar (`PointSet`); `list[PointRecord]`
is accepted and converted.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Mapping, Sequence

import numpy as np

from . import _native as N
from . import errors as E


@dataclass(frozen=True)
class Point2D:
    """SPEC.md:27-30."""
    x: float
    y: float


@dataclass(frozen=True)
class MBR:
    """SPEC.md:35-38."""
    min: Point2D
    max: Point2D


def _ring_array(ring) -> np.ndarray:
    if isinstance(ring, np.ndarray):
        a = np.asarray(ring, dtype=np.float64)
    else:
        pts = []
        for v in ring:
            if isinstance(v, Point2D):
                pts.append((v.x, v.y))
            else:
                pts.append((float(v[0]), float(v[1])))
        a = np.asarray(pts, dtype=np.float64).reshape(-1, 2)
    if a.ndim != 2 or a.shape[1] != 2:
        raise E.GeometryError("ring must be a sequence of (x, y) vertices")
    # rings are implicitly closed; drop an explicit closing vertex
    if len(a) >= 2 and a[0, 0] == a[-1, 0] and a[0, 1] == a[-1, 1]:
        a = a[:-1]
    if len(a) < 3:
        raise E.GeometryError(f"ring has {len(a)} vertices; at least 3 are required (SPEC.md:32)")
    if not np.all(np.isfinite(a)):
        raise E.GeometryError("ring has non-finite coordinates")
    return np.ascontiguousarray(a)


class Polygon:
    """Outer ring + holes; vertices stored as float64 [n, 2]."""

    __slots__ = ("outer", "holes")

    def __init__(self, outer, holes: Iterable = ()):
        self.outer = _ring_array(outer)
        self.holes = tuple(_ring_array(h) for h in holes)
        ar = _shoelace(self.outer)
        if ar == 0.0:
            raise E.GeometryError("outer ring has zero area (SPEC.md:33)")

    @property
    def rings(self) -> tuple:
        return (self.outer,) + self.holes

    def __repr__(self) -> str:
        return f"Polygon(outer={len(self.outer)} vertices, holes={len(self.holes)})"

    def __eq__(self, other) -> bool:
        return (isinstance(other, Polygon) and len(self.holes) == len(other.holes)
                and all(np.array_equal(a, b) for a, b in zip(self.rings, other.rings)))

    def __hash__(self) -> int:
        return hash(tuple(r.tobytes() for r in self.rings))


def _shoelace(a: np.ndarray) -> float:
    x, y = a[:, 0], a[:, 1]
    x2, y2 = np.roll(x, -1), np.roll(y, -1)
    return float(np.sum(x * y2 - x2 * y)) / 2.0


@dataclass
class PointRecord:
    """SPEC.md:39-42."""
    loc: Point2D
    attrs: dict = field(default_factory=dict)


@dataclass
class RegionRecord:
    """geometry is a Polygon or a list of Polygons (multi-polygon)."""
    id: int
    geometry: Polygon | list


@dataclass
class PointSet:
    """Columnar points: xy float64/float32 [N, 2] (numpy or torch) + named attributes [N]."""
    xy: object
    attrs: dict = field(default_factory=dict)

    def __len__(self) -> int:
        return int(self.xy.shape[0])


def as_point_set(points, attrs: Mapping | None = None) -> PointSet:
    """Accept PointSet, list[PointRecord], (N,2) arrays/tensors, or dict(x=, y=, **attrs)."""
    if isinstance(points, PointSet):
        if attrs:
            return PointSet(points.xy, {**points.attrs, **attrs})
        return points
    if isinstance(points, dict):
        xy = np.stack([np.asarray(points["x"], np.float64), np.asarray(points["y"], np.float64)], axis=1)
        rest = {k: v for k, v in points.items() if k not in ("x", "y")}
        return PointSet(xy, {**rest, **(attrs or {})})
    if isinstance(points, (list, tuple)):
        if len(points) == 0:
            return PointSet(np.zeros((0, 2), np.float64), dict(attrs or {}))
        if isinstance(points[0], PointRecord):
            xy = np.array([(p.loc.x, p.loc.y) for p in points], dtype=np.float64).reshape(-1, 2)
            names = list(points[0].attrs.keys())
            cols = {}
            for nm in names:
                try:
                    cols[nm] = np.array([p.attrs[nm] for p in points], dtype=np.float64)
                except KeyError as ex:
                    raise E.SchemaError(f"attribute {nm!r} missing on some points (SPEC.md:40)") from ex
            return PointSet(xy, {**cols, **(attrs or {})})
        if isinstance(points[0], Point2D):
            xy = np.array([(p.x, p.y) for p in points], dtype=np.float64).reshape(-1, 2)
            return PointSet(xy, dict(attrs or {}))
        return PointSet(np.asarray(points, dtype=np.float64).reshape(-1, 2), dict(attrs or {}))
    shape = getattr(points, "shape", None)
    if shape is not None and len(shape) == 2 and shape[1] == 2:
        return PointSet(points, dict(attrs or {}))
    raise E.ShapeError("points must be a PointSet, list of PointRecord/Point2D, or an (N, 2) array")


def mbr_of(poly: Polygon) -> MBR:
    """coordinate extrema of the outer ring."""
    o = poly.outer
    return MBR(Point2D(float(o[:, 0].min()), float(o[:, 1].min())), Point2D(float(o[:, 0].max()), float(o[:, 1].max())))


# ------------------------------------------------------------ CSR packing
@dataclass
class PackedRegions:
    """Polygon CSR shared by the native build and the oracle (host numpy)."""
    vx: np.ndarray
    vy: np.ndarray
    ring_off: np.ndarray
    poly_ring_off: np.ndarray
    poly_region: np.ndarray  # dense region index per polygon
    region_ids: np.ndarray  # dense index -> user region id

    @property
    def n_regions(self) -> int:
        return int(len(self.region_ids))

    @property
    def n_polygons(self) -> int:
        return int(len(self.poly_ring_off) - 1)

    def mbr(self) -> tuple[float, float, float, float]:
        return float(self.vx.min()), float(self.vy.min()), float(self.vx.max()), float(self.vy.max())


def _polys_of(geom) -> list:
    if isinstance(geom, Polygon):
        return [geom]
    if isinstance(geom, (list, tuple)) and geom and isinstance(geom[0], Polygon):
        return list(geom)
    if isinstance(geom, (list, tuple)) and not geom:
        raise E.GeometryError("region geometry is an empty multi-polygon")
    return [Polygon(geom)]


def pack_regions(regions: Sequence) -> PackedRegions:
    """RegionRecords (or bare Polygons, ids = position) -> CSR arrays."""
    vx, vy, ring_off, poly_ring_off, poly_region, ids = [], [], [0], [0], [], []
    seen = set()
    for k, r in enumerate(regions):
        if isinstance(r, RegionRecord):
            rid, geom = int(r.id), r.geometry
        else:
            rid, geom = k, r
        if rid in seen:
            raise E.ConfigError(f"duplicate region id {rid} (SPEC.md:45)")
        seen.add(rid)
        ridx = len(ids)
        ids.append(rid)
        for poly in _polys_of(geom):
            for ring in poly.rings:
                vx.append(ring[:, 0])
                vy.append(ring[:, 1])
                ring_off.append(ring_off[-1] + len(ring))
            poly_ring_off.append(len(ring_off) - 1)
            poly_region.append(ridx)
    if not ids:
        raise E.ConfigError("no regions")
    return PackedRegions(np.ascontiguousarray(np.concatenate(vx)), np.ascontiguousarray(np.concatenate(vy)),
                         np.asarray(ring_off, np.int64), np.asarray(poly_ring_off, np.int64),
                         np.asarray(poly_region, np.int32), np.asarray(ids, np.int64))


class DevicePolygons:
    """Device copy of a PackedRegions + the rb_polygons descriptor."""

    def __init__(self, packed: PackedRegions, device=None):
        torch = N.require_cuda()
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.packed = packed
        self.vx = torch.from_numpy(packed.vx).to(dev)
        self.vy = torch.from_numpy(packed.vy).to(dev)
        self.ring_off = torch.from_numpy(packed.ring_off).to(dev)
        self.poly_ring_off = torch.from_numpy(packed.poly_ring_off).to(dev)
        self.poly_region = torch.from_numpy(packed.poly_region).to(dev)
        self.desc = N.Polygons(self.vx.data_ptr(), self.vy.data_ptr(), len(packed.vx), self.ring_off.data_ptr(),
                               len(packed.ring_off) - 1, self.poly_ring_off.data_ptr(), len(packed.poly_ring_off) - 1,
                               self.poly_region.data_ptr(), packed.n_regions)


# ------------------------------------------------------------ exact tests
def _exact(poly: Polygon, px: np.ndarray, py: np.ndarray, fn: str):
    torch = N.require_cuda()
    L = N.load()
    dp = DevicePolygons(pack_regions([poly]))
    n = len(px)
    dx = torch.as_tensor(np.ascontiguousarray(px, np.float64), device="cuda")
    dy = torch.as_tensor(np.ascontiguousarray(py, np.float64), device="cuda")
    pp = torch.zeros(max(n, 1), dtype=torch.int32, device="cuda")
    if fn == "pip":
        out = torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")
        N.check(L.rb_exact_pip(C.byref(dp.desc), dx.data_ptr(), dy.data_ptr(), pp.data_ptr(), n, out.data_ptr(),
                               N.stream_ptr()), "point_in_polygon")
        return out[:n].bool().cpu().numpy()
    out = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    N.check(L.rb_exact_distance(C.byref(dp.desc), dx.data_ptr(), dy.data_ptr(), pp.data_ptr(), n, out.data_ptr(),
                                N.stream_ptr()), "distance_to_boundary")
    return out[:n].cpu().numpy()


def point_in_polygon(p: Point2D, poly: Polygon) -> bool:
    """SPEC.md:49-57 (boundary = inside)."""
    return bool(_exact(poly, np.array([p.x]), np.array([p.y]), "pip")[0])


def points_in_polygon(xy, poly: Polygon) -> np.ndarray:
    a = np.asarray(xy, np.float64).reshape(-1, 2)
    return _exact(poly, a[:, 0], a[:, 1], "pip")


def distance_to_boundary(p: Point2D, poly: Polygon) -> float:
    """min distance to any ring segment."""
    return float(_exact(poly, np.array([p.x]), np.array([p.y]), "dist")[0])


def distances_to_boundary(xy, poly: Polygon) -> np.ndarray:
    a = np.asarray(xy, np.float64).reshape(-1, 2)
    return _exact(poly, a[:, 0], a[:, 1], "dist")


def hausdorff_distance(A, B, step: float | None = None) -> float:
    """symmetric Hausdorff distance of two point samples.

    A and B are (n, 2) samples (the grid-sampled oracle; `step` is the
    documented slack and does not change the computation)."""
    torch = N.require_cuda()
    a = torch.as_tensor(np.asarray(A, np.float64).reshape(-1, 2), device="cuda")
    b = torch.as_tensor(np.asarray(B, np.float64).reshape(-1, 2), device="cuda")
    if a.shape[0] == 0 or b.shape[0] == 0:
        raise E.DomainError("empty sample set (SPEC.md:71)")

    def directed(x, y):
        best = torch.empty(x.shape[0], dtype=torch.float64, device="cuda")
        for i in range(0, x.shape[0], 4096):
            d = torch.cdist(x[i:i + 4096], y)
            best[i:i + 4096] = d.min(dim=1).values
        return best.max()

    return float(torch.maximum(directed(a, b), directed(b, a)).item())


__all__ = [
    "Point2D", "MBR", "Polygon", "PointRecord", "RegionRecord", "PointSet", "as_point_set", "mbr_of",
    "point_in_polygon", "points_in_polygon", "distance_to_boundary", "distances_to_boundary", "hausdorff_distance",
    "PackedRegions", "pack_regions", "DevicePolygons",
]
