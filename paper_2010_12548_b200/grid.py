"""rasterbound.grid: square quadtree domain, Z-order codes.

Scalar helpers are host arithmetic (pure integer / IEEE float64, identical
to the device code); the batched point -> cell map runs on the GPU
(rb_point_cells).  Conventions: Morton with x in the even
bits, half-open cells, level cap 31.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import errors as E
from .geometry import Point2D


@dataclass(frozen=True)
class GridConfig:
    """origin, extent (square side), max_level L in [0, 31]."""
    origin: Point2D
    extent: float
    max_level: int = 0

    def __post_init__(self):
        if not isinstance(self.origin, Point2D):
            object.__setattr__(self, "origin", Point2D(float(self.origin[0]), float(self.origin[1])))
        if not (self.extent > 0.0) or not math.isfinite(self.extent):
            raise E.ConfigError("GridConfig.extent must be finite and > 0 (SPEC.md:113)")
        if not (0 <= int(self.max_level) <= 31):
            raise E.CapacityError("GridConfig.max_level must lie in [0, 31] (SPEC.md:112)")

    def side(self, level: int | None = None) -> float:
        return math.ldexp(self.extent, -(self.max_level if level is None else level))

    def with_level(self, level: int) -> "GridConfig":
        return GridConfig(self.origin, self.extent, level)

    def native(self, level: int | None = None) -> N.Grid:
        return N.Grid(self.origin.x, self.origin.y, self.extent, self.max_level if level is None else level)


@dataclass(frozen=True, order=True)
class CellId:
    """SPEC.md:115-118."""
    level: int
    code: int

    def __post_init__(self):
        if not (0 <= self.level <= 31):
            raise E.DomainError(f"cell level {self.level} outside [0, 31]")
        if not (0 <= self.code < (1 << (2 * self.level))):
            raise E.DomainError(f"cell code {self.code} outside [0, 4^{self.level})")


@dataclass(frozen=True)
class CellInterval:
    """half-open [lo, hi) over max-level codes."""
    lo: int
    hi: int

    def __contains__(self, code: int) -> bool:
        return self.lo <= code < self.hi


def level_for_bound(cfg: GridConfig, epsilon: float) -> int:
    """SPEC.md:125-133 (computed by the native library, same rule as the device)."""
    out = C.c_int32(0)
    N.check(N.load().rb_level_for_bound(float(cfg.extent), float(epsilon), C.byref(out)), "level_for_bound")
    return int(out.value)


def _spread(v: int) -> int:
    r = 0
    b = 0
    while v:
        if v & 1:
            r |= 1 << (2 * b)
        v >>= 1
        b += 1
    return r


def _compact(v: int) -> int:
    r = 0
    b = 0
    while v:
        if v & 1:
            r |= 1 << b
        v >>= 2
        b += 1
    return r


def z_encode(ix: int, iy: int, level: int) -> CellId:
    """bit i of ix -> bit 2i, bit i of iy -> bit 2i+1."""
    if not (0 <= level <= 31):
        raise E.DomainError(f"level {level} outside [0, 31]")
    if not (0 <= ix < (1 << level) and 0 <= iy < (1 << level)):
        raise E.DomainError(f"cell coordinates ({ix}, {iy}) outside [0, 2^{level})")
    return CellId(level, _spread(ix) | (_spread(iy) << 1))


def z_decode(c: CellId) -> tuple[int, int]:
    return _compact(c.code), _compact(c.code >> 1)


def point_to_cell(cfg: GridConfig, p: Point2D, level: int) -> CellId:
    """z_encode(floor((p - origin) / side)) with half-open cells."""
    side = math.ldexp(cfg.extent, -level)
    u = (p.x - cfg.origin.x) / side
    v = (p.y - cfg.origin.y) / side
    lim = 1 << level
    if not (u >= 0.0 and v >= 0.0):
        raise E.DomainError(f"point ({p.x}, {p.y}) outside the grid domain (SPEC.md:147)")
    ix, iy = math.floor(u), math.floor(v)
    if ix >= lim or iy >= lim:
        raise E.DomainError(f"point ({p.x}, {p.y}) outside the grid domain (SPEC.md:147)")
    return z_encode(ix, iy, level)


def points_to_cells(cfg: GridConfig, xy, level: int | None = None):
    """Batched point_to_cell on the GPU: returns (ix, iy) uint32 torch tensors."""
    torch = N.require_cuda()
    t = xy if isinstance(xy, torch.Tensor) else torch.as_tensor(np.asarray(xy))
    if t.dtype not in (torch.float64, torch.float32):
        t = t.to(torch.float64)
    t = t.to("cuda").contiguous()
    n = int(t.shape[0])
    ix = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    iy = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    bad = torch.empty(1, dtype=torch.int64, device="cuda")
    g = cfg.native(level)
    N.check(N.load().rb_point_cells(C.byref(g), t.data_ptr(), N.XY_F64 if t.dtype == torch.float64 else N.XY_F32, n,
                                    ix.data_ptr(), iy.data_ptr(), bad.data_ptr(), N.stream_ptr()), "point_to_cell")
    b = int(bad.item())
    if b != (1 << 63) - 1:
        raise E.DomainError(f"point {b} outside the grid domain (SPEC.md:147)", b)
    return ix[:n], iy[:n]


def cell_interval(c: CellId, L: int) -> CellInterval:
    """SPEC.md:152-160."""
    if c.level > L:
        raise E.DomainError(f"cell level {c.level} above max level {L}")
    sh = 2 * (L - c.level)
    return CellInterval(c.code << sh, (c.code + 1) << sh)


def children(c: CellId) -> tuple[CellId, CellId, CellId, CellId]:
    """SPEC.md:161-169."""
    if c.level >= 31:
        raise E.DomainError("children of a level-31 cell")
    return tuple(CellId(c.level + 1, 4 * c.code + k) for k in range(4))


def parent(c: CellId) -> CellId:
    if c.level <= 0:
        raise E.DomainError("parent of the root cell")
    return CellId(c.level - 1, c.code >> 2)


def ingest_grid(xmin: float, ymin: float, xmax: float, ymax: float, pad: float = 0.01) -> GridConfig:
    """SPEC.md:556 ingest rule: data MBR padded by 1% of its larger span on every side."""
    span = max(xmax - xmin, ymax - ymin)
    if not (span > 0.0):
        span = 1.0
    return GridConfig(Point2D(xmin - pad * span, ymin - pad * span), (1.0 + 2.0 * pad) * span, 0)


def eps_grid(xmin: float, ymin: float, xmax: float, ymax: float, epsilon: float, pad: float = 0.01) -> GridConfig:
    """epsilon-matched GridConfig: the leaf side is exactly epsilon/sqrt(2) (the paper's "diagonal of the
    cell is epsilon"), at the smallest level whose domain holds the data MBR padded as by the
    ingest rule.  The ingest grid instead fixes the extent and lets level_for_bound round the
    side down to a power-of-two fraction of it (up to 2x finer than epsilon requires).
    level_for_bound(eps_grid(..., epsilon), epsilon) is the returned max_level."""
    if not (epsilon > 0.0) or not math.isfinite(epsilon):
        raise E.ConfigError("epsilon must be finite and > 0")
    span = max(xmax - xmin, ymax - ymin)
    if not (span > 0.0):
        span = 1.0
    side = epsilon / math.sqrt(2.0)  # the same IEEE expression as rb_level_for_bound
    need = (1.0 + 2.0 * pad) * span
    L = 0
    while math.ldexp(side, L) < need:
        L += 1
        if L > 31:
            raise E.CapacityError("epsilon requires a level above 31 (SPEC.md:129)")
    return GridConfig(Point2D(xmin - pad * span, ymin - pad * span), math.ldexp(side, L), L)


__all__ = [
    "GridConfig", "CellId", "CellInterval", "level_for_bound", "z_encode", "z_decode", "point_to_cell",
    "points_to_cells", "cell_interval", "children", "parent", "ingest_grid", "eps_grid",
]
