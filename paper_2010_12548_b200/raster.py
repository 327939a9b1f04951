"""rasterbound.raster: epsilon-bounded coverings.

Coverings are computed on the GPU (csrc/rb_build.cu: edge walk K2, scanline
K3, quadtree descent K4) and exported as `RasterApprox` cell arrays.  The
semantic ledger is in DESIGN.md ("Semantics S1-S7"):
  * a leaf is PARTIAL iff the polygon boundary meets its OPEN square;
  * a non-PARTIAL cell is INSIDE iff its centre is inside (even-odd);
  * CONSERVATIVE keeps every PARTIAL leaf, CENTER_SAMPLED keeps it iff its
    centre is inside (boundary = inside);
  * the hierarchical covering is the top-down descent that splits a block
    iff the boundary meets its open interior, so uniform == hierarchical as
    point sets by construction.
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import errors as E
from .geometry import Point2D, Polygon, RegionRecord, pack_regions
from .grid import CellId, GridConfig, level_for_bound, point_to_cell

UNIFORM_CELL_CAP = 1 << 27


class RasterMode(enum.IntEnum):
    """SPEC.md:197-200."""
    CONSERVATIVE = N.MODE_CONSERVATIVE
    CENTER_SAMPLED = N.MODE_CENTER_SAMPLED


class CellClass(enum.Enum):
    INSIDE = "INSIDE"
    OUTSIDE = "OUTSIDE"
    PARTIAL = "PARTIAL"


KIND_I, KIND_B = 1, 2


@dataclass
class RasterApprox:
    """interior cells (any level <= L) + boundary cells (level L).

    Cells are kept as arrays (levels int32, codes uint64, kinds uint8 with
    1 = interior, 2 = boundary), sorted by level-L start code."""
    region_id: int
    epsilon: float
    mode: RasterMode
    grid: GridConfig
    levels: np.ndarray
    codes: np.ndarray
    kinds: np.ndarray

    @property
    def L(self) -> int:
        return self.grid.max_level

    def _cells(self, kind: int) -> frozenset:
        m = self.kinds == kind
        return frozenset(CellId(int(l), int(c)) for l, c in zip(self.levels[m], self.codes[m]))

    @property
    def interior(self) -> frozenset:
        return self._cells(KIND_I)

    @property
    def boundary(self) -> frozenset:
        return self._cells(KIND_B)

    @property
    def n_cells(self) -> int:
        return int(len(self.codes))

    def intervals(self):
        """Sorted half-open level-L code intervals [lo, hi) and their kinds."""
        sh = (2 * (self.L - self.levels.astype(np.int64))).astype(np.uint64)
        lo = self.codes.astype(np.uint64) << sh
        hi = (self.codes.astype(np.uint64) + np.uint64(1)) << sh
        o = np.argsort(lo, kind="stable")
        return lo[o], hi[o], self.kinds[o]

    def dump(self) -> str:
        """Covering dump format of SPEC.md:258: `region_id level code kind(I|B)`."""
        return "\n".join(f"{self.region_id} {int(l)} {int(c)} {'I' if k == KIND_I else 'B'}"
                         for l, c, k in zip(self.levels, self.codes, self.kinds))


def _union_cells(levels, codes, kinds, L):
    """Union of polygon coverings of one region: dedup, coarser cell wins,
    interior wins over boundary at equal cells."""
    if len(codes) == 0:
        return levels, codes, kinds
    lv = levels.astype(np.int64)
    sh = (2 * (L - lv)).astype(np.uint64)
    start = codes.astype(np.uint64) << sh
    end = (codes.astype(np.uint64) + np.uint64(1)) << sh
    o = np.lexsort((kinds, lv, start))
    keep = np.zeros(len(o), bool)
    cur_end = np.uint64(0)
    first = True
    for t, k in enumerate(o):
        if first or start[k] >= cur_end:
            keep[t] = True
            cur_end = end[k]
            first = False
        elif end[k] > cur_end:  # cannot happen for quadtree cells (nest or disjoint)
            raise E.GeometryError("non-nested cells in covering union")
    o = o[keep]
    return levels[o], codes[o], kinds[o]


def _build(geom, cfg: GridConfig, epsilon: float, mode: RasterMode):
    from .engine import ApproxIndex

    L = level_for_bound(cfg, epsilon)
    grid = cfg.with_level(L)
    packed = pack_regions([RegionRecord(0, geom)])
    idx = ApproxIndex(packed, grid, int(mode), layout="trie", keep_cells=True)
    return idx, grid, L


def rasterize_hierarchical(poly, cfg: GridConfig, epsilon: float,
                           mode: RasterMode = RasterMode.CONSERVATIVE, region_id: int = 0) -> RasterApprox:
    """SPEC.md:216-224 (poly may be a Polygon or a list of Polygons)."""
    idx, grid, L = _build(poly, cfg, epsilon, RasterMode(mode))
    p, lv, code, kind = idx.cells()
    if idx.packed.n_polygons > 1:
        lv, code, kind = _union_cells(lv, code, kind, L)
    else:
        sh = (2 * (L - lv.astype(np.int64))).astype(np.uint64)
        o = np.lexsort((lv, code.astype(np.uint64) << sh))
        lv, code, kind = lv[o], code[o], kind[o]
    return RasterApprox(region_id, float(epsilon), RasterMode(mode), grid, lv.astype(np.int32), code.astype(np.uint64),
                        kind.astype(np.uint8))


def expand_uniform(r: RasterApprox) -> RasterApprox:
    """All cells expanded to level L."""
    L = r.L
    d = (L - r.levels.astype(np.int64))
    sizes = np.left_shift(np.int64(1), 2 * d)
    total = int(sizes.sum()) if len(sizes) else 0
    if total > UNIFORM_CELL_CAP:
        raise E.CapacityError(f"uniform covering has {total} leaves (cap {UNIFORM_CELL_CAP}); use the hierarchical form")
    starts = (r.codes.astype(np.uint64) << (2 * d).astype(np.uint64)).astype(np.int64)
    rep = np.repeat(np.arange(len(sizes)), sizes)
    off = np.arange(total, dtype=np.int64) - np.repeat(np.cumsum(sizes) - sizes, sizes)
    codes = (starts[rep] + off).astype(np.uint64)
    kinds = r.kinds[rep]
    o = np.argsort(codes, kind="stable")
    return RasterApprox(r.region_id, r.epsilon, r.mode, r.grid, np.full(total, L, np.int32), codes[o], kinds[o])


def rasterize_uniform(poly, cfg: GridConfig, epsilon: float, mode: RasterMode = RasterMode.CONSERVATIVE,
                      region_id: int = 0) -> RasterApprox:
    """the hierarchical covering with every cell at level L."""
    return expand_uniform(rasterize_hierarchical(poly, cfg, epsilon, mode, region_id))


_CLASSIFY_CACHE: dict = {}


def classify_cell(c: CellId, poly: Polygon, cfg: GridConfig | None = None) -> CellClass:
    """INSIDE / OUTSIDE / PARTIAL for a cell of the grid `cfg`
    (default: unit square at origin).  PARTIAL iff the boundary meets the open
    cell; otherwise decided by the cell centre (D2)."""
    from .engine import ApproxIndex

    cfg = cfg or GridConfig(Point2D(0.0, 0.0), 1.0, 0)
    grid = cfg.with_level(c.level)
    key = (id(poly), grid.origin.x, grid.origin.y, grid.extent, c.level)
    hit = _CLASSIFY_CACHE.get(key)
    if hit is not None and hit[0] is poly:
        idx = hit[1]
    else:  # one index per (polygon, grid level), reused by further cells of that polygon
        idx = ApproxIndex(pack_regions([RegionRecord(0, poly)]), grid, N.MODE_CONSERVATIVE, layout="trie")
        if len(_CLASSIFY_CACHE) >= 8:
            _CLASSIFY_CACHE.pop(next(iter(_CLASSIFY_CACHE)))
        _CLASSIFY_CACHE[key] = (poly, idx)
    ix, iy = _decode(c)
    side = grid.side()
    centre = np.array([[cfg.origin.x + (ix + 0.5) * side, cfg.origin.y + (iy + 0.5) * side]])
    v = int(idx.lookup(centre).cpu().numpy().view(np.uint32)[0])
    if v == 0:
        return CellClass.OUTSIDE
    return CellClass.PARTIAL if ((v - 1) & 1) else CellClass.INSIDE


def _decode(c: CellId):
    from .grid import z_decode

    return z_decode(c)


def approx_contains(r: RasterApprox, p: Point2D) -> bool:
    """p's leaf lies in the interval of some covering cell."""
    leaf = point_to_cell(r.grid, p, r.L).code
    lo, hi, _ = r.intervals()
    k = int(np.searchsorted(lo, np.uint64(leaf), side="right")) - 1
    return k >= 0 and leaf < int(hi[k])


__all__ = [
    "RasterMode", "CellClass", "RasterApprox", "rasterize_hierarchical", "rasterize_uniform", "expand_uniform",
    "classify_cell", "approx_contains",
]
