"""rasterbound.canvas (section 4): the canvas data
model and its blend / mask / affine operator algebra, the substrate of the
Bounded Raster Join (query.join_canvas).

A Canvas is a device-resident 2^level x 2^level tile of the level-L leaf grid
(pixel (ix, iy) = leaf z_encode(ix, iy, L)) with channels count,
SUM channels, region id (-1 = none) and flags (non-empty, boundary).  Every
operator runs as a kernel of librasterbound_b200.so (csrc/rb_canvas.cu); the
canvases are immutable values (operators return new canvases).
Tiles are capped at 2^13 per side: brj() tiles finer grids.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from . import _native as N
from . import errors as E
from .geometry import PackedRegions, Polygon, RegionRecord, as_point_set, pack_regions
from .grid import GridConfig
from .raster import RasterMode

CANVAS_MAX_LEVEL = 13


class BlendFn(IntEnum):
    """SUM (associative, commutative), OVERWRITE (b over a), MAX."""
    SUM = 0
    OVERWRITE = 1
    MAX = 2


@dataclass(frozen=True)
class MaskPredicate:
    """SPEC.md:397-400.  kind: NONEMPTY | REGION_EQ(arg) | BOUNDARY_ONLY |
    COUNT_GT(arg) | COVERED_BY(canvas) | BOUNDARY_OF(canvas)."""
    kind: str = "NONEMPTY"
    arg: int = 0
    canvas: "Canvas | None" = None

    _CODES = {"NONEMPTY": 0, "REGION_EQ": 1, "BOUNDARY_ONLY": 2, "COUNT_GT": 3, "COVERED_BY": 4, "BOUNDARY_OF": 5}

    @staticmethod
    def nonempty():
        return MaskPredicate("NONEMPTY")

    @staticmethod
    def region_eq(rid: int):
        return MaskPredicate("REGION_EQ", int(rid))

    @staticmethod
    def boundary_only():
        return MaskPredicate("BOUNDARY_ONLY")

    @staticmethod
    def count_gt(k: int):
        return MaskPredicate("COUNT_GT", int(k))

    @staticmethod
    def covered_by(c: "Canvas"):
        return MaskPredicate("COVERED_BY", 0, c)

    @staticmethod
    def boundary_of(c: "Canvas"):
        return MaskPredicate("BOUNDARY_OF", 0, c)


@dataclass(frozen=True)
class AffineTransform:
    """integer-pixel translation, then axis flips."""
    dx: float = 0
    dy: float = 0
    flip_x: bool = False
    flip_y: bool = False


class Canvas:
    """SPEC.md:389-392."""

    def __init__(self, cfg: GridConfig, L: int, level: int | None = None, x0: int = 0, y0: int = 0,
                 sum_attrs=()):
        torch = N.require_cuda()
        level = L if level is None else level
        if level > 16 or level < 0 or level > L:
            raise E.CapacityError(f"canvas tile level {level} out of range (grid level {L})")
        self.grid = cfg.with_level(L)
        self.L, self.level, self.x0, self.y0 = int(L), int(level), int(x0), int(y0)
        self.sum_attrs = tuple(sum_attrs)
        W = 1 << level
        self.count = torch.zeros((W, W), dtype=torch.int64, device="cuda")
        self.sums = torch.zeros((max(len(self.sum_attrs), 1), W, W), dtype=torch.float64, device="cuda")
        self.region = torch.full((W, W), -1, dtype=torch.int32, device="cuda")
        self.flags = torch.zeros((W, W), dtype=torch.uint8, device="cuda")

    # ------------------------------------------------------------ views
    @property
    def width(self) -> int:
        return 1 << self.level

    height = width

    @property
    def empty(self):
        """Per-pixel empty marker."""
        return (self.flags & 1) == 0

    @property
    def boundary_flag(self):
        return (self.flags & 2) != 0

    @property
    def region_id(self):
        return self.region

    def sum(self, attr: str):
        if attr not in self.sum_attrs:
            raise E.SchemaError(f"canvas has no SUM channel {attr!r}")
        return self.sums[self.sum_attrs.index(attr)]

    def like(self) -> "Canvas":
        return Canvas(self.grid, self.L, self.level, self.x0, self.y0, self.sum_attrs)

    def desc(self) -> N.CanvasDesc:
        return N.CanvasDesc(self.level, self.x0, self.y0, len(self.sum_attrs), self.count.data_ptr(),
                            self.sums.data_ptr(), self.region.data_ptr(), self.flags.data_ptr())

    # ------------------------------------------------------------ debug export
    def to_csv(self, path: str, channel: str = "count") -> None:
        a = (self.count if channel == "count" else self.region if channel == "region" else self.sum(channel)).cpu()
        np.savetxt(path, a.numpy(), delimiter=",", fmt="%g")

    def to_pgm(self, path: str, channel: str = "count") -> None:
        a = (self.count if channel == "count" else self.region if channel == "region" else self.sum(channel)).cpu()
        a = a.numpy().astype(np.float64)
        m = a.max() if a.size and a.max() > 0 else 1.0
        img = np.clip(a / m * 255.0, 0, 255).astype(np.uint8)[::-1]
        with open(path, "wb") as f:
            f.write(f"P5 {img.shape[1]} {img.shape[0]} 255\n".encode())
            f.write(img.tobytes())


def _same(a: Canvas, b: Canvas) -> None:
    if a.level != b.level or a.sum_attrs != b.sum_attrs:
        raise E.ShapeError("canvas dimensions or channels differ (SPEC.md:425)")


def render_points(points, cfg: GridConfig, L: int, agg_channels=(), level: int | None = None, x0: int = 0,
                  y0: int = 0, lps=None) -> Canvas:
    """per pixel COUNT and the SUM channels of the points in
    its leaf cell (from a point index built here, or the given one)."""
    from .pointindex import lps_build

    grid = cfg.with_level(L)
    if lps is None:
        lps = lps_build(as_point_set(points), grid, agg_channels)
    elif lps.grid.max_level != L:
        raise E.ConfigError("point index level differs from the canvas level")
    names = tuple(agg_channels)
    if names != tuple(lps.attrs[:len(names)]):
        raise E.SchemaError("SUM channels must be the point index's leading attributes")
    c = Canvas(grid, L, level, x0, y0, names)
    d = c.desc()
    N.check(N.load().rb_canvas_render_points(lps._h, C.byref(d), N.stream_ptr()), "render_points")
    return c


def _render_cells(c: Canvas, level, code, kind, rid: int, clear: bool = True) -> Canvas:
    torch = N.require_cuda()
    lv = torch.as_tensor(np.asarray(level, np.int32)).cuda()
    cd = torch.as_tensor(np.asarray(code, np.uint64).view(np.int64)).cuda()
    kd = torch.as_tensor(np.asarray(kind, np.uint8)).cuda()
    d = c.desc()
    N.check(N.load().rb_canvas_render_cells(int(len(lv)), lv.data_ptr(), cd.data_ptr(), kd.data_ptr(), c.L, int(rid),
                                            1 if clear else 0, C.byref(d), N.stream_ptr()), "render_polygon")
    return c


def render_polygon(poly, cfg: GridConfig, L: int, mode: RasterMode = RasterMode.CONSERVATIVE, id: int = 0,
                   level: int | None = None, x0: int = 0, y0: int = 0) -> Canvas:
    """pixels = the leaf expansion of rasterize_uniform(poly,
    eps(L), mode); region_id set, boundary_flag on boundary cells."""
    from .engine import ApproxIndex

    grid = cfg.with_level(L)
    geom = poly if isinstance(poly, (Polygon, list)) else Polygon(poly)
    packed = pack_regions([RegionRecord(int(id), geom)])
    idx = ApproxIndex(packed, grid, int(RasterMode(mode)), layout="trie", keep_cells=True)
    from .query import _region_cells

    _, lv, code, kind = _region_cells(packed, idx, L)
    return _render_cells(Canvas(grid, L, level, x0, y0), lv, code, kind, int(id))


def blend(a: Canvas, b: Canvas, f: BlendFn = BlendFn.SUM) -> Canvas:
    """SPEC.md:421-428."""
    _same(a, b)
    out = a.like()
    da, db, do = a.desc(), b.desc(), out.desc()
    N.check(N.load().rb_canvas_blend(C.byref(da), C.byref(db), int(BlendFn(f)), C.byref(do), N.stream_ptr()), "blend")
    return out


def mask(a: Canvas, m: MaskPredicate) -> Canvas:
    """pixels failing m become empty, the others unchanged."""
    code = MaskPredicate._CODES.get(m.kind)
    if code is None:
        raise E.ConfigError(f"unknown mask predicate {m.kind!r}")
    by = None
    if code >= 4:
        if m.canvas is None:
            raise E.ConfigError(f"{m.kind} needs a canvas")
        if m.canvas.level != a.level:
            raise E.ShapeError("mask canvas of another size")
        by = m.canvas.desc()
    out = a.like()
    da, do = a.desc(), out.desc()
    N.check(N.load().rb_canvas_mask(C.byref(da), code, int(m.arg), C.byref(by) if by is not None else None,
                                    C.byref(do), N.stream_ptr()), "mask")
    return out


def affine(a: Canvas, t: AffineTransform) -> Canvas:
    """payloads moved, pixels mapped outside drop; only
    integer-pixel translations and axis flips (else UnsupportedTransform)."""
    if float(t.dx) != int(t.dx) or float(t.dy) != int(t.dy):
        raise E.UnsupportedTransform("affine: only integer-pixel translations and axis flips (SPEC.md:440)")
    out = a.like()
    da, do = a.desc(), out.desc()
    N.check(N.load().rb_canvas_affine(C.byref(da), int(t.dx), int(t.dy), 1 if t.flip_x else 0, 1 if t.flip_y else 0,
                                      C.byref(do), N.stream_ptr()), "affine")
    return out


def reduce(a: Canvas):
    """Totals over non-empty pixels: (count, boundary count, {attr: (sum, boundary sum)})."""
    torch = N.require_cuda()
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    sm = torch.zeros((max(len(a.sum_attrs), 1), 2), dtype=torch.float64, device="cuda")
    d = a.desc()
    N.check(N.load().rb_canvas_reduce(C.byref(d), cnt.data_ptr(), sm.data_ptr(), N.stream_ptr()), "reduce")
    c = cnt.cpu().numpy()
    s = sm.cpu().numpy()
    return int(c[0]), int(c[1]), {k: (float(s[i, 0]), float(s[i, 1])) for i, k in enumerate(a.sum_attrs)}


def _compact1by1(v: np.ndarray) -> np.ndarray:
    """Even bits of Morton codes (x of z_encode)."""
    v = np.asarray(v, np.uint64) & np.uint64(0x5555555555555555)
    for sh, m in ((1, 0x3333333333333333), (2, 0x0F0F0F0F0F0F0F0F), (4, 0x00FF00FF00FF00FF),
                  (8, 0x0000FFFF0000FFFF), (16, 0x00000000FFFFFFFF)):
        v = (v | (v >> np.uint64(sh))) & np.uint64(m)
    return v


def brj(points, regions, q, cfg: GridConfig, tile_level: int = CANVAS_MAX_LEVEL):
    """The Bounded Raster Join plan written in the canvas algebra:
    per region, over Z-aligned canvas tiles covering its pixel bounding box
    (at most 2^tile_level per side): render_points, render_polygon
    (the region's covering cells), mask the point canvas by it, reduce
    (boundary pixels separately into beta).  Tiles are sized to the region, so
    the work is proportional to the region's pixels; the per-tile reductions
    stay on the device and are summed per region on the host in a fixed order.
    Returns [R,2] alpha/beta COUNT and SUM arrays (dense region order)."""
    from .engine import ApproxIndex
    from .grid import level_for_bound
    from .pointindex import lps_build
    from .query import _region_cells

    torch = N.require_cuda()
    lib = N.load()
    ps = as_point_set(points)
    packed = regions if isinstance(regions, PackedRegions) else pack_regions(regions)
    L = level_for_bound(cfg, q.epsilon)
    grid = cfg.with_level(L)
    a = q.agg
    attrs = () if a.kind == "COUNT" else (a.attr,)
    lps = lps_build(ps, grid, attrs)
    idx = ApproxIndex(packed, grid, int(q.mode), layout="trie", keep_cells=True)
    region, level, code, kind = _region_cells(packed, idx, L)
    del idx
    R = packed.n_regions
    beg = np.searchsorted(region, np.arange(R + 1))
    cnt = np.zeros((R, 2), np.int64)
    sm = np.zeros((R, 2), np.float64)
    if len(region) == 0:
        return cnt, sm
    lv_d = torch.as_tensor(np.asarray(level, np.int32)).cuda()
    cd_d = torch.as_tensor(np.asarray(code, np.uint64).view(np.int64)).cuda()
    kd_d = torch.as_tensor(np.asarray(kind, np.uint8)).cuda()
    # leaf-pixel extent of every cell
    c64 = np.asarray(code, np.uint64)
    sh = (L - np.asarray(level, np.int64)).astype(np.int64)
    cx = _compact1by1(c64).astype(np.int64)
    cy = _compact1by1(c64 >> np.uint64(1)).astype(np.int64)
    px0, px1, py0, py1 = cx << sh, (cx + 1) << sh, cy << sh, (cy + 1) << sh
    cap = min(L, tile_level, CANVAS_MAX_LEVEL)
    jobs = []
    for r in range(R):
        lo, hi = int(beg[r]), int(beg[r + 1])
        if lo == hi:
            continue
        bx0, bx1 = int(px0[lo:hi].min()), int(px1[lo:hi].max())
        by0, by1 = int(py0[lo:hi].min()), int(py1[lo:hi].max())
        w = max(bx1 - bx0, by1 - by0)
        tl = min(cap, max(0, int(math.ceil(math.log2(w)))))
        for ty in range(by0 >> tl, ((by1 - 1) >> tl) + 1):
            for tx in range(bx0 >> tl, ((bx1 - 1) >> tl) + 1):
                jobs.append((r, lo, hi, tl, tx, ty))
    nsum = max(len(attrs), 1)
    cnt_t = torch.zeros((len(jobs), 2), dtype=torch.int64, device="cuda")
    sum_t = torch.zeros((len(jobs), nsum, 2), dtype=torch.float64, device="cuda")
    canv = {}
    st = N.stream_ptr()
    covered = MaskPredicate._CODES["COVERED_BY"]
    for k, (r, lo, hi, tl, tx, ty) in enumerate(jobs):
        if tl not in canv:
            canv[tl] = tuple(Canvas(grid, L, tl, 0, 0, attrs) for _ in range(3))
        pc, rc, mc = canv[tl]
        for c in (pc, rc, mc):
            c.x0, c.y0 = tx << tl, ty << tl
        dp, dr, dm = pc.desc(), rc.desc(), mc.desc()
        N.check(lib.rb_canvas_render_points(lps._h, C.byref(dp), st), "render_points")
        N.check(lib.rb_canvas_render_cells(hi - lo, lv_d[lo:hi].data_ptr(), cd_d[lo:hi].data_ptr(),
                                           kd_d[lo:hi].data_ptr(), L, int(r), 1, C.byref(dr), st), "render_polygon")
        N.check(lib.rb_canvas_mask(C.byref(dp), covered, 0, C.byref(dr), C.byref(dm), st), "mask")
        N.check(lib.rb_canvas_reduce(C.byref(dm), cnt_t[k].data_ptr(), sum_t[k].data_ptr(), st), "reduce")
    c_h = cnt_t.cpu().numpy()
    s_h = sum_t.cpu().numpy()
    for k, job in enumerate(jobs):
        r = job[0]
        cnt[r] += c_h[k]
        if attrs:
            sm[r] += s_h[k, 0]
    return cnt, sm


__all__ = ["Canvas", "BlendFn", "MaskPredicate", "AffineTransform", "render_points", "render_polygon", "blend", "mask",
           "affine", "reduce", "brj", "CANVAS_MAX_LEVEL"]
