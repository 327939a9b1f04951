"""rasterbound.query: approximate spatial aggregation.

`join_act` builds the approximation + cell index on the GPU and runs the
streaming point pass (csrc/rb_point_pass.cu); `PreparedJoin` keeps the
index resident for repeated joins (the hot path the benchmark times).
`join_canvas` is the Bounded Raster Join contract: the
same leaf-level semantics evaluated on the dense canvas layout, so it equals
join_act exactly.  `result_range` implements SPEC.md:509-517.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _native as N
from . import errors as E
from .engine import ApproxIndex, PassResult
from .geometry import PackedRegions, PointSet, as_point_set, pack_regions
from .grid import GridConfig, ingest_grid, level_for_bound
from .raster import RasterMode

UNAVAILABLE = None  # "range unavailable" marker
EMPTY = float("nan")  # AVG over an empty selection


@dataclass(frozen=True)
class Agg:
    """COUNT | SUM(attr) | AVG(attr)."""
    kind: str = "COUNT"
    attr: str | None = None

    def __post_init__(self):
        k = self.kind.upper()
        object.__setattr__(self, "kind", k)
        if k not in ("COUNT", "SUM", "AVG"):
            raise E.ConfigError(f"unknown aggregate {self.kind!r}")
        if k != "COUNT" and not self.attr:
            raise E.ConfigError(f"{k} needs an attribute")

    @staticmethod
    def parse(a) -> "Agg":
        if isinstance(a, Agg):
            return a
        if isinstance(a, str):
            s = a.strip()
            if ":" in s:  # CLI form sum:attr / avg:attr
                k, at = s.split(":", 1)
                return Agg(k, at)
            return Agg(s)
        if isinstance(a, (tuple, list)) and len(a) == 2:
            return Agg(a[0], a[1])
        raise E.ConfigError(f"cannot parse aggregate {a!r}")

    def __str__(self) -> str:
        return self.kind if self.kind == "COUNT" else f"{self.kind}({self.attr})"


_OPS = {"<": "lt", "<=": "le", ">": "gt", ">=": "ge", "==": "eq", "!=": "ne"}


@dataclass(frozen=True)
class AggregationQuery:
    """SPEC.md:472-475.  filter: None, (attr, op, value) or callable(attrs) -> bool mask."""
    agg: Agg | str | tuple = "COUNT"
    epsilon: float = 1.0
    mode: RasterMode = RasterMode.CONSERVATIVE
    filter: tuple | Callable | None = None

    def __post_init__(self):
        object.__setattr__(self, "agg", Agg.parse(self.agg))
        object.__setattr__(self, "mode", RasterMode(self.mode))
        if not (self.epsilon > 0.0) or not math.isfinite(self.epsilon):
            raise E.ConfigError("epsilon must be finite and > 0 (SPEC.md:474)")


@dataclass
class RegionResult:
    """alpha, boundary part beta, guaranteed range when derivable."""
    region_id: int
    alpha: float
    boundary_part: float
    range: tuple | None = None

    def to_json(self, q: AggregationQuery, engine: str = "act") -> str:
        lo, hi = self.range if self.range is not None else (None, None)
        return json.dumps({"region_id": self.region_id, "alpha": self.alpha, "beta": self.boundary_part, "lo": lo,
                           "hi": hi, "agg": str(q.agg), "epsilon": q.epsilon, "mode": q.mode.name, "engine": engine})


def result_range(rr: RegionResult, q: AggregationQuery, nonnegative: bool = True):
    """[alpha - beta, alpha] iff CONSERVATIVE and (COUNT or a
    SUM over non-negative values -- the caller's precondition, checked on the
    data by PreparedJoin); otherwise the unavailable marker."""
    if q.mode != RasterMode.CONSERVATIVE or q.agg.kind == "AVG":
        return UNAVAILABLE
    if q.agg.kind == "SUM" and not nonnegative:
        return UNAVAILABLE
    return (rr.alpha - rr.boundary_part, rr.alpha)


# ------------------------------------------------------------------ joins
def _grid_for(points: PointSet, packed: PackedRegions, cfg: GridConfig | None) -> GridConfig:
    if cfg is not None:
        return cfg
    torch = N.require_cuda()
    x0, y0, x1, y1 = packed.mbr()
    if len(points):
        xy = points.xy if isinstance(points.xy, torch.Tensor) else torch.as_tensor(np.asarray(points.xy))
        mn = xy.min(dim=0).values.double().cpu().numpy()
        mx = xy.max(dim=0).values.double().cpu().numpy()
        if not (np.all(np.isfinite(mn)) and np.all(np.isfinite(mx))):
            raise E.DomainError("non-finite point coordinates (SPEC.md:29)")
        x0, y0 = min(x0, float(mn[0])), min(y0, float(mn[1]))
        x1, y1 = max(x1, float(mx[0])), max(y1, float(mx[1]))
    return ingest_grid(x0, y0, x1, y1)


def _apply_filter(points: PointSet, flt) -> PointSet:
    if flt is None:
        return points
    torch = N.require_cuda()
    cols = {}
    for k, v in points.attrs.items():
        cols[k] = v if isinstance(v, torch.Tensor) else torch.as_tensor(np.asarray(v))
        cols[k] = cols[k].to("cuda")
    if callable(flt):
        mask = torch.as_tensor(flt(cols), device="cuda").bool()
    else:
        attr, op, val = flt
        if attr not in cols:
            raise E.SchemaError(f"filter attribute {attr!r} not in the point schema (SPEC.md:359)")
        if op not in _OPS:
            raise E.ConfigError(f"unknown filter operator {op!r}")
        mask = getattr(cols[attr], _OPS[op])(val)
    xy = points.xy if isinstance(points.xy, torch.Tensor) else torch.as_tensor(np.asarray(points.xy))
    xy = xy.to("cuda")
    return PointSet(xy[mask], {k: v[mask] for k, v in cols.items()})


class PreparedJoin:
    """An immutable, device-resident approximation + index for one region set
    and query (SPEC.md:304 concurrency: safe for concurrent joins)."""

    def __init__(self, regions, q: AggregationQuery, cfg: GridConfig, layout: str = "trie", radix_width: int = 8,
                 root_level: int = -1, keep_cells: bool = False):
        self.q = q
        self.packed = regions if isinstance(regions, PackedRegions) else pack_regions(regions)
        L = level_for_bound(cfg, q.epsilon)
        self.grid = cfg.with_level(L)
        self.layout = layout
        self.index = ApproxIndex(self.packed, self.grid, int(q.mode), layout=layout, radix_width=radix_width,
                                 root_level=root_level, keep_cells=keep_cells)

    @property
    def n_regions(self) -> int:
        return self.packed.n_regions

    def stats(self) -> dict:
        return self.index.stats()

    def _attr(self, points: PointSet):
        a = self.q.agg
        if a.kind == "COUNT":
            return None
        if a.attr not in points.attrs:
            raise E.SchemaError(f"attribute {a.attr!r} not in the point schema (SPEC.md:359)")
        return points.attrs[a.attr]

    def run_device(self, points, out: PassResult | None = None, accumulate: bool = False, stream=None) -> PassResult:
        """Device-side join: returns device tensors, no host sync."""
        ps = _apply_filter(as_point_set(points), self.q.filter)
        return self.index.point_pass(ps.xy, self._attr(ps), out=out, accumulate=accumulate, stream=stream)

    def run(self, points) -> list:
        ps = as_point_set(points)
        r = self.run_device(ps).check()
        return self.results(r.cnt.cpu().numpy(), r.sum.cpu().numpy(), ps)

    def run_host(self, points) -> list:
        """Join from host buffers through rb_join_host (chunked H2D overlap)."""
        ps = _apply_filter(as_point_set(points), self.q.filter)
        xy = ps.xy
        attr = self._attr(ps)
        if hasattr(xy, "is_cuda") and xy.is_cuda:
            xy = xy.cpu()
        if attr is not None and hasattr(attr, "is_cuda") and attr.is_cuda:
            attr = attr.cpu()
        if attr is not None and not hasattr(attr, "data_ptr"):
            attr = np.ascontiguousarray(attr, np.float32)
        cnt, sm = self.index.join_host(xy if hasattr(xy, "data_ptr") else np.asarray(xy), attr)
        return self.results(cnt, sm, ps)

    def results(self, cnt: np.ndarray, sm: np.ndarray, points: PointSet | None = None) -> list:
        return _results(self.packed, self.q, cnt, sm, points)


def _results(packed: PackedRegions, q: AggregationQuery, cnt: np.ndarray, sm: np.ndarray,
             points: PointSet | None = None, nonneg: bool | None = None) -> list:
    """RegionResult per region from [R,2] alpha/beta COUNT and SUM."""
    a = q.agg
    if nonneg is None:
        nonneg = True
        if a.kind != "COUNT" and points is not None:
            v = points.attrs.get(a.attr)
            if v is not None:
                nonneg = bool((v.min() >= 0).item()) if len(v) else True
    out = []
    for k, rid in enumerate(packed.region_ids.tolist()):
        ac, bc = int(cnt[k, 0]), int(cnt[k, 1])
        if a.kind == "COUNT":
            alpha, beta = ac, bc
        elif a.kind == "SUM":
            alpha, beta = float(sm[k, 0]), float(sm[k, 1])
        else:
            alpha = float(sm[k, 0]) / ac if ac else EMPTY
            beta = float(sm[k, 1]) / bc if bc else EMPTY
        rr = RegionResult(int(rid), alpha, beta)
        rr.range = result_range(rr, q, nonneg)
        out.append(rr)
    return out


def join_act(points, regions, q: AggregationQuery, cfg: GridConfig | None = None, layout: str = "trie",
             radix_width: int = 8) -> list:
    """rasterize regions (hierarchical, epsilon, mode), build the
    ACT, stream every point passing the filter, accumulate into every matched
    region with boundary contributions tracked separately."""
    ps = as_point_set(points)
    packed = pack_regions(regions)
    cfg = _grid_for(ps, packed, cfg)
    return PreparedJoin(packed, q, cfg, layout=layout, radix_width=radix_width).run(ps)


def _region_cells(packed: PackedRegions, index: ApproxIndex, L: int):
    """Disjoint covering cells per region: a multi-polygon
    region's coverings are unioned, a cell inside a coarser cell of the same
    region is dropped (the coarser wins), identical cells keep interior if any
    polygon has it interior.  Returns (region, level, code, kind) grouped by region."""
    poly, level, code, kind = index.cells()
    region = packed.poly_region[poly].astype(np.int32)
    counts = np.bincount(packed.poly_region, minlength=packed.n_regions)
    multi = counts[region] > 1
    if multi.any():
        keep = ~multi
        lv = level.astype(np.int64)
        lo = code.astype(np.uint64) << (2 * (L - lv)).astype(np.uint64)
        hi = (code.astype(np.uint64) + np.uint64(1)) << (2 * (L - lv)).astype(np.uint64)
        idx = np.nonzero(multi)[0]
        # per region: by start, larger cells first, interior before boundary
        order = idx[np.lexsort((kind[idx], lv[idx], lo[idx], region[idx]))]
        kind = kind.copy()
        cur_r, cur_hi, cur_j = -1, np.uint64(0), -1
        for j in order.tolist():
            r = int(region[j])
            if r == cur_r and lo[j] < cur_hi:  # nested in (or identical to) the kept cell
                if lo[j] == lo[cur_j] and hi[j] == cur_hi and kind[j] == 1:
                    kind[cur_j] = 1
                continue
            keep[j] = True
            cur_r, cur_hi, cur_j = r, hi[j], j
        region, level, code, kind = region[keep], level[keep], code[keep], kind[keep]
    if len(region) > 1 and not np.all(region[1:] >= region[:-1]):  # cells come grouped by polygon already
        o = np.argsort(region, kind="stable")
        region, level, code, kind = region[o], level[o], code[o], kind[o]
    return region, level.astype(np.int32), code, kind.astype(np.uint8)


class PreparedPointIndexJoin:
    """The region side of join_pointindex, built once per (regions, epsilon,
    mode): the hierarchical coverings as disjoint per-region cells on the
    device.  run() answers the query from a point index."""

    def __init__(self, regions, q: AggregationQuery, grid: GridConfig):
        torch = N.require_cuda()
        if q.filter is not None:
            raise E.ConfigError("join_pointindex aggregates prefix sums over all points; filters need join_act")
        self.q = q
        self.packed = regions if isinstance(regions, PackedRegions) else pack_regions(regions)
        L = level_for_bound(grid, q.epsilon)
        self.grid = grid.with_level(L)
        index = ApproxIndex(self.packed, self.grid, int(q.mode), layout="trie", keep_cells=True)
        region, level, code, kind = _region_cells(self.packed, index, L)
        del index
        self.n_cells = int(len(region))
        self._region = torch.as_tensor(region).cuda()
        self._level = torch.as_tensor(level).cuda()
        self._code = torch.as_tensor(code.view(np.int64)).cuda()
        self._kind = torch.as_tensor(kind).cuda()

    def run_device(self, lps, rs=None, stream=None):
        """Per-region [R,2] alpha/beta COUNT (int64) and SUM (float64) device tensors."""
        torch = N.require_cuda()
        if lps.grid.max_level != self.grid.max_level:
            raise E.ConfigError(f"point index built at level {lps.grid.max_level}, "
                                f"query epsilon needs level {self.grid.max_level}")
        a = self.q.agg
        attr_idx = -1
        if a.kind != "COUNT":
            if a.attr not in lps.attrs:
                raise E.SchemaError(f"attribute {a.attr!r} has no prefix array in the point index (SPEC.md:359)")
            attr_idx = lps.attrs.index(a.attr)
        R = self.packed.n_regions
        cnt = torch.zeros((R, 2), dtype=torch.int64, device="cuda")
        sm = torch.zeros((R, 2), dtype=torch.float64, device="cuda")
        N.check(N.load().rb_join_pointindex(lps._h, rs._h if rs is not None else None, self.n_cells,
                                            self._region.data_ptr(), self._level.data_ptr(), self._code.data_ptr(),
                                            self._kind.data_ptr(), R, attr_idx, cnt.data_ptr(), sm.data_ptr(),
                                            N.stream_ptr(stream)), "join_pointindex")
        return cnt, sm

    def run(self, lps, rs=None) -> list:
        cnt, sm = self.run_device(lps, rs)
        a = self.q.agg
        nonneg = True
        if a.kind != "COUNT":
            pre = lps.prefix(a.attr)
            nonneg = bool((pre[1:] - pre[:-1] >= 0).all().item()) if lps.n else True
        return _results(self.packed, self.q, cnt.cpu().numpy(), sm.cpu().numpy(), nonneg=nonneg)


def join_pointindex(lps, rs, regions, q: AggregationQuery) -> list:
    """per region, its covering (hierarchical raster at the
    query's epsilon and mode) as cell intervals, each aggregated from the point
    index with two lower-bound lookups and a prefix difference
    (pointindex.range_aggregate); beta from the boundary cells only.  Equals
    join_act exactly for COUNT."""
    return PreparedPointIndexJoin(regions, q, lps.grid).run(lps, rs)


CANVAS_MAX_LEVEL = 17


def join_canvas(points, regions, q: AggregationQuery, cfg: GridConfig | None = None, plan: str = "fused") -> list:
    """SPEC.md:500-508 (Bounded Raster Join): point canvas x region canvases at
    the resolution chosen from epsilon.  plan="fused" (default) evaluates it as
    one pass over the dense canvas layout (pixel = leaf cell);
    plan="algebra" runs the literal canvas plan (canvas.brj: render_points,
    per region render_polygon -> mask -> reduce, tiled at 2^13 per side)."""
    ps = as_point_set(points)
    packed = pack_regions(regions)
    cfg = _grid_for(ps, packed, cfg)
    if plan == "algebra":
        from .canvas import brj

        if q.filter is not None:
            ps = _apply_filter(ps, q.filter)
        cnt, sm = brj(ps, packed, q, cfg)
        return _results(packed, q, cnt, sm, ps)
    if plan != "fused":
        raise E.ConfigError(f"unknown join_canvas plan {plan!r} (fused | algebra)")
    L = level_for_bound(cfg, q.epsilon)
    if L > CANVAS_MAX_LEVEL:
        raise E.CapacityError(f"canvas resolution 2^{L} exceeds the dense limit 2^{CANVAS_MAX_LEVEL}; use join_act")
    return PreparedJoin(packed, q, cfg, layout="dense").run(ps)


__all__ = [
    "Agg", "AggregationQuery", "RegionResult", "result_range", "PreparedJoin", "join_act", "join_canvas",
    "join_pointindex", "PreparedPointIndexJoin",
    "UNAVAILABLE", "EMPTY",
]
