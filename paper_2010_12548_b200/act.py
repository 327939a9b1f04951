"""rasterbound.act: the Adaptive Cell Trie, B200 layout.

The trie is a radix table resident in HBM (csrc/rb_build.cu, index_impl):
a dense root table of level-T0 cells followed by node levels of
`radix_width` bits (radix_width/2 quadtree levels) each, aligned at the leaf
level.  A slot holds either a child pointer or the complete owner value of
its cell; coarse cells are prefix-expanded into the slots they cover, so a
lookup reads one slot per level instead of collecting terminal lists -- the
result is the same set.  `root_level = 0` gives the
reference's pure radix trie (depth ceil(2l / radix_width)); the default
root level keeps the upper levels in one L2-resident table.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import errors as E
from .engine import ApproxIndex
from .geometry import Point2D
from .grid import GridConfig
from .raster import KIND_B, RasterApprox


@dataclass
class AdaptiveCellTrie:
    """SPEC.md:270-273."""
    radix_width: int
    grid: GridConfig | None
    region_ids: np.ndarray
    index: ApproxIndex | None

    def stats(self) -> dict:
        return self.index.stats() if self.index is not None else {}


def _layout_code(layout: str) -> int:
    from .engine import LAYOUTS

    if layout not in LAYOUTS:
        raise E.ConfigError(f"unknown layout {layout!r} (dense | trie | keys | packed)")
    return LAYOUTS[layout]


def act_build(coverings, radix_width: int = 8, root_level: int = -1, layout: str = "trie") -> AdaptiveCellTrie:
    """insert every interior/boundary cell with its region id."""
    torch = N.require_cuda()
    if radix_width not in (2, 4, 8):
        raise E.ConfigError("radix_width must be 2, 4 or 8 (SPEC.md:278)")
    coverings = list(coverings)
    if not coverings:
        return AdaptiveCellTrie(radix_width, None, np.zeros(0, np.int64), None)
    g0 = coverings[0].grid
    for r in coverings:
        if not isinstance(r, RasterApprox):
            raise E.ConfigError("act_build expects RasterApprox coverings")
        if (r.grid.origin, r.grid.extent, r.grid.max_level) != (g0.origin, g0.extent, g0.max_level):
            raise E.ConfigError("coverings use different grid configurations (SPEC.md:280)")
    ids = sorted({int(r.region_id) for r in coverings})
    dense = {rid: k for k, rid in enumerate(ids)}
    cov_region = np.array([dense[int(r.region_id)] for r in coverings], np.int32)
    cov = np.concatenate([np.full(r.n_cells, k, np.int32) for k, r in enumerate(coverings)])
    lv = np.concatenate([r.levels.astype(np.uint8) for r in coverings])
    code = np.concatenate([r.codes.astype(np.uint64) for r in coverings])
    kind = np.concatenate([r.kinds.astype(np.uint8) for r in coverings])
    n = len(code)
    d = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a) if len(a) else np.zeros(1, a.dtype)).to("cuda")
    t_cov, t_lv, t_code, t_kind = d(cov, None), d(lv, None), d(code.view(np.int64), None), d(kind, None)
    t_reg = d(cov_region, None)
    g = g0.native()
    opts = N.BuildOpts(0, _layout_code(layout), radix_width, int(root_level), 0)
    h = C.c_void_p()
    N.check(N.load().rb_index_from_cells(C.byref(g), n, t_cov.data_ptr(), t_lv.data_ptr(), t_code.data_ptr(),
                                         t_kind.data_ptr(), t_reg.data_ptr(), len(coverings), len(ids), C.byref(opts),
                                         N.stream_ptr(), C.byref(h)), "act_build")
    idx = ApproxIndex.from_handle(h, g0, len(ids), layout, radix_width)
    return AdaptiveCellTrie(radix_width, g0, np.asarray(ids, np.int64), idx)


def _from_cells(grid: GridConfig, radix_width: int, region_ids, levels, codes, kinds,
                layout: str = "trie") -> AdaptiveCellTrie:
    """Index from explicit (region id, level, code, kind) cells (one covering per region)."""
    torch = N.require_cuda()
    region_ids = np.asarray(region_ids, np.int64)
    ids = sorted({int(r) for r in region_ids.tolist()})
    dense = {rid: k for k, rid in enumerate(ids)}
    cov = np.array([dense[int(r)] for r in region_ids.tolist()], np.int32)
    cov_region = np.arange(len(ids), dtype=np.int32)
    d = lambda a: torch.as_tensor(np.ascontiguousarray(a) if len(a) else np.zeros(1, a.dtype)).to("cuda")  # noqa
    t_cov, t_lv = d(cov), d(np.asarray(levels, np.uint8))
    t_code, t_kind = d(np.asarray(codes, np.uint64).view(np.int64)), d(np.asarray(kinds, np.uint8))
    t_reg = d(cov_region)
    opts = N.BuildOpts(0, _layout_code(layout), radix_width, -1, 0)
    h = C.c_void_p()
    N.check(N.load().rb_index_from_cells(C.byref(grid.native()), len(cov), t_cov.data_ptr(), t_lv.data_ptr(),
                                         t_code.data_ptr(), t_kind.data_ptr(), t_reg.data_ptr(), len(ids), len(ids),
                                         C.byref(opts), N.stream_ptr(), C.byref(h)), "act load")
    idx = ApproxIndex.from_handle(h, grid, len(ids), layout, radix_width)
    return AdaptiveCellTrie(radix_width, grid, np.asarray(ids, np.int64), idx)


def save_act(path: str, coverings, radix_width: int = 8) -> None:
    """ACT file: versioned magic, radix_width, grid, then the
    covering cells the device index is rebuilt from (formats.write_act)."""
    from .formats import write_act

    coverings = list(coverings)
    if not coverings:
        raise E.ConfigError("no coverings to save")
    rid = np.concatenate([np.full(r.n_cells, int(r.region_id), np.int64) for r in coverings])
    lv = np.concatenate([r.levels for r in coverings])
    code = np.concatenate([r.codes for r in coverings])
    kind = np.concatenate([r.kinds for r in coverings])
    write_act(path, coverings[0].grid, radix_width, rid, lv, code, kind)


def load_act(path: str, layout: str = "trie") -> AdaptiveCellTrie:
    """Rebuild the index saved by save_act (identical lookups)."""
    from .formats import read_act

    grid, rw, rid, lv, code, kind = read_act(path)
    return _from_cells(grid, rw, rid, lv, code, kind, layout)


def act_lookup_many(t: AdaptiveCellTrie, xy) -> list[set]:
    """Batched act_lookup: per point the set of (region_id, 'I'|'B')."""
    a = np.asarray(xy.cpu().numpy() if hasattr(xy, "cpu") else xy)
    n = a.shape[0] if a.ndim == 2 else 0
    if t.index is None:
        return [set() for _ in range(n)]
    vals = t.index.lookup(xy)
    out = []
    for owners in t.index.decode(vals):
        out.append({(int(t.region_ids[r]), "B" if b else "I") for r, b in owners})
    return out


def act_lookup(t: AdaptiveCellTrie, p: Point2D) -> set:
    """every (region_id, kind) whose covering contains p's leaf."""
    return act_lookup_many(t, np.array([[p.x, p.y]], np.float64))[0]


__all__ = ["AdaptiveCellTrie", "act_build", "act_lookup", "act_lookup_many", "save_act", "load_act"]
