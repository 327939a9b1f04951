"""rasterbound.pointindex: the point-side
access path for repeated polygon queries over a fixed point set.

Points are linearised once to their leaf Z codes (the same float64 point_to_cell
and z_encode as the join), sorted on the GPU with their permutation, and
float64 prefix sums of every configured attribute are kept beside the codes
(COUNT's prefix is the position itself).  A RadixSpline (greedy spline corridor
with error <= max_error at every stored key + a radix table over the top bits)
predicts lower-bound positions; a cell interval's aggregate is then two lookups
and a prefix difference.  All bulk work is rb_lps_build / rb_rs_build /
rb_bounds_lookup / rb_join_pointindex in librasterbound_b200.so (csrc/
rb_pointindex.cu); there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native as N
from . import errors as E
from .geometry import as_point_set
from .grid import CellInterval, GridConfig

EMPTY = float("nan")  # AVG over an empty selection


class LinearizedPointSet:
    """codes (sorted leaf codes, duplicates allowed), perm
    (sorted position -> point id), prefix arrays (n + 1, prefix[0] = 0) for
    COUNT and every configured SUM attribute, grid.  Device-resident and
    immutable; concurrent lookups are safe."""

    def __init__(self, handle: C.c_void_p, grid: GridConfig, attrs: tuple):
        self._h = handle
        self.grid = grid
        self.attrs = tuple(attrs)
        self._lib = N.load()
        self._torch = N.require_cuda()
        n = C.c_int64()
        codes, perm, prefix = C.c_void_p(), C.c_void_p(), C.c_void_p()
        na = C.c_int32()
        N.check(self._lib.rb_lps_info(self._h, C.byref(n), C.byref(codes), C.byref(perm), C.byref(prefix),
                                      C.byref(na)))
        self.n = int(n.value)
        self._codes, self._perm, self._prefix = codes.value, perm.value, prefix.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._torch.cuda.synchronize()
            except Exception:
                pass
            self._lib.rb_lps_free(h)
            self._h = None

    @property
    def handle(self) -> int:
        return self._h.value

    def _view(self, ptr, count: int, dtype):
        """Copy of a device array (count elements) as a torch tensor (via
        __cuda_array_interface__, then cloned so it outlives the handle)."""
        torch = self._torch
        if count <= 0:
            return torch.empty(0, dtype=dtype, device="cuda")
        typestr = {torch.int64: "<i8", torch.float64: "<f8", torch.int32: "<i4"}[dtype]

        class _Dev:
            __cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (int(ptr), False),
                                        "version": 3, "strides": None}

        torch.cuda.synchronize()
        return torch.as_tensor(_Dev(), device="cuda").clone()

    @property
    def codes(self):
        """Sorted level-L codes (torch int64 holding the uint64 values)."""
        return self._view(self._codes, self.n, self._torch.int64)

    @property
    def perm(self):
        return self._view(self._perm, self.n, self._torch.int64)

    def prefix(self, agg: str = "COUNT"):
        """Prefix array (n + 1) of COUNT or of a configured SUM attribute."""
        torch = self._torch
        if agg.upper() == "COUNT":
            return torch.arange(self.n + 1, dtype=torch.float64, device="cuda")
        if agg not in self.attrs:
            raise E.SchemaError(f"attribute {agg!r} has no prefix array (SPEC.md:359)")
        k = self.attrs.index(agg)
        return self._view(self._prefix + k * (self.n + 1) * 8, self.n + 1, torch.float64)


class RadixSplineIndex:
    """radix table over the top radix_bits of the code space,
    spline knots (key, position) strictly increasing in key, max_error tau."""

    def __init__(self, handle: C.c_void_p, lps: LinearizedPointSet, max_error: int):
        self._h = handle
        self.lps = lps
        self.max_error = int(max_error)
        self._lib = N.load()
        self._torch = lps._torch
        nk, keys, pos, table = C.c_int64(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        rb, sh = C.c_int32(), C.c_int32()
        N.check(self._lib.rb_rs_info(self._h, C.byref(nk), C.byref(keys), C.byref(pos), C.byref(table), C.byref(rb),
                                     C.byref(sh)))
        self.n_knots = int(nk.value)
        self.radix_bits = int(rb.value)
        self.shift = int(sh.value)
        self._keys, self._pos, self._table = keys.value, pos.value, table.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._torch.cuda.synchronize()
            except Exception:
                pass
            self._lib.rb_rs_free(h)
            self._h = None

    @property
    def handle(self) -> int:
        return self._h.value

    @property
    def knots(self):
        """(keys, positions) as torch int64 tensors (keys hold uint64 values)."""
        torch = self._torch
        return (self.lps._view(self._keys, self.n_knots, torch.int64),
                self.lps._view(self._pos, self.n_knots, torch.int64))

    @property
    def radix_table(self):
        return self.lps._view(self._table, (1 << self.radix_bits) + 1, self._torch.int32)


def lps_build(points, cfg: GridConfig, sum_attrs=()) -> LinearizedPointSet:
    """linearise, sort, and prefix-sum the points (all in the
    domain; an offender raises DomainError with its index)."""
    torch = N.require_cuda()
    ps = as_point_set(points)
    xy = ps.xy if isinstance(ps.xy, torch.Tensor) else torch.as_tensor(np.asarray(ps.xy))
    if xy.dtype not in (torch.float64, torch.float32):
        xy = xy.to(torch.float64)
    if len(xy) and (xy.dim() != 2 or xy.shape[1] != 2):
        raise E.ShapeError("points must be an (N, 2) array")
    xy = xy.reshape(-1, 2).to("cuda").contiguous()
    n = int(xy.shape[0])
    names = tuple(sum_attrs)
    cols = []
    for a in names:
        if a not in ps.attrs:
            raise E.SchemaError(f"unknown attribute {a!r} (SPEC.md:359)")
        v = ps.attrs[a]
        v = v if isinstance(v, torch.Tensor) else torch.as_tensor(np.asarray(v))
        v = v.to("cuda", dtype=torch.float32).contiguous()
        if int(v.shape[0]) != n:
            raise E.ShapeError(f"attribute {a!r} length differs from the point count")
        cols.append(v)
    ptrs = (C.c_void_p * max(len(cols), 1))(*[c.data_ptr() for c in cols])
    h = C.c_void_p()
    bad = C.c_int64(-1)
    lib = N.load()
    st = lib.rb_lps_build(C.byref(cfg.native()), xy.data_ptr() if n else None,
                          N.XY_F64 if xy.dtype == torch.float64 else N.XY_F32, n, ptrs, len(cols), N.stream_ptr(),
                          C.byref(h), C.byref(bad))
    N.check(st, "lps_build", bad.value if st == -2 else None)
    return LinearizedPointSet(h, cfg, names)


def rs_build(lps: LinearizedPointSet, radix_bits: int | None = None, max_error: int = 32) -> RadixSplineIndex:
    """SPEC.md:337-345.  An explicit radix_bits above the 2L-bit code width is a
    ConfigError; the default (the paper's 25 bits) is clamped to
    the code width and, at desk scale, to ceil(log2 n) + 1."""
    width = 2 * lps.grid.max_level
    if radix_bits is None:
        radix_bits = min(25, width)
    if radix_bits > width:
        raise E.ConfigError(f"radix_bits {radix_bits} exceeds the code width {width} (SPEC.md:340)")
    rb = int(max(0, min(radix_bits, math.ceil(math.log2(max(lps.n, 1))) + 1, 30)))
    h = C.c_void_p()
    N.check(N.load().rb_rs_build(lps._h, rb, int(max_error), N.stream_ptr(), C.byref(h)), "rs_build")
    return RadixSplineIndex(h, lps, max_error)


def save_point_index(path: str, lps: LinearizedPointSet, rs: RadixSplineIndex | None = None) -> None:
    """Index file: codes + prefix arrays + spline knots, versioned."""
    from .formats import write_point_index

    write_point_index(path, lps, rs)


def load_point_index(path: str):
    """-> (LinearizedPointSet, RadixSplineIndex | None) from save_point_index."""
    from .formats import read_point_index

    d = read_point_index(path)
    lib = N.load()
    n = len(d["codes"])
    codes = np.ascontiguousarray(d["codes"])
    perm = np.ascontiguousarray(d["perm"])
    pre = np.ascontiguousarray(np.concatenate([d["prefix"][a] for a in d["attrs"]])) if d["attrs"] else \
        np.zeros(1, np.float64)
    h = C.c_void_p()
    N.check(lib.rb_lps_from_arrays(C.byref(d["grid"].native()), n, codes.ctypes.data, perm.ctypes.data,
                                   pre.ctypes.data, len(d["attrs"]), N.stream_ptr(), C.byref(h)), "load_point_index")
    lps = LinearizedPointSet(h, d["grid"], tuple(d["attrs"]))
    rs = None
    if d["radix_bits"] >= 0:
        keys = np.ascontiguousarray(d["keys"])
        pos = np.ascontiguousarray(d["pos"])
        tab = np.ascontiguousarray(d["table"])
        hr = C.c_void_p()
        N.check(lib.rb_rs_from_arrays(lps._h, d["radix_bits"], d["max_error"], len(keys), keys.ctypes.data,
                                      pos.ctypes.data, tab.ctypes.data, N.stream_ptr(), C.byref(hr)),
                "load_point_index")
        rs = RadixSplineIndex(hr, lps, d["max_error"])
    return lps, rs


def _intervals(iv):
    torch = N.require_cuda()
    if isinstance(iv, CellInterval):
        lo, hi = np.array([iv.lo], np.uint64), np.array([iv.hi], np.uint64)
    else:
        lo, hi = iv
        lo = np.asarray(lo.cpu().numpy() if hasattr(lo, "cpu") else lo).astype(np.uint64)
        hi = np.asarray(hi.cpu().numpy() if hasattr(hi, "cpu") else hi).astype(np.uint64)
    return (torch.as_tensor(lo.view(np.int64)).cuda(), torch.as_tensor(hi.view(np.int64)).cuda())


def bounds_lookup(lps: LinearizedPointSet, rs: RadixSplineIndex | None, iv):
    """(first position with code >= lo, first with code >= hi),
    for one CellInterval or a batch (lo array, hi array).  With rs the
    positions are identical to binary search."""
    torch = lps._torch
    lo, hi = _intervals(iv)
    m = int(lo.shape[0])
    lo_pos = torch.empty(m, dtype=torch.int64, device="cuda")
    hi_pos = torch.empty(m, dtype=torch.int64, device="cuda")
    N.check(N.load().rb_bounds_lookup(lps._h, rs._h if rs is not None else None, lo.data_ptr(), hi.data_ptr(), m,
                                      lo_pos.data_ptr(), hi_pos.data_ptr(), N.stream_ptr()), "bounds_lookup")
    if isinstance(iv, CellInterval):
        return int(lo_pos[0]), int(hi_pos[0])
    return lo_pos, hi_pos


def range_aggregate(lps: LinearizedPointSet, rs: RadixSplineIndex | None, cells, agg="COUNT") -> float:
    """sum over (pairwise disjoint) cell intervals of
    prefix[hi] - prefix[lo]; AVG = SUM / COUNT with 0/0 -> the empty marker."""
    from .query import Agg

    a = Agg.parse(agg)
    ivs = list(cells)
    if not ivs:
        return EMPTY if a.kind == "AVG" else 0.0
    lo = np.array([c.lo for c in ivs], np.uint64)
    hi = np.array([c.hi for c in ivs], np.uint64)
    lo_pos, hi_pos = bounds_lookup(lps, rs, (lo, hi))
    cnt = float((hi_pos - lo_pos).sum().item())
    if a.kind == "COUNT":
        return cnt
    pre = lps.prefix(a.attr)
    s = float((pre[hi_pos] - pre[lo_pos]).sum().item())
    if a.kind == "SUM":
        return s
    return s / cnt if cnt else EMPTY


__all__ = ["LinearizedPointSet", "RadixSplineIndex", "lps_build", "rs_build", "bounds_lookup", "range_aggregate",
           "save_point_index", "load_point_index", "EMPTY"]
