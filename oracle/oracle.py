"""ORACLE -- test infrastructure only (see oracle/rb_oracle.c header).

ctypes binding of the C restatement `librb_oracle.so`.  Inputs are plain
numpy arrays in the polygon CSR layout used across the repo:

  vx, vy         float64 [V]   vertex coordinates (original units)
  ring_off       int64 [nrings+1]  vertex offsets of each ring
  poly_ring_off  int64 [npolys+1]  ring offsets of each polygon (ring 0 outer)
  poly_region    int32 [npolys]    region index (0..R-1) of each polygon

Results of `join` use the layout cnt[R,2] (alpha, beta) int64 and
sum[R,2] (alpha, beta) float64 -- SPEC.md:476-479 RegionResult.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "librb_oracle.so")

OK, GEOMETRY, DOMAIN, CAPACITY, CONFIG, SCHEMA, SHAPE = 0, -1, -2, -3, -4, -5, -6
KIND_NONE, KIND_I, KIND_B = 0, 1, 2


class OracleError(RuntimeError):
    def __init__(self, status: int, first_bad: int = -1):
        super().__init__(f"oracle status {status} (first_bad={first_bad})")
        self.status = status
        self.first_bad = first_bad


class _Grid(C.Structure):
    _fields_ = [("ox", C.c_double), ("oy", C.c_double), ("extent", C.c_double), ("level", C.c_int32)]


def build_lib(force: bool = False) -> str:
    src = os.path.join(_HERE, "rb_oracle.c")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build_lib()
        L = C.CDLL(_LIB)
        p = C.c_void_p
        L.orc_level_for_bound.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_int32)]
        L.orc_z_encode.argtypes = [C.c_uint32, C.c_uint32]
        L.orc_z_encode.restype = C.c_uint64
        L.orc_point_cells.argtypes = [C.POINTER(_Grid), p, C.c_int32, C.c_int64, p, p, C.POINTER(C.c_int64)]
        L.orc_build.argtypes = [C.POINTER(_Grid), p, p, C.c_int64, p, C.c_int64, p, C.c_int64, p, C.c_int32,
                                C.c_int32, C.POINTER(C.c_int32)]
        L.orc_build.restype = p
        L.orc_free.argtypes = [p]
        L.orc_join.argtypes = [p, p, C.c_int32, C.c_int64, p, p, p, C.POINTER(C.c_int64), C.c_int32]
        L.orc_lookup.argtypes = [p, p, C.c_int32, C.c_int64, p, p, p, C.c_int64, C.POINTER(C.c_int64)]
        L.orc_partial_leaves.argtypes = [p, C.c_int64, p, p]
        L.orc_partial_leaves.restype = C.c_int64
        L.orc_spans.argtypes = [p, C.c_int64, p, p, p]
        L.orc_spans.restype = C.c_int64
        L.orc_leaf_kinds.argtypes = [p, C.c_int64, p, p, C.c_int64, p]
        L.orc_hier_cells.argtypes = [p, C.c_int64, p, p, p, C.c_int64]
        L.orc_hier_cells.restype = C.c_int64
        L.orc_pip.argtypes = [p, p, p, C.c_int64, p, p, C.c_int64, p]
        L.orc_distance.argtypes = [p, p, p, C.c_int64, p, p, C.c_int64, p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def level_for_bound(extent: float, eps: float) -> int:
    out = C.c_int32(0)
    st = lib().orc_level_for_bound(float(extent), float(eps), C.byref(out))
    if st:
        raise OracleError(st)
    return int(out.value)


def z_encode(ix: int, iy: int) -> int:
    return int(lib().orc_z_encode(ix, iy))


def point_cells(grid, xy: np.ndarray):
    """grid = (ox, oy, extent, level); xy float64/float32 [N,2] -> (ix, iy)."""
    xy = np.ascontiguousarray(xy)
    dtype = 0 if xy.dtype == np.float64 else 1
    n = xy.shape[0]
    ix = np.empty(n, np.uint32)
    iy = np.empty(n, np.uint32)
    bad = C.c_int64(-1)
    g = _Grid(*grid)
    st = lib().orc_point_cells(C.byref(g), _ptr(xy), dtype, n, _ptr(ix), _ptr(iy), C.byref(bad))
    if st:
        raise OracleError(st, bad.value)
    return ix, iy


class Approx:
    """Oracle approximation of a region set (SPEC.md:216-224 + 276-284)."""

    def __init__(self, grid, vx, vy, ring_off, poly_ring_off, poly_region, nregions: int, mode: int):
        self.grid = tuple(grid)
        self.vx = np.ascontiguousarray(vx, np.float64)
        self.vy = np.ascontiguousarray(vy, np.float64)
        self.ring_off = np.ascontiguousarray(ring_off, np.int64)
        self.poly_ring_off = np.ascontiguousarray(poly_ring_off, np.int64)
        self.poly_region = np.ascontiguousarray(poly_region, np.int32)
        self.nregions = int(nregions)
        self.mode = int(mode)
        st = C.c_int32(0)
        g = _Grid(*grid)
        self._h = lib().orc_build(C.byref(g), _ptr(self.vx), _ptr(self.vy), len(self.vx), _ptr(self.ring_off),
                                  len(self.ring_off) - 1, _ptr(self.poly_ring_off), len(self.poly_ring_off) - 1,
                                  _ptr(self.poly_region), self.nregions, self.mode, C.byref(st))
        if not self._h:
            raise OracleError(st.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            try:
                _lib.orc_free(h)
            except Exception:
                pass
            self._h = None

    @property
    def npolys(self) -> int:
        return len(self.poly_ring_off) - 1

    def join(self, xy: np.ndarray, attr: np.ndarray | None = None, nthreads: int = 1):
        xy = np.ascontiguousarray(xy)
        dtype = 0 if xy.dtype == np.float64 else 1
        n = xy.shape[0]
        if attr is not None:
            attr = np.ascontiguousarray(attr, np.float32)
        cnt = np.zeros((self.nregions, 2), np.int64)
        sm = np.zeros((self.nregions, 2), np.float64)
        bad = C.c_int64(-1)
        st = lib().orc_join(self._h, _ptr(xy), dtype, n, _ptr(attr), _ptr(cnt), _ptr(sm), C.byref(bad), nthreads)
        if st:
            raise OracleError(st, bad.value)
        return cnt, sm

    def lookup(self, xy: np.ndarray):
        """Per point owner set: CSR (off, regions, kinds)."""
        xy = np.ascontiguousarray(xy)
        dtype = 0 if xy.dtype == np.float64 else 1
        n = xy.shape[0]
        cap = max(16, 8 * n)
        off = np.zeros(n + 1, np.int64)
        reg = np.empty(cap, np.int32)
        kind = np.empty(cap, np.uint8)
        bad = C.c_int64(-1)
        st = lib().orc_lookup(self._h, _ptr(xy), dtype, n, _ptr(off), _ptr(reg), _ptr(kind), cap, C.byref(bad))
        if st:
            raise OracleError(st, bad.value)
        return off, reg[: off[-1]].copy(), kind[: off[-1]].copy()

    def partial_leaves(self, p: int):
        n = lib().orc_partial_leaves(self._h, p, None, None)
        codes = np.empty(n, np.uint64)
        kept = np.empty(n, np.uint8)
        lib().orc_partial_leaves(self._h, p, _ptr(codes), _ptr(kept))
        return codes, kept.astype(bool)

    def spans(self, p: int):
        n = lib().orc_spans(self._h, p, None, None, None)
        rows = np.empty(n, np.int32)
        c0 = np.empty(n, np.int32)
        c1 = np.empty(n, np.int32)
        lib().orc_spans(self._h, p, _ptr(rows), _ptr(c0), _ptr(c1))
        return rows, c0, c1

    def leaf_kinds(self, p: int, i: np.ndarray, j: np.ndarray):
        i = np.ascontiguousarray(i, np.uint32)
        j = np.ascontiguousarray(j, np.uint32)
        out = np.empty(len(i), np.uint8)
        lib().orc_leaf_kinds(self._h, p, _ptr(i), _ptr(j), len(i), _ptr(out))
        return out

    def hier_cells(self, p: int):
        """Hierarchical covering of polygon p: (level, code, kind) arrays."""
        n = lib().orc_hier_cells(self._h, p, None, None, None, 0)
        lv = np.empty(n, np.int32)
        code = np.empty(n, np.uint64)
        kind = np.empty(n, np.uint8)
        lib().orc_hier_cells(self._h, p, _ptr(lv), _ptr(code), _ptr(kind), n)
        return lv, code, kind


def pip(vx, vy, ring_off, px, py) -> np.ndarray:
    """Exact PIP (boundary = inside) of points against ONE polygon's rings."""
    vx = np.ascontiguousarray(vx, np.float64)
    vy = np.ascontiguousarray(vy, np.float64)
    ring_off = np.ascontiguousarray(ring_off, np.int64)
    px = np.ascontiguousarray(px, np.float64)
    py = np.ascontiguousarray(py, np.float64)
    out = np.empty(len(px), np.uint8)
    lib().orc_pip(_ptr(vx), _ptr(vy), _ptr(ring_off), len(ring_off) - 1, _ptr(px), _ptr(py), len(px), _ptr(out))
    return out.astype(bool)


def distance(vx, vy, ring_off, px, py) -> np.ndarray:
    vx = np.ascontiguousarray(vx, np.float64)
    vy = np.ascontiguousarray(vy, np.float64)
    ring_off = np.ascontiguousarray(ring_off, np.int64)
    px = np.ascontiguousarray(px, np.float64)
    py = np.ascontiguousarray(py, np.float64)
    out = np.empty(len(px), np.float64)
    lib().orc_distance(_ptr(vx), _ptr(vy), _ptr(ring_off), len(ring_off) - 1, _ptr(px), _ptr(py), len(px), _ptr(out))
    return out
