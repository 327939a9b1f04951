"""ctypes binding of librasterbound_b200.so (include/rasterbound_b200.h).

The library is the only compute path: if it is missing or no CUDA device is
visible, every entry point raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

from . import errors as E

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RASTERBOUND_B200_LIB") or os.path.join(_HERE, "lib", "librasterbound_b200.so")

RB_OK = 0
_STATUS = {
    -1: E.GeometryError, -2: E.DomainError, -3: E.CapacityError, -4: E.ConfigError, -5: E.SchemaError,
    -6: E.ShapeError, -7: E.UnsupportedTransform,
}
MODE_CONSERVATIVE, MODE_CENTER_SAMPLED = 0, 1
LAYOUT_DENSE, LAYOUT_TRIE, LAYOUT_KEYS, LAYOUT_PACKED = 0, 1, 2, 3
XY_F64, XY_F32 = 0, 1
VALUE_LIST = 0x40000000
CODE_MASK = 0x3FFFF
MAX_HOT = 4095
VALUE_PAYLOAD = 0x3FFFFFFF

# every symbol include/rasterbound_b200.h declares
EXPORTS = (
    "rb_version", "rb_last_error", "rb_level_for_bound", "rb_approx_build", "rb_approx_stats", "rb_approx_free",
    "rb_point_pass", "rb_join_host", "rb_lookup", "rb_owner_pool", "rb_point_cells", "rb_approx_cells",
    "rb_approx_partial", "rb_exact_pip", "rb_exact_distance", "rb_index_from_cells", "rb_instrument", "rb_approx_set_hot",
    "rb_lps_build", "rb_lps_info", "rb_lps_free", "rb_rs_build", "rb_rs_info", "rb_rs_free", "rb_bounds_lookup",
    "rb_join_pointindex", "rb_canvas_clear", "rb_canvas_render_points", "rb_canvas_render_cells", "rb_canvas_blend",
    "rb_canvas_mask", "rb_canvas_affine", "rb_canvas_reduce", "rb_lps_from_arrays", "rb_rs_from_arrays",
    "rb_validate_full",
)


class Grid(C.Structure):
    _fields_ = [("origin_x", C.c_double), ("origin_y", C.c_double), ("extent", C.c_double), ("max_level", C.c_int32)]


class Polygons(C.Structure):
    _fields_ = [("vx", C.c_void_p), ("vy", C.c_void_p), ("n_vertices", C.c_int64), ("ring_off", C.c_void_p),
                ("n_rings", C.c_int64), ("poly_ring_off", C.c_void_p), ("n_polygons", C.c_int64),
                ("poly_region", C.c_void_p), ("n_regions", C.c_int32)]


class BuildOpts(C.Structure):
    _fields_ = [("mode", C.c_int32), ("layout", C.c_int32), ("radix_width", C.c_int32), ("root_level", C.c_int32),
                ("keep_cells", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("n_partial_leaves", C.c_int64), ("n_interior_cells", C.c_int64), ("n_boundary_cells", C.c_int64),
                ("n_uniform_interior", C.c_int64), ("n_positions", C.c_int64), ("n_multi_owner", C.c_int64),
                ("n_nodes", C.c_int64), ("index_bytes", C.c_int64), ("root_level", C.c_int32),
                ("node_levels", C.c_int32), ("n_regions", C.c_int32), ("max_level", C.c_int32),
                ("build_ms", C.c_double), ("max_hot", C.c_int32), ("n_hot", C.c_int32)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


class CanvasDesc(C.Structure):
    _fields_ = [("level", C.c_int32), ("x0", C.c_int64), ("y0", C.c_int64), ("n_sum", C.c_int32),
                ("count", C.c_void_p), ("sums", C.c_void_p), ("region", C.c_void_p), ("flags", C.c_void_p)]


_lib = None


def load() -> C.CDLL:
    """Load the native library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise E.ConfigError(
            f"native library missing: {LIB_PATH}; build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    p, i32, i64, d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    L.rb_version.restype = i32
    L.rb_last_error.restype = C.c_char_p
    L.rb_level_for_bound.argtypes = [d, d, C.POINTER(i32)]
    L.rb_approx_build.argtypes = [C.POINTER(Grid), C.POINTER(Polygons), C.POINTER(BuildOpts), p, C.POINTER(p)]
    L.rb_index_from_cells.argtypes = [C.POINTER(Grid), i64, p, p, p, p, p, i64, i32, C.POINTER(BuildOpts), p,
                                      C.POINTER(p)]
    L.rb_approx_stats.argtypes = [p, C.POINTER(Stats)]
    L.rb_approx_free.argtypes = [p]
    L.rb_approx_free.restype = None
    L.rb_point_pass.argtypes = [p, p, i32, i64, p, p, p, p, i32, p]
    L.rb_join_host.argtypes = [p, p, i32, i64, p, p, p, p]
    L.rb_lookup.argtypes = [p, p, i32, i64, p, p, p]
    L.rb_owner_pool.argtypes = [p, p, C.POINTER(i64)]
    L.rb_point_cells.argtypes = [C.POINTER(Grid), p, i32, i64, p, p, p, p]
    L.rb_approx_cells.argtypes = [p, C.POINTER(i64), p, p, p, p, p]
    L.rb_approx_partial.argtypes = [p, C.POINTER(i64), p, p, p, p]
    L.rb_exact_pip.argtypes = [C.POINTER(Polygons), p, p, p, i64, p, p]
    L.rb_exact_distance.argtypes = [C.POINTER(Polygons), p, p, p, i64, p, p]
    L.rb_instrument.argtypes = [i32, C.POINTER(i64), C.POINTER(i64), C.POINTER(d)]
    L.rb_approx_set_hot.argtypes = [p, p, i32, p]
    L.rb_lps_build.argtypes = [C.POINTER(Grid), p, i32, i64, p, i32, p, C.POINTER(p), C.POINTER(i64)]
    L.rb_lps_info.argtypes = [p, C.POINTER(i64), C.POINTER(p), C.POINTER(p), C.POINTER(p), C.POINTER(i32)]
    L.rb_lps_free.argtypes = [p]
    L.rb_lps_free.restype = None
    L.rb_rs_build.argtypes = [p, i32, i32, p, C.POINTER(p)]
    L.rb_rs_info.argtypes = [p, C.POINTER(i64), C.POINTER(p), C.POINTER(p), C.POINTER(p), C.POINTER(i32),
                             C.POINTER(i32)]
    L.rb_rs_free.argtypes = [p]
    L.rb_rs_free.restype = None
    L.rb_bounds_lookup.argtypes = [p, p, p, p, i64, p, p, p]
    L.rb_validate_full.argtypes = [p, C.POINTER(Polygons), p, p, p, i32, d, d, d, p, i32, i64, d, p,
                                   C.POINTER(d), p]
    L.rb_lps_from_arrays.argtypes = [C.POINTER(Grid), i64, p, p, p, i32, p, C.POINTER(p)]
    L.rb_rs_from_arrays.argtypes = [p, i32, i32, i64, p, p, p, p, C.POINTER(p)]
    L.rb_join_pointindex.argtypes = [p, p, i64, p, p, p, p, i32, i32, p, p, p]
    cd = C.POINTER(CanvasDesc)
    L.rb_canvas_clear.argtypes = [cd, p]
    L.rb_canvas_render_points.argtypes = [p, cd, p]
    L.rb_canvas_render_cells.argtypes = [i64, p, p, p, i32, i32, i32, cd, p]
    L.rb_canvas_blend.argtypes = [cd, cd, i32, cd, p]
    L.rb_canvas_mask.argtypes = [cd, i32, i64, cd, cd, p]
    L.rb_canvas_affine.argtypes = [cd, i64, i64, i32, i32, cd, p]
    L.rb_canvas_reduce.argtypes = [cd, p, p, p]
    for name in EXPORTS:
        getattr(L, name)  # AttributeError if an export is missing
    _lib = L
    return L


def check(status: int, what: str = "", index: int | None = None) -> None:
    if status == RB_OK:
        return
    msg = (load().rb_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    cls = _STATUS.get(status)
    if cls is E.DomainError:
        raise E.DomainError(text, index)
    if cls is not None:
        raise cls(text)
    raise RuntimeError(f"rasterbound_b200 CUDA failure ({status}): {text}")


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise E.ConfigError("rasterbound_b200 requires a CUDA device (sm_100a); none is visible")
    return torch


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def instrument(op: int):
    """op 1: reset + time the point-pass kernel; 2: reset, no timing; 0: read
    -> (launches, timed_launches, timed_ms)."""
    a, b, c = C.c_int64(), C.c_int64(), C.c_double()
    check(load().rb_instrument(op, C.byref(a), C.byref(b), C.byref(c)), "rb_instrument")
    return int(a.value), int(b.value), float(c.value)
