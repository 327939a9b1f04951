"""Device-resident approximation + cell index (owner of an rb_approx handle).

`ApproxIndex` is what raster / act / query share: it builds the epsilon-
bounded raster approximation of a region set on the GPU (rb_approx_build),
keeps the cell index resident in HBM and runs the point pass
(rb_point_pass), the lookup (rb_lookup) and the host-buffer join
(rb_join_host).  Immutable after construction; point passes on one index may
run concurrently.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import errors as E
from .geometry import DevicePolygons, PackedRegions
from .grid import GridConfig

INT64_MAX = (1 << 63) - 1
LAYOUTS = {"dense": N.LAYOUT_DENSE, "trie": N.LAYOUT_TRIE, "keys": N.LAYOUT_KEYS, "packed": N.LAYOUT_PACKED}


@dataclass
class PassResult:
    """Device tensors of one point pass: cnt [R,2] int64 (alpha, beta), sum [R,2] float64."""
    cnt: object
    sum: object
    first_bad: object

    def check(self):
        b = int(self.first_bad.item())
        if b != INT64_MAX:
            raise E.DomainError(f"point {b} lies outside the grid domain or is NaN (SPEC.md:147)", b)
        return self


class ApproxIndex:
    def __init__(self, packed: PackedRegions, grid: GridConfig, mode: int = N.MODE_CONSERVATIVE,
                 layout: str = "trie", radix_width: int = 8, root_level: int = -1, keep_cells: bool = False,
                 stream=None):
        torch = N.require_cuda()
        if layout not in LAYOUTS:
            raise E.ConfigError(f"unknown layout {layout!r} (dense | trie | keys | packed)")
        self.packed = packed
        self.grid = grid
        self.mode = int(mode)
        self.layout = layout
        self.radix_width = int(radix_width)
        self.n_regions = packed.n_regions
        self._dev = DevicePolygons(packed)
        self._lib = N.load()
        g = grid.native()
        opts = N.BuildOpts(self.mode, LAYOUTS[layout], self.radix_width, int(root_level), 1 if keep_cells else 0)
        h = C.c_void_p()
        N.check(self._lib.rb_approx_build(C.byref(g), C.byref(self._dev.desc), C.byref(opts), N.stream_ptr(stream),
                                          C.byref(h)), "rasterize/act_build")
        self._h = h
        self._torch = torch
        self._hot = None
        self._hot_lock = threading.Lock()

    # regions beyond what one CTA's shared memory holds are accumulated with
    # global atomics; the most frequent owners are privatised ("hot" slots)
    HOT_THRESHOLD = 1024

    def set_hot(self, regions) -> None:
        """rb_approx_set_hot: privatise these (dense) region indices in shared memory."""
        torch = self._torch
        r = torch.as_tensor(np.asarray(regions, dtype=np.int32)).contiguous()
        N.check(self._lib.rb_approx_set_hot(self._h, r.data_ptr() if len(r) else None, int(len(r)),
                                            N.stream_ptr()), "set_hot")
        self._hot = r.numpy().copy()

    # hot slots the deep point pass keeps in shared memory next to its point ring (12 bytes per slot)
    DEFAULT_HOT = 4095  # 8191 fit the shared memory too, but ran slower (C4: 1.79 -> 2.60 ms per 200M points)

    def auto_hot(self, xy, k: int | None = None, sample: int = 1 << 20) -> np.ndarray:
        """Pick the k most frequent single owners of a strided point sample."""
        torch = self._torch
        if k is None:
            k = int(os.environ.get("RB_HOT_K", self.DEFAULT_HOT))  # RB_HOT_K: experiments
        k = min(k, int(self.stats()["max_hot"]))
        t, _ = self._xy(xy)
        n = int(t.shape[0])
        if n == 0:
            self.set_hot([])
            return self._hot
        step = max(1, n // sample)
        v = self.lookup(t[::step]).to(torch.int64) & 0xFFFFFFFF
        single = (v != 0) & ((v & N.VALUE_LIST) == 0)
        reg = (((v[single] & N.CODE_MASK) - 1) >> 1)
        cnt = torch.bincount(reg, minlength=self.n_regions)
        top = torch.argsort(cnt, descending=True)[:k]
        top = top[cnt[top] > 0]
        self.set_hot(top.sort().values.cpu().numpy())
        return self._hot

    @classmethod
    def from_handle(cls, handle: C.c_void_p, grid: GridConfig, n_regions: int, layout: str, radix_width: int):
        self = cls.__new__(cls)
        self.packed = None
        self.grid = grid
        self.mode = -1
        self.layout = layout
        self.radix_width = radix_width
        self.n_regions = n_regions
        self._dev = None
        self._lib = N.load()
        self._h = handle
        self._torch = N.require_cuda()
        self._hot = None
        self._hot_lock = threading.Lock()
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._torch.cuda.synchronize()
            except Exception:
                pass
            self._lib.rb_approx_free(h)
            self._h = None

    @property
    def handle(self) -> int:
        return self._h.value

    def stats(self) -> dict:
        s = N.Stats()
        N.check(self._lib.rb_approx_stats(self._h, C.byref(s)))
        return s.as_dict()

    # ------------------------------------------------------------ points
    def _xy(self, xy):
        torch = self._torch
        t = xy if isinstance(xy, torch.Tensor) else torch.as_tensor(np.asarray(xy))
        if t.dtype not in (torch.float64, torch.float32):
            t = t.to(torch.float64)
        if t.dim() != 2 or t.shape[1] != 2:
            raise E.ShapeError("points must be an (N, 2) array")
        t = t.to("cuda", non_blocking=True).contiguous()
        return t, (N.XY_F64 if t.dtype == torch.float64 else N.XY_F32)

    def _ensure_hot(self, xy) -> None:
        """Large region sets: privatise the most frequent owners once (first pass), under a lock so that
        concurrent first passes do not both rewrite the index."""
        if self._hot is None and self.n_regions > self.HOT_THRESHOLD:
            with self._hot_lock:
                if self._hot is None:
                    self.auto_hot(xy)

    def point_pass(self, xy, attr=None, out: PassResult | None = None, accumulate: bool = False,
                   stream=None) -> PassResult:
        """Stream-ordered alpha/beta COUNT + SUM over device points (no host sync).  A float64
        attribute is summed as its float32 high part plus the float32 residual (two passes)."""
        torch = self._torch
        if accumulate and out is None:
            raise E.ConfigError("accumulate=True adds into existing outputs: pass out=")
        t, dt = self._xy(xy)
        n = int(t.shape[0])
        self._ensure_hot(t)
        a = lo = None
        if attr is not None:
            a = attr if isinstance(attr, torch.Tensor) else torch.as_tensor(np.asarray(attr))
            a = a.to("cuda", non_blocking=True)
            if a.shape[0] != n:
                raise E.ShapeError("attribute length differs from the point count")
            if a.dtype == torch.float64:
                hi = a.to(torch.float32)
                lo = (a - hi.to(torch.float64)).to(torch.float32).contiguous()
                a = hi.contiguous()
            else:
                a = a.to(torch.float32).contiguous()
        if out is None:
            out = PassResult(torch.empty((self.n_regions, 2), dtype=torch.int64, device="cuda"),
                             torch.empty((self.n_regions, 2), dtype=torch.float64, device="cuda"),
                             torch.empty(1, dtype=torch.int64, device="cuda"))
        N.check(self._lib.rb_point_pass(self._h, t.data_ptr(), dt, n, a.data_ptr() if a is not None else None,
                                        out.cnt.data_ptr(), out.sum.data_ptr(), out.first_bad.data_ptr(),
                                        1 if accumulate else 0, N.stream_ptr(stream)), "join")
        if lo is not None:  # the residual part's sums (its counts repeat the first pass)
            part = PassResult(torch.empty_like(out.cnt), torch.empty_like(out.sum), torch.empty_like(out.first_bad))
            N.check(self._lib.rb_point_pass(self._h, t.data_ptr(), dt, n, lo.data_ptr(), part.cnt.data_ptr(),
                                            part.sum.data_ptr(), part.first_bad.data_ptr(), 0, N.stream_ptr(stream)),
                    "join")
            out.sum.add_(part.sum)
        return out

    def join_host(self, xy: np.ndarray, attr: np.ndarray | None = None):
        """rb_join_host: host (ideally pinned) buffers in, host results out."""
        xy = np.ascontiguousarray(xy) if isinstance(xy, np.ndarray) else xy
        if self._hot is None and self.n_regions > self.HOT_THRESHOLD:
            step = max(1, int(xy.shape[0]) // (1 << 20))
            self._ensure_hot(xy[::step])
        if attr is not None:  # float64: float32 high part + float32 residual, two joins
            dt64 = attr.dtype == np.float64 if isinstance(attr, np.ndarray) else attr.dtype == self._torch.float64
            if dt64:
                a64 = np.asarray(attr.numpy() if hasattr(attr, "numpy") else attr, np.float64)
                hi = a64.astype(np.float32)
                lo = (a64 - hi.astype(np.float64)).astype(np.float32)
                cnt, sm = self.join_host(xy, hi)
                _, sm_lo = self.join_host(xy, lo)
                return cnt, sm + sm_lo
        if isinstance(xy, np.ndarray):
            dt = N.XY_F64 if xy.dtype == np.float64 else N.XY_F32
            if xy.dtype not in (np.float64, np.float32):
                raise E.ConfigError("xy must be float64 or float32")
            ptr, n = xy.ctypes.data, xy.shape[0]
        else:  # torch CPU (possibly pinned) tensor
            dt = N.XY_F64 if xy.dtype == self._torch.float64 else N.XY_F32
            ptr, n = xy.data_ptr(), int(xy.shape[0])
        aptr = None
        if attr is not None:
            if isinstance(attr, np.ndarray):
                attr = np.ascontiguousarray(attr, np.float32)
                aptr = attr.ctypes.data
            else:
                aptr = attr.data_ptr()
        cnt = np.zeros((self.n_regions, 2), np.int64)
        sm = np.zeros((self.n_regions, 2), np.float64)
        bad = np.zeros(1, np.int64)
        N.check(self._lib.rb_join_host(self._h, ptr, dt, n, aptr, cnt.ctypes.data, sm.ctypes.data, bad.ctypes.data),
                "join")
        if int(bad[0]) != INT64_MAX:
            raise E.DomainError(f"point {int(bad[0])} lies outside the grid domain or is NaN (SPEC.md:147)", int(bad[0]))
        return cnt, sm

    def lookup(self, xy, stream=None):
        """Owner value per point (uint32 encoding of include/rasterbound_b200.h)."""
        torch = self._torch
        t, dt = self._xy(xy)
        n = int(t.shape[0])
        out = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        bad = torch.empty(1, dtype=torch.int64, device="cuda")
        N.check(self._lib.rb_lookup(self._h, t.data_ptr(), dt, n, out.data_ptr(), bad.data_ptr(), N.stream_ptr(stream)),
                "act_lookup")
        b = int(bad.item())
        if b != INT64_MAX:
            raise E.DomainError(f"point {b} lies outside the grid domain or is NaN (SPEC.md:147)", b)
        return out[:n]

    def owner_pool(self) -> np.ndarray:
        n = C.c_int64()
        N.check(self._lib.rb_owner_pool(self._h, None, C.byref(n)))
        out = np.zeros(max(n.value, 1), np.uint32)
        if n.value:
            N.check(self._lib.rb_owner_pool(self._h, out.ctypes.data, C.byref(n)))
        return out[: n.value]

    def decode(self, values) -> list[list[tuple[int, int]]]:
        """Owner values -> per point list of (dense region index, boundary flag)."""
        vals = np.asarray(values.cpu().numpy() if hasattr(values, "cpu") else values).view(np.uint32)
        pool = self.owner_pool()
        out = []
        for v in vals.tolist():
            if v == 0:
                out.append([])
            elif not (v & N.VALUE_LIST):
                s = v - 1
                out.append([(s >> 1, s & 1)])
            else:
                off = v & N.VALUE_PAYLOAD
                k = int(pool[off])
                out.append([(int(e) >> 1, int(e) & 1) for e in pool[off + 1: off + 1 + k]])
        return out

    # ------------------------------------------------------------ exports
    def cells(self):
        """Per-polygon covering cells: (poly, level, code, kind) numpy arrays."""
        torch = self._torch
        n = C.c_int64()
        N.check(self._lib.rb_approx_cells(self._h, C.byref(n), None, None, None, None, None))
        m = n.value
        poly = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
        level = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
        code = torch.empty(max(m, 1), dtype=torch.int64, device="cuda")
        kind = torch.empty(max(m, 1), dtype=torch.uint8, device="cuda")
        N.check(self._lib.rb_approx_cells(self._h, C.byref(n), poly.data_ptr(), level.data_ptr(), code.data_ptr(),
                                          kind.data_ptr(), N.stream_ptr()))
        torch.cuda.synchronize()
        return (poly[:m].cpu().numpy(), level[:m].cpu().numpy(), code[:m].cpu().numpy().view(np.uint64),
                kind[:m].cpu().numpy())

    def partial(self):
        """PARTIAL leaves: (poly, code, kept) numpy arrays sorted by (poly, code)."""
        torch = self._torch
        n = C.c_int64()
        N.check(self._lib.rb_approx_partial(self._h, C.byref(n), None, None, None, None))
        m = n.value
        poly = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
        code = torch.empty(max(m, 1), dtype=torch.int64, device="cuda")
        kept = torch.empty(max(m, 1), dtype=torch.uint8, device="cuda")
        N.check(self._lib.rb_approx_partial(self._h, C.byref(n), poly.data_ptr(), code.data_ptr(), kept.data_ptr(),
                                            N.stream_ptr()))
        torch.cuda.synchronize()
        return poly[:m].cpu().numpy(), code[:m].cpu().numpy().view(np.uint64), kept[:m].cpu().numpy().astype(bool)


__all__ = ["ApproxIndex", "PassResult", "INT64_MAX", "LAYOUTS"]
