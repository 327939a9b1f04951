"""ORACLE -- test infrastructure only.

CPU restatement of the reference's point-side access path, rasterbound.pointindex
(SPEC.md:313-382), and join_pointindex, following the spec
line by line in numpy:

  lps_build        SPEC.md:328-336  leaf codes = z_encode(floor((p - origin) / side))
                                    (float64 numpy division, same as the
                                    C oracle's point_cells), stable sort -> perm,
                                    prefix[0] = 0, prefix[i] = sum of the first i
                                    sorted values (sequential float64 cumsum)
  rs_build         SPEC.md:337-345  greedy spline corridor over the distinct-key CDF
                                    (key, first position), error <= tau at every key,
                                    radix table over the top radix_bits of the 2L-bit
                                    code space
  bounds_lookup    SPEC.md:346-354  first position with code >= lo / >= hi (binary search)
  range_aggregate  SPEC.md:355-363  sum over cells of prefix[hi] - prefix[lo]

Used only by tests/ (parity checker); the product never imports it.
"""
from __future__ import annotations

import math

import numpy as np


def _spread(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64) & np.uint64(0xFFFFFFFF)
    for s, m in ((16, 0x0000FFFF0000FFFF), (8, 0x00FF00FF00FF00FF), (4, 0x0F0F0F0F0F0F0F0F),
                 (2, 0x3333333333333333), (1, 0x5555555555555555)):
        v = (v | (v << np.uint64(s))) & np.uint64(m)
    return v


def leaf_codes(xy: np.ndarray, origin, extent: float, L: int) -> np.ndarray:
    """SPEC.md:143-151 point_to_cell + SPEC.md:134-142 z_encode (x in the even bits)."""
    xy = np.asarray(xy, np.float64).reshape(-1, 2)
    side = math.ldexp(extent, -L)
    fx = np.floor((xy[:, 0] - origin[0]) / side)
    fy = np.floor((xy[:, 1] - origin[1]) / side)
    lim = float(1 << L)
    bad = ~((fx >= 0) & (fx < lim) & (fy >= 0) & (fy < lim))
    if bad.any():
        raise ValueError(f"point {int(np.nonzero(bad)[0][0])} outside the domain")
    return _spread(fx.astype(np.uint64)) | (_spread(fy.astype(np.uint64)) << np.uint64(1))


def lps_build(xy, origin, extent: float, L: int, attrs: dict | None = None):
    """-> (codes sorted, perm, {name: prefix (n+1)})"""
    codes = leaf_codes(xy, origin, extent, L)
    perm = np.argsort(codes, kind="stable")
    prefix = {}
    for k, v in (attrs or {}).items():
        p = np.zeros(len(codes) + 1, np.float64)
        p[1:] = np.cumsum(np.asarray(v, np.float64)[perm])
        prefix[k] = p
    return codes[perm], perm.astype(np.int64), prefix


def cdf_points(codes: np.ndarray, width: int):
    """Lower-bound CDF F(q) = #{codes < q} sampled at every distinct key k and,
    when the next distinct key (or 2^width) lies beyond k + 1, at k + 1: a spline
    within tau of these points is within tau of F at every integer query."""
    first = np.ones(len(codes), bool)
    first[1:] = codes[1:] != codes[:-1]
    dk = codes[first].astype(np.uint64)
    dp = np.nonzero(first)[0].astype(np.int64)
    nxt = np.append(dk[1:], np.uint64(min(1 << width, (1 << 64) - 1)))
    nxtp = np.append(dp[1:], len(codes)).astype(np.int64)
    gap = nxt > dk + np.uint64(1)
    k = np.empty(len(dk) + int(gap.sum()), np.uint64)
    p = np.empty(len(k), np.int64)
    o = np.arange(len(dk)) + np.concatenate([[0], np.cumsum(gap)[:-1]]).astype(np.int64)
    k[o], p[o] = dk, dp
    k[o[gap] + 1], p[o[gap] + 1] = dk[gap] + np.uint64(1), nxtp[gap]
    return k, p


def spline_fit(codes: np.ndarray, tau: float, chunk: int = 4096, width: int = 62):
    """Greedy spline corridor over the lower-bound CDF points, restarted every
    `chunk` points (the GPU fits chunks in parallel; same knots)."""
    codes = np.asarray(codes, np.uint64)
    if len(codes) == 0:
        return np.zeros(0, np.uint64), np.zeros(0, np.int64)
    dk, dp = cdf_points(codes, width)
    kk, kp = [], []
    for b in range(0, len(dk), chunk):
        e = min(len(dk), b + chunk)
        kk.append(dk[b]); kp.append(dp[b])
        if e - b > 1:
            base, prev = b, b
            lo_s, hi_s = -1e300, 1e300
            for i in range(b + 1, e):
                dx = float(int(dk[i]) - int(dk[base]))
                y = float(int(dp[i]) - int(dp[base]))
                s = y / dx
                if s < lo_s or s > hi_s:
                    kk.append(dk[prev]); kp.append(dp[prev])
                    base = prev
                    dx2 = float(int(dk[i]) - int(dk[base]))
                    y2 = float(int(dp[i]) - int(dp[base]))
                    lo_s, hi_s = (y2 - tau) / dx2, (y2 + tau) / dx2
                else:
                    lo_s = max(lo_s, (y - tau) / dx)
                    hi_s = min(hi_s, (y + tau) / dx)
                prev = i
            kk.append(dk[e - 1]); kp.append(dp[e - 1])
    return np.asarray(kk, np.uint64), np.asarray(kp, np.int64)


def spline_errors(codes: np.ndarray, keys: np.ndarray, pos: np.ndarray) -> np.ndarray:
    """|interpolated position - true first position| for every distinct key."""
    codes = np.asarray(codes, np.uint64)
    first = np.ones(len(codes), bool)
    first[1:] = codes[1:] != codes[:-1]
    dk = codes[first].astype(np.float64)
    dp = np.nonzero(first)[0].astype(np.float64)
    k = keys.astype(np.float64)
    est = np.interp(dk, k, pos.astype(np.float64))
    return np.abs(est - dp)


def radix_table(keys: np.ndarray, radix_bits: int, width: int) -> np.ndarray:
    shift = width - radix_bits
    pref = (keys >> np.uint64(shift)).astype(np.int64) if len(keys) else np.zeros(0, np.int64)
    return np.searchsorted(pref, np.arange((1 << radix_bits) + 1), side="left").astype(np.int64)


def bounds_lookup(codes: np.ndarray, lo, hi):
    codes = np.asarray(codes, np.uint64)
    return (np.searchsorted(codes, np.asarray(lo, np.uint64), side="left"),
            np.searchsorted(codes, np.asarray(hi, np.uint64), side="left"))


def range_aggregate(codes: np.ndarray, prefix: np.ndarray | None, cells):
    """cells: list of (lo, hi); prefix None = COUNT."""
    if not cells:
        return 0.0
    lo, hi = bounds_lookup(codes, [c[0] for c in cells], [c[1] for c in cells])
    if prefix is None:
        return float((hi - lo).sum())
    return float((prefix[hi] - prefix[lo]).sum())
