"""Seeded synthetic workloads standing in for the paper's NYC data
(BASELINE.json configs; the taxi points and census/neighbourhood polygons are
not available here -- DESIGN.md "Workloads").

  C1  1M uniform f64 points in the unit square, 100 tiling polygons from a
      jittered 10x10 grid (corner jitter +-0.3 cell, 4-16 vertices per edge,
      +-0.02 perpendicular noise), eps = 1e-3, uniform raster, COUNT.
  C2  100M f64 points over 40 km x 40 km from 50 isotropic Gaussians
      (sigma U[200, 3000] m, Dirichlet(1) weights) + 10% uniform background,
      fare f32 ~ lognormal(2.5, 0.6); 260 jittered-Voronoi tiling polygons
      with 100-500 vertices; eps = 4.9 m; uniform raster; COUNT + SUM(fare).
  C3  C2 inputs x eps in {50, 10, 4.9, 1, 0.5} x {uniform, hierarchical}.
  C4  1B f32 offset points, same mixture over 100 km x 100 km, 40,000
      jittered-Voronoi polygons with 10-30 vertices, eps = 1 m,
      hierarchical raster, COUNT + SUM(fare).
  C5  C4 per rank (seed + rank), 1/2/4/8 GPUs.

Unspecified choices (recorded in DESIGN.md): Gaussian centres uniform over
the extent; sigma uniform; seeds = 0 (+ rank); GridConfig by the SPEC ingest
rule (data MBR + 1% padding).
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from .geometry import Polygon, RegionRecord
from .grid import GridConfig, eps_grid, ingest_grid


# ------------------------------------------------------------- validation
def _segments_intersect_any(poly: np.ndarray) -> bool:
    """True if a simple-polygon violation exists (non-adjacent edges touch)."""
    n = len(poly)
    a = poly
    b = np.roll(poly, -1, axis=0)
    i, j = np.triu_indices(n, k=2)
    keep = ~((i == 0) & (j == n - 1))
    i, j = i[keep], j[keep]
    if len(i) == 0:
        return False
    p1, p2, q1, q2 = a[i], b[i], a[j], b[j]

    def orient(p, q, r):
        return np.sign((q[:, 0] - p[:, 0]) * (r[:, 1] - p[:, 1]) - (q[:, 1] - p[:, 1]) * (r[:, 0] - p[:, 0]))

    o1, o2, o3, o4 = orient(p1, p2, q1), orient(p1, p2, q2), orient(q1, q2, p1), orient(q1, q2, p2)
    proper = (o1 * o2 < 0) & (o3 * o4 < 0)
    if proper.any():
        return True
    # touching / collinear overlaps
    def on_seg(p, q, r, o):
        return (o == 0) & (np.minimum(p[:, 0], q[:, 0]) <= r[:, 0]) & (r[:, 0] <= np.maximum(p[:, 0], q[:, 0])) & \
            (np.minimum(p[:, 1], q[:, 1]) <= r[:, 1]) & (r[:, 1] <= np.maximum(p[:, 1], q[:, 1]))
    touch = on_seg(p1, p2, q1, o1) | on_seg(p1, p2, q2, o2) | on_seg(q1, q2, p1, o3) | on_seg(q1, q2, p2, o4)
    return bool(touch.any())


def is_simple(poly: np.ndarray) -> bool:
    return not _segments_intersect_any(np.asarray(poly, np.float64))


# ------------------------------------------------------------- chains
class _Chains:
    """Shared, subdivided + noised edge chains, generated once per undirected
    edge and reused (reversed) by the neighbouring polygon, so tilings have
    no gaps or overlaps."""

    def __init__(self, rng: np.random.Generator, nsub, noise, on_boundary):
        self.rng = rng
        self.nsub = nsub  # callable(a, b) -> number of intermediate vertices
        self.noise = noise  # callable(a, b) -> max perpendicular offset
        self.on_boundary = on_boundary  # callable(a, b) -> bool (no perpendicular noise)
        self.cache: dict = {}
        self.calm: set = set()

    def chain(self, ka, kb, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        """Intermediate vertices from a to b (exclusive of both)."""
        key = (ka, kb) if ka < kb else (kb, ka)
        if key not in self.cache:
            p, q = (a, b) if ka < kb else (b, a)
            m = int(self.nsub(p, q))
            t = (np.arange(1, m + 1) / (m + 1))[:, None]
            pts = p[None, :] + t * (q - p)[None, :]
            if m and key not in self.calm and not self.on_boundary(p, q):
                d = q - p
                nrm = np.array([-d[1], d[0]]) / (np.hypot(d[0], d[1]) + 1e-300)
                amp = self.noise(p, q)
                off = self.rng.uniform(-amp, amp, size=m) * np.sin(np.pi * t[:, 0])
                pts = pts + off[:, None] * nrm[None, :]
            self.cache[key] = pts
        pts = self.cache[key]
        return pts if ka < kb else pts[::-1]

    def reset(self, key):
        self.calm.add(key)
        self.cache.pop(key, None)


def _assemble(corner_ids, corners, chains: _Chains) -> np.ndarray:
    out = []
    n = len(corner_ids)
    for k in range(n):
        ka, kb = corner_ids[k], corner_ids[(k + 1) % n]
        out.append(corners[ka][None, :])
        out.append(chains.chain(ka, kb, corners[ka], corners[kb]))
    return np.concatenate(out, axis=0)


def _build_tiling(cells, corners, chains: _Chains, max_iter: int = 8):
    """cells: list of corner-id cycles.  Returns vertex arrays, calming the
    noise of every edge of a non-simple polygon until all are simple."""
    for _ in range(max_iter):
        polys = [_assemble(c, corners, chains) for c in cells]
        bad = [k for k, p in enumerate(polys) if not is_simple(p)]
        if not bad:
            return polys
        for k in bad:
            c = cells[k]
            for i in range(len(c)):
                a, b = c[i], c[(i + 1) % len(c)]
                chains.reset((a, b) if a < b else (b, a))
    raise RuntimeError("could not generate simple polygons")


# ------------------------------------------------------------- C1 tiling
def grid_tiling(seed: int = 0, n: int = 10, jitter: float = 0.3, sub=(4, 16), noise: float = 0.02,
                extent: float = 1.0) -> list:
    """C1: n x n jittered grid tiling of [0, extent]^2."""
    rng = np.random.default_rng(seed)
    h = extent / n
    corners = {}
    for j in range(n + 1):
        for i in range(n + 1):
            x, y = i * h, j * h
            dx, dy = rng.uniform(-jitter * h, jitter * h, size=2)
            if 0 < i < n:
                x += dx
            if 0 < j < n:
                y += dy
            # boundary vertices move only along their side; corners fixed
            corners[j * (n + 1) + i] = np.array([x, y])

    def on_boundary(p, q):
        return (p[0] == q[0] and p[0] in (0.0, extent)) or (p[1] == q[1] and p[1] in (0.0, extent))

    chains = _Chains(rng, lambda p, q: rng.integers(sub[0], sub[1] + 1) - 2, lambda p, q: noise, on_boundary)
    cells = []
    for j in range(n):
        for i in range(n):
            c00 = j * (n + 1) + i
            cells.append([c00, c00 + 1, c00 + n + 2, c00 + n + 1])  # CCW
    polys = _build_tiling(cells, corners, chains)
    return [RegionRecord(k, Polygon(p)) for k, p in enumerate(polys)]


# ------------------------------------------------------------- Voronoi
def voronoi_tiling(n_polys: int, width: float, seed: int = 0, verts=(100, 500), noise_frac: float = 0.04,
                   jitter: float = 0.4) -> list:
    """Jittered-Voronoi tiling of [0, width]^2 clipped by seed mirroring;
    shared ridges are subdivided once so the tiling stays watertight."""
    from scipy.spatial import Voronoi

    rng = np.random.default_rng(seed)
    nx = int(round(math.sqrt(n_polys)))
    while n_polys % nx:
        nx -= 1
    ny = n_polys // nx
    gx, gy = width / nx, width / ny
    ii, jj = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    sx = (ii.ravel() + 0.5 + rng.uniform(-jitter, jitter, n_polys)) * gx
    sy = (jj.ravel() + 0.5 + rng.uniform(-jitter, jitter, n_polys)) * gy
    seeds = np.stack([sx, sy], axis=1)
    mirrored = [seeds, seeds * [-1, 1], seeds * [1, -1], np.stack([2 * width - sx, sy], 1),
                np.stack([sx, 2 * width - sy], 1)]
    vor = Voronoi(np.concatenate(mirrored, axis=0))
    V = vor.vertices.copy()
    tol = 1e-7 * width
    V[np.abs(V[:, 0]) < tol, 0] = 0.0
    V[np.abs(V[:, 1]) < tol, 1] = 0.0
    V[np.abs(V[:, 0] - width) < tol, 0] = width
    V[np.abs(V[:, 1] - width) < tol, 1] = width
    corners = {k: V[k] for k in range(len(V))}
    cells = []
    for k in range(n_polys):
        reg = vor.regions[vor.point_region[k]]
        if -1 in reg or not reg:
            raise RuntimeError("unbounded Voronoi cell inside the mirrored domain")
        pts = V[reg]
        # CCW order
        if np.sum(pts[:, 0] * np.roll(pts[:, 1], -1) - np.roll(pts[:, 0], -1) * pts[:, 1]) < 0:
            reg = reg[::-1]
        cells.append(list(reg))
    mean_edges = np.mean([len(c) for c in cells])
    lo, hi = verts
    # intermediate vertices per ridge so that polygons land in [lo, hi] on average
    per_lo = max(0, int(math.floor((lo - mean_edges) / mean_edges)))
    per_hi = max(per_lo, int(math.ceil((hi - mean_edges) / mean_edges)))

    def on_boundary(p, q):
        return (p[0] == q[0] and p[0] in (0.0, width)) or (p[1] == q[1] and p[1] in (0.0, width))

    chains = _Chains(rng, lambda p, q: rng.integers(per_lo, per_hi + 1),
                     lambda p, q: noise_frac * float(np.hypot(*(q - p))), on_boundary)
    polys = _build_tiling(cells, corners, chains)
    return [RegionRecord(k, Polygon(p)) for k, p in enumerate(polys)]


# ------------------------------------------------------------- points
def uniform_points(n: int, seed: int = 0, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return lo + (hi - lo) * rng.random((n, 2))


@dataclass
class Mixture:
    centres: np.ndarray
    sigmas: np.ndarray
    weights: np.ndarray
    background: float
    width: float


def make_mixture(width: float, seed: int = 0, k: int = 50, sigma=(200.0, 3000.0), background: float = 0.1) -> Mixture:
    rng = np.random.default_rng([seed, 7919])
    return Mixture(rng.uniform(0, width, (k, 2)), rng.uniform(sigma[0], sigma[1], k), rng.dirichlet(np.ones(k)),
                   background, width)


def _mixture_chunk(mx: Mixture, n: int, ss: np.random.SeedSequence, dtype) -> np.ndarray:
    rng = np.random.default_rng(ss)
    out = np.empty((n, 2), np.float64)
    todo = np.arange(n)
    while len(todo):
        m = len(todo)
        bg = rng.random(m) < mx.background
        comp = rng.choice(len(mx.weights), size=m, p=mx.weights)
        pts = mx.centres[comp] + rng.standard_normal((m, 2)) * mx.sigmas[comp][:, None]
        pts[bg] = rng.uniform(0, mx.width, (int(bg.sum()), 2))
        ok = (pts[:, 0] >= 0) & (pts[:, 0] < mx.width) & (pts[:, 1] >= 0) & (pts[:, 1] < mx.width)
        out[todo[ok]] = pts[ok]
        todo = todo[~ok]
    return out.astype(dtype, copy=False)


def mixture_points(n: int, mx: Mixture, seed: int = 0, dtype=np.float64, chunk: int = 1 << 22,
                   threads: int | None = None) -> np.ndarray:
    """Gaussian-mixture points in random order (each point draws its component),
    generated in seeded chunks (deterministic for any thread count)."""
    nch = (n + chunk - 1) // chunk
    seqs = np.random.SeedSequence([seed, 104729]).spawn(max(nch, 1))
    out = np.empty((n, 2), dtype)
    threads = threads or min(32, len(os.sched_getaffinity(0)))

    def work(c):
        a, b = c * chunk, min(n, (c + 1) * chunk)
        out[a:b] = _mixture_chunk(mx, b - a, seqs[c], dtype)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, range(nch)))
    return out


def fares(n: int, seed: int = 0, chunk: int = 1 << 22) -> np.ndarray:
    nch = (n + chunk - 1) // chunk
    seqs = np.random.SeedSequence([seed, 1299709]).spawn(max(nch, 1))
    out = np.empty(n, np.float32)

    def work(c):
        a, b = c * chunk, min(n, (c + 1) * chunk)
        out[a:b] = np.random.default_rng(seqs[c]).lognormal(2.5, 0.6, b - a).astype(np.float32)

    with ThreadPoolExecutor(min(32, len(os.sched_getaffinity(0)))) as ex:
        list(ex.map(work, range(nch)))
    return out


# ------------------------------------------------------------- configs
@dataclass
class Workload:
    name: str
    regions: list
    xy: np.ndarray
    attrs: dict
    grid: GridConfig
    epsilon: float
    layout: str
    agg: str
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.xy.shape[0])


def c1(n: int = 1_000_000, seed: int = 0) -> Workload:
    regions = grid_tiling(seed)
    xy = uniform_points(n, seed)
    return Workload("C1", regions, xy, {}, ingest_grid(0.0, 0.0, 1.0, 1.0), 1e-3, "dense", "COUNT",
                    {"points": n, "polygons": 100, "seed": seed})


def city_regions(seed: int = 0, n_polys: int = 260, width: float = 40_000.0) -> list:
    return voronoi_tiling(n_polys, width, seed, verts=(100, 500))


def c2(n: int = 100_000_000, seed: int = 0, regions: list | None = None, eps: float = 4.9) -> Workload:
    W = 40_000.0
    regions = regions if regions is not None else city_regions(seed)
    mx = make_mixture(W, seed)
    xy = mixture_points(n, mx, seed, np.float64)
    f = fares(n, seed)
    return Workload("C2", regions, xy, {"fare": f}, ingest_grid(0.0, 0.0, W, W), eps, "trie", "SUM:fare",
                    {"points": n, "polygons": len(regions), "seed": seed, "extent_m": W})


def fine_regions(seed: int = 0, n_polys: int = 40_000, width: float = 100_000.0) -> list:
    return voronoi_tiling(n_polys, width, seed, verts=(10, 30))


def c4(n: int = 1_000_000_000, seed: int = 0, regions: list | None = None, rank: int = 0,
       grid: str = "eps") -> Workload:
    """grid="eps": the epsilon-matched GridConfig (leaf side exactly eps/sqrt(2) = 0.707 m, L = 18 over a
    185 km domain holding the padded 100 km data MBR; grid.eps_grid), the north star's "cell side
    eps/sqrt(2)".  grid="ingest": the SPEC ingest rule (102 km domain, L = 18, side 0.389 m)."""
    W = 100_000.0
    eps = 1.0
    regions = regions if regions is not None else fine_regions(seed)
    mx = make_mixture(W, seed)
    xy = mixture_points(n, mx, seed + rank, np.float32)
    f = fares(n, seed + rank)
    if grid not in ("eps", "ingest"):
        raise ValueError("grid must be 'eps' or 'ingest'")
    g = eps_grid(0.0, 0.0, W, W, eps) if grid == "eps" else ingest_grid(0.0, 0.0, W, W)
    return Workload("C4", regions, xy, {"fare": f}, g, eps, "packed", "SUM:fare",
                    {"points": n, "polygons": len(regions), "seed": seed + rank, "extent_m": W, "xy": "f32 offsets",
                     "grid": grid})


__all__ = [
    "grid_tiling", "voronoi_tiling", "uniform_points", "make_mixture", "mixture_points", "fares", "Workload", "c1",
    "c2", "c4", "city_regions", "fine_regions", "is_simple",
]
