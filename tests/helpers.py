"""Shared test helpers: oracle construction from the product's CSR packing,
random polygon generators and adversarial fixtures."""
from __future__ import annotations

import numpy as np

from paper_2010_12548_b200.geometry import Polygon, RegionRecord, pack_regions
from paper_2010_12548_b200.grid import GridConfig


def oracle_approx(O, regions, grid: GridConfig, mode: int = 0):
    p = regions if hasattr(regions, "vx") else pack_regions(regions)
    return O.Approx((grid.origin.x, grid.origin.y, grid.extent, grid.max_level), p.vx, p.vy, p.ring_off,
                    p.poly_ring_off, p.poly_region, p.n_regions, mode), p


def star_polygon(rng, cx, cy, r, n=12, irregular=0.5):
    ang = np.sort(rng.uniform(0, 2 * np.pi, n))
    rad = r * (1 - irregular * rng.random(n))
    return np.stack([cx + rad * np.cos(ang), cy + rad * np.sin(ang)], 1)


def random_polygons(seed: int, k: int = 20, extent: float = 1.0, holes: bool = False):
    """k random star-shaped (simple) polygons inside [0.05, 0.95]*extent, possibly overlapping."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(k):
        r = rng.uniform(0.03, 0.2) * extent
        cx, cy = rng.uniform(0.05 * extent + r, 0.95 * extent - r, 2)
        outer = star_polygon(rng, cx, cy, r, n=int(rng.integers(3, 30)))
        hs = []
        if holes and rng.random() < 0.5:
            hs = [star_polygon(rng, cx, cy, 0.2 * r, n=6, irregular=0.2)[::-1]]
        out.append(RegionRecord(i, Polygon(outer, hs)))
    return out


def adversarial_regions():
    """Degenerate-geometry fixtures on the unit grid used with L=3 (side 1/8)."""
    sq = lambda a, b: [(a, a), (b, a), (b, b), (a, b)]
    return [
        RegionRecord(0, Polygon(sq(0.25, 0.75))),                                  # grid aligned
        RegionRecord(1, Polygon([(0.5, 0.0), (1.0, 0.5), (0.5, 1.0), (0.0, 0.5)])),  # edges through cell corners
        RegionRecord(2, Polygon([(0.0625, 0.0625), (0.9375, 0.0625), (0.5, 0.9375)])),  # vertices at cell centres
        RegionRecord(3, Polygon(sq(0.0, 1.0), [sq(0.375, 0.625)[::-1]])),          # domain-filling with aligned hole
        RegionRecord(4, Polygon([(0.0, 0.0), (0.3, 0.0), (0.0, 0.01)])),          # sliver touching the domain edge
        RegionRecord(5, Polygon([(0.1, 0.5625), (0.9, 0.5625), (0.9, 0.6), (0.1, 0.6)])),  # horizontal edge on centre line
    ]


UNIT = GridConfig((0.0, 0.0), 1.0, 0)
