"""Cache model for C4 cell-index layouts (design aid, CPU only).

For a sample of C4 points and the C4 polygon boundaries, estimate for a
candidate index layout: the fraction of points that reach each index level,
the touched bytes per level, and (Che approximation of an LRU cache of the
given size over the i.i.d. point stream) the DRAM sectors per point.

Mixedness of a level-l cell is approximated by "holds a leaf that an edge
passes through" (edges sampled at side/4), which is what the hierarchical
raster refines.

  python tools/index_model.py [points] [grid: ingest|eps]
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_12548_b200 import workloads as W  # noqa: E402


def boundary_leaves(regions, ox, oy, side, L):
    segs = []
    for r in regions:
        for p in (r.geometry if isinstance(r.geometry, list) else [r.geometry]):
            for ring in p.rings:
                a = ring
                b = np.roll(ring, -1, axis=0)
                segs.append(np.concatenate([a, b], axis=1))
    S = np.concatenate(segs)
    keys = []
    for c in range(0, len(S), 20000):
        s = S[c:c + 20000]
        ln = np.hypot(s[:, 2] - s[:, 0], s[:, 3] - s[:, 1])
        m = np.maximum(2, np.ceil(ln / (side / 4)).astype(np.int64) + 1)
        idx = np.repeat(np.arange(len(s)), m)
        off = np.arange(m.sum()) - np.repeat(np.cumsum(m) - m, m)
        t = off / (m[idx] - 1)
        x = s[idx, 0] + t * (s[idx, 2] - s[idx, 0])
        y = s[idx, 1] + t * (s[idx, 3] - s[idx, 1])
        ix = np.floor((x - ox) / side).astype(np.int64)
        iy = np.floor((y - oy) / side).astype(np.int64)
        keys.append(np.unique((iy << 32) | ix))
    return np.unique(np.concatenate(keys))


def che_miss(counts, n_acc, cache_items):
    """LRU miss ratio (Che): p_i = counts/n_acc; find T with sum(1-exp(-p T)) = C."""
    p = counts / n_acc
    if len(p) <= cache_items:
        return 0.0
    lo, hi = 0.0, 1e18
    for _ in range(200):
        T = math.sqrt(lo * hi) if lo > 0 else hi / 1e6
        occ = np.sum(1 - np.exp(-p * T))
        if occ > cache_items:
            hi = T
        else:
            lo = T
        if hi / max(lo, 1e-30) < 1.0001:
            break
    T = lo
    return float(np.sum(p * np.exp(-p * T)))


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 4_000_000
    gmode = sys.argv[2] if len(sys.argv) > 2 else "eps"
    regions = W.fine_regions(0)
    mx = W.make_mixture(100_000.0, 0)
    xy = W.mixture_points(n, mx, 0, np.float32).astype(np.float64)
    L = 18
    if gmode == "eps":
        side = 1.0 / math.sqrt(2.0)
        ox = oy = -1000.0
    else:
        g = W.ingest_grid(0.0, 0.0, 100_000.0, 100_000.0)
        side = g.extent / 2 ** L
        ox, oy = g.origin.x, g.origin.y
    bl = boundary_leaves(regions, ox, oy, side, L)
    bx = (bl & 0xffffffff)
    by = bl >> 32
    px = np.floor((xy[:, 0] - ox) / side).astype(np.int64)
    py = np.floor((xy[:, 1] - oy) / side).astype(np.int64)
    print(f"grid={gmode} side={side:.4f} boundary leaves={len(bl)/1e6:.1f}M")
    mixed = {}
    for lvl in range(8, L + 1):
        d = L - lvl
        mixed[lvl] = np.unique(((by >> d) << 32) | (bx >> d))
    frac = {}
    for lvl in range(8, L + 1):
        d = L - lvl
        k = ((py >> d) << 32) | (px >> d)
        frac[lvl] = np.isin(k, mixed[lvl])
        print(f"  level {lvl:2d} cell {side * 2**d:8.2f} m  mixed cells {len(mixed[lvl])/1e6:8.3f}M  "
              f"points in mixed {frac[lvl].mean():.4f}")
    # designs: list of (name, [(level, bytes_per_cell_record, sector key fn)])
    cache_mb = float(os.environ.get("CACHE_MB", "90"))
    for T0 in (11, 12, 13):
        for blk in (16, 32):
            # root u32 at T0; then leaf blocks of `blk` bytes covering (blk==16: 4x4, blk==32: 8x8) leaves,
            # dense per mixed root cell
            d = L - T0
            root_key = ((py >> d) << T0) | (px >> d)
            root_sector = root_key // 8
            leaf_side = 4 if blk == 16 else 8
            inb = frac[T0]
            # leaf block key: root cell id * blocks_per_root + block
            bpr = (2 ** d // leaf_side) ** 2
            bxl = (px & (2 ** d - 1)) // leaf_side
            byl = (py & (2 ** d - 1)) // leaf_side
            blk_key = root_key * bpr + byl * (2 ** d // leaf_side) + bxl
            sec_key = (blk_key * blk) // 32
            acc = np.concatenate([root_sector, (1 << 50) + sec_key[inb]])
            u, c = np.unique(acc, return_counts=True)
            miss = che_miss(c, n, cache_mb * 1e6 / 32)
            mem = len(mixed[T0]) * bpr * blk
            print(f"2L T0={T0} blk={blk}: L2 sectors/pt {1 + inb.mean():.3f}  DRAM sectors/pt {miss * len(acc) / n:.3f} "
                  f"({miss * len(acc) / n * 32:.1f} B/pt)  root {4**T0*4/1e6:.0f} MB  leaf mem {mem/1e9:.2f} GB")
    # 3-level: root T0, mid 32 B sectors (8x8 of level T0+3), leaf 32 B sectors (8x8 leaves), compact
    for T0 in (11, 12):
        M = T0 + 3
        d0, d1 = L - T0, L - M
        root_key = ((py >> d0) << T0) | (px >> d0)
        mid_cell = ((py >> d1) << 32) | (px >> d1)
        # mid sector id: rank of the mixed root cell (keyed by root id)
        mid_key = root_key
        leaf_key = mid_cell
        a1 = frac[T0]
        a2 = frac[M] if M <= L else np.zeros(n, bool)
        acc = np.concatenate([root_key // 8, (1 << 50) + mid_key[a1], (2 << 50) + leaf_key[a2]])
        u, c = np.unique(acc, return_counts=True)
        miss = che_miss(c, n, cache_mb * 1e6 / 32)
        mem = len(mixed[T0]) * 32 + len(mixed[M]) * 32
        print(f"3L T0={T0} M={M}: L2 sectors/pt {1 + a1.mean() + a2.mean():.3f}  DRAM sectors/pt "
              f"{miss * len(acc) / n:.3f} ({miss * len(acc) / n * 32:.1f} B/pt)  mid+leaf mem {mem/1e6:.0f} MB")


if __name__ == "__main__":
    main()
