"""Oracle properties (CPU): the SPEC's invariants and acceptance criteria
 on the C oracle, plus
equality of the SPEC-literal tier (i) with the C tier (ii) on generic inputs."""
import math

import numpy as np
import pytest

from helpers import random_polygons
from oracle import spec_literal as SL
from paper_2010_12548_b200.geometry import pack_regions


def _approx(O, regions, L, mode=0, extent=1.0, origin=(0.0, 0.0)):
    p = pack_regions(regions)
    return O.Approx((origin[0], origin[1], extent, L), p.vx, p.vy, p.ring_off, p.poly_ring_off, p.poly_region,
                    p.n_regions, mode), p


def _exact_owner_sets(O, packed, xy):
    """Exact PIP (boundary = inside) per region for every point (test helper)."""
    R = packed.n_regions
    inside = np.zeros((len(xy), R), bool)
    for k in range(packed.n_polygons):
        r0, r1 = packed.poly_ring_off[k], packed.poly_ring_off[k + 1]
        v0, v1 = packed.ring_off[r0], packed.ring_off[r1]
        ro = packed.ring_off[r0:r1 + 1] - v0
        inside[:, packed.poly_region[k]] |= O.pip(packed.vx[v0:v1], packed.vy[v0:v1], ro, xy[:, 0], xy[:, 1])
    return inside


def _dist(O, packed, xy, region):
    d = np.full(len(xy), np.inf)
    for k in np.nonzero(packed.poly_region == region)[0]:
        r0, r1 = packed.poly_ring_off[k], packed.poly_ring_off[k + 1]
        v0, v1 = packed.ring_off[r0], packed.ring_off[r1]
        ro = packed.ring_off[r0:r1 + 1] - v0
        d = np.minimum(d, O.distance(packed.vx[v0:v1], packed.vy[v0:v1], ro, xy[:, 0], xy[:, 1]))
    return d


def _approx_owner_sets(A, n, R, xy):
    off, reg, kind = A.lookup(xy)
    got = np.zeros((n, R), bool)
    b = np.zeros((n, R), bool)
    rows = np.repeat(np.arange(n), np.diff(off))
    got[rows, reg] = True
    b[rows[kind == 2], reg[kind == 2]] = True
    return got, b


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
@pytest.mark.parametrize("mode", [0, 1])
def test_literal_tier_equals_c_tier(oracle_lib, seed, mode):
    """Tier (i) top-down classify + radix trie == tier (ii) column walk + spans."""
    regions = random_polygons(100 + seed, k=6, holes=True)
    L = 7
    A, p = _approx(oracle_lib, regions, L, mode)
    side = math.ldexp(1.0, -L)
    for k, r in enumerate(regions):
        rings = [r.geometry.outer.tolist()] + [h.tolist() for h in r.geometry.holes]
        lit = sorted(SL.rasterize_hierarchical(SL.to_grid(rings, (0.0, 0.0), side), L, mode == 1))
        lv, code, kind = A.hier_cells(k)
        got = sorted(zip(lv.tolist(), code.tolist(), ["I" if x == 1 else "B" for x in kind]))
        assert got == lit, f"polygon {k}"
    trie, _ = SL.build([(r.id, [[r.geometry.outer.tolist()] + [h.tolist() for h in r.geometry.holes]])
                        for r in regions], (0.0, 0.0), 1.0, L, mode == 1, radix_width=8)
    xy = np.random.default_rng(seed).random((3000, 2))
    res = SL.join_act(xy.tolist(), trie, (0.0, 0.0), 1.0)
    cnt, _ = A.join(xy)
    for r in range(len(regions)):
        exp = res.get(r, [0, 0, 0.0, 0.0])
        assert [int(cnt[r, 0]), int(cnt[r, 1])] == exp[:2]


def test_trie_radix_widths_agree(oracle_lib):
    regions = random_polygons(7, k=5)
    L = 6
    tries = [SL.build([(r.id, [[r.geometry.outer.tolist()]]) for r in regions], (0.0, 0.0), 1.0, L,
                      radix_width=w)[0] for w in (2, 4, 8)]
    for leaf in range(0, 1 << (2 * L), 7):
        a = tries[0].lookup_code(leaf)
        assert a == tries[1].lookup_code(leaf) == tries[2].lookup_code(leaf)


def test_zorder_interval_exhaustive():
    """Acceptance 7: cell membership <=> code in cell_interval, L <= 5."""
    from paper_2010_12548_b200.grid import CellId, cell_interval, z_decode, z_encode

    for L in range(0, 6):
        n = 1 << L
        for level in range(0, L + 1):
            for code in range(1 << (2 * level)):
                c = CellId(level, code)
                iv = cell_interval(c, L)
                cx, cy = z_decode(c)
                s = 1 << (L - level)
                for ix in range(n):
                    for iy in range(n):
                        leaf = z_encode(ix, iy, L).code
                        inside = cx * s <= ix < (cx + 1) * s and cy * s <= iy < (cy + 1) * s
                        assert (leaf in iv) == inside


def test_uniform_equals_hierarchical_and_disjoint(oracle_lib):
    """hierarchical and uniform coverings denote the same set;
    cells of one covering are pairwise disjoint."""
    regions = random_polygons(21, k=10, holes=True)
    L = 8
    for mode in (0, 1):
        A, _ = _approx(oracle_lib, regions, L, mode)
        for k in range(len(regions)):
            lv, code, kind = A.hier_cells(k)
            sh = (2 * (L - lv)).astype(np.uint64)
            lo, hi = code.astype(np.uint64) << sh, (code.astype(np.uint64) + np.uint64(1)) << sh
            o = np.argsort(lo)
            assert np.all(lo[o][1:] >= hi[o][:-1])  # disjoint
            leaves = np.concatenate([np.arange(a, b, dtype=np.uint64) for a, b in zip(lo, hi)]) if len(lo) else []
            kinds = np.concatenate([np.full(int(b - a), k_) for a, b, k_ in zip(lo, hi, kind)]) if len(lo) else []
            # uniform (leaf-level) classification straight from the leaf rule
            n = 1 << L
            ii, jj = np.meshgrid(np.arange(n, dtype=np.uint32), np.arange(n, dtype=np.uint32), indexing="xy")
            lk = A.leaf_kinds(k, ii.ravel(), jj.ravel())
            z = np.array([SL.z_encode(int(a), int(b)) for a, b in zip(ii.ravel()[lk > 0], jj.ravel()[lk > 0])],
                         dtype=np.uint64)
            assert sorted(z.tolist()) == sorted(np.asarray(leaves, np.uint64).tolist())
            leaf_kind = dict(zip(np.asarray(leaves).tolist(), np.asarray(kinds).tolist()))
            assert all(leaf_kind[int(zz)] == int(kk) for zz, kk in zip(z, lk[lk > 0]))


@pytest.mark.parametrize("mode", [0, 1])
def test_epsilon_soundness_and_completeness(oracle_lib, mode):
    """Acceptance 1-2: >= 100 polygons x >= 1e5 points: every
    point whose approximate owner set differs from the exact one is within eps
    of that region's boundary; CONSERVATIVE has no false negatives."""
    regions = random_polygons(5, k=100, holes=True)
    eps = 0.01
    L = oracle_lib.level_for_bound(1.0, eps)
    A, p = _approx(oracle_lib, regions, L, mode)
    xy = np.random.default_rng(1).random((100_000, 2))
    exact = _exact_owner_sets(oracle_lib, p, xy)
    got, _ = _approx_owner_sets(A, len(xy), p.n_regions, xy)
    diff = exact != got
    for r in np.nonzero(diff.any(axis=0))[0]:
        idx = np.nonzero(diff[:, r])[0]
        assert np.all(_dist(oracle_lib, p, xy[idx], r) <= eps + 1e-12)
    if mode == 0:
        assert not np.any(exact & ~got)


def test_result_range_soundness(oracle_lib):
    """Acceptance 5: exact PIP count in [alpha - beta, alpha]."""
    regions = random_polygons(9, k=60, holes=True)
    L = 8
    A, p = _approx(oracle_lib, regions, L, 0)
    xy = np.random.default_rng(2).random((60_000, 2))
    exact = _exact_owner_sets(oracle_lib, p, xy).sum(axis=0)
    cnt, _ = A.join(xy)
    assert np.all(cnt[:, 0] - cnt[:, 1] <= exact)
    assert np.all(exact <= cnt[:, 0])


def test_precision_monotone_under_eps_halving(oracle_lib):
    """Acceptance 8-9: conservative alpha non-increasing as
    eps halves (grid-aligned refinement) and exact for grid-aligned polygons."""
    regions = random_polygons(13, k=30)
    xy = np.random.default_rng(3).random((200_000, 2))
    prev = None
    errs = []
    p = pack_regions(regions)
    exact = _exact_owner_sets(oracle_lib, p, xy).sum(axis=0)
    for L in range(4, 11):
        A, _ = _approx(oracle_lib, regions, L, 0)
        a = A.join(xy)[0][:, 0]
        if prev is not None:
            assert np.all(a <= prev)
        prev = a
        errs.append(np.median(np.abs(a - exact) / np.maximum(exact, 1)))
    assert errs[-1] <= errs[0]
    from paper_2010_12548_b200.geometry import Polygon, RegionRecord

    sq = [RegionRecord(0, Polygon([(0.25, 0.25), (0.75, 0.25), (0.75, 0.75), (0.25, 0.75)]))]
    A, p2 = _approx(oracle_lib, sq, 6, 0)
    cnt, _ = A.join(xy)
    assert cnt[0, 0] == _exact_owner_sets(oracle_lib, p2, xy).sum() and cnt[0, 1] == 0


def test_sampled_hausdorff_bound(oracle_lib):
    """Acceptance 3: sampled Hausdorff(polygon, covering) <= eps + step*sqrt(2)."""
    from scipy.spatial import cKDTree

    regions = random_polygons(17, k=12)
    eps = 0.02
    L = oracle_lib.level_for_bound(1.0, eps)
    step = eps / 10
    A, p = _approx(oracle_lib, regions, L, 0)
    g = np.arange(step / 2, 1.0, step)
    X, Y = np.meshgrid(g, g)
    S = np.stack([X.ravel(), Y.ravel()], 1)
    exact = _exact_owner_sets(oracle_lib, p, S)
    got, _ = _approx_owner_sets(A, len(S), p.n_regions, S)
    for r in range(p.n_regions):
        a, b = S[exact[:, r]], S[got[:, r]]
        if len(a) == 0 or len(b) == 0:
            continue
        h = max(cKDTree(b).query(a)[0].max(), cKDTree(a).query(b)[0].max())
        assert h <= eps + step * math.sqrt(2) + 1e-12
