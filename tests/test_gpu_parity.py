"""GPU parity against the oracle (through the C-ABI): COUNT and beta bit-exact,
SUM within rel 1e-6 (BASELINE north star), covering cells and PARTIAL leaves
identical, act_lookup identical."""
import math

import numpy as np
import pytest

from helpers import UNIT, adversarial_regions, oracle_approx, random_polygons

pytestmark = pytest.mark.gpu

SUM_RTOL = 1e-6


def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _prepared(regions, grid, mode=0, layout="trie", keep=False, radix_width=8, root_level=-1):
    from paper_2010_12548_b200.engine import ApproxIndex
    from paper_2010_12548_b200.geometry import pack_regions

    return ApproxIndex(pack_regions(regions), grid, mode, layout=layout, keep_cells=keep, radix_width=radix_width,
                       root_level=root_level)


def _assert_join(idx, A, xy, attr=None, nthreads=8):
    cnt_o, sum_o = A.join(xy, attr, nthreads=nthreads)
    r = idx.point_pass(xy, attr).check()
    cnt = r.cnt.cpu().numpy()
    np.testing.assert_array_equal(cnt, cnt_o)
    if attr is not None:
        s = r.sum.cpu().numpy()
        np.testing.assert_allclose(s, sum_o, rtol=SUM_RTOL, atol=1e-9)
    return cnt


@pytest.mark.parametrize("layout", ["dense", "trie"])
@pytest.mark.parametrize("mode", [0, 1])
def test_c1_full_count_parity(oracle_lib, layout, mode):
    """Config C1 at full size: 1M points, 100 tiling polygons, eps=1e-3."""
    _gpu()
    from paper_2010_12548_b200 import workloads as W
    from paper_2010_12548_b200.grid import level_for_bound

    w = W.c1()
    grid = w.grid.with_level(level_for_bound(w.grid, w.epsilon))
    A, _ = oracle_approx(oracle_lib, w.regions, grid, mode)
    idx = _prepared(w.regions, grid, mode, layout)
    cnt = _assert_join(idx, A, w.xy)
    assert cnt[:, 0].sum() >= w.n if mode == 0 else True


def test_city_downsized_count_sum(oracle_lib):
    """C2 generator (260 Voronoi polygons, eps 4.9 m) at 4M points: COUNT exact, SUM rel 1e-6."""
    _gpu()
    from paper_2010_12548_b200 import workloads as W
    from paper_2010_12548_b200.grid import level_for_bound

    w = W.c2(n=4_000_000)
    grid = w.grid.with_level(level_for_bound(w.grid, w.epsilon))
    A, _ = oracle_approx(oracle_lib, w.regions, grid, 0)
    for layout in ("trie", "dense"):
        idx = _prepared(w.regions, grid, 0, layout)
        _assert_join(idx, A, w.xy, w.attrs["fare"])


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_overlapping_polygons_with_holes(oracle_lib, seed):
    """Overlapping regions exercise the overlay (all-owners rule)."""
    _gpu()
    regions = random_polygons(seed, k=25, holes=True)
    rng = np.random.default_rng(seed)
    xy = rng.random((200_000, 2))
    attr = rng.lognormal(2.5, 0.6, 200_000).astype(np.float32)
    for L in (6, 9, 12):
        grid = UNIT.with_level(L)
        for mode in (0, 1):
            A, _ = oracle_approx(oracle_lib, regions, grid, mode)
            for layout, rw in (("trie", 8), ("trie", 2), ("dense", 8)):
                idx = _prepared(regions, grid, mode, layout, radix_width=rw)
                _assert_join(idx, A, xy, attr)


def test_lookup_parity(oracle_lib):
    _gpu()
    from paper_2010_12548_b200.act import AdaptiveCellTrie

    regions = random_polygons(7, k=30)
    grid = UNIT.with_level(10)
    rng = np.random.default_rng(0)
    xy = rng.random((20_000, 2))
    A, packed = oracle_approx(oracle_lib, regions, grid, 0)
    off, reg, kind = A.lookup(xy)
    idx = _prepared(regions, grid, 0, "trie")
    got = idx.decode(idx.lookup(xy))
    for k in range(len(xy)):
        exp = sorted((int(r), 1 if kd == 2 else 0) for r, kd in zip(reg[off[k]:off[k + 1]], kind[off[k]:off[k + 1]]))
        assert sorted(got[k]) == exp, k


@pytest.mark.parametrize("mode", [0, 1])
def test_partial_leaves_and_cells_parity(oracle_lib, mode):
    _gpu()
    regions = random_polygons(11, k=12, holes=True) + adversarial_regions()
    regions = [type(r)(k, r.geometry) for k, r in enumerate(regions)]
    for L in (3, 7, 11):
        grid = UNIT.with_level(L)
        A, packed = oracle_approx(oracle_lib, regions, grid, mode)
        idx = _prepared(regions, grid, mode, "trie", keep=True)
        poly, code, kept = idx.partial()
        cp, cl, cc, ck = idx.cells()
        for p in range(packed.n_polygons):
            oc, ok = A.partial_leaves(p)
            m = poly == p
            np.testing.assert_array_equal(code[m], oc)
            np.testing.assert_array_equal(kept[m], ok)
            lv, hc, hk = A.hier_cells(p)
            o = np.lexsort((lv, hc.astype(np.uint64) << (2 * (L - lv)).astype(np.uint64)))
            m = cp == p
            np.testing.assert_array_equal(cl[m], lv[o])
            np.testing.assert_array_equal(cc[m], hc[o])
            np.testing.assert_array_equal(ck[m], hk[o])


def test_adversarial_join_parity(oracle_lib):
    _gpu()
    regions = adversarial_regions()
    grid = UNIT.with_level(3)
    # points on cell lines, corners, centres, vertices, plus random
    g = np.arange(0, 8 * 8 + 1) / 64.0
    gx, gy = np.meshgrid(g[:-1], g[:-1])
    xy = np.concatenate([np.stack([gx.ravel(), gy.ravel()], 1), np.random.default_rng(0).random((50_000, 2))])
    for mode in (0, 1):
        A, _ = oracle_approx(oracle_lib, regions, grid, mode)
        for layout in ("trie", "dense"):
            _assert_join(_prepared(regions, grid, mode, layout), A, xy)


def test_domain_error_reports_first_offender():
    _gpu()
    from paper_2010_12548_b200 import errors as E

    idx = _prepared(adversarial_regions(), UNIT.with_level(5))
    xy = np.random.default_rng(0).random((1000, 2))
    xy[700] = (1.5, 0.2)
    xy[300] = (np.nan, 0.5)
    with pytest.raises(E.DomainError) as ei:
        idx.point_pass(xy).check()
    assert ei.value.index == 300


def test_f32_points_match_promoted_f64(oracle_lib):
    _gpu()
    regions = random_polygons(5, k=20)
    grid = UNIT.with_level(12)
    rng = np.random.default_rng(1)
    xy32 = rng.random((300_001, 2)).astype(np.float32)
    attr = rng.random(300_001).astype(np.float32)
    A, _ = oracle_approx(oracle_lib, regions, grid, 0)
    idx = _prepared(regions, grid, 0, "trie")
    _assert_join(idx, A, xy32, attr)
    r64 = idx.point_pass(xy32.astype(np.float64), attr).check()
    r32 = idx.point_pass(xy32, attr).check()
    np.testing.assert_array_equal(r64.cnt.cpu().numpy(), r32.cnt.cpu().numpy())


def test_uniform_equals_hierarchical_and_shards_sum(oracle_lib):
    _gpu()
    from paper_2010_12548_b200 import workloads as W
    from paper_2010_12548_b200.grid import level_for_bound

    w = W.c2(n=1_000_000, eps=10.0)
    grid = w.grid.with_level(level_for_bound(w.grid, w.epsilon))
    dense = _prepared(w.regions, grid, 0, "dense")
    trie = _prepared(w.regions, grid, 0, "trie")
    a = dense.point_pass(w.xy, w.attrs["fare"]).check().cnt.cpu().numpy()
    b = trie.point_pass(w.xy, w.attrs["fare"]).check().cnt.cpu().numpy()
    np.testing.assert_array_equal(a, b)
    tot = np.zeros_like(b)
    for k in range(4):
        s = slice(k * len(w.xy) // 4, (k + 1) * len(w.xy) // 4)
        tot += trie.point_pass(w.xy[s], w.attrs["fare"][s]).check().cnt.cpu().numpy()
    np.testing.assert_array_equal(tot, b)


def test_join_host_matches_device(oracle_lib):
    _gpu()
    from paper_2010_12548_b200 import workloads as W
    from paper_2010_12548_b200.grid import level_for_bound

    w = W.c2(n=3_000_001)
    grid = w.grid.with_level(level_for_bound(w.grid, w.epsilon))
    idx = _prepared(w.regions, grid, 0, "trie")
    r = idx.point_pass(w.xy, w.attrs["fare"]).check()
    cnt, sm = idx.join_host(w.xy, w.attrs["fare"])
    np.testing.assert_array_equal(cnt, r.cnt.cpu().numpy())
    np.testing.assert_allclose(sm, r.sum.cpu().numpy(), rtol=1e-12)


def test_large_region_set_global_histogram(oracle_lib):
    """3000 regions: the histogram no longer fits shared memory and the point
    pass accumulates with global REDs -- same bit-exact COUNT."""
    _gpu()
    from paper_2010_12548_b200 import workloads as W

    regions = W.voronoi_tiling(3000, 1.0, seed=4, verts=(10, 30))
    grid = UNIT.with_level(13)
    rng = np.random.default_rng(8)
    xy = rng.random((1_000_001, 2))
    xy32 = xy.astype(np.float32)
    attr = rng.lognormal(2.5, 0.6, len(xy)).astype(np.float32)
    for mode in (0, 1):
        A, _ = oracle_approx(oracle_lib, regions, grid, mode)
        idx = _prepared(regions, grid, mode, "trie")
        _assert_join(idx, A, xy, attr)
        _assert_join(idx, A, xy32, attr)


@pytest.mark.parametrize("fold", ["1", "3"])
def test_ring_drains_and_out_of_window_sums(oracle_lib, monkeypatch, fold):
    """The ring kernel's barrier-free drains of the 16-bit fixed-point halves
    (forced every `fold` warp-tiles via RB_FOLD), the per-warp rare queue, and
    attribute values outside the fixed-point window (tiny, huge, zero,
    negative) that take the float64 path: COUNT bit-exact, SUM rel 1e-6."""
    _gpu()
    from paper_2010_12548_b200 import workloads as W
    from paper_2010_12548_b200.grid import level_for_bound

    monkeypatch.setenv("RB_FOLD", fold)
    w = W.c2(n=3_000_003)  # not a multiple of 4: the trailing-point path too
    grid = w.grid.with_level(level_for_bound(w.grid, w.epsilon))
    attr = w.attrs["fare"].copy()
    rng = np.random.default_rng(5)
    k = rng.choice(len(attr), 20_000, replace=False)
    attr[k[:5000]] *= 1e-6          # below the window
    attr[k[5000:10000]] *= 1e6      # above the window
    attr[k[10000:15000]] = 0.0
    attr[k[15000:]] *= -1.0         # negative values: signed fixed point
    A, _ = oracle_approx(oracle_lib, w.regions, grid, 0)
    idx = _prepared(w.regions, grid, 0, "trie")
    _assert_join(idx, A, w.xy, attr)


def test_single_hot_region_copies(oracle_lib):
    """Every point in one region (the worst case for same-address REDs that the
    bank-staggered histogram copies absorb): exact COUNT, SUM within 1e-6."""
    _gpu()
    from paper_2010_12548_b200.geometry import Polygon, RegionRecord

    regions = [RegionRecord(0, Polygon([(0.0, 0.0), (0.5, 0.0), (0.5, 0.5), (0.0, 0.5)])),
               RegionRecord(1, Polygon([(0.5, 0.5), (1.0, 0.5), (1.0, 1.0), (0.5, 1.0)]))]
    grid = UNIT.with_level(12)
    rng = np.random.default_rng(9)
    xy = rng.random((2_000_000, 2)) * 0.49  # all inside region 0's interior
    attr = rng.lognormal(2.5, 0.6, len(xy)).astype(np.float32)
    A, _ = oracle_approx(oracle_lib, regions, grid, 0)
    idx = _prepared(regions, grid, 0, "trie")
    cnt = _assert_join(idx, A, xy, attr)
    assert cnt[0, 0] == len(xy)


@pytest.mark.parametrize("root_level,radix_width", [(8, 8), (6, 8), (2, 8), (5, 4)])
@pytest.mark.parametrize("hot", ["all", "some"])
def test_deep_index_kernel(oracle_lib, monkeypatch, root_level, radix_width, hot):
    """k_point_pass_deep: 3000 regions (histogram beyond shared memory) with two
    or more node levels below the root (root level 8 -> node split 1+4, 6 -> 3+4,
    2 -> 3+4+4, 5 with radix width 4 -> 2+2+2+2),
    hot slots for all or only some regions (cold regions and boundary leaves
    take global REDs), forced drains, out-of-window attributes, clustered
    points, a trailing partial tile: COUNT bit-exact, SUM within 1e-6."""
    _gpu()
    from paper_2010_12548_b200 import workloads as W

    monkeypatch.setenv("RB_FOLD", "2")
    regions = W.voronoi_tiling(3000, 1.0, seed=4, verts=(10, 30))
    grid = UNIT.with_level(13)
    rng = np.random.default_rng(11)
    n = 1_500_003
    cen = rng.random((12, 2))
    xy = np.clip(cen[rng.integers(0, 12, n)] + rng.normal(0, 0.05, (n, 2)), 0.0, 0.999999)
    attr = rng.lognormal(2.5, 0.6, n).astype(np.float32)
    k = rng.choice(n, 6000, replace=False)
    attr[k[:2000]] *= 1e-6
    attr[k[2000:4000]] = 0.0
    attr[k[4000:]] *= -1.0
    for mode in (0, 1):
        A, _ = oracle_approx(oracle_lib, regions, grid, mode)
        idx = _prepared(regions, grid, mode, "trie", root_level=root_level, radix_width=radix_width)
        st = idx.stats()
        assert st["root_level"] == root_level
        if hot == "some":
            idx.set_hot(np.arange(0, 3000, 7))
        _assert_join(idx, A, xy, attr)
        _assert_join(idx, A, xy.astype(np.float32), attr)
        _assert_join(idx, A, xy, None)


@pytest.mark.parametrize("mode", [0, 1])
def test_sorted_key_layout(oracle_lib, mode):
    """RB_LAYOUT_KEYS (sorted 64-bit cell keys + radix table over the top key
    bits): overlapping polygons with holes (owner lists), the C2 generator
    (SUM), and 3000 regions (global histogram), f64 and f32 points; plus
    act_lookup and the complete validator through the same index."""
    torch = _gpu()
    from paper_2010_12548_b200 import workloads as W
    from paper_2010_12548_b200.grid import level_for_bound
    from paper_2010_12548_b200.validate import validate_full

    rng = np.random.default_rng(21)
    cases = [(random_polygons(8, 25, holes=True), UNIT.with_level(11), rng.random((400_003, 2)), None)]
    w = W.c2(n=1_000_001)
    cases.append((w.regions, w.grid.with_level(level_for_bound(w.grid, w.epsilon)), w.xy, w.attrs["fare"]))
    cases.append((W.voronoi_tiling(3000, 1.0, seed=4, verts=(10, 30)), UNIT.with_level(12), rng.random((300_001, 2)),
                  rng.lognormal(2.5, 0.6, 300_001).astype(np.float32)))
    for regions, grid, xy, attr in cases:
        A, _ = oracle_approx(oracle_lib, regions, grid, mode)
        idx = _prepared(regions, grid, mode, "keys")
        _assert_join(idx, A, xy, attr)
        _assert_join(idx, A, xy.astype(np.float32), None)
        trie = _prepared(regions, grid, mode, "trie")
        sample = xy[:50_000]
        assert torch.equal(idx.lookup(sample), trie.lookup(sample))
    rep = validate_full(idx, xy, 1.0 / (1 << 12))
    assert rep.owner_set_overflows == 0


@pytest.mark.parametrize("L", [0, 1, 2])
def test_sorted_key_layout_tiny_grids(oracle_lib, L):
    """RB_LAYOUT_KEYS at L = 0..2 (a bucket table of 1..16 slots) and with no
    owner at all, against the oracle and the radix table."""
    torch = _gpu()
    rng = np.random.default_rng(40 + L)
    regions = random_polygons(9, 6)
    grid = UNIT.with_level(L)
    xy = rng.random((50_003, 2))
    A, _ = oracle_approx(oracle_lib, regions, grid, 0)
    idx = _prepared(regions, grid, 0, "keys")
    _assert_join(idx, A, xy, rng.random(len(xy)).astype(np.float32))
    assert torch.equal(idx.lookup(xy), _prepared(regions, grid, 0, "trie").lookup(xy))
    from paper_2010_12548_b200.geometry import Polygon, RegionRecord

    far = [RegionRecord(0, Polygon([(0.01, 0.01), (0.02, 0.01), (0.02, 0.02)]))]  # touches no sample point's cell
    idx2 = _prepared(far, UNIT.with_level(8), 0, "keys")
    A2, _ = oracle_approx(oracle_lib, far, UNIT.with_level(8), 0)
    _assert_join(idx2, A2, 0.5 + 0.4 * rng.random((10_001, 2)))
