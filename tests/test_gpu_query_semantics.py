"""Query-level semantics against the oracle (SPEC.md:95,240-242,
253,358,363,473,485,489-490,517): attribute filters, AVG with its empty-result
marker, multi-polygon regions (union of coverings, the coarser cell kept),
approx_contains's three properties, the join_act examples, and the SUM
numerics (fixed-point accumulation: per value relative error <= 2^-21,
exact float64 adds outside the window; mixed-sign sums bounded by
2^-21 * sum |w|)."""
import math

import numpy as np
import pytest

from helpers import UNIT, oracle_approx, random_polygons

pytestmark = pytest.mark.gpu

FIXED_POINT_REL = 2.0 ** -21


def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _workload(seed=3, n=200_000, k=25):
    regions = random_polygons(seed, k=k, holes=True)
    rng = np.random.default_rng(seed)
    xy = rng.random((n, 2))
    fare = rng.lognormal(2.5, 0.6, n).astype(np.float32)
    tip = rng.normal(0.0, 5.0, n).astype(np.float32)
    return regions, xy, fare, tip


@pytest.mark.parametrize("op,val", [(">", 15.0), ("<=", 9.5), ("!=", 0.0)])
def test_filter_matches_oracle_on_filtered_points(oracle_lib, op, val):
    """only points passing the filter are joined."""
    _gpu()
    from paper_2010_12548_b200.geometry import PointSet
    from paper_2010_12548_b200.query import AggregationQuery, join_act

    regions, xy, fare, _ = _workload()
    grid = UNIT.with_level(10)
    q = AggregationQuery(("SUM", "fare"), epsilon=grid.side() * math.sqrt(2.0), filter=("fare", op, val))
    res = join_act(PointSet(xy, {"fare": fare}), regions, q, cfg=UNIT)
    m = {">": fare > val, "<=": fare <= val, "!=": fare != val}[op]
    A, _ = oracle_approx(oracle_lib, regions, grid, 0)
    cnt_o, sum_o = A.join(xy[m], fare[m], nthreads=8)
    got_s = np.array([[r.alpha, r.boundary_part] for r in res])
    np.testing.assert_allclose(got_s, sum_o, rtol=1e-6, atol=1e-9)
    qc = AggregationQuery("COUNT", epsilon=q.epsilon, filter=("fare", op, val))
    rc = join_act(PointSet(xy, {"fare": fare}), regions, qc, cfg=UNIT)
    np.testing.assert_array_equal(np.array([[r.alpha, r.boundary_part] for r in rc]), cnt_o)


def test_avg_and_empty_marker(oracle_lib):
    """AVG = SUM / COUNT; a region without points gives the
    empty-result marker (not 0); AVG has no range."""
    _gpu()
    from paper_2010_12548_b200.geometry import Polygon, PointSet, RegionRecord
    from paper_2010_12548_b200.query import EMPTY, UNAVAILABLE, AggregationQuery, join_act

    regions, xy, fare, _ = _workload()
    # a region far from every point: points live in [0, 0.5)^2 only
    xy = xy * 0.5
    regions = regions + [RegionRecord(99, Polygon([(0.8, 0.8), (0.95, 0.8), (0.95, 0.95), (0.8, 0.95)]))]
    grid = UNIT.with_level(10)
    q = AggregationQuery(("AVG", "fare"), epsilon=grid.side() * math.sqrt(2.0))
    res = join_act(PointSet(xy, {"fare": fare}), regions, q, cfg=UNIT)
    A, packed = oracle_approx(oracle_lib, regions, grid, 0)
    cnt_o, sum_o = A.join(xy, fare, nthreads=8)
    for k, r in enumerate(res):
        assert r.range is UNAVAILABLE
        for col, got in ((0, r.alpha), (1, r.boundary_part)):
            if cnt_o[k, col] == 0:
                assert got is EMPTY or (isinstance(got, float) and math.isnan(got))
            else:
                assert got == pytest.approx(sum_o[k, col] / cnt_o[k, col], rel=1e-6)
    assert res[-1].region_id == 99 and math.isnan(res[-1].alpha)


def test_multipolygon_regions_union_and_coarser_cell(oracle_lib):
    """a region of several polygons (one nested inside
    another of the same region, one overlapping another region) counts each
    point once per region; the nested polygon's cells merge into the coarser
    covering cell."""
    _gpu()
    from paper_2010_12548_b200.geometry import Polygon, PointSet, RegionRecord
    from paper_2010_12548_b200.query import AggregationQuery, join_act
    from paper_2010_12548_b200.raster import rasterize_hierarchical

    big = Polygon([(0.1, 0.1), (0.6, 0.1), (0.6, 0.6), (0.1, 0.6)])
    inner = Polygon([(0.2, 0.2), (0.3, 0.2), (0.25, 0.33)])
    far = Polygon([(0.7, 0.7), (0.9, 0.72), (0.8, 0.9)])
    other = Polygon([(0.5, 0.5), (0.8, 0.55), (0.65, 0.8)])
    regions = [RegionRecord(0, [big, inner, far]), RegionRecord(1, other), RegionRecord(2, [inner])]
    rng = np.random.default_rng(5)
    xy = rng.random((300_000, 2))
    grid = UNIT.with_level(9)
    A, _ = oracle_approx(oracle_lib, regions, grid, 0)
    cnt_o, _ = A.join(xy, None, nthreads=8)
    res = join_act(PointSet(xy), regions, AggregationQuery("COUNT", epsilon=grid.side() * math.sqrt(2.0)), cfg=UNIT)
    np.testing.assert_array_equal(np.array([[r.alpha, r.boundary_part] for r in res]), cnt_o)
    # union covering: disjoint cells, no cell of the nested polygon survives inside a coarser cell
    r = rasterize_hierarchical([big, inner, far], UNIT, grid.side() * math.sqrt(2.0))
    lo, hi, _ = r.intervals()
    assert np.all(lo[1:] >= hi[:-1])
    single = rasterize_hierarchical(big, UNIT, grid.side() * math.sqrt(2.0))
    lo1, hi1, _ = single.intervals()
    inside = (lo >= np.uint64(lo1.min())) & (hi <= np.uint64(hi1.max()))
    assert inside.sum() <= len(lo1)  # the inner polygon adds no finer cell within big's covering


@pytest.mark.parametrize("mode", [0, 1])
def test_approx_contains_properties(oracle_lib, mode):
    """SPEC.md:240-242 on 4000 points: deep interior (distance > eps) equals exact
    PIP; CONSERVATIVE has no false negatives; distance > eps and outside gives false."""
    _gpu()
    from oracle import oracle as O
    from paper_2010_12548_b200.geometry import Point2D
    from paper_2010_12548_b200.raster import RasterMode, approx_contains, rasterize_hierarchical

    regions = random_polygons(13, k=3, holes=True)
    poly = regions[0].geometry
    eps = 0.01
    r = rasterize_hierarchical(poly, UNIT, eps, RasterMode(mode))
    rng = np.random.default_rng(7)
    pts = rng.random((4000, 2))
    rings = poly.rings
    vx = np.concatenate([g[:, 0] for g in rings])
    vy = np.concatenate([g[:, 1] for g in rings])
    ro = np.concatenate([[0], np.cumsum([len(g) for g in rings])]).astype(np.int64)
    pip = O.pip(vx, vy, ro, pts[:, 0], pts[:, 1])
    dist = O.distance(vx, vy, ro, pts[:, 0], pts[:, 1])
    got = np.array([approx_contains(r, Point2D(float(x), float(y))) for x, y in pts])
    deep = dist > eps
    assert deep.sum() > 1000
    np.testing.assert_array_equal(got[deep], pip[deep])
    assert not np.any(got[deep & ~pip])
    if mode == 0:
        assert np.all(got[pip])
    assert np.all(dist[got != pip] <= eps)


def test_join_act_spec_examples(oracle_lib):
    """whole-domain region with 7 points -> alpha 7, beta 0,
    range [7, 7]; 10 polygons x 10^4 points -> alpha per region equals the
    per-point approx_contains count over the covering; a point in a boundary
    cell only contributes to both alpha and beta."""
    _gpu()
    from paper_2010_12548_b200.geometry import Point2D, Polygon, PointSet, RegionRecord
    from paper_2010_12548_b200.query import AggregationQuery, join_act
    from paper_2010_12548_b200.raster import approx_contains, rasterize_hierarchical

    whole = [RegionRecord(5, Polygon([(0.0, 0.0), (1.0, 0.0), (1.0, 1.0), (0.0, 1.0)]))]
    pts = np.random.default_rng(1).random((7, 2)) * 0.9 + 0.05
    (r,) = join_act(PointSet(pts), whole, AggregationQuery("COUNT", epsilon=0.05), cfg=UNIT)
    assert (r.region_id, r.alpha, r.boundary_part, r.range) == (5, 7, 0, (7, 7))

    regions = random_polygons(21, k=10)
    xy = np.random.default_rng(2).random((10_000, 2))
    eps = 0.02
    res = join_act(PointSet(xy), regions, AggregationQuery("COUNT", epsilon=eps), cfg=UNIT)
    for reg, rr in zip(regions, res):
        cov = rasterize_hierarchical(reg.geometry, UNIT, eps)
        exp = sum(approx_contains(cov, Point2D(float(x), float(y))) for x, y in xy)
        assert rr.alpha == exp

    # a point inside one boundary leaf of a square that is not grid aligned
    sq = [RegionRecord(0, Polygon([(0.3, 0.3), (0.7, 0.3), (0.7, 0.7), (0.3, 0.7)]))]
    L = 5  # side 1/32: the edge x = 0.3 cuts leaf column 9 ([0.28125, 0.3125))
    eps = (1.0 / 32) * math.sqrt(2.0)
    p = np.array([[0.29, 0.5]])
    (rr,) = join_act(PointSet(p), sq, AggregationQuery("COUNT", epsilon=eps), cfg=UNIT)
    assert (rr.alpha, rr.boundary_part) == (1, 1)
    assert rr.range == (0, 1)


def test_mixed_sign_sum_within_fixed_point_bound(oracle_lib):
    """SUM numerics under cancellation: the device SUM differs from a float64
    sum of the same float32 values by at most 2^-21 * sum |w| per region (the
    fixed-point window's per-value bound); COUNT stays exact."""
    torch = _gpu()
    regions, xy, _, tip = _workload(seed=9, n=400_000)
    grid = UNIT.with_level(10)
    A, _ = oracle_approx(oracle_lib, regions, grid, 0)
    cnt_o, sum_o = A.join(xy, tip, nthreads=8)
    _, abs_o = A.join(xy, np.abs(tip), nthreads=8)
    from paper_2010_12548_b200.engine import ApproxIndex
    from paper_2010_12548_b200.geometry import pack_regions

    idx = ApproxIndex(pack_regions(regions), grid, 0, layout="trie")
    r = idx.point_pass(torch.as_tensor(xy).cuda(), torch.as_tensor(tip).cuda()).check()
    np.testing.assert_array_equal(r.cnt.cpu().numpy(), cnt_o)
    err = np.abs(r.sum.cpu().numpy() - sum_o)
    assert np.all(err <= FIXED_POINT_REL * abs_o + 1e-9), float(np.max(err / np.maximum(abs_o, 1e-30)))


def test_float64_attribute_is_summed_in_two_parts(oracle_lib):
    """A float64 attribute is not truncated to float32: it is summed as a float32
    high part plus the float32 residual, so a region's SUM is within the
    fixed-point bound of the float64 values (not of their float32 rounding)."""
    torch = _gpu()
    regions, xy, _, _ = _workload(seed=4, n=200_000)
    grid = UNIT.with_level(10)
    w = 123456789.12 + np.random.default_rng(0).random(len(xy))  # float32 would lose ~4 units per value
    A, _ = oracle_approx(oracle_lib, regions, grid, 0)
    # oracle in two exact float32 parts: hi + lo == w up to 2^-48 relative
    hi = w.astype(np.float32)
    lo = (w - hi.astype(np.float64)).astype(np.float32)
    cnt_o, s_hi = A.join(xy, hi, nthreads=8)
    _, s_lo = A.join(xy, lo, nthreads=8)
    exact = s_hi + s_lo
    from paper_2010_12548_b200.engine import ApproxIndex
    from paper_2010_12548_b200.geometry import pack_regions

    idx = ApproxIndex(pack_regions(regions), grid, 0, layout="trie")
    r = idx.point_pass(torch.as_tensor(xy).cuda(), torch.as_tensor(w).cuda()).check()
    np.testing.assert_array_equal(r.cnt.cpu().numpy(), cnt_o)
    np.testing.assert_allclose(r.sum.cpu().numpy(), exact, rtol=1e-6, atol=1e-9)
    f32_only = idx.point_pass(torch.as_tensor(xy).cuda(), torch.as_tensor(hi).cuda()).sum.cpu().numpy()
    assert np.max(np.abs(r.sum.cpu().numpy() - exact)) < np.max(np.abs(f32_only - exact))


def test_spec_literal_tier_float64_mixed_sign_sums():
    """the SPEC-literal tier (float64 attribute values, Python float
    accumulation) checks a float64, mixed-sign SUM: the device result lies within
    2^-21 * sum |w| of it (the float64 attribute takes the two-part path)."""
    torch = _gpu()
    from oracle import spec_literal as SL
    from paper_2010_12548_b200.engine import ApproxIndex
    from paper_2010_12548_b200.geometry import pack_regions

    regions = random_polygons(17, k=6, holes=True)
    L = 7
    grid = UNIT.with_level(L)
    rng = np.random.default_rng(3)
    xy = rng.random((20_000, 2))
    w = rng.normal(0.0, 1e6, len(xy)) + rng.random(len(xy)) * 1e-3  # float64, mixed sign, not float32-exact
    trie, _ = SL.build([(r.id, [p.rings]) for r in regions for p in [r.geometry]], (0.0, 0.0), 1.0, L)
    ref = SL.join_act(xy.tolist(), trie, (0.0, 0.0), 1.0, w.tolist())
    ref_abs = SL.join_act(xy.tolist(), trie, (0.0, 0.0), 1.0, np.abs(w).tolist())
    idx = ApproxIndex(pack_regions(regions), grid, 0, layout="trie")
    r = idx.point_pass(torch.as_tensor(xy).cuda(), torch.as_tensor(w).cuda()).check()
    cnt, sm = r.cnt.cpu().numpy(), r.sum.cpu().numpy()
    for k, reg in enumerate(regions):
        a = ref.get(reg.id, [0, 0, 0.0, 0.0])
        b = ref_abs.get(reg.id, [0, 0, 0.0, 0.0])
        assert (cnt[k, 0], cnt[k, 1]) == (a[0], a[1])
        assert abs(sm[k, 0] - a[2]) <= FIXED_POINT_REL * b[2] + 1e-9
        assert abs(sm[k, 1] - a[3]) <= FIXED_POINT_REL * b[3] + 1e-9
