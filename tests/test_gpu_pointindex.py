"""GPU parity of the point-side path through the
C-ABI: lps_build codes/perm bit-exact and prefix sums vs the numpy oracle,
the RadixSpline error audit, RS bounds == binary search, the SPEC examples,
and join_pointindex == join_act (COUNT and beta exact, SUM within 1e-6)."""
import json
import os

import numpy as np
import pytest

from helpers import UNIT, random_polygons

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
EX = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))["examples"]


def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_lps_matches_oracle():
    _gpu()
    from oracle import pointindex_oracle as PO
    from paper_2010_12548_b200 import pointindex as P
    from paper_2010_12548_b200 import workloads as W
    from paper_2010_12548_b200.grid import level_for_bound

    w = W.c2(n=2_000_000)
    grid = w.grid.with_level(level_for_bound(w.grid, w.epsilon))
    from paper_2010_12548_b200.geometry import PointSet

    lps = P.lps_build(PointSet(w.xy, {"fare": w.attrs["fare"]}), grid, ["fare"])
    codes, perm, prefix = PO.lps_build(w.xy, (grid.origin.x, grid.origin.y), grid.extent, grid.max_level,
                                       {"fare": w.attrs["fare"]})
    np.testing.assert_array_equal(lps.codes.cpu().numpy().view(np.uint64), codes)
    np.testing.assert_array_equal(lps.perm.cpu().numpy(), perm)
    np.testing.assert_allclose(lps.prefix("fare").cpu().numpy(), prefix["fare"], rtol=1e-9, atol=1e-6)
    c = lps.prefix("COUNT").cpu().numpy()
    assert c[0] == 0 and c[-1] == len(w.xy)


@pytest.mark.parametrize("kind", ["city", "duplicates"])
def test_radix_spline_audit_and_bounds_equal_binary_search(kind):
    torch = _gpu()
    from oracle import pointindex_oracle as PO
    from paper_2010_12548_b200 import pointindex as P
    from paper_2010_12548_b200 import workloads as W
    from paper_2010_12548_b200.grid import GridConfig, level_for_bound
    from paper_2010_12548_b200.geometry import Point2D

    if kind == "city":
        w = W.c2(n=3_000_000)
        grid = w.grid.with_level(level_for_bound(w.grid, w.epsilon))
        xy = w.xy
    else:  # few distinct leaves, many duplicates
        grid = GridConfig(Point2D(0.0, 0.0), 1.0, 6)
        xy = np.random.default_rng(2).random((500_000, 2))
    lps = P.lps_build(xy, grid)
    rs = P.rs_build(lps, radix_bits=min(18, 2 * grid.max_level), max_error=32)
    codes = lps.codes.cpu().numpy().view(np.uint64)
    keys, pos = (t.cpu().numpy() for t in rs.knots)
    keys = keys.view(np.uint64)
    assert np.all(np.diff(keys.astype(np.float64)) > 0)
    assert PO.spline_errors(codes, keys, pos).max() <= 32          # SPEC.md:366 error audit
    np.testing.assert_array_equal(rs.radix_table.cpu().numpy(),
                                  PO.radix_table(keys, rs.radix_bits, 2 * grid.max_level))
    rng = np.random.default_rng(7)
    width = 2 * grid.max_level
    lo = rng.integers(0, 1 << width, 1_000_000, dtype=np.uint64)
    ln = rng.integers(0, 1 << max(width - 6, 1), 1_000_000, dtype=np.uint64)
    hi = np.minimum(lo + ln, np.uint64(1 << width))
    lo[:1000] = codes[rng.integers(0, len(codes), 1000)]  # stored keys too
    want = PO.bounds_lookup(codes, lo, hi)
    with pytest.raises(Exception):
        P.rs_build(lps, radix_bits=width + 1)  # SPEC.md:340 configuration error
    for r in (rs, None):                                   # SPEC.md:365 RS == binary search
        a, b = P.bounds_lookup(lps, r, (lo, hi))
        np.testing.assert_array_equal(a.cpu().numpy(), want[0])
        np.testing.assert_array_equal(b.cpu().numpy(), want[1])


@pytest.mark.parametrize("e", [e for e in EX if e["op"] in ("lps_build", "range_aggregate")],
                         ids=lambda e: e["spec"])
def test_spec_examples_gpu(e):
    _gpu()
    from paper_2010_12548_b200 import pointindex as P
    from paper_2010_12548_b200.geometry import Point2D, PointSet
    from paper_2010_12548_b200.grid import CellInterval, GridConfig

    if e["op"] == "lps_build":
        xy = np.asarray(e["points"], float).reshape(-1, 2)
        lps = P.lps_build(PointSet(xy, {"w": np.ones(len(xy), np.float32)}), GridConfig(Point2D(0, 0), 1.0, e["L"]),
                          ["w"])
        codes = lps.codes.cpu().numpy().view(np.uint64).tolist()
        if "expect_codes" in e:
            assert codes == e["expect_codes"]
        if "expect_prefix" in e:
            assert lps.prefix("w").cpu().numpy().tolist() == e["expect_prefix"]
        if "expect_count_prefix" in e:
            got = [P.range_aggregate(lps, None, [CellInterval(0, c)]) for c in range(5)]
            assert got == e["expect_count_prefix"]
        if e.get("expect_codes_equal_adjacent"):
            assert codes[0] == codes[1]
    else:
        # codes [0,1,1,3,3,3] at L=1 from points in the unit square
        pts = np.array([[0.1, 0.1], [0.6, 0.2], [0.9, 0.4], [0.7, 0.7], [0.8, 0.9], [0.55, 0.6]])
        lps = P.lps_build(pts, GridConfig(Point2D(0, 0), 1.0, 1))
        assert lps.codes.cpu().numpy().tolist() == e["codes"]
        rs = P.rs_build(lps, radix_bits=2, max_error=0)
        cells = [CellInterval(*c) for c in e["cells"]]
        assert P.range_aggregate(lps, rs, cells) == e["expect"]
        assert P.range_aggregate(lps, None, cells) == e["expect"]


def test_bounds_examples_gpu():
    _gpu()
    from paper_2010_12548_b200 import pointindex as P
    from paper_2010_12548_b200.geometry import Point2D
    from paper_2010_12548_b200.grid import CellInterval, GridConfig

    # points with codes [2, 4, 4, 7, 9, 12] at L=2 (x in the even bits)
    def cell_center(z):
        x = (z & 1) | ((z >> 1) & 2)
        y = ((z >> 1) & 1) | ((z >> 2) & 2)
        return [(x + 0.5) / 4, (y + 0.5) / 4]

    pts = np.array([cell_center(z) for z in (2, 4, 4, 7, 9, 12)])
    lps = P.lps_build(pts, GridConfig(Point2D(0, 0), 1.0, 2))
    assert lps.codes.cpu().numpy().tolist() == [2, 4, 4, 7, 9, 12]
    rs = P.rs_build(lps, radix_bits=3, max_error=1)
    for e in [e for e in EX if e["op"] == "bounds_lookup"]:
        iv = CellInterval(e["iv"][0], min(e["iv"][1], 16))
        for r in (rs, None):
            assert list(P.bounds_lookup(lps, r, iv)) == e["expect"]


@pytest.mark.parametrize("seed", list(range(12)))
def test_join_pointindex_equals_join_act(oracle_lib, seed):
    """SPEC.md:497 engine cross-check on seeded workloads (random overlapping
    polygons with holes, both modes, COUNT and SUM)."""
    torch = _gpu()
    from paper_2010_12548_b200 import pointindex as P
    from paper_2010_12548_b200.geometry import PointSet
    from paper_2010_12548_b200.query import AggregationQuery, join_act, join_pointindex
    from paper_2010_12548_b200.raster import RasterMode

    rng = np.random.default_rng(100 + seed)
    regions = random_polygons(seed, k=int(rng.integers(3, 25)), holes=True)
    L = int(rng.integers(6, 13))
    eps = UNIT.extent * 2.0 ** -L * np.sqrt(2.0) * 1.000001
    grid = UNIT.with_level(L)
    xy = rng.random((int(rng.integers(1000, 300_000)), 2))
    fare = rng.lognormal(2.5, 0.6, len(xy)).astype(np.float32)
    pts = PointSet(xy, {"fare": fare})
    lps = P.lps_build(pts, grid, ["fare"])
    rs = P.rs_build(lps, radix_bits=min(16, 2 * L), max_error=32) if seed % 2 else None
    for mode in (RasterMode.CONSERVATIVE, RasterMode.CENTER_SAMPLED):
        for agg in ("COUNT", "SUM:fare"):
            q = AggregationQuery(agg, eps, mode)
            a = join_act(pts, regions, q, cfg=UNIT)
            b = join_pointindex(lps, rs, regions, q)
            assert [r.region_id for r in a] == [r.region_id for r in b]
            for x, y in zip(a, b):
                if agg == "COUNT":
                    assert (x.alpha, x.boundary_part, x.range) == (y.alpha, y.boundary_part, y.range)
                else:
                    np.testing.assert_allclose([y.alpha, y.boundary_part], [x.alpha, x.boundary_part],
                                               rtol=1e-6, atol=1e-6)


def test_join_pointindex_multipolygon_regions(oracle_lib):
    """Multi-polygon regions (overlapping parts): union of coverings, coarser
    cell wins -- equal to join_act."""
    _gpu()
    from paper_2010_12548_b200 import pointindex as P
    from paper_2010_12548_b200.geometry import RegionRecord
    from paper_2010_12548_b200.query import AggregationQuery, join_act, join_pointindex

    polys = random_polygons(11, k=12, holes=True)
    regions = [RegionRecord(7, [polys[0].geometry, polys[1].geometry, polys[2].geometry]),
               RegionRecord(3, [polys[3].geometry, polys[4].geometry]),
               RegionRecord(9, polys[5].geometry)]
    grid = UNIT.with_level(10)
    xy = np.random.default_rng(4).random((200_000, 2))
    lps = P.lps_build(xy, grid)
    rs = P.rs_build(lps)
    q = AggregationQuery("COUNT", 2.0 ** -10 * np.sqrt(2.0) * 1.000001)
    a = join_act(xy, regions, q, cfg=UNIT)
    b = join_pointindex(lps, rs, regions, q)
    assert [(r.region_id, r.alpha, r.boundary_part) for r in a] == [(r.region_id, r.alpha, r.boundary_part) for r in b]
