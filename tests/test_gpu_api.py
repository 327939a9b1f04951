"""The public rasterbound API (GPU path) on the SPEC golden vectors, error
behaviour, aggregates/filters, host-buffer join and the epsilon validator."""
import json
import math
import os

import numpy as np
import pytest

from helpers import UNIT, random_polygons

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
EX = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))["examples"]


def by_op(op):
    return [e for e in EX if e["op"] == op]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("e", by_op("point_in_polygon"), ids=lambda e: e["spec"])
def test_point_in_polygon(e):
    import rasterbound.geometry as G

    poly = G.Polygon(e["outer"], e["holes"])
    assert G.point_in_polygon(G.Point2D(*e["p"]), poly) == e["expect"]


@pytest.mark.parametrize("e", by_op("distance_to_boundary"), ids=lambda e: e["spec"])
def test_distance_to_boundary(e):
    import rasterbound.geometry as G

    d = G.distance_to_boundary(G.Point2D(*e["p"]), G.Polygon(e["outer"]))
    assert d == pytest.approx(e["expect"], abs=1e-15)


def test_hausdorff():
    import rasterbound.geometry as G

    for e in by_op("hausdorff_distance"):
        assert G.hausdorff_distance(e["A"], e["B"]) == pytest.approx(e["expect"], abs=1e-12)
    e = by_op("hausdorff_squares")[0]
    g = np.arange(0.0, 1.0 + 1e-9, 1 / 200)
    X, Y = np.meshgrid(g, g)
    B = np.stack([X.ravel(), Y.ravel()], 1)
    A = B[(B[:, 0] >= 0.25) & (B[:, 0] <= 0.75) & (B[:, 1] >= 0.25) & (B[:, 1] <= 0.75)]
    assert G.hausdorff_distance(A, B) == pytest.approx(e["expect"], abs=1e-9)


@pytest.mark.parametrize("e", by_op("classify_cell"), ids=lambda e: e["spec"])
def test_classify_cell(e):
    import rasterbound.geometry as G
    import rasterbound.grid as Gr
    import rasterbound.raster as R

    c = R.classify_cell(Gr.CellId(*e["cell"]), G.Polygon(e["outer"]), UNIT)
    assert c.value == e["expect"]


@pytest.mark.parametrize("e", by_op("rasterize_hierarchical") + by_op("rasterize_uniform"), ids=lambda e: e["spec"])
def test_rasterize(e):
    import rasterbound.geometry as G
    import rasterbound.grid as Gr
    import rasterbound.raster as R

    cfg = Gr.GridConfig((0.0, 0.0), e["extent"])
    fn = R.rasterize_hierarchical if e["op"] == "rasterize_hierarchical" else R.rasterize_uniform
    r = fn(G.Polygon(e["outer"]), cfg, e["epsilon"])
    assert sorted([c.level, c.code] for c in r.interior) == e["expect_interior"]
    assert sorted([c.level, c.code] for c in r.boundary) == e["expect_boundary"]


@pytest.mark.parametrize("e", by_op("act_lookup"), ids=lambda e: e["spec"])
def test_act_build_lookup(e):
    import rasterbound.act as A
    import rasterbound.geometry as G
    import rasterbound.raster as R

    covers = [R.rasterize_hierarchical(G.Polygon(ring), UNIT, e["epsilon"], region_id=int(rid))
              for rid, ring in e["regions"].items()]
    t = A.act_build(covers, radix_width=8)
    for p, exp in zip(e["points"], e["expect"]):
        assert sorted(A.act_lookup(t, G.Point2D(*p))) == sorted(tuple(x) for x in exp)


def test_act_duplicate_cells_idempotent_and_widths():
    import rasterbound.act as A
    import rasterbound.geometry as G
    import rasterbound.raster as R

    regs = random_polygons(3, k=8)
    covers = [R.rasterize_hierarchical(r.geometry, UNIT, 0.01, region_id=r.id) for r in regs]
    xy = np.random.default_rng(0).random((4000, 2))
    ref = A.act_lookup_many(A.act_build(covers), xy)
    for w in (2, 4):
        assert A.act_lookup_many(A.act_build(covers + covers[:3], radix_width=w, root_level=0), xy) == ref
    # every index layout the engine has is reachable from act_build (keys was not)
    for layout in ("dense", "keys", "packed"):
        assert A.act_lookup_many(A.act_build(covers + covers[:3], layout=layout), xy) == ref, layout


@pytest.mark.parametrize("engine", ["act", "canvas"])
def test_join_whole_domain(engine):
    import rasterbound.geometry as G
    import rasterbound.query as Q

    e = by_op("join_act")[0]
    fn = Q.join_act if engine == "act" else Q.join_canvas
    res = fn(e["points"], [G.RegionRecord(0, G.Polygon(e["outer"]))], Q.AggregationQuery("COUNT", e["epsilon"]), UNIT)
    assert (res[0].alpha, res[0].boundary_part, list(res[0].range)) == (7, 0, [7, 7])


def test_join_engines_agree_and_ranges_sound(oracle_lib):
    import rasterbound.geometry as G
    import rasterbound.query as Q

    regs = random_polygons(11, k=40, holes=True)
    rng = np.random.default_rng(4)
    pts = G.PointSet(rng.random((100_000, 2)), {"fare": rng.lognormal(2.5, 0.6, 100_000).astype(np.float32)})
    for agg in ("COUNT", "SUM:fare", "AVG:fare"):
        q = Q.AggregationQuery(agg, 0.005)
        a = Q.join_act(pts, regs, q, UNIT)
        c = Q.join_canvas(pts, regs, q, UNIT)
        for x, y in zip(a, c):
            assert x.region_id == y.region_id
            if agg == "COUNT":
                assert (x.alpha, x.boundary_part) == (y.alpha, y.boundary_part)
            else:
                assert x.alpha == pytest.approx(y.alpha, rel=1e-9, nan_ok=True)
    from paper_2010_12548_b200.validate import validate  # noqa: F401
    packed = __import__("paper_2010_12548_b200.geometry", fromlist=["pack_regions"]).pack_regions(regs)
    exact = np.zeros(packed.n_regions, np.int64)
    for k in range(packed.n_polygons):
        r0, r1 = packed.poly_ring_off[k], packed.poly_ring_off[k + 1]
        v0, v1 = packed.ring_off[r0], packed.ring_off[r1]
        inside = oracle_lib.pip(packed.vx[v0:v1], packed.vy[v0:v1], packed.ring_off[r0:r1 + 1] - v0,
                                pts.xy[:, 0], pts.xy[:, 1])
        exact[packed.poly_region[k]] += inside.sum()
    res = Q.join_act(pts, regs, Q.AggregationQuery("COUNT", 0.005), UNIT)
    for r in res:
        lo, hi = r.range
        assert lo <= exact[r.region_id] <= hi


def test_filter_and_schema_errors():
    import rasterbound.errors as E
    import rasterbound.geometry as G
    import rasterbound.query as Q

    regs = random_polygons(2, k=5)
    rng = np.random.default_rng(5)
    fare = rng.random(20_000).astype(np.float32)
    pts = G.PointSet(rng.random((20_000, 2)), {"fare": fare})
    base = Q.join_act(pts, regs, Q.AggregationQuery("COUNT", 0.01), UNIT)
    sub = Q.join_act(G.PointSet(pts.xy[fare > 0.5], {"fare": fare[fare > 0.5]}), regs,
                     Q.AggregationQuery("COUNT", 0.01), UNIT)
    flt = Q.join_act(pts, regs, Q.AggregationQuery("COUNT", 0.01, filter=("fare", ">", 0.5)), UNIT)
    assert [r.alpha for r in flt] == [r.alpha for r in sub]
    assert sum(r.alpha for r in flt) <= sum(r.alpha for r in base)
    with pytest.raises(E.SchemaError):
        Q.join_act(pts, regs, Q.AggregationQuery("SUM:tip", 0.01), UNIT)
    with pytest.raises(E.SchemaError):
        Q.join_act(pts, regs, Q.AggregationQuery("COUNT", 0.01, filter=("tip", ">", 1)), UNIT)


def test_error_taxonomy_through_the_abi():
    import rasterbound.errors as E
    import rasterbound.geometry as G
    import rasterbound.query as Q
    from paper_2010_12548_b200.engine import ApproxIndex
    from paper_2010_12548_b200.geometry import pack_regions

    regs = random_polygons(1, k=3)
    xy = np.random.default_rng(0).random((5000, 2))
    xy[4321] = (2.0, 0.5)
    with pytest.raises(E.DomainError) as ei:
        Q.join_act(xy, regs, Q.AggregationQuery("COUNT", 0.01), UNIT)
    assert ei.value.index == 4321
    far = [G.RegionRecord(0, G.Polygon([(0.5, 0.5), (3.0, 0.5), (0.5, 3.0)]))]
    with pytest.raises(E.DomainError):
        ApproxIndex(pack_regions(far), UNIT.with_level(4))
    with pytest.raises(E.CapacityError):
        Q.join_canvas(xy[:10], regs, Q.AggregationQuery("COUNT", 1e-6), UNIT)
    with pytest.raises(E.ConfigError):
        ApproxIndex(pack_regions(regs), UNIT.with_level(4), radix_width=3)


def test_join_host_and_device_paths_agree():
    import rasterbound.geometry as G
    import rasterbound.query as Q

    regs = random_polygons(8, k=30)
    rng = np.random.default_rng(6)
    pts = G.PointSet(rng.random((1_000_003, 2)), {"fare": rng.random(1_000_003).astype(np.float32)})
    prep = Q.PreparedJoin(regs, Q.AggregationQuery("SUM:fare", 0.002), UNIT)
    a = prep.run(pts)
    b = prep.run_host(pts)
    for x, y in zip(a, b):
        assert x.alpha == pytest.approx(y.alpha, rel=1e-12) and x.boundary_part == pytest.approx(y.boundary_part, rel=1e-12)


@pytest.mark.parametrize("mode", [0, 1])
def test_epsilon_validator(mode):
    """North star: every point assigned differently from the exact test lies
    within eps of a boundary; CONSERVATIVE has no false negatives."""
    from paper_2010_12548_b200 import workloads as W
    from paper_2010_12548_b200.engine import ApproxIndex
    from paper_2010_12548_b200.geometry import pack_regions
    from paper_2010_12548_b200.grid import level_for_bound
    from paper_2010_12548_b200.validate import validate

    w = W.c2(n=300_000, eps=10.0)
    g = w.grid.with_level(level_for_bound(w.grid, w.epsilon))
    idx = ApproxIndex(pack_regions(w.regions), g, mode)
    rep = validate(idx, w.xy, w.epsilon, max_points=300_000)
    assert rep.ok, rep.as_dict()
    assert rep.mismatched_points > 0  # the approximation is genuinely approximate
    if mode == 0:
        assert rep.false_negatives == 0


@pytest.mark.parametrize("mode", [0, 1])
def test_full_validator_matches_sampled(mode):
    """rb_validate_full (every point, one kernel) agrees with the pairwise
    validator on the same points: same mismatches, same max distance."""
    from paper_2010_12548_b200 import workloads as W
    from paper_2010_12548_b200.engine import ApproxIndex
    from paper_2010_12548_b200.geometry import pack_regions
    from paper_2010_12548_b200.grid import level_for_bound
    from paper_2010_12548_b200.validate import validate, validate_full

    w = W.c2(n=200_000, eps=10.0)
    g = w.grid.with_level(level_for_bound(w.grid, w.epsilon))
    idx = ApproxIndex(pack_regions(w.regions), g, mode)
    a = validate(idx, w.xy, w.epsilon, max_points=None)
    b = validate_full(idx, w.xy, w.epsilon)
    assert b.ok and b.owner_set_overflows == 0, b.as_dict()
    assert b.points == a.points
    assert (b.mismatched_points, b.false_positives, b.false_negatives) == \
        (a.mismatched_points, a.false_positives, a.false_negatives)
    assert b.max_mismatch_distance == pytest.approx(a.max_mismatch_distance, rel=1e-12)
    if mode == 0:
        assert b.false_negatives == 0


def test_full_validator_detects_violation():
    """A coarse index (cells far larger than eps) must be reported."""
    from paper_2010_12548_b200 import workloads as W
    from paper_2010_12548_b200.engine import ApproxIndex
    from paper_2010_12548_b200.geometry import pack_regions
    from paper_2010_12548_b200.validate import validate_full

    w = W.c2(n=100_000, eps=10.0)
    idx = ApproxIndex(pack_regions(w.regions), w.grid.with_level(4), 1)
    b = validate_full(idx, w.xy, w.epsilon)
    assert b.violations > 0 and not b.ok
