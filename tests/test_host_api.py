"""Host logic of the rasterbound API mirror (CPU): scalar grid functions on
the SPEC golden vectors, error taxonomy, aggregate/range policy, CSR packing,
workload generators, and the C-ABI library exports (no GPU compute)."""
import ctypes
import json
import math
import os
import re

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
EX = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))["examples"]


def by_op(op):
    return [e for e in EX if e["op"] == op]


def test_library_exports_every_declared_symbol():
    """librasterbound_b200.so loads on a CPU host and exports every function
    include/rasterbound_b200.h declares."""
    from paper_2010_12548_b200 import _native as N

    hdr = open(os.path.join(ROOT, "include", "rasterbound_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|int32_t|const char\*)\s+(rb_\w+)\(", hdr, re.M))
    assert declared, "no declarations parsed"
    lib = ctypes.CDLL(N.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(N.EXPORTS)
    assert N.load().rb_version() == 10000


@pytest.mark.parametrize("e", by_op("level_for_bound"), ids=lambda e: e["spec"])
def test_level_for_bound_native(e):
    from paper_2010_12548_b200.grid import GridConfig, level_for_bound

    assert level_for_bound(GridConfig((0, 0), e["extent"]), e["epsilon"]) == e["expect"]


def test_level_for_bound_capacity():
    from paper_2010_12548_b200.errors import CapacityError, ConfigError
    from paper_2010_12548_b200.grid import GridConfig, level_for_bound

    with pytest.raises(CapacityError):
        level_for_bound(GridConfig((0, 0), 1.0), 1e-12)
    with pytest.raises(ConfigError):
        level_for_bound(GridConfig((0, 0), 1.0), 0.0)


@pytest.mark.parametrize("e", by_op("z_encode"), ids=lambda e: e["spec"])
def test_z_encode_host(e):
    from paper_2010_12548_b200.grid import z_decode, z_encode

    c = z_encode(e["ix"], e["iy"], e["level"])
    assert c.code == e["expect"] and z_decode(c) == (e["ix"], e["iy"])


def test_z_roundtrip_and_errors():
    from paper_2010_12548_b200.errors import DomainError
    from paper_2010_12548_b200.grid import z_decode, z_encode

    rng = np.random.default_rng(0)
    for L in (0, 3, 10, 20, 31):
        for _ in range(50):
            ix, iy = (int(v) for v in rng.integers(0, 1 << L, 2)) if L else (0, 0)
            assert z_decode(z_encode(ix, iy, L)) == (ix, iy)
    with pytest.raises(DomainError):
        z_encode(4, 0, 2)


@pytest.mark.parametrize("e", by_op("point_to_cell"), ids=lambda e: e["spec"])
def test_point_to_cell_host(e):
    from paper_2010_12548_b200.geometry import Point2D
    from paper_2010_12548_b200.grid import GridConfig, point_to_cell

    c = point_to_cell(GridConfig(tuple(e["origin"]), e["extent"]), Point2D(*e["p"]), e["level"])
    assert [c.level, c.code] == e["expect"]


def test_point_to_cell_domain_error():
    from paper_2010_12548_b200.errors import DomainError
    from paper_2010_12548_b200.geometry import Point2D
    from paper_2010_12548_b200.grid import GridConfig, point_to_cell

    g = GridConfig((0, 0), 1.0)
    for p in (Point2D(1.0, 0.5), Point2D(-1e-9, 0.5), Point2D(float("nan"), 0.1)):
        with pytest.raises(DomainError):
            point_to_cell(g, p, 4)


@pytest.mark.parametrize("e", by_op("cell_interval") + by_op("children") + by_op("parent"), ids=lambda e: e["spec"])
def test_cell_navigation(e):
    from paper_2010_12548_b200.grid import CellId, cell_interval, children, parent

    c = CellId(*e["cell"])
    if e["op"] == "cell_interval":
        iv = cell_interval(c, e["L"])
        assert [iv.lo, iv.hi] == e["expect"]
    elif e["op"] == "children":
        assert [[k.level, k.code] for k in children(c)] == e["expect"]
        assert all(parent(k) == c for k in children(c))
    else:
        assert [parent(c).level, parent(c).code] == e["expect"]


def test_interval_prefix_property():
    """cell_interval(c) is the disjoint union of its children's."""
    from paper_2010_12548_b200.grid import CellId, cell_interval, children

    for level in range(0, 4):
        for code in range(1 << (2 * level)):
            c = CellId(level, code)
            ivs = [cell_interval(k, 6) for k in children(c)]
            iv = cell_interval(c, 6)
            assert ivs[0].lo == iv.lo and ivs[-1].hi == iv.hi
            assert all(a.hi == b.lo for a, b in zip(ivs, ivs[1:]))


@pytest.mark.parametrize("e", by_op("mbr_of"), ids=lambda e: e["spec"])
def test_mbr_of(e):
    from paper_2010_12548_b200.geometry import Polygon, mbr_of

    m = mbr_of(Polygon(e["outer"]))
    assert [m.min.x, m.min.y, m.max.x, m.max.y] == e["expect"]


@pytest.mark.parametrize("e", by_op("hausdorff_distance") + by_op("hausdorff_squares"), ids=lambda e: e["spec"])
def test_hausdorff_examples_hold(e):
    """The SPEC's Hausdorff examples, checked with an independent KD-tree oracle
    (the product's GPU version is checked in test_gpu_api.py)."""
    from scipy.spatial import cKDTree

    if e["op"] == "hausdorff_squares":
        def sq(a, b, step=1 / 400):
            g = np.arange(a, b + step / 2, step)
            X, Y = np.meshgrid(g, g)
            return np.stack([X.ravel(), Y.ravel()], 1)
        A, B = sq(*e["inner"]), sq(*e["outer"])
    else:
        A, B = np.asarray(e["A"], float), np.asarray(e["B"], float)
    h = max(cKDTree(B).query(A)[0].max(), cKDTree(A).query(B)[0].max())
    assert h == pytest.approx(e["expect"], abs=e.get("tol", 1e-12))


@pytest.mark.parametrize("e", by_op("result_range"), ids=lambda e: e["spec"])
def test_result_range(e):
    from paper_2010_12548_b200.query import AggregationQuery, RegionResult, result_range
    from paper_2010_12548_b200.raster import RasterMode

    q = AggregationQuery(e["agg"], 1.0, RasterMode[e["mode"]])
    r = result_range(RegionResult(0, e["alpha"], e["beta"]), q)
    assert (list(r) if r is not None else None) == e["expect"]


def test_range_unavailable_for_center_sampled_and_negative_sums():
    from paper_2010_12548_b200.query import AggregationQuery, RegionResult, result_range
    from paper_2010_12548_b200.raster import RasterMode

    assert result_range(RegionResult(0, 5, 1), AggregationQuery("COUNT", 1.0, RasterMode.CENTER_SAMPLED)) is None
    assert result_range(RegionResult(0, 5.0, 1.0), AggregationQuery("SUM:x", 1.0), nonnegative=False) is None
    assert result_range(RegionResult(0, 5.0, 1.0), AggregationQuery("SUM:x", 1.0)) == (4.0, 5.0)


def test_errors_hierarchy_matches_reference():
    """Same class names and base as /root/reference/pkg/src/rasterbound/errors.py:8-37."""
    from paper_2010_12548_b200 import errors as E

    names = ["GeometryError", "DomainError", "CapacityError", "ConfigError", "SchemaError", "ShapeError",
             "UnsupportedTransform"]
    for n in names:
        assert issubclass(getattr(E, n), E.RasterBoundError)
    import rasterbound.errors as RE

    assert RE.DomainError is E.DomainError


def test_agg_and_query_validation():
    from paper_2010_12548_b200.errors import ConfigError
    from paper_2010_12548_b200.query import Agg, AggregationQuery

    assert Agg.parse("sum:fare") == Agg("SUM", "fare")
    assert Agg.parse(("avg", "fare")) == Agg("AVG", "fare")
    assert str(Agg.parse("count")) == "COUNT"
    for bad in ("median", ("sum", None)):
        with pytest.raises(ConfigError):
            Agg.parse(bad)
    with pytest.raises(ConfigError):
        AggregationQuery("COUNT", -1.0)


def test_geometry_validation_and_packing():
    from paper_2010_12548_b200.errors import ConfigError, GeometryError
    from paper_2010_12548_b200.geometry import Point2D, Polygon, PointRecord, RegionRecord, as_point_set, pack_regions

    with pytest.raises(GeometryError):
        Polygon([(0, 0), (1, 1)])
    with pytest.raises(GeometryError):
        Polygon([(0, 0), (1, 1), (2, 2)])  # zero area
    with pytest.raises(GeometryError):
        Polygon([(0, 0), (1, float("nan")), (0, 1)])
    sq = Polygon([(0, 0), (1, 0), (1, 1), (0, 1), (0, 0)])  # explicit closing vertex dropped
    assert len(sq.outer) == 4
    p = pack_regions([RegionRecord(7, [sq, Polygon([(2, 2), (3, 2), (3, 3)], [])]), RegionRecord(3, sq)])
    assert p.region_ids.tolist() == [7, 3] and p.poly_region.tolist() == [0, 0, 1]
    assert p.ring_off.tolist() == [0, 4, 7, 11]
    with pytest.raises(ConfigError):
        pack_regions([RegionRecord(1, sq), RegionRecord(1, sq)])
    ps = as_point_set([PointRecord(Point2D(0.1, 0.2), {"fare": 3.0}), PointRecord(Point2D(0.3, 0.4), {"fare": 1.0})])
    assert ps.xy.shape == (2, 2) and ps.attrs["fare"].tolist() == [3.0, 1.0]


def test_workload_tilings_are_watertight():
    """C1/C2 generators: simple polygons whose areas sum to the tiled square."""
    from paper_2010_12548_b200 import workloads as W

    def area(a):
        return 0.5 * np.sum(a[:, 0] * np.roll(a[:, 1], -1) - np.roll(a[:, 0], -1) * a[:, 1])

    t = W.grid_tiling(0)
    assert len(t) == 100 and all(W.is_simple(r.geometry.outer) for r in t)
    assert sum(area(r.geometry.outer) for r in t) == pytest.approx(1.0, abs=1e-12)
    v = W.voronoi_tiling(40, 1000.0, seed=3, verts=(10, 30))
    assert len(v) == 40 and all(W.is_simple(r.geometry.outer) for r in v)
    assert sum(area(r.geometry.outer) for r in v) == pytest.approx(1e6, rel=1e-12)
    mx = W.make_mixture(1000.0, 0)
    a = W.mixture_points(10_000, mx, seed=1)
    b = W.mixture_points(10_000, mx, seed=1, threads=1)
    assert np.array_equal(a, b) and a.min() >= 0 and a.max() < 1000.0


def test_shard_ranges_partition():
    from paper_2010_12548_b200.shard import shard_range

    for n in (0, 1, 7, 1000):
        for world in (1, 2, 3, 8):
            rs = [shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))


def test_region_sets_beyond_the_owner_code_field_are_rejected():
    """Owner values carry ((region << 1) | boundary) + 1 in 18 bits: a region set of
    2^17 or more is a CapacityError before any device work."""
    from paper_2010_12548_b200 import _native as N

    lib = N.load()
    g = N.Grid(0.0, 0.0, 1.0, 8)
    for n_regions, want in ((1 << 17, N.RB_CAPACITY_ERROR if hasattr(N, "RB_CAPACITY_ERROR") else -3), (0, -3)):
        polys = N.Polygons(None, None, 0, None, 0, None, 0, None, n_regions)
        opts = N.BuildOpts(0, N.LAYOUT_TRIE, 8, -1, 0)
        h = ctypes.c_void_p()
        st = lib.rb_approx_build(ctypes.byref(g), ctypes.byref(polys), ctypes.byref(opts), None, ctypes.byref(h))
        assert st == want
        assert "n_regions" in lib.rb_last_error().decode()


def test_packed_layout_is_a_known_layout():
    from paper_2010_12548_b200 import _native as N
    from paper_2010_12548_b200.engine import LAYOUTS

    assert LAYOUTS == {"dense": 0, "trie": 1, "keys": 2, "packed": 3}
    hdr = open(os.path.join(ROOT, "include", "rasterbound_b200.h")).read()
    assert "#define RB_LAYOUT_PACKED 3" in hdr
    assert N.LAYOUT_PACKED == 3


def test_eps_grid_leaf_side_is_eps_over_sqrt2():
    """grid.eps_grid: side exactly eps/sqrt(2) and level_for_bound returns its level."""
    from paper_2010_12548_b200.grid import eps_grid, level_for_bound

    for eps, span in ((1.0, 100_000.0), (4.9, 40_000.0), (1e-3, 1.0), (0.5, 40_000.0)):
        g = eps_grid(0.0, 0.0, span, span, eps)
        assert math.ldexp(g.extent, -g.max_level) == eps / math.sqrt(2.0)
        assert g.extent >= 1.02 * span and g.extent / 2 < 1.02 * span
        assert level_for_bound(g, eps) == g.max_level
    assert eps_grid(0.0, 0.0, 100_000.0, 100_000.0, 1.0).max_level == 18


def test_integration_stub_structs_match_the_binding():
    """INTEGRATION.md section B's ctypes structs have the layout of the header's
    (as bound by _native.py); the block executes as written (library path filled in)."""
    import re

    from paper_2010_12548_b200 import _native as N

    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(.*?)```", text[text.index("## B."):], re.S).group(1)
    lib = os.path.join(ROOT, "paper_2010_12548_b200", "lib", "librasterbound_b200.so")
    ns = {}
    exec(compile(code.replace('C.CDLL("librasterbound_b200.so")', f"C.CDLL({lib!r})"), "INTEGRATION.md#B", "exec"), ns)
    for stub, ours in (("rb_grid", N.Grid), ("rb_polygons", N.Polygons), ("rb_build_opts", N.BuildOpts)):
        s = ns[stub]
        assert ctypes.sizeof(s) == ctypes.sizeof(ours), stub
        assert [f[0] for f in s._fields_] == [f[0] for f in ours._fields_], stub
        assert [getattr(s, f[0]).offset for f in s._fields_] == [getattr(ours, f[0]).offset for f in ours._fields_]
