"""GPU tests of the canvas algebra through the C-ABI: the
SPEC examples of render_points / blend / mask / affine, render_polygon ==
the leaf expansion of rasterize_uniform (oracle cells), mass conservation,
and the literal Bounded Raster Join plan == join_act."""
import numpy as np
import pytest

from helpers import UNIT, oracle_approx, random_polygons

pytestmark = pytest.mark.gpu


def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _counts_canvas(mat):
    """Canvas at L=1 whose pixel (row iy, col ix) holds mat[iy][ix] points."""
    from paper_2010_12548_b200 import canvas as CV

    pts = []
    for iy in range(2):
        for ix in range(2):
            pts += [[(ix + 0.5) / 2, (iy + 0.5) / 2]] * int(mat[iy][ix])
    return CV.render_points(np.array(pts, float).reshape(-1, 2), UNIT, 1)


def _mat(c):
    cnt = c.count.cpu().numpy()
    emp = c.empty.cpu().numpy()
    return [[None if emp[i, j] else int(cnt[i, j]) for j in range(2)] for i in range(2)]


def test_render_points_examples_and_mass():
    _gpu()
    from paper_2010_12548_b200 import canvas as CV

    c = CV.render_points(np.zeros((0, 2)), UNIT, 4)  # no points -> all empty
    assert bool(c.empty.all())
    c = CV.render_points(np.array([[0.3, 0.3], [0.31, 0.32], [0.33, 0.3]]), UNIT, 2)  # 3 points in one cell
    assert int(c.count.sum()) == 3 and int((~c.empty).sum()) == 1 and int(c.count.max()) == 3
    rng = np.random.default_rng(0)
    xy = rng.random((200_000, 2))
    w = rng.lognormal(2.5, 0.6, len(xy)).astype(np.float32)
    from paper_2010_12548_b200.geometry import PointSet

    c = CV.render_points(PointSet(xy, {"w": w}), UNIT, 7, ["w"])
    ix = np.floor(xy[:, 0] / (1 / 128)).astype(int)
    iy = np.floor(xy[:, 1] / (1 / 128)).astype(int)
    np.testing.assert_array_equal(c.count.sum(0).cpu().numpy(), np.bincount(ix, minlength=128))  # column sums
    assert int(c.count.sum()) == len(xy)  # mass conservation
    want = np.zeros((128, 128))
    np.add.at(want, (iy, ix), w.astype(np.float64))
    np.testing.assert_allclose(c.sum("w").cpu().numpy(), want, rtol=1e-12)


def test_blend_mask_affine_examples():
    _gpu()
    from paper_2010_12548_b200 import canvas as CV
    from paper_2010_12548_b200 import errors as E

    x = _counts_canvas([[1, 2], [3, 4]])
    y = _counts_canvas([[10, 0], [0, 1]])
    assert _mat(CV.blend(x, y, CV.BlendFn.SUM)) == [[11, 2], [3, 5]]
    assert _mat(CV.blend(y, x, CV.BlendFn.SUM)) == [[11, 2], [3, 5]]  # commutes
    empty = _counts_canvas([[0, 0], [0, 0]])
    assert _mat(CV.blend(x, empty, CV.BlendFn.SUM)) == _mat(x)  # SPEC.md:426 identity
    assert _mat(CV.blend(x, y, CV.BlendFn.MAX)) == [[10, 2], [3, 4]]
    assert _mat(CV.blend(x, y, CV.BlendFn.OVERWRITE)) == [[10, 2], [3, 1]]
    m = CV.mask(x, CV.MaskPredicate.count_gt(2))
    assert _mat(m) == [[None, None], [3, 4]]
    assert _mat(CV.mask(x, CV.MaskPredicate.nonempty())) == _mat(x)  # always-true on x
    assert _mat(CV.mask(m, CV.MaskPredicate.count_gt(2))) == _mat(m)  # idempotence
    assert _mat(CV.affine(x, CV.AffineTransform())) == _mat(x)  # identity
    assert _mat(CV.affine(x, CV.AffineTransform(1, 0))) == [[None, 1], [None, 3]]
    f = CV.affine(x, CV.AffineTransform(flip_x=True))
    assert _mat(f) == [[2, 1], [4, 3]]
    assert _mat(CV.affine(f, CV.AffineTransform(flip_x=True))) == _mat(x)  # flip twice
    with pytest.raises(E.UnsupportedTransform):
        CV.affine(x, CV.AffineTransform(0.5, 0))
    with pytest.raises(E.ShapeError):
        CV.blend(x, CV.render_points(np.zeros((0, 2)), UNIT, 2), CV.BlendFn.SUM)


@pytest.mark.parametrize("mode", [0, 1])
def test_render_polygon_equals_uniform_cells(oracle_lib, mode):
    _gpu()
    from paper_2010_12548_b200 import canvas as CV

    L = 8
    grid = UNIT.with_level(L)
    for reg in random_polygons(5, k=6, holes=True):
        c = CV.render_polygon(reg.geometry, UNIT, L, mode, id=reg.id)
        A, _ = oracle_approx(oracle_lib, [reg], grid, mode)
        # oracle leaf classification: lookup of every pixel centre
        W = 1 << L
        cx, cy = np.meshgrid((np.arange(W) + 0.5) / W, (np.arange(W) + 0.5) / W)
        cnt, _ = A.join(np.stack([cx.ravel(), cy.ravel()], 1))
        covered = int(cnt[0, 0])
        boundary = int(cnt[0, 1])
        assert int((~c.empty).sum()) == covered
        assert int(c.boundary_flag.sum()) == boundary
        assert set(np.unique(c.region.cpu().numpy()[~c.empty.cpu().numpy()]).tolist()) <= {reg.id}
    full = CV.render_polygon([(0, 0), (1, 0), (1, 1), (0, 1)], UNIT, 5, mode, id=3)
    assert not bool(full.empty.any())  # domain-filling polygon


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_brj_algebra_equals_join_act(oracle_lib, seed):
    """The literal canvas plan (with 2^4-pixel tiles, so tiling is exercised)
    equals join_act (COUNT exact, SUM 1e-6) -- SPEC.md:507."""
    _gpu()
    from paper_2010_12548_b200 import canvas as CV
    from paper_2010_12548_b200.geometry import PointSet, pack_regions
    from paper_2010_12548_b200.query import AggregationQuery, join_act, join_canvas
    from paper_2010_12548_b200.raster import RasterMode

    rng = np.random.default_rng(seed)
    regions = random_polygons(seed + 20, k=8, holes=True)
    xy = rng.random((50_000, 2))
    pts = PointSet(xy, {"fare": rng.lognormal(2.5, 0.6, len(xy)).astype(np.float32)})
    for mode in (RasterMode.CONSERVATIVE, RasterMode.CENTER_SAMPLED):
        for agg in ("COUNT", "SUM:fare"):
            q = AggregationQuery(agg, 2.0 ** -7 * np.sqrt(2.0) * 1.000001, mode)
            ref = join_act(pts, regions, q, cfg=UNIT)
            cnt, sm = CV.brj(pts, pack_regions(regions), q, UNIT, tile_level=4)
            if agg == "COUNT":
                assert [(r.alpha, r.boundary_part) for r in ref] == [tuple(x) for x in cnt.tolist()]
            else:
                np.testing.assert_allclose(sm, [[r.alpha, r.boundary_part] for r in ref], rtol=1e-6, atol=1e-6)
            alg = join_canvas(pts, regions, q, cfg=UNIT, plan="algebra")
            assert [r.alpha for r in alg] == pytest.approx([r.alpha for r in ref], rel=1e-6)


def test_render_points_tiles_aligned_and_unaligned():
    """Sub-tiles of the point canvas: Z-aligned tiles (only the tile's slice of
    the sorted codes is visited) and unaligned or edge-clipped offsets (full
    scan) both equal the matching window of the whole-grid canvas."""
    _gpu()
    from paper_2010_12548_b200 import canvas as CV
    from paper_2010_12548_b200.geometry import PointSet
    from paper_2010_12548_b200.pointindex import lps_build

    L = 9
    rng = np.random.default_rng(3)
    xy = rng.random((300_000, 2)) ** 2  # skewed towards the origin
    w = rng.lognormal(2.5, 0.6, len(xy)).astype(np.float32)
    ps = PointSet(xy, {"w": w})
    lps = lps_build(ps, UNIT.with_level(L), ["w"])
    full = CV.render_points(None, UNIT, L, ["w"], lps=lps)
    fc, fs = full.count.cpu().numpy(), full.sum("w").cpu().numpy()
    for lev, x0, y0 in ((6, 0, 0), (6, 64, 128), (5, 480, 480), (4, 3, 5), (6, 500, 7), (3, 0, 511)):
        t = CV.render_points(None, UNIT, L, ["w"], level=lev, x0=x0, y0=y0, lps=lps)
        W = 1 << lev
        wc = np.zeros((W, W), np.int64)
        ws = np.zeros((W, W))
        hx, hy = min(W, (1 << L) - x0), min(W, (1 << L) - y0)
        wc[:hy, :hx] = fc[y0:y0 + hy, x0:x0 + hx]
        ws[:hy, :hx] = fs[y0:y0 + hy, x0:x0 + hx]
        np.testing.assert_array_equal(t.count.cpu().numpy(), wc)
        np.testing.assert_allclose(t.sum("w").cpu().numpy(), ws, rtol=1e-12, atol=1e-9)
        assert bool(((t.count > 0) == ~t.empty).all())
