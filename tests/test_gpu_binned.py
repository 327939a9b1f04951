"""The partitioned point pass (csrc/rb_binned.cuh, RB_BINNED=1; an opt-in
experiment, slower than the one-pass deep kernel on C4): pass 1 groups the
points by a coarse cell into chunks, pass 2 joins each cell's chunks against
its slice of the root table.  Same index and quantisation as the one-pass
kernels, so COUNT (alpha, beta) is bit-exact against the oracle and SUM within
rel 1e-6; repeated runs agree (the chunk order is not deterministic, the
result must be)."""
import numpy as np
import pytest

from helpers import UNIT, oracle_approx

pytestmark = pytest.mark.gpu

SUM_RTOL = 1e-6


def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _index(regions, grid, mode=0, root_level=-1):
    from paper_2010_12548_b200.engine import ApproxIndex
    from paper_2010_12548_b200.geometry import pack_regions

    return ApproxIndex(pack_regions(regions), grid, mode, layout="trie", root_level=root_level)


@pytest.mark.timeout(900)
@pytest.mark.parametrize("root_level", [-1, 8, 4])
def test_binned_pass_equals_oracle(oracle_lib, monkeypatch, root_level):
    """3000 regions on L = 13 (bins at root level - 6, or the whole root for
    low roots), clustered points with a trailing partial tile, f64 and f32
    points, COUNT-only, zero / tiny / negative attributes, both modes."""
    _gpu()
    from paper_2010_12548_b200 import workloads as W

    monkeypatch.setenv("RB_BINNED", "1")
    regions = W.voronoi_tiling(3000, 1.0, seed=4, verts=(10, 30))
    grid = UNIT.with_level(13)
    rng = np.random.default_rng(5)
    n = 1_200_007
    cen = rng.random((12, 2))
    xy = np.clip(cen[rng.integers(0, 12, n)] + rng.normal(0, 0.05, (n, 2)), 0.0, 0.999999)
    attr = rng.lognormal(2.5, 0.6, n).astype(np.float32)
    k = rng.choice(n, 6000, replace=False)
    attr[k[:2000]] *= 1e-6
    attr[k[2000:4000]] = 0.0
    attr[k[4000:]] *= -1.0
    for mode in (0, 1):
        A, _ = oracle_approx(oracle_lib, regions, grid, mode)
        idx = _index(regions, grid, mode, root_level)
        for pts in (xy.astype(np.float32), xy):  # f32 points quantise as their f64 promotion
            cnt_o, sum_o = A.join(pts, attr, nthreads=8)
            for _ in range(2):
                r = idx.point_pass(pts, attr).check()
                np.testing.assert_array_equal(r.cnt.cpu().numpy(), cnt_o)
                np.testing.assert_allclose(r.sum.cpu().numpy(), sum_o, rtol=SUM_RTOL, atol=1e-9)
        r = idx.point_pass(xy, None).check()
        np.testing.assert_array_equal(r.cnt.cpu().numpy(), cnt_o)


@pytest.mark.parametrize("n", [1, 5, 4095, 4097])
def test_binned_pass_small_batches(oracle_lib, monkeypatch, n):
    _gpu()
    from paper_2010_12548_b200 import workloads as W

    monkeypatch.setenv("RB_BINNED", "1")
    regions = W.voronoi_tiling(300, 1.0, seed=2, verts=(6, 12))
    grid = UNIT.with_level(12)
    rng = np.random.default_rng(n)
    xy = rng.random((n, 2))
    attr = rng.random(n).astype(np.float32)
    A, _ = oracle_approx(oracle_lib, regions, grid, 0)
    cnt_o, sum_o = A.join(xy, attr, nthreads=4)
    r = _index(regions, grid).point_pass(xy, attr).check()
    np.testing.assert_array_equal(r.cnt.cpu().numpy(), cnt_o)
    np.testing.assert_allclose(r.sum.cpu().numpy(), sum_o, rtol=SUM_RTOL, atol=1e-9)


def test_binned_pass_domain_error(monkeypatch):
    _gpu()
    from paper_2010_12548_b200 import errors as E
    from paper_2010_12548_b200 import workloads as W

    monkeypatch.setenv("RB_BINNED", "1")
    idx = _index(W.voronoi_tiling(300, 1.0, seed=2, verts=(6, 12)), UNIT.with_level(12))
    xy = np.random.default_rng(0).random((100_000, 2))
    xy[70_000] = (1.5, 0.2)
    xy[30_000] = (np.nan, 0.5)
    with pytest.raises(E.DomainError) as ei:
        idx.point_pass(xy).check()
    assert ei.value.index == 30_000
