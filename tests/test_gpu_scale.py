"""Parity at config scale (at scale the pinned oracle is the
reference).  A down-sized C4 -- all 40,000 regions, L = 18 on the
epsilon-matched grid, 20M float32-offset points, hot and cold regions -- through
the packed, radix-table and sorted-key indexes; and the C3 epsilon sweep on the
C2 inputs at 10M points through the uniform (dense) and hierarchical rasters.
COUNT alpha/beta bit-exact, SUM within rel 1e-6."""
import numpy as np
import pytest

from helpers import oracle_approx

pytestmark = pytest.mark.gpu

SUM_RTOL = 1e-6


def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def c4_small():
    from paper_2010_12548_b200 import workloads as W

    return W.c4(n=20_000_000)


@pytest.fixture(scope="module")
def c4_oracle(oracle_lib, c4_small):
    from paper_2010_12548_b200.grid import level_for_bound

    w = c4_small
    grid = w.grid.with_level(level_for_bound(w.grid, w.epsilon))
    A, _ = oracle_approx(oracle_lib, w.regions, grid, 0)
    cnt, sm = A.join(w.xy, w.attrs["fare"], nthreads=16)
    return grid, cnt, sm


@pytest.mark.timeout(1200)
@pytest.mark.parametrize("layout,root_level", [("packed", -1), ("packed", 12), ("trie", -1), ("trie", 12),
                                               ("keys", -1)])
def test_c4_downsized_all_regions(c4_small, c4_oracle, layout, root_level):
    torch = _gpu()
    from paper_2010_12548_b200.engine import ApproxIndex
    from paper_2010_12548_b200.geometry import pack_regions

    w = c4_small
    grid, cnt_o, sum_o = c4_oracle
    assert grid.max_level == 18 and len(w.regions) == 40_000 and w.xy.dtype == np.float32
    idx = ApproxIndex(pack_regions(w.regions), grid, 0, layout=layout, root_level=root_level)
    xy = torch.from_numpy(w.xy).cuda()
    fare = torch.from_numpy(w.attrs["fare"]).cuda()
    r = idx.point_pass(xy, fare).check()  # first pass picks the hot regions (auto_hot)
    st = idx.stats()
    assert 0 < st["n_hot"] < 40_000  # both privatised (hot) and global-RED (cold) regions are exercised
    np.testing.assert_array_equal(r.cnt.cpu().numpy(), cnt_o)
    np.testing.assert_allclose(r.sum.cpu().numpy(), sum_o, rtol=SUM_RTOL, atol=1e-9)
    r2 = idx.point_pass(xy, None).check()  # COUNT-only instantiation
    np.testing.assert_array_equal(r2.cnt.cpu().numpy(), cnt_o)


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("eps", [50.0, 10.0, 4.9, 1.0, 0.5])
def test_c3_epsilon_sweep_both_rasters(oracle_lib, eps):
    """C3: the C2 inputs at 10M points, each epsilon, uniform raster (dense leaf
    grid; beyond 4^16 leaves the packed index stands in, same leaf semantics,
    SPEC.md:248) and hierarchical raster (radix table)."""
    torch = _gpu()
    from paper_2010_12548_b200 import workloads as W
    from paper_2010_12548_b200.engine import ApproxIndex
    from paper_2010_12548_b200.geometry import pack_regions
    from paper_2010_12548_b200.grid import level_for_bound

    w = W.c2(n=10_000_000, eps=eps)
    grid = w.grid.with_level(level_for_bound(w.grid, w.epsilon))
    A, packed = oracle_approx(oracle_lib, w.regions, grid, 0)
    cnt_o, sum_o = A.join(w.xy, w.attrs["fare"], nthreads=16)
    xy = torch.from_numpy(w.xy).cuda()
    fare = torch.from_numpy(w.attrs["fare"]).cuda()
    uniform = "dense" if grid.max_level <= 16 else "packed"
    for layout in (uniform, "trie"):
        idx = ApproxIndex(packed, grid, 0, layout=layout)
        r = idx.point_pass(xy, fare).check()
        np.testing.assert_array_equal(r.cnt.cpu().numpy(), cnt_o, err_msg=f"{layout} eps={eps}")
        np.testing.assert_allclose(r.sum.cpu().numpy(), sum_o, rtol=SUM_RTOL, atol=1e-9)
        del idx
        torch.cuda.empty_cache()
