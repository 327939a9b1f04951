"""The point-pass kernels off the fast paths, each against the oracle (COUNT
bit-exact, SUM rel 1e-6): inputs not 16-byte aligned (no bulk copies:
k_point_pass / k_point_pass_global), grids above level 20 (beyond the
quantisation window of the ring kernels: k_point_pass_tma), and every kernel
family forced through RB_KERNEL in a fresh process (the selector is read once)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from helpers import UNIT, oracle_approx, random_polygons

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUM_RTOL = 1e-6


def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _index(regions, grid, mode=0):
    from paper_2010_12548_b200.engine import ApproxIndex
    from paper_2010_12548_b200.geometry import pack_regions

    return ApproxIndex(pack_regions(regions), grid, mode)


def _check(idx, A, xy, attr):
    cnt_o, sum_o = A.join(np.ascontiguousarray(xy.cpu().numpy() if hasattr(xy, "cpu") else xy),
                          None if attr is None else np.ascontiguousarray(
                              attr.cpu().numpy() if hasattr(attr, "cpu") else attr), nthreads=8)
    r = idx.point_pass(xy, attr).check()
    np.testing.assert_array_equal(r.cnt.cpu().numpy(), cnt_o)
    if attr is not None:
        np.testing.assert_allclose(r.sum.cpu().numpy(), sum_o, rtol=SUM_RTOL, atol=1e-9)


@pytest.mark.parametrize("nreg", [20, 3000])
def test_misaligned_inputs(oracle_lib, nreg):
    """Device views offset by one element: f32 coordinates at 8 mod 16 bytes and
    the attribute at 4 mod 16 -- no bulk copies; shared (20 regions) and global
    (3000 regions) histograms."""
    torch = _gpu()
    from paper_2010_12548_b200 import workloads as W

    regions = random_polygons(3, 20) if nreg == 20 else W.voronoi_tiling(3000, 1.0, seed=4, verts=(10, 30))
    grid = UNIT.with_level(12)
    rng = np.random.default_rng(1)
    xy = torch.from_numpy(rng.random((400_001, 2)).astype(np.float32)).cuda()[1:]
    at = torch.from_numpy(rng.lognormal(2.5, 0.6, 400_001).astype(np.float32)).cuda()[1:]
    assert xy.data_ptr() % 16 == 8 and at.data_ptr() % 16 == 4
    A, _ = oracle_approx(oracle_lib, regions, grid, 0)
    idx = _index(regions, grid)
    _check(idx, A, xy, at)
    _check(idx, A, xy, None)


@pytest.mark.parametrize("mode", [0, 1])
def test_level_above_20(oracle_lib, mode):
    """L = 21 (cells of 2^-21): beyond the 2^20 quantisation window of the ring
    kernels, so the pass runs k_point_pass_tma with the exact division."""
    torch = _gpu()
    regions = random_polygons(5, 6)
    grid = UNIT.with_level(21)
    rng = np.random.default_rng(2)
    xy = rng.random((300_003, 2))
    at = rng.lognormal(2.5, 0.6, len(xy)).astype(np.float32)
    A, _ = oracle_approx(oracle_lib, regions, grid, mode)
    idx = _index(regions, grid, mode)
    _check(idx, A, xy, at)
    _check(idx, A, torch.from_numpy(xy.astype(np.float32)).cuda(), None)


_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from helpers import UNIT, oracle_approx, random_polygons
from oracle import oracle as O
from paper_2010_12548_b200 import workloads as W
from paper_2010_12548_b200.engine import ApproxIndex
from paper_2010_12548_b200.geometry import pack_regions
O.build_lib()
rng = np.random.default_rng(4)
for regions, L in ((random_polygons(7, 30, holes=True), 12), (W.voronoi_tiling(3000, 1.0, seed=4, verts=(10, 30)), 13)):
    grid = UNIT.with_level(L)
    xy = rng.random((500_003, 2))
    at = rng.lognormal(2.5, 0.6, len(xy)).astype(np.float32)
    at[:1000] *= 1e-7
    A, _ = oracle_approx(O, regions, grid, 0)
    idx = ApproxIndex(pack_regions(regions), grid, 0)
    for pts, a in ((xy, at), (xy.astype(np.float32), None)):
        cnt_o, sum_o = A.join(pts, a, nthreads=8)
        r = idx.point_pass(pts, a).check()
        np.testing.assert_array_equal(r.cnt.cpu().numpy(), cnt_o)
        if a is not None:
            np.testing.assert_allclose(r.sum.cpu().numpy(), sum_o, rtol=1e-6, atol=1e-9)
print("ok")
"""


@pytest.mark.parametrize("kernel", ["0", "3", "4"])
def test_forced_kernel_families(kernel):
    """RB_KERNEL=0: no bulk copies (k_point_pass / k_point_pass_global);
    3: k_point_pass_tma for every region-set size; 4: everything but the deep
    ring kernel.  Random overlapping polygons with holes and a 3000-region
    tiling, f64 + attribute and f32 COUNT."""
    _gpu()
    env = dict(os.environ, RB_KERNEL=kernel)
    code = _SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0 and p.stdout.strip().endswith("ok"), p.stdout[-2000:] + p.stderr[-4000:]
