"""The ctypes binding INTEGRATION.md section B shows a reference maintainer
(the code block itself, executed as written with only the library path
filled in): build an approximation and run the point pass through the
C-ABI, COUNT bit-exact and SUM within rel 1e-6 against the oracle, and the
DomainError path."""
import os
import re

import numpy as np
import pytest

from helpers import oracle_approx

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stub():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = text[text.index("## B."):]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    lib = os.path.join(ROOT, "paper_2010_12548_b200", "lib", "librasterbound_b200.so")
    code = code.replace('C.CDLL("librasterbound_b200.so")', f'C.CDLL({lib!r})')
    ns = {}
    exec(compile(code, "INTEGRATION.md#B", "exec"), ns)
    return ns


def test_integration_stub_join(oracle_lib):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2010_12548_b200 import workloads as W
    from paper_2010_12548_b200.geometry import pack_regions

    ns = _stub()
    from paper_2010_12548_b200.grid import level_for_bound

    w = W.c1(n=200_000)
    p = pack_regions(w.regions)
    grid = w.grid.with_level(level_for_bound(w.grid, w.epsilon))
    g = ns["rb_grid"](grid.origin.x, grid.origin.y, grid.extent, grid.max_level)
    dev = [torch.from_numpy(a).cuda() for a in (p.vx, p.vy, p.ring_off, p.poly_ring_off, p.poly_region)]
    h = ns["build"](g, *dev, p.n_regions, mode=0)
    rng = np.random.default_rng(1)
    xy = np.ascontiguousarray(w.xy, dtype=np.float64)
    fare = rng.lognormal(2.5, 0.6, len(xy)).astype(np.float32)
    cnt, sm = ns["point_pass"](h, torch.from_numpy(xy).cuda(), torch.from_numpy(fare).cuda(), p.n_regions)
    torch.cuda.synchronize()
    A, _ = oracle_approx(oracle_lib, p, grid, 0)
    cnt_o, sum_o = A.join(xy, fare, nthreads=4)
    np.testing.assert_array_equal(cnt.cpu().numpy(), cnt_o)
    np.testing.assert_allclose(sm.cpu().numpy(), sum_o, rtol=1e-6, atol=1e-9)
    bad = xy.copy()
    bad[123] = (grid.origin.x + 2 * grid.extent, 0.5)
    import rasterbound.errors as E

    with pytest.raises(E.DomainError):
        ns["point_pass"](h, torch.from_numpy(bad).cuda(), None, p.n_regions)
    ns["lib"].rb_approx_free(h)
