"""The largest region set the owner-code field holds: 131,071
regions = 2^17 - 1 (codes ((region << 1) | boundary) + 1 need 18 bits; the hot
annotation sits above them, 4095 slots).  A 362 x 362 jittered quad tiling plus
27 small overlapping diamonds (owner lists), 2M uniform and clustered points,
through the radix table (deep kernel: hot and cold regions), the packed and the
sorted-key layouts: COUNT bit-exact against the oracle, SUM within rel 1e-6,
act_lookup identical to the oracle's owner sets.  One region more is rejected
(tests/test_host_api.py)."""
import numpy as np
import pytest

from helpers import UNIT, oracle_approx

pytestmark = pytest.mark.gpu

N_MAX = (1 << 17) - 1


def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _max_regions():
    from paper_2010_12548_b200.geometry import PackedRegions

    g = 362
    rng = np.random.default_rng(17)
    h = 1.0 / g
    cx = np.linspace(0.0, 1.0, g + 1)
    X, Y = np.meshgrid(cx, cx)
    J = rng.uniform(-0.3 * h, 0.3 * h, (2, g + 1, g + 1))
    J[0][:, [0, g]] = 0.0
    J[1][[0, g], :] = 0.0
    X, Y = X + J[0], Y + J[1]
    j, i = np.divmod(np.arange(g * g), g)
    quad_x = np.stack([X[j, i], X[j, i + 1], X[j + 1, i + 1], X[j + 1, i]], 1)  # CCW
    quad_y = np.stack([Y[j, i], Y[j, i + 1], Y[j + 1, i + 1], Y[j + 1, i]], 1)
    extra = N_MAX - g * g
    c = rng.uniform(0.1, 0.9, (extra, 2))
    r = rng.uniform(0.5, 3.0, extra) * h
    dia_x = np.stack([c[:, 0], c[:, 0] + r, c[:, 0], c[:, 0] - r], 1)
    dia_y = np.stack([c[:, 1] - r, c[:, 1], c[:, 1] + r, c[:, 1]], 1)
    vx = np.concatenate([quad_x, dia_x]).ravel()
    vy = np.concatenate([quad_y, dia_y]).ravel()
    n = g * g + extra
    return PackedRegions(np.ascontiguousarray(vx), np.ascontiguousarray(vy), np.arange(n + 1, dtype=np.int64) * 4,
                         np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), np.arange(n, dtype=np.int64))


@pytest.mark.timeout(1200)
def test_largest_region_set_all_layouts(oracle_lib):
    torch = _gpu()
    from paper_2010_12548_b200.engine import ApproxIndex

    packed = _max_regions()
    assert packed.n_regions == N_MAX
    grid = UNIT.with_level(12)
    rng = np.random.default_rng(3)
    n = 2_000_001
    cen = rng.random((8, 2))
    xy = np.concatenate([rng.random((n // 2, 2)),
                         np.clip(cen[rng.integers(0, 8, n - n // 2)] + rng.normal(0, 0.03, (n - n // 2, 2)), 0, 0.999999)])
    attr = rng.lognormal(2.5, 0.6, n).astype(np.float32)
    A, _ = oracle_approx(oracle_lib, packed, grid, 0)
    cnt_o, sum_o = A.join(xy, attr, nthreads=16)
    assert (cnt_o[:, 0] > 0).sum() > 100_000
    sample = np.concatenate([xy[:10_000], xy[-10_000:]])
    off, reg, kind = A.lookup(sample)
    own_o = [sorted((int(g), 1 if kd == 2 else 0) for g, kd in zip(reg[off[k]:off[k + 1]], kind[off[k]:off[k + 1]]))
             for k in range(len(sample))]
    assert any(len(o) > 1 for o in own_o)  # owner lists (diamonds over quads) are exercised
    for layout in ("trie", "packed", "keys"):
        idx = ApproxIndex(packed, grid, 0, layout=layout)
        st = idx.stats()
        assert st["max_hot"] == 4095
        r = idx.point_pass(xy, attr).check()  # picks hot regions on the first pass (cold ones take global REDs)
        np.testing.assert_array_equal(r.cnt.cpu().numpy(), cnt_o, err_msg=layout)
        np.testing.assert_allclose(r.sum.cpu().numpy(), sum_o, rtol=1e-6, atol=1e-9, err_msg=layout)
        if layout == "trie":
            assert 0 < idx.stats()["n_hot"] <= 4095
        r2 = idx.point_pass(xy, attr).check()  # hot slots in place
        np.testing.assert_array_equal(r2.cnt.cpu().numpy(), cnt_o, err_msg=layout)
        got = idx.decode(idx.lookup(sample))
        bad = [k for k in range(len(sample)) if sorted(got[k]) != own_o[k]]
        assert not bad, (layout, bad[:5])
        del idx
        torch.cuda.empty_cache()
