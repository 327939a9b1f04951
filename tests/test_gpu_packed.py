"""RB_LAYOUT_PACKED (radix-table root over 16-byte palette blocks of 4x4
leaves; the C4 index): COUNT bit-exact and SUM within 1e-6 of the oracle
through the ring kernel (small region sets), the deep kernel (3000 regions,
hot and cold slots) and the generic kernel (misaligned inputs); act_lookup
identical to the radix table, escape blocks (> 3 owners in a block) included."""
import numpy as np
import pytest

from helpers import UNIT, adversarial_regions, oracle_approx, random_polygons
from test_gpu_parity import _assert_join, _gpu, _prepared

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("L,root_level", [(9, -1), (11, 5), (12, 10), (6, 0)])
def test_packed_overlapping_with_holes(oracle_lib, mode, L, root_level):
    """Overlapping holed polygons (owner lists; many blocks with > 3 distinct
    owner values -> escape blocks), ring kernel."""
    torch = _gpu()
    regions = random_polygons(5 + L, k=30, holes=True)
    rng = np.random.default_rng(L)
    xy = rng.random((300_001, 2))
    attr = rng.lognormal(2.5, 0.6, len(xy)).astype(np.float32)
    grid = UNIT.with_level(L)
    A, _ = oracle_approx(oracle_lib, regions, grid, mode)
    idx = _prepared(regions, grid, mode, "packed", root_level=root_level)
    st = idx.stats()
    assert st["root_level"] == (root_level if root_level >= 0 else (L - 6 if L >= 6 else 0))
    _assert_join(idx, A, xy, attr)
    _assert_join(idx, A, xy.astype(np.float32), None)
    trie = _prepared(regions, grid, mode, "trie")
    assert torch.equal(idx.lookup(xy[:100_000]), trie.lookup(xy[:100_000]))


def test_packed_adversarial(oracle_lib):
    _gpu()
    regions = adversarial_regions()
    rng = np.random.default_rng(3)
    g = np.arange(0, 64) / 64.0
    xy = np.concatenate([rng.random((50_000, 2)), np.stack(np.meshgrid(g, g), -1).reshape(-1, 2)])
    for L in (3, 6):
        grid = UNIT.with_level(L)
        for mode in (0, 1):
            A, _ = oracle_approx(oracle_lib, regions, grid, mode)
            idx = _prepared(regions, grid, mode, "packed", root_level=L - 2)
            _assert_join(idx, A, xy)


@pytest.mark.parametrize("hot", ["auto", "some"])
def test_packed_deep_kernel(oracle_lib, monkeypatch, hot):
    """3000 Voronoi regions (histogram beyond shared memory): k_point_pass_deep
    with the packed index, forced drains, out-of-window attributes, clustered
    points, trailing partial tile, f64 and f32."""
    _gpu()
    from paper_2010_12548_b200 import workloads as W

    monkeypatch.setenv("RB_FOLD", "2")
    regions = W.voronoi_tiling(3000, 1.0, seed=4, verts=(10, 30))
    rng = np.random.default_rng(12)
    n = 1_200_003
    cen = rng.random((12, 2))
    xy = np.clip(cen[rng.integers(0, 12, n)] + rng.normal(0, 0.05, (n, 2)), 0.0, 0.999999)
    attr = rng.lognormal(2.5, 0.6, n).astype(np.float32)
    k = rng.choice(n, 6000, replace=False)
    attr[k[:2000]] *= 1e-6
    attr[k[2000:4000]] = 0.0
    attr[k[4000:]] *= -1.0
    for L, rl in ((13, -1), (14, 7)):
        grid = UNIT.with_level(L)
        for mode in (0, 1):
            A, _ = oracle_approx(oracle_lib, regions, grid, mode)
            idx = _prepared(regions, grid, mode, "packed", root_level=rl)
            if hot == "some":
                idx.set_hot(np.arange(0, 3000, 7))
            _assert_join(idx, A, xy, attr)
            _assert_join(idx, A, xy.astype(np.float32), attr)
            _assert_join(idx, A, xy, None)


def test_packed_misaligned_generic_kernel(oracle_lib):
    """Inputs that are not 16-byte aligned take k_point_pass_global (index_lookup)."""
    torch = _gpu()
    regions = random_polygons(9, k=20, holes=True)
    grid = UNIT.with_level(10)
    rng = np.random.default_rng(1)
    buf = rng.random((200_001 * 2 + 1,))
    A, _ = oracle_approx(oracle_lib, regions, grid, 0)
    idx = _prepared(regions, grid, 0, "packed")
    t = torch.as_tensor(buf).cuda()
    xy = t[1:].view(-1, 2)  # 8-byte offset
    assert xy.data_ptr() % 16 == 8
    cnt_o, _ = A.join(buf[1:].reshape(-1, 2), None, nthreads=8)
    r = idx.point_pass(xy).check()
    np.testing.assert_array_equal(r.cnt.cpu().numpy(), cnt_o)


def test_packed_rejects_bad_root_level():
    _gpu()
    from paper_2010_12548_b200 import errors as E

    regions = random_polygons(2, k=3)
    with pytest.raises(E.ConfigError):
        _prepared(regions, UNIT.with_level(10), 0, "packed", root_level=9)
    with pytest.raises(E.ConfigError):
        _prepared(regions, UNIT.with_level(12), 0, "packed", root_level=2)
    # root slots are addressed with 32-bit indices in the point pass: root levels above 16 are refused
    # (fuzz_parity found wrong counts at root level 17 before this limit)
    with pytest.raises(E.CapacityError):
        _prepared(regions, UNIT.with_level(20), 0, "packed", root_level=17)
    with pytest.raises(E.CapacityError):
        _prepared(regions, UNIT.with_level(19), 0, "trie", root_level=17)
