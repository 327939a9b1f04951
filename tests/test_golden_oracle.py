"""Pin the oracle (C tier ii and SPEC-literal tier i) on the reference's only
golden vectors: the SPEC.md `examples:` lines (tests/golden/spec_examples.json).
CPU only."""
import json
import math
import os

import numpy as np
import pytest

from oracle import spec_literal as SL

HERE = os.path.dirname(os.path.abspath(__file__))
EX = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))["examples"]


def by_op(op):
    return [e for e in EX if e["op"] == op]


def _unit_approx(O, rings_by_region, L, extent=1.0, mode=0):
    vx, vy, ring_off, pro, preg = [], [], [0], [0], []
    for r, rings in enumerate(rings_by_region):
        for ring in rings:
            a = np.asarray(ring, float)
            vx += list(a[:, 0]); vy += list(a[:, 1])
            ring_off.append(ring_off[-1] + len(a))
        pro.append(len(ring_off) - 1)
        preg.append(r)
    return O.Approx((0.0, 0.0, extent, L), np.array(vx), np.array(vy), ring_off, pro, preg, max(1, len(preg)), mode)


@pytest.mark.parametrize("e", by_op("level_for_bound"), ids=lambda e: e["spec"])
def test_level_for_bound(oracle_lib, e):
    assert oracle_lib.level_for_bound(e["extent"], e["epsilon"]) == e["expect"]
    assert SL.level_for_bound(e["extent"], e["epsilon"]) == e["expect"]


@pytest.mark.parametrize("e", by_op("z_encode"), ids=lambda e: e["spec"])
def test_z_encode(oracle_lib, e):
    assert oracle_lib.z_encode(e["ix"], e["iy"]) == e["expect"]
    assert SL.z_encode(e["ix"], e["iy"]) == e["expect"]


@pytest.mark.parametrize("e", by_op("point_to_cell"), ids=lambda e: e["spec"])
def test_point_to_cell(oracle_lib, e):
    ix, iy = oracle_lib.point_cells((e["origin"][0], e["origin"][1], e["extent"], e["level"]), np.array([e["p"]]))
    assert [e["level"], oracle_lib.z_encode(int(ix[0]), int(iy[0]))] == e["expect"]


@pytest.mark.parametrize("e", by_op("point_in_polygon"), ids=lambda e: e["spec"])
def test_pip(oracle_lib, e):
    rings = [e["outer"]] + e["holes"]
    vx = np.concatenate([np.asarray(r, float)[:, 0] for r in rings])
    vy = np.concatenate([np.asarray(r, float)[:, 1] for r in rings])
    off = np.cumsum([0] + [len(r) for r in rings])
    got = oracle_lib.pip(vx, vy, off, [e["p"][0]], [e["p"][1]])[0]
    assert bool(got) == e["expect"]
    assert SL.point_in_polygon(e["p"][0], e["p"][1], rings) == e["expect"]


@pytest.mark.parametrize("e", by_op("distance_to_boundary"), ids=lambda e: e["spec"])
def test_distance(oracle_lib, e):
    a = np.asarray(e["outer"], float)
    d = oracle_lib.distance(a[:, 0], a[:, 1], [0, len(a)], [e["p"][0]], [e["p"][1]])[0]
    assert d == pytest.approx(e["expect"], abs=1e-15)
    assert SL.distance_to_boundary(e["p"][0], e["p"][1], [e["outer"]]) == pytest.approx(e["expect"], abs=1e-15)


@pytest.mark.parametrize("e", by_op("classify_cell"), ids=lambda e: e["spec"])
def test_classify_cell(oracle_lib, e):
    lvl, code = e["cell"]
    # tier (i): top-down classify
    assert SL.classify_cell(lvl, code, [[tuple(v) for v in e["outer"]]], lvl) == e["expect"]
    # tier (ii): leaf classification at L = cell level (CONSERVATIVE: PARTIAL -> B)
    A = _unit_approx(oracle_lib, [[e["outer"]]], lvl)
    ix, iy = SL.z_decode(code)
    k = int(A.leaf_kinds(0, np.array([ix]), np.array([iy]))[0])
    assert {0: "OUTSIDE", 1: "INSIDE", 2: "PARTIAL"}[k] == e["expect"]


@pytest.mark.parametrize("e", by_op("rasterize_hierarchical") + by_op("rasterize_uniform"), ids=lambda e: e["spec"])
def test_rasterize(oracle_lib, e):
    L = oracle_lib.level_for_bound(e["extent"], e["epsilon"])
    A = _unit_approx(oracle_lib, [[e["outer"]]], L, e["extent"])
    lv, code, kind = A.hier_cells(0)
    cells = sorted(zip(lv.tolist(), code.tolist(), kind.tolist()))
    if e["op"] == "rasterize_uniform":  # expand interior cells to level L
        cells = sorted((L, (c << (2 * (L - l))) + t, k) for l, c, k in cells for t in range(1 << (2 * (L - l))))
    interior = [[l, c] for l, c, k in cells if k == 1]
    boundary = [[l, c] for l, c, k in cells if k == 2]
    assert interior == e["expect_interior"]
    assert boundary == e["expect_boundary"]
    # tier (i) agrees (hierarchical form)
    if e["op"] == "rasterize_hierarchical":
        side = math.ldexp(e["extent"], -L)
        g = SL.to_grid([e["outer"]], (0.0, 0.0), side)
        lit = sorted(SL.rasterize_hierarchical(g, L))
        assert [[l, c] for l, c, k in lit if k == "I"] == e["expect_interior"]
        assert [[l, c] for l, c, k in lit if k == "B"] == e["expect_boundary"]


@pytest.mark.parametrize("e", by_op("act_lookup"), ids=lambda e: e["spec"])
def test_act_lookup(oracle_lib, e):
    L = oracle_lib.level_for_bound(1.0, e["epsilon"])
    ids = sorted(int(k) for k in e["regions"])
    pts = np.asarray(e["points"], float)
    # tier (i): real radix trie
    trie, _ = SL.build([(i, [[e["regions"][str(i)]]]) for i in ids], (0.0, 0.0), 1.0, L)
    for p, exp in zip(e["points"], e["expect"]):
        ix, iy = math.floor(p[0] * (1 << L)), math.floor(p[1] * (1 << L))
        assert sorted(trie.lookup_code(SL.z_encode(ix, iy))) == sorted(tuple(x) for x in exp)
    if not ids:
        return
    A = _unit_approx(oracle_lib, [[e["regions"][str(i)]] for i in ids], L)
    off, reg, kind = A.lookup(pts)
    for k, exp in enumerate(e["expect"]):
        got = sorted((ids[int(r)], "I" if kd == 1 else "B") for r, kd in zip(reg[off[k]:off[k + 1]], kind[off[k]:off[k + 1]]))
        assert got == sorted(tuple(x) for x in exp)


@pytest.mark.parametrize("e", by_op("join_act"), ids=lambda e: e["spec"])
def test_join_act(oracle_lib, e):
    L = oracle_lib.level_for_bound(1.0, e["epsilon"])
    A = _unit_approx(oracle_lib, [[e["outer"]]], L)
    cnt, _ = A.join(np.asarray(e["points"], float))
    a, b = int(cnt[0, 0]), int(cnt[0, 1])
    assert (a, b) == (e["expect"]["alpha"], e["expect"]["beta"])
    assert [a - b, a] == e["expect"]["range"]
    trie, _ = SL.build([(0, [[e["outer"]]])], (0.0, 0.0), 1.0, L)
    res = SL.join_act(e["points"], trie, (0.0, 0.0), 1.0)
    assert res[0][:2] == [e["expect"]["alpha"], e["expect"]["beta"]]


def test_all_examples_covered():
    """Every golden example is exercised by a CPU test here, in test_host_api.py
    or in test_pointindex_oracle.py."""
    ops = {e["op"] for e in EX}
    covered = {"level_for_bound", "z_encode", "point_to_cell", "point_in_polygon", "distance_to_boundary",
               "classify_cell", "rasterize_hierarchical", "rasterize_uniform", "act_lookup", "join_act",
               "cell_interval", "children", "parent", "mbr_of", "result_range", "hausdorff_distance",
               "hausdorff_squares", "lps_build", "bounds_lookup", "range_aggregate"}
    assert ops <= covered
