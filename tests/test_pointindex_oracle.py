"""Pin the pointindex oracle (oracle/pointindex_oracle.py) on the SPEC.md
examples of lps_build / bounds_lookup / range_aggregate and on the SPEC's
properties (RadixSpline error audit, RS == binary search, prefix totals).  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import pointindex_oracle as PO

HERE = os.path.dirname(os.path.abspath(__file__))
EX = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))["examples"]


def by_op(op):
    return [e for e in EX if e["op"] == op]


@pytest.mark.parametrize("e", by_op("lps_build"), ids=lambda e: e["spec"])
def test_lps_build_examples(e):
    xy = np.asarray(e["points"], float).reshape(-1, 2)
    codes, perm, prefix = PO.lps_build(xy, (0.0, 0.0), 1.0, e["L"], {"w": np.ones(len(xy))})
    if "expect_codes" in e:
        assert codes.tolist() == e["expect_codes"]
    if "expect_count_prefix" in e:
        cnt = [int((codes < c).sum()) for c in range(len(e["expect_count_prefix"]))]
        assert cnt == e["expect_count_prefix"]
        assert prefix["w"][[0, 1, 3, 3, 6]].tolist() == [0, 1, 3, 3, 6]
    if "expect_prefix" in e:
        assert prefix["w"].tolist() == e["expect_prefix"]
    if e.get("expect_codes_equal_adjacent"):
        assert codes[0] == codes[1]
    assert sorted(perm.tolist()) == list(range(len(xy)))


@pytest.mark.parametrize("e", by_op("bounds_lookup"), ids=lambda e: e["spec"])
def test_bounds_lookup_examples(e):
    lo, hi = PO.bounds_lookup(np.asarray(e["codes"], np.uint64), [e["iv"][0]], [e["iv"][1]])
    assert [int(lo[0]), int(hi[0])] == e["expect"]


@pytest.mark.parametrize("e", by_op("range_aggregate"), ids=lambda e: e["spec"])
def test_range_aggregate_examples(e):
    got = PO.range_aggregate(np.asarray(e["codes"], np.uint64), None, [tuple(c) for c in e["cells"]])
    assert got == e["expect"]


@pytest.mark.parametrize("kind", ["uniform", "clustered", "duplicates"])
def test_spline_error_audit_and_bounds(kind):
    """interpolation error <= tau at every stored key; lookups
    through the spline window equal binary search."""
    rng = np.random.default_rng(3)
    if kind == "uniform":
        codes = np.sort(rng.integers(0, 1 << 40, 200_000).astype(np.uint64))
    elif kind == "clustered":
        c = rng.integers(0, 1 << 40, 30)
        codes = np.sort((c[rng.integers(0, 30, 200_000)] + rng.geometric(1e-4, 200_000)).astype(np.uint64))
    else:
        codes = np.sort(rng.integers(0, 5000, 200_000).astype(np.uint64))
    tau = 32
    keys, pos = PO.spline_fit(codes, tau - 0.5, width=40)
    assert np.all(np.diff(keys.astype(np.float64)) > 0)
    assert PO.spline_errors(codes, keys, pos).max() <= tau
    tab = PO.radix_table(keys, 12, 40)
    assert tab[0] == 0 and tab[-1] == len(keys) and np.all(np.diff(tab) >= 0)
    q = rng.integers(0, 1 << 40, 10_000).astype(np.uint64)
    lo, _ = PO.bounds_lookup(codes, q, q)
    est = np.interp(q.astype(np.float64), keys.astype(np.float64), pos.astype(np.float64))
    # fitted on the lower-bound CDF at and after every key: every integer query is within tau
    q[:2000] = codes[rng.integers(0, len(codes), 2000)]
    lo, _ = PO.bounds_lookup(codes, q, q)
    est = np.interp(q.astype(np.float64), keys.astype(np.float64), pos.astype(np.float64))
    assert np.all(np.abs(est - lo) <= tau + 1e-6)


def test_prefix_total_equals_whole_aggregate():
    rng = np.random.default_rng(1)
    xy = rng.random((50_000, 2))
    w = rng.lognormal(2.5, 0.6, len(xy))
    codes, perm, prefix = PO.lps_build(xy, (0.0, 0.0), 1.0, 12, {"w": w})
    assert np.all(np.diff(codes.astype(np.float64)) >= 0)
    np.testing.assert_allclose(prefix["w"][-1], w.sum(), rtol=1e-12)
    # range aggregate over the whole key space = n; over the 4 level-1 quadrants = n
    L = 12
    quads = [((q << (2 * (L - 1))), ((q + 1) << (2 * (L - 1)))) for q in range(4)]
    assert PO.range_aggregate(codes, None, quads) == len(xy)
