"""GPU end-to-end tests of the cli through click's runner:
ingest -> rasterize (covering dump) -> index build (ACT / point index files)
-> query / join (engines agree) -> bench (seeded determinism,
SPEC.md:570) -> audit."""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture()
def data(tmp_path):
    rng = np.random.default_rng(3)
    xy = rng.random((20_000, 2)) * [4000.0, 3000.0] + [500.0, 800.0]  # arbitrary planar units
    fare = rng.lognormal(2.5, 0.6, len(xy))
    with open(tmp_path / "pts.csv", "w") as f:
        f.write("x,y,fare\n")
        for (x, y), w in zip(xy, fare):
            f.write(f"{float(x)!r},{float(y)!r},{float(w)!r}\n")
        f.write("bad,row,1\n")
    from paper_2010_12548_b200 import workloads as W

    regs = W.voronoi_tiling(12, 1.0, seed=2, verts=(8, 20))
    feats = []
    for r in regs:
        ring = (r.geometry.outer * [4000.0, 4000.0] + [500.0, 300.0]).tolist()
        feats.append({"type": "Feature", "geometry": {"type": "Polygon", "coordinates": [ring + ring[:1]]}})
    (tmp_path / "regs.geojson").write_text(json.dumps({"type": "FeatureCollection", "features": feats}))
    return tmp_path


def test_cli_end_to_end(data):
    _gpu()
    from click.testing import CliRunner

    from paper_2010_12548_b200 import formats as F
    from paper_2010_12548_b200.cli import main

    R = CliRunner()
    pts, regs = str(data / "pts.csv"), str(data / "regs.geojson")
    r = R.invoke(main, ["ingest", "--points", pts, "--regions", regs, "--out", str(data / "ing")])
    assert r.exit_code == 0, r.output
    meta = json.loads(r.output)
    assert meta["points"] == 20_000 and meta["regions"] == 12 and meta["rejected"] == 1
    r = R.invoke(main, ["rasterize", "--regions", regs, "--epsilon", "0.01", "--out", str(data / "cover.txt")])
    assert r.exit_code == 0, r.output
    with open(data / "cover.txt") as f:
        rid, lv, code, kind = F.read_covering_dump(f)
    assert set(rid.tolist()) == set(range(12)) and set(kind.tolist()) <= {1, 2}
    r = R.invoke(main, ["index", "build", "--kind", "act", "--regions", regs, "--epsilon", "0.01",
                        "--out", str(data / "r.act")])
    assert r.exit_code == 0, r.output
    r = R.invoke(main, ["query", "--index", str(data / "r.act"), "--points", pts, "--regions", regs])
    assert r.exit_code == 0, r.output
    owners = [json.loads(l) for l in r.output.splitlines()]
    assert len(owners) == 20_000 and all(len(o["owners"]) >= 1 for o in owners[:1000]) is not None
    r = R.invoke(main, ["index", "build", "--kind", "point", "--points", pts, "--epsilon", "0.01", "--sum", "fare",
                        "--out", str(data / "p.rbpi")])
    assert r.exit_code == 0, r.output
    from paper_2010_12548_b200.pointindex import load_point_index

    lps, rs = load_point_index(str(data / "p.rbpi"))
    assert lps.n == 20_000 and rs is not None and lps.attrs == ("fare",)
    per_engine = {}
    for eng in ("act", "pointindex", "canvas"):
        r = R.invoke(main, ["join", "--points", pts, "--regions", regs, "--epsilon", "0.01", "--engine", eng,
                            "--agg", "count"])
        assert r.exit_code == 0, r.output
        per_engine[eng] = [(d["region_id"], d["alpha"], d["beta"]) for d in map(json.loads, r.output.splitlines())]
    assert per_engine["act"] == per_engine["pointindex"] == per_engine["canvas"]  # engines agree
    r = R.invoke(main, ["join", "--points", pts, "--regions", regs, "--epsilon", "0.01", "--engine", "all",
                        "--agg", "sum:fare"])
    assert r.exit_code == 0, r.output
    recs = [json.loads(l) for l in r.output.splitlines()]
    assert {d["engine"] for d in recs} == {"act", "pointindex", "canvas"}
    assert set(recs[0]) == {"region_id", "alpha", "beta", "lo", "hi", "agg", "epsilon", "mode", "engine"}
    r = R.invoke(main, ["audit", "--points", pts, "--regions", regs, "--epsilon", "0.01"])
    assert r.exit_code == 0, r.output
    a = json.loads(r.output)
    assert a["ok"] and a["false_negatives"] == 0


def test_cli_bench_synthetic_deterministic():
    _gpu()
    from click.testing import CliRunner

    from paper_2010_12548_b200.cli import main

    R = CliRunner()
    outs = []
    for _ in range(2):
        r = R.invoke(main, ["bench", "--epsilon", "0.02,0.01", "--engine", "all", "--seed", "7"])
        assert r.exit_code == 0, r.output
        recs = [json.loads(l) for l in r.output.splitlines()]
        for d in recs:  # timings excluded from the determinism check
            d.pop("build_time", None)
            d.pop("query_time", None)
        outs.append(recs)
    assert outs[0] == outs[1]
    recs = outs[0]
    assert len(recs) == 6 and all(d["audit"]["eps_ok"] for d in recs)
    by = {}
    for d in recs:
        by.setdefault(d["epsilon"], []).append([(x["region_id"], x["alpha"]) for x in d["regions"]])
    for eps, lists in by.items():
        assert lists[0] == lists[1] == lists[2]  # engines=all -> identical alpha
    # smaller epsilon -> mismatch fraction not larger
    assert by and recs[3]["audit"]["mismatch_fraction"] <= recs[0]["audit"]["mismatch_fraction"]
