"""CPU tests of the ingest / file-format layer (SPEC.md:553-561 examples,
:185 CellId, :258 covering dump, :306 ACT file header)."""
import io
import json

import numpy as np
import pytest

from paper_2010_12548_b200 import errors as E
from paper_2010_12548_b200 import formats as F


def test_points_csv_one_point_and_rejects():
    xy, attrs, rej = F.read_points_csv("x,y,fare\n10,20,3.5\n")  # SPEC.md:559 1-point CSV
    assert xy.tolist() == [[10.0, 20.0]] and attrs["fare"].tolist() == [3.5] and rej == []
    xy, attrs, rej = F.read_points_csv("lon,lat\n1,2\nfoo,3\n4,5\n\n6,nan\n", "lon", "lat")
    assert xy.tolist() == [[1, 2], [4, 5]]
    assert [r[0] for r in rej] == [3, 6]  # rejects listed with line numbers
    with pytest.raises(E.SchemaError):
        F.read_points_csv("a,b\n1,2\n")
    with pytest.raises(E.SchemaError):
        F.read_points_csv("x,y\nq,w\n")  # empty dataset


def test_geojson_two_polygons_ids_and_multipolygon():
    fc = {"type": "FeatureCollection", "features": [
        {"type": "Feature", "geometry": {"type": "Polygon", "coordinates": [[[0, 0], [1, 0], [1, 1], [0, 1], [0, 0]]]}},
        {"type": "Feature", "geometry": {"type": "MultiPolygon", "coordinates": [
            [[[2, 2], [3, 2], [3, 3], [2, 2]]], [[[4, 4], [5, 4], [5, 5], [4, 4]]]]}}]}
    regs = F.read_regions_geojson(json.dumps(fc))
    assert [r.id for r in regs] == [0, 1]
    assert len(regs[0].geometry.outer) == 4 and isinstance(regs[1].geometry, list) and len(regs[1].geometry) == 2
    with pytest.raises(E.SchemaError):
        F.read_regions_geojson('{"type": "FeatureCollection", "features": [')


def test_wkt_polygon_with_hole_and_multipolygon():
    txt = ("POLYGON ((0 0, 10 0, 10 10, 0 10, 0 0), (2 2, 2 3, 3 3, 3 2, 2 2))\n"
           "MULTIPOLYGON (((20 20, 30 20, 30 30, 20 20)), ((40 40, 50 40, 50 50, 40 40)))\n")
    regs = F.read_regions_wkt(txt)
    assert [r.id for r in regs] == [0, 1]
    assert len(regs[0].geometry.holes) == 1 and len(regs[1].geometry) == 2


def test_normalize_unit_square_with_padding():
    regs = F.read_regions_wkt("POLYGON ((0 0, 100 0, 100 50, 0 50, 0 0))\n")
    xy = np.array([[200.0, 25.0]])  # outside every region's MBR: still ingested
    nxy, nregs, cfg, T = F.normalize(xy, regs)
    allv = np.concatenate([nxy, nregs[0].geometry.outer])
    assert allv.min() > 0.0 and allv.max() < 1.0
    np.testing.assert_allclose(allv.min(0)[0], 0.01 / 1.02)
    np.testing.assert_allclose(T.invert(nxy), xy)
    assert (cfg.origin.x, cfg.origin.y, cfg.extent) == (0.0, 0.0, 1.0)


def test_cellid_and_covering_dump_round_trip(tmp_path):
    lv = np.array([0, 3, 31], np.int32)
    code = np.array([0, 39, (1 << 62) - 1], np.uint64)
    F.write_cellids(tmp_path / "c.bin", lv, code)
    assert (tmp_path / "c.bin").stat().st_size == 27  # 9 bytes per CellId
    l2, c2 = F.read_cellids(tmp_path / "c.bin")
    assert l2.tolist() == lv.tolist() and c2.tolist() == code.tolist()
    buf = io.StringIO()
    F.write_covering_dump(buf, [5, 5, 7], lv, code, [1, 2, 1])
    assert buf.getvalue().splitlines()[1] == "5 3 39 B"
    rid, l3, c3, k3 = F.read_covering_dump(io.StringIO(buf.getvalue()))
    assert rid.tolist() == [5, 5, 7] and k3.tolist() == [1, 2, 1] and c3.tolist() == code.tolist()


def test_act_file_header_round_trip(tmp_path):
    from paper_2010_12548_b200.geometry import Point2D
    from paper_2010_12548_b200.grid import GridConfig

    g = GridConfig(Point2D(0.5, -1.0), 2.0, 9)
    F.write_act(tmp_path / "a.act", g, 4, [3, 3], [9, 2], [12345, 7], [2, 1])
    assert (tmp_path / "a.act").read_bytes()[:8] == F.ACT_MAGIC
    g2, rw, rid, lv, code, kind = F.read_act(tmp_path / "a.act")
    assert (g2.origin.x, g2.origin.y, g2.extent, g2.max_level, rw) == (0.5, -1.0, 2.0, 9, 4)
    assert rid.tolist() == [3, 3] and lv.tolist() == [9, 2] and code.tolist() == [12345, 7] and kind.tolist() == [2, 1]
    (tmp_path / "bad.act").write_bytes(b"XXXXXXXX")
    with pytest.raises(E.SchemaError):
        F.read_act(tmp_path / "bad.act")
