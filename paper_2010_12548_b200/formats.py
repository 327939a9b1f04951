"""File formats and ingestion of the reference's artifact plumbing (SPEC.md:538-586
cli.ingest; SPEC.md:185 CellId, :258 covering dump, :306 ACT file, :377 point
index file, :531 JSON-lines results).

Host-side parsing/serialisation only: the bulk work (rasterising, indexing,
joining) stays in librasterbound_b200.so.

  points CSV      header names the location columns (default x, y); other numeric
                  columns become attributes; unparsable rows are rejected with
                  their line numbers
  regions         GeoJSON FeatureCollection (Polygon / MultiPolygon features, ids
                  0, 1, ... in order) or WKT (one POLYGON / MULTIPOLYGON per line)
  normalisation   affine map of the data MBR into the unit square with 1 % padding
                  (SPEC.md:556); the transform is returned for the inverse
  covering dump   one line per cell: `region_id level code kind(I|B)`
  CellId binary   (level u8, code u64) little-endian
  ACT file        versioned magic, radix_width, grid, then the covering cells the
                  index is rebuilt from (the GPU radix table has no
                  pointer nodes to stream, so the cells are its preorder content)
  point index     versioned magic, grid, codes, permutation, prefix arrays, spline
                  knots and radix table, little-endian
"""
from __future__ import annotations

import csv
import io
import json
import re
import struct
from dataclasses import dataclass

import numpy as np

from . import errors as E
from .geometry import Point2D, PointSet, Polygon, RegionRecord
from .grid import GridConfig

ACT_MAGIC = b"RBACT\x00\x01\x00"
LPS_MAGIC = b"RBPIX\x00\x01\x00"


@dataclass(frozen=True)
class Normalization:
    """Affine map x' = (x - x0) * scale, y' = (y - y0) * scale into the unit square."""
    x0: float
    y0: float
    scale: float

    def apply(self, xy: np.ndarray) -> np.ndarray:
        out = np.empty_like(np.asarray(xy, np.float64))
        out[:, 0] = (xy[:, 0] - self.x0) * self.scale
        out[:, 1] = (xy[:, 1] - self.y0) * self.scale
        return out

    def invert(self, xy: np.ndarray) -> np.ndarray:
        return np.stack([xy[:, 0] / self.scale + self.x0, xy[:, 1] / self.scale + self.y0], 1)


# ------------------------------------------------------------------ points
def read_points_csv(path_or_text, x_col: str = "x", y_col: str = "y"):
    """-> (xy float64 [N,2], {attr: float32 [N]}, rejects [(line, reason)])."""
    f = io.StringIO(path_or_text) if "\n" in str(path_or_text) else open(path_or_text, newline="")
    with f:
        rd = csv.reader(f)
        try:
            header = [h.strip() for h in next(rd)]
        except StopIteration:
            raise E.SchemaError("points CSV is empty") from None
        if x_col not in header or y_col not in header:
            raise E.SchemaError(f"points CSV header lacks {x_col!r}/{y_col!r} (line 1)")
        ix, iy = header.index(x_col), header.index(y_col)
        others = [(k, h) for k, h in enumerate(header) if k not in (ix, iy)]
        xs, ys, cols, rejects = [], [], {h: [] for _, h in others}, []
        for line, row in enumerate(rd, start=2):
            if not row or all(not c.strip() for c in row):
                continue
            try:
                x, y = float(row[ix]), float(row[iy])
                if not (np.isfinite(x) and np.isfinite(y)):
                    raise ValueError("non-finite coordinate")
                vals = {h: float(row[k]) if k < len(row) and row[k].strip() else np.nan for k, h in others}
            except (ValueError, IndexError) as ex:
                rejects.append((line, str(ex)))
                continue
            xs.append(x)
            ys.append(y)
            for h, v in vals.items():
                cols[h].append(v)
    if not xs:
        raise E.SchemaError("points CSV holds no valid point")
    attrs = {h: np.asarray(v, np.float32) for h, v in cols.items()}
    return np.stack([np.asarray(xs), np.asarray(ys)], 1), attrs, rejects


# ------------------------------------------------------------------ regions
def _ring(coords) -> np.ndarray:
    a = np.asarray(coords, np.float64)
    if a.ndim != 2 or a.shape[1] < 2 or len(a) < 3:
        raise E.GeometryError("ring needs at least three 2-D vertices")
    a = a[:, :2]
    if np.array_equal(a[0], a[-1]):
        a = a[:-1]
    return a


def _poly_from_coords(rings) -> Polygon:
    return Polygon(_ring(rings[0]), [_ring(h) for h in rings[1:]])


def read_regions_geojson(path_or_text) -> list:
    """FeatureCollection (or a single Feature / geometry) -> RegionRecords with ids 0, 1, ..."""
    txt = path_or_text if str(path_or_text).lstrip().startswith("{") else open(path_or_text).read()
    try:
        doc = json.loads(txt)
    except json.JSONDecodeError as ex:
        raise E.SchemaError(f"GeoJSON parse error at line {ex.lineno} column {ex.colno}: {ex.msg}") from None
    feats = doc.get("features") if doc.get("type") == "FeatureCollection" else [doc]
    out = []
    for k, ft in enumerate(feats):
        g = ft.get("geometry", ft)
        t = g.get("type")
        if t == "Polygon":
            geom = _poly_from_coords(g["coordinates"])
        elif t == "MultiPolygon":
            geom = [_poly_from_coords(p) for p in g["coordinates"]]
        else:
            raise E.SchemaError(f"feature {k}: unsupported geometry type {t!r}")
        out.append(RegionRecord(len(out), geom))
    if not out:
        raise E.SchemaError("GeoJSON holds no region")
    return out


_NUM = r"[-+]?(?:\d+\.?\d*|\.\d+)(?:[eE][-+]?\d+)?"


def _wkt_rings(body: str):
    rings = re.findall(r"\(([^()]*)\)", body)
    out = []
    for r in rings:
        pts = [p.split() for p in r.split(",")]
        out.append([(float(p[0]), float(p[1])) for p in pts if p])
    return out


def read_regions_wkt(path_or_text) -> list:
    """One POLYGON((...),(hole)) or MULTIPOLYGON(((...)),((...))) per line -> RegionRecords."""
    txt = path_or_text if "(" in str(path_or_text) else open(path_or_text).read()
    out = []
    for line, raw in enumerate(txt.splitlines(), start=1):
        s = raw.strip()
        if not s:
            continue
        head = s.split("(", 1)[0].strip().upper()
        body = s[len(s.split("(", 1)[0]):]
        try:
            if head == "POLYGON":
                geom = _poly_from_coords(_wkt_rings(body))
            elif head == "MULTIPOLYGON":
                parts = re.findall(r"\(\s*(\(.*?\)(?:\s*,\s*\(.*?\))*)\s*\)", body[1:-1])
                geom = [_poly_from_coords(_wkt_rings(p)) for p in parts]
            else:
                raise E.SchemaError(f"line {line}: unsupported WKT {head!r}")
        except (ValueError, IndexError) as ex:
            raise E.SchemaError(f"WKT parse error at line {line}: {ex}") from None
        out.append(RegionRecord(len(out), geom))
    if not out:
        raise E.SchemaError("WKT holds no region")
    return out


def read_regions(path: str) -> list:
    p = str(path)
    if p.endswith((".json", ".geojson")) or p.lstrip().startswith("{"):
        return read_regions_geojson(p)
    return read_regions_wkt(p)


def _region_vertices(regions) -> np.ndarray:
    vs = []
    for r in regions:
        for poly in (r.geometry if isinstance(r.geometry, list) else [r.geometry]):
            for ring in poly.rings:
                vs.append(ring)
    return np.concatenate(vs) if vs else np.zeros((0, 2))


def normalize(xy: np.ndarray, regions, pad: float = 0.01):
    """affine map of the data MBR (points and regions) into the unit
    square with `pad` of the larger span on every side -> (xy', regions', cfg, T)."""
    pts = [np.asarray(xy, np.float64).reshape(-1, 2), _region_vertices(regions)]
    allv = np.concatenate([p for p in pts if len(p)])
    if not len(allv):
        raise E.SchemaError("empty dataset")
    lo, hi = allv.min(0), allv.max(0)
    span = float(max(hi[0] - lo[0], hi[1] - lo[1])) or 1.0
    scale = 1.0 / ((1.0 + 2.0 * pad) * span)
    T = Normalization(float(lo[0] - pad * span), float(lo[1] - pad * span), scale)

    def npoly(poly: Polygon) -> Polygon:
        rings = [T.apply(r) for r in poly.rings]
        return Polygon(rings[0], rings[1:])

    regs = [RegionRecord(r.id, [npoly(p) for p in r.geometry] if isinstance(r.geometry, list) else npoly(r.geometry))
            for r in regions]
    return T.apply(np.asarray(xy, np.float64).reshape(-1, 2)), regs, GridConfig(Point2D(0.0, 0.0), 1.0, 0), T


# ------------------------------------------------------------------ cell formats
def write_cellids(path, levels, codes) -> None:
    """CellId serialisation: (level u8, code u64) little-endian records."""
    rec = np.zeros(len(levels), dtype=[("level", "<u1"), ("code", "<u8")])
    rec["level"] = np.asarray(levels, np.uint8)
    rec["code"] = np.asarray(codes, np.uint64)
    with open(path, "wb") as f:
        f.write(rec.tobytes())


def read_cellids(path):
    rec = np.frombuffer(open(path, "rb").read(), dtype=[("level", "<u1"), ("code", "<u8")])
    return rec["level"].astype(np.int32), rec["code"].astype(np.uint64)


def write_covering_dump(f, region_ids, levels, codes, kinds) -> None:
    """one line per cell `region_id level code kind(I|B)`."""
    for r, l, c, k in zip(region_ids, levels, codes, kinds):
        f.write(f"{int(r)} {int(l)} {int(c)} {'I' if int(k) == 1 else 'B'}\n")


def read_covering_dump(f):
    rid, lv, code, kind = [], [], [], []
    for line, raw in enumerate(f, start=1):
        t = raw.split()
        if not t:
            continue
        if len(t) != 4 or t[3] not in ("I", "B"):
            raise E.SchemaError(f"covering dump line {line}: expected `region_id level code I|B`")
        rid.append(int(t[0])); lv.append(int(t[1])); code.append(int(t[2])); kind.append(1 if t[3] == "I" else 2)
    return (np.asarray(rid, np.int64), np.asarray(lv, np.int32), np.asarray(code, np.uint64),
            np.asarray(kind, np.uint8))


def _grid_bytes(g: GridConfig) -> bytes:
    return struct.pack("<dddi", g.origin.x, g.origin.y, g.extent, g.max_level)


def _grid_from(b: bytes) -> GridConfig:
    ox, oy, ext, L = struct.unpack("<dddi", b)
    return GridConfig(Point2D(ox, oy), ext, L)


def write_act(path, grid: GridConfig, radix_width: int, region_ids, levels, codes, kinds) -> None:
    """ACT file: magic, radix_width, grid, n, then the cells."""
    n = len(levels)
    with open(path, "wb") as f:
        f.write(ACT_MAGIC)
        f.write(struct.pack("<i", int(radix_width)))
        f.write(_grid_bytes(grid))
        f.write(struct.pack("<q", n))
        f.write(np.asarray(region_ids, "<i8").tobytes())
        f.write(np.asarray(levels, "<u1").tobytes())
        f.write(np.asarray(codes, "<u8").tobytes())
        f.write(np.asarray(kinds, "<u1").tobytes())


def read_act(path):
    b = open(path, "rb").read()
    if b[:8] != ACT_MAGIC:
        raise E.SchemaError("not an ACT file (bad magic or version)")
    o = 8
    (rw,) = struct.unpack_from("<i", b, o); o += 4
    grid = _grid_from(b[o:o + 28]); o += 28
    (n,) = struct.unpack_from("<q", b, o); o += 8
    rid = np.frombuffer(b, "<i8", n, o); o += 8 * n
    lv = np.frombuffer(b, "<u1", n, o); o += n
    code = np.frombuffer(b, "<u8", n, o); o += 8 * n
    kind = np.frombuffer(b, "<u1", n, o)
    return grid, rw, rid.copy(), lv.astype(np.int32), code.copy(), kind.copy()


def write_point_index(path, lps, rs=None) -> None:
    """Point index file: magic, grid, n, n_attr, attribute names,
    codes, perm, prefix arrays, then (optional) spline knots and radix table."""
    codes = lps.codes.cpu().numpy().view(np.uint64)
    perm = lps.perm.cpu().numpy()
    with open(path, "wb") as f:
        f.write(LPS_MAGIC)
        f.write(_grid_bytes(lps.grid))
        f.write(struct.pack("<qi", lps.n, len(lps.attrs)))
        for a in lps.attrs:
            nb = a.encode()
            f.write(struct.pack("<i", len(nb)) + nb)
        f.write(codes.astype("<u8").tobytes())
        f.write(perm.astype("<i8").tobytes())
        for a in lps.attrs:
            f.write(lps.prefix(a).cpu().numpy().astype("<f8").tobytes())
        if rs is None:
            f.write(struct.pack("<iiq", -1, 0, 0))
        else:
            keys, pos = (t.cpu().numpy() for t in rs.knots)
            f.write(struct.pack("<iiq", rs.radix_bits, rs.max_error, rs.n_knots))
            f.write(keys.view(np.uint64).astype("<u8").tobytes())
            f.write(pos.astype("<i8").tobytes())
            f.write(rs.radix_table.cpu().numpy().astype("<u4").tobytes())


def read_point_index(path):
    """-> dict(grid, codes, perm, attrs, prefix {attr: f64 [n+1]}, radix_bits, max_error, keys, pos, table)."""
    b = open(path, "rb").read()
    if b[:8] != LPS_MAGIC:
        raise E.SchemaError("not a point index file (bad magic or version)")
    o = 8
    grid = _grid_from(b[o:o + 28]); o += 28
    n, na = struct.unpack_from("<qi", b, o); o += 12
    attrs = []
    for _ in range(na):
        (ln,) = struct.unpack_from("<i", b, o); o += 4
        attrs.append(b[o:o + ln].decode()); o += ln
    codes = np.frombuffer(b, "<u8", n, o).copy(); o += 8 * n
    perm = np.frombuffer(b, "<i8", n, o).copy(); o += 8 * n
    prefix = {}
    for a in attrs:
        prefix[a] = np.frombuffer(b, "<f8", n + 1, o).copy(); o += 8 * (n + 1)
    rb, me, nk = struct.unpack_from("<iiq", b, o); o += 16
    out = dict(grid=grid, codes=codes, perm=perm, attrs=attrs, prefix=prefix, radix_bits=rb, max_error=me)
    if rb >= 0:
        out["keys"] = np.frombuffer(b, "<u8", nk, o).copy(); o += 8 * nk
        out["pos"] = np.frombuffer(b, "<i8", nk, o).copy(); o += 8 * nk
        out["table"] = np.frombuffer(b, "<u4", (1 << rb) + 1, o).copy()
    return out


def results_jsonl(results, q, engine: str) -> str:
    """SPEC.md:531 JSON lines {region_id, alpha, beta, lo, hi, agg, epsilon, mode, engine}."""
    return "".join(r.to_json(q, engine) + "\n" for r in results)


__all__ = [
    "Normalization", "read_points_csv", "read_regions_geojson", "read_regions_wkt", "read_regions", "normalize",
    "write_cellids", "read_cellids", "write_covering_dump", "read_covering_dump", "write_act", "read_act",
    "write_point_index", "read_point_index", "results_jsonl", "ACT_MAGIC", "LPS_MAGIC",
]
