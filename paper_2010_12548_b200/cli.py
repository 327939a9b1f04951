"""rasterbound.cli: ingestion, configuration, benchmark
orchestration and JSON-lines emission around the B200 engine.

  rasterbound ingest     --points P.csv --regions R.geojson|R.wkt --out DIR
  rasterbound rasterize  --regions ... --epsilon E [--mode ...] --out cover.txt   (covering dump)
  rasterbound index build --kind act|point --points/--regions ... --out FILE
  rasterbound query      --index FILE.act --points ...                          (act_lookup per point)
  rasterbound join       --points ... --regions ... --epsilon E --engine act|pointindex|canvas|all
                         --agg count|sum:attr|avg:attr --out results.jsonl
  rasterbound bench      [--points ... --regions ...] --epsilon E1,E2 --engine all --seed S --out bench.jsonl
  rasterbound audit      --points ... --regions ... --epsilon E                 (validator vs exact PIP)

Inputs are normalised into the unit square with 1 % padding.
Without input files, bench runs a seeded synthetic workload (clustered points +
random polygons).  Log level comes from RASTERBOUND_LOG only.
"""
from __future__ import annotations

import json
import logging
import os
import sys
import time

import click
import numpy as np

from . import errors as E
from . import formats as F

log = logging.getLogger("rasterbound")
logging.basicConfig(level=os.environ.get("RASTERBOUND_LOG", "WARNING").upper(), stream=sys.stderr)

ENGINES = ("act", "pointindex", "canvas")


def _mode(s: str):
    from .raster import RasterMode

    return RasterMode.CONSERVATIVE if s.lower().startswith("cons") else RasterMode.CENTER_SAMPLED


def _load(points, regions, x_col="x", y_col="y"):
    """ingest: parse, report rejects, normalise."""
    from .geometry import PointSet

    xy, attrs, rejects = F.read_points_csv(points, x_col, y_col)
    for line, why in rejects:
        log.warning("points line %d rejected: %s", line, why)
    regs = F.read_regions(regions)
    nxy, nregs, cfg, T = F.normalize(xy, regs)
    return PointSet(nxy, attrs), nregs, cfg, T, rejects


def _synthetic(seed: int, n: int = 200_000, k: int = 50):
    """SPEC.md:565 synthetic workload: seeded clustered points + random polygons (unit square)."""
    from .geometry import Point2D, PointSet, Polygon, RegionRecord
    from .grid import GridConfig

    rng = np.random.default_rng(seed)
    c = rng.random((8, 2)) * 0.8 + 0.1
    xy = c[rng.integers(0, 8, n)] + rng.normal(0, 0.05, (n, 2))
    xy = np.clip(xy, 0.0, 1.0 - 1e-9)
    regs = []
    for i in range(k):
        r = rng.uniform(0.02, 0.08)
        cx, cy = rng.uniform(0.1, 0.9, 2)
        ang = np.sort(rng.uniform(0, 2 * np.pi, int(rng.integers(5, 20))))
        rad = r * (1 - 0.5 * rng.random(len(ang)))
        regs.append(RegionRecord(i, Polygon(np.stack([cx + rad * np.cos(ang), cy + rad * np.sin(ang)], 1))))
    fare = rng.lognormal(2.5, 0.6, n).astype(np.float32)
    return PointSet(xy, {"fare": fare}), regs, GridConfig(Point2D(0.0, 0.0), 1.0, 0)


def _join(engine: str, pts, regs, q, cfg):
    from . import pointindex as P
    from .query import join_act, join_canvas, join_pointindex
    from .grid import level_for_bound

    t0 = time.perf_counter()
    if engine == "act":
        res = join_act(pts, regs, q, cfg)
    elif engine == "canvas":
        res = join_canvas(pts, regs, q, cfg)
    else:
        grid = cfg.with_level(level_for_bound(cfg, q.epsilon))
        attrs = () if q.agg.kind == "COUNT" else (q.agg.attr,)
        lps = P.lps_build(pts, grid, attrs)
        rs = P.rs_build(lps)
        res = join_pointindex(lps, rs, regs, q)
    return res, time.perf_counter() - t0


@click.group()
def main():
    """rasterbound -- epsilon-bounded spatial aggregation on B200."""


@main.command()
@click.option("--points", required=True, type=click.Path(exists=True))
@click.option("--regions", required=True, type=click.Path(exists=True))
@click.option("--x-col", default="x")
@click.option("--y-col", default="y")
@click.option("--out", required=True, type=click.Path())
def ingest(points, regions, x_col, y_col, out):
    """Normalise points and regions into the unit square (1 % padding)."""
    pts, regs, cfg, T, rejects = _load(points, regions, x_col, y_col)
    os.makedirs(out, exist_ok=True)
    np.save(os.path.join(out, "points_xy.npy"), pts.xy)
    for k, v in pts.attrs.items():
        np.save(os.path.join(out, f"points_{k}.npy"), v)
    feats = []
    for r in regs:
        polys = r.geometry if isinstance(r.geometry, list) else [r.geometry]
        coords = [[np.vstack([ring, ring[:1]]).tolist() for ring in p.rings] for p in polys]
        g = {"type": "Polygon", "coordinates": coords[0]} if len(coords) == 1 else \
            {"type": "MultiPolygon", "coordinates": coords}
        feats.append({"type": "Feature", "id": r.id, "geometry": g, "properties": {}})
    with open(os.path.join(out, "regions.geojson"), "w") as f:
        json.dump({"type": "FeatureCollection", "features": feats}, f)
    meta = {"points": len(pts), "regions": len(regs), "rejects": rejects,
            "normalization": {"x0": T.x0, "y0": T.y0, "scale": T.scale}}
    with open(os.path.join(out, "ingest.json"), "w") as f:
        json.dump(meta, f)
    click.echo(json.dumps({k: v for k, v in meta.items() if k != "rejects"} | {"rejected": len(rejects)}))


@main.command()
@click.option("--regions", required=True, type=click.Path(exists=True))
@click.option("--epsilon", required=True, type=float)
@click.option("--mode", default="conservative")
@click.option("--out", required=True, type=click.Path())
def rasterize(regions, epsilon, mode, out):
    """Covering dump: one line per cell `region_id level code kind(I|B)`."""
    from .raster import rasterize_hierarchical

    regs = F.read_regions(regions)
    _, nregs, cfg, _ = F.normalize(np.zeros((0, 2)), regs)
    with open(out, "w") as f:
        for r in nregs:
            ra = rasterize_hierarchical(r.geometry, cfg, epsilon, _mode(mode), region_id=r.id)
            F.write_covering_dump(f, [r.id] * ra.n_cells, ra.levels, ra.codes, ra.kinds)


@main.group()
def index():
    """Build / inspect persistent indexes."""


@index.command("build")
@click.option("--kind", type=click.Choice(["act", "point"]), default="act")
@click.option("--points", type=click.Path(exists=True))
@click.option("--regions", type=click.Path(exists=True))
@click.option("--epsilon", required=True, type=float)
@click.option("--mode", default="conservative")
@click.option("--radix-width", default=8, type=int)
@click.option("--sum", "sums", multiple=True, help="attributes with prefix sums (point index)")
@click.option("--out", required=True, type=click.Path())
def index_build(kind, points, regions, epsilon, mode, radix_width, sums, out):
    """ACT file from regions, or point index file from points."""
    from . import pointindex as P
    from .act import save_act
    from .grid import level_for_bound
    from .raster import rasterize_hierarchical

    if kind == "act":
        if not regions:
            raise click.UsageError("--regions is required for an ACT")
        regs = F.read_regions(regions)
        _, nregs, cfg, _ = F.normalize(np.zeros((0, 2)), regs)
        cov = [rasterize_hierarchical(r.geometry, cfg, epsilon, _mode(mode), region_id=r.id) for r in nregs]
        save_act(out, cov, radix_width)
    else:
        if not points:
            raise click.UsageError("--points is required for a point index")
        from .geometry import PointSet

        xy, attrs, _ = F.read_points_csv(points)
        regs = F.read_regions(regions) if regions else []
        nxy, _, cfg, _ = F.normalize(xy, regs)
        grid = cfg.with_level(level_for_bound(cfg, epsilon))
        lps = P.lps_build(PointSet(nxy, attrs), grid, sums)
        P.save_point_index(out, lps, P.rs_build(lps))
    click.echo(json.dumps({"kind": kind, "out": out}))


@main.command()
@click.option("--index", "index_path", required=True, type=click.Path(exists=True))
@click.option("--points", required=True, type=click.Path(exists=True))
@click.option("--regions", required=True, type=click.Path(exists=True),
              help="the regions the ACT was built from (its normalisation)")
def query(index_path, points, regions):
    """act_lookup per point: JSON lines {point, owners}."""
    from .act import act_lookup_many, load_act

    xy, _, _ = F.read_points_csv(points)
    _, _, _, T = F.normalize(np.zeros((0, 2)), F.read_regions(regions))
    nxy = T.apply(xy)
    t = load_act(index_path)
    for k, own in enumerate(act_lookup_many(t, nxy)):
        click.echo(json.dumps({"point": k, "owners": sorted([list(o) for o in own])}))


@main.command()
@click.option("--points", required=True, type=click.Path(exists=True))
@click.option("--regions", required=True, type=click.Path(exists=True))
@click.option("--epsilon", required=True, type=float)
@click.option("--mode", default="conservative")
@click.option("--engine", type=click.Choice(ENGINES + ("all",)), default="act")
@click.option("--agg", default="count")
@click.option("--x-col", default="x")
@click.option("--y-col", default="y")
@click.option("--out", type=click.Path(), default=None)
def join(points, regions, epsilon, mode, engine, agg, x_col, y_col, out):
    """Per-region results as JSON lines."""
    from .query import AggregationQuery

    pts, regs, cfg, _, _ = _load(points, regions, x_col, y_col)
    q = AggregationQuery(agg, epsilon, _mode(mode))
    lines = []
    for eng in (ENGINES if engine == "all" else (engine,)):
        res, _ = _join(eng, pts, regs, q, cfg)
        lines.append(F.results_jsonl(res, q, eng))
    text = "".join(lines)
    if out:
        with open(out, "w") as f:
            f.write(text)
    else:
        click.echo(text, nl=False)


def run_bench(pts, regs, cfg, epsilons, engines, agg, mode, seed, audit_sample=0):
    """per (engine, eps) build + run + audit vs the exact PIP
    oracle; yields BenchRecord dicts.  Capacity errors are reported per run.
    audit_sample 0 (default): every point (rb_validate_full); > 0: a seeded sample."""
    from .engine import ApproxIndex
    from .geometry import pack_regions
    from .grid import level_for_bound
    from .query import AggregationQuery
    from .validate import validate, validate_full

    packed = pack_regions(regs)
    for eps in epsilons:
        q = AggregationQuery(agg, eps, _mode(mode))
        grid = cfg.with_level(level_for_bound(cfg, eps))
        rep = None
        try:
            t = time.perf_counter()
            idx = ApproxIndex(packed, grid, int(q.mode))
            build_s = time.perf_counter() - t
            rep = validate_full(idx, pts.xy, eps) if audit_sample <= 0 else \
                validate(idx, pts.xy, eps, max_points=audit_sample, seed=seed)
            mem = int(idx.stats()["index_bytes"])
        except E.RasterBoundError as ex:
            yield {"engine": "all", "epsilon": eps, "error": f"{type(ex).__name__}: {ex}"}
            continue
        for eng in engines:
            rec = {"engine": eng, "epsilon": eps, "mode": q.mode.name, "agg": str(q.agg), "seed": seed}
            try:
                res, qs = _join(eng, pts, regs, q, cfg)
            except E.RasterBoundError as ex:
                rec["error"] = f"{type(ex).__name__}: {ex}"
                yield rec
                continue
            rec.update(build_time=round(build_s, 6), query_time=round(qs, 6), index_bytes=mem,
                       regions=[{"region_id": r.region_id, "alpha": r.alpha, "beta": r.boundary_part,
                                 "range": r.range} for r in res],
                       audit={"points": rep.points, "mismatch_fraction": rep.mismatch_fraction,
                              "false_negatives": rep.false_negatives,
                              "max_mismatch_distance": rep.max_mismatch_distance, "eps_ok": rep.ok,
                              "violations": getattr(rep, "violations", None)})
            yield rec


@main.command()
@click.option("--points", type=click.Path(exists=True))
@click.option("--regions", type=click.Path(exists=True))
@click.option("--epsilon", "epsilons", default="0.01,0.005", help="comma-separated list")
@click.option("--mode", default="conservative")
@click.option("--engine", type=click.Choice(ENGINES + ("all",)), default="all")
@click.option("--agg", default="count")
@click.option("--seed", default=0, type=int)
@click.option("--parallel", is_flag=True, help="accepted for compatibility: the point scan is always parallel on the GPU")
@click.option("--out", type=click.Path(), default=None)
def bench(points, regions, epsilons, mode, engine, agg, seed, parallel, out):
    """BenchRecord JSON lines."""
    if points and regions:
        pts, regs, cfg, _, _ = _load(points, regions)
    else:
        pts, regs, cfg = _synthetic(seed)
    eps = [float(e) for e in epsilons.split(",")]
    engines = ENGINES if engine == "all" else (engine,)
    f = open(out, "w") if out else None
    for rec in run_bench(pts, regs, cfg, eps, engines, agg, mode, seed):
        line = json.dumps(rec)
        (f.write(line + "\n") if f else click.echo(line))
    if f:
        f.close()


@main.command()
@click.option("--points", required=True, type=click.Path(exists=True))
@click.option("--regions", required=True, type=click.Path(exists=True))
@click.option("--epsilon", required=True, type=float)
@click.option("--mode", default="conservative")
@click.option("--sample", default=0, type=int, help="0 (default): every point; N > 0: a seeded sample of N")
def audit(points, regions, epsilon, mode, sample):
    """Validator: every point assigned differently from the exact test lies within eps."""
    from .engine import ApproxIndex
    from .geometry import pack_regions
    from .grid import level_for_bound
    from .validate import validate, validate_full

    pts, regs, cfg, _, _ = _load(points, regions)
    grid = cfg.with_level(level_for_bound(cfg, epsilon))
    idx = ApproxIndex(pack_regions(regs), grid, int(_mode(mode)))
    rep = validate_full(idx, pts.xy, epsilon) if sample <= 0 else validate(idx, pts.xy, epsilon, max_points=sample)
    click.echo(json.dumps(rep.as_dict()))


if __name__ == "__main__":
    main()
