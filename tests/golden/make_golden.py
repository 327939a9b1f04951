"""Writes tests/golden/spec_examples.json: every `examples:` line of the
reference SPEC.md on the join path, transcribed with its SPEC.md line number.
The reference ships no implementation or test fixtures,
so these examples are its only golden vectors.  Re-run to regenerate:
    python tests/golden/make_golden.py
"""
import json
import math
import os

R2 = math.sqrt(2.0)
UNIT = [[0, 0], [1, 0], [1, 1], [0, 1]]
SQ = lambda a, b: [[a, a], [b, a], [b, b], [a, b]]

EXAMPLES = [
    # geometry.point_in_polygon
    {"op": "point_in_polygon", "spec": "SPEC.md:55", "p": [0.5, 0.5], "outer": UNIT, "holes": [], "expect": True},
    {"op": "point_in_polygon", "spec": "SPEC.md:56", "p": [2, 2], "outer": UNIT, "holes": [], "expect": False},
    {"op": "point_in_polygon", "spec": "SPEC.md:57", "p": [0.5, 0.5], "outer": UNIT,
     "holes": [SQ(0.4, 0.6)[::-1]], "expect": False},
    # geometry.distance_to_boundary
    {"op": "distance_to_boundary", "spec": "SPEC.md:64", "p": [0.5, 0.5], "outer": UNIT, "expect": 0.5},
    {"op": "distance_to_boundary", "spec": "SPEC.md:65", "p": [1, 0], "outer": UNIT, "expect": 0.0},
    {"op": "distance_to_boundary", "spec": "SPEC.md:66", "p": [2, 0.5], "outer": UNIT, "expect": 1.0},
    # geometry.hausdorff_distance
    {"op": "hausdorff_distance", "spec": "SPEC.md:73", "A": [[0, 0], [1, 2]], "B": [[0, 0], [1, 2]], "expect": 0.0},
    {"op": "hausdorff_distance", "spec": "SPEC.md:74", "A": [[0, 0]], "B": [[3, 4]], "expect": 5.0},
    {"op": "hausdorff_squares", "spec": "SPEC.md:75", "inner": [0.25, 0.75], "outer": [0, 1],
     "expect": 0.3535533905932738, "tol": 1e-9},
    # geometry.mbr_of
    {"op": "mbr_of", "spec": "SPEC.md:82", "outer": UNIT, "expect": [0, 0, 1, 1]},
    {"op": "mbr_of", "spec": "SPEC.md:83", "outer": [[0, 0], [2, 0], [1, 3]], "expect": [0, 0, 2, 3]},
    {"op": "mbr_of", "spec": "SPEC.md:84", "outer": [[1, 0], [2, 1], [1, 2], [0, 1]], "expect": [0, 0, 2, 2]},
    # grid.level_for_bound
    {"op": "level_for_bound", "spec": "SPEC.md:131", "extent": 1.0, "epsilon": R2, "expect": 0},
    {"op": "level_for_bound", "spec": "SPEC.md:132", "extent": 1.0, "epsilon": R2 / 4, "expect": 2},
    {"op": "level_for_bound", "spec": "SPEC.md:133", "extent": 1.0, "epsilon": 0.1, "expect": 4},
    # grid.z_encode
    {"op": "z_encode", "spec": "SPEC.md:140", "ix": 0, "iy": 0, "level": 7, "expect": 0},
    {"op": "z_encode", "spec": "SPEC.md:141", "ix": 1, "iy": 0, "level": 1, "expect": 1},
    {"op": "z_encode", "spec": "SPEC.md:141", "ix": 0, "iy": 1, "level": 1, "expect": 2},
    {"op": "z_encode", "spec": "SPEC.md:142", "ix": 3, "iy": 5, "level": 3, "expect": 39},
    # grid.point_to_cell
    {"op": "point_to_cell", "spec": "SPEC.md:149", "origin": [0, 0], "extent": 1.0, "level": 1, "p": [0.3, 0.7],
     "expect": [1, 2]},
    {"op": "point_to_cell", "spec": "SPEC.md:150", "origin": [0, 0], "extent": 1.0, "level": 9, "p": [0, 0],
     "expect": [9, 0]},
    {"op": "point_to_cell", "spec": "SPEC.md:151", "origin": [0, 0], "extent": 1.0, "level": 1,
     "p": [0.9999999999, 0.9999999999], "expect": [1, 3]},
    # grid.cell_interval
    {"op": "cell_interval", "spec": "SPEC.md:158", "cell": [4, 77], "L": 4, "expect": [77, 78]},
    {"op": "cell_interval", "spec": "SPEC.md:159", "cell": [0, 0], "L": 2, "expect": [0, 16]},
    {"op": "cell_interval", "spec": "SPEC.md:160", "cell": [1, 2], "L": 2, "expect": [8, 12]},
    # grid.children / parent
    {"op": "children", "spec": "SPEC.md:168", "cell": [0, 0], "expect": [[1, 0], [1, 1], [1, 2], [1, 3]]},
    {"op": "parent", "spec": "SPEC.md:169", "cell": [2, 9], "expect": [1, 2]},
    # raster.classify_cell (grid: unit square domain)
    {"op": "classify_cell", "spec": "SPEC.md:213", "cell": [0, 0], "outer": SQ(0.25, 0.75), "expect": "PARTIAL"},
    {"op": "classify_cell", "spec": "SPEC.md:214", "cell": [2, 0], "outer": UNIT, "expect": "INSIDE"},
    {"op": "classify_cell", "spec": "SPEC.md:215", "cell": [2, 5], "outer": SQ(0, 0.5), "expect": "OUTSIDE"},
    # raster.rasterize_hierarchical (extent 1, origin 0)
    {"op": "rasterize_hierarchical", "spec": "SPEC.md:222", "outer": UNIT, "extent": 1.0, "epsilon": R2,
     "expect_interior": [[0, 0]], "expect_boundary": []},
    {"op": "rasterize_hierarchical", "spec": "SPEC.md:223", "outer": SQ(0.25, 0.75), "extent": 1.0,
     "epsilon": R2 / 2, "expect_interior": [], "expect_boundary": [[1, 0], [1, 1], [1, 2], [1, 3]]},
    {"op": "rasterize_hierarchical", "spec": "SPEC.md:224", "outer": SQ(0.25, 0.75), "extent": 1.0,
     "epsilon": R2 / 8, "expect_interior": [[2, 3], [2, 6], [2, 9], [2, 12]], "expect_boundary": []},
    # raster.rasterize_uniform
    {"op": "rasterize_uniform", "spec": "SPEC.md:231", "outer": UNIT, "extent": 1.0, "epsilon": R2 / 2,
     "expect_interior": [[1, 0], [1, 1], [1, 2], [1, 3]], "expect_boundary": []},
    {"op": "rasterize_uniform", "spec": "SPEC.md:232", "outer": UNIT, "extent": 2.0, "epsilon": R2,
     "expect_interior": [[1, 0]], "expect_boundary": []},
    # act_build / act_lookup (regions: id -> outer ring; grid unit square)
    {"op": "act_lookup", "spec": "SPEC.md:282", "regions": {"5": UNIT}, "epsilon": R2,
     "points": [[0.1, 0.1], [0.9, 0.5]], "expect": [[[5, "I"]], [[5, "I"]]]},
    {"op": "act_lookup", "spec": "SPEC.md:283", "regions": {"0": [[0, 0], [0.5, 0], [0.5, 1], [0, 1]],
                                                             "1": [[0.5, 0], [1, 0], [1, 1], [0.5, 1]]},
     "epsilon": R2 / 2, "points": [[0.2, 0.7], [0.8, 0.2]], "expect": [[[0, "I"]], [[1, "I"]]]},
    {"op": "act_lookup", "spec": "SPEC.md:291", "regions": {}, "epsilon": R2, "points": [[0.3, 0.3]],
     "expect": [[]]},
    # pointindex.lps_build: leaf codes at L=1 over the unit square (code 0 = (0,0), 1 = (1,0),
    # 2 = (0,1), 3 = (1,1)); counts per code [1, 2, 0, 3] -> COUNT prefix [0, 1, 3, 3, 6]
    {"op": "lps_build", "spec": "SPEC.md:334", "L": 1,
     "points": [[0.1, 0.1], [0.6, 0.2], [0.9, 0.4], [0.7, 0.7], [0.8, 0.9], [0.55, 0.6]],
     "expect_codes": [0, 1, 1, 3, 3, 3], "expect_count_prefix": [0, 1, 3, 3, 6]},
    {"op": "lps_build", "spec": "SPEC.md:333", "L": 3, "points": [], "expect_codes": [], "expect_prefix": [0]},
    {"op": "lps_build", "spec": "SPEC.md:335", "L": 4, "points": [[0.3, 0.3], [0.3, 0.3]],
     "expect_codes_equal_adjacent": True},
    # pointindex.bounds_lookup
    {"op": "bounds_lookup", "spec": "SPEC.md:352", "codes": [2, 4, 4, 7, 9, 12], "iv": [0, 1 << 40],
     "expect": [0, 6]},
    {"op": "bounds_lookup", "spec": "SPEC.md:353", "codes": [2, 4, 4, 7, 9, 12], "iv": [4, 8], "expect": [1, 4]},
    {"op": "bounds_lookup", "spec": "SPEC.md:354", "codes": [2, 4, 4, 7, 9, 12], "iv": [5, 5], "expect": [3, 3]},
    # pointindex.range_aggregate: counts per code [1, 2, 0, 3], cells covering codes {1, 2} -> 2
    {"op": "range_aggregate", "spec": "SPEC.md:361", "codes": [0, 1, 1, 3, 3, 3], "cells": [[1, 3]], "expect": 2},
    {"op": "range_aggregate", "spec": "SPEC.md:362", "codes": [0, 1, 1, 3, 3, 3], "cells": [[0, 4]], "expect": 6},
    # query.join_act
    {"op": "join_act", "spec": "SPEC.md:488", "outer": UNIT, "epsilon": 0.1,
     "points": [[0.1, 0.1], [0.2, 0.9], [0.5, 0.5], [0.7, 0.3], [0.9, 0.9], [0.05, 0.6], [0.6, 0.05]],
     "expect": {"alpha": 7, "beta": 0, "range": [7, 7]}},
    # query.result_range
    {"op": "result_range", "spec": "SPEC.md:515", "alpha": 10, "beta": 3, "agg": "COUNT",
     "mode": "CONSERVATIVE", "expect": [7, 10]},
    {"op": "result_range", "spec": "SPEC.md:516", "alpha": 4, "beta": 0, "agg": "COUNT",
     "mode": "CONSERVATIVE", "expect": [4, 4]},
    {"op": "result_range", "spec": "SPEC.md:517", "alpha": 4.5, "beta": 1.0, "agg": "AVG:fare",
     "mode": "CONSERVATIVE", "expect": None},
]

if __name__ == "__main__":
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "spec_examples.json")
    with open(out, "w") as f:
        json.dump({"source": "/root/reference/SPEC.md examples (transcribed)", "examples": EXAMPLES}, f, indent=1)
    print("wrote", out, len(EXAMPLES), "examples")
