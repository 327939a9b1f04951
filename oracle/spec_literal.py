"""ORACLE tier (i) -- SPEC-literal, pure Python; test infrastructure only.

A line-by-line restatement of the reference algorithm as SPEC.md words it,
with its own geometric predicates, used at small sizes to validate the C
oracle (tier ii, oracle/rb_oracle.c) on generic inputs:

  * classify_cell: PARTIAL iff some polygon edge meets the
    OPEN cell square (segment / open-rectangle test by parametric clipping,
    a different float formulation from the C column walk); otherwise
    INSIDE/OUTSIDE by point_in_polygon of the cell centre (D2);
  * rasterize_hierarchical: recursive quadtree descent
    from the root cell;
  * AdaptiveCellTrie: a real radix trie over padded Z codes,
    `radix_width` bits per node, cells terminating at depth
    ceil(2*level/radix_width) with their (region_id, kind) terminal entries,
    lookups collecting every terminal on the path;
  * join_act: per point leaf code -> trie lookup ->
    accumulate alpha into every owner, beta for boundary owners.

Everything is computed in grid units u = (v - origin) / side (the map of
SPEC.md:146 applied to vertices and points alike).
"""
from __future__ import annotations

import math

INSIDE, OUTSIDE, PARTIAL = "INSIDE", "OUTSIDE", "PARTIAL"


def level_for_bound(extent: float, eps: float) -> int:
    """SPEC.md:125-133."""
    t = eps / math.sqrt(2.0)
    for l in range(32):
        if math.ldexp(extent, -l) <= t:
            return l
    raise OverflowError("capacity: level > 31")


def z_encode(ix: int, iy: int) -> int:
    """x bit i -> 2i, y bit i -> 2i+1."""
    z = 0
    for b in range(32):
        z |= ((ix >> b) & 1) << (2 * b)
        z |= ((iy >> b) & 1) << (2 * b + 1)
    return z


def z_decode(z: int):
    ix = iy = 0
    for b in range(32):
        ix |= ((z >> (2 * b)) & 1) << b
        iy |= ((z >> (2 * b + 1)) & 1) << b
    return ix, iy


def to_grid(rings, origin, side):
    ox, oy = origin
    return [[((x - ox) / side, (y - oy) / side) for (x, y) in ring] for ring in rings]


def edges(rings):
    for ring in rings:
        n = len(ring)
        for k in range(n):
            yield ring[k], ring[(k + 1) % n]


def seg_meets_open_rect(a, b, x0, y0, x1, y1) -> bool:
    """Does segment [a, b] contain a point strictly inside (x0,x1) x (y0,y1)?"""
    lo, hi = 0.0, 1.0
    for p, d, r0, r1 in ((a[0], b[0] - a[0], x0, x1), (a[1], b[1] - a[1], y0, y1)):
        if d == 0.0:
            if not (r0 < p < r1):
                return False
            continue
        t0, t1 = (r0 - p) / d, (r1 - p) / d
        if t0 > t1:
            t0, t1 = t1, t0
        lo, hi = max(lo, t0), min(hi, t1)
    return lo < hi


def point_in_polygon(px, py, rings) -> bool:
    """even-odd over all rings, boundary counts as inside."""
    inside = False
    for (ax, ay), (bx, by) in edges(rings):
        if min(ax, bx) <= px <= max(ax, bx) and min(ay, by) <= py <= max(ay, by):
            if (bx - ax) * (py - ay) - (by - ay) * (px - ax) == 0.0:
                return True
        if (ay > py) != (by > py):
            xl, yl, xh, yh = (ax, ay, bx, by) if ay < by else (bx, by, ax, ay)
            xc = xl + ((py - yl) * (xh - xl)) / (yh - yl)
            if px == xc:
                return True
            if px < xc:
                inside = not inside
    return inside


def distance_to_boundary(px, py, rings) -> float:
    best = math.inf
    for (ax, ay), (bx, by) in edges(rings):
        dx, dy, wx, wy = bx - ax, by - ay, px - ax, py - ay
        L2 = dx * dx + dy * dy
        t = 0.0 if L2 == 0 else min(1.0, max(0.0, (wx * dx + wy * dy) / L2))
        best = min(best, math.hypot(wx - t * dx, wy - t * dy))
    return best


def classify_cell(level: int, code: int, grings, L: int) -> str:
    """SPEC.md:207-215 for a cell of `level` in grid units of level L."""
    s = 1 << (L - level)
    cx, cy = z_decode(code)
    x0, y0 = cx * s, cy * s
    x1, y1 = x0 + s, y0 + s
    for a, b in edges(grings):
        if seg_meets_open_rect(a, b, x0, y0, x1, y1):
            return PARTIAL
    return INSIDE if point_in_polygon(x0 + 0.5 * s, y0 + 0.5 * s, grings) else OUTSIDE


def rasterize_hierarchical(grings, L: int, center_sampled: bool = False):
    """list of (level, code, kind 'I'|'B')."""
    out = []

    def visit(level, code):
        c = classify_cell(level, code, grings, L)
        if c == OUTSIDE:
            return
        if c == INSIDE:
            out.append((level, code, "I"))
            return
        if level == L:
            if not center_sampled:
                out.append((level, code, "B"))
            else:
                cx, cy = z_decode(code)
                if point_in_polygon(cx + 0.5, cy + 0.5, grings):
                    out.append((level, code, "B"))
            return
        for k in range(4):
            visit(level + 1, 4 * code + k)

    visit(0, 0)
    return out


class AdaptiveCellTrie:
    """radix trie over Z codes, `radix_width` bits per node."""

    def __init__(self, L: int, radix_width: int = 8):
        if radix_width not in (2, 4, 8):
            raise ValueError("radix_width must be 2, 4 or 8 (SPEC.md:278)")
        self.L, self.w = L, radix_width
        self.root = self._node()

    def _node(self):
        return {"child": {}, "term": {}}

    def insert(self, level: int, code: int, region: int, kind: str):
        w = self.w
        depth = max(1, -(-2 * level // w))  # ceil(2l/w), root cell at depth 1
        pad = depth * w - 2 * level
        base = code << pad
        node = self.root
        for d in range(depth - 1):
            chunk = (base >> ((depth - 1 - d) * w)) & ((1 << w) - 1)
            node = node["child"].setdefault(chunk, self._node())
        lo = base & ((1 << w) - 1)
        for slot in range(lo, lo + (1 << pad)):
            node["term"].setdefault(slot, set()).add((region, kind))

    def lookup_code(self, leaf: int):
        """Every terminal on the path of the level-L leaf code."""
        w = self.w
        depth = max(1, -(-2 * self.L // w))
        code = leaf << (depth * w - 2 * self.L)
        out = set()
        node = self.root
        for d in range(depth):
            chunk = (code >> ((depth - 1 - d) * w)) & ((1 << w) - 1)
            out |= node["term"].get(chunk, set())
            node = node["child"].get(chunk)
            if node is None:
                break
        return out


def build(regions, origin, extent: float, L: int, center_sampled: bool = False, radix_width: int = 8):
    """regions: list of (region_id, [polygon rings...]) with polygons given as
    lists of rings in original units.  Returns (trie, per-polygon coverings)."""
    side = math.ldexp(extent, -L)
    trie = AdaptiveCellTrie(L, radix_width)
    covers = []
    for rid, polys in regions:
        for rings in polys:
            g = to_grid(rings, origin, side)
            cells = rasterize_hierarchical(g, L, center_sampled)
            covers.append((rid, cells))
            for lv, code, kind in cells:
                trie.insert(lv, code, rid, kind)
    return trie, covers


def join_act(points, trie: AdaptiveCellTrie, origin, extent: float, attr=None):
    """{region: [alpha_cnt, beta_cnt, alpha_sum, beta_sum]}."""
    L = trie.L
    side = math.ldexp(extent, -L)
    res = {}
    for k, (x, y) in enumerate(points):
        ix = math.floor((x - origin[0]) / side)
        iy = math.floor((y - origin[1]) / side)
        if not (0 <= ix < (1 << L) and 0 <= iy < (1 << L)):
            raise ValueError(f"domain: point {k}")
        owners = {}
        for rid, kind in trie.lookup_code(z_encode(ix, iy)):
            owners[rid] = "I" if (kind == "I" or owners.get(rid) == "I") else "B"
        w = attr[k] if attr is not None else 0.0
        for rid, kind in owners.items():
            r = res.setdefault(rid, [0, 0, 0.0, 0.0])
            r[0] += 1
            r[2] += w
            if kind == "B":
                r[1] += 1
                r[3] += w
    return res
