/*
 * rb_oracle.c -- ORACLE / TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C, scalar float64, no FMA contraction: build with
 * -ffp-contract=off) of the reference `rasterbound` package's approximate
 * point-polygon aggregation path.  The reference ships no implementation
 * (/root/reference holds only SPEC.md, PAPER.md and errors.py), so this file
 * restates SPEC.md directly; every function cites the SPEC line it follows.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * `--impl reference`) may load this library, and only as the checker / the
 * CPU baseline.  The product package (paper_2010_12548_b200/) never links it.
 *
 * Parity pinning: SPEC.md `examples:` golden vectors (tests/golden/) and the
 * SPEC-literal Python tier (oracle/spec_literal.py).  No reference artifact
 * pins results at config scale ("parity pinned to SPEC examples only").
 *
 * Semantics (DESIGN.md "Semantic ledger" restates these):
 *  S1 grid coordinates: u = (v - origin) / side, side = extent * 2^-L, IEEE
 *     float64 in that order.  Points and polygon vertices go
 *     through the same map; all rasterization happens in grid units where
 *     leaf (i,j) is the half-open square [i,i+1) x [j,j+1).
 *  S2 PARTIAL leaf: the polygon boundary meets the OPEN leaf square
 *     (pinned by the aligned example SPEC.md:224).  Computed by
 *     a per-edge column walk with one fixed formula (edge_walk below).
 *  S3 non-PARTIAL leaf: INSIDE iff its centre is inside by the even-odd
 *     scanline rule at y = j + 0.5 (centre instead of corner,
 *     see DESIGN.md D2).
 *  S4 CONSERVATIVE keeps every PARTIAL leaf as boundary; CENTER_SAMPLED keeps
 *     it iff point_in_polygon(centre) with boundary = inside.
 *  S5 region kind of a leaf: I if any polygon of the region says INSIDE, else
 *     B if any polygon keeps it as boundary.
 *  S6 ownership: a point adds to alpha of EVERY region owning its leaf and to
 *     beta when that region's kind is B.
 *  S7 hierarchical covering: top-down quadtree descent; a block is split iff
 *     it contains a PARTIAL leaf or a grid-line-aligned boundary piece crosses
 *     its open interior (= SPEC classify_cell PARTIAL).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_GEOMETRY (-1)
#define ORC_DOMAIN (-2)
#define ORC_CAPACITY (-3)
#define ORC_CONFIG (-4)
#define ORC_SCHEMA (-5)
#define ORC_SHAPE (-6)
#define ORC_NOMEM (-100)

#define MODE_CONSERVATIVE 0
#define MODE_CENTER 1

#define KIND_NONE 0
#define KIND_I 1
#define KIND_B 2

typedef struct {
  double ox, oy, extent;
  int32_t level;
} orc_grid;

/* ------------------------------------------------------------------ grid */

/* SPEC.md:125-133 level_for_bound: smallest l with extent*2^-l <= eps/sqrt(2). */
int orc_level_for_bound(double extent, double eps, int32_t* out) {
  if (!(eps > 0.0) || !(extent > 0.0)) return ORC_CONFIG;
  double t = eps / sqrt(2.0);
  for (int l = 0; l <= 31; ++l) {
    if (ldexp(extent, -l) <= t) { *out = l; return ORC_OK; }
  }
  return ORC_CAPACITY;
}

/* SPEC.md:134-142 z_encode: bit i of ix -> bit 2i, bit i of iy -> bit 2i+1. */
static inline uint64_t part1by1(uint64_t v) {
  v &= 0xffffffffull;
  v = (v | (v << 16)) & 0x0000ffff0000ffffull;
  v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
  v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}
static inline uint64_t zenc(uint64_t ix, uint64_t iy) { return part1by1(ix) | (part1by1(iy) << 1); }
static inline uint32_t compact1by1(uint64_t v) {
  v &= 0x5555555555555555ull;
  v = (v | (v >> 1)) & 0x3333333333333333ull;
  v = (v | (v >> 2)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v >> 4)) & 0x00ff00ff00ff00ffull;
  v = (v | (v >> 8)) & 0x0000ffff0000ffffull;
  v = (v | (v >> 16)) & 0x00000000ffffffffull;
  return (uint32_t)v;
}

uint64_t orc_z_encode(uint32_t ix, uint32_t iy) { return zenc(ix, iy); }

/* S1: grid coordinate of a coordinate value. */
static inline double gcoord(double v, double o, double side) { return (v - o) / side; }

/* SPEC.md:143-151 point_to_cell for a batch; dtype 0 = f64 xy, 1 = f32 xy.
 * Returns ORC_DOMAIN and *first_bad = first offending index. */
int orc_point_cells(const orc_grid* g, const void* xy, int32_t dtype, int64_t n, uint32_t* ix, uint32_t* iy,
                    int64_t* first_bad) {
  double side = ldexp(g->extent, -g->level);
  double lim = ldexp(1.0, g->level);
  *first_bad = -1;
  for (int64_t k = 0; k < n; ++k) {
    double x, y;
    if (dtype == 0) { x = ((const double*)xy)[2 * k]; y = ((const double*)xy)[2 * k + 1]; }
    else { x = (double)((const float*)xy)[2 * k]; y = (double)((const float*)xy)[2 * k + 1]; }
    double u = floor(gcoord(x, g->ox, side)), v = floor(gcoord(y, g->oy, side));
    if (!(u >= 0.0 && u < lim && v >= 0.0 && v < lim)) { *first_bad = k; return ORC_DOMAIN; }
    ix[k] = (uint32_t)u; iy[k] = (uint32_t)v;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------ containers */

typedef struct { uint64_t* a; int64_t n, cap; } u64vec;
static int u64push(u64vec* v, uint64_t x) {
  if (v->n == v->cap) {
    int64_t nc = v->cap ? v->cap * 2 : 64;
    uint64_t* na = (uint64_t*)realloc(v->a, (size_t)nc * sizeof(uint64_t));
    if (!na) return ORC_NOMEM;
    v->a = na; v->cap = nc;
  }
  v->a[v->n++] = x;
  return ORC_OK;
}
static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}
typedef struct { int64_t row; double x; } xing;
static int cmp_xing(const void* a, const void* b) {
  const xing* p = (const xing*)a; const xing* q = (const xing*)b;
  if (p->row != q->row) return p->row < q->row ? -1 : 1;
  return p->x < q->x ? -1 : (p->x > q->x);
}

/* per-polygon rasterization state */
typedef struct { int32_t row, c0, c1; } span_t;
typedef struct { double a, lo, hi; int vertical; } aligned_t; /* x=a (vertical) or y=a, extent (lo,hi) */
typedef struct {
  int64_t v0, v1;             /* ring range [r0, r1) */
  int32_t region;
  uint32_t imin, imax, jmin, jmax; /* leaf MBR (inclusive) */
  uint64_t* partial;          /* sorted unique Z codes of PARTIAL leaves */
  uint8_t* kept;              /* per partial leaf: kept as boundary under the mode */
  int64_t npartial;
  span_t* spans; int64_t nspans; /* sorted by (row, c0), disjoint */
  aligned_t* aligned; int64_t naligned;
} poly_t;

struct orc_approx {
  orc_grid g;
  int32_t mode, nregions;
  int64_t npolys;
  double* gx; double* gy;      /* vertex grid coords */
  int64_t* ring_off; int64_t nrings;
  int64_t* poly_ring_off;
  poly_t* polys;
  /* bucket grid over polygons */
  int32_t blevel; uint32_t bside;
  int64_t* boff; int32_t* bpoly;
};
typedef struct orc_approx orc_approx;

/* ------------------------------------------------------------ geometry */

/* S2 fixed formula: y of the (canonical, x-ordered) edge at abscissa c. */
static inline double y_at(double x1, double y1, double x2, double y2, double c) {
  if (c == x1) return y1;
  if (c == x2) return y2;
  double t = (c - x1) * (y2 - y1);
  t = t / (x2 - x1);
  return y1 + t;
}

/* S2: open leaves crossed by segment (x1,y1)-(x2,y2).  Endpoints are ordered
 * lexicographically first so a shared edge yields identical leaves in both
 * neighbouring polygons. */
static int edge_walk(double x1, double y1, double x2, double y2, u64vec* out) {
  if (x2 < x1 || (x2 == x1 && y2 < y1)) { double t = x1; x1 = x2; x2 = t; t = y1; y1 = y2; y2 = t; }
  if (x1 == x2 && y1 == y2) return ORC_OK; /* zero-length edge */
  if (x1 == x2) {                           /* vertical */
    if (x1 == floor(x1)) return ORC_OK;     /* on a grid line: meets no open leaf */
    int64_t i = (int64_t)floor(x1);
    int64_t j0 = (int64_t)floor(y1), j1 = (int64_t)ceil(y2) - 1;
    for (int64_t j = j0; j <= j1; ++j) if (u64push(out, zenc((uint64_t)i, (uint64_t)j))) return ORC_NOMEM;
    return ORC_OK;
  }
  int64_t i0 = (int64_t)floor(x1), i1 = (int64_t)ceil(x2) - 1;
  for (int64_t i = i0; i <= i1; ++i) {
    double xa = x1 > (double)i ? x1 : (double)i;
    double xb = x2 < (double)(i + 1) ? x2 : (double)(i + 1);
    double ya = y_at(x1, y1, x2, y2, xa), yb = y_at(x1, y1, x2, y2, xb);
    double lo = ya < yb ? ya : yb, hi = ya < yb ? yb : ya;
    if (lo == hi) {
      if (lo == floor(lo)) continue; /* horizontal piece on a grid line */
      if (u64push(out, zenc((uint64_t)i, (uint64_t)floor(lo)))) return ORC_NOMEM;
      continue;
    }
    int64_t j0 = (int64_t)floor(lo), j1 = (int64_t)ceil(hi) - 1;
    for (int64_t j = j0; j <= j1; ++j) if (u64push(out, zenc((uint64_t)i, (uint64_t)j))) return ORC_NOMEM;
  }
  return ORC_OK;
}

/* Scanline crossing abscissa of edge with yc, edge ordered so ylo < yhi. */
static inline double x_cross(double xl, double yl, double xh, double yh, double yc) {
  double t = (yc - yl) * (xh - xl);
  t = t / (yh - yl);
  return xl + t;
}

/* SPEC.md:49-57 point_in_polygon, boundary = inside, even-odd
 * over all rings.  Used (in grid units) for the CENTER_SAMPLED keep rule and,
 * in original units, as the exact test of the validator. */
static int pip_rings(const double* X, const double* Y, const int64_t* ring_off, int64_t r0, int64_t r1, double px,
                     double py) {
  int inside = 0;
  for (int64_t r = r0; r < r1; ++r) {
    int64_t a = ring_off[r], b = ring_off[r + 1], m = b - a;
    for (int64_t k = 0; k < m; ++k) {
      double ax = X[a + k], ay = Y[a + k];
      double bx = X[a + (k + 1) % m], by = Y[a + (k + 1) % m];
      /* on-segment (boundary = inside) */
      double minx = ax < bx ? ax : bx, maxx = ax < bx ? bx : ax;
      double miny = ay < by ? ay : by, maxy = ay < by ? by : ay;
      if (px >= minx && px <= maxx && py >= miny && py <= maxy) {
        double cr = (bx - ax) * (py - ay) - (by - ay) * (px - ax);
        if (cr == 0.0) return 1;
      }
      if ((ay > py) != (by > py)) {
        double xl, yl, xh, yh;
        if (ay < by) { xl = ax; yl = ay; xh = bx; yh = by; } else { xl = bx; yl = by; xh = ax; yh = ay; }
        double xc = x_cross(xl, yl, xh, yh, py);
        if (px == xc) return 1;
        if (px < xc) inside = !inside;
      }
    }
  }
  return inside;
}

/* SPEC.md:58-66 distance_to_boundary: min point-segment distance over rings. */
static double dist_rings(const double* X, const double* Y, const int64_t* ring_off, int64_t r0, int64_t r1, double px,
                         double py) {
  double best = INFINITY;
  for (int64_t r = r0; r < r1; ++r) {
    int64_t a = ring_off[r], b = ring_off[r + 1], m = b - a;
    for (int64_t k = 0; k < m; ++k) {
      double ax = X[a + k], ay = Y[a + k];
      double bx = X[a + (k + 1) % m], by = Y[a + (k + 1) % m];
      double dx = bx - ax, dy = by - ay, wx = px - ax, wy = py - ay;
      double L2 = dx * dx + dy * dy, t = 0.0;
      if (L2 > 0.0) { t = (wx * dx + wy * dy) / L2; if (t < 0.0) t = 0.0; if (t > 1.0) t = 1.0; }
      double ex = wx - t * dx, ey = wy - t * dy;
      double d = sqrt(ex * ex + ey * ey);
      if (d < best) best = d;
    }
  }
  return best;
}

int orc_pip(const double* vx, const double* vy, const int64_t* ring_off, int64_t nrings, const double* px,
            const double* py, int64_t n, uint8_t* out) {
  for (int64_t k = 0; k < n; ++k) out[k] = (uint8_t)pip_rings(vx, vy, ring_off, 0, nrings, px[k], py[k]);
  return ORC_OK;
}
int orc_distance(const double* vx, const double* vy, const int64_t* ring_off, int64_t nrings, const double* px,
                 const double* py, int64_t n, double* out) {
  for (int64_t k = 0; k < n; ++k) out[k] = dist_rings(vx, vy, ring_off, 0, nrings, px[k], py[k]);
  return ORC_OK;
}

/* ------------------------------------------------------------- build */

static int64_t lower_u64(const uint64_t* a, int64_t n, uint64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (a[mid] < key) lo = mid + 1; else hi = mid; }
  return lo;
}

static int build_poly(orc_approx* A, int64_t p) {
  poly_t* P = &A->polys[p];
  double lim = ldexp(1.0, A->g.level);
  int64_t r0 = A->poly_ring_off[p], r1 = A->poly_ring_off[p + 1];
  double mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
  u64vec pv = {0, 0, 0};
  int64_t nx = 0, xcap = 64;
  xing* xs = (xing*)malloc((size_t)xcap * sizeof(xing));
  int64_t nal = 0, alcap = 8;
  aligned_t* al = (aligned_t*)malloc((size_t)alcap * sizeof(aligned_t));
  if (!xs || !al) return ORC_NOMEM;
  for (int64_t k = A->ring_off[r0]; k < A->ring_off[r1]; ++k) {
    double x1 = A->gx[k], y1 = A->gy[k];
    if (x1 < mnx) mnx = x1;
    if (x1 > mxx) mxx = x1;
    if (y1 < mny) mny = y1;
    if (y1 > mxy) mxy = y1;
  }
  if (!(mnx >= 0.0 && mny >= 0.0 && mxx <= lim && mxy <= lim)) { free(xs); free(al); return ORC_DOMAIN; }
  for (int64_t r = r0; r < r1; ++r) {
    int64_t a = A->ring_off[r], b = A->ring_off[r + 1], m = b - a;
    for (int64_t k = 0; k < m; ++k) {
      double x1 = A->gx[a + k], y1 = A->gy[a + k];
      double x2 = A->gx[a + (k + 1) % m], y2 = A->gy[a + (k + 1) % m];
      if (edge_walk(x1, y1, x2, y2, &pv)) return ORC_NOMEM;
      /* grid-aligned pieces (S7) */
      if (x1 == x2 && x1 == floor(x1) && y1 != y2) {
        if (nal == alcap) { alcap *= 2; al = (aligned_t*)realloc(al, (size_t)alcap * sizeof(aligned_t)); if (!al) return ORC_NOMEM; }
        al[nal].a = x1; al[nal].lo = y1 < y2 ? y1 : y2; al[nal].hi = y1 < y2 ? y2 : y1; al[nal].vertical = 1; ++nal;
      } else if (y1 == y2 && y1 == floor(y1) && x1 != x2) {
        if (nal == alcap) { alcap *= 2; al = (aligned_t*)realloc(al, (size_t)alcap * sizeof(aligned_t)); if (!al) return ORC_NOMEM; }
        al[nal].a = y1; al[nal].lo = x1 < x2 ? x1 : x2; al[nal].hi = x1 < x2 ? x2 : x1; al[nal].vertical = 0; ++nal;
      }
      /* scanline crossings at row centres j + 0.5 in [ylo, yhi) (S3) */
      if (y1 != y2) {
        double xl, yl, xh, yh;
        if (y1 < y2) { xl = x1; yl = y1; xh = x2; yh = y2; } else { xl = x2; yl = y2; xh = x1; yh = y1; }
        int64_t j0 = (int64_t)ceil(yl - 0.5), j1 = (int64_t)ceil(yh - 0.5) - 1;
        for (int64_t j = j0; j <= j1; ++j) {
          if (nx == xcap) { xcap *= 2; xs = (xing*)realloc(xs, (size_t)xcap * sizeof(xing)); if (!xs) return ORC_NOMEM; }
          xs[nx].row = j; xs[nx].x = x_cross(xl, yl, xh, yh, (double)j + 0.5); ++nx;
        }
      }
    }
  }
  uint32_t top = (uint32_t)(lim - 1.0);
  P->imin = (uint32_t)floor(mnx); P->jmin = (uint32_t)floor(mny);
  P->imax = (uint32_t)floor(mxx); P->jmax = (uint32_t)floor(mxy);
  if (P->imax > top) P->imax = top;
  if (P->jmax > top) P->jmax = top;
  /* PARTIAL leaves: sort + unique */
  qsort(pv.a, (size_t)pv.n, sizeof(uint64_t), cmp_u64);
  int64_t u = 0;
  for (int64_t k = 0; k < pv.n; ++k) if (u == 0 || pv.a[k] != pv.a[u - 1]) pv.a[u++] = pv.a[k];
  P->partial = pv.a; P->npartial = u;
  P->kept = (uint8_t*)malloc((size_t)(u ? u : 1));
  for (int64_t k = 0; k < u; ++k) {
    if (A->mode == MODE_CONSERVATIVE) { P->kept[k] = 1; continue; }
    uint64_t z = pv.a[k];
    double cx = (double)compact1by1(z) + 0.5, cy = (double)compact1by1(z >> 1) + 0.5;
    P->kept[k] = (uint8_t)pip_rings(A->gx, A->gy, A->ring_off, r0, r1, cx, cy);
  }
  /* spans */
  qsort(xs, (size_t)nx, sizeof(xing), cmp_xing);
  P->spans = (span_t*)malloc((size_t)(nx / 2 + 1) * sizeof(span_t));
  int64_t ns = 0;
  for (int64_t k = 0; k + 1 < nx; k += 2) {
    /* crossings come in pairs per row (half-open rule, closed rings) */
    double a = xs[k].x, b = xs[k + 1].x;
    int64_t c0 = (int64_t)ceil(a - 0.5), c1 = (int64_t)floor(b - 0.5);
    if (c0 > c1) continue;
    int32_t row = (int32_t)xs[k].row;
    if (ns > 0 && P->spans[ns - 1].row == row && c0 <= (int64_t)P->spans[ns - 1].c1 + 1) {
      if (c1 > P->spans[ns - 1].c1) P->spans[ns - 1].c1 = (int32_t)c1;
      continue;
    }
    P->spans[ns].row = row; P->spans[ns].c0 = (int32_t)c0; P->spans[ns].c1 = (int32_t)c1; ++ns;
  }
  P->nspans = ns;
  P->aligned = al; P->naligned = nal;
  free(xs);
  return ORC_OK;
}

static inline int in_spans(const poly_t* P, uint32_t i, uint32_t j) {
  int64_t lo = 0, hi = P->nspans;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    const span_t* s = &P->spans[mid];
    if (s->row < (int32_t)j || (s->row == (int32_t)j && s->c0 <= (int32_t)i)) lo = mid + 1; else hi = mid;
  }
  if (lo == 0) return 0;
  const span_t* s = &P->spans[lo - 1];
  return s->row == (int32_t)j && (int32_t)i <= s->c1;
}

/* S2-S4: kind of leaf (i,j) for polygon P. */
static inline int leaf_kind(const poly_t* P, uint32_t i, uint32_t j) {
  if (i < P->imin || i > P->imax || j < P->jmin || j > P->jmax) return KIND_NONE;
  uint64_t z = zenc(i, j);
  int64_t k = lower_u64(P->partial, P->npartial, z);
  if (k < P->npartial && P->partial[k] == z) return P->kept[k] ? KIND_B : KIND_NONE;
  return in_spans(P, i, j) ? KIND_I : KIND_NONE;
}

void orc_free(orc_approx* A);

orc_approx* orc_build(const orc_grid* g, const double* vx, const double* vy, int64_t nverts, const int64_t* ring_off,
                      int64_t nrings, const int64_t* poly_ring_off, int64_t npolys, const int32_t* poly_region,
                      int32_t nregions, int32_t mode, int32_t* status) {
  *status = ORC_OK;
  if (g->level < 0 || g->level > 31 || !(g->extent > 0.0) || (mode != 0 && mode != 1)) { *status = ORC_CONFIG; return NULL; }
  for (int64_t r = 0; r < nrings; ++r) if (ring_off[r + 1] - ring_off[r] < 3) { *status = ORC_GEOMETRY; return NULL; }
  for (int64_t p = 0; p < npolys; ++p) {
    if (poly_ring_off[p + 1] <= poly_ring_off[p]) { *status = ORC_GEOMETRY; return NULL; }
    if (poly_region[p] < 0 || poly_region[p] >= nregions) { *status = ORC_CONFIG; return NULL; }
  }
  for (int64_t k = 0; k < nverts; ++k) if (!isfinite(vx[k]) || !isfinite(vy[k])) { *status = ORC_GEOMETRY; return NULL; }
  orc_approx* A = (orc_approx*)calloc(1, sizeof(orc_approx));
  A->g = *g; A->mode = mode; A->nregions = nregions; A->npolys = npolys; A->nrings = nrings;
  A->gx = (double*)malloc((size_t)(nverts ? nverts : 1) * sizeof(double));
  A->gy = (double*)malloc((size_t)(nverts ? nverts : 1) * sizeof(double));
  A->ring_off = (int64_t*)malloc((size_t)(nrings + 1) * sizeof(int64_t));
  A->poly_ring_off = (int64_t*)malloc((size_t)(npolys + 1) * sizeof(int64_t));
  A->polys = (poly_t*)calloc((size_t)(npolys ? npolys : 1), sizeof(poly_t));
  memcpy(A->ring_off, ring_off, (size_t)(nrings + 1) * sizeof(int64_t));
  memcpy(A->poly_ring_off, poly_ring_off, (size_t)(npolys + 1) * sizeof(int64_t));
  double side = ldexp(g->extent, -g->level);
  for (int64_t k = 0; k < nverts; ++k) { A->gx[k] = gcoord(vx[k], g->ox, side); A->gy[k] = gcoord(vy[k], g->oy, side); }
  for (int64_t p = 0; p < npolys; ++p) {
    /* outer ring must have nonzero area */
    int64_t a = ring_off[poly_ring_off[p]], b = ring_off[poly_ring_off[p] + 1];
    double ar = 0.0;
    for (int64_t k = a; k < b; ++k) { int64_t k2 = (k + 1 < b) ? k + 1 : a; ar += vx[k] * vy[k2] - vx[k2] * vy[k]; }
    if (ar == 0.0) { *status = ORC_GEOMETRY; orc_free(A); return NULL; }
    A->polys[p].region = poly_region[p];
    int st = build_poly(A, p);
    if (st) { *status = st; orc_free(A); return NULL; }
  }
  /* bucket grid: 4^blevel ~ 4 * npolys */
  int bl = 0;
  while (bl < g->level && ((int64_t)1 << (2 * bl)) < 4 * npolys) ++bl;
  A->blevel = bl; A->bside = 1u << bl;
  int sh = g->level - bl;
  int64_t nb = (int64_t)A->bside * A->bside;
  A->boff = (int64_t*)calloc((size_t)nb + 1, sizeof(int64_t));
  for (int64_t p = 0; p < npolys; ++p) {
    poly_t* P = &A->polys[p];
    for (uint32_t by = P->jmin >> sh; by <= (P->jmax >> sh); ++by)
      for (uint32_t bx = P->imin >> sh; bx <= (P->imax >> sh); ++bx) A->boff[(int64_t)by * A->bside + bx + 1]++;
  }
  for (int64_t b = 0; b < nb; ++b) A->boff[b + 1] += A->boff[b];
  A->bpoly = (int32_t*)malloc((size_t)(A->boff[nb] ? A->boff[nb] : 1) * sizeof(int32_t));
  int64_t* fill = (int64_t*)malloc((size_t)nb * sizeof(int64_t));
  memcpy(fill, A->boff, (size_t)nb * sizeof(int64_t));
  for (int64_t p = 0; p < npolys; ++p) {
    poly_t* P = &A->polys[p];
    for (uint32_t by = P->jmin >> sh; by <= (P->jmax >> sh); ++by)
      for (uint32_t bx = P->imin >> sh; bx <= (P->imax >> sh); ++bx) A->bpoly[fill[(int64_t)by * A->bside + bx]++] = (int32_t)p;
  }
  free(fill);
  return A;
}

void orc_free(orc_approx* A) {
  if (!A) return;
  for (int64_t p = 0; p < A->npolys; ++p) {
    free(A->polys[p].partial); free(A->polys[p].kept); free(A->polys[p].spans); free(A->polys[p].aligned);
  }
  free(A->polys); free(A->gx); free(A->gy); free(A->ring_off); free(A->poly_ring_off); free(A->boff); free(A->bpoly);
  free(A);
}

/* ------------------------------------------------------- lookup / join */

#define MAXOWN 256
/* S5/S6: owner set of leaf (i,j): regions + kinds, I dominating B per region.
 * Returns count; entries sorted by region. */
static int leaf_owners(const orc_approx* A, uint32_t i, uint32_t j, int32_t* reg, uint8_t* kind) {
  int sh = A->g.level - A->blevel;
  int64_t b = (int64_t)(j >> sh) * A->bside + (i >> sh);
  int n = 0;
  for (int64_t t = A->boff[b]; t < A->boff[b + 1]; ++t) {
    const poly_t* P = &A->polys[A->bpoly[t]];
    int k = leaf_kind(P, i, j);
    if (k == KIND_NONE) continue;
    int q = 0;
    while (q < n && reg[q] != P->region) ++q;
    if (q < n) { if (k == KIND_I) kind[q] = KIND_I; continue; }
    if (n == MAXOWN) return -1;
    /* insertion sort by region */
    int pos = n;
    while (pos > 0 && reg[pos - 1] > P->region) { reg[pos] = reg[pos - 1]; kind[pos] = kind[pos - 1]; --pos; }
    reg[pos] = P->region; kind[pos] = (uint8_t)k; ++n;
  }
  return n;
}

/* act_lookup restated: owners of each point's leaf, CSR. */
int orc_lookup(const orc_approx* A, const void* xy, int32_t dtype, int64_t n, int64_t* off /*n+1*/, int32_t* reg_out,
               uint8_t* kind_out, int64_t cap, int64_t* first_bad) {
  double side = ldexp(A->g.extent, -A->g.level), lim = ldexp(1.0, A->g.level);
  int32_t reg[MAXOWN]; uint8_t kd[MAXOWN];
  int64_t w = 0; off[0] = 0; *first_bad = -1;
  for (int64_t k = 0; k < n; ++k) {
    double x, y;
    if (dtype == 0) { x = ((const double*)xy)[2 * k]; y = ((const double*)xy)[2 * k + 1]; }
    else { x = (double)((const float*)xy)[2 * k]; y = (double)((const float*)xy)[2 * k + 1]; }
    double u = floor(gcoord(x, A->g.ox, side)), v = floor(gcoord(y, A->g.oy, side));
    if (!(u >= 0.0 && u < lim && v >= 0.0 && v < lim)) { *first_bad = k; return ORC_DOMAIN; }
    int c = leaf_owners(A, (uint32_t)u, (uint32_t)v, reg, kd);
    if (c < 0) return ORC_CAPACITY;
    for (int q = 0; q < c; ++q) {
      if (w >= cap) return ORC_SHAPE;
      reg_out[w] = reg[q]; kind_out[w] = kd[q]; ++w;
    }
    off[k + 1] = w;
  }
  return ORC_OK;
}

typedef struct {
  const orc_approx* A; const void* xy; int32_t dtype; const float* attr;
  int64_t k0, k1; int64_t* cnt; double* sum; int64_t bad; int status;
} job_t;

static void* join_worker(void* arg) {
  job_t* J = (job_t*)arg;
  const orc_approx* A = J->A;
  double side = ldexp(A->g.extent, -A->g.level), lim = ldexp(1.0, A->g.level);
  int32_t reg[MAXOWN]; uint8_t kd[MAXOWN];
  for (int64_t k = J->k0; k < J->k1; ++k) {
    double x, y;
    if (J->dtype == 0) { x = ((const double*)J->xy)[2 * k]; y = ((const double*)J->xy)[2 * k + 1]; }
    else { x = (double)((const float*)J->xy)[2 * k]; y = (double)((const float*)J->xy)[2 * k + 1]; }
    double u = floor(gcoord(x, A->g.ox, side)), v = floor(gcoord(y, A->g.oy, side));
    if (!(u >= 0.0 && u < lim && v >= 0.0 && v < lim)) { J->bad = k; J->status = ORC_DOMAIN; return NULL; }
    int c = leaf_owners(A, (uint32_t)u, (uint32_t)v, reg, kd);
    if (c < 0) { J->status = ORC_CAPACITY; return NULL; }
    double w = J->attr ? (double)J->attr[k] : 0.0;
    for (int q = 0; q < c; ++q) {
      int64_t r = reg[q];
      J->cnt[2 * r] += 1; J->sum[2 * r] += w;
      if (kd[q] == KIND_B) { J->cnt[2 * r + 1] += 1; J->sum[2 * r + 1] += w; }
    }
  }
  return NULL;
}

/* join_act restated: per region alpha/beta COUNT and SUM.
 * cnt[2r] = alpha count, cnt[2r+1] = beta count; sum likewise (float64).
 * Points split into nthreads contiguous chunks; partials combined in chunk
 * order (deterministic for a given nthreads). */
int orc_join(const orc_approx* A, const void* xy, int32_t dtype, int64_t n, const float* attr, int64_t* cnt,
             double* sum, int64_t* first_bad, int32_t nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (n < 4096 * nthreads) nthreads = 1;
  int32_t R = A->nregions;
  job_t* jobs = (job_t*)calloc((size_t)nthreads, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].A = A; jobs[t].xy = xy; jobs[t].dtype = dtype; jobs[t].attr = attr;
    jobs[t].k0 = n * t / nthreads; jobs[t].k1 = n * (t + 1) / nthreads;
    jobs[t].cnt = (int64_t*)calloc((size_t)2 * R + 1, sizeof(int64_t));
    jobs[t].sum = (double*)calloc((size_t)2 * R + 1, sizeof(double));
    jobs[t].bad = -1;
    if (nthreads == 1) join_worker(&jobs[t]); else pthread_create(&th[t], NULL, join_worker, &jobs[t]);
  }
  int status = ORC_OK;
  *first_bad = -1;
  for (int t = 0; t < nthreads; ++t) {
    if (nthreads > 1) pthread_join(th[t], NULL);
  }
  for (int t = 0; t < nthreads; ++t) {
    if (jobs[t].status && status == ORC_OK) { status = jobs[t].status; *first_bad = jobs[t].bad; }
  }
  if (status == ORC_OK) {
    memset(cnt, 0, (size_t)2 * R * sizeof(int64_t));
    memset(sum, 0, (size_t)2 * R * sizeof(double));
    for (int t = 0; t < nthreads; ++t)
      for (int64_t q = 0; q < 2 * (int64_t)R; ++q) { cnt[q] += jobs[t].cnt[q]; sum[q] += jobs[t].sum[q]; }
  }
  for (int t = 0; t < nthreads; ++t) { free(jobs[t].cnt); free(jobs[t].sum); }
  free(jobs); free(th);
  return status;
}

/* ------------------------------------------------------------ exports */

int64_t orc_npolys(const orc_approx* A) { return A->npolys; }

/* PARTIAL leaves of polygon p (Z codes) and kept flags; two-call pattern. */
int64_t orc_partial_leaves(const orc_approx* A, int64_t p, uint64_t* codes, uint8_t* kept) {
  const poly_t* P = &A->polys[p];
  if (codes) { memcpy(codes, P->partial, (size_t)P->npartial * sizeof(uint64_t)); memcpy(kept, P->kept, (size_t)P->npartial); }
  return P->npartial;
}

/* Interior spans of polygon p: rows, c0, c1 (inclusive), before PARTIAL
 * exclusion (a leaf in a span that is PARTIAL is boundary, not interior). */
int64_t orc_spans(const orc_approx* A, int64_t p, int32_t* rows, int32_t* c0, int32_t* c1) {
  const poly_t* P = &A->polys[p];
  if (rows) for (int64_t k = 0; k < P->nspans; ++k) { rows[k] = P->spans[k].row; c0[k] = P->spans[k].c0; c1[k] = P->spans[k].c1; }
  return P->nspans;
}

/* leaf kinds for explicit leaves of polygon p (KIND_NONE/I/B) */
int orc_leaf_kinds(const orc_approx* A, int64_t p, const uint32_t* i, const uint32_t* j, int64_t n, uint8_t* out) {
  for (int64_t k = 0; k < n; ++k) out[k] = (uint8_t)leaf_kind(&A->polys[p], i[k], j[k]);
  return ORC_OK;
}

/* S7 hierarchical covering of polygon p: (level, code, kind) cells. */
typedef struct { u64vec lv; u64vec code; u64vec kind; } cellvec;

static int block_aligned_cut(const poly_t* P, double bx0, double by0, double bx1, double by1) {
  for (int64_t k = 0; k < P->naligned; ++k) {
    const aligned_t* a = &P->aligned[k];
    if (a->vertical) {
      if (bx0 < a->a && a->a < bx1) {
        double lo = a->lo > by0 ? a->lo : by0, hi = a->hi < by1 ? a->hi : by1;
        if (lo < hi) return 1;
      }
    } else {
      if (by0 < a->a && a->a < by1) {
        double lo = a->lo > bx0 ? a->lo : bx0, hi = a->hi < bx1 ? a->hi : bx1;
        if (lo < hi) return 1;
      }
    }
  }
  return 0;
}

static int hier_visit(const orc_approx* A, const poly_t* P, int lvl, uint64_t code, cellvec* out) {
  int L = A->g.level;
  int d = L - lvl;
  uint32_t bi = compact1by1(code) << d, bj = compact1by1(code >> 1) << d;
  uint32_t bw = 1u << d;
  /* outside the polygon's leaf MBR: all OUTSIDE */
  if (bi > P->imax || bj > P->jmax || bi + (bw - 1) < P->imin || bj + (bw - 1) < P->jmin) return ORC_OK;
  if (d == 0) {
    int k = leaf_kind(P, bi, bj);
    if (k != KIND_NONE) { u64push(&out->lv, (uint64_t)lvl); u64push(&out->code, code); u64push(&out->kind, (uint64_t)k); }
    return ORC_OK;
  }
  uint64_t lo = code << (2 * d), hi = (code + 1) << (2 * d);
  int64_t q = lower_u64(P->partial, P->npartial, lo);
  int mixed = (q < P->npartial && P->partial[q] < hi);
  if (!mixed) mixed = block_aligned_cut(P, (double)bi, (double)bj, (double)bi + (double)bw, (double)bj + (double)bw);
  if (!mixed) {
    if (in_spans(P, bi, bj)) { u64push(&out->lv, (uint64_t)lvl); u64push(&out->code, code); u64push(&out->kind, KIND_I); }
    return ORC_OK;
  }
  for (uint64_t c = 0; c < 4; ++c) { int st = hier_visit(A, P, lvl + 1, code * 4 + c, out); if (st) return st; }
  return ORC_OK;
}

/* Returns number of cells; fills when arrays non-NULL and cap suffices. */
int64_t orc_hier_cells(const orc_approx* A, int64_t p, int32_t* level, uint64_t* code, uint8_t* kind, int64_t cap) {
  cellvec cv; memset(&cv, 0, sizeof(cv));
  hier_visit(A, &A->polys[p], 0, 0, &cv);
  int64_t n = cv.lv.n;
  if (level && n <= cap) for (int64_t k = 0; k < n; ++k) { level[k] = (int32_t)cv.lv.a[k]; code[k] = cv.code.a[k]; kind[k] = (uint8_t)cv.kind.a[k]; }
  free(cv.lv.a); free(cv.code.a); free(cv.kind.a);
  return n;
}
