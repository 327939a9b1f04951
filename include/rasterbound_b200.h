/*
 * rasterbound_b200.h -- C-ABI of the B200-native epsilon-bounded
 * point-polygon aggregation engine (librasterbound_b200.so).
 *
 * The reference (`rasterbound`, SPEC.md) is a Python package with no FFI; this
 * header is the boundary its Python API (rasterbound.{grid,raster,act,query})
 * binds through ctypes (INTEGRATION.md shows the binding).  Each entry point
 * names the reference operation it replaces.
 *
 * Conventions
 *  - Plain C types only; no exceptions cross the boundary.  Every function
 *    returns an rb status; rb_last_error() gives a thread-local message.
 *  - Status codes map 1:1 onto /root/reference/pkg/src/rasterbound/errors.py.
 *  - "device" pointers are CUDA global-memory pointers (e.g. torch tensors);
 *    "host" pointers are ordinary CPU memory.  `stream` is a cudaStream_t
 *    (NULL = legacy default stream).  rb_point_pass / rb_lookup are
 *    stream-ordered and never synchronise the host.
 *  - An rb_approx is immutable after rb_approx_build returns; concurrent
 *    rb_point_pass / rb_lookup calls on one handle are safe.
 */
#ifndef RASTERBOUND_B200_H
#define RASTERBOUND_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (errors.py:8-37) */
#define RB_OK 0
#define RB_GEOMETRY_ERROR (-1)        /* errors.py:12 GeometryError */
#define RB_DOMAIN_ERROR (-2)          /* errors.py:16 DomainError */
#define RB_CAPACITY_ERROR (-3)        /* errors.py:20 CapacityError */
#define RB_CONFIG_ERROR (-4)          /* errors.py:24 ConfigError */
#define RB_SCHEMA_ERROR (-5)          /* errors.py:28 SchemaError */
#define RB_SHAPE_ERROR (-6)           /* errors.py:32 ShapeError */
#define RB_UNSUPPORTED_TRANSFORM (-7) /* errors.py:36 UnsupportedTransform */
#define RB_CUDA_ERROR (-100)          /* device / driver failure */

/* RasterMode */
#define RB_MODE_CONSERVATIVE 0
#define RB_MODE_CENTER_SAMPLED 1

/* cell-index layouts (north star subsystem 2) */
#define RB_LAYOUT_DENSE 0 /* dense leaf grid of owner values (uniform raster)   */
#define RB_LAYOUT_TRIE 1  /* multi-level radix table (ACT, hierarchical raster) */
#define RB_LAYOUT_KEYS 2  /* sorted 64-bit cell keys (disjoint covering cells, leaf-level start keys)
                           with a radix table over the top key bits: radix + binary search */
#define RB_LAYOUT_PACKED 3 /* radix table whose last level is palette-packed: each 4x4-leaf block is 16
                            bytes (three owner values + 16 two-bit palette indices).  L - root_level in
                            [2, 5]: the blocks sit right below the root; in [6, 8] (default root_level
                            L - 6): one u32 node level, then packed nodes of 16 x 16 leaves.  C4: a 1.2 GB
                            index against 4.5 GB for RB_LAYOUT_TRIE at the same speed */

/* point coordinate storage */
#define RB_XY_F64 0 /* interleaved float64 (x,y) */
#define RB_XY_F32 1 /* interleaved float32 (x,y), promoted exactly to float64 */

/* owner-value encoding returned by rb_lookup (one uint32 per point):
 *   0                       no owner
 *   v in [1, 2^18)          single owner: region = (v-1)>>1, boundary = (v-1)&1
 *                           (region sets are limited to n_regions < 2^17: RB_CAPACITY_ERROR beyond)
 *   RB_VALUE_LIST | off     several owners: pool[off] = k, pool[off+1..k] = (region<<1)|boundary */
#define RB_VALUE_LIST 0x40000000u
#define RB_VALUE_PAYLOAD 0x3fffffffu

/* GridConfig */
typedef struct rb_grid {
  double origin_x, origin_y;
  double extent;     /* side of the square domain */
  int32_t max_level; /* L in [0, 31] */
} rb_grid;

/* Polygon set in CSR form (device pointers).  Ring 0 of every polygon is the
 * outer ring, further rings are holes; a region may own
 * several polygons (multi-polygon). */
typedef struct rb_polygons {
  const double* vx;
  const double* vy;
  int64_t n_vertices;
  const int64_t* ring_off; /* [n_rings+1] vertex offsets */
  int64_t n_rings;
  const int64_t* poly_ring_off; /* [n_polygons+1] ring offsets */
  int64_t n_polygons;
  const int32_t* poly_region; /* [n_polygons] region index in [0, n_regions) */
  int32_t n_regions;
} rb_polygons;

typedef struct rb_build_opts {
  int32_t mode;        /* RB_MODE_* */
  int32_t layout;      /* RB_LAYOUT_* */
  int32_t radix_width; /* ACT bits per node: 2, 4, 8; default 8 */
  int32_t root_level;  /* TRIE / PACKED root table level; -1 = automatic (TRIE: min(L, 12); PACKED: L - 6) */
  int32_t keep_cells;  /* keep per-polygon covering cells for export */
} rb_build_opts;

typedef struct rb_stats {
  int64_t n_partial_leaves;   /* (polygon, leaf) pairs whose open leaf meets the boundary */
  int64_t n_interior_cells;   /* hierarchical interior cells over all polygons */
  int64_t n_boundary_cells;   /* kept boundary leaves over all polygons */
  int64_t n_uniform_interior; /* interior leaves after expansion to level L */
  int64_t n_positions;        /* disjoint indexed cells after overlay */
  int64_t n_multi_owner;      /* positions with more than one owner */
  int64_t n_nodes;            /* TRIE nodes below the root table */
  int64_t index_bytes;        /* root + nodes + owner pool */
  int32_t root_level;
  int32_t node_levels; /* quad levels per node (radix_width / 2) */
  int32_t n_regions;
  int32_t max_level;
  double build_ms;
  int32_t max_hot; /* hot slots rb_approx_set_hot accepts for this region count (4095 .. 16383) */
  int32_t n_hot;   /* hot slots set */
} rb_stats;

typedef struct rb_approx rb_approx;

int32_t rb_version(void);
const char* rb_last_error(void);

/* grid.level_for_bound */
int rb_level_for_bound(double extent, double epsilon, int32_t* level_out);

/* raster.rasterize_hierarchical/uniform for a region set + act.act_build
 * (SPEC.md:216-233, 276-284).  Synchronises `stream` (sizes come back to the
 * host).  Errors: GeometryError (ring < 3 vertices, NaN, zero area),
 * DomainError (vertex outside the domain), CapacityError, ConfigError. */
int rb_approx_build(const rb_grid* grid, const rb_polygons* polys, const rb_build_opts* opts, void* stream,
                    rb_approx** out);
/* act.act_build from explicit coverings: device arrays of
 * n_cells cells (covering index, level <= L, Z code at that level, kind
 * 1 = interior / 2 = boundary); covering c belongs to region cov_region[c].
 * Duplicate cells are idempotent (set semantics). */
int rb_index_from_cells(const rb_grid* grid, int64_t n_cells, const int32_t* cov, const uint8_t* level,
                        const uint64_t* code, const uint8_t* kind, const int32_t* cov_region, int64_t n_cov,
                        int32_t n_regions, const rb_build_opts* opts, void* stream, rb_approx** out);
int rb_approx_stats(const rb_approx* a, rb_stats* out);
/* Mark frequently hit regions (device or host int32 array) whose
 * alpha COUNT/SUM the point pass privatises in shared memory when the full
 * per-region histogram does not fit there (large region sets, e.g. 40,000
 * census blocks).  Results are unchanged.  At most rb_stats.max_hot regions: 2^(30 - b) - 1 (capped at
 * 16383) where b = max(16, bit length of 2 * n_regions) is the width of the owner codes.  Rewrites the
 * index's owner values in place, once (a second call is RB_CONFIG_ERROR): call it before, not during,
 * concurrent point passes (the Python layer does so under a lock on the first pass). */
int rb_approx_set_hot(rb_approx* a, const int32_t* regions, int32_t n_hot, void* stream);
void rb_approx_free(rb_approx* a);

/* query.join_act point loop: per region alpha/beta COUNT and
 * SUM over n points.  cnt_out: device int64 [n_regions*2] (alpha, beta);
 * sum_out: device float64 [n_regions*2]; attr: device float32 [n] or NULL.
 * accumulate=0 overwrites the outputs, 1 adds to them.  first_bad: device
 * int64 [1], set to the smallest out-of-domain / NaN point index (or left at
 * INT64_MAX); the caller raises DomainError.  Never syncs. */
int rb_point_pass(const rb_approx* a, const void* xy, int32_t xy_dtype, int64_t n, const float* attr,
                  int64_t* cnt_out, double* sum_out, int64_t* first_bad, int32_t accumulate, void* stream);

/* Same as rb_point_pass on HOST buffers: pinned staging, chunked H2D copies
 * overlapped with the point pass, results copied back to host; synchronous.
 * The end-to-end entry a CPU caller of the reference would bind. */
int rb_join_host(const rb_approx* a, const void* xy_host, int32_t xy_dtype, int64_t n, const float* attr_host,
                 int64_t* cnt_host, double* sum_host, int64_t* first_bad_host);

/* act.act_lookup: owner value per point (encoding above). */
int rb_lookup(const rb_approx* a, const void* xy, int32_t xy_dtype, int64_t n, uint32_t* value_out,
              int64_t* first_bad, void* stream);
/* owner-list pool used by RB_VALUE_LIST values: *n = length; when dst is not
 * NULL, copies the pool to dst (host or device memory, synchronous). */
int rb_owner_pool(const rb_approx* a, uint32_t* dst, int64_t* n);

/* grid.point_to_cell for a batch: leaf column/row. */
int rb_point_cells(const rb_grid* grid, const void* xy, int32_t xy_dtype, int64_t n, uint32_t* ix, uint32_t* iy,
                   int64_t* first_bad, void* stream);

/* Covering export (RasterApprox) -- requires keep_cells.
 * Two-call pattern: pass NULL arrays to get *n.  Device arrays, sorted by
 * (polygon, level-L start code, level).  kind: 1 = interior, 2 = boundary. */
int rb_approx_cells(const rb_approx* a, int64_t* n, int32_t* poly, int32_t* level, uint64_t* code, uint8_t* kind,
                    void* stream);
/* PARTIAL leaves (polygon, Z code, kept flag), sorted by (polygon, code). */
int rb_approx_partial(const rb_approx* a, int64_t* n, int32_t* poly, uint64_t* code, uint8_t* kept, void* stream);

/* geometry.point_in_polygon / distance_to_boundary on the
 * GPU, for the epsilon validator: point k is tested against polygon
 * poly_of_point[k] of `polys` (original coordinates). */
int rb_exact_pip(const rb_polygons* polys, const double* px, const double* py, const int32_t* poly_of_point, int64_t n,
                 uint8_t* inside_out, void* stream);
int rb_exact_distance(const rb_polygons* polys, const double* px, const double* py, const int32_t* poly_of_point,
                      int64_t n, double* dist_out, void* stream);

/* ---- point-side access path: pointindex + join_pointindex (SPEC.md:313-382,
 * 491-499).  The reference has no FFI for these either; they
 * replace the Python operations named below. */
typedef struct rb_lps rb_lps; /* pointindex.LinearizedPointSet */
typedef struct rb_rs rb_rs;   /* pointindex.RadixSplineIndex */

/* pointindex.lps_build: leaf Z codes (grid level L) of n
 * device points sorted with their permutation (stable: equal codes keep point
 * order), float64 prefix sums (n + 1 entries, prefix[0] = 0) of n_attr device
 * float32 attribute arrays in sorted order.  Synchronous.  An out-of-domain or
 * NaN point gives RB_DOMAIN_ERROR with its index in *first_bad (host). */
int rb_lps_build(const rb_grid* grid, const void* xy, int32_t xy_dtype, int64_t n, const float* const* attrs,
                 int32_t n_attr, void* stream, rb_lps** out, int64_t* first_bad);
/* device views: codes u64 [n], perm i64 [n], prefix f64 [n_attr][n + 1] */
int rb_lps_info(const rb_lps* lps, int64_t* n, const uint64_t** codes, const int64_t** perm, const double** prefix,
                int32_t* n_attr);
void rb_lps_free(rb_lps* lps);

/* point index file load: a LinearizedPointSet from its arrays
 * (host or device memory; copied). */
int rb_lps_from_arrays(const rb_grid* grid, int64_t n, const uint64_t* codes, const int64_t* perm, const double* prefix,
                       int32_t n_attr, void* stream, rb_lps** out);

/* pointindex.rs_build: RadixSpline over the distinct-key
 * CDF of the codes -- spline knots with interpolation error <= max_error at
 * every stored key, radix table over the top radix_bits of the 2L-bit code
 * space.  radix_bits > 2L (or > 30) is RB_CONFIG_ERROR.  Synchronous. */
int rb_rs_build(const rb_lps* lps, int32_t radix_bits, int32_t max_error, void* stream, rb_rs** out);
/* device views: knot keys u64 / positions i64 [n_knots], radix table u32 [2^radix_bits + 1] */
int rb_rs_info(const rb_rs* rs, int64_t* n_knots, const uint64_t** keys, const int64_t** pos, const uint32_t** table,
               int32_t* radix_bits, int32_t* shift);
void rb_rs_free(rb_rs* rs);
/* RadixSpline from stored knots and radix table (host or device; copied) */
int rb_rs_from_arrays(const rb_lps* lps, int32_t radix_bits, int32_t max_error, int64_t n_knots, const uint64_t* keys,
                      const int64_t* pos, const uint32_t* table, void* stream, rb_rs** out);

/* pointindex.bounds_lookup, batched: for m intervals
 * [lo, hi) of level-L codes (device u64), lo_pos / hi_pos (device i64) = first
 * sorted position with code >= lo / >= hi.  rs may be NULL (binary search);
 * with rs the result is identical.  Stream-ordered. */
int rb_bounds_lookup(const rb_lps* lps, const rb_rs* rs, const uint64_t* lo, const uint64_t* hi, int64_t m,
                     int64_t* lo_pos, int64_t* hi_pos, void* stream);

/* query.join_pointindex over pointindex.range_aggregate
 * (SPEC.md:355-363): covering cells (device arrays, grouped by region: region
 * ids non-decreasing; level, Z code at that level, kind 1 = interior /
 * 2 = boundary) -> per region alpha/beta COUNT (device int64 [n_regions*2]) and
 * SUM of prefix attribute attr_idx (device float64 [n_regions*2]; attr_idx < 0:
 * sums left 0).  Cells of one region must be disjoint.  Deterministic;
 * stream-ordered (no host synchronisation). */
int rb_join_pointindex(const rb_lps* lps, const rb_rs* rs, int64_t n_cells, const int32_t* region,
                       const int32_t* level, const uint64_t* code, const uint8_t* kind, int32_t n_regions,
                       int32_t attr_idx, int64_t* cnt_out, double* sum_out, void* stream);

/* ---- canvas algebra (section 4) and the Bounded
 * Raster Join plan.  A canvas tile is a dense row-major
 * 2^level x 2^level block of the level-L leaf grid at pixel offset (x0, y0);
 * pixel (ix, iy) is leaf z_encode(ix, iy, L).  Caller-owned
 * device channels: */
typedef struct rb_canvas_desc {
  int32_t level;  /* tile side 2^level pixels (<= 16) */
  int64_t x0, y0; /* pixel offset of the tile in the level-L grid */
  int32_t n_sum;  /* SUM channels */
  int64_t* count; /* [2^(2 level)] point count */
  double* sums;   /* [n_sum][2^(2 level)] */
  int32_t* region; /* [2^(2 level)] region id, -1 = none */
  uint8_t* flags;  /* [2^(2 level)] bit 0 non-empty, bit 1 boundary cell */
} rb_canvas_desc;

#define RB_BLEND_SUM 0
#define RB_BLEND_OVERWRITE 1
#define RB_BLEND_MAX 2
#define RB_MASK_NONEMPTY 0
#define RB_MASK_REGION_EQ 1     /* arg = region id */
#define RB_MASK_BOUNDARY_ONLY 2
#define RB_MASK_COUNT_GT 3      /* arg = threshold */
#define RB_MASK_COVERED_BY 4    /* by = region canvas: keep pixels it covers (inherit its boundary flag) */
#define RB_MASK_BOUNDARY_OF 5   /* by = region canvas: keep pixels on its boundary cells */

int rb_canvas_clear(rb_canvas_desc* c, void* stream);
/* canvas.render_points: per pixel COUNT and the first n_sum
 * prefix attributes of the point index (exact per-pixel reductions of the
 * sorted points, deterministic); out-of-tile points are skipped. */
int rb_canvas_render_points(const rb_lps* lps, rb_canvas_desc* out, void* stream);
/* canvas.render_polygon from a region's covering cells
 * (device arrays: level, code at that level, kind 1/2): every leaf pixel of a
 * cell gets region_id, the non-empty flag, and the boundary flag for kind 2.
 * clear = 1 empties the tile first. */
int rb_canvas_render_cells(int64_t n_cells, const int32_t* level, const uint64_t* code, const uint8_t* kind, int32_t L,
                           int32_t region_id, int32_t clear, rb_canvas_desc* out, void* stream);
/* canvas.blend: pixel-wise fn; empty (.) x = x. */
int rb_canvas_blend(const rb_canvas_desc* a, const rb_canvas_desc* b, int32_t fn, rb_canvas_desc* out, void* stream);
/* canvas.mask: pixels failing the predicate become empty. */
int rb_canvas_mask(const rb_canvas_desc* a, int32_t pred, int64_t arg, const rb_canvas_desc* by, rb_canvas_desc* out,
                   void* stream);
/* canvas.affine: integer translation (dx, dy) then axis
 * flips; pixels mapped outside drop.  out must not alias a.  Non-integer
 * transforms are rejected by the caller (UnsupportedTransform). */
int rb_canvas_affine(const rb_canvas_desc* a, int64_t dx, int64_t dy, int32_t flip_x, int32_t flip_y,
                     rb_canvas_desc* out, void* stream);
/* reduce over non-empty pixels: cnt_out (device int64 [2]: all, boundary
 * pixels), sum_out (device float64 [n_sum][2]).  Fixed-order, deterministic. */
int rb_canvas_reduce(const rb_canvas_desc* a, int64_t* cnt_out, double* sum_out, void* stream);

/* The complete epsilon validator (K5): for EVERY point, the
 * approximate owner regions (index lookup) against the exact owner regions
 * (point_in_polygon over the candidate polygons of its bucket: a uniform
 * n_buckets_side^2 grid of side bucket_side at (bucket_x0, bucket_y0), CSR
 * lists bucket_off [n^2+1] / bucket_poly of the polygons whose MBR expanded by
 * epsilon meets the bucket; poly_mbr = device f64 [n_polygons][4] xmin ymin
 * xmax ymax).  Each region in only one of the two sets is a mismatch whose
 * distance to the region's boundary must be <= epsilon.  out6 (host) = points,
 * mismatched points, false positives, false negatives, violations (distance >
 * epsilon), owner-set overflows; *max_dist (host) = largest mismatch distance.
 * All polygon and bucket arrays are device arrays.  Synchronous. */
int rb_validate_full(const rb_approx* a, const rb_polygons* polys, const double* poly_mbr, const int32_t* bucket_off,
                     const int32_t* bucket_poly, int32_t n_buckets_side, double bucket_x0, double bucket_y0,
                     double bucket_side, const void* xy, int32_t xy_dtype, int64_t n, double epsilon, int64_t* out6,
                     double* max_dist, void* stream);

/* Instrumentation (benchmarks): op 1 = reset counters and enable CUDA-event
 * timing of the point-pass main kernel, op 2 = reset and disable, op 0 = read
 * (synchronises the recorded events): launches of this library's point-pass
 * kernels since the reset, number of timed main-kernel launches and their
 * summed device time in ms. */
int rb_instrument(int32_t op, int64_t* launches, int64_t* timed_launches, double* timed_ms);

#ifdef __cplusplus
}
#endif
#endif /* RASTERBOUND_B200_H */
