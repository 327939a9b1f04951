// rb_internal.cuh -- shared device helpers and the rb_approx handle.
//
// Geometry predicates here restate SPEC.md's semantics with the SAME float64
// operation order as oracle/rb_oracle.c (the library is compiled with
// --fmad=false so no multiply-add is contracted); that is what makes COUNT
// parity bit-exact by construction.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/rasterbound_b200.h"

#define RB_KIND_NONE 0
#define RB_KIND_I 1
#define RB_KIND_B 2

// TRIE slot tag for "child node" (never returned by rb_lookup).
#define RB_VALUE_NODE 0x80000000u
// Hot-slot annotation (rb_approx_set_hot): bits 18..29 of a single-owner
// value / owner-list entry carry (hot slot + 1); stripped by rb_lookup and
// rb_owner_pool.  Owner-list count words carry RB_POOL_COUNT_FLAG.
#define RB_HOT_SHIFT 18
#define RB_HOT_BITS 0xfffu
#define RB_CODE_MASK 0x3ffffu
#define RB_POOL_COUNT_FLAG 0x80000000u
#define RB_MAX_HOT 4095
#define RB_MAX_HOT_CAP 16383  // hot slots with narrower owner codes (fewer regions), rb_approx::set_code_format
// single owner codes ((region << 1) | boundary) + 1 must fit RB_CODE_MASK
#define RB_MAX_REGIONS (1 << 17)

namespace rb {

void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define RB_CUDA(call)                                   \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return rb::cuda_fail(_e, #call); \
  } while (0)

// ------------------------------------------------------------------ grid
struct GridD {
  double ox, oy, side;
  double lim;  // 2^L
  int L;
};

__host__ __device__ inline uint64_t part1by1(uint64_t v) {
  v &= 0xffffffffull;
  v = (v | (v << 16)) & 0x0000ffff0000ffffull;
  v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
  v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}
__host__ __device__ inline uint64_t zenc(uint64_t ix, uint64_t iy) { return part1by1(ix) | (part1by1(iy) << 1); }
__host__ __device__ inline uint32_t compact1by1(uint64_t v) {
  v &= 0x5555555555555555ull;
  v = (v | (v >> 1)) & 0x3333333333333333ull;
  v = (v | (v >> 2)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v >> 4)) & 0x00ff00ff00ff00ffull;
  v = (v | (v >> 8)) & 0x0000ffff0000ffffull;
  v = (v | (v >> 16)) & 0x00000000ffffffffull;
  return (uint32_t)v;
}

// S1: grid coordinate, correctly rounded division.
__device__ __forceinline__ double gcoord(double v, double o, double side) { return __ddiv_rn(__dsub_rn(v, o), side); }

// floor(RN((v - o) / side)) without a division on the common path: the
// product with RN(1/side) is within 4e-16 relative of the quotient, so unless
// it lies within 2^-20 of an integer its floor is the floor of the quotient;
// otherwise fall back to the exact division (bit-identical to the oracle).
__device__ __forceinline__ double cell_floor(double v, double o, double side, double inv_side) {
  double d = __dsub_rn(v, o);
  double q = __dmul_rn(d, inv_side);
  double f = floor(q);
  double fr = __dsub_rn(q, f);
  if (fabs(__dsub_rn(fr, 0.5)) > 0.4999990463256836) f = floor(__ddiv_rn(d, side));
  return f;
}

// S2 fixed formula (oracle y_at)
__host__ __device__ inline double y_at(double x1, double y1, double x2, double y2, double c) {
  if (c == x1) return y1;
  if (c == x2) return y2;
#ifdef __CUDA_ARCH__
  double t = __dmul_rn(__dsub_rn(c, x1), __dsub_rn(y2, y1));
  t = __ddiv_rn(t, __dsub_rn(x2, x1));
  return __dadd_rn(y1, t);
#else
  double t = (c - x1) * (y2 - y1);
  t = t / (x2 - x1);
  return y1 + t;
#endif
}

// scanline crossing abscissa (oracle x_cross), edge ordered yl < yh
__host__ __device__ inline double x_cross(double xl, double yl, double xh, double yh, double yc) {
#ifdef __CUDA_ARCH__
  double t = __dmul_rn(__dsub_rn(yc, yl), __dsub_rn(xh, xl));
  t = __ddiv_rn(t, __dsub_rn(yh, yl));
  return __dadd_rn(xl, t);
#else
  double t = (yc - yl) * (xh - xl);
  t = t / (yh - yl);
  return xl + t;
#endif
}

// SPEC.md:49-57 PIP, boundary = inside, even-odd over rings [r0, r1).
__device__ inline int pip_rings(const double* X, const double* Y, const int64_t* ring_off, int64_t r0, int64_t r1,
                                double px, double py) {
  int inside = 0;
  for (int64_t r = r0; r < r1; ++r) {
    int64_t a = ring_off[r], b = ring_off[r + 1];
    for (int64_t k = a; k < b; ++k) {
      int64_t k2 = (k + 1 < b) ? k + 1 : a;
      double ax = X[k], ay = Y[k], bx = X[k2], by = Y[k2];
      double minx = ax < bx ? ax : bx, maxx = ax < bx ? bx : ax;
      double miny = ay < by ? ay : by, maxy = ay < by ? by : ay;
      if (px >= minx && px <= maxx && py >= miny && py <= maxy) {
        double cr = __dsub_rn(__dmul_rn(__dsub_rn(bx, ax), __dsub_rn(py, ay)),
                              __dmul_rn(__dsub_rn(by, ay), __dsub_rn(px, ax)));
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

// SPEC.md:58-66 distance_to_boundary
__device__ inline double dist_rings(const double* X, const double* Y, const int64_t* ring_off, int64_t r0, int64_t r1,
                                    double px, double py) {
  double best = INFINITY;
  for (int64_t r = r0; r < r1; ++r) {
    int64_t a = ring_off[r], b = ring_off[r + 1];
    for (int64_t k = a; k < b; ++k) {
      int64_t k2 = (k + 1 < b) ? k + 1 : a;
      double ax = X[k], ay = Y[k], bx = X[k2], by = Y[k2];
      double dx = bx - ax, dy = by - ay, wx = px - ax, wy = py - ay;
      double L2 = dx * dx + dy * dy, t = 0.0;
      if (L2 > 0.0) { t = (wx * dx + wy * dy) / L2; t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t); }
      double ex = wx - t * dx, ey = wy - t * dy;
      double d = sqrt(ex * ex + ey * ey);
      best = d < best ? d : best;
    }
  }
  return best;
}

// ----------------------------------------------------------- device memory
// The library's private stream-ordered pool (one per device; freed blocks stay cached up to a release
// threshold, so repeated builds and point passes do not pay cudaMalloc / cudaFree -- which synchronise
// the device -- and the process-wide default pool is left alone).
cudaMemPool_t mem_pool();
template <class T>
inline cudaError_t pool_alloc(T** p, size_t bytes, cudaStream_t s) {
  return cudaMallocFromPoolAsync((void**)p, bytes ? bytes : 1, mem_pool(), s);
}
// Build-time allocation scope: while alive on this thread, DBuf allocations are stream-ordered on `s`
// from the private pool (temporaries are freed stream-ordered; buffers kept by an rb_approx are
// detached at the end of the build and later freed with cudaFree, which orders itself).
cudaStream_t& alloc_stream_tls();
bool& alloc_scope_tls();
struct AllocScope {
  cudaStream_t prev_s;
  bool prev_on;
  explicit AllocScope(cudaStream_t s) : prev_s(alloc_stream_tls()), prev_on(alloc_scope_tls()) {
    alloc_stream_tls() = s;
    alloc_scope_tls() = true;
  }
  ~AllocScope() {
    alloc_stream_tls() = prev_s;
    alloc_scope_tls() = prev_on;
  }
};
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  bool pooled = false;  // stream-ordered: freed with cudaFreeAsync on `s` until detached
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes), s(o.s), pooled(o.pooled) { o.p = nullptr; o.bytes = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    release();
    p = o.p; bytes = o.bytes; s = o.s; pooled = o.pooled;
    o.p = nullptr; o.bytes = 0;
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) {
      if (pooled) cudaFreeAsync(p, s); else cudaFree(p);
    }
    p = nullptr;
    bytes = 0;
  }
  cudaError_t alloc(size_t b) {
    release();
    bytes = b;
    if (!b) return cudaSuccess;
    if (alloc_scope_tls()) {
      s = alloc_stream_tls();
      pooled = true;
      return pool_alloc(&p, b, s);
    }
    pooled = false;
    return cudaMalloc(&p, b);
  }
  // index data that outlives the build: plain cudaMalloc, so the pool holds only build scratch and its
  // working set (and so the build time) stays the same from one build to the next
  cudaError_t alloc_persistent(size_t b) {
    release();
    bytes = b;
    pooled = false;
    return b ? cudaMalloc(&p, b) : cudaSuccess;
  }
  void detach() { pooled = false; }  // outlives the allocating stream: cudaFree later (synchronising)
  template <class T> T* as() const { return (T*)p; }
};

// Index geometry: root table at level T0 (row-major, 2^T0 x 2^T0 slots) and
// node levels T0 + ks[0], T0 + ks[0] + ks[1], ..., L; a node of level i holds
// 2^ks[i] x 2^ks[i] row-major slots.  T0 == L is the dense uniform grid.
#define RB_MAX_NODE_LEVELS 8
struct IndexView {
  const uint32_t* root;
  const uint32_t* nodes[RB_MAX_NODE_LEVELS];
  int ks[RB_MAX_NODE_LEVELS];
  int nlev;
  const uint32_t* pool;
  int L, T0;
  const uint16_t* summary;  // level-S table of single owner values (0xffff = consult the index)
  int S;
  int64_t nodes0_len;  // entries of the first node level (32-bit offsets when < 2^32)
  // RB_LAYOUT_KEYS: disjoint cells as sorted leaf-level start keys, their levels and owner values,
  // and a radix table over the top key bits (ktab[p] = first key with key >> kshift >= p)
  const uint4* krec;    // per cell: start key (lo, hi words), owner value, level -- one 16-byte load
  const uint32_t* ktab;
  int64_t nkeys;
  int kshift;
  // RB_LAYOUT_PACKED: the radix table (root, then nlev = 0 or 1 node levels of u32 slots) ends in packed
  // nodes of 2^pd x 2^pd leaves: a slot RB_VALUE_NODE | b points at the node's 4^(pd-2) blocks of 4x4
  // leaves, pblk[b ..] (row-major over the node's 2^(pd-2) x 2^(pd-2) blocks).  Block {p0, p1, p2, idx}:
  // leaf s = (y & 3) * 4 + (x & 3) owns p[(idx >> 2s) & 3]; a block with more than three distinct owner
  // values has p0 = RB_VALUE_NODE | e, idx = 0: its 16 values are pwide[16e ..]
  const uint4* pblk;
  const uint32_t* pwide;
  int pd;
  // owner-value format: code = value & code_mask; hot slot + 1 = value >> hot_shift (bits up to 29)
  uint32_t code_mask;
  uint32_t hot_shift;
};

// RB_LAYOUT_PACKED helpers: the block of leaf (ix, iy) in the root cell whose first block is b, and the
// owner value of the leaf in a loaded block (escape blocks resolved with one more load)
__device__ __forceinline__ uint32_t packed_block(uint32_t b, uint32_t ix, uint32_t iy, int pd) {
  const uint32_t bm = (1u << (pd - 2)) - 1u;
  return b + ((((iy >> 2) & bm) << (pd - 2)) | ((ix >> 2) & bm));
}
__device__ __forceinline__ uint32_t packed_slot(uint32_t ix, uint32_t iy) { return ((iy & 3u) << 2) | (ix & 3u); }
__device__ __forceinline__ uint32_t packed_pick(const uint4& k, uint32_t s) {
  const uint32_t i = (k.w >> (2u * s)) & 3u;
  return i == 0u ? k.x : (i == 1u ? k.y : k.z);
}


__device__ __forceinline__ uint64_t spread_bits(uint32_t v) {
  uint64_t x = v;
  x = (x | (x << 16)) & 0x0000ffff0000ffffull;
  x = (x | (x << 8)) & 0x00ff00ff00ff00ffull;
  x = (x | (x << 4)) & 0x0f0f0f0f0f0f0f0full;
  x = (x | (x << 2)) & 0x3333333333333333ull;
  x = (x | (x << 1)) & 0x5555555555555555ull;
  return x;
}

// RB_LAYOUT_KEYS lookup: the leaf's Z code (x in the even bits); the radix table
// narrows the sorted cells to one prefix bucket (plus the cell before it).  Buckets hold ~1 cell, so
// the few records are read at once (one dependent step after the table); larger buckets binary-search.
// The owner is the last cell starting at or before the leaf, if the leaf lies inside it.
__device__ __forceinline__ uint64_t leaf_z(uint32_t ix, uint32_t iy) { return spread_bits(ix) | (spread_bits(iy) << 1); }

// the owner of leaf z among the cells [lo, hi) of its radix bucket (lo = table[p], hi = table[p + 1])
__device__ __forceinline__ uint32_t keys_resolve(const IndexView& v, uint64_t z, int64_t lo, int64_t hi) {
  lo = lo > 0 ? lo - 1 : 0;
  uint4 best = make_uint4(0u, 0u, 0u, 0u);
  bool found = false;
  if (hi - lo <= 4) {
    uint4 r[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) r[t] = lo + t < hi ? __ldg(v.krec + lo + t) : make_uint4(0xffffffffu, 0xffffffffu, 0u, 0u);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint64_t k = ((uint64_t)r[t].y << 32) | r[t].x;
      if (lo + t < hi && k <= z) { best = r[t]; found = true; }
    }
  } else {
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      const uint4 rm = __ldg(v.krec + m);
      if ((((uint64_t)rm.y << 32) | rm.x) <= z) { best = rm; found = true; lo = m + 1; } else hi = m;
    }
  }
  if (!found) return 0u;
  const uint64_t start = ((uint64_t)best.y << 32) | best.x;
  const uint64_t end = start + ((uint64_t)1 << (2 * (v.L - (int)best.w)));
  return z < end ? best.z : 0u;
}

__device__ __forceinline__ uint32_t keys_lookup(const IndexView& v, uint32_t ix, uint32_t iy) {
  const uint64_t z = leaf_z(ix, iy);
  const uint64_t p = z >> v.kshift;
  return keys_resolve(v, z, (int64_t)v.ktab[p], (int64_t)v.ktab[p + 1]);
}

__device__ __forceinline__ uint32_t index_lookup(const IndexView& v, uint32_t ix, uint32_t iy) {
  if (v.krec) return keys_lookup(v, ix, iy);
  int s = v.L - v.T0;
  uint32_t val = __ldg(&v.root[((size_t)(iy >> s) << v.T0) | (ix >> s)]);
  if (v.pblk) {
    for (int li = 0; li < v.nlev && (val & RB_VALUE_NODE); ++li) {  // u32 node levels above the packed nodes
      const int k = v.ks[li];
      s -= k;
      const uint32_t m = (1u << k) - 1u;
      val = __ldg(&v.nodes[li][((size_t)(val & RB_VALUE_PAYLOAD) << (2 * k)) + ((((iy >> s) & m) << k) | ((ix >> s) & m))]);
    }
    if (val & RB_VALUE_NODE) {
      const uint32_t sl = packed_slot(ix, iy);
      val = packed_pick(__ldg(v.pblk + packed_block(val & RB_VALUE_PAYLOAD, ix, iy, v.pd)), sl);
      if (val & RB_VALUE_NODE) val = __ldg(v.pwide + (((size_t)(val & RB_VALUE_PAYLOAD)) << 4) + sl);
    }
    return val;
  }
#pragma unroll
  for (int li = 0; li < RB_MAX_NODE_LEVELS; ++li) {
    if (!(val & RB_VALUE_NODE)) break;
    int k = v.ks[li];
    s -= k;
    uint32_t m = (1u << k) - 1u;
    size_t node = val & RB_VALUE_PAYLOAD;
    uint32_t slot = (((iy >> s) & m) << k) | ((ix >> s) & m);
    val = __ldg(&v.nodes[li][(node << (2 * k)) + slot]);
  }
  return val;
}

}  // namespace rb

struct rb_approx {
  rb_grid grid;
  rb_build_opts opts;
  int32_t n_regions = 0;
  int64_t n_polygons = 0;
  rb::DBuf root, pool;
  std::vector<rb::DBuf> node_bufs;
  std::vector<int> node_levels;
  int64_t root_entries = 0, n_nodes = 0, pool_len = 0;
  int T0 = 0, k = 4;
  rb::DBuf summary;  // u16 [4^S] or empty
  int S = -1;
  rb::DBuf keys, ktab;  // RB_LAYOUT_KEYS: uint4 records (start key, owner value, level), radix table
  int64_t nkeys = 0;
  int kshift = 0;
  rb::DBuf pblk, pwide;  // RB_LAYOUT_PACKED: palette blocks (uint4) and escape blocks (16 x u32)
  int64_t n_pblk = 0, n_pwide = 0;
  int pd = 0;
  rb::DBuf hot_region;  // int32 [n_hot]: hot slot -> region
  int32_t n_hot = 0;
  // partitioned point pass (rb_binned.cuh): per level-bin_level cell, whether any root slot below it is set
  // (points in uncovered bins have no owner); computed on first use
  rb::DBuf bin_flags;
  int bin_level = -1, bin_used = 0;
  std::mutex bin_mu;
  // Owner codes ((region << 1) | boundary) + 1 take code_bits = bit length of 2 * n_regions (<= 18); the hot
  // slot annotation (slot + 1) sits above them, up to bit 29: 2^(30 - code_bits) - 1 slots (4095 .. 16383)
  uint32_t code_mask = RB_CODE_MASK, hot_shift = RB_HOT_SHIFT;
  int32_t max_hot = RB_MAX_HOT;
  void set_code_format() {
    uint32_t cb = 1;
    while (cb < 18 && ((uint64_t)2 * (uint64_t)n_regions) >> cb) ++cb;
    if (cb < 16) cb = 16;
    code_mask = (1u << cb) - 1u;
    hot_shift = cb;
    const int64_t mh = ((int64_t)1 << (30 - cb)) - 1;
    max_hot = (int32_t)(mh < RB_MAX_HOT_CAP ? mh : RB_MAX_HOT_CAP);
  }
  // optional exports
  rb::DBuf cell_poly, cell_level, cell_code, cell_kind;
  int64_t n_cells = 0;
  rb::DBuf part_poly, part_code, part_kept;
  int64_t n_partial = 0;
  rb_stats stats{};
  // buffers kept past the build no longer belong to the build stream
  void detach_all() {
    for (rb::DBuf* b : {&root, &pool, &summary, &keys, &ktab, &pblk, &pwide, &hot_region, &bin_flags, &cell_poly,
                        &cell_level, &cell_code, &cell_kind, &part_poly, &part_code, &part_kept})
      b->detach();
    for (auto& b : node_bufs) b.detach();
  }
  ~rb_approx() { cudaDeviceSynchronize(); }  // no pass may still read the index when it is freed
  rb::IndexView view() const {
    rb::IndexView v{};
    v.root = root.as<uint32_t>();
    v.nlev = (int)node_levels.size();
    for (int i = 0; i < v.nlev; ++i) { v.nodes[i] = node_bufs[i].as<uint32_t>(); v.ks[i] = node_levels[i]; }
    v.pool = pool.as<uint32_t>();
    v.L = grid.max_level;
    v.T0 = T0;
    v.summary = summary.as<uint16_t>();
    v.S = S;
    v.nodes0_len = v.nlev > 0 ? (int64_t)(node_bufs[0].bytes / 4) : 0;
    v.krec = keys.as<uint4>();
    v.ktab = ktab.as<uint32_t>();
    v.nkeys = nkeys;
    v.kshift = kshift;
    v.pblk = pblk.as<uint4>();
    v.pwide = pwide.as<uint32_t>();
    v.pd = pd;
    v.code_mask = code_mask;
    v.hot_shift = hot_shift;
    return v;
  }
};
