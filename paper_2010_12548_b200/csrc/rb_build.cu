// rb_build.cu -- GPU construction of the epsilon-bounded raster approximation
// and its cell index (north star subsystems 1 and 2).
//
// Pipeline (all on the stream given to rb_approx_build):
//   K0  vertex -> grid units (SPEC.md:146 map, shared with points)
//   K2  conservative edge walk: PARTIAL leaves per polygon
//   K3  scanline crossings at row centres -> interior spans     (D2)
//   K4  level-synchronous quadtree descent: hierarchical cells
//   K5  overlay of all regions' cells into disjoint positions with owner
//       lists ("all owners" rule) and the radix-table index
//       (ACT): root table at level T0 + nodes of radix_width
//       bits; T0 == L is the dense uniform grid.
// Every predicate restates oracle/rb_oracle.c with identical float64 order.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <memory>

#include "rb_internal.cuh"

#ifndef RB_SUMMARY_DEFAULT
#define RB_SUMMARY_DEFAULT 7
#endif

namespace rb {

// ------------------------------------------------------------ CUB helpers
static cudaError_t excl_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s);
  if (e) return e;
  DBuf t;
  if ((e = t.alloc(tb ? tb : 1))) return e;
  return cub::DeviceScan::ExclusiveSum(t.p, tb, in, out, n, s);
}

// in-place inclusive max-scan (run heads)
static cudaError_t incl_max_scan_i64(int64_t* a, int64_t n, cudaStream_t s) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceScan::InclusiveScan(nullptr, tb, a, a, cub::Max(), n, s);
  if (e) return e;
  DBuf t;
  if ((e = t.alloc(tb ? tb : 1))) return e;
  return cub::DeviceScan::InclusiveScan(t.p, tb, a, a, cub::Max(), n, s);
}

template <class T>
static cudaError_t seg_sort_keys(T* keys, int64_t n, int64_t nseg, const int64_t* beg, const int64_t* end,
                                 cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  DBuf alt;
  cudaError_t e = alt.alloc(n * sizeof(T));
  if (e) return e;
  cub::DoubleBuffer<T> db(keys, alt.as<T>());
  size_t tb = 0;
  e = cub::DeviceSegmentedSort::SortKeys(nullptr, tb, db, n, nseg, beg, end, s);
  if (e) return e;
  DBuf t;
  if ((e = t.alloc(tb ? tb : 1))) return e;
  e = cub::DeviceSegmentedSort::SortKeys(t.p, tb, db, n, nseg, beg, end, s);
  if (e) return e;
  if (db.Current() != keys) e = cudaMemcpyAsync(keys, db.Current(), n * sizeof(T), cudaMemcpyDeviceToDevice, s);
  if (e) return e;
  return cudaStreamSynchronize(s);
}

static cudaError_t radix_sort_pairs(uint64_t* keys, uint32_t* vals, int64_t n, int end_bit, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  DBuf ka, va;
  cudaError_t e;
  if ((e = ka.alloc(n * 8))) return e;
  if ((e = va.alloc(n * 4))) return e;
  cub::DoubleBuffer<uint64_t> dk(keys, ka.as<uint64_t>());
  cub::DoubleBuffer<uint32_t> dv(vals, va.as<uint32_t>());
  size_t tb = 0;
  if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, n, 0, end_bit, s))) return e;
  DBuf t;
  if ((e = t.alloc(tb ? tb : 1))) return e;
  if ((e = cub::DeviceRadixSort::SortPairs(t.p, tb, dk, dv, n, 0, end_bit, s))) return e;
  if (dk.Current() != keys) {
    if ((e = cudaMemcpyAsync(keys, dk.Current(), n * 8, cudaMemcpyDeviceToDevice, s))) return e;
    if ((e = cudaMemcpyAsync(vals, dv.Current(), n * 4, cudaMemcpyDeviceToDevice, s))) return e;
  }
  return cudaStreamSynchronize(s);
}

template <class T>
static T d2h(const T* p, cudaStream_t s) {
  T v{};
  cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  return v;
}

static inline int nblk(int64_t n, int t = 256) {
  int64_t b = (n + t - 1) / t;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 64));
}
#define GRID_STRIDE(k, n) for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < (n); k += (int64_t)gridDim.x * blockDim.x)

// ------------------------------------------------------------------- K0
__global__ void k_ring_poly(const int64_t* poly_ring_off, int64_t np, int32_t* ring_poly) {
  GRID_STRIDE(p, np) {
    for (int64_t r = poly_ring_off[p]; r < poly_ring_off[p + 1]; ++r) ring_poly[r] = (int32_t)p;
  }
}

__global__ void k_vertex(const double* vx, const double* vy, int64_t nv, const int64_t* ring_off, int64_t nr,
                         const int32_t* ring_poly, GridD g, double* gx, double* gy, int64_t* vnext, int32_t* vpoly,
                         int* flags) {
  GRID_STRIDE(k, nv) {
    double x = vx[k], y = vy[k];
    if (!isfinite(x) || !isfinite(y)) atomicOr(flags, 1);
    double u = gcoord(x, g.ox, g.side), v = gcoord(y, g.oy, g.side);
    if (!(u >= 0.0 && u <= g.lim && v >= 0.0 && v <= g.lim)) atomicOr(flags, 2);
    gx[k] = u;
    gy[k] = v;
    // ring of vertex k: last r with ring_off[r] <= k
    int64_t lo = 0, hi = nr;
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if (ring_off[mid] <= k) lo = mid; else hi = mid;
    }
    vnext[k] = (k + 1 < ring_off[lo + 1]) ? k + 1 : ring_off[lo];
    vpoly[k] = ring_poly[lo];
  }
}

// per polygon: outer-ring shoelace (SPEC.md:33 nonzero area, same order as
// the oracle) and the leaf MBR of all its vertices.
__global__ void k_poly_info(const double* vx, const double* vy, const double* gx, const double* gy,
                            const int64_t* ring_off, const int64_t* poly_ring_off, int64_t np, double lim,
                            uint32_t* mbr, int* flags) {
  GRID_STRIDE(p, np) {
    int64_t a = ring_off[poly_ring_off[p]], b = ring_off[poly_ring_off[p] + 1];
    double ar = 0.0;
    for (int64_t k = a; k < b; ++k) {
      int64_t k2 = (k + 1 < b) ? k + 1 : a;
      ar = __dadd_rn(ar, __dsub_rn(__dmul_rn(vx[k], vy[k2]), __dmul_rn(vx[k2], vy[k])));
    }
    if (ar == 0.0) atomicOr(flags, 4);
    double mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    for (int64_t k = a; k < ring_off[poly_ring_off[p + 1]]; ++k) {
      mnx = fmin(mnx, gx[k]); mxx = fmax(mxx, gx[k]);
      mny = fmin(mny, gy[k]); mxy = fmax(mxy, gy[k]);
    }
    double top = lim - 1.0;
    mbr[4 * p + 0] = (uint32_t)floor(mnx);
    mbr[4 * p + 1] = (uint32_t)floor(mny);
    mbr[4 * p + 2] = (uint32_t)fmin(floor(mxx), top);
    mbr[4 * p + 3] = (uint32_t)fmin(floor(mxy), top);
  }
}

// ------------------------------------------------------------------- K2
// S2: open leaves crossed by an edge (oracle edge_walk, identical order).
template <class F>
__device__ inline void edge_walk(double x1, double y1, double x2, double y2, F& emit) {
  if (x2 < x1 || (x2 == x1 && y2 < y1)) {
    double t = x1; x1 = x2; x2 = t;
    t = y1; y1 = y2; y2 = t;
  }
  if (x1 == x2 && y1 == y2) return;
  if (x1 == x2) {
    if (x1 == floor(x1)) return;
    int64_t i = (int64_t)floor(x1);
    int64_t j0 = (int64_t)floor(y1), j1 = (int64_t)ceil(y2) - 1;
    for (int64_t j = j0; j <= j1; ++j) emit(i, j);
    return;
  }
  int64_t i0 = (int64_t)floor(x1), i1 = (int64_t)ceil(x2) - 1;
  for (int64_t i = i0; i <= i1; ++i) {
    double xa = x1 > (double)i ? x1 : (double)i;
    double xb = x2 < (double)(i + 1) ? x2 : (double)(i + 1);
    double ya = y_at(x1, y1, x2, y2, xa), yb = y_at(x1, y1, x2, y2, xb);
    double lo = ya < yb ? ya : yb, hi = ya < yb ? yb : ya;
    if (lo == hi) {
      if (lo == floor(lo)) continue;
      emit(i, (int64_t)floor(lo));
      continue;
    }
    int64_t j0 = (int64_t)floor(lo), j1 = (int64_t)ceil(hi) - 1;
    for (int64_t j = j0; j <= j1; ++j) emit(i, j);
  }
}

struct CountEmit {
  int64_t n = 0;
  __device__ void operator()(int64_t, int64_t) { ++n; }
};
struct ZEmit {
  uint64_t* out;
  __device__ void operator()(int64_t i, int64_t j) { *out++ = zenc((uint64_t)i, (uint64_t)j); }
};

__global__ void k_walk_count(const double* gx, const double* gy, const int64_t* vnext, int64_t nv, int64_t* cnt) {
  GRID_STRIDE(k, nv) {
    CountEmit c;
    int64_t k2 = vnext[k];
    edge_walk(gx[k], gy[k], gx[k2], gy[k2], c);
    cnt[k] = c.n;
  }
}
__global__ void k_walk_emit(const double* gx, const double* gy, const int64_t* vnext, int64_t nv, const int64_t* off,
                            uint64_t* out) {
  GRID_STRIDE(k, nv) {
    ZEmit e{out + off[k]};
    int64_t k2 = vnext[k];
    edge_walk(gx[k], gy[k], gx[k2], gy[k2], e);
  }
}

// ------------------------------------------------------------------- K3
template <class F>
__device__ inline void edge_crossings(double x1, double y1, double x2, double y2, F& emit) {
  if (y1 == y2) return;
  double xl, yl, xh, yh;
  if (y1 < y2) { xl = x1; yl = y1; xh = x2; yh = y2; } else { xl = x2; yl = y2; xh = x1; yh = y1; }
  int64_t j0 = (int64_t)ceil(yl - 0.5), j1 = (int64_t)ceil(yh - 0.5) - 1;
  for (int64_t j = j0; j <= j1; ++j) {
    double x = x_cross(xl, yl, xh, yh, (double)j + 0.5);
    emit(j, (int64_t)ceil(x - 0.5));
  }
}
struct XEmit {
  uint64_t* out;
  __device__ void operator()(int64_t j, int64_t t) { *out++ = ((uint64_t)j << 32) | (uint64_t)t; }
};
__global__ void k_xing_count(const double* gx, const double* gy, const int64_t* vnext, int64_t nv, int64_t* cnt) {
  GRID_STRIDE(k, nv) {
    CountEmit c;
    int64_t k2 = vnext[k];
    edge_crossings(gx[k], gy[k], gx[k2], gy[k2], c);
    cnt[k] = c.n;
  }
}
__global__ void k_xing_emit(const double* gx, const double* gy, const int64_t* vnext, int64_t nv, const int64_t* off,
                            uint64_t* out) {
  GRID_STRIDE(k, nv) {
    XEmit e{out + off[k]};
    int64_t k2 = vnext[k];
    edge_crossings(gx[k], gy[k], gx[k2], gy[k2], e);
  }
}

// segment bounds per polygon from a per-vertex exclusive scan (size nv+1)
__global__ void k_seg_bounds(const int64_t* scan, const int64_t* ring_off, const int64_t* poly_ring_off, int64_t np,
                             int64_t* beg, int64_t* end) {
  GRID_STRIDE(p, np) {
    beg[p] = scan[ring_off[poly_ring_off[p]]];
    end[p] = scan[ring_off[poly_ring_off[p + 1]]];
  }
}

// unique flags within polygon segments of a sorted array; seg_of via binary search
__global__ void k_unique_flags(const uint64_t* a, int64_t n, const int64_t* beg, int64_t np, int64_t* flag) {
  GRID_STRIDE(k, n) {
    int64_t lo = 0, hi = np;  // last p with beg[p] <= k (skip empty segments by taking the last)
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if (beg[mid] <= k) lo = mid; else hi = mid;
    }
    flag[k] = (k == beg[lo] || a[k] != a[k - 1]) ? 1 : 0;
  }
}
__global__ void k_compact_u64(const uint64_t* a, const int64_t* flag, const int64_t* pos, int64_t n, uint64_t* out) {
  GRID_STRIDE(k, n) if (flag[k]) out[pos[k]] = a[k];
}
__global__ void k_remap_bounds(const int64_t* pos, const int64_t* beg, const int64_t* end, int64_t np, int64_t* nbeg,
                               int64_t* nend, int64_t n, int64_t total) {
  GRID_STRIDE(p, np) {
    nbeg[p] = beg[p] < n ? pos[beg[p]] : total;
    nend[p] = end[p] < n ? pos[end[p]] : total;
  }
}

// spans from sorted crossing keys: pairs (2m, 2m+1) inside each polygon segment
__global__ void k_span_count(const uint64_t* x, const int64_t* beg, const int64_t* end, int64_t np, int64_t* cnt) {
  GRID_STRIDE(p, np) {
    int64_t c = 0;
    for (int64_t k = beg[p]; k + 1 < end[p]; k += 2) {
      uint32_t t0 = (uint32_t)x[k], t1 = (uint32_t)x[k + 1];
      if (t0 < t1) ++c;
    }
    cnt[p] = c;
  }
}
__global__ void k_span_emit(const uint64_t* x, const int64_t* beg, const int64_t* end, int64_t np, const int64_t* off,
                            uint64_t* skey, int32_t* sc1) {
  GRID_STRIDE(p, np) {
    int64_t w = off[p];
    for (int64_t k = beg[p]; k + 1 < end[p]; k += 2) {
      uint32_t t0 = (uint32_t)x[k], t1 = (uint32_t)x[k + 1];
      if (t0 < t1) {
        skey[w] = (x[k] & 0xffffffff00000000ull) | t0;
        sc1[w] = (int32_t)(t1 - 1);
        ++w;
      }
    }
  }
}

// aligned (grid-line) boundary pieces, S7
__global__ void k_aligned_count(const double* gx, const double* gy, const int64_t* vnext, int64_t nv, int64_t* flag) {
  GRID_STRIDE(k, nv) {
    int64_t k2 = vnext[k];
    double x1 = gx[k], y1 = gy[k], x2 = gx[k2], y2 = gy[k2];
    flag[k] = ((x1 == x2 && x1 == floor(x1) && y1 != y2) || (y1 == y2 && y1 == floor(y1) && x1 != x2)) ? 1 : 0;
  }
}
__global__ void k_aligned_emit(const double* gx, const double* gy, const int64_t* vnext, int64_t nv,
                               const int64_t* flag, const int64_t* pos, double4* out) {
  GRID_STRIDE(k, nv) {
    if (!flag[k]) continue;
    int64_t k2 = vnext[k];
    double x1 = gx[k], y1 = gy[k], x2 = gx[k2], y2 = gy[k2];
    if (x1 == x2) out[pos[k]] = make_double4(x1, fmin(y1, y2), fmax(y1, y2), 1.0);
    else out[pos[k]] = make_double4(y1, fmin(x1, x2), fmax(x1, x2), 0.0);
  }
}

// CENTER_SAMPLED keep rule for PARTIAL leaves (S4)
__global__ void k_kept(const uint64_t* part, int64_t n, const int64_t* beg, int64_t np, const double* gx,
                       const double* gy, const int64_t* ring_off, const int64_t* poly_ring_off, int mode,
                       uint8_t* kept, int32_t* part_poly) {
  GRID_STRIDE(k, n) {
    int64_t lo = 0, hi = np;
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if (beg[mid] <= k) lo = mid; else hi = mid;
    }
    part_poly[k] = (int32_t)lo;
    if (mode == RB_MODE_CONSERVATIVE) { kept[k] = 1; continue; }
    uint64_t z = part[k];
    double cx = (double)compact1by1(z) + 0.5, cy = (double)compact1by1(z >> 1) + 0.5;
    kept[k] = (uint8_t)pip_rings(gx, gy, ring_off, poly_ring_off[lo], poly_ring_off[lo + 1], cx, cy);
  }
}

// ------------------------------------------------------------------- K4
struct PolyView {
  const uint32_t* mbr;
  const uint64_t* part; const int64_t* pbeg; const int64_t* pend; const uint8_t* kept;
  const uint64_t* skey; const int32_t* sc1; const int64_t* sbeg; const int64_t* send;
  const double4* al; const int64_t* abeg; const int64_t* aend;
};

__device__ inline int64_t lower_u64(const uint64_t* a, int64_t lo, int64_t hi, uint64_t key) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ inline int in_spans(const PolyView& V, int p, uint32_t i, uint32_t j) {
  uint64_t key = ((uint64_t)j << 32) | i;
  int64_t lo = V.sbeg[p], hi = V.send[p];
  // upper bound of key
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (V.skey[mid] <= key) lo = mid + 1; else hi = mid;
  }
  if (lo == V.sbeg[p]) return 0;
  uint64_t s = V.skey[lo - 1];
  return (uint32_t)(s >> 32) == j && (int32_t)i <= V.sc1[lo - 1];
}

__device__ inline int leaf_kind(const PolyView& V, int p, uint32_t i, uint32_t j) {
  if (i < V.mbr[4 * p] || j < V.mbr[4 * p + 1] || i > V.mbr[4 * p + 2] || j > V.mbr[4 * p + 3]) return RB_KIND_NONE;
  uint64_t z = zenc(i, j);
  int64_t k = lower_u64(V.part, V.pbeg[p], V.pend[p], z);
  if (k < V.pend[p] && V.part[k] == z) return V.kept[k] ? RB_KIND_B : RB_KIND_NONE;
  return in_spans(V, p, i, j) ? RB_KIND_I : RB_KIND_NONE;
}

__device__ inline int aligned_cut(const PolyView& V, int p, double bx0, double by0, double bx1, double by1) {
  for (int64_t k = V.abeg[p]; k < V.aend[p]; ++k) {
    double4 a = V.al[k];
    if (a.w != 0.0) {
      if (bx0 < a.x && a.x < bx1 && fmax(a.y, by0) < fmin(a.z, by1)) return 1;
    } else {
      if (by0 < a.x && a.x < by1 && fmax(a.y, bx0) < fmin(a.z, bx1)) return 1;
    }
  }
  return 0;
}

// one frontier item (S7, oracle hier_visit)
template <class Child, class Cell>
__device__ inline void hier_item(const PolyView& V, int p, uint64_t code, int lvl, int L, Child& child, Cell& cell) {
  int d = L - lvl;
  uint64_t bi = (uint64_t)compact1by1(code) << d, bj = (uint64_t)compact1by1(code >> 1) << d;
  uint64_t bw = 1ull << d;
  if (bi > V.mbr[4 * p + 2] || bj > V.mbr[4 * p + 3] || bi + (bw - 1) < V.mbr[4 * p] || bj + (bw - 1) < V.mbr[4 * p + 1])
    return;
  if (d == 0) {
    int k = leaf_kind(V, p, (uint32_t)bi, (uint32_t)bj);
    if (k) cell(lvl, code, k);
    return;
  }
  uint64_t lo = code << (2 * d), hi = (code + 1) << (2 * d);
  int64_t q = lower_u64(V.part, V.pbeg[p], V.pend[p], lo);
  bool mixed = q < V.pend[p] && V.part[q] < hi;
  if (!mixed) mixed = aligned_cut(V, p, (double)bi, (double)bj, (double)bi + (double)bw, (double)bj + (double)bw);
  if (!mixed) {
    if (in_spans(V, p, (uint32_t)bi, (uint32_t)bj)) cell(lvl, code, RB_KIND_I);
    return;
  }
  if (d == 1) {
    for (uint64_t c = 0; c < 4; ++c) {
      uint64_t cc = code * 4 + c;
      int k = leaf_kind(V, p, compact1by1(cc), compact1by1(cc >> 1));
      if (k) cell(L, cc, k);
    }
  } else {
    for (uint64_t c = 0; c < 4; ++c) child(code * 4 + c);
  }
}

struct CntChild { int n = 0; __device__ void operator()(uint64_t) { ++n; } };
struct CntCell { int n = 0; __device__ void operator()(int, uint64_t, int) { ++n; } };
struct WChild {
  int32_t* fp; uint64_t* fc; int64_t w; int p;
  __device__ void operator()(uint64_t c) { fp[w] = p; fc[w] = c; ++w; }
};
struct WCell {
  int32_t* cp; uint8_t* cl; uint64_t* cc; uint8_t* ck; int64_t w; int p;
  __device__ void operator()(int l, uint64_t c, int k) { cp[w] = p; cl[w] = (uint8_t)l; cc[w] = c; ck[w] = (uint8_t)k; ++w; }
};

__global__ void k_hier_count(PolyView V, const int32_t* fp, const uint64_t* fc, int64_t nf, int lvl, int L,
                             int64_t* nchild, int64_t* ncell) {
  GRID_STRIDE(k, nf) {
    CntChild a; CntCell b;
    hier_item(V, fp[k], fc[k], lvl, L, a, b);
    nchild[k] = a.n;
    ncell[k] = b.n;
  }
}
__global__ void k_hier_emit(PolyView V, const int32_t* fp, const uint64_t* fc, int64_t nf, int lvl, int L,
                            const int64_t* coff, const int64_t* eoff, int32_t* nfp, uint64_t* nfc, int32_t* cp,
                            uint8_t* cl, uint64_t* cc, uint8_t* ck) {
  GRID_STRIDE(k, nf) {
    int p = fp[k];
    WChild a{nfp, nfc, coff[k], p};
    WCell b{cp, cl, cc, ck, eoff[k], p};
    hier_item(V, p, fc[k], lvl, L, a, b);
  }
}

// ------------------------------------------------------------------- K5
__global__ void k_cell_keys(const int32_t* cp, const uint8_t* cl, const uint64_t* cc, const uint8_t* ck,
                            const int32_t* poly_region, int64_t n, int L, uint64_t* start, uint64_t* sec,
                            uint32_t* idx) {
  GRID_STRIDE(k, n) {
    int l = cl[k];
    start[k] = cc[k] << (2 * (L - l));
    sec[k] = ((uint64_t)l << 40) | ((uint64_t)(uint32_t)poly_region[cp[k]] << 2) | ck[k];
    idx[k] = (uint32_t)k;
  }
}
// overlay record (SoA): start (level-L code), level, region, kind
struct Recs {
  uint64_t* start; uint8_t* level; int32_t* region; uint8_t* kind;
};
__global__ void k_gather_recs(const uint32_t* idx, int64_t n, const int32_t* cp, const uint8_t* cl, const uint64_t* cc,
                              const uint8_t* ck, const int32_t* poly_region, int L, Recs out) {
  GRID_STRIDE(k, n) {
    uint32_t s = idx[k];
    int l = cl[s];
    out.start[k] = cc[s] << (2 * (L - l));
    out.level[k] = (uint8_t)l;
    out.region[k] = poly_region[cp[s]];
    out.kind[k] = ck[s];
  }
}
__global__ void k_rec_keys(Recs r, int64_t n, uint64_t* start, uint64_t* sec, uint32_t* idx) {
  GRID_STRIDE(k, n) {
    start[k] = r.start[k];
    sec[k] = ((uint64_t)r.level[k] << 40) | ((uint64_t)(uint32_t)r.region[k] << 2) | r.kind[k];
    idx[k] = (uint32_t)k;
  }
}
__global__ void k_rec_gather(const uint32_t* idx, int64_t n, Recs in, Recs out) {
  GRID_STRIDE(k, n) {
    uint32_t s = idx[k];
    out.start[k] = in.start[s]; out.level[k] = in.level[s]; out.region[k] = in.region[s]; out.kind[k] = in.kind[s];
  }
}
__global__ void k_gather_u64(const uint64_t* src, const uint32_t* idx, int64_t n, uint64_t* dst) {
  GRID_STRIDE(k, n) dst[k] = src[idx[k]];
}
// head flag: first record of each (start, level) position
__global__ void k_pos_head(Recs r, int64_t n, int64_t* head) {
  GRID_STRIDE(k, n) head[k] = (k == 0 || r.start[k] != r.start[k - 1] || r.level[k] != r.level[k - 1]) ? 1 : 0;
}
__global__ void k_pos_list(const int64_t* head, const int64_t* hpos, int64_t n, int64_t* pbeg) {
  GRID_STRIDE(k, n) if (head[k]) pbeg[hpos[k]] = k;
}
// container flag per record: its position contains the next position
__global__ void k_container(Recs r, int64_t n, const int64_t* head, const int64_t* hpos, const int64_t* pbeg,
                            int64_t npos, int L, int64_t* split) {
  GRID_STRIDE(k, n) {
    int64_t P = hpos[k] + head[k] - 1;  // inclusive position index
    int64_t b = pbeg[P], e = (P + 1 < npos) ? pbeg[P + 1] : n;
    uint64_t size = 1ull << (2 * (L - r.level[b]));
    split[k] = (e < n && r.start[e] < r.start[b] + size) ? 1 : 0;
  }
}
__global__ void k_split(Recs in, int64_t n, const int64_t* split, const int64_t* off, int L, Recs out) {
  GRID_STRIDE(k, n) {
    int64_t w = off[k];
    if (!split[k]) {
      out.start[w] = in.start[k]; out.level[w] = in.level[k]; out.region[w] = in.region[k]; out.kind[w] = in.kind[k];
    } else {
      int l = in.level[k] + 1;
      uint64_t q = 1ull << (2 * (L - l));
      for (int c = 0; c < 4; ++c) {
        out.start[w + c] = in.start[k] + c * q; out.level[w + c] = (uint8_t)l;
        out.region[w + c] = in.region[k]; out.kind[w + c] = in.kind[k];
      }
    }
  }
}
// owners per position: distinct regions (records sorted by region, kind within position; I=1 first)
// RB_LAYOUT_KEYS records: start key, owner value and level of each disjoint cell in one uint4
__global__ void k_key_records(const uint64_t* start, const uint8_t* level, const uint32_t* val, int64_t n,
                              uint4* rec) {
  GRID_STRIDE(i, n) rec[i] = make_uint4((uint32_t)start[i], (uint32_t)(start[i] >> 32), val[i], level[i]);
}
// RB_LAYOUT_KEYS summary: a level-S block is answered by one owner value when a single cell covers
// it (value <= 0xfffe: single owners), 0 when no cell meets it, else 0xffff (consult the keys)
__global__ void k_key_summary(const uint4* rec, int64_t n, int L, int S, uint16_t* out) {
  GRID_STRIDE(b, (int64_t)1 << (2 * S)) {
    const uint64_t span = (uint64_t)1 << (2 * (L - S));
    const uint32_t bx = (uint32_t)(b & ((1 << S) - 1)), by = (uint32_t)(b >> S);  // row-major, as the kernels read it
    const uint64_t z0 = spread_bits(bx << (L - S)) | (spread_bits(by << (L - S)) << 1), z1 = z0 + span;
    int64_t lo = 0, hi = n;  // first cell with start > z0
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if ((((uint64_t)rec[m].y << 32) | rec[m].x) <= z0) lo = m + 1; else hi = m;
    }
    uint16_t v = 0xffffu;
    const int64_t c = lo - 1;
    const uint64_t nxt = lo < n ? (((uint64_t)rec[lo].y << 32) | rec[lo].x) : ~0ull;
    if (c >= 0) {
      const uint64_t st = ((uint64_t)rec[c].y << 32) | rec[c].x;
      const uint64_t en = st + ((uint64_t)1 << (2 * (L - (int)rec[c].w)));
      if (en >= z1) v = rec[c].z <= 0xfffeu ? (uint16_t)rec[c].z : 0xffffu;  // one cell covers the block
      else if (en <= z0 && nxt >= z1) v = 0;                                   // no cell meets the block
    } else if (nxt >= z1) {
      v = 0;
    }
    out[b] = v;
  }
}
// RB_LAYOUT_KEYS radix table: tab[p] = first key index with key >> shift >= p
__global__ void k_key_table(const uint64_t* keys, int64_t n, int shift, int64_t nslots, uint32_t* tab) {
  GRID_STRIDE(p, nslots) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if ((keys[m] >> shift) < (uint64_t)p) lo = m + 1; else hi = m;
    }
    tab[p] = (uint32_t)lo;
  }
}
__global__ void k_pos_owners(Recs r, int64_t n, const int64_t* pbeg, int64_t npos, int64_t* nown) {
  GRID_STRIDE(P, npos) {
    int64_t b = pbeg[P], e = (P + 1 < npos) ? pbeg[P + 1] : n;
    int64_t c = 0;
    for (int64_t k = b; k < e; ++k) if (k == b || r.region[k] != r.region[k - 1]) ++c;
    nown[P] = c;
  }
}
// Owner lists are shared: positions with the same owner set (e.g. every boundary leaf between regions A
// and B) get one pool entry, so a block of the index holds few distinct owner values.  Lists are hashed,
// sorted by hash (stable: equal hashes keep position order), and a position whose list equals the first
// list of its hash run uses that run head's entry (a hash collision just keeps its own entry).
__device__ inline uint32_t list_entry(const Recs& r, int64_t k) {
  return ((uint32_t)r.region[k] << 1) | (r.kind[k] == RB_KIND_B ? 1u : 0u);
}
__global__ void k_list_hash(Recs r, int64_t n, const int64_t* pbeg, int64_t npos, const int64_t* nown, uint64_t* key,
                            uint32_t* idx) {
  GRID_STRIDE(P, npos) {
    uint64_t h = 0x9E3779B97F4A7C15ull;
    if (nown[P] > 1) {
      const int64_t b = pbeg[P], e = (P + 1 < npos) ? pbeg[P + 1] : n;
      for (int64_t k = b; k < e; ++k)
        if (k == b || r.region[k] != r.region[k - 1]) {
          h ^= list_entry(r, k) + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
          h *= 0xff51afd7ed558ccdull;
        }
      h ^= h >> 33;
      key[P] = h >> 1;  // < 2^63: single owners (all ones) sort last
    } else {
      key[P] = ~0ull;
    }
    idx[P] = (uint32_t)P;
  }
}
__global__ void k_run_head(const uint64_t* key, int64_t n, int64_t* head) {
  GRID_STRIDE(i, n) head[i] = (i == 0 || key[i] != key[i - 1]) ? i : 0;
}
__device__ inline bool lists_equal(const Recs& r, int64_t n, const int64_t* pbeg, int64_t npos, int64_t P, int64_t Q) {
  int64_t a = pbeg[P], ae = (P + 1 < npos) ? pbeg[P + 1] : n;
  int64_t b = pbeg[Q], be = (Q + 1 < npos) ? pbeg[Q + 1] : n;
  for (;;) {
    while (a < ae && a > pbeg[P] && r.region[a] == r.region[a - 1]) ++a;
    while (b < be && b > pbeg[Q] && r.region[b] == r.region[b - 1]) ++b;
    if (a == ae || b == be) return a == ae && b == be;
    if (list_entry(r, a) != list_entry(r, b)) return false;
    ++a;
    ++b;
  }
}
__global__ void k_list_rep(Recs r, int64_t n, const int64_t* pbeg, int64_t npos, const int64_t* nown,
                           const uint64_t* key, const uint32_t* idx, const int64_t* head, uint32_t* rep) {
  GRID_STRIDE(i, npos) {
    const uint32_t P = idx[i];
    uint32_t q = P;
    if (nown[P] > 1) {
      const uint32_t H = idx[head[i]];
      if (H != P && lists_equal(r, n, pbeg, npos, P, H)) q = H;
    }
    rep[P] = q;
  }
}
__global__ void k_pool_size(const int64_t* nown, const uint32_t* rep, int64_t npos, int64_t* psz) {
  GRID_STRIDE(P, npos) psz[P] = (nown[P] > 1 && rep[P] == (uint32_t)P) ? nown[P] + 1 : 0;
}
__global__ void k_pos_values(Recs r, int64_t n, const int64_t* pbeg, int64_t npos, const int64_t* nown,
                             const uint32_t* rep, const int64_t* poff, uint32_t* pool, uint64_t* pstart, uint8_t* plevel,
                             uint32_t* pval) {
  GRID_STRIDE(P, npos) {
    int64_t b = pbeg[P], e = (P + 1 < npos) ? pbeg[P + 1] : n;
    pstart[P] = r.start[b];
    plevel[P] = r.level[b];
    if (nown[P] == 1) {
      pval[P] = (uint32_t)((((uint32_t)r.region[b] << 1) | (r.kind[b] == RB_KIND_B ? 1u : 0u)) + 1u);
    } else if (rep[P] != (uint32_t)P) {
      pval[P] = RB_VALUE_LIST | (uint32_t)poff[rep[P]];
    } else {
      int64_t w = poff[P];
      pool[w++] = RB_POOL_COUNT_FLAG | (uint32_t)nown[P];
      for (int64_t k = b; k < e; ++k)
        if (k == b || r.region[k] != r.region[k - 1]) pool[w++] = list_entry(r, k);
      pval[P] = RB_VALUE_LIST | (uint32_t)poff[P];
    }
  }
}

// ---- index: root table level T0, node levels T0 + sum(ks[..]); row-major slots
struct IndexBuild {
  uint32_t* root;
  uint32_t* nodes[8];
  int ks[8];
  int nlev;
  int L, T0;
};

// pointer to the slot covering level-`lvl` cell (cx, cy) where lvl is T0 or a
// node level; descends existing pointers.
__device__ inline uint32_t* slot_ptr(const IndexBuild& B, uint64_t cx, uint64_t cy, int lvl) {
  // (cx, cy) at level lvl -> slot at the structure level == lvl
  int s = lvl - B.T0;
  uint32_t* slot = &B.root[((size_t)(cy >> s) << B.T0) | (size_t)(cx >> s)];
  int cur = B.T0;
  int li = 0;
  while (cur < lvl) {
    uint32_t v = *slot;
    int k = B.ks[li];
    cur += k;
    s = lvl - cur;
    uint64_t m = (1ull << k) - 1;
    size_t node = v & RB_VALUE_PAYLOAD;
    slot = &B.nodes[li][(node << (2 * k)) + ((((cy >> s) & m) << k) | ((cx >> s) & m))];
    ++li;
  }
  return slot;
}

// rows to fill for position P: cell at level l filled at structure level T
// (the smallest structure level >= l): side = 2^(T - l) slots.
__device__ inline int fill_level(const IndexBuild& B, int l) {
  if (l <= B.T0) return B.T0;
  int T = B.T0;
  for (int i = 0; i < B.nlev; ++i) { T += B.ks[i]; if (l <= T) return T; }
  return T;
}
// rows of the positions whose square spans more than 2^RB_FILL_WARP_D x 2^RB_FILL_WARP_D slots (smaller squares
// take k_fill_small, single slots k_fill_single)
#define RB_FILL_WARP_D 5
__global__ void k_fill_rows(IndexBuild B, const uint8_t* plevel, int64_t npos, int lo_excl, int hi_incl,
                            int64_t* rows) {
  GRID_STRIDE(P, npos) {
    int l = plevel[P];
    const int d = fill_level(B, l) - l;
    rows[P] = (l > lo_excl && l <= hi_incl && d > RB_FILL_WARP_D) ? (1ll << d) : 0;
  }
}
// positions whose square is 2^d x 2^d slots with 1 <= d <= RB_FILL_WARP_D: one warp per position, row by row
__global__ void k_fill_small(IndexBuild B, const uint64_t* pstart, const uint8_t* plevel, const uint32_t* pval,
                             int64_t npos, int lo_excl, int hi_incl) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t P = warp; P < npos; P += nw) {
    const int l = plevel[P];
    if (!(l > lo_excl && l <= hi_incl)) continue;
    const int T = fill_level(B, l), d = T - l;
    if (d < 1 || d > RB_FILL_WARP_D) continue;
    const uint64_t code = pstart[P] >> (2 * (B.L - l));
    const uint64_t cx = (uint64_t)compact1by1(code) << d, cy = (uint64_t)compact1by1(code >> 1) << d;
    const uint32_t w = 1u << d, v = pval[P];
    for (uint32_t r = 0; r < w; ++r) {
      uint32_t* base = slot_ptr(B, cx, cy + r, T);
      for (uint32_t t = lane; t < w; t += 32) base[t] = v;
    }
  }
}
// positions at a structure level (most of them: boundary leaves): one thread writes the one slot
__global__ void k_fill_single(IndexBuild B, const uint64_t* pstart, const uint8_t* plevel, const uint32_t* pval,
                              int64_t npos, int lo_excl, int hi_incl) {
  GRID_STRIDE(P, npos) {
    const int l = plevel[P];
    if (!(l > lo_excl && l <= hi_incl) || fill_level(B, l) != l) continue;
    const uint64_t code = pstart[P] >> (2 * (B.L - l));
    *slot_ptr(B, compact1by1(code), compact1by1(code >> 1), l) = pval[P];
  }
}
// one warp per row: fill 2^(T-l) slots of row `r` of position P's square
__global__ void k_fill(IndexBuild B, const uint64_t* pstart, const uint8_t* plevel, const uint32_t* pval,
                       const int64_t* roff, int64_t npos, int64_t nrows) {
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = warp; row < nrows; row += nw) {
    int64_t lo = 0, hi = npos;  // last P with roff[P] <= row
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if (roff[mid] <= row) lo = mid; else hi = mid;
    }
    int64_t P = lo;
    while (P + 1 < npos && roff[P + 1] <= row) ++P;  // skip empties
    int l = plevel[P];
    int T = fill_level(B, l);
    int d = T - l;
    uint64_t code = pstart[P] >> (2 * (B.L - l));
    uint64_t cx = (uint64_t)compact1by1(code) << d, cy = ((uint64_t)compact1by1(code >> 1) << d) + (row - roff[P]);
    uint64_t w = 1ull << d;
    uint32_t* base = slot_ptr(B, cx, cy, T);  // slots of one row are contiguous (row-major)
    for (uint64_t t = lane; t < w; t += 32) base[t] = pval[P];
  }
}
// node pointers: unique ancestors of positions finer than structure level T
__global__ void k_anc(const uint64_t* pstart, const uint8_t* plevel, int64_t npos, int T, int L, uint64_t* anc,
                      int64_t* flag) {
  GRID_STRIDE(P, npos) {
    flag[P] = plevel[P] > T ? 1 : 0;
    anc[P] = pstart[P] >> (2 * (L - T));
  }
}
__global__ void k_anc_unique(const uint64_t* a, int64_t n, int64_t* flag) {
  GRID_STRIDE(k, n) flag[k] = (k == 0 || a[k] != a[k - 1]) ? 1 : 0;
}
__global__ void k_set_ptr(IndexBuild B, const uint64_t* anc, int64_t n, int T) {
  GRID_STRIDE(k, n) {
    uint64_t c = anc[k];
    *slot_ptr(B, compact1by1(c), compact1by1(c >> 1), T) = RB_VALUE_NODE | (uint32_t)k;
  }
}
__global__ void k_compact_anc(const uint64_t* anc, const int64_t* flag, const int64_t* pos, int64_t n, uint64_t* out) {
  GRID_STRIDE(k, n) if (flag[k]) out[pos[k]] = anc[k];
}

// ---- shared-memory summary: level-S cell -> its single owner value when the
// whole cell has one (non-list, non-node) root value, else 0xffff
__global__ void k_summary(const uint32_t* root, int T0, int S, uint16_t* out) {
  const int d = T0 - S;
  const int64_t ncell = (int64_t)1 << (2 * S);
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t sub = (int64_t)1 << (2 * d);
  for (int64_t c = warp; c < ncell; c += nw) {
    const uint64_t sx = (uint64_t)c & ((1ull << S) - 1), sy = (uint64_t)c >> S;
    const uint32_t first = root[((sy << d) << T0) | (sx << d)];
    bool same = !(first & (RB_VALUE_NODE | RB_VALUE_LIST)) && first < 0xffffu;
    // warp-uniform trip count: every lane runs every iteration
    for (int64_t e0 = 0; e0 < sub && __all_sync(0xffffffffu, same); e0 += 32) {
      const int64_t e = e0 + lane;
      if (e < sub) {
        const uint64_t rx = (sx << d) | ((uint64_t)e & ((1ull << d) - 1)), ry = (sy << d) | ((uint64_t)e >> d);
        if (root[(ry << T0) | rx] != first) same = false;
      }
    }
    same = __all_sync(0xffffffffu, same);
    if (lane == 0) out[c] = same ? (uint16_t)first : (uint16_t)0xffffu;
  }
}

// ---- RB_LAYOUT_PACKED: palette blocks from the dense leaf nodes of the mixed root cells.
// Node n (2^pd x 2^pd leaves, row-major u32) -> 4^(pd-2) blocks of 4x4 leaves; block j of node n is
// pblk[n * 4^(pd-2) + j].  The 16 owner values of a block with <= 3 distinct values become a palette
// (in order of first appearance, unused entries = p0) and 2-bit indices; otherwise an escape block.
__device__ inline int pack_gather(const uint32_t* nodes, int64_t blk, int pd, uint32_t v[16]) {
  const int bw = pd - 2;
  const int64_t n = blk >> (2 * bw);
  const uint32_t j = (uint32_t)(blk & ((1ll << (2 * bw)) - 1));
  const uint32_t bx = j & ((1u << bw) - 1u), by = j >> bw;
  const uint32_t* nb = nodes + (n << (2 * pd));
  int nd = 0;
  uint32_t d0 = 0, d1 = 0, d2 = 0;
  for (int s = 0; s < 16; ++s) {
    const uint32_t x = (bx << 2) | (s & 3), y = (by << 2) | (s >> 2);
    v[s] = nb[((size_t)y << pd) | x];
    const uint32_t q = v[s];
    if (nd > 0 && q == d0) continue;
    if (nd > 1 && q == d1) continue;
    if (nd > 2 && q == d2) continue;
    if (nd == 0) d0 = q; else if (nd == 1) d1 = q; else if (nd == 2) d2 = q;
    ++nd;
  }
  return nd;
}
__global__ void k_pack_count(const uint32_t* nodes, int64_t nblocks, int pd, uint32_t* esc) {
  GRID_STRIDE(b, nblocks) {
    uint32_t v[16];
    esc[b] = pack_gather(nodes, b, pd, v) > 3 ? 1u : 0u;
  }
}
__global__ void k_pack_emit(const uint32_t* nodes, int64_t nblocks, int pd, const uint32_t* esc_off, uint4* blk,
                            uint32_t* wide) {
  GRID_STRIDE(b, nblocks) {
    uint32_t v[16];
    const int nd = pack_gather(nodes, b, pd, v);
    if (nd > 3) {
      const uint32_t e = esc_off[b];
      for (int s = 0; s < 16; ++s) wide[((size_t)e << 4) + s] = v[s];
      blk[b] = make_uint4(RB_VALUE_NODE | e, 0u, 0u, 0u);
      continue;
    }
    uint32_t p[3] = {v[0], v[0], v[0]};
    int np = 1;
    uint32_t idx = 0;
    for (int s = 0; s < 16; ++s) {
      int i = 0;
      while (i < np && p[i] != v[s]) ++i;
      if (i == np) p[np++] = v[s];
      idx |= (uint32_t)i << (2 * s);
    }
    blk[b] = make_uint4(p[0], p[1], p[2], idx);
  }
}
// root slots: node pointer n -> first block of node n
__global__ void k_pack_root(uint32_t* root, int64_t n, int pd) {
  GRID_STRIDE(k, n) {
    const uint32_t v = root[k];
    if (v & RB_VALUE_NODE) root[k] = RB_VALUE_NODE | ((v & RB_VALUE_PAYLOAD) << (2 * (pd - 2)));
  }
}
static cudaError_t excl_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, cudaStream_t s) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s);
  if (e) return e;
  DBuf t;
  if ((e = t.alloc(tb ? tb : 1))) return e;
  return cub::DeviceScan::ExclusiveSum(t.p, tb, in, out, n, s);
}

__global__ void k_split_off(const int64_t* soffs, int64_t n, int64_t* o2) {
  GRID_STRIDE(k, n) o2[k] = k + 3 * soffs[k];
}
__global__ void k_count_multi(const int64_t* nown, int64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  GRID_STRIDE(k, n) c += nown[k] > 1 ? 1 : 0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}
// interior cells, boundary cells, interior leaves after expansion to level L
__global__ void k_cell_stats(const uint8_t* level, const uint8_t* kind, int64_t n, int L, unsigned long long* out) {
  unsigned long long ni = 0, nb = 0, uni = 0;
  GRID_STRIDE(k, n) {
    if (kind[k] == RB_KIND_I) { ++ni; uni += 1ull << (2 * (L - level[k])); } else ++nb;
  }
  for (int o = 16; o > 0; o >>= 1) {
    ni += __shfl_xor_sync(0xffffffffu, ni, o);
    nb += __shfl_xor_sync(0xffffffffu, nb, o);
    uni += __shfl_xor_sync(0xffffffffu, uni, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (ni) atomicAdd(out, ni);
    if (nb) atomicAdd(out + 1, nb);
    if (uni) atomicAdd(out + 2, uni);
  }
}

// ---------------------------------------------------------------- driver
struct Ctx {
  cudaStream_t s;
  int64_t nv, nr, np;
};

// K5: overlay + index from hierarchical cells (cell k belongs to covering
// cp[k]; covering -> region via cov_region).  Cells are only read.
// RB_BUILD_TRACE=1: per-phase wall time of the build (stream-synchronised), on stderr
struct BuildTrace {
  cudaStream_t s;
  bool on;
  std::chrono::steady_clock::time_point t;
  explicit BuildTrace(cudaStream_t st) : s(st), on(getenv("RB_BUILD_TRACE") != nullptr), t(std::chrono::steady_clock::now()) {}
  void operator()(const char* phase) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "rb build %-28s %9.2f ms\n", phase, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};
static int index_impl(int L, int64_t total_cells, const int32_t* cp_in, const uint8_t* cl_in, const uint64_t* cc_in,
                      const uint8_t* ck_in, const int32_t* cov_region, const rb_build_opts* opts, cudaStream_t s,
                      rb_approx* A) {
  BuildTrace trace(s);
  // ---- K5 overlay: records sorted by (start, level, region, kind)
  int64_t n = total_cells;
  DBuf rs, rl, rr, rk;
  RB_CUDA(rs.alloc(std::max<int64_t>(n, 1) * 8));
  RB_CUDA(rl.alloc(std::max<int64_t>(n, 1)));
  RB_CUDA(rr.alloc(std::max<int64_t>(n, 1) * 4));
  RB_CUDA(rk.alloc(std::max<int64_t>(n, 1)));
  Recs R{rs.as<uint64_t>(), rl.as<uint8_t>(), rr.as<int32_t>(), rk.as<uint8_t>()};
  {
    DBuf st, sec, idx, tmp;
    RB_CUDA(st.alloc(std::max<int64_t>(n, 1) * 8));
    RB_CUDA(sec.alloc(std::max<int64_t>(n, 1) * 8));
    RB_CUDA(idx.alloc(std::max<int64_t>(n, 1) * 4));
    RB_CUDA(tmp.alloc(std::max<int64_t>(n, 1) * 8));
    if (n) k_cell_keys<<<nblk(n), 256, 0, s>>>(cp_in, cl_in, cc_in,
                                               ck_in, cov_region, n, L, st.as<uint64_t>(),
                                               sec.as<uint64_t>(), idx.as<uint32_t>());
    RB_CUDA(cudaGetLastError());
    RB_CUDA(radix_sort_pairs(sec.as<uint64_t>(), idx.as<uint32_t>(), n, 46, s));
    if (n) k_gather_u64<<<nblk(n), 256, 0, s>>>(st.as<uint64_t>(), idx.as<uint32_t>(), n, tmp.as<uint64_t>());
    RB_CUDA(radix_sort_pairs(tmp.as<uint64_t>(), idx.as<uint32_t>(), n, std::max(1, 2 * L), s));
    if (n) k_gather_recs<<<nblk(n), 256, 0, s>>>(idx.as<uint32_t>(), n, cp_in, cl_in,
                                                 cc_in, ck_in, cov_region, L, R);
    RB_CUDA(cudaGetLastError());
  }
  DBuf head, hpos, pb;
  int64_t npos = 0;
  for (int iter = 0; iter <= L + 1; ++iter) {
    RB_CUDA(head.alloc((n + 1) * 8));
    RB_CUDA(hpos.alloc((n + 1) * 8));
    RB_CUDA(cudaMemsetAsync(head.p, 0, (n + 1) * 8, s));
    if (n) k_pos_head<<<nblk(n), 256, 0, s>>>(R, n, head.as<int64_t>());
    RB_CUDA(excl_scan_i64(head.as<int64_t>(), hpos.as<int64_t>(), n + 1, s));
    npos = d2h(hpos.as<int64_t>() + n, s);
    RB_CUDA(pb.alloc(std::max<int64_t>(npos, 1) * 8));
    if (n) k_pos_list<<<nblk(n), 256, 0, s>>>(head.as<int64_t>(), hpos.as<int64_t>(), n, pb.as<int64_t>());
    DBuf split, soffs;
    RB_CUDA(split.alloc((n + 1) * 8));
    RB_CUDA(soffs.alloc((n + 1) * 8));
    RB_CUDA(cudaMemsetAsync(split.p, 0, (n + 1) * 8, s));
    if (n) k_container<<<nblk(n), 256, 0, s>>>(R, n, head.as<int64_t>(), hpos.as<int64_t>(), pb.as<int64_t>(), npos,
                                               L, split.as<int64_t>());
    RB_CUDA(cudaGetLastError());
    RB_CUDA(excl_scan_i64(split.as<int64_t>(), soffs.as<int64_t>(), n + 1, s));
    int64_t nsplit = d2h(soffs.as<int64_t>() + n, s);
    if (nsplit == 0) break;
    if (iter > L) return fail(RB_CAPACITY_ERROR, "overlay did not converge");
    // new offsets: k + 3 * (#splits before k)
    int64_t n2 = n + 3 * nsplit;
    DBuf o2;
    RB_CUDA(o2.alloc((n + 1) * 8));
    k_split_off<<<nblk(n + 1), 256, 0, s>>>(soffs.as<int64_t>(), n + 1, o2.as<int64_t>());  // k + 3 * splits before k
    RB_CUDA(cudaGetLastError());
    DBuf s2, l2, r2, k2;
    RB_CUDA(s2.alloc(n2 * 8));
    RB_CUDA(l2.alloc(n2));
    RB_CUDA(r2.alloc(n2 * 4));
    RB_CUDA(k2.alloc(n2));
    Recs R2{s2.as<uint64_t>(), l2.as<uint8_t>(), r2.as<int32_t>(), k2.as<uint8_t>()};
    k_split<<<nblk(n), 256, 0, s>>>(R, n, split.as<int64_t>(), o2.as<int64_t>(), L, R2);
    RB_CUDA(cudaGetLastError());
    // re-sort R2 by (start, level, region, kind)
    DBuf st, sec, idx, tmp, s3, l3, r3, k3;
    RB_CUDA(st.alloc(n2 * 8));
    RB_CUDA(sec.alloc(n2 * 8));
    RB_CUDA(idx.alloc(n2 * 4));
    RB_CUDA(tmp.alloc(n2 * 8));
    k_rec_keys<<<nblk(n2), 256, 0, s>>>(R2, n2, st.as<uint64_t>(), sec.as<uint64_t>(), idx.as<uint32_t>());
    RB_CUDA(radix_sort_pairs(sec.as<uint64_t>(), idx.as<uint32_t>(), n2, 46, s));
    k_gather_u64<<<nblk(n2), 256, 0, s>>>(st.as<uint64_t>(), idx.as<uint32_t>(), n2, tmp.as<uint64_t>());
    RB_CUDA(radix_sort_pairs(tmp.as<uint64_t>(), idx.as<uint32_t>(), n2, std::max(1, 2 * L), s));
    RB_CUDA(s3.alloc(n2 * 8));
    RB_CUDA(l3.alloc(n2));
    RB_CUDA(r3.alloc(n2 * 4));
    RB_CUDA(k3.alloc(n2));
    Recs R3{s3.as<uint64_t>(), l3.as<uint8_t>(), r3.as<int32_t>(), k3.as<uint8_t>()};
    k_rec_gather<<<nblk(n2), 256, 0, s>>>(idx.as<uint32_t>(), n2, R2, R3);
    RB_CUDA(cudaGetLastError());
    RB_CUDA(cudaStreamSynchronize(s));
    rs = std::move(s3); rl = std::move(l3); rr = std::move(r3); rk = std::move(k3);
    R = Recs{rs.as<uint64_t>(), rl.as<uint8_t>(), rr.as<int32_t>(), rk.as<uint8_t>()};
    n = n2;
  }
  trace("K5 overlay (sort + split)");
  // owner values per position
  DBuf nown, psz, poff, pstart, plevel, pval;
  RB_CUDA(nown.alloc((npos + 1) * 8));
  RB_CUDA(psz.alloc((npos + 1) * 8));
  RB_CUDA(poff.alloc((npos + 1) * 8));
  RB_CUDA(cudaMemsetAsync(nown.p, 0, (npos + 1) * 8, s));
  RB_CUDA(cudaMemsetAsync(psz.p, 0, (npos + 1) * 8, s));
  if (npos) k_pos_owners<<<nblk(npos), 256, 0, s>>>(R, n, pb.as<int64_t>(), npos, nown.as<int64_t>());
  DBuf rep;
  RB_CUDA(rep.alloc(std::max<int64_t>(npos, 1) * 4));
  if (npos) {  // shared owner lists (identical owner sets -> one pool entry)
    if (npos >= ((int64_t)1 << 32)) return fail(RB_CAPACITY_ERROR, "more than 2^32 indexed positions");
    DBuf hkey, hidx, hhead;
    RB_CUDA(hkey.alloc(npos * 8));
    RB_CUDA(hidx.alloc(npos * 4));
    RB_CUDA(hhead.alloc(npos * 8));
    k_list_hash<<<nblk(npos), 256, 0, s>>>(R, n, pb.as<int64_t>(), npos, nown.as<int64_t>(), hkey.as<uint64_t>(),
                                           hidx.as<uint32_t>());
    RB_CUDA(cudaGetLastError());
    RB_CUDA(radix_sort_pairs(hkey.as<uint64_t>(), hidx.as<uint32_t>(), npos, 64, s));
    k_run_head<<<nblk(npos), 256, 0, s>>>(hkey.as<uint64_t>(), npos, hhead.as<int64_t>());
    RB_CUDA(cudaGetLastError());
    RB_CUDA(incl_max_scan_i64(hhead.as<int64_t>(), npos, s));
    k_list_rep<<<nblk(npos), 256, 0, s>>>(R, n, pb.as<int64_t>(), npos, nown.as<int64_t>(), hkey.as<uint64_t>(),
                                          hidx.as<uint32_t>(), hhead.as<int64_t>(), rep.as<uint32_t>());
    RB_CUDA(cudaGetLastError());
  }
  if (npos) k_pool_size<<<nblk(npos), 256, 0, s>>>(nown.as<int64_t>(), rep.as<uint32_t>(), npos, psz.as<int64_t>());
  RB_CUDA(excl_scan_i64(psz.as<int64_t>(), poff.as<int64_t>(), npos + 1, s));
  int64_t npool = d2h(poff.as<int64_t>() + npos, s);
  if (npool >= (int64_t)RB_VALUE_PAYLOAD) return fail(RB_CAPACITY_ERROR, "owner pool exceeds 2^30 entries");
  RB_CUDA(A->pool.alloc_persistent(std::max<int64_t>(npool, 1) * 4));
  A->pool_len = npool;
  RB_CUDA(pstart.alloc(std::max<int64_t>(npos, 1) * 8));
  RB_CUDA(plevel.alloc(std::max<int64_t>(npos, 1)));
  RB_CUDA(pval.alloc(std::max<int64_t>(npos, 1) * 4));
  if (npos) k_pos_values<<<nblk(npos), 256, 0, s>>>(R, n, pb.as<int64_t>(), npos, nown.as<int64_t>(),
                                                    rep.as<uint32_t>(), poff.as<int64_t>(), A->pool.as<uint32_t>(), pstart.as<uint64_t>(),
                                                    plevel.as<uint8_t>(), pval.as<uint32_t>());
  RB_CUDA(cudaGetLastError());
  {
    DBuf cm;
    RB_CUDA(cm.alloc(8));
    RB_CUDA(cudaMemsetAsync(cm.p, 0, 8, s));
    if (npos) k_count_multi<<<nblk(npos), 256, 0, s>>>(nown.as<int64_t>(), npos, cm.as<unsigned long long>());
    RB_CUDA(cudaGetLastError());
    A->stats.n_multi_owner = (int64_t)d2h(cm.as<unsigned long long>(), s);
    A->stats.n_positions = npos;
  }
  rs.release(); rl.release(); rr.release(); rk.release(); head.release(); hpos.release(); pb.release();

  if (opts->layout == RB_LAYOUT_KEYS) {
    // sorted 64-bit cell keys: the disjoint positions already come sorted by start key
    A->T0 = 0;
    A->k = std::max(1, opts->radix_width / 2);
    A->nkeys = npos;
    int bits = 0;  // ~1 cell per bucket up to 2^28 cells (a 2 GB table); 0 bits for L = 0
    while (bits < std::min(2 * L, 29) && ((int64_t)1 << bits) < 2 * std::max<int64_t>(npos, 1)) ++bits;
    A->kshift = 2 * L - bits;
    const int64_t nslots = ((int64_t)1 << bits) + 1;
    RB_CUDA(A->ktab.alloc_persistent(nslots * 4));
    k_key_table<<<nblk(nslots), 256, 0, s>>>(pstart.as<uint64_t>(), npos, A->kshift, nslots, A->ktab.as<uint32_t>());
    RB_CUDA(cudaGetLastError());
    RB_CUDA(A->keys.alloc_persistent(std::max<int64_t>(npos, 1) * 16));
    if (npos) k_key_records<<<nblk(npos), 256, 0, s>>>(pstart.as<uint64_t>(), plevel.as<uint8_t>(), pval.as<uint32_t>(),
                                                       npos, A->keys.as<uint4>());
    RB_CUDA(A->root.alloc_persistent(4));  // unused (no radix table levels)
    RB_CUDA(cudaMemsetAsync(A->root.p, 0, 4, s));
    A->root_entries = 1;
    A->S = -1;
    {  // level-S summary for the shared-memory fast path, as for the radix table
      int Smax = RB_SUMMARY_DEFAULT;
      if (const char* e = getenv("RB_SUMMARY_LEVEL")) Smax = std::min(atoi(e), 8);
      if (Smax >= 0 && 2 * (int64_t)A->n_regions + 1 < 0xffff) {
        const int S = std::min(Smax, L);
        RB_CUDA(A->summary.alloc_persistent(((size_t)2 << (2 * S))));
        k_key_summary<<<nblk((int64_t)1 << (2 * S)), 256, 0, s>>>(A->keys.as<uint4>(), npos, L, S,
                                                                  A->summary.as<uint16_t>());
        RB_CUDA(cudaGetLastError());
        A->S = S;
      }
    }
    A->stats.root_level = 0;
    A->stats.node_levels = 0;
    A->stats.n_nodes = 0;
    A->stats.index_bytes = npos * 16 + nslots * 4 + npool * 4;
    RB_CUDA(cudaStreamSynchronize(s));
    return RB_OK;
  }

  trace("K5 owner values + lists");
  // ---- index geometry
  int k = std::max(1, opts->radix_width / 2);
  int T0;
  std::vector<int> ks;
  if (opts->layout == RB_LAYOUT_DENSE) {
    T0 = L;
  } else {
    // automatic root level: a 2^12 x 2^12 root (64 MB, L2-resident) leaves one node level up to L = 16
    // (C2: 0.503 -> 0.487 ms over T0 = 10) and two up to L = 20 (C4, eps-matched grid: 1.70 -> 1.64 ms
    // per 200M points over T0 = 11; only the data's 19 MB of it is touched)
    T0 = opts->root_level >= 0 ? std::min(opts->root_level, L) : (L <= 20 ? std::min(L, 12) : 11);
    if (opts->layout == RB_LAYOUT_PACKED) {
      // L - T0 in [2, 5]: nodes of 4x4-leaf palette blocks right below the root; in [6, 8]: one radix node
      // level of u32 slots (L - T0 - 4 bits a side), then packed nodes of 16 x 16 leaves
      T0 = opts->root_level >= 0 ? opts->root_level : (L >= 6 ? L - 6 : 0);
      if (L < 2) return fail(RB_CONFIG_ERROR, "the packed layout needs max_level >= 2");
      if (L - T0 < 2 || L - T0 > 8)
        return fail(RB_CONFIG_ERROR, "packed layout: root_level must lie in [max_level - 8, max_level - 2]");
    }
    int rem = L - T0;
    if (const char* e = getenv("RB_NODE_KS")) {  // experiments: explicit node split, e.g. "2,5"
      for (const char* c = e; *c;) {
        const int v = atoi(c);
        if (v <= 0 || v > rem) { ks.clear(); break; }
        ks.push_back(v);
        rem -= v;
        while (*c && *c != ',') ++c;
        if (*c == ',') ++c;
      }
      if (rem != 0) return fail(RB_CONFIG_ERROR, "RB_NODE_KS must split L - root_level exactly");
    }
    if (opts->layout == RB_LAYOUT_PACKED) {  // dense nodes, packed below
      ks.clear();
      if (rem >= 6) { ks.push_back(rem - 4); ks.push_back(4); } else ks.push_back(rem);
    }
    if (ks.empty() && rem > 0) {
      int first = rem % k ? rem % k : k;
      ks.push_back(first);
      rem -= first;
      while (rem > 0) { ks.push_back(k); rem -= k; }
    }
  }
  if ((int)ks.size() > 8) return fail(RB_CONFIG_ERROR, "too many index levels (raise root_level or radix_width)");
  // the point-pass kernels address root slots with 32-bit indices ((row << T0) | col): T0 <= 16 (17.2 GB)
  if (T0 > 16)
    return fail(RB_CAPACITY_ERROR, "root table above level 16 (17.2 GB) is not supported; use the trie or packed "
                                   "layout with a lower root_level");
  {
    size_t fr = 0, tot = 0;
    RB_CUDA(cudaMemGetInfo(&fr, &tot));
    if ((double)((int64_t)4 << (2 * T0)) > 0.9 * (double)fr)
      return fail(RB_CAPACITY_ERROR, "root table of level " + std::to_string(T0) + " does not fit in free device memory");
  }
  A->T0 = T0;
  A->k = k;
  A->root_entries = (int64_t)1 << (2 * T0);
  RB_CUDA(A->root.alloc_persistent(A->root_entries * 4));
  RB_CUDA(cudaMemsetAsync(A->root.p, 0, A->root_entries * 4, s));
  IndexBuild B{};
  B.root = A->root.as<uint32_t>();
  B.nlev = (int)ks.size();
  B.L = L;
  B.T0 = T0;
  for (int i = 0; i < B.nlev; ++i) B.ks[i] = ks[i];
  // count nodes per level: unique ancestors at structure level T_{i-1} of positions finer than it
  std::vector<int64_t> nnodes(B.nlev, 0);
  std::vector<DBuf> ancs(B.nlev);
  {
    int T = T0;
    for (int i = 0; i < B.nlev; ++i) {
      DBuf anc, fl2, pos2, sel, uf, up;
      RB_CUDA(anc.alloc(std::max<int64_t>(npos, 1) * 8));
      RB_CUDA(fl2.alloc((npos + 1) * 8));
      RB_CUDA(pos2.alloc((npos + 1) * 8));
      RB_CUDA(cudaMemsetAsync(fl2.p, 0, (npos + 1) * 8, s));
      if (npos) k_anc<<<nblk(npos), 256, 0, s>>>(pstart.as<uint64_t>(), plevel.as<uint8_t>(), npos, T, L,
                                                 anc.as<uint64_t>(), fl2.as<int64_t>());
      RB_CUDA(excl_scan_i64(fl2.as<int64_t>(), pos2.as<int64_t>(), npos + 1, s));
      int64_t nsel = d2h(pos2.as<int64_t>() + npos, s);
      RB_CUDA(sel.alloc(std::max<int64_t>(nsel, 1) * 8));
      if (npos) k_compact_anc<<<nblk(npos), 256, 0, s>>>(anc.as<uint64_t>(), fl2.as<int64_t>(), pos2.as<int64_t>(),
                                                         npos, sel.as<uint64_t>());
      RB_CUDA(uf.alloc((nsel + 1) * 8));
      RB_CUDA(up.alloc((nsel + 1) * 8));
      RB_CUDA(cudaMemsetAsync(uf.p, 0, (nsel + 1) * 8, s));
      if (nsel) k_anc_unique<<<nblk(nsel), 256, 0, s>>>(sel.as<uint64_t>(), nsel, uf.as<int64_t>());
      RB_CUDA(excl_scan_i64(uf.as<int64_t>(), up.as<int64_t>(), nsel + 1, s));
      int64_t nu = d2h(up.as<int64_t>() + nsel, s);
      DBuf u;
      RB_CUDA(u.alloc(std::max<int64_t>(nu, 1) * 8));
      if (nsel) k_compact_anc<<<nblk(nsel), 256, 0, s>>>(sel.as<uint64_t>(), uf.as<int64_t>(), up.as<int64_t>(), nsel,
                                                         u.as<uint64_t>());
      RB_CUDA(cudaGetLastError());
      if (nu >= (int64_t)RB_VALUE_PAYLOAD) return fail(RB_CAPACITY_ERROR, "index node count exceeds 2^30");
      nnodes[i] = nu;
      ancs[i] = std::move(u);
      T += ks[i];
    }
  }
  std::vector<DBuf> node_bufs(B.nlev);
  int64_t total_nodes = 0, node_bytes = 0;
  for (int i = 0; i < B.nlev; ++i) {
    int64_t bytes = nnodes[i] * ((int64_t)4 << (2 * ks[i]));
    RB_CUDA(node_bufs[i].alloc_persistent(std::max<int64_t>(bytes, 4)));
    RB_CUDA(cudaMemsetAsync(node_bufs[i].p, 0, std::max<int64_t>(bytes, 4), s));
    B.nodes[i] = node_bufs[i].as<uint32_t>();
    total_nodes += nnodes[i];
    node_bytes += bytes;
  }
  // fill: root, then per node level: pointers, then positions
  auto fill_range = [&](int lo_excl, int hi_incl) -> int {
    DBuf rows, roff;
    RB_CUDA(rows.alloc((npos + 1) * 8));
    RB_CUDA(roff.alloc((npos + 1) * 8));
    RB_CUDA(cudaMemsetAsync(rows.p, 0, (npos + 1) * 8, s));
    if (npos) {
      k_fill_rows<<<nblk(npos), 256, 0, s>>>(B, plevel.as<uint8_t>(), npos, lo_excl, hi_incl, rows.as<int64_t>());
      k_fill_single<<<nblk(npos), 256, 0, s>>>(B, pstart.as<uint64_t>(), plevel.as<uint8_t>(), pval.as<uint32_t>(),
                                               npos, lo_excl, hi_incl);
      k_fill_small<<<nblk(npos * 32), 256, 0, s>>>(B, pstart.as<uint64_t>(), plevel.as<uint8_t>(), pval.as<uint32_t>(),
                                                   npos, lo_excl, hi_incl);
    }
    RB_CUDA(excl_scan_i64(rows.as<int64_t>(), roff.as<int64_t>(), npos + 1, s));
    int64_t nrows = d2h(roff.as<int64_t>() + npos, s);
    if (nrows) k_fill<<<nblk(nrows * 32), 256, 0, s>>>(B, pstart.as<uint64_t>(), plevel.as<uint8_t>(),
                                                      pval.as<uint32_t>(), roff.as<int64_t>(), npos, nrows);
    RB_CUDA(cudaGetLastError());
    RB_CUDA(cudaStreamSynchronize(s));
    return RB_OK;
  };
  trace("index node counts");
  int st = fill_range(-1, T0);
  if (st) return st;
  {
    int T = T0;
    for (int i = 0; i < B.nlev; ++i) {
      if (nnodes[i]) k_set_ptr<<<nblk(nnodes[i]), 256, 0, s>>>(B, ancs[i].as<uint64_t>(), nnodes[i], T);
      RB_CUDA(cudaGetLastError());
      RB_CUDA(cudaStreamSynchronize(s));
      st = fill_range(T, T + ks[i]);
      if (st) return st;
      T += ks[i];
    }
  }
  A->node_levels.clear();
  if (opts->layout == RB_LAYOUT_PACKED && B.nlev == 2) {
    // radix node level 0 stays u32; the level-1 nodes (16 x 16 leaves) become 16 palette blocks each
    const int pd = ks[1];
    const int64_t bpn = (int64_t)1 << (2 * (pd - 2));
    const int64_t nblocks = nnodes[1] * bpn;
    if (nblocks >= (int64_t)RB_VALUE_PAYLOAD) return fail(RB_CAPACITY_ERROR, "packed index exceeds 2^30 blocks");
    DBuf esc, eoff;
    RB_CUDA(esc.alloc((nblocks + 1) * 4));
    RB_CUDA(eoff.alloc((nblocks + 1) * 4));
    RB_CUDA(cudaMemsetAsync(esc.p, 0, (nblocks + 1) * 4, s));
    if (nblocks) k_pack_count<<<nblk(nblocks), 256, 0, s>>>(node_bufs[1].as<uint32_t>(), nblocks, pd, esc.as<uint32_t>());
    RB_CUDA(cudaGetLastError());
    RB_CUDA(excl_scan_u32(esc.as<uint32_t>(), eoff.as<uint32_t>(), nblocks + 1, s));
    const int64_t nwide = d2h(eoff.as<uint32_t>() + nblocks, s);
    RB_CUDA(A->pblk.alloc_persistent(std::max<int64_t>(nblocks, 1) * 16));
    RB_CUDA(A->pwide.alloc_persistent(std::max<int64_t>(nwide, 1) * 64));
    if (nblocks)
      k_pack_emit<<<nblk(nblocks), 256, 0, s>>>(node_bufs[1].as<uint32_t>(), nblocks, pd, eoff.as<uint32_t>(),
                                                A->pblk.as<uint4>(), A->pwide.as<uint32_t>());
    const int64_t n0 = nnodes[0] << (2 * ks[0]);  // level-0 slots: node pointer n -> first block of node n
    if (n0) k_pack_root<<<nblk(n0), 256, 0, s>>>(node_bufs[0].as<uint32_t>(), n0, pd);
    RB_CUDA(cudaGetLastError());
    RB_CUDA(cudaStreamSynchronize(s));
    node_bufs.pop_back();
    A->pd = pd;
    A->n_pblk = nblocks;
    A->n_pwide = nwide;
    node_bytes = (nnodes[0] << (2 * ks[0])) * 4 + nblocks * 16 + nwide * 64;
  } else if (opts->layout == RB_LAYOUT_PACKED) {
    const int pd = L - T0;
    const int64_t bpr = (int64_t)1 << (2 * (pd - 2));
    const int64_t nblocks = nnodes[0] * bpr;
    if (nblocks >= (int64_t)RB_VALUE_PAYLOAD) return fail(RB_CAPACITY_ERROR, "packed index exceeds 2^30 blocks");
    DBuf esc, eoff;
    RB_CUDA(esc.alloc((nblocks + 1) * 4));
    RB_CUDA(eoff.alloc((nblocks + 1) * 4));
    RB_CUDA(cudaMemsetAsync(esc.p, 0, (nblocks + 1) * 4, s));
    if (nblocks) k_pack_count<<<nblk(nblocks), 256, 0, s>>>(node_bufs[0].as<uint32_t>(), nblocks, pd, esc.as<uint32_t>());
    RB_CUDA(cudaGetLastError());
    RB_CUDA(excl_scan_u32(esc.as<uint32_t>(), eoff.as<uint32_t>(), nblocks + 1, s));
    const int64_t nwide = d2h(eoff.as<uint32_t>() + nblocks, s);
    RB_CUDA(A->pblk.alloc_persistent(std::max<int64_t>(nblocks, 1) * 16));
    RB_CUDA(A->pwide.alloc_persistent(std::max<int64_t>(nwide, 1) * 64));
    if (nblocks)
      k_pack_emit<<<nblk(nblocks), 256, 0, s>>>(node_bufs[0].as<uint32_t>(), nblocks, pd, eoff.as<uint32_t>(),
                                                A->pblk.as<uint4>(), A->pwide.as<uint32_t>());
    k_pack_root<<<nblk(A->root_entries), 256, 0, s>>>(A->root.as<uint32_t>(), A->root_entries, pd);
    RB_CUDA(cudaGetLastError());
    RB_CUDA(cudaStreamSynchronize(s));
    node_bufs.clear();
    A->pd = pd;
    A->n_pblk = nblocks;
    A->n_pwide = nwide;
    node_bytes = nblocks * 16 + nwide * 64;
  }
  for (size_t i = 0; i < node_bufs.size(); ++i) {
    A->node_levels.push_back(ks[i]);
    A->node_bufs.push_back(std::move(node_bufs[i]));
  }
  A->n_nodes = total_nodes;
  A->stats.n_nodes = total_nodes;
  trace("index fill + pack");
  // summary table for the shared-memory fast path (owner values must fit u16)
  {
    int Smax = RB_SUMMARY_DEFAULT;
    if (const char* e = getenv("RB_SUMMARY_LEVEL")) Smax = std::min(atoi(e), 8);  // <= 128 KB of shared memory
    A->S = -1;
    if (Smax >= 0 && 2 * (int64_t)A->n_regions + 1 < 0xffff) {
      const int S = std::min(Smax, T0);
      RB_CUDA(A->summary.alloc_persistent(((size_t)2 << (2 * S))));
      k_summary<<<nblk(((int64_t)32 << (2 * S))), 256, 0, s>>>(A->root.as<uint32_t>(), T0, S, A->summary.as<uint16_t>());
      RB_CUDA(cudaGetLastError());
      A->S = S;
    }
  }
  A->stats.root_level = T0;
  A->stats.node_levels = k;
  A->stats.index_bytes = A->root_entries * 4 + node_bytes + npool * 4;
  RB_CUDA(cudaStreamSynchronize(s));
  RB_CUDA(cudaStreamSynchronize(s));
  return RB_OK;
}

static int build_impl(const rb_grid* grid, const rb_polygons* P, const rb_build_opts* opts, cudaStream_t s,
                      rb_approx* A) {
  auto t_start = std::chrono::steady_clock::now();
  const int L = grid->max_level;
  const int64_t nv = P->n_vertices, nr = P->n_rings, np = P->n_polygons;
  GridD g{grid->origin_x, grid->origin_y, ldexp(grid->extent, -L), ldexp(1.0, L), L};
  A->stats.max_level = L;
  A->stats.n_regions = P->n_regions;

  BuildTrace trace(s);
  // ---- host-side structural checks (copy small offset arrays)
  std::vector<int64_t> h_ring(nr + 1), h_pr(np + 1);
  RB_CUDA(cudaMemcpyAsync(h_ring.data(), P->ring_off, (nr + 1) * 8, cudaMemcpyDeviceToHost, s));
  RB_CUDA(cudaMemcpyAsync(h_pr.data(), P->poly_ring_off, (np + 1) * 8, cudaMemcpyDeviceToHost, s));
  RB_CUDA(cudaStreamSynchronize(s));
  if (h_ring[0] != 0 || h_ring[nr] != nv || h_pr[0] != 0 || h_pr[np] != nr)
    return fail(RB_GEOMETRY_ERROR, "polygon CSR offsets inconsistent");
  for (int64_t r = 0; r < nr; ++r)
    if (h_ring[r + 1] - h_ring[r] < 3) return fail(RB_GEOMETRY_ERROR, "ring " + std::to_string(r) + " has fewer than 3 vertices");
  for (int64_t p = 0; p < np; ++p)
    if (h_pr[p + 1] <= h_pr[p]) return fail(RB_GEOMETRY_ERROR, "polygon " + std::to_string(p) + " has no ring");
  {
    std::vector<int32_t> h_reg(np);
    if (np) RB_CUDA(cudaMemcpyAsync(h_reg.data(), P->poly_region, np * 4, cudaMemcpyDeviceToHost, s));
    RB_CUDA(cudaStreamSynchronize(s));
    for (int64_t p = 0; p < np; ++p)
      if (h_reg[p] < 0 || h_reg[p] >= P->n_regions) return fail(RB_CONFIG_ERROR, "poly_region out of range");
  }

  // ---- K0
  DBuf ring_poly, gx, gy, vnext, vpoly, flags, mbr;
  RB_CUDA(ring_poly.alloc(std::max<int64_t>(nr, 1) * 4));
  RB_CUDA(gx.alloc(std::max<int64_t>(nv, 1) * 8));
  RB_CUDA(gy.alloc(std::max<int64_t>(nv, 1) * 8));
  RB_CUDA(vnext.alloc(std::max<int64_t>(nv, 1) * 8));
  RB_CUDA(vpoly.alloc(std::max<int64_t>(nv, 1) * 4));
  RB_CUDA(flags.alloc(4));
  RB_CUDA(mbr.alloc(std::max<int64_t>(np, 1) * 16));
  RB_CUDA(cudaMemsetAsync(flags.p, 0, 4, s));
  if (np) k_ring_poly<<<nblk(np), 256, 0, s>>>(P->poly_ring_off, np, ring_poly.as<int32_t>());
  if (nv) k_vertex<<<nblk(nv), 256, 0, s>>>(P->vx, P->vy, nv, P->ring_off, nr, ring_poly.as<int32_t>(), g,
                                            gx.as<double>(), gy.as<double>(), vnext.as<int64_t>(), vpoly.as<int32_t>(),
                                            flags.as<int>());
  if (np) k_poly_info<<<nblk(np), 256, 0, s>>>(P->vx, P->vy, gx.as<double>(), gy.as<double>(), P->ring_off,
                                               P->poly_ring_off, np, g.lim, mbr.as<uint32_t>(), flags.as<int>());
  RB_CUDA(cudaGetLastError());
  int fl = d2h(flags.as<int>(), s);
  if (fl & 1) return fail(RB_GEOMETRY_ERROR, "non-finite polygon vertex");
  if (fl & 4) return fail(RB_GEOMETRY_ERROR, "polygon outer ring has zero area");
  if (fl & 2) return fail(RB_DOMAIN_ERROR, "polygon vertex outside the grid domain");

  const double* dgx = gx.as<double>();
  const double* dgy = gy.as<double>();
  const int64_t* dvn = vnext.as<int64_t>();

  trace("checks + K0 vertices");
  // ---- K2 edge walk
  DBuf cnt, off;
  RB_CUDA(cnt.alloc((nv + 1) * 8));
  RB_CUDA(off.alloc((nv + 1) * 8));
  RB_CUDA(cudaMemsetAsync(cnt.p, 0, (nv + 1) * 8, s));
  if (nv) k_walk_count<<<nblk(nv), 256, 0, s>>>(dgx, dgy, dvn, nv, cnt.as<int64_t>());
  RB_CUDA(excl_scan_i64(cnt.as<int64_t>(), off.as<int64_t>(), nv + 1, s));
  int64_t nwalk = d2h(off.as<int64_t>() + nv, s);
  DBuf walk, pbeg, pend;
  RB_CUDA(walk.alloc(std::max<int64_t>(nwalk, 1) * 8));
  RB_CUDA(pbeg.alloc(std::max<int64_t>(np, 1) * 8));
  RB_CUDA(pend.alloc(std::max<int64_t>(np, 1) * 8));
  if (nv) k_walk_emit<<<nblk(nv), 256, 0, s>>>(dgx, dgy, dvn, nv, off.as<int64_t>(), walk.as<uint64_t>());
  if (np) k_seg_bounds<<<nblk(np), 256, 0, s>>>(off.as<int64_t>(), P->ring_off, P->poly_ring_off, np,
                                                pbeg.as<int64_t>(), pend.as<int64_t>());
  RB_CUDA(cudaGetLastError());
  RB_CUDA(seg_sort_keys(walk.as<uint64_t>(), nwalk, np, pbeg.as<int64_t>(), pend.as<int64_t>(), s));
  // unique within polygon segments
  DBuf uflag, upos, part, ubeg, uend;
  RB_CUDA(uflag.alloc((nwalk + 1) * 8));
  RB_CUDA(upos.alloc((nwalk + 1) * 8));
  RB_CUDA(cudaMemsetAsync(uflag.p, 0, (nwalk + 1) * 8, s));
  if (nwalk) k_unique_flags<<<nblk(nwalk), 256, 0, s>>>(walk.as<uint64_t>(), nwalk, pbeg.as<int64_t>(), np,
                                                        uflag.as<int64_t>());
  RB_CUDA(excl_scan_i64(uflag.as<int64_t>(), upos.as<int64_t>(), nwalk + 1, s));
  int64_t npart = d2h(upos.as<int64_t>() + nwalk, s);
  RB_CUDA(part.alloc(std::max<int64_t>(npart, 1) * 8));
  RB_CUDA(ubeg.alloc(std::max<int64_t>(np, 1) * 8));
  RB_CUDA(uend.alloc(std::max<int64_t>(np, 1) * 8));
  if (nwalk) k_compact_u64<<<nblk(nwalk), 256, 0, s>>>(walk.as<uint64_t>(), uflag.as<int64_t>(), upos.as<int64_t>(),
                                                       nwalk, part.as<uint64_t>());
  if (np) k_remap_bounds<<<nblk(np), 256, 0, s>>>(upos.as<int64_t>(), pbeg.as<int64_t>(), pend.as<int64_t>(), np,
                                                  ubeg.as<int64_t>(), uend.as<int64_t>(), nwalk, npart);
  walk.release(); uflag.release(); upos.release();
  DBuf kept, part_poly;
  RB_CUDA(kept.alloc(std::max<int64_t>(npart, 1)));
  RB_CUDA(part_poly.alloc(std::max<int64_t>(npart, 1) * 4));
  if (npart) k_kept<<<nblk(npart), 256, 0, s>>>(part.as<uint64_t>(), npart, ubeg.as<int64_t>(), np, dgx, dgy,
                                                P->ring_off, P->poly_ring_off, opts->mode, kept.as<uint8_t>(),
                                                part_poly.as<int32_t>());
  RB_CUDA(cudaGetLastError());
  A->stats.n_partial_leaves = npart;

  trace("K2 edge walk");
  // ---- K3 crossings -> spans
  RB_CUDA(cudaMemsetAsync(cnt.p, 0, (nv + 1) * 8, s));
  if (nv) k_xing_count<<<nblk(nv), 256, 0, s>>>(dgx, dgy, dvn, nv, cnt.as<int64_t>());
  RB_CUDA(excl_scan_i64(cnt.as<int64_t>(), off.as<int64_t>(), nv + 1, s));
  int64_t nx = d2h(off.as<int64_t>() + nv, s);
  DBuf xs, xbeg, xend;
  RB_CUDA(xs.alloc(std::max<int64_t>(nx, 1) * 8));
  RB_CUDA(xbeg.alloc(std::max<int64_t>(np, 1) * 8));
  RB_CUDA(xend.alloc(std::max<int64_t>(np, 1) * 8));
  if (nv) k_xing_emit<<<nblk(nv), 256, 0, s>>>(dgx, dgy, dvn, nv, off.as<int64_t>(), xs.as<uint64_t>());
  if (np) k_seg_bounds<<<nblk(np), 256, 0, s>>>(off.as<int64_t>(), P->ring_off, P->poly_ring_off, np,
                                                xbeg.as<int64_t>(), xend.as<int64_t>());
  RB_CUDA(cudaGetLastError());
  RB_CUDA(seg_sort_keys(xs.as<uint64_t>(), nx, np, xbeg.as<int64_t>(), xend.as<int64_t>(), s));
  DBuf scnt, soff, skey, sc1, sbeg, send;
  RB_CUDA(scnt.alloc((np + 1) * 8));
  RB_CUDA(soff.alloc((np + 1) * 8));
  RB_CUDA(cudaMemsetAsync(scnt.p, 0, (np + 1) * 8, s));
  if (np) k_span_count<<<nblk(np), 256, 0, s>>>(xs.as<uint64_t>(), xbeg.as<int64_t>(), xend.as<int64_t>(), np,
                                                scnt.as<int64_t>());
  RB_CUDA(excl_scan_i64(scnt.as<int64_t>(), soff.as<int64_t>(), np + 1, s));
  int64_t nspan = d2h(soff.as<int64_t>() + np, s);
  RB_CUDA(skey.alloc(std::max<int64_t>(nspan, 1) * 8));
  RB_CUDA(sc1.alloc(std::max<int64_t>(nspan, 1) * 4));
  if (np) k_span_emit<<<nblk(np), 256, 0, s>>>(xs.as<uint64_t>(), xbeg.as<int64_t>(), xend.as<int64_t>(), np,
                                               soff.as<int64_t>(), skey.as<uint64_t>(), sc1.as<int32_t>());
  RB_CUDA(cudaGetLastError());
  xs.release();
  // span segment bounds: beg = soff[p], end = soff[p+1]
  const int64_t* dsoff = soff.as<int64_t>();

  // ---- aligned pieces
  RB_CUDA(cudaMemsetAsync(cnt.p, 0, (nv + 1) * 8, s));
  if (nv) k_aligned_count<<<nblk(nv), 256, 0, s>>>(dgx, dgy, dvn, nv, cnt.as<int64_t>());
  RB_CUDA(excl_scan_i64(cnt.as<int64_t>(), off.as<int64_t>(), nv + 1, s));
  int64_t nal = d2h(off.as<int64_t>() + nv, s);
  DBuf al, abeg, aend;
  RB_CUDA(al.alloc(std::max<int64_t>(nal, 1) * 32));
  RB_CUDA(abeg.alloc(std::max<int64_t>(np, 1) * 8));
  RB_CUDA(aend.alloc(std::max<int64_t>(np, 1) * 8));
  if (nv) k_aligned_emit<<<nblk(nv), 256, 0, s>>>(dgx, dgy, dvn, nv, cnt.as<int64_t>(), off.as<int64_t>(),
                                                  al.as<double4>());
  if (np) k_seg_bounds<<<nblk(np), 256, 0, s>>>(off.as<int64_t>(), P->ring_off, P->poly_ring_off, np,
                                                abeg.as<int64_t>(), aend.as<int64_t>());
  RB_CUDA(cudaGetLastError());

  PolyView V{mbr.as<uint32_t>(), part.as<uint64_t>(), ubeg.as<int64_t>(), uend.as<int64_t>(), kept.as<uint8_t>(),
             skey.as<uint64_t>(), sc1.as<int32_t>(), dsoff, dsoff + 1, al.as<double4>(), abeg.as<int64_t>(),
             aend.as<int64_t>()};

  trace("K3 spans + aligned pieces");
  // ---- K4 hierarchical descent
  std::vector<DBuf> cpl, cll, ccl, ckl;
  std::vector<int64_t> ncl;
  DBuf fp, fc;
  RB_CUDA(fp.alloc(std::max<int64_t>(np, 1) * 4));
  RB_CUDA(fc.alloc(std::max<int64_t>(np, 1) * 8));
  {
    std::vector<int32_t> h(np);
    for (int64_t p = 0; p < np; ++p) h[p] = (int32_t)p;
    if (np) RB_CUDA(cudaMemcpyAsync(fp.p, h.data(), np * 4, cudaMemcpyHostToDevice, s));
    RB_CUDA(cudaMemsetAsync(fc.p, 0, std::max<int64_t>(np, 1) * 8, s));
    RB_CUDA(cudaStreamSynchronize(s));
  }
  int64_t nf = np;
  int64_t total_cells = 0, n_int = 0, n_bnd = 0;
  for (int lvl = 0; lvl <= L && nf > 0; ++lvl) {
    DBuf nch, nce, cho, ceo;
    RB_CUDA(nch.alloc((nf + 1) * 8));
    RB_CUDA(nce.alloc((nf + 1) * 8));
    RB_CUDA(cho.alloc((nf + 1) * 8));
    RB_CUDA(ceo.alloc((nf + 1) * 8));
    RB_CUDA(cudaMemsetAsync(nch.p, 0, (nf + 1) * 8, s));
    RB_CUDA(cudaMemsetAsync(nce.p, 0, (nf + 1) * 8, s));
    k_hier_count<<<nblk(nf), 256, 0, s>>>(V, fp.as<int32_t>(), fc.as<uint64_t>(), nf, lvl, L, nch.as<int64_t>(),
                                          nce.as<int64_t>());
    RB_CUDA(cudaGetLastError());
    RB_CUDA(excl_scan_i64(nch.as<int64_t>(), cho.as<int64_t>(), nf + 1, s));
    RB_CUDA(excl_scan_i64(nce.as<int64_t>(), ceo.as<int64_t>(), nf + 1, s));
    int64_t nchild = d2h(cho.as<int64_t>() + nf, s), ncell = d2h(ceo.as<int64_t>() + nf, s);
    DBuf nfp, nfc, cp, cl, cc, ck;
    RB_CUDA(nfp.alloc(std::max<int64_t>(nchild, 1) * 4));
    RB_CUDA(nfc.alloc(std::max<int64_t>(nchild, 1) * 8));
    RB_CUDA(cp.alloc(std::max<int64_t>(ncell, 1) * 4));
    RB_CUDA(cl.alloc(std::max<int64_t>(ncell, 1)));
    RB_CUDA(cc.alloc(std::max<int64_t>(ncell, 1) * 8));
    RB_CUDA(ck.alloc(std::max<int64_t>(ncell, 1)));
    k_hier_emit<<<nblk(nf), 256, 0, s>>>(V, fp.as<int32_t>(), fc.as<uint64_t>(), nf, lvl, L, cho.as<int64_t>(),
                                         ceo.as<int64_t>(), nfp.as<int32_t>(), nfc.as<uint64_t>(), cp.as<int32_t>(),
                                         cl.as<uint8_t>(), cc.as<uint64_t>(), ck.as<uint8_t>());
    RB_CUDA(cudaGetLastError());
    if (ncell) {
      cpl.push_back(std::move(cp)); cll.push_back(std::move(cl)); ccl.push_back(std::move(cc)); ckl.push_back(std::move(ck));
      ncl.push_back(ncell);
      total_cells += ncell;
    }
    fp = std::move(nfp);
    fc = std::move(nfc);
    nf = nchild;
  }
  RB_CUDA(cudaStreamSynchronize(s));
  // concatenate
  DBuf c_poly, c_level, c_code, c_kind;
  RB_CUDA(c_poly.alloc(std::max<int64_t>(total_cells, 1) * 4));
  RB_CUDA(c_level.alloc(std::max<int64_t>(total_cells, 1)));
  RB_CUDA(c_code.alloc(std::max<int64_t>(total_cells, 1) * 8));
  RB_CUDA(c_kind.alloc(std::max<int64_t>(total_cells, 1)));
  {
    int64_t w = 0;
    for (size_t i = 0; i < ncl.size(); ++i) {
      int64_t c = ncl[i];
      RB_CUDA(cudaMemcpyAsync(c_poly.as<int32_t>() + w, cpl[i].p, c * 4, cudaMemcpyDeviceToDevice, s));
      RB_CUDA(cudaMemcpyAsync(c_level.as<uint8_t>() + w, cll[i].p, c, cudaMemcpyDeviceToDevice, s));
      RB_CUDA(cudaMemcpyAsync(c_code.as<uint64_t>() + w, ccl[i].p, c * 8, cudaMemcpyDeviceToDevice, s));
      RB_CUDA(cudaMemcpyAsync(c_kind.as<uint8_t>() + w, ckl[i].p, c, cudaMemcpyDeviceToDevice, s));
      w += c;
    }
    RB_CUDA(cudaStreamSynchronize(s));
    cpl.clear(); cll.clear(); ccl.clear(); ckl.clear();
  }
  {
    // stats: interior / boundary cells and expanded interior leaves (device reduce)
    DBuf cs3;
    RB_CUDA(cs3.alloc(24));
    RB_CUDA(cudaMemsetAsync(cs3.p, 0, 24, s));
    if (total_cells)
      k_cell_stats<<<nblk(total_cells), 256, 0, s>>>(c_level.as<uint8_t>(), c_kind.as<uint8_t>(), total_cells, L,
                                                     cs3.as<unsigned long long>());
    RB_CUDA(cudaGetLastError());
    unsigned long long h3[3] = {0, 0, 0};
    RB_CUDA(cudaMemcpyAsync(h3, cs3.p, 24, cudaMemcpyDeviceToHost, s));
    RB_CUDA(cudaStreamSynchronize(s));
    n_int = (int64_t)h3[0];
    n_bnd = (int64_t)h3[1];
    A->stats.n_interior_cells = n_int;
    A->stats.n_boundary_cells = n_bnd;
    A->stats.n_uniform_interior = (int64_t)h3[2];
  }

  trace("K4 descent + concat + stats");
  int ist = index_impl(L, total_cells, c_poly.as<int32_t>(), c_level.as<uint8_t>(), c_code.as<uint64_t>(),
                       c_kind.as<uint8_t>(), P->poly_region, opts, s, A);
  if (ist) return ist;
  if (opts->keep_cells) {
    A->cell_poly = std::move(c_poly); A->cell_level = std::move(c_level);
    A->cell_code = std::move(c_code); A->cell_kind = std::move(c_kind);
    A->n_cells = total_cells;
    A->part_poly = std::move(part_poly); A->part_code = std::move(part); A->part_kept = std::move(kept);
    A->n_partial = npart;
  }

  A->stats.build_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  return RB_OK;
}

}  // namespace rb

extern "C" int rb_approx_build(const rb_grid* grid, const rb_polygons* polys, const rb_build_opts* opts, void* stream,
                               rb_approx** out) {
  using namespace rb;
  if (!grid || !polys || !opts || !out) return fail(RB_CONFIG_ERROR, "null argument");
  *out = nullptr;
  if (grid->max_level < 0 || grid->max_level > 31) return fail(RB_CAPACITY_ERROR, "max_level outside [0, 31]");
  if (!(grid->extent > 0.0) || !std::isfinite(grid->extent) || !std::isfinite(grid->origin_x) ||
      !std::isfinite(grid->origin_y))
    return fail(RB_CONFIG_ERROR, "grid extent must be finite and > 0");
  if (opts->mode != RB_MODE_CONSERVATIVE && opts->mode != RB_MODE_CENTER_SAMPLED)
    return fail(RB_CONFIG_ERROR, "unknown raster mode");
  if (opts->layout != RB_LAYOUT_DENSE && opts->layout != RB_LAYOUT_TRIE && opts->layout != RB_LAYOUT_KEYS &&
      opts->layout != RB_LAYOUT_PACKED)
    return fail(RB_CONFIG_ERROR, "unknown layout");
  if (opts->radix_width != 2 && opts->radix_width != 4 && opts->radix_width != 8)
    return fail(RB_CONFIG_ERROR, "radix_width must be 2, 4 or 8 (SPEC.md:278)");
  if (polys->n_regions <= 0 || polys->n_regions >= RB_MAX_REGIONS)  // the 18-bit code field of owner values
    return fail(RB_CAPACITY_ERROR, "n_regions outside [1, 2^17)");
  if (polys->n_polygons < 0 || polys->n_rings < 0 || polys->n_vertices < 0) return fail(RB_CONFIG_ERROR, "negative sizes");
  if (polys->n_polygons >= ((int64_t)1 << 31)) return fail(RB_CAPACITY_ERROR, "too many polygons");
  std::unique_ptr<rb_approx> A(new rb_approx());
  A->grid = *grid;
  A->opts = *opts;
  A->n_regions = polys->n_regions;
  A->n_polygons = polys->n_polygons;
  A->set_code_format();
  int st;
  {
    AllocScope scope((cudaStream_t)stream);  // stream-ordered scratch from the private pool
    st = build_impl(grid, polys, opts, (cudaStream_t)stream, A.get());
    if (st == RB_OK) st = cudaStreamSynchronize((cudaStream_t)stream) ? cuda_fail(cudaGetLastError(), "build") : RB_OK;
  }
  if (st != RB_OK) return st;
  A->detach_all();
  *out = A.release();
  return RB_OK;
}

namespace rb {
__global__ void k_validate_cells(const int32_t* cov, const uint8_t* lv, const uint64_t* code, const uint8_t* kind,
                                 int64_t n, int64_t ncov, int L, int* flag) {
  GRID_STRIDE(k, n) {
    if (cov[k] < 0 || cov[k] >= ncov || lv[k] > L || kind[k] < 1 || kind[k] > 2) atomicOr(flag, 1);
    else if ((code[k] >> (2 * lv[k])) != 0) atomicOr(flag, 2);
  }
}
}  // namespace rb

// act.act_build from explicit coverings: cells of covering
// c (interior kind 1 / boundary kind 2, any level <= L) map to region
// cov_region[c]; duplicates are idempotent.
extern "C" int rb_index_from_cells(const rb_grid* grid, int64_t n_cells, const int32_t* cov, const uint8_t* level,
                                   const uint64_t* code, const uint8_t* kind, const int32_t* cov_region, int64_t n_cov,
                                   int32_t n_regions, const rb_build_opts* opts, void* stream, rb_approx** out) {
  using namespace rb;
  if (!grid || !opts || !out) return fail(RB_CONFIG_ERROR, "null argument");
  *out = nullptr;
  if (grid->max_level < 0 || grid->max_level > 31) return fail(RB_CAPACITY_ERROR, "max_level outside [0, 31]");
  if (opts->layout != RB_LAYOUT_DENSE && opts->layout != RB_LAYOUT_TRIE && opts->layout != RB_LAYOUT_KEYS &&
      opts->layout != RB_LAYOUT_PACKED)
    return fail(RB_CONFIG_ERROR, "unknown layout");
  if (opts->radix_width != 2 && opts->radix_width != 4 && opts->radix_width != 8)
    return fail(RB_CONFIG_ERROR, "radix_width must be 2, 4 or 8 (SPEC.md:278)");
  if (n_regions <= 0 || n_regions >= RB_MAX_REGIONS)  // the 18-bit code field of owner values
    return fail(RB_CAPACITY_ERROR, "n_regions outside [1, 2^17)");
  if (n_cells < 0 || n_cov < 0) return fail(RB_SHAPE_ERROR, "negative sizes");
  cudaStream_t s = (cudaStream_t)stream;
  AllocScope scope(s);
  auto t_start = std::chrono::steady_clock::now();
  {
    std::vector<int32_t> hr(n_cov);
    if (n_cov) RB_CUDA(cudaMemcpyAsync(hr.data(), cov_region, n_cov * 4, cudaMemcpyDeviceToHost, s));
    RB_CUDA(cudaStreamSynchronize(s));
    for (int64_t c = 0; c < n_cov; ++c)
      if (hr[c] < 0 || hr[c] >= n_regions) return fail(RB_CONFIG_ERROR, "covering region out of range");
  }
  const int L = grid->max_level;
  if (n_cells) {
    DBuf flag;
    RB_CUDA(flag.alloc(4));
    RB_CUDA(cudaMemsetAsync(flag.p, 0, 4, s));
    k_validate_cells<<<nblk(n_cells), 256, 0, s>>>(cov, level, code, kind, n_cells, n_cov, L, flag.as<int>());
    RB_CUDA(cudaGetLastError());
    int f = d2h(flag.as<int>(), s);
    if (f & 1) return fail(RB_CONFIG_ERROR, "cell with bad covering index, level > L or kind not in {1,2}");
    if (f & 2) return fail(RB_DOMAIN_ERROR, "cell code >= 4^level");
  }
  std::unique_ptr<rb_approx> A(new rb_approx());
  A->grid = *grid;
  A->opts = *opts;
  A->opts.keep_cells = 0;
  A->n_regions = n_regions;
  A->n_polygons = n_cov;
  A->set_code_format();
  A->stats.max_level = L;
  A->stats.n_regions = n_regions;
  int st = index_impl(L, n_cells, cov, level, code, kind, cov_region, opts, s, A.get());
  if (st != RB_OK) return st;
  RB_CUDA(cudaStreamSynchronize(s));
  A->stats.build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  A->detach_all();
  *out = A.release();
  return RB_OK;
}

namespace rb {
__global__ void k_hot_remap(const int32_t* regions, int32_t K, int32_t* remap) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x) remap[regions[k]] = k + 1;
}
// annotate single-owner values (root / nodes) with their region's hot slot
__global__ void k_hot_values(uint32_t* v, int64_t n, const int32_t* remap, uint32_t cm, uint32_t hs) {
  GRID_STRIDE(k, n) {
    const uint32_t x = v[k];
    if (x == 0u || (x & (RB_VALUE_NODE | RB_VALUE_LIST))) continue;
    const uint32_t code = x & cm;
    const uint32_t r = (code - 1u) >> 1;
    v[k] = code | ((uint32_t)remap[r] << hs);
  }
}
__device__ __forceinline__ uint32_t hot_value(uint32_t x, const int32_t* remap, uint32_t cm, uint32_t hs) {
  if (x == 0u || (x & (RB_VALUE_NODE | RB_VALUE_LIST))) return x;
  const uint32_t code = x & cm;
  return code | ((uint32_t)remap[(code - 1u) >> 1] << hs);
}
// RB_LAYOUT_PACKED: the three palette entries of every block (escape pointers are left alone)
__global__ void k_hot_blocks(uint4* blk, int64_t n, const int32_t* remap, uint32_t cm, uint32_t hs) {
  GRID_STRIDE(k, n) {
    uint4 b = blk[k];
    b.x = hot_value(b.x, remap, cm, hs);
    b.y = hot_value(b.y, remap, cm, hs);
    b.z = hot_value(b.z, remap, cm, hs);
    blk[k] = b;
  }
}
// RB_LAYOUT_KEYS: annotate the single owner values of the cell records
__global__ void k_hot_records(uint4* rec, int64_t n, const int32_t* remap, uint32_t cm, uint32_t hs) {
  GRID_STRIDE(k, n) rec[k].z = hot_value(rec[k].z, remap, cm, hs);
}
// annotate owner-list entries ((region<<1)|boundary); count words are flagged
__global__ void k_hot_pool(uint32_t* p, int64_t n, const int32_t* remap, uint32_t cm, uint32_t hs) {
  GRID_STRIDE(k, n) {
    const uint32_t x = p[k];
    if (x & RB_POOL_COUNT_FLAG) continue;
    const uint32_t e = x & cm;
    p[k] = e | ((uint32_t)remap[e >> 1] << hs);
  }
}
}  // namespace rb

// Mark up to 4095 "hot" regions (e.g. the most frequent owners of a point
// sample): their alpha COUNT/SUM are accumulated in shared memory by the
// point pass when the full histogram does not fit there.  Results are
// unchanged; only where the accumulation happens.  Synchronises `stream`.
extern "C" int rb_approx_set_hot(rb_approx* a, const int32_t* regions, int32_t n_hot, void* stream) {
  using namespace rb;
  if (!a) return fail(RB_CONFIG_ERROR, "null approximation");
  if (a->n_hot) return fail(RB_CONFIG_ERROR, "hot regions already set");
  if (n_hot < 0 || n_hot > a->max_hot)
    return fail(RB_CAPACITY_ERROR, "at most " + std::to_string(a->max_hot) + " hot regions for this region count");
  if (n_hot == 0) return RB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  AllocScope scope(s);
  std::vector<int32_t> h(n_hot);
  RB_CUDA(cudaMemcpyAsync(h.data(), regions, n_hot * 4, cudaMemcpyDefault, s));
  RB_CUDA(cudaStreamSynchronize(s));
  {
    std::vector<char> seen(a->n_regions, 0);
    for (int32_t r : h) {
      if (r < 0 || r >= a->n_regions) return fail(RB_CONFIG_ERROR, "hot region out of range");
      if (seen[r]++) return fail(RB_CONFIG_ERROR, "duplicate hot region");
    }
  }
  RB_CUDA(a->hot_region.alloc_persistent(n_hot * 4));
  RB_CUDA(cudaMemcpyAsync(a->hot_region.p, h.data(), n_hot * 4, cudaMemcpyHostToDevice, s));
  DBuf remap;
  RB_CUDA(remap.alloc((size_t)a->n_regions * 4));
  RB_CUDA(cudaMemsetAsync(remap.p, 0, (size_t)a->n_regions * 4, s));
  k_hot_remap<<<nblk(n_hot), 256, 0, s>>>(a->hot_region.as<int32_t>(), n_hot, remap.as<int32_t>());
  k_hot_values<<<nblk(a->root_entries), 256, 0, s>>>(a->root.as<uint32_t>(), a->root_entries, remap.as<int32_t>(), a->code_mask, a->hot_shift);
  for (size_t i = 0; i < a->node_bufs.size(); ++i) {
    const int64_t n = (int64_t)(a->node_bufs[i].bytes / 4);
    k_hot_values<<<nblk(n), 256, 0, s>>>(a->node_bufs[i].as<uint32_t>(), n, remap.as<int32_t>(), a->code_mask, a->hot_shift);
  }
  if (a->n_pblk) k_hot_blocks<<<nblk(a->n_pblk), 256, 0, s>>>(a->pblk.as<uint4>(), a->n_pblk, remap.as<int32_t>(), a->code_mask, a->hot_shift);
  if (a->n_pwide)
    k_hot_values<<<nblk(a->n_pwide * 16), 256, 0, s>>>(a->pwide.as<uint32_t>(), a->n_pwide * 16, remap.as<int32_t>(), a->code_mask, a->hot_shift);
  if (a->pool_len) k_hot_pool<<<nblk(a->pool_len), 256, 0, s>>>(a->pool.as<uint32_t>(), a->pool_len, remap.as<int32_t>(), a->code_mask, a->hot_shift);
  RB_CUDA(cudaGetLastError());
  if (a->keys.p && a->nkeys)
    k_hot_records<<<nblk(a->nkeys), 256, 0, s>>>(a->keys.as<uint4>(), a->nkeys, remap.as<int32_t>(), a->code_mask, a->hot_shift);
  if (a->S >= 0 && a->keys.p)  // annotated values exceed u16: the summary refers them to the index
    k_key_summary<<<nblk((int64_t)1 << (2 * a->S)), 256, 0, s>>>(a->keys.as<uint4>(), a->nkeys, a->grid.max_level,
                                                                 a->S, a->summary.as<uint16_t>());
  else if (a->S >= 0)
    k_summary<<<nblk(((int64_t)32 << (2 * a->S))), 256, 0, s>>>(a->root.as<uint32_t>(), a->T0, a->S,
                                                                 a->summary.as<uint16_t>());
  RB_CUDA(cudaGetLastError());
  RB_CUDA(cudaStreamSynchronize(s));
  a->hot_region.detach();
  a->n_hot = n_hot;
  return RB_OK;
}
