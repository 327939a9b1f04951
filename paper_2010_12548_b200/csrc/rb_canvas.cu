// rb_canvas.cu -- the canvas data model and its blend / mask / affine operator
// algebra (section 4), the substrate of the Bounded
// Raster Join (join_canvas).
//
// A canvas tile is a dense row-major 2^level x 2^level block of the level-L
// leaf grid at pixel offset (x0, y0): pixel (ix, iy) is leaf z_encode(ix, iy, L)
// (SPEC.md:391).  Channels: count (int64), n_sum float64 SUM channels, region
// id (int32, -1 = none) and flags (bit 0 = non-empty, bit 1 = boundary).
// Every operator is a pure elementwise or gather kernel; render_points reduces
// each pixel from a point index (sorted codes + prefix sums), so real-valued
// channels are deterministic, and the reduction of a canvas is a fixed-order
// two-pass tree.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>

#include "rb_internal.cuh"

namespace rb {
int lps_view(const rb_lps* L, int64_t* n, const uint64_t** codes, const double** prefix, int32_t* n_attr,
             int32_t* level);
}

namespace rb {

#define RB_PX_VALID 1u
#define RB_PX_BOUNDARY 2u

static inline int cb(int64_t n, int t = 256) {
  int64_t b = (n + t - 1) / t;
  return (int)std::min<int64_t>(std::max<int64_t>(b, 1), 148 * 64);
}

static bool desc_ok(const rb_canvas_desc* c) {
  return c && c->level >= 0 && c->level <= 16 && c->count && c->region && c->flags && (c->n_sum == 0 || c->sums);
}
static inline int64_t npx(const rb_canvas_desc* c) { return (int64_t)1 << (2 * c->level); }

__global__ void k_canvas_clear(int64_t n, int n_sum, int64_t* count, double* sums, int32_t* region, uint8_t* flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    count[i] = 0;
    for (int s = 0; s < n_sum; ++s) sums[(size_t)s * n + i] = 0.0;
    region[i] = -1;
    flags[i] = 0;
  }
}

// render_points: one thread per sorted point; the first point of each run of
// equal codes writes the pixel (count = run length, sums = prefix differences)
__global__ void k_render_points(const uint64_t* codes, int64_t n, const double* prefix, int n_attr, int L, int64_t x0,
                                int64_t y0, int lev, int64_t* count, double* sums) {
  const int64_t W = (int64_t)1 << lev;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (i > 0 && codes[i] == codes[i - 1]) continue;
    const uint64_t c = codes[i];
    const int64_t ix = (int64_t)compact1by1(c) - x0, iy = (int64_t)compact1by1(c >> 1) - y0;
    if (ix < 0 || iy < 0 || ix >= W || iy >= W) continue;
    // run end: next different code (binary search over the sorted codes)
    int64_t lo = i + 1, hi = n;
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if (codes[m] <= c) lo = m + 1; else hi = m;
    }
    const int64_t p = iy * W + ix;
    count[p] = lo - i;
    for (int s = 0; s < n_attr; ++s) {
      const double* pre = prefix + (size_t)s * (n + 1);
      sums[(size_t)s * W * W + p] = pre[lo] - pre[i];
    }
  }
}
// Z-aligned tiles: the leaves of an aligned 2^lev x 2^lev block are the Z-code
// range [zlo, zlo + 4^lev), so only that slice of the sorted codes is visited.
__device__ __forceinline__ uint64_t spread1by1(uint64_t v) {
  v &= 0xffffffffull;
  v = (v | (v << 16)) & 0x0000ffff0000ffffull;
  v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
  v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}
__global__ void k_tile_range(const uint64_t* codes, int64_t n, int64_t x0, int64_t y0, int lev, int64_t* range) {
  const uint64_t zlo = spread1by1((uint64_t)x0) | (spread1by1((uint64_t)y0) << 1);
  const uint64_t zhi = zlo + ((uint64_t)1 << (2 * lev));
  for (int b = 0; b < 2; ++b) {
    const uint64_t key = b ? zhi : zlo;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if (codes[m] < key) lo = m + 1; else hi = m;
    }
    range[b] = lo;
  }
}
__global__ void k_render_points_range(const uint64_t* codes, int64_t n, const int64_t* range, const double* prefix,
                                      int n_attr, int L, int64_t x0, int64_t y0, int lev, int64_t* count,
                                      double* sums) {
  const int64_t W = (int64_t)1 << lev;
  const int64_t b = range[0], e = range[1];
  for (int64_t i = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
    if (i > b && codes[i] == codes[i - 1]) continue;
    const uint64_t c = codes[i];
    const int64_t ix = (int64_t)compact1by1(c) - x0, iy = (int64_t)compact1by1(c >> 1) - y0;
    int64_t lo = i + 1, hi = e;  // run end within the tile's slice
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if (codes[m] <= c) lo = m + 1; else hi = m;
    }
    const int64_t p = iy * W + ix;
    count[p] = lo - i;
    for (int s = 0; s < n_attr; ++s) {
      const double* pre = prefix + (size_t)s * (n + 1);
      sums[(size_t)s * W * W + p] = pre[lo] - pre[i];
    }
  }
}
__global__ void k_flag_nonempty(int64_t n, const int64_t* count, uint8_t* flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = count[i] > 0 ? RB_PX_VALID : 0u;
}

// render_polygon from covering cells (level, code at that level, kind): each
// cell fills its 2^(L-l) x 2^(L-l) pixel block (clipped to the tile)
__global__ void k_render_cells(int64_t m, const int32_t* lev, const uint64_t* code, const uint8_t* kind, int L,
                               int64_t x0, int64_t y0, int tlev, int32_t rid, int32_t* region, uint8_t* flags) {
  const int64_t W = (int64_t)1 << tlev;
  for (int64_t c = blockIdx.x; c < m; c += gridDim.x) {
    const int d = L - lev[c];
    const int64_t bx = ((int64_t)compact1by1(code[c]) << d) - x0, by = ((int64_t)compact1by1(code[c] >> 1) << d) - y0;
    const int64_t side = (int64_t)1 << d;
    const int64_t xa = bx < 0 ? 0 : bx, ya = by < 0 ? 0 : by;
    const int64_t xb = bx + side > W ? W : bx + side, yb = by + side > W ? W : by + side;
    if (xa >= xb || ya >= yb) continue;
    const uint8_t f = RB_PX_VALID | (kind[c] == RB_KIND_B ? RB_PX_BOUNDARY : 0u);
    const int64_t w = xb - xa, tot = w * (yb - ya);
    for (int64_t k = threadIdx.x; k < tot; k += blockDim.x) {
      const int64_t p = (ya + k / w) * W + xa + k % w;
      region[p] = rid;
      flags[p] = f;
    }
  }
}

// blend: fn 0 = SUM, 1 = OVERWRITE (b over a), 2 = MAX
__global__ void k_blend(int64_t n, int n_sum, int fn, const int64_t* ac, const double* as, const int32_t* ar,
                        const uint8_t* af, const int64_t* bc, const double* bs, const int32_t* br, const uint8_t* bf,
                        int64_t* oc, double* os, int32_t* orr, uint8_t* of) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool va = af[i] & RB_PX_VALID, vb = bf[i] & RB_PX_VALID;
    if (!vb) {  // empty (.) x = x for every fn
      oc[i] = ac[i];
      for (int s = 0; s < n_sum; ++s) os[(size_t)s * n + i] = as[(size_t)s * n + i];
      orr[i] = ar[i];
      of[i] = af[i];
      continue;
    }
    if (!va || fn == 1) {
      oc[i] = bc[i];
      for (int s = 0; s < n_sum; ++s) os[(size_t)s * n + i] = bs[(size_t)s * n + i];
      orr[i] = br[i];
      of[i] = bf[i];
      continue;
    }
    if (fn == 0) {
      oc[i] = ac[i] + bc[i];
      for (int s = 0; s < n_sum; ++s) os[(size_t)s * n + i] = as[(size_t)s * n + i] + bs[(size_t)s * n + i];
    } else {
      oc[i] = ac[i] > bc[i] ? ac[i] : bc[i];
      for (int s = 0; s < n_sum; ++s) {
        const double x = as[(size_t)s * n + i], y = bs[(size_t)s * n + i];
        os[(size_t)s * n + i] = x > y ? x : y;
      }
    }
    orr[i] = ar[i] >= 0 ? ar[i] : br[i];
    of[i] = af[i] | bf[i];
  }
}

// mask: predicate 0 NONEMPTY, 1 REGION_EQ(arg), 2 BOUNDARY_ONLY,
// 3 COUNT_GT(arg), 4 COVERED_BY(canvas `by`: its pixel is non-empty),
// 5 BOUNDARY_OF(canvas `by`: its pixel is a boundary pixel)
__global__ void k_mask(int64_t n, int n_sum, int pred, int64_t arg, const int64_t* ac, const double* as,
                       const int32_t* ar, const uint8_t* af, const uint8_t* byf, int64_t* oc, double* os,
                       int32_t* orr, uint8_t* of) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool keep = af[i] & RB_PX_VALID;
    if (pred == 1) keep = keep && ar[i] == (int32_t)arg;
    else if (pred == 2) keep = keep && (af[i] & RB_PX_BOUNDARY);
    else if (pred == 3) keep = keep && ac[i] > arg;
    else if (pred == 4) keep = keep && (byf[i] & RB_PX_VALID);
    else if (pred == 5) keep = keep && (byf[i] & RB_PX_BOUNDARY);
    oc[i] = keep ? ac[i] : 0;
    for (int s = 0; s < n_sum; ++s) os[(size_t)s * n + i] = keep ? as[(size_t)s * n + i] : 0.0;
    orr[i] = keep ? ar[i] : -1;
    // a pixel kept through COVERED_BY inherits the covering canvas's boundary flag
    uint8_t f = keep ? af[i] : 0u;
    if (keep && pred == 4) f = (uint8_t)((f & RB_PX_VALID) | (byf[i] & RB_PX_BOUNDARY));
    of[i] = f;
  }
}

// affine: integer translation + axis flips; out(x, y) = a(src)
__global__ void k_affine(int lev, int n_sum, int64_t dx, int64_t dy, int fx, int fy, const int64_t* ac,
                         const double* as, const int32_t* ar, const uint8_t* af, int64_t* oc, double* os, int32_t* orr,
                         uint8_t* of) {
  const int64_t W = (int64_t)1 << lev, n = W * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = i % W, y = i / W;
    int64_t sx = x - dx, sy = y - dy;  // translate first, then flip
    if (fx) sx = W - 1 - sx;
    if (fy) sy = W - 1 - sy;
    if (sx < 0 || sy < 0 || sx >= W || sy >= W) {
      oc[i] = 0;
      for (int s = 0; s < n_sum; ++s) os[(size_t)s * n + i] = 0.0;
      orr[i] = -1;
      of[i] = 0;
      continue;
    }
    const int64_t j = sy * W + sx;
    oc[i] = ac[j];
    for (int s = 0; s < n_sum; ++s) os[(size_t)s * n + i] = as[(size_t)s * n + j];
    orr[i] = ar[j];
    of[i] = af[j];
  }
}

// reduce: count and sums over non-empty pixels (all, and boundary only);
// fixed-order two-pass tree (deterministic)
#define RB_RED_BLOCKS 592
__global__ void __launch_bounds__(256) k_reduce_px(int64_t n, int n_sum, const int64_t* c, const double* s,
                                                   const uint8_t* f, long long* pc, double* ps) {
  __shared__ long long sc[2][256];
  __shared__ double ss[2][256];
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = b0 + per < n ? b0 + per : n;
  for (int ch = -1; ch < n_sum; ++ch) {
    long long ca = 0, cbn = 0;
    double sa = 0.0, sbn = 0.0;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
      if (!(f[i] & RB_PX_VALID)) continue;
      const bool bnd = f[i] & RB_PX_BOUNDARY;
      if (ch < 0) { ca += c[i]; if (bnd) cbn += c[i]; }
      else { const double v = s[(size_t)ch * n + i]; sa += v; if (bnd) sbn += v; }
    }
    sc[0][threadIdx.x] = ca; sc[1][threadIdx.x] = cbn;
    ss[0][threadIdx.x] = sa; ss[1][threadIdx.x] = sbn;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if (threadIdx.x < o) {
        sc[0][threadIdx.x] += sc[0][threadIdx.x + o]; sc[1][threadIdx.x] += sc[1][threadIdx.x + o];
        ss[0][threadIdx.x] += ss[0][threadIdx.x + o]; ss[1][threadIdx.x] += ss[1][threadIdx.x + o];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      if (ch < 0) { pc[2 * blockIdx.x] = sc[0][0]; pc[2 * blockIdx.x + 1] = sc[1][0]; }
      else { ps[((size_t)ch * gridDim.x + blockIdx.x) * 2] = ss[0][0]; ps[((size_t)ch * gridDim.x + blockIdx.x) * 2 + 1] = ss[1][0]; }
    }
    __syncthreads();
  }
}
__global__ void k_reduce_px2(int nb, int n_sum, const long long* pc, const double* ps, int64_t* cnt_out,
                             double* sum_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  long long a = 0, b = 0;
  for (int i = 0; i < nb; ++i) { a += pc[2 * i]; b += pc[2 * i + 1]; }
  cnt_out[0] = a;
  cnt_out[1] = b;
  for (int s = 0; s < n_sum; ++s) {
    double x = 0.0, y = 0.0;
    for (int i = 0; i < nb; ++i) { x += ps[((size_t)s * nb + i) * 2]; y += ps[((size_t)s * nb + i) * 2 + 1]; }
    sum_out[2 * s] = x;
    sum_out[2 * s + 1] = y;
  }
}

}  // namespace rb

using namespace rb;

extern "C" int rb_canvas_clear(rb_canvas_desc* c, void* stream) {
  if (!desc_ok(c)) return fail(RB_CONFIG_ERROR, "invalid canvas");
  k_canvas_clear<<<cb(npx(c)), 256, 0, (cudaStream_t)stream>>>(npx(c), c->n_sum, c->count, c->sums, c->region, c->flags);
  RB_CUDA(cudaGetLastError());
  return RB_OK;
}

extern "C" int rb_canvas_render_points(const rb_lps* lps, rb_canvas_desc* out, void* stream) {
  if (!lps || !desc_ok(out)) return fail(RB_CONFIG_ERROR, "invalid argument");
  int64_t n = 0;
  const uint64_t* codes = nullptr;
  const double* prefix = nullptr;
  int32_t na = 0, L = 0;
  int st = lps_view(lps, &n, &codes, &prefix, &na, &L);
  if (st) return st;
  if (out->n_sum > na) return fail(RB_SCHEMA_ERROR, "more SUM channels than point-index attributes (SPEC.md:359)");
  if (out->level > L) return fail(RB_SHAPE_ERROR, "canvas tile finer than the point index level");
  cudaStream_t s = (cudaStream_t)stream;
  k_canvas_clear<<<cb(npx(out)), 256, 0, s>>>(npx(out), out->n_sum, out->count, out->sums, out->region, out->flags);
  const int64_t W = (int64_t)1 << out->level;
  const bool aligned = out->x0 >= 0 && out->y0 >= 0 && (out->x0 % W) == 0 && (out->y0 % W) == 0 &&
                       out->x0 + W <= ((int64_t)1 << L) && out->y0 + W <= ((int64_t)1 << L);
  if (n && aligned) {  // only the tile's slice of the sorted codes
    int64_t* range = nullptr;
    RB_CUDA(pool_alloc(&range, 16, s));
    k_tile_range<<<1, 1, 0, s>>>(codes, n, out->x0, out->y0, out->level, range);
    k_render_points_range<<<cb(std::min<int64_t>(n, (int64_t)npx(out) * 4)), 256, 0, s>>>(
        codes, n, range, prefix, out->n_sum, L, out->x0, out->y0, out->level, out->count, out->sums);
    RB_CUDA(cudaFreeAsync(range, s));
  } else if (n) {
    k_render_points<<<cb(n), 256, 0, s>>>(codes, n, prefix, out->n_sum, L, out->x0, out->y0, out->level, out->count,
                                          out->sums);
  }
  k_flag_nonempty<<<cb(npx(out)), 256, 0, s>>>(npx(out), out->count, out->flags);
  RB_CUDA(cudaGetLastError());
  return RB_OK;
}

extern "C" int rb_canvas_render_cells(int64_t n_cells, const int32_t* level, const uint64_t* code, const uint8_t* kind,
                                      int32_t L, int32_t region_id, int32_t clear, rb_canvas_desc* out, void* stream) {
  if (!desc_ok(out) || n_cells < 0) return fail(RB_CONFIG_ERROR, "invalid argument");
  if (out->level > L) return fail(RB_SHAPE_ERROR, "canvas tile finer than the raster level");
  cudaStream_t s = (cudaStream_t)stream;
  if (clear)
    k_canvas_clear<<<cb(npx(out)), 256, 0, s>>>(npx(out), out->n_sum, out->count, out->sums, out->region, out->flags);
  if (n_cells)
    k_render_cells<<<(int)std::min<int64_t>(n_cells, 148 * 32), 256, 0, s>>>(n_cells, level, code, kind, L, out->x0,
                                                                            out->y0, out->level, region_id,
                                                                            out->region, out->flags);
  RB_CUDA(cudaGetLastError());
  return RB_OK;
}

static bool same_shape(const rb_canvas_desc* a, const rb_canvas_desc* b) {
  return a->level == b->level && a->n_sum == b->n_sum;
}

extern "C" int rb_canvas_blend(const rb_canvas_desc* a, const rb_canvas_desc* b, int32_t fn, rb_canvas_desc* out,
                               void* stream) {
  if (!desc_ok(a) || !desc_ok(b) || !desc_ok(out)) return fail(RB_CONFIG_ERROR, "invalid canvas");
  if (!same_shape(a, b) || !same_shape(a, out)) return fail(RB_SHAPE_ERROR, "canvas dimensions differ (SPEC.md:425)");
  if (fn < 0 || fn > 2) return fail(RB_CONFIG_ERROR, "unknown blend function");
  k_blend<<<cb(npx(a)), 256, 0, (cudaStream_t)stream>>>(npx(a), a->n_sum, fn, a->count, a->sums, a->region, a->flags,
                                                        b->count, b->sums, b->region, b->flags, out->count, out->sums,
                                                        out->region, out->flags);
  RB_CUDA(cudaGetLastError());
  return RB_OK;
}

extern "C" int rb_canvas_mask(const rb_canvas_desc* a, int32_t pred, int64_t arg, const rb_canvas_desc* by,
                              rb_canvas_desc* out, void* stream) {
  if (!desc_ok(a) || !desc_ok(out)) return fail(RB_CONFIG_ERROR, "invalid canvas");
  if (!same_shape(a, out)) return fail(RB_SHAPE_ERROR, "canvas dimensions differ");
  if (pred < 0 || pred > 5) return fail(RB_CONFIG_ERROR, "unknown mask predicate");
  if (pred >= 4 && (!by || !by->flags || by->level != a->level))
    return fail(RB_SHAPE_ERROR, "mask canvas missing or of another size");
  k_mask<<<cb(npx(a)), 256, 0, (cudaStream_t)stream>>>(npx(a), a->n_sum, pred, arg, a->count, a->sums, a->region,
                                                       a->flags, pred >= 4 ? by->flags : nullptr, out->count,
                                                       out->sums, out->region, out->flags);
  RB_CUDA(cudaGetLastError());
  return RB_OK;
}

extern "C" int rb_canvas_affine(const rb_canvas_desc* a, int64_t dx, int64_t dy, int32_t flip_x, int32_t flip_y,
                                rb_canvas_desc* out, void* stream) {
  if (!desc_ok(a) || !desc_ok(out)) return fail(RB_CONFIG_ERROR, "invalid canvas");
  if (!same_shape(a, out)) return fail(RB_SHAPE_ERROR, "canvas dimensions differ");
  if (a->count == out->count) return fail(RB_CONFIG_ERROR, "affine needs a distinct output canvas");
  k_affine<<<cb(npx(a)), 256, 0, (cudaStream_t)stream>>>(a->level, a->n_sum, dx, dy, flip_x != 0, flip_y != 0,
                                                         a->count, a->sums, a->region, a->flags, out->count, out->sums,
                                                         out->region, out->flags);
  RB_CUDA(cudaGetLastError());
  return RB_OK;
}

extern "C" int rb_canvas_reduce(const rb_canvas_desc* a, int64_t* cnt_out, double* sum_out, void* stream) {
  if (!desc_ok(a) || !cnt_out || (a->n_sum && !sum_out)) return fail(RB_CONFIG_ERROR, "invalid argument");
  cudaStream_t s = (cudaStream_t)stream;
  long long* pc = nullptr;
  double* ps = nullptr;  // stream-ordered scratch: no host synchronisation
  RB_CUDA(pool_alloc(&pc, RB_RED_BLOCKS * 16, s));
  RB_CUDA(pool_alloc(&ps, (size_t)std::max(a->n_sum, 1) * RB_RED_BLOCKS * 16, s));
  k_reduce_px<<<RB_RED_BLOCKS, 256, 0, s>>>(npx(a), a->n_sum, a->count, a->sums, a->flags, pc, ps);
  k_reduce_px2<<<1, 32, 0, s>>>(RB_RED_BLOCKS, a->n_sum, pc, ps, cnt_out, sum_out);
  RB_CUDA(cudaGetLastError());
  RB_CUDA(cudaFreeAsync(pc, s));
  RB_CUDA(cudaFreeAsync(ps, s));
  return RB_OK;
}
