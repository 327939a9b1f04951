// rb_pointindex.cu -- the point-side access path (
// PAPER.md:238-254): points linearised to sorted leaf Z codes with prefix sums,
// a RadixSpline over the codes, and join_pointindex = per covering cell two
// lower-bound lookups and a prefix-sum difference.
//
// B200 layout: codes (u64, sorted, CUB radix sort of (code, point id) pairs --
// stable, so equal codes keep point order), perm (i64), one float64 prefix
// array of n+1 entries per attribute (CUB inclusive scan of the permuted
// attribute).  The RadixSpline is fitted greedily in parallel chunks of the
// distinct-key CDF (one thread per chunk, knots at chunk borders), so its
// error bound <= max_error holds for every key by construction and the fit is
// deterministic.  Lookups: radix table -> knot segment -> interpolation ->
// binary search in [estimate - tau - 1, estimate + tau + 2), with a full binary
// search fallback whenever the window does not bracket the answer, so results
// are identical to plain binary search.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <vector>

#include "rb_internal.cuh"

struct rb_lps {
  rb_grid grid;
  int64_t n = 0;
  int32_t n_attr = 0;
  rb::DBuf codes, perm, prefix;  // u64 [n], i64 [n], f64 [n_attr][n+1]
};

struct rb_rs {
  int32_t radix_bits = 0, shift = 0, max_error = 0;
  int64_t n_knots = 0;
  rb::DBuf keys, pos, table;  // u64 [n_knots], i64 [n_knots], u32 [2^r + 1]
};

namespace rb {

static inline int nb(int64_t n, int t = 256) {
  int64_t b = (n + t - 1) / t;
  return (int)std::min<int64_t>(std::max<int64_t>(b, 1), 148 * 64);
}

// leaf Z code of each point (x in the even bits), the same
// float64 formula as the point pass and the oracle (floor(RN((v - o) / side)))
__global__ void k_leaf_codes(double ox, double oy, double side, double inv_side, double lim, int L, const void* xy,
                             int dtype, int64_t n, uint64_t* codes, int64_t* ids, unsigned long long* first_bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double x, y;
    if (dtype == RB_XY_F64) { x = ((const double*)xy)[2 * i]; y = ((const double*)xy)[2 * i + 1]; }
    else { x = (double)((const float*)xy)[2 * i]; y = (double)((const float*)xy)[2 * i + 1]; }
    const double fx = cell_floor(x, ox, side, inv_side), fy = cell_floor(y, oy, side, inv_side);
    uint64_t c = 0;
    if (!(fx >= 0.0 && fx < lim && fy >= 0.0 && fy < lim)) atomicMin(first_bad, (unsigned long long)i);
    else c = zenc((uint64_t)fx, (uint64_t)fy);
    codes[i] = c;
    ids[i] = i;
  }
}

__global__ void k_gather_attr(const float* attr, const int64_t* perm, int64_t n, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (double)attr[perm[i]];
}

__global__ void k_reset_first_bad(unsigned long long* p) { *p = (unsigned long long)LLONG_MAX; }

// ---------------------------------------------------------------- RadixSpline
// distinct keys: flag[i] = (i == 0 || codes[i] != codes[i-1]); the CDF point of
// a key is (key, first position).
__global__ void k_first_flags(const uint64_t* codes, int64_t n, int64_t* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i == 0 || codes[i] != codes[i - 1]) ? 1 : 0;
}
__global__ void k_compact_keys(const uint64_t* codes, const int64_t* flag, const int64_t* off, int64_t n, uint64_t* dk,
                               int64_t* dp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) { dk[off[i]] = codes[i]; dp[off[i]] = i; }
}
// lower-bound CDF points F(q) = #{codes < q}: (k, F(k)) for every distinct key k,
// plus (k + 1, F(next key)) when the next distinct key (or the end of the key
// space) lies beyond k + 1 -- with both in the fit, the spline is within tau of
// F at every integer query, stored or not, so the lookup window always brackets.
__global__ void k_cdf_count(const uint64_t* dk, int64_t nd, uint64_t kend, int64_t* cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nd; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t nxt = i + 1 < nd ? dk[i + 1] : kend;
    cnt[i] = 1 + (nxt > dk[i] + 1 ? 1 : 0);
  }
}
__global__ void k_cdf_points(const uint64_t* dk, const int64_t* dp, int64_t nd, int64_t n, uint64_t kend,
                             const int64_t* off, uint64_t* pk, int64_t* pp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nd; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t nxt = i + 1 < nd ? dk[i + 1] : kend;
    const int64_t o = off[i];
    pk[o] = dk[i];
    pp[o] = dp[i];
    if (nxt > dk[i] + 1) { pk[o + 1] = dk[i] + 1; pp[o + 1] = i + 1 < nd ? dp[i + 1] : n; }
  }
}

// greedy spline corridor over the distinct-key CDF, one chunk per thread:
// knots are the chunk's first and last point plus every point where the
// corridor from the previous knot would be violated (|interpolation error| <=
// tau for every point strictly between two knots).  mode 0 counts the knots
// of each chunk, mode 1 writes them at out_off[chunk].
template <int MODE>
__global__ void k_spline_chunks(const uint64_t* dk, const int64_t* dp, int64_t nd, int64_t chunk, double tau,
                                int64_t* nknots, const int64_t* out_off, uint64_t* kk, int64_t* kp) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t b = c * chunk;
  if (b >= nd) return;
  const int64_t e = nd < b + chunk ? nd : b + chunk;
  int64_t cnt = 0, w = MODE ? out_off[c] : 0;
  auto emit = [&](int64_t i) {
    if (MODE) { kk[w] = dk[i]; kp[w] = dp[i]; ++w; }
    ++cnt;
  };
  emit(b);
  if (e - b > 1) {
    int64_t base = b;  // last knot
    // corridor of admissible slopes from the last knot (position per key unit)
    double lo_s = -1e300, hi_s = 1e300;
    int64_t prev = b;
    for (int64_t i = b + 1; i < e; ++i) {
      const double dx = (double)(dk[i] - dk[base]);
      const double y = (double)(dp[i] - dp[base]);
      const double s = y / dx;
      if (s < lo_s || s > hi_s) {  // the segment base..i cannot cover i-1's corridor: knot at prev
        emit(prev);
        base = prev;
        const double dx2 = (double)(dk[i] - dk[base]);
        const double y2 = (double)(dp[i] - dp[base]);
        lo_s = (y2 - tau) / dx2;
        hi_s = (y2 + tau) / dx2;
      } else {
        const double l = (y - tau) / dx, h = (y + tau) / dx;
        lo_s = l > lo_s ? l : lo_s;
        hi_s = h < hi_s ? h : hi_s;
      }
      prev = i;
    }
    emit(e - 1);
  }
  if (!MODE) nknots[c] = cnt;
}

// radix table: table[p] = index of the first knot whose key >> shift >= p, p in [0, 2^r]
// (one thread per slot, binary search over the knots)
__global__ void k_radix_table(const uint64_t* kk, int64_t nk, int shift, int64_t nslots, uint32_t* table) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nslots; p += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nk;
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if ((int64_t)(kk[m] >> shift) < p) lo = m + 1; else hi = m;
    }
    table[p] = (uint32_t)lo;
  }
}

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* a, int64_t lo, int64_t hi, uint64_t key) {
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (a[m] < key) lo = m + 1; else hi = m;
  }
  return lo;
}

struct RsView {
  const uint64_t* keys;
  const int64_t* pos;
  const uint32_t* table;
  int64_t nk;
  int shift;
  int64_t nslots;
  int tau;
};

// first position with code >= key
__device__ int64_t bound(const uint64_t* codes, int64_t n, const RsView* rs, uint64_t key) {
  if (!rs || rs->nk < 2) return lower_bound_u64(codes, 0, n, key);
  const RsView& R = *rs;
  // knot segment: last knot with key <= query
  const int64_t p = (int64_t)(key >> R.shift);
  int64_t a = p < R.nslots ? (int64_t)R.table[p] : R.nk;  // first knot with prefix >= p
  int64_t b = p + 1 < R.nslots ? (int64_t)R.table[p + 1] : R.nk;
  a = a > 0 ? a - 1 : 0;
  // upper_bound over knots in [a, b] for key, minus one
  int64_t lo = a, hi = b < R.nk ? b + 1 : R.nk;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (R.keys[m] <= key) lo = m + 1; else hi = m;
  }
  const int64_t k0 = lo - 1;
  double est;
  if (k0 < 0) est = 0.0;
  else if (k0 + 1 >= R.nk) est = (double)R.pos[R.nk - 1] + (key == R.keys[R.nk - 1] ? 0.0 : 1.0);
  else {
    const double t = (double)(key - R.keys[k0]) / (double)(R.keys[k0 + 1] - R.keys[k0]);
    est = (double)R.pos[k0] + t * (double)(R.pos[k0 + 1] - R.pos[k0]);
  }
  int64_t wlo = (int64_t)est - R.tau - 1, whi = (int64_t)est + R.tau + 2;
  wlo = wlo < 0 ? 0 : (wlo > n ? n : wlo);
  whi = whi < wlo ? wlo : (whi > n ? n : whi);
  const int64_t r = lower_bound_u64(codes, wlo, whi, key);
  // the window must bracket the answer; otherwise fall back (identical results by construction)
  const bool left_ok = r > wlo || wlo == 0 || codes[wlo - 1] < key;
  const bool right_ok = r < whi || whi == n || codes[whi] >= key;
  if (left_ok && right_ok) return r;
  return lower_bound_u64(codes, 0, n, key);
}

__global__ void k_bounds(const uint64_t* codes, int64_t n, RsView rs, int use_rs, const uint64_t* lo,
                         const uint64_t* hi, int64_t m, int64_t* lo_pos, int64_t* hi_pos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    lo_pos[i] = bound(codes, n, use_rs ? &rs : nullptr, lo[i]);
    hi_pos[i] = bound(codes, n, use_rs ? &rs : nullptr, hi[i]);
  }
}

// join_pointindex, pass 1: one thread per covering cell -- its two lower
// bounds (RadixSpline window or binary search) and the prefix differences
__global__ void k_cell_vals(const uint64_t* codes, int64_t n, RsView rs, int use_rs, int64_t n_cells,
                            const int32_t* lev, const uint64_t* code, int L, const double* prefix, int64_t* kv,
                            double* sv) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_cells; c += (int64_t)gridDim.x * blockDim.x) {
    const int sh = 2 * (L - lev[c]);
    const uint64_t lo = code[c] << sh, hi = (code[c] + 1) << sh;  // SPEC.md:152-160 cell_interval
    const int64_t p0 = bound(codes, n, use_rs ? &rs : nullptr, lo);
    const int64_t p1 = bound(codes, n, use_rs ? &rs : nullptr, hi);
    kv[c] = p1 - p0;  // COUNT prefix is the position itself
    sv[c] = prefix ? prefix[p1] - prefix[p0] : 0.0;
  }
}

// pass 2: one block per region over its (region-grouped) cells, thread-strided
// order + fixed-order block reduction: deterministic COUNT and SUM
__global__ void __launch_bounds__(256) k_region_sums(const int64_t* cell_beg, const uint8_t* kind, const int64_t* kv,
                                                     const double* sv, int64_t* cnt_out, double* sum_out) {
  __shared__ int64_t sc[2][8];
  __shared__ double ss[2][8];
  const int r = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t ca = 0, cb = 0;
  double sa = 0.0, sb = 0.0;
  for (int64_t c = cell_beg[r] + threadIdx.x; c < cell_beg[r + 1]; c += 256) {
    const int64_t k = kv[c];
    const double v = sv[c];
    ca += k;
    sa += v;
    if (kind[c] == RB_KIND_B) { cb += k; sb += v; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    ca += __shfl_xor_sync(0xffffffffu, ca, o);
    cb += __shfl_xor_sync(0xffffffffu, cb, o);
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
  }
  if (lane == 0) { sc[0][warp] = ca; sc[1][warp] = cb; ss[0][warp] = sa; ss[1][warp] = sb; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) { ca += sc[0][w]; cb += sc[1][w]; sa += ss[0][w]; sb += ss[1][w]; }
    cnt_out[2 * r] = ca;
    cnt_out[2 * r + 1] = cb;
    sum_out[2 * r] = sa;
    sum_out[2 * r + 1] = sb;
  }
}

__global__ void k_cell_counts(const int32_t* reg, int64_t m, int64_t* beg_counts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd((unsigned long long*)&beg_counts[reg[i]], 1ull);
}

static RsView view_of(const rb_rs* rs) {
  RsView v{};
  if (!rs) return v;
  v.keys = rs->keys.as<uint64_t>();
  v.pos = rs->pos.as<int64_t>();
  v.table = rs->table.as<uint32_t>();
  v.nk = rs->n_knots;
  v.shift = rs->shift;
  v.nslots = (int64_t)1 << rs->radix_bits;
  v.tau = rs->max_error;
  return v;
}

}  // namespace rb

namespace rb {
// internal view for the canvas module (rb_canvas.cu)
int lps_view(const rb_lps* L, int64_t* n, const uint64_t** codes, const double** prefix, int32_t* n_attr,
             int32_t* level) {
  if (!L) return fail(RB_CONFIG_ERROR, "null point index");
  *n = L->n;
  *codes = L->codes.as<uint64_t>();
  *prefix = L->prefix.as<double>();
  *n_attr = L->n_attr;
  *level = L->grid.max_level;
  return RB_OK;
}
}  // namespace rb

using namespace rb;

extern "C" int rb_lps_build(const rb_grid* grid, const void* xy, int32_t xy_dtype, int64_t n, const float* const* attrs,
                            int32_t n_attr, void* stream, rb_lps** out, int64_t* first_bad) {
  if (!grid || !out || !first_bad) return fail(RB_CONFIG_ERROR, "null argument");
  if (xy_dtype != RB_XY_F64 && xy_dtype != RB_XY_F32) return fail(RB_CONFIG_ERROR, "unknown xy dtype");
  if (n < 0 || n_attr < 0) return fail(RB_SHAPE_ERROR, "negative size");
  if (grid->max_level < 0 || grid->max_level > 31) return fail(RB_CAPACITY_ERROR, "level must be in [0, 31]");
  if (n > 0 && !xy) return fail(RB_CONFIG_ERROR, "null points");
  cudaStream_t s = (cudaStream_t)stream;
  auto* L = new rb_lps();
  L->grid = *grid;
  L->n = n;
  L->n_attr = n_attr;
  *first_bad = LLONG_MAX;
  auto bail = [&](int st) { delete L; return st; };
  DBuf k0, i0, bad;
  if (bad.alloc(8) || L->codes.alloc(std::max<int64_t>(n, 1) * 8) || L->perm.alloc(std::max<int64_t>(n, 1) * 8) ||
      L->prefix.alloc(std::max<int32_t>(n_attr, 1) * (n + 1) * 8) || k0.alloc(std::max<int64_t>(n, 1) * 8) ||
      i0.alloc(std::max<int64_t>(n, 1) * 8))
    return bail(fail(RB_CAPACITY_ERROR, "out of device memory for the point index"));
  k_reset_first_bad<<<1, 1, 0, s>>>(bad.as<unsigned long long>());
  const int Lv = grid->max_level;
  const double side = ldexp(grid->extent, -Lv);
  if (n > 0) {
    k_leaf_codes<<<nb(n), 256, 0, s>>>(grid->origin_x, grid->origin_y, side, 1.0 / side, ldexp(1.0, Lv), Lv, xy,
                                      xy_dtype, n, k0.as<uint64_t>(), i0.as<int64_t>(),
                                      bad.as<unsigned long long>());
    size_t tb = 0;
    const int bits = std::max(1, 2 * Lv);
    cub::DeviceRadixSort::SortPairs(nullptr, tb, k0.as<uint64_t>(), L->codes.as<uint64_t>(), i0.as<int64_t>(),
                                    L->perm.as<int64_t>(), n, 0, bits, s);
    DBuf t;
    if (t.alloc(std::max<size_t>(tb, 1))) return bail(fail(RB_CAPACITY_ERROR, "out of device memory (sort)"));
    cudaError_t e = cub::DeviceRadixSort::SortPairs(t.p, tb, k0.as<uint64_t>(), L->codes.as<uint64_t>(),
                                                    i0.as<int64_t>(), L->perm.as<int64_t>(), n, 0, bits, s);
    if (e) return bail(cuda_fail(e, "lps sort"));
  }
  for (int a = 0; a < n_attr; ++a) {
    double* pre = L->prefix.as<double>() + (size_t)a * (n + 1);
    cudaError_t e = cudaMemsetAsync(pre, 0, 8, s);  // prefix[0] = 0
    if (e) return bail(cuda_fail(e, "lps prefix"));
    if (n == 0) continue;
    if (!attrs || !attrs[a]) return bail(fail(RB_SCHEMA_ERROR, "null attribute array"));
    DBuf g;
    if (g.alloc(n * 8)) return bail(fail(RB_CAPACITY_ERROR, "out of device memory (prefix)"));
    k_gather_attr<<<nb(n), 256, 0, s>>>(attrs[a], L->perm.as<int64_t>(), n, g.as<double>());
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, g.as<double>(), pre + 1, n, s);
    DBuf t;
    if (t.alloc(std::max<size_t>(tb, 1))) return bail(fail(RB_CAPACITY_ERROR, "out of device memory (scan)"));
    e = cub::DeviceScan::InclusiveSum(t.p, tb, g.as<double>(), pre + 1, n, s);
    if (e) return bail(cuda_fail(e, "lps scan"));
    e = cudaStreamSynchronize(s);  // g and t go out of scope
    if (e) return bail(cuda_fail(e, "lps scan sync"));
  }
  unsigned long long fb = 0;
  cudaError_t e = cudaMemcpyAsync(&fb, bad.p, 8, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  if (e) return bail(cuda_fail(e, "lps build"));
  if (fb != (unsigned long long)LLONG_MAX) {
    *first_bad = (int64_t)fb;
    return bail(fail(RB_DOMAIN_ERROR, "point outside the grid domain (SPEC.md:332)"));
  }
  *out = L;
  return RB_OK;
}

extern "C" int rb_lps_info(const rb_lps* L, int64_t* n, const uint64_t** codes, const int64_t** perm,
                           const double** prefix, int32_t* n_attr) {
  if (!L) return fail(RB_CONFIG_ERROR, "null point index");
  if (n) *n = L->n;
  if (codes) *codes = L->codes.as<uint64_t>();
  if (perm) *perm = L->perm.as<int64_t>();
  if (prefix) *prefix = L->prefix.as<double>();
  if (n_attr) *n_attr = L->n_attr;
  return RB_OK;
}

extern "C" void rb_lps_free(rb_lps* L) { delete L; }

extern "C" int rb_rs_build(const rb_lps* L, int32_t radix_bits, int32_t max_error, void* stream, rb_rs** out) {
  if (!L || !out) return fail(RB_CONFIG_ERROR, "null argument");
  const int width = 2 * L->grid.max_level;
  if (radix_bits < 0 || radix_bits > width || radix_bits > 30)
    return fail(RB_CONFIG_ERROR, "radix_bits exceeds the code width (SPEC.md:340)");
  if (max_error < 0) return fail(RB_CONFIG_ERROR, "max_error must be >= 0");
  cudaStream_t s = (cudaStream_t)stream;
  auto* R = new rb_rs();
  R->radix_bits = radix_bits;
  R->shift = width - radix_bits;
  R->max_error = max_error;
  auto bail = [&](int st) { delete R; return st; };
  const int64_t n = L->n;
  const int64_t nslots = (int64_t)1 << radix_bits;
  if (R->table.alloc((nslots + 1) * 4)) return bail(fail(RB_CAPACITY_ERROR, "out of device memory (radix table)"));
  if (n == 0) {
    cudaMemsetAsync(R->table.p, 0, (nslots + 1) * 4, s);
    cudaStreamSynchronize(s);
    *out = R;
    return RB_OK;
  }
  DBuf flag, off, dk, dp;
  if (flag.alloc((n + 1) * 8) || off.alloc((n + 1) * 8)) return bail(fail(RB_CAPACITY_ERROR, "out of memory"));
  cudaMemsetAsync(flag.p, 0, (n + 1) * 8, s);
  k_first_flags<<<nb(n), 256, 0, s>>>(L->codes.as<uint64_t>(), n, flag.as<int64_t>());
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.as<int64_t>(), off.as<int64_t>(), n + 1, s);
  {
    DBuf t;
    if (t.alloc(std::max<size_t>(tb, 1))) return bail(fail(RB_CAPACITY_ERROR, "out of memory"));
    cub::DeviceScan::ExclusiveSum(t.p, tb, flag.as<int64_t>(), off.as<int64_t>(), n + 1, s);
    cudaStreamSynchronize(s);
  }
  int64_t nd = 0;
  cudaMemcpy(&nd, off.as<int64_t>() + n, 8, cudaMemcpyDeviceToHost);
  if (dk.alloc(nd * 8) || dp.alloc(nd * 8)) return bail(fail(RB_CAPACITY_ERROR, "out of memory"));
  k_compact_keys<<<nb(n), 256, 0, s>>>(L->codes.as<uint64_t>(), flag.as<int64_t>(), off.as<int64_t>(), n,
                                       dk.as<uint64_t>(), dp.as<int64_t>());
  {  // the fitted points: the lower-bound CDF at and just after every distinct key
    const uint64_t kend = width >= 64 ? ~0ull : (1ull << width);
    DBuf pc, po, pk, pp;
    if (pc.alloc((nd + 1) * 8) || po.alloc((nd + 1) * 8)) return bail(fail(RB_CAPACITY_ERROR, "out of memory"));
    cudaMemsetAsync(pc.p, 0, (nd + 1) * 8, s);
    k_cdf_count<<<nb(nd), 256, 0, s>>>(dk.as<uint64_t>(), nd, kend, pc.as<int64_t>());
    tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, pc.as<int64_t>(), po.as<int64_t>(), nd + 1, s);
    {
      DBuf t;
      if (t.alloc(std::max<size_t>(tb, 1))) return bail(fail(RB_CAPACITY_ERROR, "out of memory"));
      cub::DeviceScan::ExclusiveSum(t.p, tb, pc.as<int64_t>(), po.as<int64_t>(), nd + 1, s);
      cudaStreamSynchronize(s);
    }
    int64_t np = 0;
    cudaMemcpy(&np, po.as<int64_t>() + nd, 8, cudaMemcpyDeviceToHost);
    if (pk.alloc(np * 8) || pp.alloc(np * 8)) return bail(fail(RB_CAPACITY_ERROR, "out of memory"));
    k_cdf_points<<<nb(nd), 256, 0, s>>>(dk.as<uint64_t>(), dp.as<int64_t>(), nd, n, kend, po.as<int64_t>(),
                                        pk.as<uint64_t>(), pp.as<int64_t>());
    cudaStreamSynchronize(s);
    dk = std::move(pk);
    dp = std::move(pp);
    nd = np;
  }
  const int64_t chunk = 4096;
  const int64_t nch = (nd + chunk - 1) / chunk;
  DBuf kc, ko;
  if (kc.alloc((nch + 1) * 8) || ko.alloc((nch + 1) * 8)) return bail(fail(RB_CAPACITY_ERROR, "out of memory"));
  cudaMemsetAsync(kc.p, 0, (nch + 1) * 8, s);
  // fit with half a position of margin: the corridor slopes are float64 quotients of 62-bit key gaps
  const double tau_fit = max_error > 0 ? (double)max_error - 0.5 : 0.0;
  k_spline_chunks<0><<<nb(nch, 128), 128, 0, s>>>(dk.as<uint64_t>(), dp.as<int64_t>(), nd, chunk, tau_fit,
                                                  kc.as<int64_t>(), nullptr, nullptr, nullptr);
  tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, kc.as<int64_t>(), ko.as<int64_t>(), nch + 1, s);
  {
    DBuf t;
    if (t.alloc(std::max<size_t>(tb, 1))) return bail(fail(RB_CAPACITY_ERROR, "out of memory"));
    cub::DeviceScan::ExclusiveSum(t.p, tb, kc.as<int64_t>(), ko.as<int64_t>(), nch + 1, s);
    cudaStreamSynchronize(s);
  }
  int64_t nk = 0;
  cudaMemcpy(&nk, ko.as<int64_t>() + nch, 8, cudaMemcpyDeviceToHost);
  if (R->keys.alloc(nk * 8) || R->pos.alloc(nk * 8)) return bail(fail(RB_CAPACITY_ERROR, "out of memory"));
  k_spline_chunks<1><<<nb(nch, 128), 128, 0, s>>>(dk.as<uint64_t>(), dp.as<int64_t>(), nd, chunk, tau_fit,
                                                  nullptr, ko.as<int64_t>(), R->keys.as<uint64_t>(),
                                                  R->pos.as<int64_t>());
  R->n_knots = nk;
  // knots at chunk borders can repeat a key only if a chunk had one point; keys stay non-decreasing
  k_radix_table<<<nb(nslots + 1), 256, 0, s>>>(R->keys.as<uint64_t>(), nk, R->shift, nslots + 1, R->table.as<uint32_t>());
  cudaError_t e = cudaGetLastError();
  if (!e) e = cudaStreamSynchronize(s);
  if (e) return bail(cuda_fail(e, "rs build"));
  *out = R;
  return RB_OK;
}

extern "C" int rb_rs_info(const rb_rs* R, int64_t* n_knots, const uint64_t** keys, const int64_t** pos,
                          const uint32_t** table, int32_t* radix_bits, int32_t* shift) {
  if (!R) return fail(RB_CONFIG_ERROR, "null spline");
  if (n_knots) *n_knots = R->n_knots;
  if (keys) *keys = R->keys.as<uint64_t>();
  if (pos) *pos = R->pos.as<int64_t>();
  if (table) *table = R->table.as<uint32_t>();
  if (radix_bits) *radix_bits = R->radix_bits;
  if (shift) *shift = R->shift;
  return RB_OK;
}

extern "C" void rb_rs_free(rb_rs* R) { delete R; }

extern "C" int rb_bounds_lookup(const rb_lps* L, const rb_rs* R, const uint64_t* lo, const uint64_t* hi, int64_t m,
                                int64_t* lo_pos, int64_t* hi_pos, void* stream) {
  if (!L) return fail(RB_CONFIG_ERROR, "null point index");
  if (m < 0) return fail(RB_SHAPE_ERROR, "negative interval count");
  if (m == 0) return RB_OK;
  if (!lo || !hi || !lo_pos || !hi_pos) return fail(RB_CONFIG_ERROR, "null interval arrays");
  k_bounds<<<nb(m), 256, 0, (cudaStream_t)stream>>>(L->codes.as<uint64_t>(), L->n, view_of(R), R != nullptr, lo, hi,
                                                     m, lo_pos, hi_pos);
  RB_CUDA(cudaGetLastError());
  return RB_OK;
}

// stream-ordered scratch (cudaMallocAsync / cudaFreeAsync): no device-wide sync on the query path
struct SBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  explicit SBuf(cudaStream_t st) : s(st) {}
  SBuf(const SBuf&) = delete;
  SBuf& operator=(const SBuf&) = delete;
  ~SBuf() { if (p) cudaFreeAsync(p, s); }
  cudaError_t alloc(size_t b) { return pool_alloc(&p, b, s); }
  template <class T> T* as() const { return (T*)p; }
};

extern "C" int rb_join_pointindex(const rb_lps* L, const rb_rs* R, int64_t n_cells, const int32_t* region,
                                  const int32_t* level, const uint64_t* code, const uint8_t* kind, int32_t n_regions,
                                  int32_t attr_idx, int64_t* cnt_out, double* sum_out, void* stream) {
  if (!L) return fail(RB_CONFIG_ERROR, "null point index");
  if (n_cells < 0 || n_regions < 0) return fail(RB_SHAPE_ERROR, "negative size");
  if (attr_idx >= L->n_attr) return fail(RB_SCHEMA_ERROR, "attribute not in the point index (SPEC.md:359)");
  if (!cnt_out || !sum_out) return fail(RB_CONFIG_ERROR, "null outputs");
  cudaStream_t s = (cudaStream_t)stream;
  // cells must be grouped by region (non-decreasing region ids): counts -> offsets
  SBuf beg(s), off(s);
  RB_CUDA(beg.alloc(((int64_t)n_regions + 1) * 8));
  RB_CUDA(off.alloc(((int64_t)n_regions + 1) * 8));
  RB_CUDA(cudaMemsetAsync(beg.p, 0, ((int64_t)n_regions + 1) * 8, s));
  if (n_cells) k_cell_counts<<<nb(n_cells), 256, 0, s>>>(region, n_cells, beg.as<int64_t>());
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, beg.as<int64_t>(), off.as<int64_t>(), n_regions + 1, s);
  {
    SBuf t(s);
    RB_CUDA(t.alloc(std::max<size_t>(tb, 1)));
    RB_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tb, beg.as<int64_t>(), off.as<int64_t>(), n_regions + 1, s));
    SBuf vals(s);
    RB_CUDA(vals.alloc(std::max<int64_t>(n_cells, 1) * 16));
    int64_t* kv = vals.as<int64_t>();
    double* sv = (double*)((char*)vals.p + std::max<int64_t>(n_cells, 1) * 8);
    if (n_cells)
      k_cell_vals<<<nb(n_cells), 256, 0, s>>>(
          L->codes.as<uint64_t>(), L->n, view_of(R), R != nullptr, n_cells, level, code, L->grid.max_level,
          attr_idx >= 0 ? L->prefix.as<double>() + (size_t)attr_idx * (L->n + 1) : nullptr, kv, sv);
    if (n_regions) k_region_sums<<<n_regions, 256, 0, s>>>(off.as<int64_t>(), kind, kv, sv, cnt_out, sum_out);
    RB_CUDA(cudaGetLastError());
  }
  return RB_OK;  // stream-ordered: the caller's read of the outputs synchronises
}

extern "C" int rb_lps_from_arrays(const rb_grid* grid, int64_t n, const uint64_t* codes, const int64_t* perm,
                                  const double* prefix, int32_t n_attr, void* stream, rb_lps** out) {
  if (!grid || !out || n < 0 || n_attr < 0) return fail(RB_CONFIG_ERROR, "invalid argument");
  if (n > 0 && (!codes || !perm)) return fail(RB_CONFIG_ERROR, "null arrays");
  if (n_attr > 0 && !prefix) return fail(RB_CONFIG_ERROR, "null prefix arrays");
  cudaStream_t s = (cudaStream_t)stream;
  auto* L = new rb_lps();
  L->grid = *grid;
  L->n = n;
  L->n_attr = n_attr;
  auto bail = [&](int st) { delete L; return st; };
  if (L->codes.alloc(std::max<int64_t>(n, 1) * 8) || L->perm.alloc(std::max<int64_t>(n, 1) * 8) ||
      L->prefix.alloc(std::max<int32_t>(n_attr, 1) * (n + 1) * 8))
    return bail(fail(RB_CAPACITY_ERROR, "out of device memory for the point index"));
  cudaError_t e = cudaSuccess;
  if (n) e = cudaMemcpyAsync(L->codes.p, codes, n * 8, cudaMemcpyDefault, s);
  if (!e && n) e = cudaMemcpyAsync(L->perm.p, perm, n * 8, cudaMemcpyDefault, s);
  if (!e && n_attr) e = cudaMemcpyAsync(L->prefix.p, prefix, (size_t)n_attr * (n + 1) * 8, cudaMemcpyDefault, s);
  if (!e) e = cudaStreamSynchronize(s);
  if (e) return bail(cuda_fail(e, "lps from arrays"));
  *out = L;
  return RB_OK;
}

extern "C" int rb_rs_from_arrays(const rb_lps* L, int32_t radix_bits, int32_t max_error, int64_t n_knots,
                                 const uint64_t* keys, const int64_t* pos, const uint32_t* table, void* stream,
                                 rb_rs** out) {
  if (!L || !out || n_knots < 0) return fail(RB_CONFIG_ERROR, "invalid argument");
  const int width = 2 * L->grid.max_level;
  if (radix_bits < 0 || radix_bits > width || radix_bits > 30) return fail(RB_CONFIG_ERROR, "radix_bits out of range");
  cudaStream_t s = (cudaStream_t)stream;
  auto* R = new rb_rs();
  R->radix_bits = radix_bits;
  R->shift = width - radix_bits;
  R->max_error = max_error;
  R->n_knots = n_knots;
  auto bail = [&](int st) { delete R; return st; };
  const int64_t nslots = ((int64_t)1 << radix_bits) + 1;
  if (R->keys.alloc(std::max<int64_t>(n_knots, 1) * 8) || R->pos.alloc(std::max<int64_t>(n_knots, 1) * 8) ||
      R->table.alloc(nslots * 4))
    return bail(fail(RB_CAPACITY_ERROR, "out of device memory for the spline"));
  cudaError_t e = cudaSuccess;
  if (n_knots) e = cudaMemcpyAsync(R->keys.p, keys, n_knots * 8, cudaMemcpyDefault, s);
  if (!e && n_knots) e = cudaMemcpyAsync(R->pos.p, pos, n_knots * 8, cudaMemcpyDefault, s);
  if (!e) e = cudaMemcpyAsync(R->table.p, table, nslots * 4, cudaMemcpyDefault, s);
  if (!e) e = cudaStreamSynchronize(s);
  if (e) return bail(cuda_fail(e, "rs from arrays"));
  *out = R;
  return RB_OK;
}
