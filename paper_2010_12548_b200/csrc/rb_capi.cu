// rb_capi.cu -- extern "C" entry points of librasterbound_b200.so
// (declared in include/rasterbound_b200.h).  Status codes mirror
// /root/reference/pkg/src/rasterbound/errors.py:8-37.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <mutex>

#include "rb_internal.cuh"

namespace rb {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

cudaStream_t& alloc_stream_tls() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}
bool& alloc_scope_tls() {
  static thread_local bool on = false;
  return on;
}
cudaMemPool_t mem_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[dev & 63]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &props) != cudaSuccess) {
      cudaDeviceGetDefaultMemPool(&p, dev);  // (never expected) the device pool, attributes untouched
    } else {
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      uint64_t thr = tot / 2;  // cache up to half the device between builds / passes (a C4 build peaks near 50 GB;
                               // trimming below that made every rebuild remap its scratch: 0.5 -> 1.4 s)
      cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pools[dev & 63] = p;
  }
  return pools[dev & 63];
}
int fail(int status, const std::string& msg) {
  g_err = msg;
  return status;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ") in " + what;
  return RB_CUDA_ERROR;
}

int point_pass(const rb_approx* A, const void* xy, int32_t dtype, int64_t n, const float* attr, int64_t* cnt_out,
               double* sum_out, int64_t* first_bad, int flags, int64_t idx_base, cudaStream_t s);
int lookup(const rb_approx* A, const void* xy, int32_t dtype, int64_t n, uint32_t* out, int64_t* first_bad,
           cudaStream_t s);
int point_cells(const rb_grid* g, const void* xy, int32_t dtype, int64_t n, uint32_t* ix, uint32_t* iy,
                int64_t* first_bad, cudaStream_t s);
int exact_pip(const rb_polygons* P, const double* px, const double* py, const int32_t* pp, int64_t n, uint8_t* out,
              cudaStream_t s);
int instrument(int op, int64_t* launches, int64_t* timed, double* ms);
int exact_distance(const rb_polygons* P, const double* px, const double* py, const int32_t* pp, int64_t n,
                   double* out, cudaStream_t s);

}  // namespace rb

using namespace rb;

extern "C" int32_t rb_version(void) { return 10000; /* 0.1.0 */ }

extern "C" const char* rb_last_error(void) { return g_err.c_str(); }

extern "C" int rb_level_for_bound(double extent, double epsilon, int32_t* level_out) {
  // smallest l with extent * 2^-l <= epsilon / sqrt(2)
  if (!level_out) return fail(RB_CONFIG_ERROR, "null output");
  if (!(epsilon > 0.0) || !std::isfinite(epsilon)) return fail(RB_CONFIG_ERROR, "epsilon must be finite and > 0");
  if (!(extent > 0.0) || !std::isfinite(extent)) return fail(RB_CONFIG_ERROR, "extent must be finite and > 0");
  double t = epsilon / std::sqrt(2.0);
  for (int l = 0; l <= 31; ++l) {
    if (std::ldexp(extent, -l) <= t) {
      *level_out = l;
      return RB_OK;
    }
  }
  return fail(RB_CAPACITY_ERROR, "epsilon requires a level above 31 (SPEC.md:129)");
}

extern "C" int rb_approx_stats(const rb_approx* a, rb_stats* out) {
  if (!a || !out) return fail(RB_CONFIG_ERROR, "null argument");
  *out = a->stats;
  out->max_hot = a->max_hot;
  out->n_hot = a->n_hot;
  return RB_OK;
}

extern "C" void rb_approx_free(rb_approx* a) { delete a; }

static int check_xy(const rb_approx* a, int32_t dtype, int64_t n) {
  if (!a) return fail(RB_CONFIG_ERROR, "null approximation");
  if (dtype != RB_XY_F64 && dtype != RB_XY_F32) return fail(RB_CONFIG_ERROR, "unknown xy dtype");
  if (n < 0) return fail(RB_SHAPE_ERROR, "negative point count");
  return RB_OK;
}

extern "C" int rb_point_pass(const rb_approx* a, const void* xy, int32_t xy_dtype, int64_t n, const float* attr,
                             int64_t* cnt_out, double* sum_out, int64_t* first_bad, int32_t accumulate, void* stream) {
  int st = check_xy(a, xy_dtype, n);
  if (st) return st;
  if (!cnt_out || !sum_out || !first_bad) return fail(RB_CONFIG_ERROR, "null output buffer");
  return point_pass(a, xy, xy_dtype, n, attr, cnt_out, sum_out, first_bad, accumulate ? 0 : 3, 0,
                    (cudaStream_t)stream);
}

extern "C" int rb_lookup(const rb_approx* a, const void* xy, int32_t xy_dtype, int64_t n, uint32_t* value_out,
                         int64_t* first_bad, void* stream) {
  int st = check_xy(a, xy_dtype, n);
  if (st) return st;
  return lookup(a, xy, xy_dtype, n, value_out, first_bad, (cudaStream_t)stream);
}

extern "C" int rb_owner_pool(const rb_approx* a, uint32_t* dst, int64_t* n) {
  if (!a || !n) return fail(RB_CONFIG_ERROR, "null argument");
  *n = a->pool_len;
  if (dst && a->pool_len) {
    // public form: count words and (region<<1)|boundary entries, no internal annotations
    std::vector<uint32_t> h(a->pool_len);
    RB_CUDA(cudaMemcpy(h.data(), a->pool.p, a->pool_len * 4, cudaMemcpyDeviceToHost));
    for (auto& x : h) x = (x & RB_POOL_COUNT_FLAG) ? (x & ~RB_POOL_COUNT_FLAG) : (x & a->code_mask);
    RB_CUDA(cudaMemcpy(dst, h.data(), a->pool_len * 4, cudaMemcpyDefault));
  }
  return RB_OK;
}

extern "C" int rb_point_cells(const rb_grid* grid, const void* xy, int32_t xy_dtype, int64_t n, uint32_t* ix,
                              uint32_t* iy, int64_t* first_bad, void* stream) {
  if (!grid) return fail(RB_CONFIG_ERROR, "null grid");
  if (grid->max_level < 0 || grid->max_level > 31) return fail(RB_CAPACITY_ERROR, "max_level outside [0, 31]");
  if (xy_dtype != RB_XY_F64 && xy_dtype != RB_XY_F32) return fail(RB_CONFIG_ERROR, "unknown xy dtype");
  return point_cells(grid, xy, xy_dtype, n, ix, iy, first_bad, (cudaStream_t)stream);
}

extern "C" int rb_approx_cells(const rb_approx* a, int64_t* n, int32_t* poly, int32_t* level, uint64_t* code,
                               uint8_t* kind, void* stream) {
  if (!a || !n) return fail(RB_CONFIG_ERROR, "null argument");
  if (!a->opts.keep_cells) return fail(RB_CONFIG_ERROR, "approximation built without keep_cells");
  *n = a->n_cells;
  if (!poly) return RB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  // cells are stored level-major; export sorted by (polygon, start code, level)
  // via a host-side stable sort (export path, not the hot path)
  int64_t m = a->n_cells;
  std::vector<int32_t> hp(m);
  std::vector<uint8_t> hl(m), hk(m);
  std::vector<uint64_t> hc(m);
  if (m) {
    RB_CUDA(cudaMemcpyAsync(hp.data(), a->cell_poly.p, m * 4, cudaMemcpyDeviceToHost, s));
    RB_CUDA(cudaMemcpyAsync(hl.data(), a->cell_level.p, m, cudaMemcpyDeviceToHost, s));
    RB_CUDA(cudaMemcpyAsync(hc.data(), a->cell_code.p, m * 8, cudaMemcpyDeviceToHost, s));
    RB_CUDA(cudaMemcpyAsync(hk.data(), a->cell_kind.p, m, cudaMemcpyDeviceToHost, s));
    RB_CUDA(cudaStreamSynchronize(s));
  }
  const int L = a->grid.max_level;
  std::vector<int64_t> ord(m);
  for (int64_t i = 0; i < m; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) {
    if (hp[x] != hp[y]) return hp[x] < hp[y];
    uint64_t sx = hc[x] << (2 * (L - hl[x])), sy = hc[y] << (2 * (L - hl[y]));
    if (sx != sy) return sx < sy;
    return hl[x] < hl[y];
  });
  std::vector<int32_t> op(m), ol(m);
  std::vector<uint64_t> oc(m);
  std::vector<uint8_t> ok(m);
  for (int64_t i = 0; i < m; ++i) { op[i] = hp[ord[i]]; ol[i] = hl[ord[i]]; oc[i] = hc[ord[i]]; ok[i] = hk[ord[i]]; }
  if (m) {
    RB_CUDA(cudaMemcpyAsync(poly, op.data(), m * 4, cudaMemcpyHostToDevice, s));
    RB_CUDA(cudaMemcpyAsync(level, ol.data(), m * 4, cudaMemcpyHostToDevice, s));
    RB_CUDA(cudaMemcpyAsync(code, oc.data(), m * 8, cudaMemcpyHostToDevice, s));
    RB_CUDA(cudaMemcpyAsync(kind, ok.data(), m, cudaMemcpyHostToDevice, s));
    RB_CUDA(cudaStreamSynchronize(s));
  }
  return RB_OK;
}

extern "C" int rb_approx_partial(const rb_approx* a, int64_t* n, int32_t* poly, uint64_t* code, uint8_t* kept,
                                 void* stream) {
  if (!a || !n) return fail(RB_CONFIG_ERROR, "null argument");
  if (!a->opts.keep_cells) return fail(RB_CONFIG_ERROR, "approximation built without keep_cells");
  *n = a->n_partial;
  if (!poly || !a->n_partial) return RB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  RB_CUDA(cudaMemcpyAsync(poly, a->part_poly.p, a->n_partial * 4, cudaMemcpyDeviceToDevice, s));
  RB_CUDA(cudaMemcpyAsync(code, a->part_code.p, a->n_partial * 8, cudaMemcpyDeviceToDevice, s));
  RB_CUDA(cudaMemcpyAsync(kept, a->part_kept.p, a->n_partial, cudaMemcpyDeviceToDevice, s));
  return RB_OK;
}

extern "C" int rb_exact_pip(const rb_polygons* polys, const double* px, const double* py, const int32_t* poly_of_point,
                            int64_t n, uint8_t* inside_out, void* stream) {
  if (!polys) return fail(RB_CONFIG_ERROR, "null polygons");
  return exact_pip(polys, px, py, poly_of_point, n, inside_out, (cudaStream_t)stream);
}

extern "C" int rb_exact_distance(const rb_polygons* polys, const double* px, const double* py,
                                 const int32_t* poly_of_point, int64_t n, double* dist_out, void* stream) {
  if (!polys) return fail(RB_CONFIG_ERROR, "null polygons");
  return exact_distance(polys, px, py, poly_of_point, n, dist_out, (cudaStream_t)stream);
}

// ------------------------------------------------------------- host join
// Chunked pipeline: H2D copies of chunk i+1 on a copy stream overlap the
// point pass of chunk i on the compute stream (double-buffered device
// chunks); pinned host inputs are copied directly, pageable ones are staged
// through pinned buffers by the CUDA driver.

extern "C" int rb_join_host(const rb_approx* a, const void* xy_host, int32_t xy_dtype, int64_t n,
                            const float* attr_host, int64_t* cnt_host, double* sum_host, int64_t* first_bad_host) {
  int st = check_xy(a, xy_dtype, n);
  if (st) return st;
  if (!cnt_host || !sum_host || !first_bad_host) return fail(RB_CONFIG_ERROR, "null output buffer");
  const int R2 = 2 * a->n_regions;
  const size_t pt_bytes = xy_dtype == RB_XY_F64 ? 16 : 8;
  const int64_t chunk = std::min<int64_t>(std::max<int64_t>(n, 1), (int64_t)1 << 23);
  const int64_t nchunks = (n + chunk - 1) / chunk;
  cudaStream_t cs = nullptr, ks = nullptr;
  cudaEvent_t copied[2] = {}, consumed[2] = {};
  void* dxy[2] = {};
  void* dat[2] = {};
  void* dout = nullptr;
  int rc = RB_OK;
  cudaError_t e = cudaSuccess;
#define JH(call) do { e = (call); if (e != cudaSuccess) { rc = cuda_fail(e, #call); goto done; } } while (0)
  JH(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  JH(cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    JH(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
    JH(cudaEventCreateWithFlags(&consumed[i], cudaEventDisableTiming));
    JH(pool_alloc(&dxy[i], chunk * pt_bytes, cs));
    if (attr_host) JH(pool_alloc(&dat[i], chunk * 4, cs));
  }
  JH(pool_alloc(&dout, (size_t)std::max(R2, 1) * 16 + 8, ks));
  {
    int64_t* dcnt = (int64_t*)dout;
    double* dsum = (double*)((char*)dout + (size_t)std::max(R2, 1) * 8);
    int64_t* dbad = (int64_t*)((char*)dout + (size_t)std::max(R2, 1) * 16);
    rc = point_pass(a, nullptr, xy_dtype, 0, nullptr, dcnt, dsum, dbad, 3, 0, ks);
    if (rc) goto done;
    JH(cudaEventRecord(consumed[0], ks));
    JH(cudaStreamWaitEvent(cs, consumed[0], 0));  // buffers allocated on cs are ordered before use on ks
    for (int64_t c = 0; c < nchunks; ++c) {
      int b = (int)(c & 1);
      int64_t off = c * chunk, m = std::min<int64_t>(chunk, n - off);
      if (c >= 2) JH(cudaStreamWaitEvent(cs, consumed[b], 0));
      JH(cudaMemcpyAsync(dxy[b], (const char*)xy_host + off * pt_bytes, m * pt_bytes, cudaMemcpyHostToDevice, cs));
      if (attr_host) JH(cudaMemcpyAsync(dat[b], attr_host + off, m * 4, cudaMemcpyHostToDevice, cs));
      JH(cudaEventRecord(copied[b], cs));
      JH(cudaStreamWaitEvent(ks, copied[b], 0));
      rc = point_pass(a, dxy[b], xy_dtype, m, attr_host ? (const float*)dat[b] : nullptr, dcnt, dsum, dbad, 0, off, ks);
      if (rc) goto done;
      JH(cudaEventRecord(consumed[b], ks));
    }
    JH(cudaMemcpyAsync(cnt_host, dcnt, (size_t)R2 * 8, cudaMemcpyDeviceToHost, ks));
    JH(cudaMemcpyAsync(sum_host, dsum, (size_t)R2 * 8, cudaMemcpyDeviceToHost, ks));
    JH(cudaMemcpyAsync(first_bad_host, dbad, 8, cudaMemcpyDeviceToHost, ks));
    JH(cudaStreamSynchronize(ks));
  }
done:
#undef JH
  if (ks) cudaStreamSynchronize(ks);
  if (cs) cudaStreamSynchronize(cs);
  for (int i = 0; i < 2; ++i) {
    if (dxy[i]) cudaFreeAsync(dxy[i], ks ? ks : cs);
    if (dat[i]) cudaFreeAsync(dat[i], ks ? ks : cs);
    if (copied[i]) cudaEventDestroy(copied[i]);
    if (consumed[i]) cudaEventDestroy(consumed[i]);
  }
  if (dout) cudaFreeAsync(dout, ks);
  if (ks) { cudaStreamSynchronize(ks); cudaStreamDestroy(ks); }
  if (cs) cudaStreamDestroy(cs);
  return rc;
}

extern "C" int rb_instrument(int32_t op, int64_t* launches, int64_t* timed_launches, double* timed_ms) {
  if (op < 0 || op > 2) return fail(RB_CONFIG_ERROR, "rb_instrument op must be 0, 1 or 2");
  return instrument(op, launches, timed_launches, timed_ms);
}
