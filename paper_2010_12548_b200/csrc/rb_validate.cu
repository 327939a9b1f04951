// rb_validate.cu -- K5, the complete epsilon validator (north star: "a validator
// confirms that every point the approximation assigns differently from the
// exact test lies within eps of a polygon boundary").
//
// Every point, not a sample: its approximate owner set comes from the index
// (act_lookup semantics); its exact owner set from
// point_in_polygon (boundary = inside) over the candidate polygons
// of its bucket in a uniform grid of polygon MBRs expanded by eps (so every
// polygon within eps of the point is a candidate).  Each region in exactly one
// of the two sets is a mismatch; its distance to the region's boundary
// (min over the region's candidate polygons) must be <= eps.
// Counters and the maximum mismatch distance are reduced with atomics.
#include <algorithm>
#include <climits>
#include <cstring>

#include "rb_internal.cuh"

namespace rb {

#define RB_VAL_MAXSET 16

struct ValOut {
  unsigned long long points, mismatched_points, false_pos, false_neg, violations, max_dist_bits, overflow;
};

__device__ __forceinline__ bool set_has(const int32_t* s, int n, int32_t r) {
  for (int i = 0; i < n; ++i)
    if (s[i] == r) return true;
  return false;
}

__global__ void k_validate(IndexView V, double ox, double oy, double side, double inv_side, double lim,
                           const void* xy, int dtype, int64_t n, const double* vx, const double* vy,
                           const int64_t* ring_off, const int64_t* poly_ring_off, const int32_t* poly_region,
                           const double* mbr, const int32_t* bucket_off, const int32_t* bucket_poly, int nb,
                           double bx0, double by0, double bs, double eps, ValOut* out) {
  unsigned long long pts = 0, mis = 0, fp = 0, fn = 0, vio = 0, ovf = 0;
  double maxd = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double x, y;
    if (dtype == RB_XY_F64) { x = ((const double*)xy)[2 * i]; y = ((const double*)xy)[2 * i + 1]; }
    else { x = (double)((const float*)xy)[2 * i]; y = (double)((const float*)xy)[2 * i + 1]; }
    const double fx = cell_floor(x, ox, side, inv_side), fy = cell_floor(y, oy, side, inv_side);
    if (!(fx >= 0.0 && fx < lim && fy >= 0.0 && fy < lim)) continue;  // out of domain: not joined
    ++pts;
    // approximate owner regions (alpha owners) of the point's leaf
    int32_t aset[RB_VAL_MAXSET];
    int na = 0;
    const uint32_t v = index_lookup(V, (uint32_t)fx, (uint32_t)fy);
    if (v & RB_VALUE_LIST) {
      const uint32_t* Lp = V.pool + (v & RB_VALUE_PAYLOAD);
      const uint32_t k = Lp[0] & ~RB_POOL_COUNT_FLAG;
      for (uint32_t e = 1; e <= k; ++e) {
        const int32_t r = (int32_t)((Lp[e] & V.code_mask) >> 1);
        if (na < RB_VAL_MAXSET) { if (!set_has(aset, na, r)) aset[na++] = r; } else ++ovf;
      }
    } else if (v != 0u) {
      aset[na++] = (int32_t)(((v & V.code_mask) - 1u) >> 1);
    }
    // exact owner regions among the bucket's candidate polygons
    int32_t eset[RB_VAL_MAXSET];
    int ne = 0;
    int bxi = (int)floor((x - bx0) / bs), byi = (int)floor((y - by0) / bs);
    bxi = bxi < 0 ? 0 : (bxi >= nb ? nb - 1 : bxi);
    byi = byi < 0 ? 0 : (byi >= nb ? nb - 1 : byi);
    const int bk = byi * nb + bxi;
    for (int c = bucket_off[bk]; c < bucket_off[bk + 1]; ++c) {
      const int32_t p = bucket_poly[c];
      const double* m = mbr + 4 * (size_t)p;
      if (x < m[0] || x > m[2] || y < m[1] || y > m[3]) continue;
      if (pip_rings(vx, vy, ring_off, poly_ring_off[p], poly_ring_off[p + 1], x, y)) {
        const int32_t r = poly_region[p];
        if (ne < RB_VAL_MAXSET) { if (!set_has(eset, ne, r)) eset[ne++] = r; } else ++ovf;
      }
    }
    // mismatches: symmetric difference, each within eps of its region's boundary
    bool any = false;
    for (int pass = 0; pass < 2; ++pass) {
      const int32_t* A = pass == 0 ? aset : eset;
      const int32_t* B = pass == 0 ? eset : aset;
      const int nA = pass == 0 ? na : ne, nB = pass == 0 ? ne : na;
      for (int t = 0; t < nA; ++t) {
        const int32_t r = A[t];
        if (set_has(B, nB, r)) continue;
        any = true;
        if (pass == 0) ++fp; else ++fn;
        double d = INFINITY;
        for (int c = bucket_off[bk]; c < bucket_off[bk + 1]; ++c) {
          const int32_t p = bucket_poly[c];
          if (poly_region[p] != r) continue;
          const double dd = dist_rings(vx, vy, ring_off, poly_ring_off[p], poly_ring_off[p + 1], x, y);
          d = dd < d ? dd : d;
        }
        if (!(d <= eps)) ++vio;  // includes a region with no candidate polygon (d = inf)
        if (d < INFINITY && d > maxd) maxd = d;
      }
    }
    if (any) ++mis;
  }
  // warp-aggregate, then one atomic per warp
  for (int o = 16; o > 0; o >>= 1) {
    pts += __shfl_xor_sync(0xffffffffu, pts, o);
    mis += __shfl_xor_sync(0xffffffffu, mis, o);
    fp += __shfl_xor_sync(0xffffffffu, fp, o);
    fn += __shfl_xor_sync(0xffffffffu, fn, o);
    vio += __shfl_xor_sync(0xffffffffu, vio, o);
    ovf += __shfl_xor_sync(0xffffffffu, ovf, o);
    const double od = __shfl_xor_sync(0xffffffffu, maxd, o);
    maxd = od > maxd ? od : maxd;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out->points, pts);
    atomicAdd(&out->mismatched_points, mis);
    atomicAdd(&out->false_pos, fp);
    atomicAdd(&out->false_neg, fn);
    atomicAdd(&out->violations, vio);
    atomicAdd(&out->overflow, ovf);
    atomicMax(&out->max_dist_bits, (unsigned long long)__double_as_longlong(maxd));  // d >= 0: bit order = value order
  }
}

}  // namespace rb

using namespace rb;

extern "C" int rb_validate_full(const rb_approx* a, const rb_polygons* P, const double* poly_mbr,
                                const int32_t* bucket_off, const int32_t* bucket_poly, int32_t n_buckets_side,
                                double bucket_x0, double bucket_y0, double bucket_side, const void* xy,
                                int32_t xy_dtype, int64_t n, double epsilon, int64_t* out6, double* max_dist,
                                void* stream) {
  if (!a || !P || !poly_mbr || !bucket_off || !bucket_poly || !out6 || !max_dist)
    return fail(RB_CONFIG_ERROR, "null argument");
  if (xy_dtype != RB_XY_F64 && xy_dtype != RB_XY_F32) return fail(RB_CONFIG_ERROR, "unknown xy dtype");
  if (n < 0 || n_buckets_side <= 0 || !(bucket_side > 0.0)) return fail(RB_SHAPE_ERROR, "bad sizes");
  cudaStream_t s = (cudaStream_t)stream;
  DBuf o;
  RB_CUDA(o.alloc(sizeof(ValOut)));
  RB_CUDA(cudaMemsetAsync(o.p, 0, sizeof(ValOut), s));
  const int L = a->grid.max_level;
  const double side = ldexp(a->grid.extent, -L);
  if (n > 0) {
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    k_validate<<<blocks, 256, 0, s>>>(a->view(), a->grid.origin_x, a->grid.origin_y, side, 1.0 / side, ldexp(1.0, L),
                                      xy, xy_dtype, n, P->vx, P->vy, P->ring_off, P->poly_ring_off, P->poly_region,
                                      poly_mbr, bucket_off, bucket_poly, n_buckets_side, bucket_x0, bucket_y0,
                                      bucket_side, epsilon, o.as<ValOut>());
    RB_CUDA(cudaGetLastError());
  }
  ValOut h{};
  RB_CUDA(cudaMemcpyAsync(&h, o.p, sizeof(ValOut), cudaMemcpyDeviceToHost, s));
  RB_CUDA(cudaStreamSynchronize(s));
  out6[0] = (int64_t)h.points;
  out6[1] = (int64_t)h.mismatched_points;
  out6[2] = (int64_t)h.false_pos;
  out6[3] = (int64_t)h.false_neg;
  out6[4] = (int64_t)h.violations;
  out6[5] = (int64_t)h.overflow;
  std::memcpy(max_dist, &h.max_dist_bits, sizeof(double));
  return RB_OK;
}
