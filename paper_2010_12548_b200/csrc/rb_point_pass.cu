// rb_point_pass.cu -- K1: the streaming point pass of join_act
// (north star subsystem 3).
//
// One persistent grid; every thread streams 32-byte chunks of the
// interleaved coordinates with 256-bit non-allocating, evict-first loads
// (plus the matching attribute words), quantises each point to its leaf
// (floor((p - origin)/side), bit-identical to the oracle),
// descends the L2-resident radix table to the owner value and accumulates
// alpha/beta COUNT and SUM for EVERY owner:
//   COUNT: u32 shared-memory atomics (native ATOMS.ADD)
//   SUM  : float64 shared-memory accumulators
// Each CTA then writes its private histogram to a scratch row and a second
// kernel reduces the rows in CTA order -- deterministic, no global atomics.
// Region sets too large for shared memory accumulate straight into global
// memory with native REDG.ADD.64 / REDG.ADD.F64.
#include <atomic>
#include <climits>
#include <mutex>
#include <utility>
#include <vector>

#include "rb_internal.cuh"

namespace rb {

// ---- instrumentation (rb_instrument): launches of this library's kernels and
// CUDA-event time of the point-pass main kernel (bench.py roofline).
std::atomic<int64_t> g_launches{0};
static std::atomic<bool> g_timing{false};
static std::mutex g_ev_mu;
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_events;

int instrument(int op, int64_t* launches, int64_t* timed, double* ms) {
  std::lock_guard<std::mutex> lk(g_ev_mu);
  if (op == 0) {
    double tot = 0.0;
    for (auto& e : g_events) {
      RB_CUDA(cudaEventSynchronize(e.second));
      float t = 0.f;
      RB_CUDA(cudaEventElapsedTime(&t, e.first, e.second));
      tot += t;
    }
    if (launches) *launches = g_launches.load();
    if (timed) *timed = (int64_t)g_events.size();
    if (ms) *ms = tot;
    return RB_OK;
  }
  for (auto& e : g_events) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  g_events.clear();
  g_launches = 0;
  g_timing = (op == 1);
  return RB_OK;
}

__device__ __forceinline__ void ld256(const void* p, uint64_t& a, uint64_t& b, uint64_t& c, uint64_t& d) {
  asm("ld.global.nc.L1::no_allocate.L2::evict_first.v4.u64 {%0,%1,%2,%3}, [%4];"
      : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
      : "l"(p));
}
__device__ __forceinline__ void ld64f2(const float* p, float& a, float& b) {
  asm("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(a), "=f"(b) : "l"(p));
}
__device__ __forceinline__ void ld128f4(const float* p, float& a, float& b, float& c, float& d) {
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
      : "l"(p));
}

struct PassArgs {
  IndexView V;
  double ox, oy, side, inv_side, lim;
  const void* xy;
  const float* attr;
  int64_t n;
  int R2;  // 2 * n_regions
  uint32_t* part_cnt;
  double* part_sum;
  unsigned long long* gcnt;
  double* gsum;
  unsigned long long* first_bad;
  int64_t idx_base;  // global index of point 0 (chunked host joins)
};

template <bool SMEM, bool ATTR>
struct Hist {
  uint32_t* scnt;
  double* ssum;
  const PassArgs* a;
  __device__ __forceinline__ void add(uint32_t q, double w) {
    if (SMEM) {
      atomicAdd(&scnt[q], 1u);
      if (ATTR) atomicAdd(&ssum[q], w);
    } else {
      atomicAdd(&a->gcnt[q], 1ull);
      if (ATTR) atomicAdd(&a->gsum[q], w);
    }
  }
};

template <bool SMEM, bool ATTR>
__device__ __forceinline__ void point(const PassArgs& a, Hist<SMEM, ATTR>& h, double x, double y, float wf,
                                      int64_t idx) {
  double fx = cell_floor(x, a.ox, a.side, a.inv_side);
  double fy = cell_floor(y, a.oy, a.side, a.inv_side);
  if (!(fx >= 0.0 && fx < a.lim && fy >= 0.0 && fy < a.lim)) {
    atomicMin(a.first_bad, (unsigned long long)(a.idx_base + idx));
    return;
  }
  uint32_t val = index_lookup(a.V, (uint32_t)fx, (uint32_t)fy);
  if (val == 0) return;
  double w = (double)wf;
  if (!(val & RB_VALUE_LIST)) {
    uint32_t s = val - 1u;
    uint32_t q = s & ~1u;  // 2 * region
    h.add(q, w);
    if (s & 1u) h.add(q + 1, w);
  } else {
    const uint32_t* L = a.V.pool + (val & RB_VALUE_PAYLOAD);
    uint32_t k = __ldg(L);
    for (uint32_t e = 1; e <= k; ++e) {
      uint32_t ent = __ldg(L + e);
      uint32_t q = ent & ~1u;
      h.add(q, w);
      if (ent & 1u) h.add(q + 1, w);
    }
  }
}

// XY: 0 = f64 interleaved, 1 = f32 interleaved.  VEC: vectorised main loop.
template <int XY, bool SMEM, bool ATTR, bool VEC>
__global__ void __launch_bounds__(512) k_point_pass(PassArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  Hist<SMEM, ATTR> h;
  h.a = &a;
  h.ssum = (double*)smem;
  h.scnt = (uint32_t*)(smem + (SMEM ? (size_t)a.R2 * 8 : 0));
  if (SMEM) {
    for (int q = threadIdx.x; q < a.R2; q += blockDim.x) { h.scnt[q] = 0; h.ssum[q] = 0.0; }
    __syncthreads();
  }
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (VEC) {
    if (XY == 0) {
      // chunk = 2 points = 32 bytes of xy + 8 bytes of attr
      const int64_t nch = a.n >> 1;
      const char* base = (const char*)a.xy;
      int64_t c = tid;
      for (; c + nth < nch; c += 2 * nth) {
        uint64_t u0, u1, u2, u3, v0, v1, v2, v3;
        float w0 = 0.f, w1 = 0.f, w2 = 0.f, w3 = 0.f;
        ld256(base + c * 32, u0, u1, u2, u3);
        ld256(base + (c + nth) * 32, v0, v1, v2, v3);
        if (ATTR) { ld64f2(a.attr + 2 * c, w0, w1); ld64f2(a.attr + 2 * (c + nth), w2, w3); }
        point(a, h, __longlong_as_double(u0), __longlong_as_double(u1), w0, 2 * c);
        point(a, h, __longlong_as_double(u2), __longlong_as_double(u3), w1, 2 * c + 1);
        point(a, h, __longlong_as_double(v0), __longlong_as_double(v1), w2, 2 * (c + nth));
        point(a, h, __longlong_as_double(v2), __longlong_as_double(v3), w3, 2 * (c + nth) + 1);
      }
      for (; c < nch; c += nth) {
        uint64_t u0, u1, u2, u3;
        float w0 = 0.f, w1 = 0.f;
        ld256(base + c * 32, u0, u1, u2, u3);
        if (ATTR) ld64f2(a.attr + 2 * c, w0, w1);
        point(a, h, __longlong_as_double(u0), __longlong_as_double(u1), w0, 2 * c);
        point(a, h, __longlong_as_double(u2), __longlong_as_double(u3), w1, 2 * c + 1);
      }
      done = nch << 1;
    } else {
      // chunk = 4 points = 32 bytes of xy + 16 bytes of attr
      const int64_t nch = a.n >> 2;
      const char* base = (const char*)a.xy;
      for (int64_t c = tid; c < nch; c += nth) {
        uint64_t u[4];
        float w[4] = {0.f, 0.f, 0.f, 0.f};
        ld256(base + c * 32, u[0], u[1], u[2], u[3]);
        if (ATTR) ld128f4(a.attr + 4 * c, w[0], w[1], w[2], w[3]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float x = __uint_as_float((uint32_t)u[j]), y = __uint_as_float((uint32_t)(u[j] >> 32));
          point(a, h, (double)x, (double)y, w[j], 4 * c + j);
        }
      }
      done = nch << 2;
    }
  }
  for (int64_t i = done + tid; i < a.n; i += nth) {
    double x, y;
    if (XY == 0) { x = ((const double*)a.xy)[2 * i]; y = ((const double*)a.xy)[2 * i + 1]; }
    else { x = (double)((const float*)a.xy)[2 * i]; y = (double)((const float*)a.xy)[2 * i + 1]; }
    point(a, h, x, y, ATTR ? a.attr[i] : 0.f, i);
  }
  if (SMEM) {
    __syncthreads();
    uint32_t* pc = a.part_cnt + (size_t)blockIdx.x * a.R2;
    double* ps = a.part_sum + (size_t)blockIdx.x * a.R2;
    for (int q = threadIdx.x; q < a.R2; q += blockDim.x) {
      pc[q] = h.scnt[q];
      if (ATTR) ps[q] = h.ssum[q];
    }
  }
}

// deterministic reduction of the per-CTA rows (fixed CTA order)
__global__ void k_reduce_rows(const uint32_t* part_cnt, const double* part_sum, int nrows, int R2, bool attr,
                              int accumulate, int64_t* cnt_out, double* sum_out) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < R2; q += gridDim.x * blockDim.x) {
    uint64_t c = 0;
    double s = 0.0;
    for (int r = 0; r < nrows; ++r) {
      c += part_cnt[(size_t)r * R2 + q];
      if (attr) s += part_sum[(size_t)r * R2 + q];
    }
    if (accumulate) { cnt_out[q] += (int64_t)c; sum_out[q] += s; }
    else { cnt_out[q] = (int64_t)c; sum_out[q] = s; }
  }
}

__global__ void k_init_out(int64_t* cnt_out, double* sum_out, int R2, int flags, unsigned long long* first_bad) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < R2; q += gridDim.x * blockDim.x) {
    if (flags & 1) { cnt_out[q] = 0; sum_out[q] = 0.0; }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (flags & 2)) *first_bad = (unsigned long long)LLONG_MAX;
}

template <int XY, bool SMEM, bool ATTR, bool VEC>
static cudaError_t launch_t(const PassArgs& a, int blocks, size_t smem, cudaStream_t s) {
  auto kern = k_point_pass<XY, SMEM, ATTR, VEC>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  kern<<<blocks, 512, smem, s>>>(a);
  return cudaGetLastError();
}

template <int XY, bool SMEM, bool ATTR>
static cudaError_t launch_v(const PassArgs& a, bool vec, int blocks, size_t smem, cudaStream_t s) {
  return vec ? launch_t<XY, SMEM, ATTR, true>(a, blocks, smem, s) : launch_t<XY, SMEM, ATTR, false>(a, blocks, smem, s);
}

template <int XY, bool SMEM>
static cudaError_t launch_a(const PassArgs& a, bool vec, int blocks, size_t smem, cudaStream_t s) {
  return a.attr ? launch_v<XY, SMEM, true>(a, vec, blocks, smem, s) : launch_v<XY, SMEM, false>(a, vec, blocks, smem, s);
}

static int g_num_sms = 0;

// flags: bit0 = zero the outputs first, bit1 = reset first_bad first
int point_pass(const rb_approx* A, const void* xy, int32_t dtype, int64_t n, const float* attr, int64_t* cnt_out,
               double* sum_out, int64_t* first_bad, int flags, int64_t idx_base, cudaStream_t s) {
  if (!g_num_sms) {
    int dev = 0;
    RB_CUDA(cudaGetDevice(&dev));
    RB_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int R2 = 2 * A->n_regions;
  PassArgs a{};
  a.V = A->view();
  const int L = A->grid.max_level;
  a.side = ldexp(A->grid.extent, -L);
  a.inv_side = 1.0 / a.side;
  a.ox = A->grid.origin_x;
  a.oy = A->grid.origin_y;
  a.lim = ldexp(1.0, L);
  a.xy = xy;
  a.attr = attr;
  a.n = n;
  a.R2 = R2;
  a.first_bad = (unsigned long long*)first_bad;
  a.gcnt = (unsigned long long*)cnt_out;
  a.gsum = sum_out;
  a.idx_base = idx_base;
  const bool smem_hist = (size_t)R2 * 12 <= 96 * 1024;
  const size_t smem = smem_hist ? (size_t)R2 * 12 : 0;
  bool vec = ((uintptr_t)xy % 32 == 0) && (!attr || (uintptr_t)attr % (dtype == RB_XY_F64 ? 8 : 16) == 0);
  int per_sm = smem_hist ? std::max(1, std::min(4, (int)((200 * 1024) / std::max<size_t>(smem, 1)))) : 4;
  int blocks = g_num_sms * per_sm;
  if (flags) {
    k_init_out<<<std::max(1, (R2 + 255) / 256), 256, 0, s>>>(cnt_out, sum_out, R2, flags, a.first_bad);
    RB_CUDA(cudaGetLastError());
    ++g_launches;
  }
  if (n == 0) return RB_OK;
  void* scratch = nullptr;
  if (smem_hist) {
    size_t bytes = (size_t)blocks * R2 * (4 + (attr ? 8 : 0));
    RB_CUDA(cudaMallocAsync(&scratch, bytes, s));
    a.part_cnt = (uint32_t*)scratch;
    a.part_sum = (double*)((char*)scratch + (size_t)blocks * R2 * 4);
  }
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (g_timing) {
    RB_CUDA(cudaEventCreate(&ev0));
    RB_CUDA(cudaEventCreate(&ev1));
    RB_CUDA(cudaEventRecord(ev0, s));
  }
  cudaError_t e;
  if (dtype == RB_XY_F64)
    e = smem_hist ? launch_a<0, true>(a, vec, blocks, smem, s) : launch_a<0, false>(a, vec, blocks, smem, s);
  else
    e = smem_hist ? launch_a<1, true>(a, vec, blocks, smem, s) : launch_a<1, false>(a, vec, blocks, smem, s);
  if (e) return cuda_fail(e, "k_point_pass");
  ++g_launches;
  if (g_timing) {
    RB_CUDA(cudaEventRecord(ev1, s));
    std::lock_guard<std::mutex> lk(g_ev_mu);
    g_events.emplace_back(ev0, ev1);
  }
  if (smem_hist) {
    k_reduce_rows<<<std::max(1, (R2 + 255) / 256), 256, 0, s>>>(a.part_cnt, a.part_sum, blocks, R2, attr != nullptr,
                                                                1, cnt_out, sum_out);
    RB_CUDA(cudaGetLastError());
    ++g_launches;
    RB_CUDA(cudaFreeAsync(scratch, s));
  }
  return RB_OK;
}

// act_lookup for a batch: owner value per point
__global__ void k_lookup(IndexView V, double ox, double oy, double side, double inv_side, double lim, const void* xy,
                         int dtype, int64_t n, uint32_t* out, unsigned long long* first_bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double x, y;
    if (dtype == 0) { x = ((const double*)xy)[2 * i]; y = ((const double*)xy)[2 * i + 1]; }
    else { x = (double)((const float*)xy)[2 * i]; y = (double)((const float*)xy)[2 * i + 1]; }
    double fx = cell_floor(x, ox, side, inv_side), fy = cell_floor(y, oy, side, inv_side);
    if (!(fx >= 0.0 && fx < lim && fy >= 0.0 && fy < lim)) {
      atomicMin(first_bad, (unsigned long long)i);
      out[i] = 0;
      continue;
    }
    out[i] = index_lookup(V, (uint32_t)fx, (uint32_t)fy);
  }
}

__global__ void k_point_cells(double ox, double oy, double side, double inv_side, double lim, const void* xy, int dtype,
                              int64_t n, uint32_t* ix, uint32_t* iy, unsigned long long* first_bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double x, y;
    if (dtype == 0) { x = ((const double*)xy)[2 * i]; y = ((const double*)xy)[2 * i + 1]; }
    else { x = (double)((const float*)xy)[2 * i]; y = (double)((const float*)xy)[2 * i + 1]; }
    double fx = cell_floor(x, ox, side, inv_side), fy = cell_floor(y, oy, side, inv_side);
    if (!(fx >= 0.0 && fx < lim && fy >= 0.0 && fy < lim)) {
      atomicMin(first_bad, (unsigned long long)i);
      ix[i] = 0xffffffffu; iy[i] = 0xffffffffu;
      continue;
    }
    ix[i] = (uint32_t)fx; iy[i] = (uint32_t)fy;
  }
}

__global__ void k_reset_bad(unsigned long long* first_bad) { *first_bad = (unsigned long long)LLONG_MAX; }

int lookup(const rb_approx* A, const void* xy, int32_t dtype, int64_t n, uint32_t* out, int64_t* first_bad,
           cudaStream_t s) {
  const int L = A->grid.max_level;
  double side = ldexp(A->grid.extent, -L);
  k_reset_bad<<<1, 1, 0, s>>>((unsigned long long*)first_bad);
  if (n > 0)
    k_lookup<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, s>>>(
        A->view(), A->grid.origin_x, A->grid.origin_y, side, 1.0 / side, ldexp(1.0, L), xy, dtype, n, out,
        (unsigned long long*)first_bad);
  RB_CUDA(cudaGetLastError());
  return RB_OK;
}

int point_cells(const rb_grid* g, const void* xy, int32_t dtype, int64_t n, uint32_t* ix, uint32_t* iy,
                int64_t* first_bad, cudaStream_t s) {
  const int L = g->max_level;
  double side = ldexp(g->extent, -L);
  k_reset_bad<<<1, 1, 0, s>>>((unsigned long long*)first_bad);
  if (n > 0)
    k_point_cells<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, s>>>(
        g->origin_x, g->origin_y, side, 1.0 / side, ldexp(1.0, L), xy, dtype, n, ix, iy,
        (unsigned long long*)first_bad);
  RB_CUDA(cudaGetLastError());
  return RB_OK;
}

// ---- K5 validator kernels: exact PIP / distance of point k vs polygon poly_of_point[k]
__global__ void k_exact_pip(const double* vx, const double* vy, const int64_t* ring_off, const int64_t* poly_ring_off,
                            const double* px, const double* py, const int32_t* pp, int64_t n, uint8_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int p = pp[i];
    out[i] = (uint8_t)pip_rings(vx, vy, ring_off, poly_ring_off[p], poly_ring_off[p + 1], px[i], py[i]);
  }
}
__global__ void k_exact_dist(const double* vx, const double* vy, const int64_t* ring_off, const int64_t* poly_ring_off,
                             const double* px, const double* py, const int32_t* pp, int64_t n, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int p = pp[i];
    out[i] = dist_rings(vx, vy, ring_off, poly_ring_off[p], poly_ring_off[p + 1], px[i], py[i]);
  }
}

int exact_pip(const rb_polygons* P, const double* px, const double* py, const int32_t* pp, int64_t n, uint8_t* out,
              cudaStream_t s) {
  if (n > 0)
    k_exact_pip<<<(int)std::min<int64_t>((n + 127) / 128, 148 * 32), 128, 0, s>>>(P->vx, P->vy, P->ring_off,
                                                                                  P->poly_ring_off, px, py, pp, n, out);
  RB_CUDA(cudaGetLastError());
  return RB_OK;
}
int exact_distance(const rb_polygons* P, const double* px, const double* py, const int32_t* pp, int64_t n,
                   double* out, cudaStream_t s) {
  if (n > 0)
    k_exact_dist<<<(int)std::min<int64_t>((n + 127) / 128, 148 * 32), 128, 0, s>>>(P->vx, P->vy, P->ring_off,
                                                                                   P->poly_ring_off, px, py, pp, n, out);
  RB_CUDA(cudaGetLastError());
  return RB_OK;
}

}  // namespace rb
