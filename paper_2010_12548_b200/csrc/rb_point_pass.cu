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
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
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
  long long* part_acc;
  int* scale_exp;
  const int32_t* hot_region;  // global mode: hot slot -> region
  int n_hot;
  int hcopies;  // warp kernel: copies of the shared histogram (lane & (hcopies-1) picks one)
  int hstride;  // warp kernel: words per histogram copy (== 1 mod 32: a bin's copies sit in distinct banks)
  int ablate;   // timing experiments only (RB_ABLATE): 1 skip the rare path
  int fold;     // ring kernel: cap on the drain period in warp-tiles (RB_FOLD, tests); 0 = automatic
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
    uint32_t s = (val & a.V.code_mask) - 1u;
    uint32_t q = s & ~1u;  // 2 * region
    h.add(q, w);
    if (s & 1u) h.add(q + 1, w);
  } else {
    const uint32_t* L = a.V.pool + (val & RB_VALUE_PAYLOAD);
    uint32_t k = __ldg(L) & ~RB_POOL_COUNT_FLAG;
    for (uint32_t e = 1; e <= k; ++e) {
      uint32_t ent = __ldg(L + e) & a.V.code_mask;
      uint32_t q = ent & ~1u;
      h.add(q, w);
      if (ent & 1u) h.add(q + 1, w);
    }
  }
}

// Large region sets (histogram does not fit in shared memory): accumulate
// straight into global memory.  XY: 0 = f64, 1 = f32.  VEC: 32-byte loads.
template <int XY, bool SMEM, bool ATTR, bool VEC>
__global__ void __launch_bounds__(512) k_point_pass_global(PassArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
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


// ---------------------------------------------------------------------------
// Shared-memory histogram kernel (region sets up to RB_SMEM_MAX_REGIONS).
//
// * grid = SMs x resident CTAs (occupancy API); CTA b streams a contiguous
//   range of 32-byte chunks, lane-interleaved so every load instruction of a
//   warp covers 1 KB of consecutive memory;
// * each thread handles PB = 8 points per iteration: all coordinates are
//   loaded first, all leaf cells computed, then all root-table reads issued
//   together, then each node level -- the dependent index chain overlaps
//   across the 8 points instead of serialising per point;
// * COUNT: native u32 smem atomics.  SUM: per-launch binary scale 2^S chosen
//   from a sample of the attribute (k_attr_scale); values whose scaled
//   magnitude lies in [2^20, 2^30) are accumulated exactly as int32 fixed
//   point split over two u32 atomics (low 16 / signed high 16 bits), folded
//   into int64 every 65536 points of the CTA; everything else (huge, tiny,
//   non-finite) goes to a float64 slow path.  Relative quantisation error per
//   value <= 2^-21 (< 1e-6), and the fixed-point part is order-independent.
// ---------------------------------------------------------------------------
#define RB_PB 8
#ifndef RB_MINB
#define RB_MINB 2
#endif

struct LevelDesc {
  const uint32_t* nodes[RB_MAX_NODE_LEVELS];
  int ks[RB_MAX_NODE_LEVELS];
};

template <bool ATTR>
struct SHist {
  uint32_t* cnt;
  uint32_t* lo;
  uint32_t* hi;
  double* slow;
  __device__ __forceinline__ void add_fast(uint32_t q, int32_t qv) {
    atomicAdd(&cnt[q], 1u);
    if (ATTR) {
      atomicAdd(&lo[q], (uint32_t)qv & 0xffffu);
      atomicAdd(&hi[q], (uint32_t)(qv >> 16));
    }
  }
  __device__ __forceinline__ void add_slow(uint32_t q, float w) {
    atomicAdd(&cnt[q], 1u);
    if (ATTR) atomicAdd(&slow[q], (double)w);
  }
  __device__ __forceinline__ void add(uint32_t q, float w, int32_t qv, bool fast) {
    if (fast) add_fast(q, qv); else add_slow(q, w);
  }
};

// Interleaved shared-memory histogram for the TMA kernel: bin q owns words
// h3[3q] (count), h3[3q+1] (fixed-point low 16 bits), h3[3q+2] (signed high
// part); stride 3 is coprime with the 32 banks, one base IMAD per update.
template <bool ATTR>
struct IHist {
  uint32_t* h3;              // shared bins: count, fixed-point low 16 bits, signed high part
  double* slow;              // shared float64 sums of out-of-window values (smem mode)
  unsigned long long* gcnt;  // non-null: global mode (region set beyond shared memory)
  double* gsum;
  __device__ __forceinline__ void fixed(uint32_t b, int32_t qv) {
    uint32_t* p = h3 + (ATTR ? 3u * b : b);
    atomicAdd(p, 1u);
    if (ATTR) {
      atomicAdd(p + 1, (uint32_t)qv & 0xffffu);
      atomicAdd(p + 2, (uint32_t)(qv >> 16));
    }
  }
  // bin q = 2*region (+1 for beta); slot = hot slot + 1 of the region (global mode)
  __device__ __forceinline__ void add(uint32_t q, uint32_t slot, float w, int32_t qv, bool fast) {
    if (gcnt) {
      if (slot && !(q & 1u) && fast) { fixed(slot - 1u, qv); return; }
      atomicAdd(&gcnt[q], 1ull);  // REDG.ADD.64
      if (ATTR) atomicAdd(&gsum[q], (double)w);  // REDG.ADD.F64
      return;
    }
    if (fast) { fixed(q, qv); return; }
    atomicAdd(h3 + (ATTR ? 3u * q : q), 1u);
    if (ATTR) atomicAdd(&slow[q], (double)w);
  }
};

template <bool ATTR>
__device__ __noinline__ void add_owners_i(IHist<ATTR> h, const uint32_t* __restrict__ pool, uint32_t v, float w,
                                          int32_t qv, bool fast, uint32_t cm, uint32_t hs) {
  if (!(v & RB_VALUE_LIST)) {
    const uint32_t sv = (v & cm) - 1u, q = sv & ~1u;
    h.add(q, v >> hs, w, qv, fast);
    if (sv & 1u) h.add(q + 1, 0u, w, qv, fast);
    return;
  }
  const uint32_t* Lp = pool + (v & RB_VALUE_PAYLOAD);
  const uint32_t kk = __ldg(Lp) & ~RB_POOL_COUNT_FLAG;
  for (uint32_t e = 1; e <= kk; ++e) {
    const uint32_t x = __ldg(Lp + e);
    const uint32_t ent = x & cm;
    const uint32_t q = ent & ~1u;
    h.add(q, x >> hs, w, qv, fast);
    if (ent & 1u) h.add(q + 1, 0u, w, qv, fast);
  }
}

// predicated 32-bit read-only load: returns dflt without touching memory when !pred
__device__ __forceinline__ uint32_t ldg_pred(const uint32_t* ptr, bool pred, uint32_t dflt) {
  uint32_t v;
  // not volatile: a pure read of the immutable index, free to be scheduled with its neighbours
  asm("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n mov.u32 %0, %3;\n @p ld.global.nc.u32 %0, [%1];\n}\n"
      : "=r"(v)
      : "l"(ptr), "r"((uint32_t)pred), "r"(dflt));
  return v;
}

// predicated 16-byte read-only load (RB_LAYOUT_PACKED block): {dflt, 0, 0, 0} when !pred, which
// packed_pick resolves to dflt (palette index 0)
__device__ __forceinline__ uint4 ldg4_pred(const uint4* ptr, bool pred, uint32_t dflt) {
  uint4 v;
  asm("{\n .reg .pred p;\n setp.ne.u32 p, %4, 0;\n mov.u32 %0, %5;\n mov.u32 %1, 0;\n mov.u32 %2, 0;\n"
      " mov.u32 %3, 0;\n @p ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%6];\n}\n"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "r"((uint32_t)pred), "r"(dflt), "l"(ptr));
  return v;
}

struct PassConst {
  double ox, oy, side, inv_side, lim;
  const uint32_t* root;
  const uint32_t* pool;
  uint32_t hmax;   // (2^L - 1) >> 12: bound on t's high word minus 0x41F00000
  uint32_t lim_u;  // 2^L (exclusive, for L < 12)
  int L, T0, s0, nlev;
};

// Rare path 1: exact division + domain check for a point
// whose fast quantisation was not conclusive.  Returns false if out of domain.
__device__ __noinline__ uint64_t quantize_exact(const void* xy, int64_t pidx, int XY, double ox, double oy, double side,
                                                double lim, unsigned long long* first_bad, int64_t idx_base) {
  double xx, yy;
  if (XY == 0) { xx = ((const double*)xy)[2 * pidx]; yy = ((const double*)xy)[2 * pidx + 1]; }
  else { xx = (double)((const float*)xy)[2 * pidx]; yy = (double)((const float*)xy)[2 * pidx + 1]; }
  const double fx = floor(__ddiv_rn(__dsub_rn(xx, ox), side));
  const double fy = floor(__ddiv_rn(__dsub_rn(yy, oy), side));
  if (!(fx >= 0.0 && fx < lim && fy >= 0.0 && fy < lim)) {
    atomicMin(first_bad, (unsigned long long)(idx_base + pidx));
    return ~0ull;
  }
  return ((uint64_t)(uint32_t)fy << 32) | (uint32_t)fx;
}

// Rare path 2: owner lists and boundary owners (multi-owner cells).
template <bool ATTR>
__device__ __noinline__ void add_owners(SHist<ATTR> h, const uint32_t* __restrict__ pool, uint32_t v, float w,
                                        int32_t qv, bool fast, uint32_t cm) {
  if (!(v & RB_VALUE_LIST)) {
    const uint32_t sv = (v & cm) - 1u, q = sv & ~1u;
    h.add(q, w, qv, fast);
    if (sv & 1u) h.add(q + 1, w, qv, fast);
    return;
  }
  const uint32_t* Lp = pool + (v & RB_VALUE_PAYLOAD);
  const uint32_t kk = __ldg(Lp) & ~RB_POOL_COUNT_FLAG;
  for (uint32_t e = 1; e <= kk; ++e) {
    const uint32_t ent = __ldg(Lp + e) & cm;
    const uint32_t q = ent & ~1u;
    h.add(q, w, qv, fast);
    if (ent & 1u) h.add(q + 1, w, qv, fast);
  }
}

template <int XY, bool ATTR, bool VEC>
__global__ void __launch_bounds__(256, RB_MINB) k_point_pass(PassArgs a) {
  constexpr int PPC = XY == 0 ? 2 : 4;  // points per 32-byte chunk
  constexpr int CPT = RB_PB / PPC;      // chunks per thread per iteration
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ LevelDesc lv;
  const int R2 = a.R2;
  long long* acc = (long long*)smem;
  double* slow = (double*)(smem + (size_t)R2 * 8);
  uint32_t* cnt = (uint32_t*)(smem + (size_t)R2 * (ATTR ? 16 : 0));
  SHist<ATTR> h{cnt, cnt + R2, cnt + 2 * R2, slow};
  for (int q = threadIdx.x; q < R2; q += blockDim.x) {
    cnt[q] = 0;
    if (ATTR) { h.lo[q] = 0; h.hi[q] = 0; acc[q] = 0; slow[q] = 0.0; }
  }
  if (threadIdx.x < RB_MAX_NODE_LEVELS) {
    lv.nodes[threadIdx.x] = a.V.nodes[threadIdx.x];
    lv.ks[threadIdx.x] = a.V.ks[threadIdx.x];
  }
  __syncthreads();
  float sc = 1.f, wmax = 0.f, wmin = 0.f;
  if (ATTR) {
    const int S = *a.scale_exp;
    sc = __int_as_float((S + 127) << 23);
    wmax = __int_as_float((30 - S + 127) << 23);
    wmin = __int_as_float((20 - S + 127) << 23);
  }
  PassConst c;
  c.ox = a.ox; c.oy = a.oy; c.side = a.side; c.inv_side = a.inv_side; c.lim = a.lim;
  c.root = a.V.root; c.pool = a.V.pool;
  c.L = a.V.L; c.T0 = a.V.T0; c.s0 = c.L - c.T0; c.nlev = a.V.nlev;
  c.lim_u = c.L >= 32 ? 0xffffffffu : (1u << c.L);
  c.hmax = (uint32_t)(((1ull << c.L) - 1ull) >> 12);
  const int64_t nchunks = a.n / PPC;
  const int64_t per_cta = (nchunks + gridDim.x - 1) / gridDim.x;
  const int64_t c_beg = (int64_t)blockIdx.x * per_cta;
  const int64_t c_end = c_beg + per_cta < nchunks ? c_beg + per_cta : nchunks;
  const int64_t span = (int64_t)blockDim.x * CPT;
  const int64_t iters = c_end > c_beg ? (c_end - c_beg + span - 1) / span : 0;
  const int64_t epi = (65536 / (blockDim.x * RB_PB)) > 0 ? (65536 / (blockDim.x * RB_PB)) : 1;
  const char* base = (const char*)a.xy;

  for (int64_t it0 = 0; it0 < iters; it0 += epi) {
    const int64_t it1 = it0 + epi < iters ? it0 + epi : iters;
    for (int64_t it = it0; it < it1; ++it) {
      uint32_t ix[RB_PB], iy[RB_PB], val[RB_PB];
      float w[RB_PB];
      uint32_t okm = 0, slowm = 0;
      const int64_t cb = c_beg + it * span + threadIdx.x;
      // 1. loads + quantisation.  t = RN(RN(RN(v - o) * inv_side) + 2^32)
      //    holds floor(q) in mantissa bits 20..51 and q's fraction rounded to
      //    2^-20 in bits 0..19; its high word minus 0x41F00000 is <= hmax iff
      //    0 <= q < 2^32 and floor(q) >> 12 < 2^(L-12).  A point whose fraction
      //    lies within 2^-19 of an integer, or that fails the range test, takes
      //    the exact path (bit-identical to floor(RN(d / side))).
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const int64_t ch = cb + (int64_t)k * blockDim.x;
        const bool v = ch < c_end;
        uint64_t u[4] = {0, 0, 0, 0};
        if (v) {
          if (VEC) ld256(base + ch * 32, u[0], u[1], u[2], u[3]);
          else {
            const uint64_t* p = (const uint64_t*)(base + ch * 32);
            u[0] = p[0]; u[1] = p[1]; u[2] = p[2]; u[3] = p[3];
          }
        }
        if (ATTR) {
          if (XY == 0) {
            if (v) {
              if (VEC) ld64f2(a.attr + 2 * ch, w[2 * k], w[2 * k + 1]);
              else { w[2 * k] = a.attr[2 * ch]; w[2 * k + 1] = a.attr[2 * ch + 1]; }
            } else { w[2 * k] = 0.f; w[2 * k + 1] = 0.f; }
          } else {
            if (v) {
              if (VEC) ld128f4(a.attr + 4 * ch, w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
              else {
#pragma unroll
                for (int j = 0; j < 4; ++j) w[4 * k + j] = a.attr[4 * ch + j];
              }
            } else {
#pragma unroll
              for (int j = 0; j < 4; ++j) w[4 * k + j] = 0.f;
            }
          }
        }
#pragma unroll
        for (int j = 0; j < PPC; ++j) {
          const int i = k * PPC + j;
          double x, y;
          if (XY == 0) { x = __longlong_as_double(u[2 * j]); y = __longlong_as_double(u[2 * j + 1]); }
          else {
            x = (double)__uint_as_float((uint32_t)u[j]);
            y = (double)__uint_as_float((uint32_t)(u[j] >> 32));
          }
          const double tx = __dadd_rn(__dmul_rn(__dsub_rn(x, c.ox), c.inv_side), 4294967296.0);
          const double ty = __dadd_rn(__dmul_rn(__dsub_rn(y, c.oy), c.inv_side), 4294967296.0);
          const uint32_t lx = (uint32_t)__double2loint(tx), hx = (uint32_t)__double2hiint(tx);
          const uint32_t ly = (uint32_t)__double2loint(ty), hy = (uint32_t)__double2hiint(ty);
          ix[i] = __funnelshift_r(lx, hx, 20);
          iy[i] = __funnelshift_r(ly, hy, 20);
          const bool good = ((hx - 0x41F00000u) <= c.hmax) & ((hy - 0x41F00000u) <= c.hmax) &
                            (((lx + 2u) & 0xfffffu) >= 4u) & (((ly + 2u) & 0xfffffu) >= 4u) &
                            (ix[i] < c.lim_u) & (iy[i] < c.lim_u);
          okm |= (v & good) ? (1u << i) : 0u;
          slowm |= (v & !good) ? (1u << i) : 0u;
        }
      }
      if (slowm) {
#pragma unroll 1
        for (uint32_t m = slowm; m; m &= m - 1) {
          const int i = __ffs(m) - 1;
          const int64_t pidx = (cb + (int64_t)(i / PPC) * blockDim.x) * PPC + (i % PPC);
          const uint64_t qq = quantize_exact(a.xy, pidx, XY, c.ox, c.oy, c.side, c.lim, a.first_bad, a.idx_base);
          const uint32_t qx = (uint32_t)qq, qy = (uint32_t)(qq >> 32);
          if (qq != ~0ull) {
            // write back through a switch so the arrays stay in registers
#pragma unroll
            for (int t = 0; t < RB_PB; ++t)
              if (t == i) { ix[t] = qx; iy[t] = qy; }
            okm |= 1u << i;
          }
        }
      }
      // 2. root reads for all points, then node levels (ACT descent); the sorted-key
      //    layout (RB_LAYOUT_KEYS) instead searches its keys per point
      if (a.V.krec) {
#pragma unroll
        for (int i = 0; i < RB_PB; ++i) val[i] = (okm >> i) & 1u ? keys_lookup(a.V, ix[i], iy[i]) : 0u;
      } else {
#pragma unroll
        for (int i = 0; i < RB_PB; ++i) {
          const uint32_t ri = ((iy[i] >> c.s0) << c.T0) | (ix[i] >> c.s0);
          val[i] = (okm >> i) & 1u ? __ldg(c.root + ri) : 0u;
        }
      }
      uint32_t nodem = 0;
#pragma unroll
      for (int i = 0; i < RB_PB; ++i) nodem |= (val[i] >> 31) << i;
      if (nodem) {
        int s = c.s0;
#pragma unroll 1
        for (int li = 0; li < c.nlev; ++li) {
          const int k = lv.ks[li];
          const uint32_t* __restrict__ nodes = lv.nodes[li];
          s -= k;
          const uint32_t m = (1u << k) - 1u;
#pragma unroll
          for (int i = 0; i < RB_PB; ++i) {
            if (val[i] & RB_VALUE_NODE) {
              const uint32_t slot = (((iy[i] >> s) & m) << k) | ((ix[i] >> s) & m);
              val[i] = __ldg(nodes + (((val[i] & RB_VALUE_PAYLOAD) << (2 * k)) + slot));
            }
          }
        }
      }
      // 3. accumulate: single interior owner inline, every
      //    other owner value (boundary owner, owner list) on the outlined path
#pragma unroll
      for (int i = 0; i < RB_PB; ++i) {
        const uint32_t v = val[i];
        int32_t qv = 0;
        bool fast = true;
        if (ATTR) {
          const float aw = fabsf(w[i]);
          fast = (aw < wmax) & ((aw >= wmin) | (aw == 0.f));
          qv = __float2int_rn(w[i] * sc);
        }
        const uint32_t sv = (v & a.V.code_mask) - 1u;
        if (v != 0u && !(v & RB_VALUE_LIST) && (sv & 1u) == 0u) {
          if (fast) h.add_fast(sv, qv); else h.add_slow(sv, w[i]);
        } else if (v != 0u) {
          add_owners<ATTR>(h, c.pool, v, w[i], qv, fast, a.V.code_mask);
        }
      }
    }
    if (ATTR) {
      __syncthreads();
      for (int q = threadIdx.x; q < R2; q += blockDim.x) {
        acc[q] += ((long long)(int32_t)h.hi[q] << 16) + (long long)h.lo[q];
        h.lo[q] = 0;
        h.hi[q] = 0;
      }
      __syncthreads();
    }
  }
  // remainder points (n not a multiple of the chunk): last CTA, float64 path
  if (blockIdx.x == gridDim.x - 1) {
    for (int64_t i = nchunks * PPC + threadIdx.x; i < a.n; i += blockDim.x) {
      const uint64_t qq = quantize_exact(a.xy, i, XY, c.ox, c.oy, c.side, c.lim, a.first_bad, a.idx_base);
      if (qq == ~0ull) continue;
      const uint32_t qx = (uint32_t)qq, qy = (uint32_t)(qq >> 32);
      const uint32_t v = index_lookup(a.V, qx, qy);
      if (v == 0) continue;
      const float ww = ATTR ? a.attr[i] : 0.f;
      if (!(v & RB_VALUE_LIST) && !(((v & a.V.code_mask) - 1u) & 1u)) h.add_slow((v & a.V.code_mask) - 1u, ww);
      else add_owners<ATTR>(h, c.pool, v, ww, 0, false, a.V.code_mask);
    }
  }
  __syncthreads();
  uint32_t* pc = a.part_cnt + (size_t)blockIdx.x * R2;
  long long* pa = a.part_acc + (size_t)blockIdx.x * R2;
  double* ps = a.part_sum + (size_t)blockIdx.x * R2;
  for (int q = threadIdx.x; q < R2; q += blockDim.x) {
    pc[q] = cnt[q];
    if (ATTR) { pa[q] = acc[q]; ps[q] = slow[q]; }
  }
}

// ---------------------------------------------------------------------------
// TMA-staged point pass (the production path).
//
// Warp 0 is the producer: one elected lane streams fixed-size tiles of the
// coordinate and attribute columns into a 4-stage shared-memory ring with
// cp.async.bulk (1-D TMA, L2 evict-first policy, completion on an mbarrier).
// Warps 1..8 consume: each thread takes 4 points of the tile from shared
// memory, quantises them, walks the radix table and accumulates.  DRAM
// latency is absorbed by the ring; no registers are tied up by in-flight
// loads, so the consumers only wait on the L2-resident index.
// ---------------------------------------------------------------------------
#ifndef RB_TP
#define RB_TP 1024     // points per tile
#endif
#ifndef RB_NST
#define RB_NST 3       // ring stages
#endif
#ifndef RB_CONS
#define RB_CONS 256    // consumer threads
#endif
#define RB_MINB_TMA (RB_CONS >= 512 ? 1 : 2)
#define RB_PPT (RB_TP / RB_CONS)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// warp-uniform wait: every lane polls and the warp leaves together (a per-lane
// spin lets lanes leave at different times, and ITS keeps such a warp split)
__device__ __forceinline__ uint32_t mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 100000;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok;
}
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
  while (!__all_sync(0xffffffffu, mbar_try(bar, parity))) {
  }
}
// the same on a precomputed shared-memory address (keeps the address computation out of the loop)
__device__ __forceinline__ uint32_t mbar_try_a(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 100000;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok;
}
__device__ __forceinline__ void mbar_wait_warp_a(uint32_t addr, uint32_t parity) {
  while (!__all_sync(0xffffffffu, mbar_try_a(addr, parity))) {
  }
}
__device__ __forceinline__ void mbar_arrive_a(uint32_t addr) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

template <int XY, bool ATTR, bool GH = false>
__global__ void __launch_bounds__(RB_CONS + 32, RB_MINB_TMA) k_point_pass_tma(PassArgs a) {
  constexpr int PB_BYTES = XY == 0 ? 16 : 8;
  constexpr uint32_t XY_TILE = RB_TP * PB_BYTES;
  constexpr uint32_t AT_TILE = ATTR ? RB_TP * 4 : 0;
  constexpr uint32_t STAGE = XY_TILE + AT_TILE;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ LevelDesc lv;
  __shared__ __align__(8) uint64_t full_bar[RB_NST], empty_bar[RB_NST];
  const int R2 = a.R2;
  // layout: [ring][h3: R2*(ATTR?3:1) u32][acc: R2 i64][slow: R2 f64][summary u16]
  // smem mode: all R2 bins [h3 | acc | slow]; global mode: the n_hot hot alpha bins only
  const int NB = GH ? a.n_hot : R2;
  unsigned char* hist = smem + (size_t)RB_NST * STAGE;
  uint32_t* h3 = (uint32_t*)hist;
  const size_t h3_bytes = (((size_t)NB * (ATTR ? 12 : 4)) + 15) & ~(size_t)15;
  long long* acc = (long long*)(hist + h3_bytes);
  double* slow = (double*)(hist + h3_bytes + (ATTR && !GH ? (size_t)R2 * 8 : 0));
  uint16_t* summ = (uint16_t*)(hist + h3_bytes + (ATTR && !GH ? (size_t)R2 * 16 : 0));
  IHist<ATTR> h{h3, slow, GH ? a.gcnt : nullptr, GH ? a.gsum : nullptr};
  const int tid = threadIdx.x;
  const int S = a.V.S;
  for (int q = tid; q < NB * (ATTR ? 3 : 1); q += blockDim.x) h3[q] = 0;
  if (ATTR && !GH)
    for (int q = tid; q < R2; q += blockDim.x) { acc[q] = 0; slow[q] = 0.0; }
  if (ATTR && GH)
    for (int q = tid; q < NB; q += blockDim.x) a.part_acc[(size_t)blockIdx.x * NB + q] = 0;
  if (S >= 0) {
    const int nsum = 1 << (2 * S);
    const uint4* src = (const uint4*)a.V.summary;
    uint4* dst = (uint4*)summ;
    for (int q = tid; q < (nsum >> 3); q += blockDim.x) dst[q] = __ldg(src + q);
    for (int q = (nsum & ~7) + tid; q < nsum; q += blockDim.x) summ[q] = a.V.summary[q];
  }
  if (tid < RB_MAX_NODE_LEVELS) {
    lv.nodes[tid] = a.V.nodes[tid];
    lv.ks[tid] = a.V.ks[tid];
  }
  if (tid == 0) {
    for (int s = 0; s < RB_NST; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], RB_CONS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nmain = a.n & ~(int64_t)3;  // bulk copies need 16-byte granules
  const int64_t ntiles = (nmain + RB_TP - 1) / RB_TP;
  const int64_t G = gridDim.x;

  if (tid < 32) {
    // ------------------------------------------------------------ producer
    if (tid == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int st = 0;
      uint32_t ph = 0;
      int64_t k = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += G, ++k) {
        if (k >= RB_NST) mbar_wait(&empty_bar[st], ph ^ 1u);
        const int64_t p0 = t * RB_TP;
        const uint32_t m = (uint32_t)(p0 + RB_TP <= nmain ? RB_TP : nmain - p0);
        unsigned char* dst = smem + (size_t)st * STAGE;
        mbar_expect_tx(&full_bar[st], m * PB_BYTES + (ATTR ? m * 4 : 0));
        bulk_g2s(dst, (const char*)a.xy + p0 * PB_BYTES, m * PB_BYTES, &full_bar[st], pol);
        if (ATTR) bulk_g2s(dst + XY_TILE, a.attr + p0, m * 4, &full_bar[st], pol);
        if (++st == RB_NST) { st = 0; ph ^= 1u; }
      }
    }
    return;
  }
  // -------------------------------------------------------------- consumers
  const int ct = tid - 32;
  float sc = 1.f, wmax = 0.f, wmin = 0.f;
  if (ATTR) {
    const int Sx = *a.scale_exp;
    sc = __int_as_float((Sx + 127) << 23);
    wmax = __int_as_float((30 - Sx + 127) << 23);
    wmin = __int_as_float((20 - Sx + 127) << 23);
  }
  const double ox = a.ox, oy = a.oy, inv_side = a.inv_side;
  const uint32_t* __restrict__ root = a.V.root;
  const uint32_t* __restrict__ pool = a.V.pool;
  const int T0 = a.V.T0, s0 = a.V.L - a.V.T0, nlev = a.V.nlev;
  const int sS = a.V.L - (S >= 0 ? S : 0);
  const uint32_t lim_u = a.V.L >= 32 ? 0xffffffffu : (1u << a.V.L);
  const uint32_t hmax = (uint32_t)(((1ull << a.V.L) - 1ull) >> 12);
  int st = 0;
  uint32_t ph = 0;
  int ep = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += G) {
    mbar_wait(&full_bar[st], ph);
    const int64_t p0 = t * RB_TP;
    const int m = (int)(p0 + RB_TP <= nmain ? RB_TP : nmain - p0);
    const unsigned char* tile = smem + (size_t)st * STAGE;
    uint32_t ix[RB_PPT], iy[RB_PPT], val[RB_PPT];
    float w[RB_PPT];
    int32_t qv[RB_PPT];
    uint32_t okm = 0, slowm = 0, fastm = 0;
    // A. quantise (t = RN(RN(RN(v - o) * inv_side) + 2^32), see rb_point_pass.cu header).
    //    Every value read from the tile is consumed here, before the slot is
    //    released to the producer (a pending LDS must not race the refill).
#pragma unroll
    for (int j = 0; j < RB_PPT; ++j) {
      const int pi = ct + j * RB_CONS;
      const bool in = pi < m;
      double x, y;
      if (XY == 0) {
        const double2 v2 = ((const double2*)tile)[in ? pi : 0];
        x = v2.x; y = v2.y;
      } else {
        const float2 v2 = ((const float2*)tile)[in ? pi : 0];
        x = (double)v2.x; y = (double)v2.y;
      }
      w[j] = ATTR ? ((const float*)(tile + XY_TILE))[in ? pi : 0] : 0.f;
      const double tx = __dadd_rn(__dmul_rn(__dsub_rn(x, ox), inv_side), 4294967296.0);
      const double ty = __dadd_rn(__dmul_rn(__dsub_rn(y, oy), inv_side), 4294967296.0);
      const uint32_t lx = (uint32_t)__double2loint(tx), hx = (uint32_t)__double2hiint(tx);
      const uint32_t ly = (uint32_t)__double2loint(ty), hy = (uint32_t)__double2hiint(ty);
      ix[j] = __funnelshift_r(lx, hx, 20);
      iy[j] = __funnelshift_r(ly, hy, 20);
      const bool good = ((hx - 0x41F00000u) <= hmax) & ((hy - 0x41F00000u) <= hmax) &
                        (((lx + 2u) & 0xffffcu) != 0u) & (((ly + 2u) & 0xffffcu) != 0u) & (ix[j] < lim_u) &
                        (iy[j] < lim_u);
      okm |= (in & good) ? (1u << j) : 0u;
      slowm |= (in & !good) ? (1u << j) : 0u;
      qv[j] = 0;
      if (ATTR) {
        const float aw = fabsf(w[j]);
        fastm |= ((aw < wmax) & ((aw >= wmin) | (aw == 0.f))) ? (1u << j) : 0u;
        qv[j] = __float2int_rn(w[j] * sc);
      }
    }
    // WAR hazard across proxies: an mbarrier arrive does not wait for LDS
    // still in flight, so order this warp's generic-proxy reads of the slot
    // before the async-proxy (bulk copy) refill that the arrive enables.
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if ((ct & 31) == 0) mbar_arrive(&empty_bar[st]);  // slot may be refilled
    if (++st == RB_NST) { st = 0; ph ^= 1u; }
    if (slowm) {  // rare: exact division + domain check
#pragma unroll
      for (int j = 0; j < RB_PPT; ++j) {
        if (slowm & (1u << j)) {
          const uint64_t qq = quantize_exact(a.xy, p0 + ct + j * RB_CONS, XY, ox, oy, a.side, a.lim, a.first_bad,
                                             a.idx_base);
          if (qq != ~0ull) { ix[j] = (uint32_t)qq; iy[j] = (uint32_t)(qq >> 32); okm |= 1u << j; }
        }
      }
    }
    // B. summary in shared memory, then the L2-resident radix table
#pragma unroll
    for (int j = 0; j < RB_PPT; ++j) {
      const bool okj = (okm >> j) & 1u;
      uint32_t sv = 0xffffu;
      if (S >= 0) sv = okj ? (uint32_t)summ[((iy[j] >> sS) << S) | (ix[j] >> sS)] : 0u;
      const uint32_t* rp = root + (((iy[j] >> s0) << T0) | (ix[j] >> s0));
      val[j] = ldg_pred(rp, okj & (sv == 0xffffu), okj ? sv : 0u);
    }
    // C. node levels (ACT descent), warp-uniform skip
    uint32_t anyn = 0;
#pragma unroll
    for (int j = 0; j < RB_PPT; ++j) anyn |= val[j];
    if (__any_sync(0xffffffffu, (anyn & RB_VALUE_NODE) != 0u)) {
      int s = s0;
#pragma unroll 1
      for (int li = 0; li < nlev; ++li) {
        const int kk = lv.ks[li];
        const uint32_t* __restrict__ nodes = lv.nodes[li];
        s -= kk;
        const uint32_t msk = (1u << kk) - 1u;
#pragma unroll
        for (int j = 0; j < RB_PPT; ++j) {
          const bool nd = (val[j] & RB_VALUE_NODE) != 0u;
          const uint32_t slot = (((iy[j] >> s) & msk) << kk) | ((ix[j] >> s) & msk);
          const uint32_t* np = nodes + (((val[j] & RB_VALUE_PAYLOAD) << (2 * kk)) + slot);
          val[j] = ldg_pred(np, nd, val[j]);
        }
      }
    }
    // D. common case inline: one interior owner and an in-window attribute
    uint32_t rarem = 0;
#pragma unroll
    for (int j = 0; j < RB_PPT; ++j) {
      const uint32_t v = val[j];
      const bool fast = !ATTR || ((fastm >> j) & 1u);
      // single interior owner: code = v & CODE_MASK (= 2*region + 1), hot slot in bits 18..29
      const uint32_t sv = (v & a.V.code_mask) - 1u;
      const bool common = (v != 0u) & ((v & RB_VALUE_LIST) == 0u) & ((sv & 1u) == 0u) & fast;
      if (common) h.add(sv, v >> a.V.hot_shift, w[j], qv[j], true);
      rarem |= (!common & (v != 0u)) ? (1u << j) : 0u;
    }
    // E. boundary owners, owner lists, out-of-window attributes
    if (rarem) {
#pragma unroll
      for (int j = 0; j < RB_PPT; ++j) {
        if (rarem & (1u << j)) {
          const bool fast = !ATTR || ((fastm >> j) & 1u);
          add_owners_i<ATTR>(h, pool, val[j], w[j], qv[j], fast, a.V.code_mask, a.V.hot_shift);
        }
      }
    }
    if (ATTR && ++ep == 65536 / RB_TP) {  // fold the 16-bit fixed-point halves every 65536 points
      ep = 0;
      asm volatile("bar.sync 1, %0;" ::"r"(RB_CONS) : "memory");
      for (int q = ct; q < NB; q += RB_CONS) {
        const long long f = ((long long)(int32_t)h3[3 * q + 2] << 16) + (long long)h3[3 * q + 1];
        if (GH) a.part_acc[(size_t)blockIdx.x * NB + q] += f; else acc[q] += f;
        h3[3 * q + 1] = 0;
        h3[3 * q + 2] = 0;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(RB_CONS) : "memory");
    }
  }
  // up to 3 trailing points (n not a multiple of 4): CTA 0, float64 path
  if (blockIdx.x == 0 && ct < (int)(a.n - nmain)) {
    const int64_t i = nmain + ct;
    const uint64_t qq = quantize_exact(a.xy, i, XY, ox, oy, a.side, a.lim, a.first_bad, a.idx_base);
    if (qq != ~0ull) {
      const uint32_t v = index_lookup(a.V, (uint32_t)qq, (uint32_t)(qq >> 32));
      if (v != 0u) add_owners_i<ATTR>(h, pool, v, ATTR ? a.attr[i] : 0.f, 0, false, a.V.code_mask, a.V.hot_shift);
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(RB_CONS) : "memory");
  if (GH) {  // flush the hot bins into the global per-region outputs
    const int Sx = ATTR ? *a.scale_exp : 0;
    for (int q = ct; q < NB; q += RB_CONS) {
      const uint32_t c = h3[ATTR ? 3 * q : q];
      if (!c) continue;
      const int32_t r = a.hot_region[q];
      atomicAdd(&a.gcnt[2 * r], (unsigned long long)c);
      if (ATTR) {
        const long long f = a.part_acc[(size_t)blockIdx.x * NB + q] + ((long long)(int32_t)h3[3 * q + 2] << 16) +
                            (long long)h3[3 * q + 1];
        atomicAdd(&a.gsum[2 * r], ldexp((double)f, -Sx));
      }
    }
    return;
  }
  uint32_t* pc = a.part_cnt + (size_t)blockIdx.x * R2;
  long long* pa = a.part_acc + (size_t)blockIdx.x * R2;
  double* ps = a.part_sum + (size_t)blockIdx.x * R2;
  for (int q = ct; q < R2; q += RB_CONS) {
    pc[q] = h3[ATTR ? 3 * q : q];
    if (ATTR) {
      pa[q] = acc[q] + ((long long)(int32_t)h3[3 * q + 2] << 16) + (long long)h3[3 * q + 1];
      ps[q] = slow[q];
    }
  }
}

// ---------------------------------------------------------------------------
// The TMA ring kernel (the production path for L <= 20 and a shared-memory
// histogram).
//
// One CTA per SM: a producer warp whose lane 0 streams CTA tiles (NW * PPT *
// 32 points of coordinates + attribute) with cp.async.bulk into an NST-stage
// shared-memory ring (full / empty mbarriers), and NW consumer warps that run
// a software pipeline over the tiles (below).  A stage is refilled once all
// consumer warps have released it.
//
// Quantisation, bit-identical to floor(RN((v - o) / side)):
// t = RN(RN(RN(v - o) * RN(1/side)) + 2^20).  For 0 <= q < 2^20 the high word
// of t is 0x41300000 + floor(q) and the low word is q's fraction in units of
// 2^-32; the product differs from the quotient by < 2^-31 (L <= 20), so unless
// the fraction lies within 2^-29 of an integer floor(q) is exact.  Range:
// (hx - 0x41300000) | (hy - 0x41300000) < 2^L covers q < 0, q >= 2^L, NaN and
// infinities.  Points failing either test take the exact division.
//
// Lookup: level-S summary in shared memory (single owner of a whole summary
// cell), else the L2-resident root table, then node levels (ACT descent,
// SPEC.md:285-288).  Accumulation: a single owner with an
// in-window attribute -> three unconditional u32 shared REDs (count, fixed-
// point low 16 bits, signed high part) into its (region << 1) | boundary bin;
// owner lists and out-of-window attributes through the per-warp rare queue.
// ---------------------------------------------------------------------------
// shared-memory REDs on 32-bit shared addresses (the generic atomicAdd on a
// pointer the compiler cannot prove shared becomes a generic ATOM)
__device__ __forceinline__ void reds(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// Rare path of the ring kernel: every owner of value v (owner list) or an
// attribute outside the fixed-point window.  bins: shared address of bin 0
// (stride 12 bytes with an attribute, 4 without).  The ring kernel's bins are
// (region << 1) | boundary: interior-leaf and boundary-leaf points of a region
// (k_reduce_fixed turns them into alpha = both, beta = boundary), so every
// owner entry adds to exactly one bin.
template <bool ATTR>
__device__ __forceinline__ void add_owners_w(uint32_t bins, double* slow, const uint32_t* __restrict__ pool, uint32_t v,
                                          float w, int32_t qv, bool fast, uint32_t cm) {
  uint32_t n = 1, e = v;
  const uint32_t* Lp = nullptr;
  if (v & RB_VALUE_LIST) {
    Lp = pool + (v & RB_VALUE_PAYLOAD);
    n = __ldg(Lp) & ~RB_POOL_COUNT_FLAG;
  } else {
    e = (v & cm) - 1u;  // (region << 1) | boundary
  }
#pragma unroll 1
  for (uint32_t i = 0; i < n; ++i) {
    if (Lp) e = __ldg(Lp + 1 + i) & cm;
    const uint32_t ad = bins + e * (ATTR ? 12u : 4u);
    reds(ad, 1u);
    if (ATTR) {
      if (fast) { reds(ad + 4, (uint32_t)qv & 0xffffu); reds(ad + 8, (uint32_t)(qv >> 16)); }
      else atomicAdd(&slow[e], (double)w);
    }
  }
}

// LAY: 0 = radix table (RB_LAYOUT_TRIE / DENSE), 1 = sorted keys (RB_LAYOUT_KEYS), 2 = palette blocks (RB_LAYOUT_PACKED)
template <int XY, bool ATTR, int NW, int PPT, int NST, int LAY = 0>
__global__ void __launch_bounds__(NW * 32 + 32, NW <= 8 ? 2 : 1) k_point_pass_ring(PassArgs a) {
  constexpr bool KEYS = LAY == 1, PK = LAY == 2;
  constexpr int PB = XY == 0 ? 16 : 8;
  constexpr int WT = PPT * 32;  // points per consumer warp per tile
  constexpr int TP = NW * WT;   // points per CTA tile
  constexpr uint32_t XYB = TP * PB, ATB = ATTR ? TP * 4 : 0, STAGE = XYB + ATB;
  constexpr uint32_t BS = ATTR ? 12u : 4u;  // bytes per shared bin
  // The histogram has C copies (lane & (C-1) picks one) so lanes of a warp that hit the same hot
  // region add to different words in different banks: same-address REDs with distinct values
  // serialise, and with clustered points a warp often holds several points of one region.
  // Drain period: every consumer warp drains ALL bins of all copies after each FOLD of its tiles;
  // between two drains of a copy-bin each warp adds <= FOLD * WT / C points to it, <= 63488 + 3 in
  // total, so the low-half sums stay < 2^32 and the signed high-half sums within +-2^30 (|qv| < 2^30).
  const int C = a.hcopies, P = a.hstride;
  // (62000 leaves room for the <= 63 points a warp's rare queue carries across a drain)
  int FOLD = C * (62000 / (NW * WT) > 0 ? 62000 / (NW * WT) : 1);
  if (a.fold > 0 && a.fold < FOLD) FOLD = a.fold;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ LevelDesc lv;
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  const int R2 = a.R2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;  // warp NW is the producer
  // layout: [NST stages][per-warp rare queues: NW x 64 x 8 B][32 dummy bins][C histogram copies of
  // P words][slow f64: R2][summary u16]
  uint2* rq = (uint2*)(smem + (size_t)NST * STAGE) + (size_t)(warp < NW ? warp : 0) * 64;
  unsigned char* dummy = smem + (size_t)NST * STAGE + NW * 64 * 8;
  uint32_t* h3 = (uint32_t*)(dummy + 32 * BS);
  const size_t h3b = (((size_t)C * P * 4) + 15) & ~(size_t)15;
  double* slow = (double*)((unsigned char*)h3 + h3b);
  uint16_t* summ = (uint16_t*)((unsigned char*)h3 + h3b + (ATTR ? (size_t)R2 * 8 : 0));
  long long* prow = a.part_acc + (size_t)blockIdx.x * R2;  // this CTA's fixed-point sums (global, REDG.64)
  const int S = a.V.S >= 0 ? a.V.S : 0;
  constexpr int NT = NW * 32 + 32;
  for (int q = tid; q < C * P; q += NT) h3[q] = 0;
  if (ATTR)
    for (int q = tid; q < R2; q += NT) { slow[q] = 0.0; prow[q] = 0; }
  if (a.V.S >= 0) {
    const int nsum = 1 << (2 * S);
    const uint4* src = (const uint4*)a.V.summary;
    for (int q = tid; q < (nsum >> 3); q += NT) ((uint4*)summ)[q] = __ldg(src + q);
    for (int q = (nsum & ~7) + tid; q < nsum; q += NT) summ[q] = a.V.summary[q];
  } else if (tid == 0) {
    summ[0] = 0xffffu;  // no summary: every point consults the index
  }
  if (tid < RB_MAX_NODE_LEVELS) {
    lv.nodes[tid] = a.V.nodes[tid];
    lv.ks[tid] = a.V.ks[tid];
  }
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t nmain = a.n & ~(int64_t)3;  // bulk copies move 16-byte granules
  const int64_t ntiles = (nmain + TP - 1) / TP;
  const int64_t G = gridDim.x;
  if (warp == NW) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int st = 0;
      uint32_t ph = 0;
      int64_t k = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += G, ++k) {
        if (k >= NST) mbar_wait(&empty[st], ph ^ 1u);
        const int64_t p0 = t * TP;
        const uint32_t m = (uint32_t)(p0 + TP <= nmain ? TP : nmain - p0);
        unsigned char* dst = smem + (size_t)st * STAGE;
        mbar_expect_tx(&full[st], m * (PB + (ATTR ? 4 : 0)));
        bulk_g2s(dst, (const char*)a.xy + p0 * PB, m * PB, &full[st], pol);
        if (ATTR) bulk_g2s(dst + XYB, a.attr + p0, m * 4, &full[st], pol);
        if (++st == NST) { st = 0; ph ^= 1u; }
      }
    }
    return;
  }
  // -------------------------------------------------------------- consumers
  float sc = 1.f;
  uint32_t wminb = 0, wspan = 0;
  if (ATTR) {
    // binary scale of the SUM fixed point from the same strided 4096-value sample in every CTA
    // (deterministic, identical to k_attr_scale; its loads overlap the producer's first tiles)
    __shared__ float smax[NW];
    float mx = 0.f;
    const int64_t stride = a.n / 4096 > 0 ? a.n / 4096 : 1;
    constexpr int NSAMP = (4096 + NW * 32 - 1) / (NW * 32);
    float sv[NSAMP];
#pragma unroll
    for (int j = 0; j < NSAMP; ++j) {  // all loads in flight at once (one DRAM latency, not NSAMP)
      const int64_t q = tid + (int64_t)j * NW * 32;
      sv[j] = (q < 4096 && q * stride < a.n) ? __ldg(a.attr + q * stride) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < NSAMP; ++j) {
      const float v = fabsf(sv[j]);
      if (isfinite(v)) mx = fmaxf(mx, v);
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) smax[warp] = mx;
    asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
    mx = 0.f;
    for (int w2 = 0; w2 < NW; ++w2) mx = fmaxf(mx, smax[w2]);
    int Sx = 0;
    if (mx > 0.f) {
      int e = 0;
      frexpf(mx, &e);  // mx < 2^e
      Sx = 29 - e;     // fast window [2^(e-9), 2^(e+1))
    }
    Sx = Sx < -96 ? -96 : (Sx > 126 ? 126 : Sx);
    if (blockIdx.x == 0 && tid == 0) *a.scale_exp = Sx;  // for k_reduce_fixed
    sc = __int_as_float((Sx + 127) << 23);
    wminb = (uint32_t)((20 - Sx + 127) << 23);  // |w| in [2^(20-S), 2^(30-S)): exact 30-bit fixed point
    wspan = (uint32_t)((30 - Sx + 127) << 23) - wminb;
  }
  const double ox = a.ox, oy = a.oy, inv_side = a.inv_side;
  const uint32_t* __restrict__ root = a.V.root;
  const uint32_t* __restrict__ pool = a.V.pool;
  const uint32_t* __restrict__ nodes0 = a.V.nodes[0];
  const int L = a.V.L, T0 = a.V.T0, s0 = L - T0, nlev = a.V.nlev, sS = L - S;
  const uint32_t hibits = ~((1u << L) - 1u);
  const uint32_t m0 = (1u << s0) - 1u;
  // the single node level is the leaf level (k = L - T0), addressable with 32-bit offsets
  const bool onelevel = nlev == 1 && a.V.ks[0] == s0 && a.V.nodes0_len < (int64_t(1) << 32);
  const uint32_t bins = smem_u32(h3) + (uint32_t)((lane & (C - 1)) * P) * 4u;  // this lane's copy
  const uint32_t h3s = bins - BS;  // single owner v: code (v & CODE_MASK) = ((region << 1) | boundary) + 1 -> bin code-1
  const uint32_t dms = smem_u32(dummy) + lane * BS;
  // ---- software pipeline over this CTA's tiles (k = 0, 1, ...); iteration k runs
  //   C(k-2): accumulate the owner values nv[] loaded during iteration k-1
  //   B(k-1): node levels of tile k-1 from its root values rv[] (loaded during iteration k-1) -> nv[]
  //   A(k)  : tile k: ring -> quantise -> summary -> root loads -> rv[]
  // Each load is consumed one iteration after it is issued, and a load's destination register is
  // only read by the consuming stage (no register copy waits on a load in flight).
  int qh = 0, qn = 0;  // this warp's rare queue: head, count (warp-uniform)
  auto rare_flush = [&](int nitems) {
    if (lane < nitems) {
      const uint2 it = rq[(qh + lane) & 63];
      const float ww = __uint_as_float(it.y);
      const bool fast = !ATTR || (((it.y & 0x7fffffffu) - wminb) < wspan);
      add_owners_w<ATTR>(bins, slow, pool, it.x, ww, ATTR ? __float2int_rn(ww * sc) : 0, fast, a.V.code_mask);
    }
    __syncwarp();
  };
  uint32_t rv[PPT], bx[PPT], by[PPT], nv[PPT];
  uint32_t hv[PPT];  // KEYS: radix bucket end (rv = bucket start, ~0u = no lookup); PK: leaf slot in its block
  uint4 pb[PPT];     // PK: the palette blocks loaded in B(k-1)
  const uint4* __restrict__ pblk = a.V.pblk;
  const uint32_t* __restrict__ pwide = a.V.pwide;
  const int pd = a.V.pd;
  float w1[PPT], w2[PPT];
#pragma unroll
  for (int j = 0; j < PPT; ++j) { rv[j] = bx[j] = by[j] = nv[j] = hv[j] = 0u; w1[j] = w2[j] = 0.f; pb[j] = make_uint4(0u, 0u, 0u, 0u); }
  int st = 0;
  uint32_t ph = 0;
  int dk = 0;
  const int64_t K = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / G + 1 : 0;
  for (int64_t k = 0; k < K + 2; ++k) {
    // ------------------------------------------------------------ C(k-2)
    if (k >= 2) {
      if constexpr (PK) {  // palette select; escape blocks (> 3 owner values) take one more load
        bool esc = false;
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          nv[j] = packed_pick(pb[j], hv[j]);
          esc |= (int32_t)nv[j] < 0;
        }
        if (__any_sync(0xffffffffu, esc)) {
#pragma unroll
          for (int j = 0; j < PPT; ++j)
            nv[j] = ldg_pred(pwide + ((size_t)(nv[j] & RB_VALUE_PAYLOAD) << 4) + hv[j], (int32_t)nv[j] < 0, nv[j]);
        }
      }
      bool anyrare = false;
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const uint32_t v = nv[j];
        int32_t qv = 0;
        bool fast = true;
        if (ATTR) {
          qv = __float2int_rn(w2[j] * sc);
          fast = ((__float_as_uint(w2[j]) & 0x7fffffffu) - wminb) < wspan;
        }
        // single owner (no list), interior or boundary leaf, with an in-window attribute
        // (v == 0, no owner, lands on bin -1: the dummy slot before copy 0, or >= 3 pad words of the copy before)
        const bool common = ((v & RB_VALUE_LIST) == 0u) & fast;
        // unconditional REDs (a predicated RED becomes a branch): off-path points hit this lane's dummy bin
        const uint32_t ad = common ? h3s + (v & a.V.code_mask) * BS : dms;
        reds(ad, 1u);
        if (ATTR) {
          reds(ad + 4, (uint32_t)qv & 0xffffu);
          reds(ad + 8, (uint32_t)(qv >> 16));
        }
        anyrare |= !common & (v != 0u);
      }
      // boundary owners, owner lists, out-of-window attributes: queue them per warp and process
      // 32 at a time, one per lane (divergent one-lane processing cost a quarter of the pass)
      if (!(a.ablate & 1) && __any_sync(0xffffffffu, anyrare)) {
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          const uint32_t v = nv[j];
          const bool fast = !ATTR || (((__float_as_uint(w2[j]) & 0x7fffffffu) - wminb) < wspan);
          const bool rare = (((v & RB_VALUE_LIST) != 0u) | !fast) & (v != 0u);
          const uint32_t mk = __ballot_sync(0xffffffffu, rare);
          if (mk) {
            if (rare) rq[(qh + qn + __popc(mk & ((1u << lane) - 1u))) & 63] = make_uint2(v, __float_as_uint(w2[j]));
            qn += __popc(mk);
            if (qn >= 32) {
              __syncwarp();
              rare_flush(32);
              qh = (qh + 32) & 63;
              qn -= 32;
            }
          }
        }
      }
      if (ATTR && ++dk == FOLD) {  // drain the 16-bit fixed-point halves into this CTA's global row
        dk = 0;
        __syncwarp();
        for (int q = lane; q < R2; q += 32) {
          long long f = 0;
          for (int c = 0; c < C; ++c) {
            const uint32_t lo = atomicExch(&h3[c * P + 3 * q + 1], 0u);
            const uint32_t hi = atomicExch(&h3[c * P + 3 * q + 2], 0u);
            f += ((long long)(int32_t)hi << 16) + (long long)lo;
          }
          if (f) atomicAdd((unsigned long long*)&prow[q], (unsigned long long)f);
        }
      }
    }
    // ------------------------------------------------------------ B(k-1)
    if constexpr (PK) {  // the 16-byte palette block of each point in a mixed root cell
      if (k >= 1 && k <= K) {
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          w2[j] = w1[j];
          hv[j] = packed_slot(bx[j], by[j]);
          pb[j] = ldg4_pred(pblk + packed_block(rv[j] & RB_VALUE_PAYLOAD, bx[j], by[j], pd), (int32_t)rv[j] < 0, rv[j]);
        }
      }
    } else
    if constexpr (KEYS) {  // the bucket's cell records for the bucket read in A(k-1)
      if (k >= 1 && k <= K) {
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          w2[j] = w1[j];
          nv[j] = hv[j] == ~0u ? rv[j] : keys_resolve(a.V, leaf_z(bx[j], by[j]), (int64_t)rv[j], (int64_t)hv[j]);
        }
      }
    } else
    if (k >= 1 && k <= K) {
#pragma unroll
      for (int j = 0; j < PPT; ++j) w2[j] = w1[j];
      uint32_t anyn = 0;
#pragma unroll
      for (int j = 0; j < PPT; ++j) anyn |= rv[j];
      if (__any_sync(0xffffffffu, (int32_t)anyn < 0)) {  // RB_VALUE_NODE = bit 31
        if (onelevel) {  // one node level = the leaf cells of a root cell, row-major (32-bit offsets)
#pragma unroll
          for (int j = 0; j < PPT; ++j) {
            const uint32_t off = ((rv[j] & RB_VALUE_PAYLOAD) << (2 * s0)) | ((by[j] & m0) << s0) | (bx[j] & m0);
            nv[j] = ldg_pred(nodes0 + off, (int32_t)rv[j] < 0, rv[j]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < PPT; ++j) nv[j] = rv[j];
          int s = s0;
#pragma unroll 1
          for (int li = 0; li < nlev; ++li) {
            const int kk = lv.ks[li];
            const uint32_t* __restrict__ nodes = lv.nodes[li];
            s -= kk;
            const uint32_t msk = (1u << kk) - 1u;
#pragma unroll
            for (int j = 0; j < PPT; ++j) {
              const uint32_t slot = (((by[j] >> s) & msk) << kk) | ((bx[j] >> s) & msk);
              const uint32_t* np = nodes + (((size_t)(nv[j] & RB_VALUE_PAYLOAD) << (2 * kk)) + slot);
              nv[j] = ldg_pred(np, (int32_t)nv[j] < 0, nv[j]);
            }
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < PPT; ++j) nv[j] = rv[j];
      }
    }
    // ------------------------------------------------------------ A(k)
    if (k < K) {
      const int64_t t = blockIdx.x + k * G;
      mbar_wait_warp(&full[st], ph);
      const unsigned char* tile = smem + (size_t)st * STAGE;
      double x[PPT], y[PPT];
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const int pi = warp * WT + lane + 32 * j;
        if (XY == 0) {
          const double2 v2 = ((const double2*)tile)[pi];
          x[j] = v2.x; y[j] = v2.y;
        } else {
          const float2 v2 = ((const float2*)tile)[pi];
          x[j] = (double)v2.x; y[j] = (double)v2.y;
        }
        w1[j] = ATTR ? ((const float*)(tile + XYB))[pi] : 0.f;
      }
      // the stage's generic-proxy reads precede the async-proxy refill that the arrive enables
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == NST) { st = 0; ph ^= 1u; }
      // quantise: t = RN((v - o) * RN(1/side) + 2^20) (one rounding); high word = 0x41300000 +
      // floor(q) for 0 <= q < 2^20, low word = fraction * 2^32; |t - 2^20 - RN(d/side)| < 2^-31
      bool anybad = false;
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const double tx = __fma_rn(__dsub_rn(x[j], ox), inv_side, 1048576.0);
        const double ty = __fma_rn(__dsub_rn(y[j], oy), inv_side, 1048576.0);
        bx[j] = (uint32_t)__double2hiint(tx) - 0x41300000u;
        by[j] = (uint32_t)__double2hiint(ty) - 0x41300000u;
        const uint32_t fx = (uint32_t)__double2loint(tx) + 8u, fy = (uint32_t)__double2loint(ty) + 8u;
        anybad |= ((bx[j] | by[j]) & hibits) != 0u;  // q < 0, q >= 2^L, NaN, inf
        anybad |= (fx < 16u) | (fy < 16u);             // within 2^-29 of a cell edge
      }
      const int64_t p0 = t * TP + warp * WT;  // this warp's slice of the tile
      uint32_t killm = 0;
      if (__any_sync(0xffffffffu, anybad) || p0 + WT > nmain) {  // rare: exact division, domain errors, partial tile
        const int64_t mm = nmain - p0;
        const int m = (int)(mm >= WT ? WT : (mm > 0 ? mm : 0));
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          const double tx = __fma_rn(__dsub_rn(x[j], ox), inv_side, 1048576.0);
          const double ty = __fma_rn(__dsub_rn(y[j], oy), inv_side, 1048576.0);
          const uint32_t fx = (uint32_t)__double2loint(tx) + 8u, fy = (uint32_t)__double2loint(ty) + 8u;
          const bool bad = (((bx[j] | by[j]) & hibits) != 0u) | (fx < 16u) | (fy < 16u);
          if (lane + 32 * j >= m) {
            bx[j] = 0; by[j] = 0; killm |= 1u << j;
          } else if (bad) {
            const uint64_t qq =
                quantize_exact(a.xy, p0 + lane + 32 * j, XY, ox, oy, a.side, a.lim, a.first_bad, a.idx_base);
            if (qq != ~0ull) { bx[j] = (uint32_t)qq; by[j] = (uint32_t)(qq >> 32); }
            else { bx[j] = 0; by[j] = 0; killm |= 1u << j; }
          }
        }
      }
      if constexpr (KEYS) {  // RB_LAYOUT_KEYS: summary, else the radix bucket now and its cell records in B(k)
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          uint32_t sv = summ[((by[j] >> sS) << S) | (bx[j] >> sS)];
          if ((killm >> j) & 1u) sv = 0u;
          const uint64_t p = leaf_z(bx[j], by[j]) >> a.V.kshift;
          rv[j] = ldg_pred(a.V.ktab + p, sv == 0xffffu, sv);     // bucket start, or the answered value
          hv[j] = ldg_pred(a.V.ktab + p + 1, sv == 0xffffu, ~0u);  // bucket end, or ~0u: answered
        }
      } else {
      // summary (shared memory), else the radix table (L2)
      uint32_t sv[PPT];
#pragma unroll
      for (int j = 0; j < PPT; ++j) sv[j] = summ[((by[j] >> sS) << S) | (bx[j] >> sS)];
      if (killm) {
#pragma unroll
        for (int j = 0; j < PPT; ++j)
          if (killm & (1u << j)) sv[j] = 0u;  // no owner, no lookup
      }
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const uint32_t* rp = root + (((by[j] >> s0) << T0) | (bx[j] >> s0));
        rv[j] = ldg_pred(rp, sv[j] == 0xffffu, sv[j]);
      }
      }
    }
  }
  __syncwarp();
  if (qn) rare_flush(qn);
  // up to 3 trailing points (n not a multiple of 4): CTA 0, float64 path
  if (blockIdx.x == 0 && tid < (int)(a.n - nmain)) {
    const int64_t i = nmain + tid;
    const uint64_t qq = quantize_exact(a.xy, i, XY, ox, oy, a.side, a.lim, a.first_bad, a.idx_base);
    if (qq != ~0ull) {
      const uint32_t v = index_lookup(a.V, (uint32_t)qq, (uint32_t)(qq >> 32));
      if (v != 0u) add_owners_w<ATTR>(bins, slow, pool, v, ATTR ? a.attr[i] : 0.f, 0, false, a.V.code_mask);
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");  // consumers only (the producer has left)
  uint32_t* pc = a.part_cnt + (size_t)blockIdx.x * R2;
  double* ps = a.part_sum + (size_t)blockIdx.x * R2;
  for (int q = tid; q < R2; q += NW * 32) {
    uint32_t cnt = 0;
    long long f = 0;
    for (int c = 0; c < C; ++c) {
      const uint32_t* b = h3 + c * P + (ATTR ? 3 * q : q);
      cnt += b[0];
      if (ATTR) f += ((long long)(int32_t)b[2] << 16) + (long long)b[1];
    }
    pc[q] = cnt;
    if (ATTR) {
      if (f) atomicAdd((unsigned long long*)&prow[q], (unsigned long long)f);  // after this CTA's drains
      ps[q] = slow[q];
    }
  }
}

// ---------------------------------------------------------------------------
// Deep-index variant of the ring kernel (C4 class: a region set beyond shared
// memory and two or more node levels below the root, L <= 20, L - T0 <= 16).
//
// The same producer warp + 16 consumer warps and TMA ring, with the node
// descent spread over the software pipeline so that every dependent index load
// is consumed one iteration after it is issued:
//   C(k-3): accumulate the owner values nv2[] of tile k-3
//   B2(k-2): node levels 1.. of tile k-2 from nv1[] -> nv2[]
//   B1(k-1): node level 0 of tile k-1 from its root values rv[] -> nv1[]
//   A(k):   tile k: ring -> quantise -> summary -> root loads -> rv[]
// Only the low L - T0 bits of a point's cell coordinates address its node
// slots, so a tile in flight carries them packed in one register per point.
//
// Index forms (LAY): 0 radix table (node levels as above), 1 sorted keys (bucket in A,
// records in B1), 2 packed below the root (block in B1, palette select in C, three
// stages), 3 packed leaves below one u32 node level (node in B1, block in B2, select
// in C; 15 consumer warps for its 128 registers).
//
// Accumulation keeps the global-histogram semantics of
// k_point_pass_tma: interior single owners of a hot region (rb_approx_set_hot,
// value bits hot_shift..29 = slot + 1) with an in-window attribute take three
// shared REDs into the region's privatised alpha slot; cold interior single
// owners take two predicated global REDs (u64 count, f64 sum); boundary leaves,
// owner lists and out-of-window attributes go through the per-warp rare queue.
// Hot slots drain to the CTA's fixed-point row like the ring kernel's bins and
// are flushed into the global outputs at the end.
//
// The C4 pass is bound by random global requests per point (about 1.3 index
// loads and 0.5 REDs), not by HBM bytes: DESIGN.md section 5 measures the SM's
// request rates and puts this kernel at 0.81 of the resulting ceiling.
// ---------------------------------------------------------------------------
template <bool ATTR>
__device__ __forceinline__ void add_owners_g(uint32_t bins, const uint32_t* __restrict__ pool, uint32_t v, float w,
                                             int32_t qv, bool fast, unsigned long long* gcnt, double* gsum, uint32_t cm,
                                             uint32_t hs) {
  const uint32_t hm = ((1u << (30 - hs)) - 1u) << hs;  // hot field
  uint32_t n = 1, x = v;
  const uint32_t* Lp = nullptr;
  if (v & RB_VALUE_LIST) {
    Lp = pool + (v & RB_VALUE_PAYLOAD);
    n = __ldg(Lp) & ~RB_POOL_COUNT_FLAG;
  } else {
    x = ((v & cm) - 1u) | (v & hm);  // (region << 1) | boundary, hot slot
  }
#pragma unroll 1
  for (uint32_t i = 0; i < n; ++i) {
    if (Lp) {
      const uint32_t y = __ldg(Lp + 1 + i);
      x = (y & cm) | (y & hm);
    }
    const uint32_t e = x & cm, q = e & ~1u, slot = x >> hs;
    if (slot && !(e & 1u) && fast) {  // privatised alpha slot
      const uint32_t ad = bins + (slot - 1u) * (ATTR ? 12u : 4u);
      reds(ad, 1u);
      if (ATTR) { reds(ad + 4, (uint32_t)qv & 0xffffu); reds(ad + 8, (uint32_t)(qv >> 16)); }
      continue;
    }
    atomicAdd(&gcnt[q], 1ull);
    if (ATTR) atomicAdd(&gsum[q], (double)w);
    if (e & 1u) {  // boundary leaf: beta as well
      atomicAdd(&gcnt[q + 1], 1ull);
      if (ATTR) atomicAdd(&gsum[q + 1], (double)w);
    }
  }
}

// predicated global REDs (a C++ `if` around an atomic compiles to a branch per point)
__device__ __forceinline__ void redg_count(unsigned long long* p, bool pred) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %1, 0;\n @q red.global.add.u64 [%0], 1;\n}\n" ::"l"(p),
               "r"((uint32_t)pred)
               : "memory");
}
__device__ __forceinline__ void redg_sum(double* p, double w, bool pred) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %1, 0;\n @q red.global.add.f64 [%0], %2;\n}\n" ::"l"(p),
               "r"((uint32_t)pred), "d"(w)
               : "memory");
}

// ABL (timing experiments only, RB_DEEP_ABLATE; results are wrong): 1 = drop cold-region REDs (LAY 0 and 2),
// 2 = no palette-block loads (every point of a mixed root cell counts as hot slot 0), 4 = no root loads
template <int XY, bool ATTR, int NW, int PPT, int NST, int LAY = 0, int ABL = 0>
__global__ void __launch_bounds__(NW * 32 + 32, 1) k_point_pass_deep(PassArgs a) {
  constexpr bool KEYS = LAY == 1, PK = LAY == 2, PK3 = LAY == 3;  // PK3: radix node level over packed leaves
  constexpr int PB = XY == 0 ? 16 : 8;
  constexpr int WT = PPT * 32;
  constexpr int TP = NW * WT;
  constexpr uint32_t XYB = TP * PB, ATB = ATTR ? TP * 4 : 0, STAGE = XYB + ATB;
  constexpr uint32_t BS = ATTR ? 12u : 4u;
  const int C = a.hcopies, P = a.hstride, NH = a.n_hot;
  // Drains are partitioned: warp w drains hot slots q with (q / 32) % NW == w every FOLD of its own tiles.
  // Warps stay within NST tiles of each other (one ring), so between two drains of a copy-slot every
  // warp adds at most (FOLD + NST) * WT / C values to it: <= NW * 30 * WT (61440 for NW = 16, WT = 128)
  // plus <= 63 queued per warp, which keeps the low halves below 2^32 and the high halves within 2^30.
  int FOLD = C * (61440 / (NW * WT) > 0 ? 61440 / (NW * WT) : 1) - NST;
  if (FOLD < 1) FOLD = 1;
  if (a.fold > 0 && a.fold < FOLD) FOLD = a.fold;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  __shared__ float smax[NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // layout: [NST stages][per-warp rare queues: NW x 64 x 8 B][32 dummy bins][C hot-slot copies of P words][summary u16]
  uint2* rq = (uint2*)(smem + (size_t)NST * STAGE) + (size_t)(warp < NW ? warp : 0) * 64;
  unsigned char* dummy = smem + (size_t)NST * STAGE + NW * 64 * 8;
  uint32_t* h3 = (uint32_t*)(dummy + 32 * BS);
  const size_t h3b = (((size_t)C * P * 4) + 15) & ~(size_t)15;
  uint16_t* summ = (uint16_t*)((unsigned char*)h3 + h3b);
  long long* prow = a.part_acc + (size_t)blockIdx.x * (NH > 0 ? NH : 1);
  const bool has_summ = a.V.S >= 0;
  const int S = has_summ ? a.V.S : 0;
  constexpr int NT = NW * 32 + 32;
  for (int q = tid; q < C * P; q += NT) h3[q] = 0;
  if (ATTR)
    for (int q = tid; q < NH; q += NT) prow[q] = 0;
  if (has_summ) {
    const int nsum = 1 << (2 * S);
    const uint4* src = (const uint4*)a.V.summary;
    for (int q = tid; q < (nsum >> 3); q += NT) ((uint4*)summ)[q] = __ldg(src + q);
    for (int q = (nsum & ~7) + tid; q < nsum; q += NT) summ[q] = a.V.summary[q];
  }
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t nmain = a.n & ~(int64_t)3;
  const int64_t ntiles = (nmain + TP - 1) / TP;
  const int64_t G = gridDim.x;
  if (warp == NW) {  // producer
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int st = 0;
      uint32_t ph = 0;
      int64_t k = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += G, ++k) {
        if (k >= NST) mbar_wait(&empty[st], ph ^ 1u);
        const int64_t p0 = t * TP;
        const uint32_t m = (uint32_t)(p0 + TP <= nmain ? TP : nmain - p0);
        unsigned char* dst = smem + (size_t)st * STAGE;
        mbar_expect_tx(&full[st], m * (PB + (ATTR ? 4 : 0)));
        bulk_g2s(dst, (const char*)a.xy + p0 * PB, m * PB, &full[st], pol);
        if (ATTR) bulk_g2s(dst + XYB, a.attr + p0, m * 4, &full[st], pol);
        if (++st == NST) { st = 0; ph ^= 1u; }
      }
    }
    return;
  }
  // consumers: fixed-point scale from the same strided sample as every other CTA
  float sc = 1.f;
  uint32_t wminb = 0, wspan = 0;
  int Sx = 0;
  if (ATTR) {
    float mx = 0.f;
    const int64_t stride = a.n / 4096 > 0 ? a.n / 4096 : 1;
    constexpr int NSAMP = (4096 + NW * 32 - 1) / (NW * 32);
    float sv[NSAMP];
#pragma unroll
    for (int j = 0; j < NSAMP; ++j) {
      const int64_t q = tid + (int64_t)j * NW * 32;
      sv[j] = (q < 4096 && q * stride < a.n) ? __ldg(a.attr + q * stride) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < NSAMP; ++j) {
      const float v = fabsf(sv[j]);
      if (isfinite(v)) mx = fmaxf(mx, v);
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) smax[warp] = mx;
    asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
    mx = 0.f;
    for (int w2 = 0; w2 < NW; ++w2) mx = fmaxf(mx, smax[w2]);
    if (mx > 0.f) {
      int e = 0;
      frexpf(mx, &e);
      Sx = 29 - e;
    }
    Sx = Sx < -96 ? -96 : (Sx > 126 ? 126 : Sx);
    sc = __int_as_float((Sx + 127) << 23);
    wminb = (uint32_t)((20 - Sx + 127) << 23);
    wspan = (uint32_t)((30 - Sx + 127) << 23) - wminb;
  }
  const double ox = a.ox, oy = a.oy, inv_side = a.inv_side;
  const uint32_t* __restrict__ root = a.V.root;
  const uint32_t* __restrict__ pool = a.V.pool;
  const uint32_t* __restrict__ nodes0 = a.V.nodes[0];
  const uint32_t* __restrict__ nodes1 = a.V.nodes[a.V.nlev > 1 ? 1 : 0];
  const int L = a.V.L, T0 = a.V.T0, s0 = L - T0, nlev = a.V.nlev, sS = L - S;
  // node slots from the packed low coordinates c = (bx & m0) | (by & m0) << 16 (32-bit node offsets)
  const int k0 = a.V.ks[0], s1 = s0 - k0, k1 = nlev > 1 ? a.V.ks[1] : 0, s2 = s1 - k1;
  const uint32_t hibits = ~((1u << L) - 1u);
  const uint32_t m0 = (1u << s0) - 1u, mk0 = (1u << k0) - 1u, mk1 = (1u << k1) - 1u;
  const uint32_t bins = smem_u32(h3) + (uint32_t)((lane & (C - 1)) * P) * 4u;
  const uint32_t h3s = bins - BS;  // hot field (slot + 1) -> slot bin at h3s + field * BS
  const uint32_t dms = smem_u32(dummy) + lane * BS;
  const uint32_t cmask = a.V.code_mask, hsh = a.V.hot_shift;
  const uint32_t full_a = smem_u32(full), empty_a = smem_u32(empty);  // mbarrier addresses, hoisted
  unsigned long long* gcnt = a.gcnt;
  double* gsum = a.gsum;
  int qh = 0, qn = 0;
  auto rare_flush = [&](int nitems) {
    if (lane < nitems) {
      const uint2 it = rq[(qh + lane) & 63];
      const float ww = __uint_as_float(it.y);
      const bool fast = !ATTR || (((it.y & 0x7fffffffu) - wminb) < wspan);
      add_owners_g<ATTR>(bins, pool, it.x, ww, ATTR ? __float2int_rn(ww * sc) : 0, fast, gcnt, gsum, a.V.code_mask,
                          a.V.hot_shift);
    }
    __syncwarp();
  };
  uint32_t rv[PPT], c1[PPT], c2[PPT], nv1[PPT], nv2[PPT];
  uint32_t hv[PPT], zh[PPT];  // KEYS: radix bucket end (~0u: answered) and the leaf code's high word (c1: low word)
  uint4 pb[PPT];              // PK: palette blocks loaded in B1 (c2: the leaf's slot in its block); PK3: in B2
  const uint4* __restrict__ pblk = a.V.pblk;
  const uint32_t* __restrict__ pwide = a.V.pwide;
  const int pd = a.V.pd;
  float w1[PPT], w2[PPT], w3[PPT];
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    rv[j] = c1[j] = c2[j] = nv1[j] = nv2[j] = 0u;
    w1[j] = w2[j] = w3[j] = 0.f;
    pb[j] = make_uint4(0u, 0u, 0u, 0u);
    hv[j] = 0u;
  }
  int st = 0;
  uint32_t ph = 0;
  int dk = 0;
  const int64_t K = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / G + 1 : 0;
  // PK: three stages (A, B1 = block load, C = palette select + accumulate), the others four
  constexpr int CD = PK ? 2 : 3;
  for (int64_t k = 0; k < K + CD; ++k) {
    // ------------------------------------------------------------ C(k-CD)
    if (k >= CD) {
      if constexpr (PK3) {  // leaf palette select (blocks loaded in B2; hv: the leaf's slot); escapes: one more load
        bool esc = false;
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          nv2[j] = packed_pick(pb[j], hv[j]);
          esc |= (int32_t)nv2[j] < 0;
        }
        if (__any_sync(0xffffffffu, esc)) {
#pragma unroll
          for (int j = 0; j < PPT; ++j)
            nv2[j] = ldg_pred(pwide + ((size_t)(nv2[j] & RB_VALUE_PAYLOAD) << 4) + hv[j], (int32_t)nv2[j] < 0, nv2[j]);
        }
      }
      if constexpr (PK) {  // palette select; escape blocks (> 3 owner values) load their leaf's value
        bool esc = false;
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          w3[j] = w2[j];
          nv2[j] = packed_pick(pb[j], c2[j]);
          esc |= (int32_t)nv2[j] < 0;
        }
        if (__any_sync(0xffffffffu, esc)) {
#pragma unroll
          for (int j = 0; j < PPT; ++j)
            nv2[j] = ldg_pred(pwide + ((size_t)(nv2[j] & RB_VALUE_PAYLOAD) << 4) + c2[j], (int32_t)nv2[j] < 0, nv2[j]);
        }
      }
      bool anyrare = false;
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const uint32_t v = nv2[j];
        int32_t qv = 0;
        bool fast = true;
        if (ATTR) {
          qv = __float2int_rn(w3[j] * sc);
          fast = ((__float_as_uint(w3[j]) & 0x7fffffffu) - wminb) < wspan;
        }
        const uint32_t hot = (v & ~(RB_VALUE_NODE | RB_VALUE_LIST)) >> hsh;
        // interior single owner with an in-window attribute: a hot region's privatised slot, else
        // predicated global REDs on its alpha bin; everything else takes the rare queue
        const bool single = ((v & (RB_VALUE_LIST | 1u)) == 1u) & fast;
        const bool common = single & (hot != 0u);
        const uint32_t ad = common ? h3s + hot * BS : dms;
        reds(ad, 1u);
        if (ATTR) {
          reds(ad + 4, (uint32_t)qv & 0xffffu);
          reds(ad + 8, (uint32_t)(qv >> 16));
        }
        const bool cold = single & (hot == 0u);
        const uint32_t q = (v & cmask) - 1u;
        if constexpr (!(ABL & 1)) {
          redg_count(gcnt + q, cold);
          if (ATTR) redg_sum(gsum + q, (double)w3[j], cold);
        }
        anyrare |= !single & (v != 0u);
      }
      if (__any_sync(0xffffffffu, anyrare)) {
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          const uint32_t v = nv2[j];
          const bool fast = !ATTR || (((__float_as_uint(w3[j]) & 0x7fffffffu) - wminb) < wspan);
          const bool rare = !(((v & (RB_VALUE_LIST | 1u)) == 1u) & fast) & (v != 0u);
          const uint32_t mk = __ballot_sync(0xffffffffu, rare);
          if (mk) {
            if (rare) rq[(qh + qn + __popc(mk & ((1u << lane) - 1u))) & 63] = make_uint2(v, __float_as_uint(w3[j]));
            qn += __popc(mk);
            if (qn >= 32) {
              __syncwarp();
              rare_flush(32);
              qh = (qh + 32) & 63;
              qn -= 32;
            }
          }
        }
      }
      if (ATTR && ++dk == FOLD) {  // drain this warp's share of the hot slots into the CTA's row
        dk = 0;
        __syncwarp();
        for (int q = warp * 32 + lane; q < NH; q += NW * 32) {
          long long f = 0;
          for (int c = 0; c < C; ++c) {
            const uint32_t lo = atomicExch(&h3[c * P + 3 * q + 1], 0u);
            const uint32_t hi = atomicExch(&h3[c * P + 3 * q + 2], 0u);
            f += ((long long)(int32_t)hi << 16) + (long long)lo;
          }
          if (f) atomicAdd((unsigned long long*)&prow[q], (unsigned long long)f);
        }
      }
    }
    // ------------------------------------------------------------ B2(k-2): node levels 1..
    if constexpr (PK) {  // (no second node stage: C selects from the block)
    } else
    if constexpr (PK3) {  // the 16-byte palette block below a node-level-0 slot (radix node, then packed leaves)
      if (k >= 2 && k <= K + 1) {
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          w3[j] = w2[j];
          const uint32_t lx = c2[j] & 0xffffu, ly = c2[j] >> 16;
          hv[j] = packed_slot(lx, ly);
          pb[j] = ldg4_pred(pblk + packed_block(nv1[j] & RB_VALUE_PAYLOAD, lx, ly, pd), (int32_t)nv1[j] < 0, nv1[j]);
        }
      }
    } else
    if constexpr (KEYS) {
      if (k >= 2 && k <= K + 1) {
#pragma unroll
        for (int j = 0; j < PPT; ++j) { w3[j] = w2[j]; nv2[j] = nv1[j]; }
      }
    } else
    if (k >= 2 && k <= K + 1) {
#pragma unroll
      for (int j = 0; j < PPT; ++j) { w3[j] = w2[j]; nv2[j] = nv1[j]; }
      uint32_t anyn = 0;
#pragma unroll
      for (int j = 0; j < PPT; ++j) anyn |= nv2[j];
      if (nlev > 1 && __any_sync(0xffffffffu, (int32_t)anyn < 0)) {
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          const uint32_t slot = (((c2[j] >> (16 + s2)) & mk1) << k1) | ((c2[j] >> s2) & mk1);
          const uint32_t off = ((nv2[j] & RB_VALUE_PAYLOAD) << (2 * k1)) | slot;
          nv2[j] = ldg_pred(nodes1 + off, (int32_t)nv2[j] < 0, nv2[j]);
        }
        if (nlev > 2) {  // deeper trees: the remaining levels in place (one more dependent load each)
          int s = s2;
#pragma unroll 1
          for (int li = 2; li < nlev; ++li) {
            const int kk = a.V.ks[li];
            const uint32_t* __restrict__ nodes = a.V.nodes[li];
            s -= kk;
            const uint32_t msk = (1u << kk) - 1u;
#pragma unroll
            for (int j = 0; j < PPT; ++j) {
              const uint32_t slot = (((c2[j] >> (16 + s)) & msk) << kk) | ((c2[j] >> s) & msk);
              const uint32_t off = ((nv2[j] & RB_VALUE_PAYLOAD) << (2 * kk)) | slot;
              nv2[j] = ldg_pred(nodes + off, (int32_t)nv2[j] < 0, nv2[j]);
            }
          }
        }
      }
    }
    // ------------------------------------------------------------ B1(k-1): node level 0
    if constexpr (PK3) {  // node level 0 (radix slots over the root cell) as for the radix table
      if (k >= 1 && k <= K) {
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          w2[j] = w1[j];
          c2[j] = c1[j];
          const uint32_t slot = (((c1[j] >> (16 + s1)) & mk0) << k0) | ((c1[j] >> s1) & mk0);
          const uint32_t off = ((rv[j] & RB_VALUE_PAYLOAD) << (2 * k0)) | slot;
          nv1[j] = ldg_pred(nodes0 + off, (int32_t)rv[j] < 0, rv[j]);
        }
      }
    } else
    if constexpr (PK) {  // the 16-byte palette block of each point in a mixed root cell
      if (k >= 1 && k <= K) {
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          w2[j] = w1[j];
          const uint32_t lx = c1[j] & 0xffffu, ly = c1[j] >> 16;
          c2[j] = packed_slot(lx, ly);
          if constexpr (ABL & 2)
            pb[j] = make_uint4((int32_t)rv[j] < 0 ? (1u << hsh) | 1u : rv[j], 0u, 0u, 0u);
          else
            pb[j] = ldg4_pred(pblk + packed_block(rv[j] & RB_VALUE_PAYLOAD, lx, ly, pd), (int32_t)rv[j] < 0, rv[j]);
        }
      }
    } else
    if constexpr (KEYS) {  // RB_LAYOUT_KEYS: the bucket's cell records
      if (k >= 1 && k <= K) {
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          w2[j] = w1[j];
          nv1[j] = hv[j] == ~0u ? rv[j]
                                : keys_resolve(a.V, ((uint64_t)zh[j] << 32) | c1[j], (int64_t)rv[j], (int64_t)hv[j]);
        }
      }
    } else
    if (k >= 1 && k <= K) {
#pragma unroll
      for (int j = 0; j < PPT; ++j) { w2[j] = w1[j]; c2[j] = c1[j]; }
      uint32_t anyn = 0;
#pragma unroll
      for (int j = 0; j < PPT; ++j) anyn |= rv[j];
      if (__any_sync(0xffffffffu, (int32_t)anyn < 0)) {
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          const uint32_t slot = (((c1[j] >> (16 + s1)) & mk0) << k0) | ((c1[j] >> s1) & mk0);
          const uint32_t off = ((rv[j] & RB_VALUE_PAYLOAD) << (2 * k0)) | slot;
          nv1[j] = ldg_pred(nodes0 + off, (int32_t)rv[j] < 0, rv[j]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < PPT; ++j) nv1[j] = rv[j];
      }
    }
    // ------------------------------------------------------------ A(k)
    if (k < K) {
      const int64_t t = blockIdx.x + k * G;
      mbar_wait_warp_a(full_a + 8u * st, ph);
      const unsigned char* tile = smem + (size_t)st * STAGE;
      double x[PPT], y[PPT];
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const int pi = warp * WT + lane + 32 * j;
        if (XY == 0) {
          const double2 v2 = ((const double2*)tile)[pi];
          x[j] = v2.x; y[j] = v2.y;
        } else {
          const float2 v2 = ((const float2*)tile)[pi];
          x[j] = (double)v2.x; y[j] = (double)v2.y;
        }
        w1[j] = ATTR ? ((const float*)(tile + XYB))[pi] : 0.f;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_a(empty_a + 8u * st);
      if (++st == NST) { st = 0; ph ^= 1u; }
      uint32_t bx[PPT], by[PPT];
      bool anybad = false;
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const double tx = __fma_rn(__dsub_rn(x[j], ox), inv_side, 1048576.0);
        const double ty = __fma_rn(__dsub_rn(y[j], oy), inv_side, 1048576.0);
        bx[j] = (uint32_t)__double2hiint(tx) - 0x41300000u;
        by[j] = (uint32_t)__double2hiint(ty) - 0x41300000u;
        const uint32_t fx = (uint32_t)__double2loint(tx) + 8u, fy = (uint32_t)__double2loint(ty) + 8u;
        anybad |= ((bx[j] | by[j]) & hibits) != 0u;
        anybad |= (fx < 16u) | (fy < 16u);
      }
      const int64_t p0 = t * TP + warp * WT;
      uint32_t killm = 0;
      if (__any_sync(0xffffffffu, anybad) || p0 + WT > nmain) {
        const int64_t mm = nmain - p0;
        const int m = (int)(mm >= WT ? WT : (mm > 0 ? mm : 0));
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          const double tx = __fma_rn(__dsub_rn(x[j], ox), inv_side, 1048576.0);
          const double ty = __fma_rn(__dsub_rn(y[j], oy), inv_side, 1048576.0);
          const uint32_t fx = (uint32_t)__double2loint(tx) + 8u, fy = (uint32_t)__double2loint(ty) + 8u;
          const bool bad = (((bx[j] | by[j]) & hibits) != 0u) | (fx < 16u) | (fy < 16u);
          if (lane + 32 * j >= m) {
            bx[j] = 0; by[j] = 0; killm |= 1u << j;
          } else if (bad) {
            const uint64_t qq =
                quantize_exact(a.xy, p0 + lane + 32 * j, XY, ox, oy, a.side, a.lim, a.first_bad, a.idx_base);
            if (qq != ~0ull) { bx[j] = (uint32_t)qq; by[j] = (uint32_t)(qq >> 32); }
            else { bx[j] = 0; by[j] = 0; killm |= 1u << j; }
          }
        }
      }
      uint32_t sv[PPT];
#pragma unroll
      for (int j = 0; j < PPT; ++j) sv[j] = has_summ ? (uint32_t)summ[((by[j] >> sS) << S) | (bx[j] >> sS)] : 0xffffu;
      if (killm) {
#pragma unroll
        for (int j = 0; j < PPT; ++j)
          if (killm & (1u << j)) sv[j] = 0u;
      }
      if constexpr (KEYS) {  // the radix bucket now, its records in B1
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          const uint64_t z = leaf_z(bx[j], by[j]);
          const uint64_t p = z >> a.V.kshift;
          rv[j] = ldg_pred(a.V.ktab + p, sv[j] == 0xffffu, sv[j]);
          hv[j] = ldg_pred(a.V.ktab + p + 1, sv[j] == 0xffffu, ~0u);
          c1[j] = (uint32_t)z;
          zh[j] = (uint32_t)(z >> 32);
        }
      } else {
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const uint32_t* rp = root + (((by[j] >> s0) << T0) | (bx[j] >> s0));
        if constexpr (ABL & 4)
          rv[j] = (1u << hsh) | 1u + (rp == nullptr);
        else
          rv[j] = ldg_pred(rp, sv[j] == 0xffffu, sv[j]);
        c1[j] = (bx[j] & m0) | ((by[j] & m0) << 16);
      }
      }
    }
  }
  __syncwarp();
  if (qn) rare_flush(qn);
  if (blockIdx.x == 0 && tid < (int)(a.n - nmain)) {  // up to 3 trailing points
    const int64_t i = nmain + tid;
    const uint64_t qq = quantize_exact(a.xy, i, XY, ox, oy, a.side, a.lim, a.first_bad, a.idx_base);
    if (qq != ~0ull) {
      const uint32_t v = index_lookup(a.V, (uint32_t)qq, (uint32_t)(qq >> 32));
      if (v != 0u) add_owners_g<ATTR>(bins, pool, v, ATTR ? a.attr[i] : 0.f, 0, false, gcnt, gsum, a.V.code_mask, a.V.hot_shift);
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
  // flush the hot slots into the global outputs (alpha bin of the slot's region)
  for (int q = tid; q < NH; q += NW * 32) {
    uint32_t cnt = 0;
    long long f = 0;
    for (int c = 0; c < C; ++c) {
      const uint32_t* b = h3 + c * P + (ATTR ? 3 * q : q);
      cnt += b[0];
      if (ATTR) f += ((long long)(int32_t)b[2] << 16) + (long long)b[1];
    }
    if (!cnt) continue;
    const int32_t r = a.hot_region[q];
    atomicAdd(&gcnt[2 * r], (unsigned long long)cnt);
    if (ATTR) atomicAdd(&gsum[2 * r], ldexp((double)(__ldcg(&prow[q]) + f), -Sx));  // drains are L2 REDs
  }
}

// binary scale of the SUM fixed point from a strided sample of the attribute
__global__ void k_attr_scale(const float* attr, int64_t n, int* scale_exp) {
  __shared__ float red[1024];
  float m = 0.f;
  const int64_t stride = n / 4096 > 0 ? n / 4096 : 1;
  for (int64_t k = threadIdx.x; k < 4096 && k * stride < n; k += blockDim.x) {
    const float v = fabsf(attr[k * stride]);
    if (isfinite(v)) m = fmaxf(m, v);
  }
  red[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmaxf(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int e = 0;
    int S = 0;
    if (red[0] > 0.f) {
      frexpf(red[0], &e);  // red[0] < 2^e
      S = 29 - e;          // fast window [2^(e-9), 2^(e+1))
    }
    S = S < -96 ? -96 : (S > 126 ? 126 : S);
    *scale_exp = S;
  }
}

// deterministic reduction of the per-CTA rows: a block owns 32 consecutive
// bins (lane = bin, coalesced row reads); its 32 warps stride over the rows
// and are combined in fixed warp order.
__global__ void __launch_bounds__(1024) k_reduce_fixed(const uint32_t* part_cnt, const long long* part_acc,
                                                       const double* part_sum, int nrows, int R2, bool attr,
                                                       bool ib, const int* scale_exp, int64_t* cnt_out,
                                                       double* sum_out) {
  __shared__ unsigned long long sc[32][32];
  __shared__ long long sa[32][32];
  __shared__ double ss[32][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = blockIdx.x * 32 + lane;
  unsigned long long c = 0;
  long long f = 0;
  double s = 0.0;
  if (q < R2) {
    for (int r = warp; r < nrows; r += 32) {
      c += part_cnt[(size_t)r * R2 + q];
      if (attr) { f += part_acc[(size_t)r * R2 + q]; s += part_sum[(size_t)r * R2 + q]; }
    }
  }
  sc[warp][lane] = c;
  sa[warp][lane] = f;
  ss[warp][lane] = s;
  __syncthreads();
  if (warp == 0) {
    for (int w2 = 1; w2 < 32; ++w2) { c += sc[w2][lane]; f += sa[w2][lane]; s += ss[w2][lane]; }
    if (ib) {  // ring kernel bins: 2r = interior-leaf points, 2r+1 = boundary-leaf points -> alpha = both
      const unsigned long long c1 = __shfl_down_sync(0xffffffffu, c, 1);
      const long long f1 = __shfl_down_sync(0xffffffffu, f, 1);
      const double s1 = __shfl_down_sync(0xffffffffu, s, 1);
      if ((lane & 1) == 0) { c += c1; f += f1; s += s1; }
    }
  }
  if (warp == 0 && q < R2) {
    cnt_out[q] += (int64_t)c;
    if (attr) sum_out[q] += ldexp((double)f, -*scale_exp) + s;
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
  auto kern = k_point_pass_global<XY, SMEM, ATTR, VEC>;
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


// largest region count whose histogram (28 B per bin pair entry) fits the
// 200 KB shared-memory budget of one CTA
#define RB_SMEM_BUDGET (226 * 1024)

template <int XY, bool ATTR, bool VEC>
static cudaError_t launch_smem(const PassArgs& a, size_t smem, cudaStream_t s, int* blocks_out) {
  auto kern = k_point_pass<XY, ATTR, VEC>;
  static int cached_blocks = -1;
  static size_t cached_smem = 0;
  if (cached_blocks < 0 || cached_smem != smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, RB_SMEM_BUDGET);
    if (e) return e;
    if (const char* cv = getenv("RB_CARVEOUT")) {  // experiments: shared-memory share of the L1 (percent)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv));
      if (e) return e;
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
    if (e) return e;
    cached_blocks = std::max(1, per_sm) * g_num_sms;
    cached_smem = smem;
  }
  *blocks_out = cached_blocks;
  return cudaSuccess;
}
static int g_kernel_sel = -1;  // 0 = synchronous loads (fallback), 1 = TMA ring (default)

template <int XY, bool ATTR, bool GH>
static cudaError_t tma_blocks(size_t smem, int* blocks_out) {
  auto kern = k_point_pass_tma<XY, ATTR, GH>;
  static int cached_blocks = -1;
  static size_t cached_smem = 0;
  if (cached_blocks < 0 || cached_smem != smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, RB_SMEM_BUDGET);
    if (e) return e;
    if (const char* cv = getenv("RB_CARVEOUT")) {  // experiments: shared-memory share of the L1 (percent)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv));
      if (e) return e;
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, RB_CONS + 32, smem);
    if (e) return e;
    cached_blocks = std::max(1, per_sm) * g_num_sms;
    cached_smem = smem;
  }
  *blocks_out = cached_blocks;
  return cudaSuccess;
}

template <int XY, bool ATTR, bool GH>
static cudaError_t tma_run(const PassArgs& a, int blocks, size_t smem, cudaStream_t s) {
  k_point_pass_tma<XY, ATTR, GH><<<blocks, RB_CONS + 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <int XY, bool ATTR, bool VEC>
static cudaError_t run_smem(const PassArgs& a, int blocks, size_t smem, cudaStream_t s) {
  k_point_pass<XY, ATTR, VEC><<<blocks, 256, smem, s>>>(a);
  return cudaGetLastError();
}

// per-warp-ring kernel configurations (consumer warps, points per lane, stages)
struct WarpCfg { int nw, ppt, nst; };
// Preference order.  Shared memory and the L1 data cache share 256 KB per SM, and the carveout is the
// smallest step (..., 164, 196, 228 KB) that holds the CTA's shared memory.  The index lookups rarely
// hit in L1 (1.8 %), but each global load in flight holds an L1 line, so the L1 that is left bounds
// the lookups in flight.  A 3-stage ring with <= 4 histogram copies (~190 KB for C2 SUM -> 60 KB of
// L1) beat the 4-stage ring (~220 KB -> 28 KB of L1): 0.475 -> 0.444 ms; forcing the 3-stage ring to a
// 228 KB carveout gave 0.469 ms.  2 points per lane (0.54 ms), 3 points per lane (0.48 ms) and 2-stage
// rings (0.47 ms) were slower (profiles/round1/ring_config_sweep.txt).
static const WarpCfg kWarpCfgs[] = {{16, 4, 3}, {16, 4, 4}, {16, 4, 2}, {15, 4, 2}};

template <int XY, bool ATTR, int NW, int PPT, int NST, int LAY = 0>
static cudaError_t warp_run(const PassArgs& a, size_t smem, cudaStream_t s, int* blocks, bool launch) {
  auto kern = k_point_pass_ring<XY, ATTR, NW, PPT, NST, LAY>;
  static int cached_blocks = -1;
  static size_t cached_smem = 0;
  if (cached_blocks < 0 || cached_smem != smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, RB_SMEM_BUDGET);
    if (e) return e;
    if (const char* cv = getenv("RB_CARVEOUT")) {  // experiments: shared-memory share of the L1 (percent)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv));
      if (e) return e;
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32 + 32, smem);
    if (e) return e;
    cached_blocks = per_sm * g_num_sms;
    cached_smem = smem;
  }
  *blocks = cached_blocks;
  if (!launch || cached_blocks <= 0) return cudaSuccess;
  kern<<<cached_blocks, NW * 32 + 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <int XY, bool ATTR, int LAY = 0>
static cudaError_t warp_dispatch(int ci, const PassArgs& a, size_t smem, cudaStream_t s, int* blocks, bool launch) {
  if constexpr (LAY == 3) return cudaErrorNotSupported;  // the three-level packed index: deep kernel only
  else if constexpr (LAY != 0) return warp_run<XY, ATTR, 16, 4, 3, LAY>(a, smem, s, blocks, launch);  // default shape only
  switch (ci) {
    case 0: return warp_run<XY, ATTR, 16, 4, 3>(a, smem, s, blocks, launch);
    case 1: return warp_run<XY, ATTR, 16, 4, 4>(a, smem, s, blocks, launch);
    case 2: return warp_run<XY, ATTR, 16, 4, 2>(a, smem, s, blocks, launch);
    default: return warp_run<XY, ATTR, 15, 4, 2>(a, smem, s, blocks, launch);
  }
}

// Experiments (RB_PERSIST_MB = persisting L2 carve-out, RB_PERSIST_HIT = hit ratio): an L2 access policy
// window over the root table, so that the index's first level is not evicted by the point stream.
static bool persist_window(const PassArgs& a, cudaLaunchAttribute* at) {
  static int mb = -1;
  static float hr = 1.f;
  static size_t maxwin = 0;
  if (mb < 0) {
    const char* e = getenv("RB_PERSIST_MB");
    mb = e ? atoi(e) : 0;
    if (const char* h = getenv("RB_PERSIST_HIT")) hr = (float)atof(h);
    if (mb > 0) {
      int dev = 0, mx = 0, mw = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev);
      cudaDeviceGetAttribute(&mw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
      size_t want = std::min<size_t>((size_t)mb << 20, (size_t)mx);
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
      maxwin = (size_t)mw;
      fprintf(stderr, "rb: persisting L2 %zu of max %d bytes, window max %d bytes\n", want, mx, mw);
    }
  }
  if (mb <= 0) return false;
  at->id = cudaLaunchAttributeAccessPolicyWindow;
  at->val.accessPolicyWindow.base_ptr = (void*)a.V.root;
  at->val.accessPolicyWindow.num_bytes = std::min<size_t>(((size_t)4) << (2 * a.V.T0), maxwin);
  at->val.accessPolicyWindow.hitRatio = hr;
  at->val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  at->val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  return true;
}

template <int XY, bool ATTR, int NW, int PPT, int NST, int LAY = 0, int ABL = 0>
static cudaError_t deep_run(const PassArgs& a, size_t smem, cudaStream_t s, int* blocks, bool launch) {
  auto kern = k_point_pass_deep<XY, ATTR, NW, PPT, NST, LAY, ABL>;
  static int cached_blocks = -1;
  static size_t cached_smem = 0;
  if (cached_blocks < 0 || cached_smem != smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, RB_SMEM_BUDGET);
    if (e) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32 + 32, smem);
    if (e) return e;
    cached_blocks = per_sm * g_num_sms;
    cached_smem = smem;
  }
  *blocks = cached_blocks;
  if (!launch || cached_blocks <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cached_blocks);
  cfg.blockDim = dim3(NW * 32 + 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  if (persist_window(a, &at[0])) { cfg.attrs = at; cfg.numAttrs = 1; }
  return cudaLaunchKernelEx(&cfg, kern, a);
}

// C4 (200M points, 4095 hot slots): 3 stages + 1 hot-slot copy 1.64 ms; 2 stages 1.67; 4 stages 1.73;
// 2 copies 2.07 (less L1 for lookups in flight); 2048 hot slots 2.35, 1024 2.98 (profiles/round1/deep_sweep.txt)
// 3: 15 consumer warps (128 registers); the same speed for the radix table (C4 1.67 vs 1.65 ms)
static const WarpCfg kDeepCfgs[] = {{16, 4, 3}, {16, 4, 2}, {16, 4, 4}, {15, 4, 3}};

template <int XY, bool ATTR, int LAY = 0>
static cudaError_t deep_dispatch(int ci, const PassArgs& a, size_t smem, cudaStream_t s, int* blocks, bool launch) {
  if constexpr (XY == 1 && ATTR && (LAY == 2 || LAY == 0)) {  // timing ablations of the C4 kernel (tools/, RB_DEEP_ABLATE)
    static int abl = -1;
    if (abl < 0) { const char* e = getenv("RB_DEEP_ABLATE"); abl = e ? atoi(e) : 0; }
    switch (abl) {
      case 1: return deep_run<XY, ATTR, 16, 4, 3, LAY, 1>(a, smem, s, blocks, launch);
      case 3: if constexpr (LAY == 2) return deep_run<XY, ATTR, 16, 4, 3, LAY, 3>(a, smem, s, blocks, launch); break;
      case 7: if constexpr (LAY == 2) return deep_run<XY, ATTR, 16, 4, 3, LAY, 7>(a, smem, s, blocks, launch); break;
      case 6: if constexpr (LAY == 2) return deep_run<XY, ATTR, 16, 4, 3, LAY, 6>(a, smem, s, blocks, launch); break;
      default: break;
    }
  }
  if constexpr (LAY == 3) {  // 15 consumer warps (4 per SM sub-partition: 128 registers, no spills): C4 1.68 ms per
                             // 200M points; RB_PK3_CFG=1: 16 warps at 96 registers spill, 2.29 ms
    static int cfg = -1;
    if (cfg < 0) { const char* e = getenv("RB_PK3_CFG"); cfg = e ? atoi(e) : 0; }
    if (cfg == 1) return deep_run<XY, ATTR, 16, 4, 3, LAY>(a, smem, s, blocks, launch);
    return deep_run<XY, ATTR, 15, 4, 3, LAY>(a, smem, s, blocks, launch);
  }
  if constexpr (LAY != 0) return deep_run<XY, ATTR, 16, 4, 3, LAY>(a, smem, s, blocks, launch);  // default shape only
  switch (ci) {
    case 0: return deep_run<XY, ATTR, 16, 4, 3>(a, smem, s, blocks, launch);
    case 1: return deep_run<XY, ATTR, 16, 4, 2>(a, smem, s, blocks, launch);
    case 3: return deep_run<XY, ATTR, 15, 4, 3>(a, smem, s, blocks, launch);
    default: return deep_run<XY, ATTR, 16, 4, 4>(a, smem, s, blocks, launch);
  }
}

#include "rb_binned.cuh"

#define RB_DISPATCH_TMA(FN, GHV, ...)                                                          \
  (dtype == RB_XY_F64 ? (attr ? FN<0, true, GHV>(__VA_ARGS__) : FN<0, false, GHV>(__VA_ARGS__)) \
                      : (attr ? FN<1, true, GHV>(__VA_ARGS__) : FN<1, false, GHV>(__VA_ARGS__)))
#define RB_DISPATCH_SYNC(FN, ...)                                                                           \
  (dtype == RB_XY_F64                                                                                       \
       ? (attr ? (vec ? FN<0, true, true>(__VA_ARGS__) : FN<0, true, false>(__VA_ARGS__))                   \
               : (vec ? FN<0, false, true>(__VA_ARGS__) : FN<0, false, false>(__VA_ARGS__)))                \
       : (attr ? (vec ? FN<1, true, true>(__VA_ARGS__) : FN<1, true, false>(__VA_ARGS__))                   \
               : (vec ? FN<1, false, true>(__VA_ARGS__) : FN<1, false, false>(__VA_ARGS__))))

// dtype x attribute x layout instantiation of warp_dispatch / deep_dispatch
#define RB_DISPATCH_LAY(FN, ...)                                                                      \
  (dtype == RB_XY_F64                                                                                 \
       ? (attr ? (lay == 1 ? FN<0, true, 1>(__VA_ARGS__) : lay == 2 ? FN<0, true, 2>(__VA_ARGS__)     \
                  : lay == 3 ? FN<0, true, 3>(__VA_ARGS__) : FN<0, true, 0>(__VA_ARGS__))                  \
               : (lay == 1 ? FN<0, false, 1>(__VA_ARGS__) : lay == 2 ? FN<0, false, 2>(__VA_ARGS__)   \
                  : lay == 3 ? FN<0, false, 3>(__VA_ARGS__) : FN<0, false, 0>(__VA_ARGS__)))               \
       : (attr ? (lay == 1 ? FN<1, true, 1>(__VA_ARGS__) : lay == 2 ? FN<1, true, 2>(__VA_ARGS__)     \
                  : lay == 3 ? FN<1, true, 3>(__VA_ARGS__) : FN<1, true, 0>(__VA_ARGS__))                  \
               : (lay == 1 ? FN<1, false, 1>(__VA_ARGS__) : lay == 2 ? FN<1, false, 2>(__VA_ARGS__)   \
                  : lay == 3 ? FN<1, false, 3>(__VA_ARGS__) : FN<1, false, 0>(__VA_ARGS__))))

// flags: bit0 = zero the outputs first, bit1 = reset first_bad first
int point_pass(const rb_approx* A, const void* xy, int32_t dtype, int64_t n, const float* attr, int64_t* cnt_out,
               double* sum_out, int64_t* first_bad, int flags, int64_t idx_base, cudaStream_t s) {
  if (!g_num_sms) {
    int dev = 0;
    RB_CUDA(cudaGetDevice(&dev));
    RB_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  if (g_kernel_sel < 0) {
    const char* ks = getenv("RB_KERNEL");
    g_kernel_sel = ks ? atoi(ks) : 1;
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
  a.hot_region = A->hot_region.as<int32_t>();
  a.n_hot = A->n_hot;
  if (flags) {
    k_init_out<<<std::max(1, (R2 + 255) / 256), 256, 0, s>>>(cnt_out, sum_out, R2, flags, a.first_bad);
    RB_CUDA(cudaGetLastError());
    ++g_launches;
  }
  if (n == 0) return RB_OK;
  const size_t pt_bytes = (dtype == RB_XY_F64 ? 16 : 8) + (attr ? 4 : 0);
  const size_t ring = (size_t)RB_NST * RB_TP * pt_bytes;
  const size_t summ_bytes = A->S >= 0 ? ((size_t)2 << (2 * A->S)) + 32 : 0;
  const size_t all_bins = (size_t)R2 * (attr ? 28 : 4) + 16;
  const size_t hot_bins = (((size_t)A->n_hot * (attr ? 12 : 4)) + 15) & ~(size_t)15;
  const bool aligned = ((uintptr_t)xy % 16 == 0) && (!attr || (uintptr_t)attr % 16 == 0);
  const bool vec = ((uintptr_t)xy % 32 == 0) && (!attr || (uintptr_t)attr % (dtype == RB_XY_F64 ? 8 : 16) == 0);
  const bool keys = A->keys.p != nullptr;  // RB_LAYOUT_KEYS: the ring kernel (KEYS) or the generic kernels
  const bool packed = A->pblk.p != nullptr;  // RB_LAYOUT_PACKED: ring / deep kernels (PK) or the generic kernel
  const int lay = keys ? 1 : (packed ? (A->node_bufs.empty() ? 2 : 3) : 0);
  const bool use_tma = g_kernel_sel != 0 && aligned && !keys && !packed;
  // histogram placement: every bin in shared memory when it fits next to the ring
  const bool smem_hist = use_tma ? ring + all_bins + summ_bytes <= RB_SMEM_BUDGET
                                 : (size_t)R2 * (attr ? 28 : 4) <= RB_SMEM_BUDGET;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  auto tstart = [&]() -> int {
    if (g_timing) {
      RB_CUDA(cudaEventCreate(&ev0));
      RB_CUDA(cudaEventCreate(&ev1));
      RB_CUDA(cudaEventRecord(ev0, s));
    }
    return RB_OK;
  };
  auto tstop = [&]() -> int {
    ++g_launches;
    if (g_timing) {
      RB_CUDA(cudaEventRecord(ev1, s));
      std::lock_guard<std::mutex> lk(g_ev_mu);
      g_events.emplace_back(ev0, ev1);
    }
    return RB_OK;
  };
  cudaError_t e = cudaSuccess;
  const bool keys_deep = (keys || packed) && g_kernel_sel != 0 && aligned && L <= 20 && g_kernel_sel != 3 && g_kernel_sel != 4;
  if ((!smem_hist || packed) && !use_tma && !keys_deep) {  // fallback: misaligned inputs with large region sets,
                                                          // or the packed layout beyond the ring kernels' L <= 20
    const int blocks = g_num_sms * 4;
    if (tstart()) return RB_CUDA_ERROR;
    e = dtype == RB_XY_F64 ? launch_a<0, false>(a, vec, blocks, 0, s) : launch_a<1, false>(a, vec, blocks, 0, s);
    if (e) return cuda_fail(e, "k_point_pass_global");
    return tstop();
  }
  // partitioned pass (rb_binned.cuh): large batches on the radix table with region sets beyond shared memory
  if (g_kernel_sel != 0 && g_kernel_sel != 3 && g_kernel_sel != 4 && binned_wanted(A, n, aligned, smem_hist)) {
    if (tstart()) return RB_CUDA_ERROR;
    int nl = 0;
    if (int st = binned_pass(A, a, dtype, attr != nullptr, s, &nl)) return st;
    g_launches += nl - 1;  // tstop counts one
    return tstop();
  }
  int blocks = 0;
  size_t smem = 0;
  // per-warp rings: shared-memory histogram, L <= 20 (the 2^20 quantisation window)
  int wci = -1;
  if (g_kernel_sel != 0 && aligned && smem_hist && L <= 20 && g_kernel_sel != 3 && lay != 3) {
    static int env_ci = -2;
    if (env_ci == -2) {
      const char* e = getenv("RB_WARP_CFG");
      env_ci = e ? atoi(e) : -1;
    }
    static int env_copies = -2;
    if (env_copies == -2) {
      const char* e = getenv("RB_HIST_COPIES");
      env_copies = e ? atoi(e) : -1;
    }
    const size_t summ_w = A->S >= 0 ? ((size_t)2 << (2 * A->S)) : 16;
    const int ncfg = (int)(sizeof(kWarpCfgs) / sizeof(kWarpCfgs[0]));
    // histogram copies: up to 4 with an attribute (distinct-value REDs to one word serialise;
    // same-address count increments are aggregated by the hardware), 1 for COUNT; 8 copies cost
    // more L1 (carveout) than they save in RED conflicts
    for (int c = 0; c < ncfg && wci < 0; ++c) {
      if (env_ci >= 0 && c != env_ci) continue;
      if (lay != 0 && c != 0) continue;  // the KEYS / PK rings are instantiated for the default shape only
      const WarpCfg& W = kWarpCfgs[c];
      const int wpb = attr ? 3 : 1;
      const int P = R2 * wpb + 3 + (int)((33 - (R2 * wpb + 3) % 32) % 32);  // P % 32 == 1, >= 3 pad words
      for (int C = env_copies > 0 ? env_copies : (attr ? 4 : 1); C >= 1; C >>= 1) {
        const size_t bins_w = (size_t)W.nw * 512 + 32 * (attr ? 12 : 4) + ((((size_t)C * P * 4) + 15) & ~(size_t)15) +
                              (attr ? (size_t)R2 * 8 : 0);
        const size_t need = (size_t)W.nw * W.nst * W.ppt * 32 * pt_bytes + bins_w + summ_w;
        if (need <= RB_SMEM_BUDGET - 1024) { wci = c; smem = need; a.hcopies = C; a.hstride = P; break; }
      }
    }
    if (wci >= 0) {
      e = RB_DISPATCH_LAY(warp_dispatch, wci, a, smem, s, &blocks, false);
      if (e) return cuda_fail(e, "k_point_pass_ring setup");
      if (blocks <= 0) wci = -1;
    }
  }
  if (wci >= 0) {
    static int env_ablate = -1;
    if (env_ablate < 0) {
      const char* e = getenv("RB_ABLATE");
      env_ablate = e ? atoi(e) : 0;
    }
    a.ablate = env_ablate;
    {
      const char* e = getenv("RB_FOLD");  // read per call: tests shorten the drain period
      a.fold = e ? atoi(e) : 0;
    }
    void* scratch = nullptr;
    const size_t rows = (size_t)blocks * R2;
    RB_CUDA(pool_alloc(&scratch, rows * 20 + 16, s));
    a.part_acc = (long long*)scratch;
    a.part_sum = (double*)((char*)scratch + rows * 8);
    a.part_cnt = (uint32_t*)((char*)scratch + rows * 16);
    int* scale = (int*)((char*)scratch + rows * 20);
    a.scale_exp = scale;  // written by the ring kernel (CTA 0) for k_reduce_fixed
    if (tstart()) return RB_CUDA_ERROR;
    e = RB_DISPATCH_LAY(warp_dispatch, wci, a, smem, s, &blocks, true);
    if (e) return cuda_fail(e, "k_point_pass_ring");
    if (tstop()) return RB_CUDA_ERROR;
    k_reduce_fixed<<<std::max(1, (R2 + 31) / 32), 1024, 0, s>>>(a.part_cnt, a.part_acc, a.part_sum, blocks, R2,
                                                                attr != nullptr, true, scale, cnt_out, sum_out);
    RB_CUDA(cudaGetLastError());
    ++g_launches;
    RB_CUDA(cudaFreeAsync(scratch, s));
    return RB_OK;
  }
  // deep-index ring: region sets beyond shared memory, node levels spread over the pipeline
  int dci = -1;
  bool nodes32 = true;
  for (const auto& nb : A->node_bufs) nodes32 = nodes32 && (int64_t)(nb.bytes / 4) < (int64_t(1) << 32);
  const bool deep_shape = keys || packed || (a.V.nlev >= 1 && L - a.V.T0 <= 16 && nodes32);
  if (g_kernel_sel != 0 && aligned && !smem_hist && L <= 20 && deep_shape && g_kernel_sel != 3 && g_kernel_sel != 4) {
    static int env_dci = -2, env_dc = -2;
    if (env_dci == -2) {
      const char* e = getenv("RB_DEEP_CFG");
      env_dci = e ? atoi(e) : -1;
      e = getenv("RB_DEEP_COPIES");
      env_dc = e ? atoi(e) : -1;
    }
    const size_t summ_w = A->S >= 0 ? ((size_t)2 << (2 * A->S)) : 16;
    const int ncfg = (int)(sizeof(kDeepCfgs) / sizeof(kDeepCfgs[0]));
    const int wpb = attr ? 3 : 1;
    const int NH = A->n_hot;
    const int P = NH * wpb + 3 + (int)((33 - (NH * wpb + 3) % 32) % 32);  // P % 32 == 1, >= 3 pad words
    for (int c = 0; c < ncfg && dci < 0; ++c) {
      if (env_dci >= 0 && c != env_dci) continue;
      if (lay != 0 && c != 0) continue;  // the KEYS / PK variants exist for the default shape only
      const WarpCfg& W = kDeepCfgs[c];
      for (int C = env_dc > 0 ? env_dc : 1; C >= 1; C >>= 1) {  // one copy: the L1 is worth more (root table)
        const size_t need = (size_t)W.nw * W.nst * W.ppt * 32 * pt_bytes + (size_t)W.nw * 512 + 32 * (attr ? 12 : 4) +
                            ((((size_t)C * P * 4) + 15) & ~(size_t)15) + summ_w;
        if (need <= RB_SMEM_BUDGET - 1024) { dci = c; smem = need; a.hcopies = C; a.hstride = P; break; }
      }
    }
    if (dci >= 0) {
      e = RB_DISPATCH_LAY(deep_dispatch, dci, a, smem, s, &blocks, false);
      if (e) return cuda_fail(e, "k_point_pass_deep setup");
      if (blocks <= 0) dci = -1;
    }
  }
  if (dci >= 0) {
    {
      const char* e = getenv("RB_FOLD");
      a.fold = e ? atoi(e) : 0;
    }
    void* scratch = nullptr;
    const size_t rows = (size_t)blocks * std::max(A->n_hot, 1);
    RB_CUDA(pool_alloc(&scratch, rows * 8 + 16, s));
    a.part_acc = (long long*)scratch;
    if (tstart()) return RB_CUDA_ERROR;
    e = RB_DISPATCH_LAY(deep_dispatch, dci, a, smem, s, &blocks, true);
    if (e) return cuda_fail(e, "k_point_pass_deep");
    if (tstop()) return RB_CUDA_ERROR;
    RB_CUDA(cudaFreeAsync(scratch, s));
    return RB_OK;
  }
  if ((!smem_hist && !use_tma) || packed) {  // keys / packed layout whose ring and deep kernels did not fit: global histogram
    if (tstart()) return RB_CUDA_ERROR;
    e = dtype == RB_XY_F64 ? launch_a<0, false>(a, vec, g_num_sms * 4, 0, s) : launch_a<1, false>(a, vec, g_num_sms * 4, 0, s);
    if (e) return cuda_fail(e, "k_point_pass_global");
    return tstop();
  }
  if (use_tma) {
    smem = ring + (smem_hist ? all_bins : hot_bins) + summ_bytes;
    e = smem_hist ? RB_DISPATCH_TMA(tma_blocks, false, smem, &blocks) : RB_DISPATCH_TMA(tma_blocks, true, smem, &blocks);
  } else {
    smem = (size_t)R2 * (attr ? 28 : 4);
    e = RB_DISPATCH_SYNC(launch_smem, a, smem, s, &blocks);
  }
  if (e) return cuda_fail(e, "k_point_pass setup");
  // scratch: per-CTA rows (smem mode: all bins; global mode: hot fixed-point accumulators) + scale
  void* scratch = nullptr;
  const size_t rows = smem_hist ? (size_t)blocks * R2 : (size_t)blocks * std::max(A->n_hot, 1);
  const size_t sbytes = smem_hist ? rows * (4 + 8 + 8) + 16 : rows * 8 + 16;
  RB_CUDA(pool_alloc(&scratch, sbytes, s));
  a.part_acc = (long long*)scratch;
  a.part_sum = smem_hist ? (double*)((char*)scratch + rows * 8) : nullptr;
  a.part_cnt = smem_hist ? (uint32_t*)((char*)scratch + rows * 16) : nullptr;
  int* scale = (int*)((char*)scratch + (smem_hist ? rows * 20 : rows * 8));
  a.scale_exp = scale;
  if (attr) {
    k_attr_scale<<<1, 1024, 0, s>>>(attr, n, scale);
    RB_CUDA(cudaGetLastError());
    ++g_launches;
  }
  if (tstart()) return RB_CUDA_ERROR;
  if (use_tma) e = smem_hist ? RB_DISPATCH_TMA(tma_run, false, a, blocks, smem, s) : RB_DISPATCH_TMA(tma_run, true, a, blocks, smem, s);
  else e = RB_DISPATCH_SYNC(run_smem, a, blocks, smem, s);
  if (e) return cuda_fail(e, "k_point_pass");
  if (tstop()) return RB_CUDA_ERROR;
  if (smem_hist) {
    k_reduce_fixed<<<std::max(1, (R2 + 31) / 32), 1024, 0, s>>>(a.part_cnt, a.part_acc, a.part_sum, blocks, R2,
                                                                attr != nullptr, false, scale, cnt_out, sum_out);
    RB_CUDA(cudaGetLastError());
    ++g_launches;
  }
  RB_CUDA(cudaFreeAsync(scratch, s));
  return RB_OK;
}
#undef RB_DISPATCH_TMA
#undef RB_DISPATCH_SYNC
#undef RB_DISPATCH_LAY

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
    const uint32_t v = index_lookup(V, (uint32_t)fx, (uint32_t)fy);
    out[i] = (v & RB_VALUE_LIST) ? v : (v & V.code_mask);  // public encoding (no hot annotation)
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
