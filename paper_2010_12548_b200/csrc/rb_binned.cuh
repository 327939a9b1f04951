// Partitioned point pass for region sets beyond shared memory on the radix
// table (C4: 40,000 regions, L = 18).  Included by rb_point_pass.cu (shares
// PassArgs and the device helpers there).
//
// Why: the one-pass deep kernel (k_point_pass_deep) makes every point's root
// lookup a random global request and every cold-region point two random global
// REDs; at the measured request rate of an SM that is its ceiling, not HBM.
// Here the points are first grouped by a coarse cell (a "bin", level BL =
// T0 - 6: 64 x 64 root slots, 16 KB), so the second pass finds each bin's
// root slots in shared memory and accumulates its few hundred regions in a
// shared hash table; only the points of mixed root cells read index nodes.
//
//   pass 1  k_bin_scatter   stream the points (12 B/pt for f32 + attribute), quantise exactly as the
//                           one-pass kernels do, count-sort each 4096-point tile by bin in shared memory
//                           and append each bin's run to this CTA's open 256-record chunk of that bin
//                           (u32 leaf code within the bin + f32 attribute: 8 B/pt written)
//   plan    k_chunk_count / k_bin_plan / k_chunk_scatter: chunk ids grouped by bin, join items of
//                           <= 1024 chunks of one bin
//   pass 2  k_bin_join      per item: the bin's root slots into shared memory, each warp streams its
//                           chunks through a private cp.async.bulk ring, node levels pipelined as in the
//                           deep kernel, interior single owners into the shared hash table (count +
//                           16-bit-split fixed point, 4 copies), the rest (owner lists, boundary leaves,
//                           out-of-window attributes) through exact global REDs; the table is flushed
//                           into the outputs at the end of the item.
//
// Measured (B200, C4 at 100M points, ncu launch times): pass 1 1.84 ms, plan 0.08 ms, pass 2 1.21 ms
// against 0.83 ms for k_point_pass_deep (profiles/round2/binned_experiment.txt).  At the HBM rate the ring
// kernel sustains (4.8 TB/s) the two passes' 28 B/pt would take 0.58 ms per 100M points (1.4x), but only
// if both ran near that rate: pass 2 streams 8 B/pt, so it would have to spend <= ~40 instructions per point
// at the achieved IPC, against 147 in the one-pass kernel; the first cut spends 175 (pass 1: plus a global
// chunk-allocation atomic per tile) and 210 (pass 2: a shared hash probe per point).  It stays an opt-in
// experiment (RB_BINNED=1), parity-tested; the one-pass deep kernel remains the C4 path.
//
// The index, the quantisation and the owner semantics are those of the one-pass kernels, so COUNT is
// bit-identical; SUM has the fixed-point error bound of the hot slots (DESIGN.md SUM numerics) for
// every in-window interior point.
// Bounds: a chunk holds 256 records; pass 1 has at most one partly filled chunk per (CTA, covered bin),
// so ceil(n / 256) + CTAs * covered bins chunks always suffice.  An item holds <= 1024 chunks (262,144
// points); copy c of a hash slot receives exactly a quarter of them (lane & 3), so the low halves stay
// below 65,536 * 65,535 < 2^32 and the high halves within 65,536 * 2^14 = 2^30 without drains.

namespace binned {
constexpr int CH = 256;                           // records per chunk
constexpr int BLMAX = 6;                          // bins: level <= 6 (<= 4096)
constexpr int NBMAX = 1 << (2 * BLMAX);
constexpr int SWB_MAX = 6;                        // a bin's slice of the root: <= 64 x 64 slots
constexpr int P1_NT = 512, P1_PPT = 8, P1_TILE = P1_NT * P1_PPT;
constexpr int ITEM_CH = 1024;                     // chunks per join item
constexpr int HTB = 9, HT = 1 << HTB;             // hash slots per item (regions of one bin)
constexpr int HC = 4;                             // accumulator copies
constexpr int HP = HT * 3 + 1;                    // words per copy (== 1 mod 32)
constexpr int NW2 = 8, PPT2 = 4, NST2 = 4, WT2 = PPT2 * 32;
constexpr uint32_t NONE = 0xffffffffu;
static_assert(CH == 2 * WT2, "a chunk is two warp groups");
static_assert(HP % 32 == 1, "hash copies in distinct banks");
}  // namespace binned

struct BinArgs {
  PassArgs a;
  int BL;                 // bin level
  int swb;                // log2 of the slice side (T0 - BL)
  uint32_t cap;           // chunk capacity
  uint32_t* rc;           // record leaf codes [cap * CH]: (x & m) | (y & m) << 16 within the bin
  float* ra;              // record attributes [cap * CH]
  uint32_t* cbin;         // chunk -> bin
  uint32_t* ccnt;         // chunk -> records
  uint32_t* ctr;          // [0] chunks allocated, [1] join items, [2] next item, [3] capacity overflow
  const uint8_t* bflags;  // bin covered by the index
  uint32_t* bin_nch;      // chunks per bin
  uint32_t* bin_off;      // first position of each bin in `sorted` [NB + 1]
  uint32_t* bin_cur;
  uint32_t* sorted;       // chunk ids grouped by bin
  uint32_t* item_bin;
  uint32_t* item_start;
  uint32_t* item_nch;
};

__global__ void k_bin_flags(const uint32_t* __restrict__ root, int T0, int BL, int64_t nroot, uint8_t* flags) {
  const int sw = T0 - BL;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nroot; s += (int64_t)gridDim.x * blockDim.x) {
    if (!root[s]) continue;
    const uint32_t row = (uint32_t)(s >> T0), col = (uint32_t)(s & ((1ll << T0) - 1));
    flags[((row >> sw) << BL) | (col >> sw)] = 1;
  }
}

// ---- pass 1: quantise, count-sort by bin per tile, append runs to per-CTA open chunks
template <int XY, bool ATTR>
__global__ void __launch_bounds__(binned::P1_NT, 2) k_bin_scatter(BinArgs b) {
  using namespace binned;
  extern __shared__ __align__(128) unsigned char sm[];
  const int NB = 1 << (2 * b.BL);
  uint32_t* hc = (uint32_t*)sm;          // [NB + 1]: tile counts, then exclusive offsets (hc[NB] = tile total)
  uint32_t* scur = hc + NBMAX + 4;       // open chunk per bin (NONE: none yet)
  uint32_t* sfill = scur + NBMAX;        // records in it
  uint32_t* sbase = sfill + NBMAX;       // first chunk allocated for this tile's run
  uint32_t* scode = sbase + NBMAX;       // tile records sorted by bin
  float* sattr = (float*)(scode + P1_TILE);
  uint16_t* sbin = (uint16_t*)(sattr + P1_TILE);
  uint8_t* sflag = (uint8_t*)(sbin + P1_TILE);
  __shared__ uint32_t wtot[P1_NT / 32];
  constexpr int BPT = NBMAX / P1_NT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < NB; i += P1_NT) {
    hc[i] = 0;
    scur[i] = NONE;
    sfill[i] = 0;
    sflag[i] = b.bflags[i];
  }
  if (tid == 0) hc[NB] = 0;
  __syncthreads();  // sflag is read by the first tile's quantisation
  const PassArgs& a = b.a;
  const double ox = a.ox, oy = a.oy, inv_side = a.inv_side;
  const int L = a.V.L, sb = L - b.BL;
  const uint32_t lm = (1u << sb) - 1u, hibits = ~((1u << L) - 1u);
  const int64_t ntiles = (a.n + P1_TILE - 1) / P1_TILE;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t p0 = t * P1_TILE + (int64_t)tid * P1_PPT;
    float fxv[XY == 1 ? 2 * P1_PPT : 1];
    double dxv[XY == 0 ? 2 * P1_PPT : 1];
    float w[P1_PPT];
    const bool full = p0 + P1_PPT <= a.n;
    if (full) {
      if constexpr (XY == 1) {
        const float4* src = (const float4*)((const float*)a.xy + 2 * p0);
#pragma unroll
        for (int q = 0; q < P1_PPT / 2; ++q) {
          const float4 v = __ldcs(src + q);
          fxv[4 * q] = v.x; fxv[4 * q + 1] = v.y; fxv[4 * q + 2] = v.z; fxv[4 * q + 3] = v.w;
        }
      } else {
        const double2* src = (const double2*)a.xy + p0;
#pragma unroll
        for (int q = 0; q < P1_PPT; ++q) {
          const double2 v = __ldcs(src + q);
          dxv[2 * q] = v.x; dxv[2 * q + 1] = v.y;
        }
      }
      if (ATTR) {
        const float4* s4 = (const float4*)(a.attr + p0);
#pragma unroll
        for (int q = 0; q < P1_PPT / 4; ++q) {
          const float4 v = __ldcs(s4 + q);
          w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < P1_PPT; ++j) {
        const bool in = p0 + j < a.n;
        if constexpr (XY == 1) {
          fxv[2 * j] = in ? ((const float*)a.xy)[2 * (p0 + j)] : 0.f;
          fxv[2 * j + 1] = in ? ((const float*)a.xy)[2 * (p0 + j) + 1] : 0.f;
        } else {
          dxv[2 * j] = in ? ((const double*)a.xy)[2 * (p0 + j)] : 0.0;
          dxv[2 * j + 1] = in ? ((const double*)a.xy)[2 * (p0 + j) + 1] : 0.0;
        }
        w[j] = (ATTR && in) ? a.attr[p0 + j] : 0.f;
      }
    }
    // quantisation: the one-pass kernels' fast path, the exact division where it is not conclusive
    uint32_t bn[P1_PPT], cd[P1_PPT];
#pragma unroll
    for (int j = 0; j < P1_PPT; ++j) {
      const double x = XY == 1 ? (double)fxv[2 * j] : dxv[2 * j];
      const double y = XY == 1 ? (double)fxv[2 * j + 1] : dxv[2 * j + 1];
      const double tx = __fma_rn(__dsub_rn(x, ox), inv_side, 1048576.0);
      const double ty = __fma_rn(__dsub_rn(y, oy), inv_side, 1048576.0);
      uint32_t bx = (uint32_t)__double2hiint(tx) - 0x41300000u;
      uint32_t by = (uint32_t)__double2hiint(ty) - 0x41300000u;
      const uint32_t fx = (uint32_t)__double2loint(tx) + 8u, fy = (uint32_t)__double2loint(ty) + 8u;
      const bool bad = (((bx | by) & hibits) != 0u) | (fx < 16u) | (fy < 16u);
      bool live = full || p0 + j < a.n;
      if (live && bad) {
        const uint64_t qq = quantize_exact(a.xy, p0 + j, XY, ox, oy, a.side, a.lim, a.first_bad, a.idx_base);
        if (qq == ~0ull) live = false;
        else { bx = (uint32_t)qq; by = (uint32_t)(qq >> 32); }
      }
      const uint32_t bin = live ? (((by >> sb) << b.BL) | (bx >> sb)) : 0u;
      bn[j] = (live && sflag[bin]) ? bin : NONE;  // uncovered bins: no owner, nothing to add
      cd[j] = (bx & lm) | ((by & lm) << 16);
    }
    __syncthreads();  // the previous tile's reset of hc is complete
    uint32_t rk[P1_PPT];
#pragma unroll
    for (int j = 0; j < P1_PPT; ++j) rk[j] = bn[j] != NONE ? atomicAdd(&hc[bn[j]], 1u) : 0u;
    __syncthreads();
    // exclusive offsets over the bins; chunks for runs that overflow the open chunk
    const int i0 = tid * BPT;
    uint32_t cnt[BPT], s = 0;
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      cnt[k] = i0 + k < NB ? hc[i0 + k] : 0u;
      s += cnt[k];
    }
    uint32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    if (lane == 31) wtot[warp] = inc;
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      if (!cnt[k]) continue;
      const int i = i0 + k;
      const uint32_t cur = scur[i], f = sfill[i];
      const uint32_t space = cur == NONE ? 0u : (uint32_t)CH - f;
      if (cnt[k] > space) {
        const uint32_t need = (cnt[k] - space + CH - 1) / CH;
        uint32_t base = atomicAdd(&b.ctr[0], need);
        if ((uint64_t)base + need > b.cap) {
          atomicOr(&b.ctr[3], 1u);  // cannot happen: the capacity bound above
          base = NONE;
        } else {
          for (uint32_t q = 0; q < need; ++q) { b.cbin[base + q] = (uint32_t)i; b.ccnt[base + q] = CH; }
        }
        sbase[i] = base;
      }
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t v = lane < P1_NT / 32 ? wtot[lane] : 0u;
      uint32_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane < P1_NT / 32) wtot[lane] = x - v;
    }
    __syncthreads();
    {
      uint32_t ex = inc - s + wtot[warp];
#pragma unroll
      for (int k = 0; k < BPT; ++k) {
        if (i0 + k < NB) hc[i0 + k] = ex;
        ex += cnt[k];
      }
      if (tid == P1_NT - 1) hc[NB] = ex;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < P1_PPT; ++j) {
      if (bn[j] == NONE) continue;
      const uint32_t pos = hc[bn[j]] + rk[j];
      scode[pos] = cd[j];
      if (ATTR) sattr[pos] = w[j];
      sbin[pos] = (uint16_t)bn[j];
    }
    __syncthreads();
    const uint32_t total = hc[NB];
    for (uint32_t i = tid; i < total; i += P1_NT) {  // runs of one bin are consecutive: coalesced stores
      const uint32_t bb = sbin[i], ri = i - hc[bb], cur = scur[bb], f = sfill[bb];
      const uint32_t space = cur == NONE ? 0u : (uint32_t)CH - f;
      size_t dst;
      if (ri < space) dst = (size_t)cur * CH + f + ri;
      else if (sbase[bb] != NONE) dst = (size_t)sbase[bb] * CH + (ri - space);
      else continue;
      b.rc[dst] = scode[i];
      if (ATTR) b.ra[dst] = sattr[i];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      const int i = i0 + k;
      if (i >= NB) continue;
      hc[i] = 0;
      if (!cnt[k]) continue;
      const uint32_t cur = scur[i], f = sfill[i];
      const uint32_t space = cur == NONE ? 0u : (uint32_t)CH - f;
      if (cnt[k] <= space) {
        sfill[i] = f + cnt[k];
      } else if (sbase[i] == NONE) {
        scur[i] = NONE;
        sfill[i] = 0;
      } else {
        const uint32_t rem = cnt[k] - space, need = (rem + CH - 1) / CH;
        scur[i] = sbase[i] + need - 1;
        sfill[i] = rem - (need - 1) * CH;
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < NB; i += P1_NT)
    if (scur[i] != NONE) b.ccnt[scur[i]] = sfill[i];
}

// ---- plan: chunks grouped by bin, join items
__global__ void k_chunk_count(BinArgs b) {
  const uint32_t n = b.ctr[0];
  for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id < n; id += gridDim.x * blockDim.x)
    atomicAdd(&b.bin_nch[b.cbin[id]], 1u);
}

__global__ void __launch_bounds__(1024) k_bin_plan(BinArgs b, int NB) {
  using namespace binned;
  constexpr int BPT = NBMAX / 1024;
  __shared__ uint32_t wc[32], wi[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i0 = tid * BPT;
  uint32_t nch[BPT], sc = 0, si = 0;
#pragma unroll
  for (int k = 0; k < BPT; ++k) {
    nch[k] = i0 + k < NB ? b.bin_nch[i0 + k] : 0u;
    sc += nch[k];
    si += (nch[k] + ITEM_CH - 1) / ITEM_CH;
  }
  uint32_t ic = sc, ii = si;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, ic, o), v = __shfl_up_sync(0xffffffffu, ii, o);
    if (lane >= o) { ic += u; ii += v; }
  }
  if (lane == 31) { wc[warp] = ic; wi[warp] = ii; }
  __syncthreads();
  if (warp == 0) {
    const uint32_t u = wc[lane], v = wi[lane];
    uint32_t x = u, y = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t p = __shfl_up_sync(0xffffffffu, x, o), q = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) { x += p; y += q; }
    }
    wc[lane] = x - u;
    wi[lane] = y - v;
    if (lane == 31) { b.ctr[1] = y; b.ctr[2] = 0; b.bin_off[NB] = x; }
  }
  __syncthreads();
  uint32_t oc = ic - sc + wc[warp], oi = ii - si + wi[warp];
#pragma unroll
  for (int k = 0; k < BPT; ++k) {
    if (i0 + k >= NB) break;
    b.bin_off[i0 + k] = oc;
    for (uint32_t q = 0; q * ITEM_CH < nch[k]; ++q, ++oi) {
      b.item_bin[oi] = (uint32_t)(i0 + k);
      b.item_start[oi] = oc + q * ITEM_CH;
      b.item_nch[oi] = min((uint32_t)ITEM_CH, nch[k] - q * ITEM_CH);
    }
    oc += nch[k];
  }
}

__global__ void k_chunk_scatter(BinArgs b) {
  const uint32_t n = b.ctr[0];
  for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id < n; id += gridDim.x * blockDim.x) {
    const uint32_t bb = b.cbin[id];
    b.sorted[b.bin_off[bb] + atomicAdd(&b.bin_cur[bb], 1u)] = id;
  }
}

// slot of region r in the item's hash table (inserted on first use); NONE after 8 probes
__device__ __forceinline__ uint32_t bin_hash_slot(uint32_t* hkey, uint32_t r) {
  using namespace binned;
  uint32_t h = (r * 0x9E3779B1u) >> (32 - HTB);
#pragma unroll 1
  for (int p = 0; p < 8; ++p) {
    uint32_t k = *(volatile uint32_t*)&hkey[h];
    if (k == r) return h;
    if (k == NONE) {
      k = atomicCAS(&hkey[h], NONE, r);
      if (k == NONE || k == r) return h;
    }
    h = (h + 1) & (HT - 1);
  }
  return NONE;
}

// ---- pass 2: per item (one bin), slice lookups in shared memory, shared hash accumulation
template <bool ATTR>
__global__ void __launch_bounds__(binned::NW2 * 32, 2) k_bin_join(BinArgs b) {
  using namespace binned;
  constexpr int NT = NW2 * 32, WT = WT2, PPT = PPT2;
  constexpr uint32_t RS = WT * (ATTR ? 2 : 1);  // words per ring stage
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t mb[NW2 * NST2];
  __shared__ uint32_t s_item;
  __shared__ float smax[NW2];
  const PassArgs& a = b.a;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* ring = (uint32_t*)sm;
  uint32_t* wring = ring + (size_t)warp * NST2 * RS;
  uint32_t* slice = ring + (size_t)NW2 * NST2 * RS;
  uint32_t* ilist = slice + (1 << (2 * SWB_MAX));
  uint32_t* icnt = ilist + ITEM_CH;
  uint32_t* hkey = icnt + ITEM_CH;
  uint32_t* hacc = hkey + HT;
  unsigned char* dummy = (unsigned char*)(hacc + HC * HP);
  uint2* rq = (uint2*)(dummy + 32 * 12) + (size_t)warp * 64;
  for (int q = tid; q < HT; q += NT) hkey[q] = NONE;
  for (int q = tid; q < HC * HP; q += NT) hacc[q] = 0;
  if (tid < NW2 * NST2) mbar_init(&mb[tid], 1);
  if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  // fixed-point scale from the same strided attribute sample as the one-pass kernels
  float sc = 1.f;
  uint32_t wminb = 0, wspan = 0;
  int Sx = 0;
  if (ATTR) {
    float mx = 0.f;
    const int64_t stride = a.n / 4096 > 0 ? a.n / 4096 : 1;
    for (int q = tid; q < 4096; q += NT) {
      const float v = (q * stride < a.n) ? fabsf(__ldg(a.attr + q * stride)) : 0.f;
      if (isfinite(v)) mx = fmaxf(mx, v);
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) smax[warp] = mx;
    __syncthreads();
    mx = 0.f;
    for (int w2 = 0; w2 < NW2; ++w2) mx = fmaxf(mx, smax[w2]);
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
  __syncthreads();
  const uint32_t* __restrict__ root = a.V.root;
  const uint32_t* __restrict__ pool = a.V.pool;
  const uint32_t* __restrict__ nodes0 = a.V.nodes[0];
  const uint32_t* __restrict__ nodes1 = a.V.nodes[a.V.nlev > 1 ? 1 : 0];
  const int L = a.V.L, T0 = a.V.T0, s0 = L - T0, nlev = a.V.nlev, SWB = b.swb;
  const int k0 = nlev > 0 ? a.V.ks[0] : 0, s1 = s0 - k0, k1 = nlev > 1 ? a.V.ks[1] : 0, s2 = s1 - k1;
  const uint32_t m0 = (1u << s0) - 1u, mk0 = (1u << k0) - 1u, mk1 = (1u << k1) - 1u;
  const uint32_t cmask = a.V.code_mask;
  const uint32_t hbase = smem_u32(hacc) + (uint32_t)((lane & (HC - 1)) * HP) * 4u;
  const uint32_t dms = smem_u32(dummy) + lane * 12u;
  const uint32_t mb0 = smem_u32(&mb[warp * NST2]);
  unsigned long long* gcnt = a.gcnt;
  double* gsum = a.gsum;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  int qh = 0, qn = 0;
  auto rare_flush = [&](int nitems) {  // owner lists, boundary leaves, out-of-window attributes: exact REDs
    if (lane < nitems) {
      const uint2 it = rq[(qh + lane) & 63];
      add_owners_g<ATTR>(0u, pool, it.x, __uint_as_float(it.y), 0, false, gcnt, gsum, cmask, a.V.hot_shift);
    }
    __syncwarp();
  };
  uint32_t seq = 0;  // groups this warp has consumed (ring stage = seq % NST2, parity = (seq / NST2) & 1)
  const int nbs = 1 << b.BL;
  for (;;) {
    if (tid == 0) s_item = atomicAdd(&b.ctr[2], 1u);
    __syncthreads();
    const uint32_t it = s_item;
    if (it >= b.ctr[1]) break;
    const uint32_t bin = b.item_bin[it], cs = b.item_start[it], nch = b.item_nch[it];
    {
      const uint32_t bx0 = (bin & (nbs - 1)) << SWB, by0 = (bin >> b.BL) << SWB;
      const int SW = 1 << SWB;
      for (int q = tid; q < SW * SW; q += NT)
        slice[q] = __ldg(root + ((size_t)(by0 + (q >> SWB)) << T0) + bx0 + (q & (SW - 1)));
      for (uint32_t q = tid; q < nch; q += NT) {
        const uint32_t id = b.sorted[cs + q];
        ilist[q] = id;
        icnt[q] = b.ccnt[id];
      }
    }
    __syncthreads();
    const uint32_t ng = 2 * nch;
    const int K = ng > (uint32_t)warp ? (int)((ng - 1 - warp) / NW2) + 1 : 0;
    auto issue = [&](int kk) {  // lane 0: group kk of this warp into its ring stage
      const uint32_t g = warp + NW2 * kk, ci = g >> 1, half = g & 1u;
      const uint32_t id = ilist[ci], cnt = icnt[ci];
      const uint32_t valid = cnt > half * WT ? min((uint32_t)WT, cnt - half * WT) : 0u;
      uint32_t bytes = (valid * 4u + 15u) & ~15u;
      if (!bytes) bytes = 16u;
      const uint32_t stg = (seq + kk) % NST2;
      uint32_t* dst = wring + stg * RS;
      const size_t off = (size_t)id * CH + half * WT;
      mbar_expect_tx(&mb[warp * NST2 + stg], bytes * (ATTR ? 2u : 1u));
      bulk_g2s(dst, b.rc + off, bytes, &mb[warp * NST2 + stg], pol);
      if (ATTR) bulk_g2s(dst + WT, b.ra + off, bytes, &mb[warp * NST2 + stg], pol);
    };
    if (lane == 0)
      for (int kk = 0; kk < K && kk < NST2; ++kk) issue(kk);
    __syncwarp();
    uint32_t rv[PPT], c1[PPT], c2[PPT], nv1[PPT], nv2[PPT];
    float w1[PPT], w2[PPT], w3[PPT];
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      rv[j] = c1[j] = c2[j] = nv1[j] = nv2[j] = 0u;
      w1[j] = w2[j] = w3[j] = 0.f;
    }
    for (int k = 0; k < K + 3; ++k) {
      // ---------------------------------------------------------- C(k-3): accumulate
      if (k >= 3) {
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
          const bool single = ((v & (RB_VALUE_LIST | 1u)) == 1u) & fast;
          const uint32_t r = ((v & cmask) - 1u) >> 1;
          const uint32_t slot = single ? bin_hash_slot(hkey, r) : NONE;
          const uint32_t ad = slot != NONE ? hbase + slot * 12u : dms;
          reds(ad, 1u);
          if (ATTR) {
            reds(ad + 4, (uint32_t)qv & 0xffffu);
            reds(ad + 8, (uint32_t)(qv >> 16));
          }
          if (single && slot == NONE) {  // table full (> 512 regions in a bin): exact global REDs
            atomicAdd(&gcnt[2 * r], 1ull);
            if (ATTR) atomicAdd(&gsum[2 * r], (double)w3[j]);
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
      }
      // ---------------------------------------------------------- B2(k-2): node levels 1..
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
          if (nlev > 2) {
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
      // ---------------------------------------------------------- B1(k-1): node level 0
      if (k >= 1 && k <= K) {
#pragma unroll
        for (int j = 0; j < PPT; ++j) { w2[j] = w1[j]; c2[j] = c1[j]; }
        uint32_t anyn = 0;
#pragma unroll
        for (int j = 0; j < PPT; ++j) anyn |= rv[j];
        if (nlev > 0 && __any_sync(0xffffffffu, (int32_t)anyn < 0)) {
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
      // ---------------------------------------------------------- A(k): records -> root slot (shared)
      if (k < K) {
        const uint32_t sq = seq + k, stg = sq % NST2;
        mbar_wait_warp_a(mb0 + 8u * stg, (sq / NST2) & 1u);
        const uint32_t* src = wring + stg * RS;
        const uint32_t g = warp + NW2 * k, cnt = icnt[g >> 1], lo = (g & 1u) * WT;
        const int valid = (int)cnt - (int)lo;
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          const int pi = lane + 32 * j;
          const uint32_t code = src[pi];
          w1[j] = ATTR ? __uint_as_float(src[WT + pi]) : 0.f;
          const uint32_t lx = code & 0xffffu, ly = code >> 16;
          rv[j] = pi < valid ? slice[((ly >> s0) << SWB) | (lx >> s0)] : 0u;
          c1[j] = (lx & m0) | ((ly & m0) << 16);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0 && k + NST2 < K) issue(k + NST2);
      }
    }
    __syncwarp();
    if (qn) {
      rare_flush(qn);
      qh = (qh + qn) & 63;
      qn = 0;
    }
    seq += (uint32_t)K;
    __syncthreads();
    for (int h = tid; h < HT; h += NT) {  // the item's regions into the outputs (alpha bins)
      const uint32_t r = hkey[h];
      if (r == NONE) continue;
      uint32_t cnt = 0;
      long long f = 0;
#pragma unroll
      for (int c = 0; c < HC; ++c) {
        uint32_t* e = hacc + c * HP + 3 * h;
        cnt += e[0];
        if (ATTR) f += ((long long)(int32_t)e[2] << 16) + (long long)e[1];
        e[0] = 0; e[1] = 0; e[2] = 0;
      }
      hkey[h] = NONE;
      if (cnt) atomicAdd(&gcnt[2 * r], (unsigned long long)cnt);
      if (ATTR && f) atomicAdd(&gsum[2 * r], ldexp((double)f, -Sx));
    }
  }
}


// bins of the partitioned pass for this index, or -1 (layout / level shape it does not cover)
static int binned_level(const rb_approx* A) {
  const int L = A->grid.max_level, T0 = A->T0;
  if (A->keys.p || A->pblk.p || L > 20 || T0 > 12) return -1;
  const int BL = std::max(0, T0 - binned::SWB_MAX);
  if (L - BL > 16) return -1;
  for (const auto& nb : A->node_bufs)
    if ((int64_t)(nb.bytes / 4) >= (int64_t(1) << 32)) return -1;
  return BL;
}

static bool binned_wanted(const rb_approx* A, int64_t n, bool aligned, bool smem_hist) {
  // RB_BINNED=1: whenever the index shape allows (read per call: tests and tools switch it).  Off by default:
  // on C4 it is slower than the one-pass kernel (see the header comment)
  (void)n;
  (void)smem_hist;
  const char* e = getenv("RB_BINNED");
  return e && atoi(e) == 1 && aligned && binned_level(A) >= 0;
}

static int binned_flags(rb_approx* A, int BL, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(A->bin_mu);
  if (A->bin_level == BL) return RB_OK;
  const int NB = 1 << (2 * BL);
  RB_CUDA(A->bin_flags.alloc_persistent(NB));
  RB_CUDA(cudaMemsetAsync(A->bin_flags.p, 0, NB, s));
  const int64_t nroot = (int64_t)1 << (2 * A->T0);
  k_bin_flags<<<(int)std::min<int64_t>((nroot + 255) / 256, 148 * 16), 256, 0, s>>>(A->root.as<uint32_t>(), A->T0, BL,
                                                                                     nroot, A->bin_flags.as<uint8_t>());
  RB_CUDA(cudaGetLastError());
  std::vector<uint8_t> h(NB);
  RB_CUDA(cudaMemcpyAsync(h.data(), A->bin_flags.p, NB, cudaMemcpyDeviceToHost, s));
  RB_CUDA(cudaStreamSynchronize(s));
  int used = 0;
  for (uint8_t f : h) used += f != 0;
  A->bin_used = used;
  A->bin_level = BL;
  return RB_OK;
}

template <int XY, bool ATTR>
static cudaError_t binned_launch(BinArgs& b, int NB, int g1, int g2, size_t sm1, size_t sm2, int nplan, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(k_bin_scatter<XY, ATTR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
  if (e) return e;
  e = cudaFuncSetAttribute(k_bin_join<ATTR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
  if (e) return e;
  k_bin_scatter<XY, ATTR><<<g1, binned::P1_NT, sm1, s>>>(b);
  k_chunk_count<<<nplan, 256, 0, s>>>(b);
  k_bin_plan<<<1, 1024, 0, s>>>(b, NB);
  k_chunk_scatter<<<nplan, 256, 0, s>>>(b);
  k_bin_join<ATTR><<<g2, binned::NW2 * 32, sm2, s>>>(b);
  return cudaGetLastError();
}

// the partitioned pass; `a` is the one-pass kernels' argument block (outputs already initialised)
static int binned_pass(const rb_approx* Ac, const PassArgs& a, int32_t dtype, bool attr, cudaStream_t s, int* launches) {
  using namespace binned;
  rb_approx* A = const_cast<rb_approx*>(Ac);  // the bin flags are a lazily computed cache of the index
  const int BL = binned_level(A);
  if (int st = binned_flags(A, BL, s)) return st;
  const int NB = 1 << (2 * BL);
  const size_t sm1 = (size_t)(NBMAX + 4) * 4 + (size_t)3 * NBMAX * 4 + (size_t)P1_TILE * (4 + 4 + 2) + NBMAX;
  const size_t ring_w = (size_t)NW2 * NST2 * WT2 * (attr ? 2 : 1);
  const size_t sm2 = (ring_w + ((size_t)1 << (2 * SWB_MAX)) + 2 * ITEM_CH + HT + (size_t)HC * HP) * 4 + 32 * 12 +
                     (size_t)NW2 * 64 * 8;
  const int g1 = 2 * g_num_sms, g2 = 2 * g_num_sms;
  const uint64_t cap64 = (uint64_t)((a.n + CH - 1) / CH) + (uint64_t)g1 * std::max(A->bin_used, 1) + 1;
  if (cap64 >= ((uint64_t)1 << 32) / CH) return fail(RB_CAPACITY_ERROR, "partitioned pass: too many points per call");
  const uint32_t cap = (uint32_t)cap64;
  const uint32_t max_items = cap / ITEM_CH + NB + 1;
  // scratch: records, chunk tables, plan
  const size_t rec = (size_t)cap * CH;
  const size_t bytes = rec * 4 * (attr ? 2 : 1) + (size_t)cap * 12 + 64 + (size_t)NB * 12 + 4 + (size_t)max_items * 12;
  void* scratch = nullptr;
  RB_CUDA(pool_alloc(&scratch, bytes, s));
  char* p = (char*)scratch;
  BinArgs b{};
  b.a = a;
  b.BL = BL;
  b.swb = A->T0 - BL;
  b.cap = cap;
  b.rc = (uint32_t*)p; p += rec * 4;
  b.ra = attr ? (float*)p : nullptr; p += attr ? rec * 4 : 0;
  b.cbin = (uint32_t*)p; p += (size_t)cap * 4;
  b.ccnt = (uint32_t*)p; p += (size_t)cap * 4;
  b.sorted = (uint32_t*)p; p += (size_t)cap * 4;
  b.ctr = (uint32_t*)p; p += 64;
  b.bin_nch = (uint32_t*)p; p += (size_t)NB * 4;
  b.bin_cur = (uint32_t*)p; p += (size_t)NB * 4;
  b.bin_off = (uint32_t*)p; p += (size_t)NB * 4 + 4;
  b.item_bin = (uint32_t*)p; p += (size_t)max_items * 4;
  b.item_start = (uint32_t*)p; p += (size_t)max_items * 4;
  b.item_nch = (uint32_t*)p;
  b.bflags = A->bin_flags.as<uint8_t>();
  RB_CUDA(cudaMemsetAsync(b.ctr, 0, 64 + (size_t)NB * 8, s));  // ctr, bin_nch, bin_cur (contiguous)
  const int nplan = (int)std::min<uint64_t>((cap + 255) / 256, (uint64_t)g_num_sms * 8);
  const cudaError_t e = dtype == RB_XY_F64
                            ? (attr ? binned_launch<0, true>(b, NB, g1, g2, sm1, sm2, nplan, s)
                                    : binned_launch<0, false>(b, NB, g1, g2, sm1, sm2, nplan, s))
                            : (attr ? binned_launch<1, true>(b, NB, g1, g2, sm1, sm2, nplan, s)
                                    : binned_launch<1, false>(b, NB, g1, g2, sm1, sm2, nplan, s));
  if (e) return cuda_fail(e, "partitioned point pass");
  *launches += 5;
  RB_CUDA(cudaFreeAsync(scratch, s));
  return RB_OK;
}
