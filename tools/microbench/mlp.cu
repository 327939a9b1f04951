// Random-lookup throughput vs memory-level parallelism (design aid for the point
// pass's index lookups).  Every thread issues PPT random 4-byte lookups per
// iteration into a table of `mb` MB and consumes them one iteration later:
//   mode 0: ld.global.nc.u32            (L1-allocating; in-flight misses hold L1 lines)
//   mode 1: ld.global.nc.L1::no_allocate.u32
//   mode 2: cp.async.cg.shared.global 16 B (L2 only) into a per-thread shared-memory slot,
//           cp.async.commit_group / wait_group 1
//   mode 5: cp.async.bulk 16 B per lookup (the TMA unit, not the LSU), completing on a per-warp mbarrier
//   mode 6: half the lookups as mode 5, half as mode 0 (do the two request paths add up?)
// The kernel also reserves `pad` KB of shared memory to emulate the point pass's ring.
// Output: one JSON line per (table size, mode, PPT, warps, pad).
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t xs(uint32_t& s) { s ^= s << 13; s ^= s >> 17; s ^= s << 5; return s; }

template <int MODE, int PPT>
__global__ void k(const uint32_t* __restrict__ tab, uint32_t mask16, int iters, uint32_t* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint4* slot = (uint4*)sm + (size_t)threadIdx.x * PPT * 2;  // 2 stages x PPT x 16 B per thread
  uint32_t s = 0x9e3779b9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  uint32_t acc = 0;
  uint32_t v[PPT];
#pragma unroll
  for (int j = 0; j < PPT; ++j) v[j] = 0;
  __shared__ __align__(8) uint64_t bar[64];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (MODE >= 5) {
    if (lane == 0)
      for (int q = 0; q < 2; ++q)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[2 * wid + q])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
  }
  constexpr int NTMA = MODE == 5 ? PPT : PPT / 2;
  for (int it = 0; it < iters; ++it) {
    const int st = it & 1;
    if (MODE == 5 || MODE == 6) {
      const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[2 * wid + st]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(32 * NTMA * 16) : "memory");
      __syncwarp();
#pragma unroll
      for (int j = 0; j < NTMA; ++j) {
        const uint32_t q = xs(s) & mask16;
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&slot[st * PPT + j]);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(dst),
                     "l"(tab + (size_t)q * 4), "r"(b)
                     : "memory");
      }
      if (MODE == 6) {
#pragma unroll
        for (int j = NTMA; j < PPT; ++j) acc += v[j];
#pragma unroll
        for (int j = NTMA; j < PPT; ++j) {
          const uint32_t q = xs(s) & mask16;
          asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v[j]) : "l"(tab + (size_t)q * 4));
        }
      }
      if (it > 0) {
        const uint32_t bo = (uint32_t)__cvta_generic_to_shared(&bar[2 * wid + (st ^ 1)]);
        const uint32_t par = ((it - 1) >> 1) & 1;
        asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(bo),
                     "r"(par)
                     : "memory");
#pragma unroll
        for (int j = 0; j < NTMA; ++j) acc += slot[(st ^ 1) * PPT + j].x;
      }
    } else if (MODE == 2) {
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const uint32_t q = xs(s) & mask16;  // 16-byte granule
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&slot[st * PPT + j]);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(tab + (size_t)q * 4) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 1;" ::: "memory");
#pragma unroll
      for (int j = 0; j < PPT; ++j) acc += slot[(st ^ 1) * PPT + j].x;
    } else if (MODE == 3 || MODE == 4) {  // 3: random u64 REDs into an 80k x 8 B table; 4: loads + half as many REDs
      unsigned long long* red = (unsigned long long*)out + 2;
      if (MODE == 4) {
#pragma unroll
        for (int j = 0; j < PPT; ++j) acc += v[j];
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          const uint32_t q = xs(s) & mask16;
          asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v[j]) : "l"(tab + (size_t)q * 4));
        }
      }
#pragma unroll
      for (int j = 0; j < (MODE == 4 ? PPT / 2 : PPT); ++j) {
        const uint32_t r = xs(s) % 80000u;
        asm volatile("red.global.add.u64 [%0], 1;" ::"l"(red + r) : "memory");
      }
    } else {
#pragma unroll
      for (int j = 0; j < PPT; ++j) acc += v[j];
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const uint32_t q = xs(s) & mask16;
        const uint32_t* p = tab + (size_t)q * 4;
        if (MODE == 0) asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v[j]) : "l"(p));
        else asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v[j]) : "l"(p));
      }
    }
  }
  if (MODE == 2) asm volatile("cp.async.wait_group 0;" ::: "memory");
  if ((MODE == 5 || MODE == 6) && iters > 0) {  // the last stage's copies land before the CTA exits
    const int st = (iters - 1) & 1;
    const uint32_t bo = (uint32_t)__cvta_generic_to_shared(&bar[2 * wid + st]);
    const uint32_t par = ((iters - 1) >> 1) & 1;
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(bo),
                 "r"(par)
                 : "memory");
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int MODE, int PPT>
static void run(const uint32_t* tab, size_t mb, int warps, int pad_kb, int sms, int clk, uint32_t* out) {
  const int threads = warps * 32;
  const size_t smem = (size_t)threads * PPT * 32 + (size_t)pad_kb * 1024;
  if (smem > 227 * 1024 - 1024) return;
  auto kern = k<MODE, PPT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - 1024);  // static mbarriers
  const uint32_t mask16 = (uint32_t)((getenv("MLP_KB") ? (mb << 10) : (mb << 20)) / 16 - 1);  // MLP_KB: sizes in KB
  const int iters = 400;
  kern<<<sms, threads, smem>>>(tab, mask16, iters, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<sms, threads, smem>>>(tab, mask16, iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double n = (double)sms * threads * iters * (MODE == 4 ? PPT + PPT / 2 : PPT);  // global requests
  printf("{\"table_mb\":%zu,\"mode\":%d,\"ppt\":%d,\"warps\":%d,\"smem_kb\":%zu,\"err\":\"%s\",\"Glookups_s\":%.1f,"
         "\"lookups_per_sm_clk\":%.3f}\n",
         mb, MODE, PPT, warps, smem / 1024, cudaGetErrorString(cudaGetLastError()), n / ms / 1e6,
         n / (ms * 1e-3) / sms / (clk * 1e3));
  fflush(stdout);
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (const char* g = getenv("MLP_SMS")) sms = atoi(g);  // CTAs (one per SM): per-SM vs chip-wide limits
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const size_t maxmb = 4096;
  uint32_t* tab;
  uint32_t* out;
  cudaMalloc(&tab, maxmb << 20);
  cudaMemset(tab, 1, maxmb << 20);
  cudaMalloc(&out, 16 + 80000 * 8);
  const char* sweep = getenv("MLP_SWEEP");
  if (sweep && sweep[0] == '5') {  // the TMA unit as a second request path (L2-resident table)
    for (int warps : {16, 32})
      for (size_t mb : {32ul}) {
        run<0, 8>(tab, mb, warps, 0, sms, clk, out);
        run<5, 4>(tab, mb, warps, 0, sms, clk, out);
        run<5, 8>(tab, mb, warps, 0, sms, clk, out);
        run<6, 8>(tab, mb, warps, 0, sms, clk, out);
        run<6, 16>(tab, mb, warps, 0, sms, clk, out);
      }
    return 0;
  }
  if (sweep && sweep[0] == '4') {  // L1-resident tables (MLP_KB=1): is the 1/clk limit the L1 or the L2?
    for (size_t kb : {16ul, 64ul, 256ul, 32768ul})
      for (int warps : {16}) {
        run<0, 8>(tab, kb, warps, 0, sms, clk, out);
        run<1, 8>(tab, kb, warps, 0, sms, clk, out);
      }
    return 0;
  }
  if (sweep && sweep[0] == '3') {  // REDs alone and mixed with loads (L2-resident table)
    for (int warps : {8, 16})
      for (int pad : {0, 128}) {
        run<3, 8>(tab, 32, warps, pad, sms, clk, out);
        run<4, 8>(tab, 32, warps, pad, sms, clk, out);
        run<0, 8>(tab, 32, warps, pad, sms, clk, out);
      }
    return 0;
  }
  if (sweep && sweep[0] == '2') {  // in-flight depth: warps x lookups per thread, L2-resident table
    for (size_t mb : {32ul, 256ul})
      for (int warps : {8, 16, 32})
        for (int pad : {0, 128}) {
          run<0, 4>(tab, mb, warps, pad, sms, clk, out);
          run<0, 8>(tab, mb, warps, pad, sms, clk, out);
          run<0, 16>(tab, mb, warps, pad, sms, clk, out);
          run<1, 8>(tab, mb, warps, pad, sms, clk, out);
        }
    return 0;
  }
  for (size_t mb : {32ul, 4096ul})
    for (int pad : {0, 96, 160})
      for (int warps : {16}) {
        run<0, 4>(tab, mb, warps, pad, sms, clk, out);
        run<0, 8>(tab, mb, warps, pad, sms, clk, out);
        run<1, 4>(tab, mb, warps, pad, sms, clk, out);
        run<2, 4>(tab, mb, warps, pad, sms, clk, out);
        run<2, 8>(tab, mb, warps, pad, sms, clk, out);
      }
  return 0;
}
