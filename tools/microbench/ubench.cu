// Microbenchmarks that decide the point-pass histogram design on B200.
// Each test reports throughput in "lane-ops per ns" (whole chip) and per SM-cycle.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t xs(uint32_t& s) { s ^= s << 13; s ^= s >> 17; s ^= s << 5; return s; }

template <int MODE>
__global__ void k_smem(unsigned* out, int iters, uint32_t nbins) {
  extern __shared__ unsigned char sm[];
  unsigned* hu = (unsigned*)sm; float* hf = (float*)sm; double* hd = (double*)sm;
  for (uint32_t i = threadIdx.x; i < nbins * 2; i += blockDim.x) hu[i] = 0;
  __syncthreads();
  uint32_t s = 0x9e3779b9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  for (int it = 0; it < iters; ++it) {
    uint32_t b = xs(s) % nbins;
    if (MODE == 0) atomicAdd(&hu[b], 1u);
    if (MODE == 1) atomicAdd(&hf[b], 1.5f);
    if (MODE == 2) atomicAdd(&hd[b >> 1], 1.5);
    if (MODE == 3) {  // warp match_any aggregation + u32 add by leader
      unsigned m = __match_any_sync(0xffffffffu, b);
      if ((threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(&hu[b], (unsigned)__popc(m));
    }
    if (MODE == 4) { atomicAdd(&hu[b], 1u); atomicAdd(&hu[nbins + b], (unsigned)s & 0xffff); }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) if (hu[i] == 0xdeadbeef) out[0] = 1;
}

template <int MODE>
__global__ void k_gmem(void* g, int iters, uint32_t nbins) {
  uint32_t s = 0x9e3779b9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  for (int it = 0; it < iters; ++it) {
    uint32_t b = xs(s) % nbins;
    if (MODE == 0) atomicAdd(&((double*)g)[b], 1.5);
    if (MODE == 1) atomicAdd(&((unsigned long long*)g)[b], 1ull);
    if (MODE == 2) atomicAdd(&((unsigned*)g)[b], 1u);
  }
}

__global__ void k_read256(const double4* __restrict__ in, size_t n4, double* out) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride * 2) {
    double4 v0, v1;
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v0.x), "=d"(v0.y), "=d"(v0.z), "=d"(v0.w) : "l"(in + i));
    size_t j = i + stride; if (j >= n4) j = i;
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v1.x), "=d"(v1.y), "=d"(v1.z), "=d"(v1.w) : "l"(in + j));
    acc += v0.x + v0.y + v0.z + v0.w + v1.x + v1.y + v1.z + v1.w;
  }
  if (acc == 1234.5) out[0] = acc;
}

__global__ void k_read128(const double2* __restrict__ in, size_t n2, double* out) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride * 4) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { size_t j = i + u * stride; if (j >= n2) j = i; v[u] = __ldcs(in + j); }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y;
  }
  if (acc == 1234.5) out[0] = acc;
}

__global__ void k_fp64div(double* out, int iters, double s) {
  double x = threadIdx.x * 0.37 + blockIdx.x, acc = 0;
  for (int it = 0; it < iters; ++it) { acc += floor((x - 0.125) / s); x += 1.0; }
  if (acc == 1234.5) out[0] = acc;
}
__global__ void k_fp64mul(double* out, int iters, double r) {
  double x = threadIdx.x * 0.37 + blockIdx.x, acc = 0;
  for (int it = 0; it < iters; ++it) { acc += floor((x - 0.125) * r); x += 1.0; }
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount; int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"clk_mhz\":%d}\n", p.name, sms, clk_khz / 1000);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  unsigned* dout; CK(cudaMalloc(&dout, 1 << 20));
  void* g; CK(cudaMalloc(&g, 64 << 20)); CK(cudaMemset(g, 0, 64 << 20));
  const int threads = 512; const int blocks = sms * 4; const int iters = 2000;
  double lanes = (double)blocks * threads * iters;
  auto timeit = [&](auto launch) { launch(); cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms; };
  const char* names[] = {"smem_u32_atomic", "smem_f32_atomic(cas)", "smem_f64_atomic(cas)", "smem_match_any+u32", "smem_u32x2_atomic"};
  uint32_t binsets[] = {260, 4096, 40000};
  for (uint32_t nb : binsets) {
    size_t shb = (size_t)nb * 8; if (shb > 200000) shb = 200000;
    uint32_t nbe = (uint32_t)(shb / 8);
    for (int m = 0; m < 5; ++m) {
      float ms = 0;
      auto L = [&]() {
        int bl = shb > 48000 ? sms : blocks;
        switch (m) {
          case 0: cudaFuncSetAttribute(k_smem<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000); k_smem<0><<<bl, threads, shb>>>(dout, iters, nbe); break;
          case 1: cudaFuncSetAttribute(k_smem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000); k_smem<1><<<bl, threads, shb>>>(dout, iters, nbe); break;
          case 2: cudaFuncSetAttribute(k_smem<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000); k_smem<2><<<bl, threads, shb>>>(dout, iters, nbe); break;
          case 3: cudaFuncSetAttribute(k_smem<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000); k_smem<3><<<bl, threads, shb>>>(dout, iters, nbe); break;
          case 4: cudaFuncSetAttribute(k_smem<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000); k_smem<4><<<bl, threads, shb>>>(dout, iters, nbe / 2); break;
        }
      };
      ms = timeit(L); CK(cudaGetLastError());
      double ln = lanes * ((shb > 48000 ? (double)sms : (double)blocks) / blocks);
      printf("{\"test\":\"%s\",\"bins\":%u,\"ms\":%.3f,\"Glane_per_s\":%.1f,\"lane_per_sm_clk\":%.3f}\n", names[m], nbe, ms, ln / ms / 1e6, ln / (ms * 1e-3) / sms / (clk_khz * 1e3));
    }
  }
  const char* gn[] = {"gmem_f64_red", "gmem_u64_red", "gmem_u32_red"};
  for (uint32_t nb : binsets) for (int m = 0; m < 3; ++m) {
    auto L = [&]() { if (m == 0) k_gmem<0><<<blocks, threads>>>(g, iters / 4, nb); if (m == 1) k_gmem<1><<<blocks, threads>>>(g, iters / 4, nb); if (m == 2) k_gmem<2><<<blocks, threads>>>(g, iters / 4, nb); };
    float ms = timeit(L); CK(cudaGetLastError());
    double ln = lanes / 4;
    printf("{\"test\":\"%s\",\"bins\":%u,\"ms\":%.3f,\"Glane_per_s\":%.1f,\"lane_per_sm_clk\":%.3f}\n", gn[m], nb, ms, ln / ms / 1e6, ln / (ms * 1e-3) / sms / (clk_khz * 1e3));
  }
  size_t bytes = (size_t)4 << 30; void* big; CK(cudaMalloc(&big, bytes)); CK(cudaMemset(big, 0, bytes));
  for (int bpsm : {2, 4, 8}) {
    float ms = timeit([&]() { k_read256<<<sms * bpsm, 256>>>((const double4*)big, bytes / 32, (double*)dout); });
    printf("{\"test\":\"read256_nc_evict_first\",\"blocks_per_sm\":%d,\"GBps\":%.1f}\n", bpsm, bytes / ms / 1e6);
    ms = timeit([&]() { k_read128<<<sms * bpsm, 256>>>((const double2*)big, bytes / 16, (double*)dout); });
    printf("{\"test\":\"read128_ldcs_x4\",\"blocks_per_sm\":%d,\"GBps\":%.1f}\n", bpsm, bytes / ms / 1e6);
  }
  {
    float ms = timeit([&]() { k_fp64div<<<blocks, threads>>>((double*)dout, iters, 2.4901); });
    printf("{\"test\":\"fp64_div_floor\",\"Gop_per_s\":%.1f}\n", lanes / ms / 1e6);
    ms = timeit([&]() { k_fp64mul<<<blocks, threads>>>((double*)dout, iters, 1.0 / 2.4901); });
    printf("{\"test\":\"fp64_mul_floor\",\"Gop_per_s\":%.1f}\n", lanes / ms / 1e6);
  }
  return 0;
}
