// DSMEM atomic throughput: clusters of C CTAs, each holding nb/C bins of a
// u32 histogram; every thread adds to random bins anywhere in the cluster.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;
__device__ __forceinline__ uint32_t xs(uint32_t& s) { s ^= s << 13; s ^= s >> 17; s ^= s << 5; return s; }

template <int MODE>
__global__ void k(unsigned* out, int iters, uint32_t nb) {
  extern __shared__ unsigned h[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t C = cl.num_blocks();
  const uint32_t per = nb / C;
  for (uint32_t i = threadIdx.x; i < per * 3; i += blockDim.x) h[i] = 0;
  cl.sync();
  uint32_t s = 0x9e3779b9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  for (int it = 0; it < iters; ++it) {
    uint32_t b = xs(s) % nb;
    uint32_t r = b / per, o = b % per;
    unsigned* dst = cl.map_shared_rank(h, r);
    if (MODE == 0) atomicAdd(&dst[o], 1u);
    if (MODE == 1) { atomicAdd(&dst[3 * o], 1u); atomicAdd(&dst[3 * o + 1], s & 0xffff); atomicAdd(&dst[3 * o + 2], 7u); }
    if (MODE == 2) { unsigned* d2 = h; uint32_t o2 = b % per; atomicAdd(&d2[o2], 1u); }  // local only
  }
  cl.sync();
  for (uint32_t i = threadIdx.x; i < per; i += blockDim.x) if (h[i] == 0xdeadbeef) out[0] = 1;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned* d; cudaMalloc(&d, 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 2000, threads = 512;
  for (int C : {1, 2, 4, 8}) for (int mode : {0, 1, 2}) for (uint32_t nb : {40000u}) {
    size_t smem = (size_t)(nb / C) * 12;
    if (smem > 220 * 1024) { printf("{\"C\":%d,\"mode\":%d,\"skip\":\"smem %zu\"}\n", C, mode, smem); continue; }
    void (*kern)(unsigned*, int, uint32_t) = mode == 0 ? k<0> : (mode == 1 ? k<1> : k<2>);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((sms / C) * C); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1]; attr[0].id = cudaLaunchAttributeClusterDimension; attr[0].val.clusterDim.x = C; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, d, iters, nb);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, kern, d, iters, nb);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaError_t e = cudaGetLastError();
    float ms; cudaEventElapsedTime(&ms, a, b);
    double lanes = (double)cfg.gridDim.x * threads * iters * (mode == 1 ? 3 : 1);
    printf("{\"C\":%d,\"mode\":%d,\"err\":\"%s\",\"ms\":%.3f,\"Gatom_per_s\":%.1f,\"atom_per_sm_clk\":%.3f}\n", C, mode, cudaGetErrorString(e), ms, lanes / ms / 1e6, lanes / (ms * 1e-3) / sms / (clk * 1e3));
  }
  return 0;
}
