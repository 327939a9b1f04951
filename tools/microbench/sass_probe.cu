#include <cstdint>
__global__ void k_u32(unsigned* out, const unsigned* idx){ __shared__ unsigned h[1024]; h[threadIdx.x]=0; __syncthreads(); atomicAdd(&h[idx[threadIdx.x]&1023],1u); __syncthreads(); out[threadIdx.x]=h[threadIdx.x];}
__global__ void k_f32(float* out, const unsigned* idx){ __shared__ float h[1024]; h[threadIdx.x]=0; __syncthreads(); atomicAdd(&h[idx[threadIdx.x]&1023],1.5f); __syncthreads(); out[threadIdx.x]=h[threadIdx.x];}
__global__ void k_f64(double* out, const unsigned* idx){ __shared__ double h[1024]; h[threadIdx.x]=0; __syncthreads(); atomicAdd(&h[idx[threadIdx.x]&1023],1.5); __syncthreads(); out[threadIdx.x]=h[threadIdx.x];}
__global__ void k_u64(unsigned long long* out, const unsigned* idx){ __shared__ unsigned long long h[1024]; h[threadIdx.x]=0; __syncthreads(); atomicAdd(&h[idx[threadIdx.x]&1023],3ull); __syncthreads(); out[threadIdx.x]=h[threadIdx.x];}
__global__ void k_gf64(double* out, const unsigned* idx){ atomicAdd(&out[idx[threadIdx.x]&1023],1.5);}
__global__ void k_gu64(unsigned long long* out, const unsigned* idx){ atomicAdd(&out[idx[threadIdx.x]&1023],3ull);}
__global__ void k_gf32(float* out, const unsigned* idx){ atomicAdd(&out[idx[threadIdx.x]&1023],1.5f);}
__global__ void k_match(unsigned* out, const unsigned* idx){ out[threadIdx.x]=__match_any_sync(0xffffffff, idx[threadIdx.x]);}
__global__ void k_ld256(double* out, const double4* in){ double4 v; asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x),"=d"(v.y),"=d"(v.z),"=d"(v.w) : "l"(in+threadIdx.x)); out[threadIdx.x]=v.x+v.y+v.z+v.w;}
