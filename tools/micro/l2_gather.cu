// L2 -> SM throughput ceiling for the gather pattern of the compress / Y-build
// kernels (not product code).  A warp reads 512-byte row segments (one
// LDG.128 per lane) at pseudo-random rows of an L2-resident buffer, U loads in
// flight per warp, W warps per SM; reports bytes delivered to the SMs per
// second.  Also a coalesced streaming read of the same buffer for reference.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2_gather l2_gather.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ unsigned hash(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int U, bool NA>
__global__ void gather(const float4* __restrict__ p, unsigned rows, int iters, float* out) {
  const int lane = threadIdx.x & 31;
  const unsigned wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  unsigned s = hash(wid * 7919u + 1);
  for (int it = 0; it < iters; ++it) {
    float4 g[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      s = hash(s + u);
      const float4* a = p + (size_t)(s % rows) * 32 + lane;
      if (NA) {
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(g[u].x), "=f"(g[u].y), "=f"(g[u].z), "=f"(g[u].w) : "l"(a));
      } else {
        g[u] = __ldg(a);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) { acc.x += g[u].x; acc.y += g[u].y; acc.z += g[u].z; acc.w += g[u].w; }
  }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

__global__ void stream(const float4* __restrict__ p, size_t n4, int reps, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
      float4 v = __ldg(p + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

template <int U, bool NA>
void run_gather(const float4* p, unsigned rows, int warps_per_sm, float* out) {
  const int threads = 256;
  const int blocks = 148 * warps_per_sm / 8;
  const int iters = 2000 / U;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  gather<U, NA><<<blocks, threads>>>(p, rows, 4, out);
  CK(cudaEventRecord(a));
  gather<U, NA><<<blocks, threads>>>(p, rows, iters, out);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  const double bytes = (double)blocks * threads / 32 * iters * U * 512.0;
  printf("gather U=%2d NA=%d warps/SM=%2d buf=%5.1f MB: %7.2f TB/s (%.3f ms)\n", U, (int)NA, warps_per_sm,
         rows * 512.0 / 1e6, bytes / ms / 1e9, ms);
}

int main() {
  const size_t bytes = 512ull << 20;
  float4* p; float* out;
  CK(cudaMalloc(&p, bytes)); CK(cudaMalloc(&out, 4));
  CK(cudaMemset(p, 0, bytes));
  for (size_t mb : {32, 64, 96}) {
    const size_t n4 = (mb << 20) / 16;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    stream<<<148 * 8, 256>>>(p, n4, 2, out);
    CK(cudaEventRecord(a));
    stream<<<148 * 8, 256>>>(p, n4, 20, out);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    printf("stream buf=%zu MB: %.2f TB/s\n", mb, 20.0 * (mb << 20) / ms / 1e9);
  }
  for (unsigned mb : {32u, 64u}) {
    const unsigned rows = (mb << 20) / 512;
    for (int w : {16, 32, 48, 64}) {
      run_gather<8, false>(p, rows, w, out);
      run_gather<16, false>(p, rows, w, out);
    }
    run_gather<8, true>(p, rows, 32, out);
    run_gather<16, true>(p, rows, 32, out);
  }
  const unsigned rows = (512u << 20) / 512;  // HBM-resident
  run_gather<8, false>(p, rows, 32, out);
  run_gather<16, false>(p, rows, 32, out);
  return 0;
}
