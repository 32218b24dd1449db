// Microbenchmark: shared-memory pipe cost (cycles per warp instruction per SM)
// of broadcast LDS.128 / LDS.64 / LDS.32, per-lane LDS.32 / LDS.64, SHFL.IDX.
// 8 independent ops per iteration with fixed addresses; one STS per iteration
// keeps ptxas from hoisting the loads out of the loop.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_pipe smem_pipe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

template <int MODE>
__device__ __forceinline__ unsigned op(unsigned a, unsigned lane, unsigned i, unsigned r) {
  unsigned x = 0, y = 0, z = 0, w = 0;
  if (MODE == 0) {
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a));
    return x ^ y ^ z ^ w;
  } else if (MODE == 1) {
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(a));
    return x ^ y;
  } else if (MODE == 2) {
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(a));
    return x;
  } else if (MODE == 3) {
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(a + lane * 4));
    return x;
  } else if (MODE == 4) {
    return __shfl_sync(0xffffffffu, r + i, a & 31);
  } else if (MODE == 5) {
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(a + lane * 8));
    return x ^ y;
  } else if (MODE == 6) {
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a + lane * 16));
    return x ^ y ^ z ^ w;
  } else if (MODE == 7) {  // per-lane LDS.32 + one SHFL.IDX
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(a + lane * 4));
    return x + __shfl_sync(0xffffffffu, r + i, a & 31);
  } else if (MODE == 8) {  // per-lane LDS.32 + two SHFL.IDX
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(a + lane * 4));
    return x + __shfl_sync(0xffffffffu, r + i, a & 31) * __shfl_sync(0xffffffffu, r ^ i, (a >> 5) & 31);
  } else {  // per-lane LDS.32 + broadcast LDS.64
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(a + lane * 4));
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(y), "=r"(z) : "r"(a + 8192));
    return x + y * z;
  }
}

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(unsigned* out, unsigned long long* cyc) {
  __shared__ __align__(16) unsigned sm[12288];
  for (int i = threadIdx.x; i < 12288; i += blockDim.x) sm[i] = i * 2654435761u;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  const unsigned base = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  const unsigned w = (threadIdx.x >> 5);
  unsigned acc = 0;
  unsigned* st = sm + 11264 + threadIdx.x;
  __syncthreads();
  const unsigned long long t0 = clock64();
#pragma unroll 1
  for (unsigned i = 0; i < ITERS; ++i) {
    unsigned s = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += op<MODE>(base + ((w * 8 + u) & 31) * 512, lane, i, u);
    acc ^= s;
    *st = acc;  // aliasing store: loads stay in the loop
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int sms) {
  unsigned* out;
  unsigned long long* cyc;
  cudaMalloc(&out, sms * 1024 * 4);
  cudaMalloc(&cyc, sms * 8);
  k<MODE><<<sms, 1024>>>(out, cyc);
  k<MODE><<<sms, 1024>>>(out, cyc);
  cudaDeviceSynchronize();
  unsigned long long h[1024];
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  printf("%-34s %.3f cycles per warp-op per SM\n", name, avg / (32.0 * ITERS * 8));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("broadcast LDS.128", sms);
  run<1>("broadcast LDS.64", sms);
  run<2>("broadcast LDS.32", sms);
  run<3>("per-lane LDS.32 (128 B)", sms);
  run<4>("SHFL.IDX", sms);
  run<5>("per-lane LDS.64 (256 B)", sms);
  run<6>("per-lane LDS.128 (512 B)", sms);
  run<7>("per-lane LDS.32 + 1 SHFL", sms);
  run<8>("per-lane LDS.32 + 2 SHFL", sms);
  run<9>("per-lane LDS.32 + bcast LDS.64", sms);
  return 0;
}
