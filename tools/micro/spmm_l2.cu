// Microbenchmarks for the compress stage-1 design space (not product code):
//  (1) L2 -> SM read bandwidth: all SMs stream a buffer that fits in L2.
//  (2) "SpMM from L2" stage 1: Z^T = G^T P with one warp per (bin, 128-column
//      tile), gathering the bin's G rows straight from global memory (L2 hits
//      after the first touch) -- no shared-memory staging, no padding.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o spmm_l2 spmm_l2.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void l2read(const float4* __restrict__ p, size_t n4, int reps, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
      float4 v = __ldg(p + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  if (acc.x == 12345.f) out[0] = acc.y + acc.z + acc.w;
}

// CSC of P: for bin b, rows csc_row[ptr[b]..ptr[b+1]) with values csc_val.
// grid: x = bin group (32 bins) fastest, y = column tile of 128 columns.
template <int U>
__global__ void __launch_bounds__(256) spmm_stage1(const float* __restrict__ G, long long ldg, int m, int n,
    const int* __restrict__ ptr, const int* __restrict__ row, const float* __restrict__ val,
    float* __restrict__ zt, int ldz, int d) {
  __shared__ float zs[32][129];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b0 = blockIdx.x * 32;
  const int j0 = blockIdx.y * 128;
  const float* gcol = G + j0 + 4 * lane;
  for (int bb = warp; bb < 32; bb += 8) {
    const int b = b0 + bb;
    float4 acc = make_float4(0, 0, 0, 0);
    if (b < d) {
      const int e0 = __ldg(ptr + b), e1 = __ldg(ptr + b + 1);
      int e = e0;
      for (; e + U <= e1; e += U) {
        float4 g[U]; float p[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = __ldg(row + e + u);
          p[u] = __ldg(val + e + u);
          g[u] = __ldg(reinterpret_cast<const float4*>(gcol + (long long)i * ldg));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          acc.x = fmaf(p[u], g[u].x, acc.x); acc.y = fmaf(p[u], g[u].y, acc.y);
          acc.z = fmaf(p[u], g[u].z, acc.z); acc.w = fmaf(p[u], g[u].w, acc.w);
        }
      }
      for (; e < e1; ++e) {
        const int i = __ldg(row + e);
        const float pp = __ldg(val + e);
        const float4 g = __ldg(reinterpret_cast<const float4*>(gcol + (long long)i * ldg));
        acc.x = fmaf(pp, g.x, acc.x); acc.y = fmaf(pp, g.y, acc.y);
        acc.z = fmaf(pp, g.z, acc.z); acc.w = fmaf(pp, g.w, acc.w);
      }
    }
    zs[bb][4 * lane] = acc.x; zs[bb][4 * lane + 1] = acc.y;
    zs[bb][4 * lane + 2] = acc.z; zs[bb][4 * lane + 3] = acc.w;
  }
  __syncthreads();
  // Z^T[j0 + c][b0 + lane] for c = warp, warp+8, ...
  for (int c = warp; c < 128; c += 8) {
    const int j = j0 + c;
    if (j < n && b0 + lane < d) zt[(long long)j * ldz + b0 + lane] = zs[lane][c];
  }
}

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  const int sms = pr.multiProcessorCount;
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float* junk; CK(cudaMalloc(&junk, 64));
  // (1) L2 bandwidth over buffers of several sizes
  for (size_t mb : {8, 32, 64, 96, 512}) {
    size_t bytes = mb << 20; float4* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes));
    int reps = mb >= 512 ? 2 : (int)(2048 / mb);
    for (int bs : {256, 512}) {
      int grid = sms * (2048 / bs);
      l2read<<<grid, bs>>>(buf, bytes / 16, 1, junk);
      CK(cudaEventRecord(e0));
      l2read<<<grid, bs>>>(buf, bytes / 16, reps, junk);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      printf("read %4zu MB x%d  block %d: %.1f GB/s\n", mb, reps, bs, bytes * (double)reps / ms / 1e6);
    }
    CK(cudaFree(buf));
  }
  // (2) SpMM stage 1 on Llama shapes, d=1024, r=4
  const int d = 1024, r = 4;
  struct Sh { int m, n; } shapes[] = {{4096, 4096}, {4096, 11008}, {11008, 4096}};
  for (auto sh : shapes) {
    const int m = sh.m, n = sh.n;
    std::mt19937_64 rng(m * 31 + n);
    std::vector<int> pos(m * r); std::vector<float> pv(m * r);
    std::normal_distribution<float> nd(0.f, 0.5f);
    for (int i = 0; i < m; ++i) {
      std::vector<int> s; while ((int)s.size() < r) { int b = rng() % d; if (std::find(s.begin(), s.end(), b) == s.end()) s.push_back(b); }
      std::sort(s.begin(), s.end());
      for (int l = 0; l < r; ++l) { pos[i * r + l] = s[l]; pv[i * r + l] = nd(rng); }
    }
    std::vector<int> ptr(d + 1, 0), crow(m * r); std::vector<float> cval(m * r);
    for (int i = 0; i < m * r; ++i) ptr[pos[i] + 1]++;
    for (int b = 0; b < d; ++b) ptr[b + 1] += ptr[b];
    std::vector<int> fill(ptr.begin(), ptr.end() - 1);
    for (int i = 0; i < m; ++i) for (int l = 0; l < r; ++l) { int b = pos[i * r + l]; crow[fill[b]] = i; cval[fill[b]++] = pv[i * r + l]; }
    int *dptr, *drow; float *dval, *G, *zt;
    CK(cudaMalloc(&dptr, (d + 1) * 4)); CK(cudaMalloc(&drow, m * r * 4)); CK(cudaMalloc(&dval, m * r * 4));
    CK(cudaMemcpy(dptr, ptr.data(), (d + 1) * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(drow, crow.data(), m * r * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dval, cval.data(), m * r * 4, cudaMemcpyHostToDevice));
    // 8 copies of G so that the timed loop streams > L2 from HBM
    const int copies = 8; size_t gsz = (size_t)m * n;
    CK(cudaMalloc(&G, gsz * 4 * copies)); CK(cudaMemset(G, 0, gsz * 4 * copies));
    CK(cudaMalloc(&zt, (size_t)n * d * 4));
    dim3 grid(d / 32, (n + 127) / 128);
    spmm_stage1<8><<<grid, 256>>>(G, n, m, n, dptr, drow, dval, zt, d, d);
    CK(cudaEventRecord(e0));
    for (int c = 0; c < copies; ++c) spmm_stage1<8><<<grid, 256>>>(G + gsz * c, n, m, n, dptr, drow, dval, zt, d, d);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ms /= copies;
    printf("spmm stage1 %dx%d: %.1f us  G %.1f GB/s  (L2->SM %.1f GB/s)\n", m, n, ms * 1e3, gsz * 4 / ms / 1e6, gsz * 16 / ms / 1e6);
    CK(cudaFree(dptr)); CK(cudaFree(drow)); CK(cudaFree(dval)); CK(cudaFree(G)); CK(cudaFree(zt));
  }
  return 0;
}
