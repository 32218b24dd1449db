// Row-gather throughput into shared memory (not product code): can TMA keep
// more 512-byte random-row gathers in flight than LDG.128 into registers?
//   tmag : one lane per warp issues cp.async.bulk.tensor tile::gather4 (4 rows of
//          128 fp32 per instruction) into a per-warp S-stage ring; all lanes read
//          the rows back with LDS.128 and accumulate.
//   bulk : the same ring filled by four 512-byte cp.async.bulk copies per stage.
//   ldg  : the register path of k_compress_spmm (U loads in flight per warp).
// Reports bytes delivered to the SMs per second from an L2-resident buffer.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tma_gather tma_gather.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ unsigned hash(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}
__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(b)));
}
__device__ __forceinline__ void mb_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
// bounded wait: trap instead of hanging the GPU
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned par) {
  for (long long i = 0;; ++i) {
    unsigned ok;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
    if (ok) return;
    if (i > (1LL << 26)) __trap();
  }
}

template <int MODE>  // 0 = gather4 tensor, 1 = 4 bulk copies
__global__ void ring(const __grid_constant__ CUtensorMap map, const float* buf, unsigned rows, int iters, int S,
                     float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned char* ring = sm + warp * S * 2048;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + nw * S * 2048) + warp * S;
  unsigned s = hash((blockIdx.x * nw + warp) * 7919u + 1);
  auto issue = [&](int st) {
    int r[4];
    for (int k = 0; k < 4; ++k) { s = hash(s + k); r[k] = s % rows; }
    mb_expect(bar + st, 2048);
    if (MODE == 0) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(sa(ring + st * 2048)),
          "l"(reinterpret_cast<unsigned long long>(&map)), "r"(sa(bar + st)), "r"(0), "r"(r[0]), "r"(r[1]),
          "r"(r[2]), "r"(r[3])
          : "memory");
    } else {
      for (int k = 0; k < 4; ++k)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
                         sa(ring + st * 2048 + k * 512)),
                     "l"(buf + (size_t)r[k] * 128), "r"(sa(bar + st))
                     : "memory");
    }
  };
  if (lane == 0) {
    for (int st = 0; st < S; ++st) mb_init(bar + st);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (lane == 0)
    for (int st = 0; st < S; ++st) issue(st);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
    const int st = it % S;
    mb_wait(bar + st, (it / S) & 1);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 v = *reinterpret_cast<const float4*>(ring + st * 2048 + k * 512 + lane * 16);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    __syncwarp();
    if (lane == 0 && it + S < iters) issue(st);
  }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

// LDGSTS ring: each lane copies its 16 bytes of 4 rows per stage (cp.async.cg),
// S stages per warp, then reads them back with LDS.128.
__global__ void ldgsts(const float4* __restrict__ p, unsigned rows, int iters, int S, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* ring = sm + warp * S * 2048;
  unsigned s = hash((blockIdx.x * (blockDim.x >> 5) + warp) * 7919u + 1);
  auto issue = [&](int st) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      s = hash(s + k);
      const float4* src = p + (size_t)(s % rows) * 32 + lane;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(ring + st * 2048 + k * 512 + lane * 16)),
                   "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int st = 0; st < S; ++st) issue(st);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
    const int st = it % S;
    // groups complete in order: wait until at most S-1 are pending
    switch (S) {
      case 2: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
      case 4: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
      case 6: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
      default: asm volatile("cp.async.wait_group 7;" ::: "memory"); break;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 v = *reinterpret_cast<const float4*>(ring + st * 2048 + k * 512 + lane * 16);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (it + S < iters) issue(st); else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

template <int U>
__global__ void ldg(const float4* __restrict__ p, unsigned rows, int iters, float* out) {
  const int lane = threadIdx.x & 31;
  const unsigned wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  unsigned s = hash(wid * 7919u + 1);
  for (int it = 0; it < iters; ++it) {
    float4 g[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { s = hash(s + u); g[u] = __ldg(p + (size_t)(s % rows) * 32 + lane); }
#pragma unroll
    for (int u = 0; u < U; ++u) { acc.x += g[u].x; acc.y += g[u].y; acc.z += g[u].z; acc.w += g[u].w; }
  }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

int main() {
  const size_t bytes = 32ull << 20;
  const unsigned rows = bytes / 512;
  float* p; float* out;
  CK(cudaMalloc(&p, bytes)); CK(cudaMalloc(&out, 4)); CK(cudaMemset(p, 0, bytes));
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto enc = (PFN_cuTensorMapEncodeTiled)fn;
  CUtensorMap map;
  cuuint64_t dims[2] = {128, rows}; cuuint64_t str[1] = {512};
  cuuint32_t box[2] = {128, 1}; cuuint32_t es[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n"); return 1;
  }
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  auto run = [&](const char* name, auto launch, double bytes_moved) {
    launch(); CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a)); launch(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    printf("%-40s %7.2f TB/s\n", name, bytes_moved / ms / 1e9);
  };
  const int iters = 4000;
  for (int w : {16}) for (int S : {4}) {
    const int smem = w * S * (2048 + 8);
    if (smem > 227 * 1024) continue;
    char nm[64];
    CK(cudaFuncSetAttribute(ring<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(ring<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const double mv = 148.0 * w * iters * 2048.0;
    snprintf(nm, 64, "gather4 warps=%d stages=%d (%d KB)", w, S, smem / 1024);
    run(nm, [&] { ring<0><<<148, w * 32, smem>>>(map, p, rows, iters, S, out); }, mv);
    snprintf(nm, 64, "bulk x4 warps=%d stages=%d", w, S);
    run(nm, [&] { ring<1><<<148, w * 32, smem>>>(map, p, rows, iters, S, out); }, mv);
  }
  for (int w : {16, 24, 32}) for (int S : {2, 4, 6, 8}) {
    const int smem = w * S * 2048;
    if (smem > 227 * 1024) continue;
    char nm[64];
    CK(cudaFuncSetAttribute(ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    snprintf(nm, 64, "ldgsts warps=%d stages=%d (%d KB)", w, S, smem / 1024);
    run(nm, [&] { ldgsts<<<148, w * 32, smem>>>(reinterpret_cast<const float4*>(p), rows, iters, S, out); },
        148.0 * w * iters * 2048.0);
  }
  for (int w : {16, 32}) {
    char nm[64];
    snprintf(nm, 64, "ldg U=16 warps=%d", w);
    run(nm, [&] { ldg<16><<<148 * w / 8, 256>>>(reinterpret_cast<const float4*>(p), rows, 1000, out); },
        148.0 * w * 1000 * 16 * 512.0);
  }
  return 0;
}
