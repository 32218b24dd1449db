// Microbenchmark: stream an m x n fp32 matrix through shared memory with 2-D
// TMA boxes of BC columns x box_rows rows (the compress stage-1 access
// pattern), no compute.  Reports GB/s for several band widths / stage sizes /
// stage counts / CTAs per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

struct Args {
  CUtensorMap map;
  int m, n, bc, box_rows, nbox, stages, bands, stage_bytes, work_per_cta;
  unsigned long long pol_first;
};

__global__ void __launch_bounds__(128) k(const __grid_constant__ Args A, int* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned long long* full = (unsigned long long*)(sm + A.stages * A.stage_bytes);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < A.stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(full + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int bm = A.box_rows * A.nbox;
  const int chunks = (A.m + bm - 1) / bm;
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  int acc = 0;
  // flattened per-CTA item list: (band = blockIdx.x + t*gridDim.x, chunk)
  const int my_bands = (A.bands - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int items = my_bands * chunks;
  auto issue = [&](int it) {
    const int band = blockIdx.x + (it / chunks) * gridDim.x, c = it % chunks;
    const int s = it % A.stages;
    unsigned char* base = sm + s * A.stage_bytes;
    const int row0 = c * bm;
    int nb = (A.m - row0 + A.box_rows - 1) / A.box_rows;
    if (nb > A.nbox) nb = A.nbox;
    const unsigned bytes = nb * A.box_rows * A.bc * 4;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(bytes) : "memory");
    for (int i = 0; i < nb; ++i)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
          " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(sa(base + i * A.box_rows * A.bc * 4)),
          "l"((unsigned long long)&A.map), "r"(band * A.bc), "r"(row0 + i * A.box_rows),
          "r"(sa(full + s)), "l"(pol)
          : "memory");
  };
  if (tid == 0)
    for (int it = 0; it < A.stages - 1 && it < items; ++it) issue(it);
  for (int it = 0; it < items; ++it) {
    if (tid == 0 && it + A.stages - 1 < items) issue(it + A.stages - 1);
    const int s = it % A.stages;
    const unsigned par = (it / A.stages) & 1;
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(sa(full + s)),
        "r"(par)
        : "memory");
    acc += sm[s * A.stage_bytes + tid * 4];
    __syncthreads();  // stage s is refilled at iteration it+1
  }
  if (acc == 123456789) sink[0] = acc;
}

int main() {
  PFN_cuTensorMapEncodeTiled enc;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
  const int m = 4096, n = 11008 * 4;  // 720 MB fp32
  float* g;
  cudaMalloc(&g, (size_t)m * n * 4);
  cudaMemset(g, 0, (size_t)m * n * 4);
  int* sink;
  cudaMalloc(&sink, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long pol;
  struct Cfg { int bc, box_rows, nbox, stages, ctas_per_sm; bool persistent; };
  std::vector<Cfg> cfgs = {
      {32, 192, 4, 2, 1, false}, {64, 208, 2, 2, 1, false}, {64, 208, 2, 2, 1, true},
      {64, 104, 2, 4, 1, true},  {64, 52, 2, 8, 1, true},   {32, 128, 1, 4, 1, true},
      {128, 96, 2, 2, 1, true},  {64, 104, 1, 4, 2, true},  {32, 192, 4, 2, 1, true},
      {256, 48, 2, 2, 1, true},  {64, 256, 1, 3, 1, true},
  };
  for (const Cfg& c : cfgs) {
    Args A{};
    A.m = m, A.n = n, A.bc = c.bc, A.box_rows = c.box_rows, A.nbox = c.nbox, A.stages = c.stages;
    A.bands = n / c.bc;
    A.stage_bytes = c.box_rows * c.nbox * c.bc * 4;
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)m};
    cuuint64_t strides[1] = {(cuuint64_t)n * 4};
    cuuint32_t box[2] = {(cuuint32_t)c.bc, (cuuint32_t)c.box_rows};
    cuuint32_t es[2] = {1, 1};
    if (enc(&A.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("encode failed bc=%d\n", c.bc);
      continue;
    }
    // evict_first policy value (createpolicy.fractional.L2::evict_first 1.0)
    A.pol_first = 0x12F0000000000000ull;
    const int smem = c.stages * A.stage_bytes + 64;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = c.persistent ? sms * c.ctas_per_sm : A.bands;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<grid, 128, smem>>>(A, sink);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k<<<grid, 128, smem>>>(A, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("bc=%3d box_rows=%3d nbox=%d stages=%d stage=%6d B ctas/sm=%d persistent=%d : %7.1f GB/s %s\n",
           c.bc, c.box_rows, c.nbox, c.stages, A.stage_bytes, c.ctas_per_sm, c.persistent,
           (double)m * n * 4 * reps / (ms * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
  }
  (void)pol;
  return 0;
}
