// Microbenchmark (not product code): in-place read-modify-write streaming of a
// large fp32 matrix W (m x n), w = 0.999*w + 1e-3, in the decompress-apply
// access pattern.  Variants:
//   plain : grid-stride LDG.128 / STG.128 over the flat array (upper bound)
//   ring  : persistent CTA per SM, column bands of BN columns, W tiles of TR
//           rows via 2-D TMA through an S-stage mbarrier ring, consumer warps
//           in NG groups (group g takes tiles g, g+NG, ...), results written
//           with STG from registers; `reserve` bytes of smem left unused (the
//           Y block of the real kernel).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_rmw stream_rmw.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)
__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void mb_expect(unsigned long long* b, unsigned n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_arrive(unsigned long long* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned ph) {
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(sa(b)), "r"(ph) : "memory"); }

__global__ void plain(float4* w, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = w[i]; v.x = 0.999f * v.x + 1e-3f; v.y = 0.999f * v.y + 1e-3f; v.z = 0.999f * v.z + 1e-3f; v.w = 0.999f * v.w + 1e-3f; w[i] = v;
  }
}

// same RMW with plain loads/stores, 32-column bands: item i -> (band i % nb,
// 64-row block i / nb); one warp per item, 8 lanes x float4 per row
__global__ void band_plain(float* w, int m, int n, int bn) {
  const int lane = threadIdx.x & 31;
  const long long warp_g = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int nb = n / bn, rbs = (m + 63) / 64;
  const int lpr = bn / 4, rpi = 32 / lpr;
  for (long long it = warp_g; it < (long long)nb * rbs; it += nwarps) {
    const int b = it % nb, rb = it / nb;
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = rb * 64 + k * 8 * rpi / 8 * 1 + (lane / lpr) + k * rpi;
      (void)r;
    }
    for (int q0 = 0; q0 < 64; q0 += 8 * rpi) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int r = rb * 64 + q0 + k * rpi + lane / lpr;
        v[k] = r < m ? *(const float4*)(w + (size_t)r * n + b * bn + (lane % lpr) * 4) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int r = rb * 64 + q0 + k * rpi + lane / lpr;
        float4 x = v[k]; x.x = 0.999f * x.x + 1e-3f; x.y = 0.999f * x.y + 1e-3f; x.z = 0.999f * x.z + 1e-3f; x.w = 0.999f * x.w + 1e-3f;
        if (r < m) *(float4*)(w + (size_t)r * n + b * bn + (lane % lpr) * 4) = x;
      }
    }
  }
}

struct RArgs { CUtensorMap map; float* w; int m, n, bn, tr, stages, ng, nc, reserve, tile_bytes, tstore; };

__global__ void ring(const __grid_constant__ RArgs A) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* rg = sm + A.reserve;
  unsigned long long* full = (unsigned long long*)(rg + A.stages * A.tile_bytes);
  unsigned long long* empty = full + A.stages;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, S = A.stages;
  const int per_group = A.nc / A.ng;
  if (tid == 0) { for (int s = 0; s < S; ++s) { mb_init(full + s, 1); mb_init(empty + s, A.tstore ? 1 : per_group); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  const int nb = (A.n + A.bn - 1) / A.bn, rbs = (A.m + A.tr - 1) / A.tr;
  if (warp == A.nc) {  // producer
    if (lane == 0) {
      unsigned long long pol; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int s = 0;
      for (int b = blockIdx.x; b < nb; b += gridDim.x)
        for (int rb = 0; rb < rbs; ++rb, ++s) {
          const int st = s % S;
          if (s >= S) mb_wait(empty + st, ((s / S) - 1) & 1);
          mb_expect(full + st, A.tile_bytes);
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;"
            ::"r"(sa(rg + st * A.tile_bytes)), "l"(&A.map), "r"(b * A.bn), "r"(rb * A.tr), "r"(sa(full + st)), "l"(pol) : "memory");
        }
    }
    return;
  }
  const int g = warp / per_group, wg = warp % per_group;
  const int lanes_per_row = A.bn / 4 < 32 ? A.bn / 4 : 32;  // float4 per lane
  const int rows_per_instr = 32 / lanes_per_row;
  int s = 0;
  for (int b = blockIdx.x; b < nb; b += gridDim.x)
    for (int rb = 0; rb < rbs; ++rb, ++s) {
      if (s % A.ng != g) continue;
      const int st = s % S;
      mb_wait(full + st, (s / S) & 1);
      float* t = (float*)(rg + st * A.tile_bytes);
      for (int q = wg * rows_per_instr + lane / lanes_per_row; q < A.tr; q += per_group * rows_per_instr) {
        for (int c4 = lane % lanes_per_row; c4 < A.bn / 4; c4 += lanes_per_row) {
          float4 v = *(const float4*)(t + q * A.bn + c4 * 4);
          v.x = 0.999f * v.x + 1e-3f; v.y = 0.999f * v.y + 1e-3f; v.z = 0.999f * v.z + 1e-3f; v.w = 0.999f * v.w + 1e-3f;
          if (A.tstore) { *(float4*)(t + q * A.bn + c4 * 4) = v; continue; }
          const int r = rb * A.tr + q, c = b * A.bn + c4 * 4;
          if (r < A.m && c < A.n) *(float4*)(A.w + (size_t)r * A.n + c) = v;
        }
      }
      if (A.tstore) {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(per_group * 32) : "memory");
        if (wg == 0 && lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&A.map), "r"(b * A.bn), "r"(rb * A.tr), "r"(sa(t)) : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          mb_arrive(empty + st);
        }
        continue;
      }
      __syncwarp();
      if (lane == 0) mb_arrive(empty + st);
    }
}

// ring3: `ring` with clusters of CL CTAs that stream adjacent bands b0..b0+CL-1
// at the same row blocks in lockstep: before each TMA load the producer
// arrives (remote mbarrier arrive) on every cluster peer's sync barrier and
// waits for all CL arrivals on its own, so the CL 128-byte segments of each
// W row are requested together (a 128*CL-byte span of the row).
__global__ void ring3(const __grid_constant__ RArgs A) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* rg = sm + A.reserve;
  unsigned long long* full = (unsigned long long*)(rg + A.stages * A.tile_bytes);
  unsigned long long* empty = full + A.stages;
  unsigned long long* sync = empty + A.stages;
  unsigned cr, CL;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(CL));
  const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, S = A.stages;
  const int per_group = A.nc / A.ng;
  if (tid == 0) { for (int s = 0; s < S; ++s) { mb_init(full + s, 1); mb_init(empty + s, per_group); }
    mb_init(sync, CL);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("barrier.cluster.arrive.aligned; barrier.cluster.wait.aligned;" ::: "memory");
  const int nb = (A.n + A.bn - 1) / A.bn, rbs = (A.m + A.tr - 1) / A.tr;
  if (warp == A.nc) {  // producer
    if (lane == 0) {
      unsigned long long pol; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int s = 0;
      for (int b0 = cid * CL; b0 < nb; b0 += ncl * CL)
        for (int rb = 0; rb < rbs; ++rb, ++s) {
          if (!A.tstore) {  // tstore = 1: no lockstep (control)
          for (unsigned p = 0; p < CL; ++p) {
            unsigned ra; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(sa(sync)), "r"(p));
            asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
          }
          asm volatile("{\n.reg .pred p;\nW3:\nmbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%0], %1;\n@!p bra W3;\n}" ::"r"(sa(sync)), "r"(s & 1) : "memory");
          }
          const int b = b0 + cr;
          if (b >= nb) continue;
          const int st = s % S;
          if (s >= S) mb_wait(empty + st, ((s / S) - 1) & 1);
          mb_expect(full + st, A.tile_bytes);
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;"
            ::"r"(sa(rg + st * A.tile_bytes)), "l"(&A.map), "r"(b * A.bn), "r"(rb * A.tr), "r"(sa(full + st)), "l"(pol) : "memory");
        }
    }
  } else {
    const int g = warp / per_group, wg = warp % per_group;
    const int lanes_per_row = A.bn / 4 < 32 ? A.bn / 4 : 32;
    const int rows_per_instr = 32 / lanes_per_row;
    int s = 0;
    for (int b0 = cid * CL; b0 < nb; b0 += ncl * CL)
      for (int rb = 0; rb < rbs; ++rb, ++s) {
        const int b = b0 + cr;
        if (b >= nb || s % A.ng != g) continue;
        const int st = s % S;
        mb_wait(full + st, (s / S) & 1);
        float* t = (float*)(rg + st * A.tile_bytes);
        for (int q = wg * rows_per_instr + lane / lanes_per_row; q < A.tr; q += per_group * rows_per_instr) {
          for (int c4 = lane % lanes_per_row; c4 < A.bn / 4; c4 += lanes_per_row) {
            float4 v = *(const float4*)(t + q * A.bn + c4 * 4);
            v.x = 0.999f * v.x + 1e-3f; v.y = 0.999f * v.y + 1e-3f; v.z = 0.999f * v.z + 1e-3f; v.w = 0.999f * v.w + 1e-3f;
            const int r = rb * A.tr + q, c = b * A.bn + c4 * 4;
            if (r < A.m && c < A.n) *(float4*)(A.w + (size_t)r * A.n + c) = v;
          }
        }
        __syncwarp();
        if (lane == 0) mb_arrive(empty + st);
      }
  }
  __syncwarp();
  asm volatile("barrier.cluster.arrive.aligned; barrier.cluster.wait.aligned;" ::: "memory");
}

// ring4: clusters of CL CTAs own "super-bands" of CL*32 columns; CTA k of the
// cluster streams columns [32k, 32k+32) of it.  Only the leader's producer
// issues loads: per tile CL boxes side by side (one W row segment of CL*128
// bytes, back to back from one TMA unit), box k multicast to CTA k alone
// (ctaMask = 1 << k).  Consumers free a stage by a remote arrive on the
// leader's empty barrier.
__global__ void ring4(const __grid_constant__ RArgs A) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* rg = sm + A.reserve;
  unsigned long long* full = (unsigned long long*)(rg + A.stages * A.tile_bytes);
  unsigned long long* empty = full + A.stages;
  unsigned cr, CL;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(CL));
  const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, S = A.stages;
  const int per_group = A.nc / A.ng;
  if (tid == 0) { for (int s = 0; s < S; ++s) { mb_init(full + s, 1); mb_init(empty + s, per_group * CL); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("barrier.cluster.arrive.aligned; barrier.cluster.wait.aligned;" ::: "memory");
  const int sbw = 32 * CL;
  const int nsb = (A.n + sbw - 1) / sbw, rbs = (A.m + A.tr - 1) / A.tr;
  if (warp == A.nc) {  // producer
    if (lane == 0) {
      unsigned long long pol; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int s = 0;
      for (int sb = cid; sb < nsb; sb += ncl)
        for (int rb = 0; rb < rbs; ++rb, ++s) {
          const int st = s % S;
          const int ph = (s / S) & 1;
          if (s >= S) mb_wait(full + st, ph ^ 1);  // own previous phase landed before re-arming
          mb_expect(full + st, A.tile_bytes);
          if (cr == 0) {
            if (s >= S) mb_wait(empty + st, ph ^ 1);
            for (unsigned k = 0; k < CL; ++k) {
              const unsigned short mask = (unsigned short)(1u << k);
              asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5, %6;"
                ::"r"(sa(rg + st * A.tile_bytes)), "l"(&A.map), "r"(sb * sbw + 32 * k), "r"(rb * A.tr), "r"(sa(full + st)), "h"(mask), "l"(pol) : "memory");
            }
          }
        }
    }
  } else {
    const int g = warp / per_group, wg = warp % per_group;
    unsigned rempty; asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rempty) : "r"(sa(empty)));
    int s = 0;
    for (int sb = cid; sb < nsb; sb += ncl)
      for (int rb = 0; rb < rbs; ++rb, ++s) {
        if (s % A.ng != g) continue;
        const int st = s % S;
        mb_wait(full + st, (s / S) & 1);
        float* t = (float*)(rg + st * A.tile_bytes);
        for (int q = wg * 4 + lane / 8; q < A.tr; q += per_group * 4) {
          float4 v = *(const float4*)(t + q * 32 + (lane % 8) * 4);
          v.x = 0.999f * v.x + 1e-3f; v.y = 0.999f * v.y + 1e-3f; v.z = 0.999f * v.z + 1e-3f; v.w = 0.999f * v.w + 1e-3f;
          const int r = rb * A.tr + q, c = sb * sbw + cr * 32 + (lane % 8) * 4;
          if (r < A.m && c < A.n) *(float4*)(A.w + (size_t)r * A.n + c) = v;
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(rempty + st * 8) : "memory");
      }
  }
  __syncwarp();
  asm volatile("barrier.cluster.arrive.aligned; barrier.cluster.wait.aligned;" ::: "memory");
}


// ring2: tiles of NB boxes side by side (box = 32 fp32 cols x TR rows, 128B
// swizzle), i.e. a TR x 32*NB tile whose rows are 128*NB bytes of W; lane =
// row reads 16-byte chunks (swizzle makes the 8-lane phases conflict-free),
// results written back in place and TMA-stored (the row-orientation apply).
struct R2Args { CUtensorMap map; float* w; int m, n, nb, tr, stages, ng, nc, reserve, tile_bytes; };
__global__ void ring2(const __grid_constant__ R2Args A) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* rg = sm + A.reserve;
  unsigned long long* full = (unsigned long long*)(rg + A.stages * A.tile_bytes);
  unsigned long long* empty = full + A.stages;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, S = A.stages;
  const int per_group = A.nc / A.ng;
  if (tid == 0) { for (int s = 0; s < S; ++s) { mb_init(full + s, 1); mb_init(empty + s, 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  const int tc = 32 * A.nb;
  const int ntc = (A.n + tc - 1) / tc, nrb = (A.m + A.tr - 1) / A.tr;
  const long long tiles = (long long)ntc * nrb;
  if (warp == A.nc) {
    if (lane == 0) {
      unsigned long long pol; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int s = 0;
      for (long long t = blockIdx.x; t < tiles; t += gridDim.x, ++s) {
        const int rb = t / ntc, cb = t % ntc;  // concurrent tiles: same rows, adjacent columns
        const int st = s % S;
        if (s >= S) mb_wait(empty + st, ((s / S) - 1) & 1);
        mb_expect(full + st, A.tile_bytes);
        for (int b = 0; b < A.nb; ++b)
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;"
            ::"r"(sa(rg + st * A.tile_bytes + b * 32 * 4 * A.tr)), "l"(&A.map), "r"(cb * tc + b * 32), "r"(rb * A.tr), "r"(sa(full + st)), "l"(pol) : "memory");
      }
    }
    return;
  }
  const int g = warp / per_group, wg = warp % per_group;
  int s = 0;
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x, ++s) {
    if (s % A.ng != g) continue;
    const int rb = t / ntc, cb = t % ntc;
    const int st = s % S;
    mb_wait(full + st, (s / S) & 1);
    unsigned char* tile = rg + st * A.tile_bytes;
    // rows: lane + 32*k; column chunks (16 B): spread over the group's warps
    for (int rr = lane; rr < A.tr; rr += 32)
      for (int ch = wg; ch < 8 * A.nb; ch += per_group) {
        const int b = ch / 8, c = ch % 8;
        float4* p = (float4*)(tile + b * 32 * 4 * A.tr + rr * 128 + ((c ^ (rr & 7)) * 16));
        float4 v = *p;
        v.x = 0.999f * v.x + 1e-3f; v.y = 0.999f * v.y + 1e-3f; v.z = 0.999f * v.z + 1e-3f; v.w = 0.999f * v.w + 1e-3f;
        *p = v;
      }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(per_group * 32) : "memory");
    if (wg == 0 && lane == 0) {
      for (int b = 0; b < A.nb; ++b)
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&A.map), "r"(cb * tc + b * 32), "r"(rb * A.tr), "r"(sa(tile + b * 32 * 4 * A.tr)) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      mb_arrive(empty + st);
    }
  }
}

int main() {
  CK(cudaSetDevice(0)); int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int m = 4096 * 7, n = 11008;  // ~1.26 GB fp32
  float* w; size_t bytes = (size_t)m * n * 4; CK(cudaMalloc(&w, bytes)); CK(cudaMemset(w, 0, bytes));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto timeit = [&](auto f) { f(); CK(cudaDeviceSynchronize()); CK(cudaEventRecord(e0)); for (int i = 0; i < 5; ++i) f(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); return 2.0 * bytes * 5 / ms / 1e6; };
  printf("plain: %.0f GB/s\n", timeit([&] { plain<<<sms * 8, 256>>>((float4*)w, bytes / 16); }));
  for (int bn : {32, 64, 128})
    for (int bpsm : {4, 8})
      printf("band_plain bn=%d blocks/SM=%d: %.0f GB/s\n", bn, bpsm, timeit([&] { band_plain<<<sms * bpsm, 256>>>(w, m, n, bn); }));
  void* fn = nullptr; cudaDriverEntryPointQueryResult q; CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto enc = (PFN_cuTensorMapEncodeTiled)fn;
  struct C2 { int nb, tr, stages, ng, nc, reserve; } c2s[] = {
    {4, 32, 4, 2, 16, 128 * 1024}, {4, 32, 5, 2, 16, 128 * 1024}, {4, 32, 4, 4, 16, 128 * 1024},
    {8, 32, 2, 2, 16, 128 * 1024}, {4, 64, 2, 2, 16, 128 * 1024}, {2, 32, 8, 2, 16, 128 * 1024},
    {4, 32, 8, 2, 16, 0}, {8, 32, 6, 2, 16, 0}};
  for (auto c : c2s) {
    R2Args A{}; A.w = w; A.m = m; A.n = n; A.nb = c.nb; A.tr = c.tr; A.stages = c.stages; A.ng = c.ng; A.nc = c.nc; A.reserve = c.reserve;
    A.tile_bytes = c.nb * 32 * 4 * c.tr;
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)m}; cuuint64_t str[1] = {(cuuint64_t)n * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)c.tr}; cuuint32_t es[2] = {1, 1};
    if (enc(&A.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode2 failed\n"); continue; }
    int smem = c.reserve + c.stages * A.tile_bytes + 2 * c.stages * 8 + 1024;
    if (smem > 227 * 1024) { printf("skip smem %d\n", smem); continue; }
    CK(cudaFuncSetAttribute(ring2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    double gbs = timeit([&] { ring2<<<sms, (c.nc + 1) * 32, smem>>>(A); });
    printf("ring2 rows=%3d B x %d, tr=%d S=%d ng=%d reserve=%3dK: %.0f GB/s\n", 128 * c.nb, 1, c.tr, c.stages, c.ng, c.reserve / 1024, gbs);
  }
  struct Cfg { int bn, tr, stages, ng, nc, reserve, ts; } cfgs[] = {
    {32, 64, 8, 1, 16, 128 * 1024, 0}, {32, 64, 8, 4, 16, 128 * 1024, 0}, {32, 64, 8, 8, 16, 128 * 1024, 0},
    {32, 64, 8, 4, 16, 128 * 1024, 1}, {32, 64, 8, 8, 16, 128 * 1024, 1},
    {32, 128, 4, 2, 16, 128 * 1024, 0}, {32, 128, 4, 4, 16, 128 * 1024, 0}, {32, 128, 4, 4, 16, 128 * 1024, 1},
    
    {32, 256, 2, 2, 16, 128 * 1024, 0}, {32, 64, 12, 4, 16, 64 * 1024, 0}, {32, 64, 12, 4, 16, 64 * 1024, 1},
    {32, 64, 8, 4, 24, 128 * 1024, 0}, {32, 64, 8, 8, 24, 128 * 1024, 0},
    {64, 64, 6, 3, 24, 128 * 1024, 0}, {64, 128, 3, 3, 24, 0, 0}, {128, 64, 6, 2, 16, 0, 0}, {128, 64, 6, 2, 16, 0, 1},
    {128, 64, 6, 3, 24, 0, 0}, {64, 64, 12, 4, 16, 0, 0}, {64, 64, 12, 4, 16, 0, 1}};
  for (auto c : cfgs) {
    RArgs A{}; A.w = w; A.m = m; A.n = n; A.bn = c.bn; A.tr = c.tr; A.stages = c.stages; A.ng = c.ng; A.nc = c.nc; A.reserve = c.reserve;
    A.tile_bytes = c.bn * c.tr * 4; A.tstore = c.ts;
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)m}; cuuint64_t str[1] = {(cuuint64_t)n * 4};
    cuuint32_t box[2] = {(cuuint32_t)c.bn, (cuuint32_t)c.tr}; cuuint32_t es[2] = {1, 1};
    if (enc(&A.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode failed\n"); continue; }
    int smem = c.reserve + c.stages * A.tile_bytes + 2 * c.stages * 8;
    if (smem > 227 * 1024) { printf("skip smem %d\n", smem); continue; }
    CK(cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    double gbs = timeit([&] { ring<<<sms, (c.nc + 1) * 32, smem>>>(A); });
    printf("ring bn=%3d tr=%3d S=%2d ng=%d nc=%d reserve=%3dK inflight=%3dK tstore=%d: %.0f GB/s\n", c.bn, c.tr, c.stages, c.ng, c.nc, c.reserve / 1024, c.stages * A.tile_bytes / 1024, c.ts, gbs);
  }
  for (int ns : {1, 0}) for (int cl : {1, 2, 4, 8}) for (int tr : {64, 128}) {
    const int stages = tr == 64 ? 8 : 4;
    RArgs A{}; A.w = w; A.m = m; A.n = n; A.bn = 32; A.tr = tr; A.stages = stages; A.ng = 2; A.nc = 16; A.reserve = 128 * 1024;
    A.tile_bytes = 32 * tr * 4; A.tstore = ns;
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)m}; cuuint64_t str[1] = {(cuuint64_t)n * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)tr}; cuuint32_t es[2] = {1, 1};
    if (enc(&A.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode failed\n"); continue; }
    int smem = A.reserve + stages * A.tile_bytes + 2 * stages * 8 + 16;
    CK(cudaFuncSetAttribute(ring3, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaLaunchConfig_t lc{}; cudaLaunchAttribute at[1];
    lc.gridDim = dim3(sms / cl * cl); lc.blockDim = dim3(17 * 32); lc.dynamicSmemBytes = smem;
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    lc.attrs = at; lc.numAttrs = 1;
    double gbs = timeit([&] { CK(cudaLaunchKernelEx(&lc, ring3, A)); });
    printf("ring3 lockstep=%d cluster=%d bn=32 tr=%d S=%d ng=2 reserve=128K: %.0f GB/s\n", !ns, cl, tr, stages, gbs);
  }
  for (int cl : {1, 2, 4, 8}) for (int tr : {32, 64, 128}) {
    const int stages = 4 * 128 / tr > 12 ? 12 : 4 * 128 / tr;
    RArgs A{}; A.w = w; A.m = m; A.n = n; A.bn = 32; A.tr = tr; A.stages = stages; A.ng = 2; A.nc = 16; A.reserve = 128 * 1024;
    A.tile_bytes = 32 * tr * 4;
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)m}; cuuint64_t str[1] = {(cuuint64_t)n * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)tr}; cuuint32_t es[2] = {1, 1};
    if (enc(&A.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode failed\n"); continue; }
    int smem = A.reserve + stages * A.tile_bytes + 2 * stages * 8 + 16;
    CK(cudaFuncSetAttribute(ring4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (cl > 1) CK(cudaFuncSetAttribute(ring4, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t lc{}; cudaLaunchAttribute at[1];
    lc.blockDim = dim3(17 * 32); lc.dynamicSmemBytes = smem;
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    lc.attrs = at; lc.numAttrs = 1;
    lc.gridDim = dim3(sms / cl * cl);
    int ncl = 0; CK(cudaOccupancyMaxActiveClusters(&ncl, ring4, &lc));
    lc.gridDim = dim3(ncl * cl);
    double gbs = timeit([&] { CK(cudaLaunchKernelEx(&lc, ring4, A)); });
    printf("ring4 multicast cluster=%d (active %d -> %d CTAs) tr=%d S=%d: %.0f GB/s\n", cl, ncl, ncl * cl, tr, stages, gbs);
  }
  return 0;
}
