// Compress stage 1, fixed-slot TMA kernel: Z^T = G^T P (n x d) for fp32
// accumulation of fp32 / bf16 G (reference: proj/src/projector.cpp:119-168,
// the G^T P half of S = P^T G Q).
//
// Same decomposition as k_compress_stage1 (compress.cu): one CTA = a band of
// columns of G x a range of subspace bins, accumulators in registers, G
// streamed once through shared memory in row chunks.  Each lane owns CPL
// adjacent columns (CPL = 1: 32-column bands, 32 bins per warp; CPL = 2:
// 64-column bands, 16 bins per warp, one 8-byte tile load per entry and lane),
// so an entry fetched once feeds 32*CPL column FMAs.  What changes is the
// entry walk.  The variable-length per-(chunk, bin) segments of the CSC table
// cost a loop, a bound test and a shuffle per bin; here every (chunk, bin)
// owns exactly K slots (rows ascending, padding slots read a zero row), so the
// per-chunk walk is a branch-free, fully unrolled sequence of 32 x K/2
// broadcast LDS.128 (two entries each) and 32 x K conflict-free tile loads +
// FMAs.  The few entries beyond K of a (chunk, bin) sit in a per-(chunk,
// 32-bin group) overflow list, prefetched one per lane while the slots run
// and applied afterwards through a warp-uniform switch on the bin.  The
// summation order per bin is still ascending rows, so results are bitwise
// those of k_compress_stage1.
//
// Data movement: per chunk, ceil(bm/256) 2-D TMA loads of the G tile
// (evict-first: G is read once) plus one 1-D bulk copy of the CTA's slot
// block, all completing on the stage's "full" mbarrier.  Thread 0 issues the
// first two chunks; afterwards the LAST warp to finish a chunk (elected with a
// shared-memory counter, after every warp arrived on the stage's "empty"
// mbarrier) refills that stage two chunks ahead.  No block-wide barrier in the
// loop, and the refill never waits for one particular warp.
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "core.cuh"
#include "tma.cuh"

namespace lspb {

namespace {

struct alignas(64) SMat {
  CUtensorMap tmap;  // G: box (32*CPL) cols x box_rows
  const EntryF* slots;
  const int* ovf_split;
  const EntryF* ovf;
  void* zt;
  int ldz, m, n, nchunks, band_end;
};
struct SArgs {
  SMat mat[kMaxGroup];
  int count, dpad, nwg, cpb, bm, nbox, box_rows;
  int stage_bytes, slot_off;
};

__device__ __forceinline__ uint4 lds128(unsigned a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}
// CPL consecutive tile elements of the lane, widened to float.
template <typename Tin, int CPL>
__device__ __forceinline__ void lds_g(unsigned a, float (&g)[CPL]) {
  if constexpr (std::is_same<Tin, float>::value) {
    if constexpr (CPL == 1) {
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(g[0]) : "r"(a));
    } else {
      asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(g[0]), "=f"(g[1]) : "r"(a));
    }
  } else {
    if constexpr (CPL == 1) {
      unsigned short h;
      asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(a));
      g[0] = __uint_as_float(static_cast<unsigned>(h) << 16);
    } else {
      unsigned w;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(a));
      g[0] = __uint_as_float(w << 16);
      g[1] = __uint_as_float(w & 0xffff0000u);
    }
  }
}

template <int CPL>
__device__ __forceinline__ void fma_bin(float (&acc)[32], int b, float v, const float (&g)[CPL]) {
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[b * CPL + c] = fmaf(v, g[c], acc[b * CPL + c]);
}

// acc[b*CPL + c] += v * g[c] for a warp-uniform runtime bin b < 32/CPL: one
// indirect branch (brx.idx jump table) instead of a compiler-built search tree.
// fma.rn.f32 is exactly fmaf, so results match the unrolled slot FMAs bitwise.
template <int CPL>
__device__ __forceinline__ void fma_bin_dyn(float (&acc)[32], int b, float v, const float (&g)[CPL]);
template <>
__device__ __forceinline__ void fma_bin_dyn<1>(float (&acc)[32], int b, float v, const float (&g)[1]) {
  asm volatile(
      "{\n"
      "ts%=: .branchtargets c0%=, c1%=, c2%=, c3%=, c4%=, c5%=, c6%=, c7%=, c8%=, c9%=, c10%=, c11%=, c12%=, c13%=, c14%=, c15%=, c16%=, c17%=, c18%=, c19%=, c20%=, c21%=, c22%=, c23%=, c24%=, c25%=, c26%=, c27%=, c28%=, c29%=, c30%=, c31%=;\n"
      "brx.idx.uni %32, ts%=;\n"
      "c0%=: fma.rn.f32 %0, %33, %34, %0; bra.uni e%=;\n"
      "c1%=: fma.rn.f32 %1, %33, %34, %1; bra.uni e%=;\n"
      "c2%=: fma.rn.f32 %2, %33, %34, %2; bra.uni e%=;\n"
      "c3%=: fma.rn.f32 %3, %33, %34, %3; bra.uni e%=;\n"
      "c4%=: fma.rn.f32 %4, %33, %34, %4; bra.uni e%=;\n"
      "c5%=: fma.rn.f32 %5, %33, %34, %5; bra.uni e%=;\n"
      "c6%=: fma.rn.f32 %6, %33, %34, %6; bra.uni e%=;\n"
      "c7%=: fma.rn.f32 %7, %33, %34, %7; bra.uni e%=;\n"
      "c8%=: fma.rn.f32 %8, %33, %34, %8; bra.uni e%=;\n"
      "c9%=: fma.rn.f32 %9, %33, %34, %9; bra.uni e%=;\n"
      "c10%=: fma.rn.f32 %10, %33, %34, %10; bra.uni e%=;\n"
      "c11%=: fma.rn.f32 %11, %33, %34, %11; bra.uni e%=;\n"
      "c12%=: fma.rn.f32 %12, %33, %34, %12; bra.uni e%=;\n"
      "c13%=: fma.rn.f32 %13, %33, %34, %13; bra.uni e%=;\n"
      "c14%=: fma.rn.f32 %14, %33, %34, %14; bra.uni e%=;\n"
      "c15%=: fma.rn.f32 %15, %33, %34, %15; bra.uni e%=;\n"
      "c16%=: fma.rn.f32 %16, %33, %34, %16; bra.uni e%=;\n"
      "c17%=: fma.rn.f32 %17, %33, %34, %17; bra.uni e%=;\n"
      "c18%=: fma.rn.f32 %18, %33, %34, %18; bra.uni e%=;\n"
      "c19%=: fma.rn.f32 %19, %33, %34, %19; bra.uni e%=;\n"
      "c20%=: fma.rn.f32 %20, %33, %34, %20; bra.uni e%=;\n"
      "c21%=: fma.rn.f32 %21, %33, %34, %21; bra.uni e%=;\n"
      "c22%=: fma.rn.f32 %22, %33, %34, %22; bra.uni e%=;\n"
      "c23%=: fma.rn.f32 %23, %33, %34, %23; bra.uni e%=;\n"
      "c24%=: fma.rn.f32 %24, %33, %34, %24; bra.uni e%=;\n"
      "c25%=: fma.rn.f32 %25, %33, %34, %25; bra.uni e%=;\n"
      "c26%=: fma.rn.f32 %26, %33, %34, %26; bra.uni e%=;\n"
      "c27%=: fma.rn.f32 %27, %33, %34, %27; bra.uni e%=;\n"
      "c28%=: fma.rn.f32 %28, %33, %34, %28; bra.uni e%=;\n"
      "c29%=: fma.rn.f32 %29, %33, %34, %29; bra.uni e%=;\n"
      "c30%=: fma.rn.f32 %30, %33, %34, %30; bra.uni e%=;\n"
      "c31%=: fma.rn.f32 %31, %33, %34, %31;\n"
      "e%=:\n}\n"
      : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3]), "+f"(acc[4]), "+f"(acc[5]), "+f"(acc[6]), "+f"(acc[7]), "+f"(acc[8]), "+f"(acc[9]), "+f"(acc[10]), "+f"(acc[11]), "+f"(acc[12]), "+f"(acc[13]), "+f"(acc[14]), "+f"(acc[15]), "+f"(acc[16]), "+f"(acc[17]), "+f"(acc[18]), "+f"(acc[19]), "+f"(acc[20]), "+f"(acc[21]), "+f"(acc[22]), "+f"(acc[23]), "+f"(acc[24]), "+f"(acc[25]), "+f"(acc[26]), "+f"(acc[27]), "+f"(acc[28]), "+f"(acc[29]), "+f"(acc[30]), "+f"(acc[31])
      : "r"(b), "f"(v), "f"(g[0]));
}
template <>
__device__ __forceinline__ void fma_bin_dyn<2>(float (&acc)[32], int b, float v, const float (&g)[2]) {
  asm volatile(
      "{\n"
      "ts%=: .branchtargets c0%=, c1%=, c2%=, c3%=, c4%=, c5%=, c6%=, c7%=, c8%=, c9%=, c10%=, c11%=, c12%=, c13%=, c14%=, c15%=;\n"
      "brx.idx.uni %32, ts%=;\n"
      "c0%=: fma.rn.f32 %0, %33, %34, %0; fma.rn.f32 %1, %33, %35, %1; bra.uni e%=;\n"
      "c1%=: fma.rn.f32 %2, %33, %34, %2; fma.rn.f32 %3, %33, %35, %3; bra.uni e%=;\n"
      "c2%=: fma.rn.f32 %4, %33, %34, %4; fma.rn.f32 %5, %33, %35, %5; bra.uni e%=;\n"
      "c3%=: fma.rn.f32 %6, %33, %34, %6; fma.rn.f32 %7, %33, %35, %7; bra.uni e%=;\n"
      "c4%=: fma.rn.f32 %8, %33, %34, %8; fma.rn.f32 %9, %33, %35, %9; bra.uni e%=;\n"
      "c5%=: fma.rn.f32 %10, %33, %34, %10; fma.rn.f32 %11, %33, %35, %11; bra.uni e%=;\n"
      "c6%=: fma.rn.f32 %12, %33, %34, %12; fma.rn.f32 %13, %33, %35, %13; bra.uni e%=;\n"
      "c7%=: fma.rn.f32 %14, %33, %34, %14; fma.rn.f32 %15, %33, %35, %15; bra.uni e%=;\n"
      "c8%=: fma.rn.f32 %16, %33, %34, %16; fma.rn.f32 %17, %33, %35, %17; bra.uni e%=;\n"
      "c9%=: fma.rn.f32 %18, %33, %34, %18; fma.rn.f32 %19, %33, %35, %19; bra.uni e%=;\n"
      "c10%=: fma.rn.f32 %20, %33, %34, %20; fma.rn.f32 %21, %33, %35, %21; bra.uni e%=;\n"
      "c11%=: fma.rn.f32 %22, %33, %34, %22; fma.rn.f32 %23, %33, %35, %23; bra.uni e%=;\n"
      "c12%=: fma.rn.f32 %24, %33, %34, %24; fma.rn.f32 %25, %33, %35, %25; bra.uni e%=;\n"
      "c13%=: fma.rn.f32 %26, %33, %34, %26; fma.rn.f32 %27, %33, %35, %27; bra.uni e%=;\n"
      "c14%=: fma.rn.f32 %28, %33, %34, %28; fma.rn.f32 %29, %33, %35, %29; bra.uni e%=;\n"
      "c15%=: fma.rn.f32 %30, %33, %34, %30; fma.rn.f32 %31, %33, %35, %31;\n"
      "e%=:\n}\n"
      : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3]), "+f"(acc[4]), "+f"(acc[5]), "+f"(acc[6]), "+f"(acc[7]), "+f"(acc[8]), "+f"(acc[9]), "+f"(acc[10]), "+f"(acc[11]), "+f"(acc[12]), "+f"(acc[13]), "+f"(acc[14]), "+f"(acc[15]), "+f"(acc[16]), "+f"(acc[17]), "+f"(acc[18]), "+f"(acc[19]), "+f"(acc[20]), "+f"(acc[21]), "+f"(acc[22]), "+f"(acc[23]), "+f"(acc[24]), "+f"(acc[25]), "+f"(acc[26]), "+f"(acc[27]), "+f"(acc[28]), "+f"(acc[29]), "+f"(acc[30]), "+f"(acc[31])
      : "r"(b), "f"(v), "f"(g[0]), "f"(g[1]));
}

template <typename Tin, int K, int CPL, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) k_compress_slots(const __grid_constant__ SArgs A) {
  constexpr int BPW = 32 / CPL;  // bins per warp (32 accumulators per lane)
  constexpr int NB = WARPS * BPW;  // bins per CTA
  constexpr int BC = 32 * CPL;     // band columns
  constexpr int ES = static_cast<int>(sizeof(Tin));
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem_raw + 2 * A.stage_bytes);
  unsigned long long* empty = full + 2;
  unsigned* done = reinterpret_cast<unsigned*>(empty + 2);  // [2] warps finished per stage
  // the CTAs of one band (bin ranges) are adjacent in launch order: G tiles
  // are fetched from HBM once and re-read from L2
  const int gband = blockIdx.x / A.cpb;
  const int bin_base = (blockIdx.x % A.cpb) * NB;
  int mi = 0;
  while (mi + 1 < A.count && gband >= A.mat[mi].band_end) ++mi;
  const SMat& M = A.mat[mi];
  const int band = gband - (mi ? A.mat[mi - 1].band_end : 0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int j0 = band * BC;
  const int bins = min(NB, A.dpad - bin_base);  // multiple of BPW
  const bool active = warp * BPW < bins;
  const int nchunks = M.nchunks;
  const unsigned slot_bytes = static_cast<unsigned>(bins) * K * 8u;

  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, WARPS);
      done[s] = 0u;
    }
    fence_mbar_init();
  }
  // zero rows (never written by TMA) right after each stage's tile
  if (tid < 2 * BC * ES / 4) {
    const int per = BC * ES / 4, s = tid / per;
    reinterpret_cast<float*>(smem_raw + s * A.stage_bytes + A.slot_off - BC * ES)[tid % per] = 0.0f;
  }
  __syncthreads();

  auto issue = [&](int c) {
    const int s = c & 1;
    unsigned char* base = smem_raw + s * A.stage_bytes;
    const int row0 = c * A.bm;
    const int nbox = min(A.nbox, (M.m - row0 + A.box_rows - 1) / A.box_rows);
    const unsigned box_bytes = static_cast<unsigned>(A.box_rows) * BC * ES;
    mbar_arrive_expect_tx(full + s, nbox * box_bytes + slot_bytes);
    const unsigned long long pol = policy_evict_first();
    for (int i = 0; i < nbox; ++i)
      tma_load_2d(base + i * box_bytes, &M.tmap, j0, row0 + i * A.box_rows, full + s, pol);
    bulk_load(base + A.slot_off,
              M.slots + (static_cast<long long>(c) * A.dpad + bin_base) * K, slot_bytes, full + s);
  };
  if (tid == 0) {
    issue(0);
    if (nchunks > 1) issue(1);
  }

  float acc[32];
#pragma unroll
  for (int b = 0; b < 32; ++b) acc[b] = 0.0f;
  const unsigned smem0 = smem_addr(smem_raw);
  const int wg = bin_base / BPW + warp;  // global bin group of this warp

  for (int c = 0; c < nchunks; ++c) {
    const int s = c & 1;
    const unsigned stage = smem0 + static_cast<unsigned>(s * A.stage_bytes);
    if (active) {
      // overflow bounds + the first 32 overflow entries, in flight during the slots
      const int* os = M.ovf_split + static_cast<long long>(c) * A.nwg + wg;
      const int o0 = __ldg(os), o1 = __ldg(os + 1);
      uint2 mine = make_uint2(0u, 0u);
      if (o0 + lane < o1) mine = __ldg(reinterpret_cast<const uint2*>(M.ovf + o0 + lane));
      mbar_wait(full + s, (c >> 1) & 1);
      const unsigned tl = stage + lane * CPL * ES;
      const unsigned sl = stage + A.slot_off + warp * BPW * K * 8;
#pragma unroll
      for (int b = 0; b < BPW; ++b) {
#pragma unroll
        for (int q = 0; q < K / 2; ++q) {
          const uint4 e = lds128(sl + (b * K + 2 * q) * 8);
          float g0[CPL], g1[CPL];
          lds_g<Tin, CPL>(tl + e.x, g0);
          lds_g<Tin, CPL>(tl + e.z, g1);
          fma_bin<CPL>(acc, b, __uint_as_float(e.y), g0);
          fma_bin<CPL>(acc, b, __uint_as_float(e.w), g1);
        }
      }
#pragma unroll 1
      for (int ob = o0; ob < o1; ob += 32) {
        if (ob != o0) {
          mine = make_uint2(0u, 0u);
          if (ob + lane < o1) mine = __ldg(reinterpret_cast<const uint2*>(M.ovf + ob + lane));
        }
        const int cnt = min(32, o1 - ob);
#pragma unroll 1
        for (int t = 0; t < cnt; ++t) {
          const unsigned pk = __shfl_sync(0xffffffffu, mine.x, t);
          const float v = __uint_as_float(__shfl_sync(0xffffffffu, mine.y, t));
          float g[CPL];
          lds_g<Tin, CPL>(tl + (pk & 0x7ffffffu), g);
          fma_bin_dyn<CPL>(acc, static_cast<int>(pk >> 27), v, g);
        }
      }
    } else {
      mbar_wait(full + s, (c >> 1) & 1);
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(empty + s);
      // the LAST warp to finish the chunk refills its stage (no coupling of
      // the refill to one warp's progress)
      if (c + 2 < nchunks && atomicAdd(done + s, 1u) == WARPS - 1) {
        done[s] = 0u;
        mbar_wait(empty + s, (c >> 1) & 1);
        issue(c + 2);
      }
    }
  }
  if (!active) return;
  const int bin0 = bin_base + warp * BPW;
#pragma unroll
  for (int cc = 0; cc < CPL; ++cc) {
    const int j = j0 + lane * CPL + cc;
    if (j >= M.n || bin0 >= M.ldz) continue;
    float* dst = static_cast<float*>(M.zt) + static_cast<long long>(j) * M.ldz + bin0;
    if (bin0 + BPW <= M.ldz && (M.ldz % 4) == 0) {
#pragma unroll
      for (int b = 0; b < BPW; b += 4)
        *reinterpret_cast<float4*>(dst + b) =
            make_float4(acc[b * CPL + cc], acc[(b + 1) * CPL + cc], acc[(b + 2) * CPL + cc],
                        acc[(b + 3) * CPL + cc]);
    } else {
#pragma unroll
      for (int b = 0; b < BPW; ++b)
        if (bin0 + b < M.ldz) dst[b] = acc[b * CPL + cc];
    }
  }
}

struct Geom {
  int K = 0, CPL = 0, bm = 0, nbox = 0, box_rows = 0, stage_bytes = 0, slot_off = 0;
};

// Chunk geometry: the largest bm whose double-buffered stage (tile + zero row
// + the CTA's slot block) fits the per-CTA shared-memory budget.
Geom geometry(int K, int CPL, int esize, int cta_bins, int budget) {
  Geom g{};
  const int row_bytes = 32 * CPL * esize;
  const int slot_bytes = cta_bins * K * 8;
  const int per_stage = (budget - 64) / 2;
  const int bm_max = (per_stage - 128 - slot_bytes - row_bytes) / row_bytes;
  if (bm_max < 8) return g;
  g.K = K, g.CPL = CPL;
  g.nbox = ceil_div(bm_max, 256);
  g.box_rows = std::max(8, (bm_max / g.nbox) / 8 * 8);
  g.bm = g.box_rows * g.nbox;
  g.slot_off = slot_zero_off(g.bm, row_bytes) + row_bytes;
  g.stage_bytes = static_cast<int>(round_up(g.slot_off + slot_bytes, 128));
  return g;
}

template <typename Tin, int K, int CPL>
void launch_slots(const SArgs& A, int warps, dim3 grid, int smem, cudaStream_t st) {
  auto go = [&](auto kern, int nt) {
    LSP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, nt, smem, st>>>(A);
  };
  if (warps == 32)
    go(k_compress_slots<Tin, K, CPL, 32>, 1024);
  else
    go(k_compress_slots<Tin, K, CPL, 8>, 256);
}

template <typename Tin>
bool slots_impl(const std::vector<S1Job>& jobs, lsp_dtype gdt, cudaStream_t st) {
  const int d = jobs[0].pr->d;
  const int dpad = static_cast<int>(round_up(d, 32));
  const int esize = static_cast<int>(sizeof(Tin));
  // Candidates (CPL, K); time model per (chunk, warp): issue slots / 4 +
  // shared-memory wavefronts (broadcast LDS.128 = 2, a lane-row load = CPL);
  // an overflow entry ~(24 instructions, CPL + 1 wavefronts).
  static const int kCand[][2] = {{1, 2}, {1, 4}, {1, 8}, {2, 2}, {2, 4}};
  // LSP_COMPRESS_SLOTS="CPL,K" pins a candidate (benchmarking aid)
  int pin_cpl = 0, pin_k = 0;
  if (const char* pin = std::getenv("LSP_COMPRESS_SLOTS")) std::sscanf(pin, "%d,%d", &pin_cpl, &pin_k);
  Geom best{};
  int best_warps = 32;
  double best_cost = 0.0;
  for (const auto& cand : kCand) {
    const int CPL = cand[0], K = cand[1], BPW = 32 / CPL;
    if (pin_cpl && (CPL != pin_cpl || K != pin_k)) continue;
    const int warps = dpad / BPW > 8 ? 32 : 8;
    const int cta_bins = std::min(warps * BPW, dpad);
    const int budget = warps == 32 ? 226 * 1024 : 72 * 1024;
    const Geom g = geometry(K, CPL, esize, cta_bins, budget);
    if (g.bm == 0) continue;
    double cost = 0.0;
    for (const S1Job& J : jobs) {
      const double bands = ceil_div(J.pr->n, 32 * CPL);
      const double chunks = ceil_div(J.pr->m, g.bm);
      const double per_warp = BPW * (K / 2 * 2.0 + K * CPL + (K / 2 + K * (2 + CPL)) / 4.0) + 20;
      cost += bands * chunks * (dpad / BPW) * per_warp +
              bands * (CPL + 1 + 24 / 4.0) * J.pr->p->overflow(K, g.bm);
    }
    if (best.bm == 0 || cost < best_cost) best = g, best_cost = cost, best_warps = warps;
  }
  if (best.bm == 0) return false;
  const int BPW = 32 / best.CPL, BC = 32 * best.CPL;
  SArgs A{};
  A.count = static_cast<int>(jobs.size());
  A.dpad = dpad;
  A.nwg = dpad / BPW;
  A.cpb = ceil_div(dpad, best_warps * BPW);
  A.bm = best.bm;
  A.nbox = best.nbox;
  A.box_rows = best.box_rows;
  A.stage_bytes = best.stage_bytes;
  A.slot_off = best.slot_off;
  int bands = 0;
  for (size_t i = 0; i < jobs.size(); ++i) {
    const S1Job& J = jobs[i];
    const Pair& pr = *J.pr;
    SMat& M = A.mat[i];
    if (!cached_tmap(&M.tmap, J.g, gdt, pr.m, pr.n, J.ldg, BC, best.box_rows)) return false;
    const SlotTable& t = pr.p->slot_table(best.bm, BC * esize, best.K, BPW);
    M.slots = t.slots.as<EntryF>();
    M.ovf_split = t.ovf_split.as<int>();
    M.ovf = t.ovf.as<EntryF>();
    M.zt = J.zt;
    M.ldz = pr.ldz();
    M.m = pr.m, M.n = pr.n;
    M.nchunks = t.nchunks;
    bands += ceil_div(pr.n, BC);
    M.band_end = bands;
  }
  if (bands == 0) return true;
  const int smem = 2 * best.stage_bytes + 64;
  const dim3 grid(bands * A.cpb);
  switch (best.CPL * 16 + best.K) {
    case 16 + 2: launch_slots<Tin, 2, 1>(A, best_warps, grid, smem, st); break;
    case 16 + 4: launch_slots<Tin, 4, 1>(A, best_warps, grid, smem, st); break;
    case 16 + 8: launch_slots<Tin, 8, 1>(A, best_warps, grid, smem, st); break;
    case 32 + 2: launch_slots<Tin, 2, 2>(A, best_warps, grid, smem, st); break;
    default: launch_slots<Tin, 4, 2>(A, best_warps, grid, smem, st); break;
  }
  after_launch("compress_slots");
  return true;
}

}  // namespace

// Fixed-slot fast path of launch_compress_stage1_group; false when the group
// is not eligible (fp64 accumulation, fp64 G, G not TMA-describable, or
// LSP_COMPRESS_GENERIC=1), in which case the caller runs k_compress_stage1.
bool launch_compress_slots_group(const std::vector<S1Job>& jobs, lsp_dtype gdt, cudaStream_t st) {
  if (jobs.empty()) return false;
  const Pair& p0 = *jobs[0].pr;
  if (p0.compute != LSP_F32 || gdt == LSP_F64) return false;
  const char* env = std::getenv("LSP_COMPRESS_GENERIC");
  if (env && env[0] == '1') return false;
  return gdt == LSP_F32 ? slots_impl<float>(jobs, gdt, st) : slots_impl<bf16>(jobs, gdt, st);
}

}  // namespace lspb
