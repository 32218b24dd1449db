// Compress stage 1, gather form: Z^T = G^T P (n x d) for fp32 accumulation of
// fp32 / bf16 G, and fp64 accumulation of fp64 G (the reference's precision)
// (reference: the G^T P half of S = P^T G Q, proj/src/projector.cpp:119-168;
// compress :163-168).
//
// Z[b][:] = sum_{i in CSC_P(b)} p(i,b) * G[i][:] is a sparse x dense product
// whose sparse factor has ~m*r/d entries per output row.  One warp computes
// one bin b for one column tile (128 fp32 / 256 bf16 columns, 16 bytes per
// lane): it walks the bin's CSC entries (rows ascending, the reference's
// summation order) and gathers the 512-byte row segments G[i][tile] straight
// from global memory with 16-byte loads, U of them in flight per warp.  The
// 32 CTAs that cover the bin groups of one column tile run together, so each
// G tile is fetched from HBM once and re-read r times from L2; there is no
// shared-memory staging of G, no padding and no overflow path, and warps of a
// CTA never wait on each other inside a bin.  A CTA owns one (column tile,
// 32-bin group) item at a time and writes its Z^T block (tile rows x 32 bins,
// 128-byte row segments) through a shared-memory transpose.
//
// Persistent grid, two 8-warp CTAs per SM (one streams while the other is in
// its item barrier / transposed write); items are ordered (matrix, column
// tile, bin group) and handed out with a stride of gridDim.x, so the tiles in
// flight at any moment are a small L2-resident window of G.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "core.cuh"
#include "tma.cuh"  // mbarrier / bulk-copy helpers

namespace lspb {

namespace {

constexpr int kBG = 32;      // bins per item (kBG / kSWarps per warp; 64 measured slower)
constexpr int kSWarps = 8;   // warps per CTA
constexpr int kSCtas = 2;    // CTAs per SM: one streams while the other syncs/transposes
constexpr int kSThreads = kSWarps * 32;

struct PMat {
  const void* g;
  long long ldg;
  const int* ptr;       // CSC_P offsets [d + 1]
  const void* ent;      // CSC_P entries {row, value}: EntryF (fp32) / EntryD (fp64)
  void* zt;
  int ldz, n, ntiles;
  long long item_end;
};
struct PArgs {
  PMat mat[kMaxGroup];
  int count, d, ngroups, ebuf_bytes;
  long long total;
};

__host__ __device__ constexpr int round_up16(int b) { return (b + 15) & ~15; }

template <typename Tin>
struct Vec;
template <>
struct Vec<float> {
  static constexpr int CPL = 4;
  __device__ __forceinline__ static void load(const void* p, float (&g)[4]) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    g[0] = v.x, g[1] = v.y, g[2] = v.z, g[3] = v.w;
  }
};
template <>
struct Vec<double> {
  static constexpr int CPL = 2;
  __device__ __forceinline__ static void load(const void* p, double (&g)[2]) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(p));
    g[0] = v.x, g[1] = v.y;
  }
};
template <>
struct Vec<bf16> {
  static constexpr int CPL = 8;
  __device__ __forceinline__ static void load(const void* p, float (&g)[8]) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      g[2 * t] = __uint_as_float(w[t] << 16);
      g[2 * t + 1] = __uint_as_float(w[t] & 0xffff0000u);
    }
  }
};

// entry words as loaded: {row, fp32 value bits} / {row, pad, fp64 value}
template <typename Tacc>
struct EntW;
template <>
struct EntW<float> {
  using E = EntryF;
  using W = uint2;
  __device__ __forceinline__ static float val(const W& w) { return __uint_as_float(w.y); }
};
template <>
struct EntW<double> {
  using E = EntryD;
  using W = uint4;
  __device__ __forceinline__ static double val(const W& w) {
    return __hiloint2double(static_cast<int>(w.w), static_cast<int>(w.z));
  }
};

template <typename Tin, typename Tacc, int U>
__global__ void __launch_bounds__(kSThreads, kSCtas) k_compress_spmm(const __grid_constant__ PArgs A) {
  constexpr int CPL = Vec<Tin>::CPL;
  constexpr int CT = 32 * CPL;  // columns per tile
  constexpr int LDS = CT + 1;   // padded row of the transpose buffer
  using E = typename EntW<Tacc>::E;
  using EW = typename EntW<Tacc>::W;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Tacc* zs = reinterpret_cast<Tacc*>(smem_raw);                         // [2][kBG][LDS]
  unsigned char* ebuf = smem_raw + 2 * kBG * LDS * sizeof(Tacc);        // [2][A.ebuf_bytes]
  unsigned long long* ebar = reinterpret_cast<unsigned long long*>(ebuf + 2 * A.ebuf_bytes);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rot = lane / (32 / CPL);  // store rotation: conflict-free transposed writes

  struct It {
    int mi, j0, b0, elo;
  };
  auto item_at = [&](long long item) {
    int mi = 0;
    while (mi + 1 < A.count && item >= A.mat[mi].item_end) ++mi;
    // 32-bit arithmetic: a matrix has < 2^31 items
    const int lt = static_cast<int>(item - (mi ? A.mat[mi - 1].item_end : 0));
    const int tile = lt / A.ngroups;
    const int b0 = (lt - tile * A.ngroups) * kBG;
    const int elo = __ldg(A.mat[mi].ptr + b0);  // padded table: 64-byte aligned
    return It{mi, tile * CT, b0, elo};
  };
  // bulk-copy the CSC entries of an item's 32 bins into entry buffer `b`
  auto stage = [&](long long item, int b) {
    const It t = item_at(item);
    const PMat& M = A.mat[t.mi];
    const int ehi = __ldg(M.ptr + min(t.b0 + kBG, A.d));
    const unsigned bytes = static_cast<unsigned>(round_up16((ehi - t.elo) * static_cast<int>(sizeof(E))));
    mbar_arrive_expect_tx(ebar + b, bytes);
    if (bytes) bulk_load(ebuf + b * A.ebuf_bytes, static_cast<const E*>(M.ent) + t.elo, bytes, ebar + b);
  };

  if (threadIdx.x == 0) {
    mbar_init(ebar, 1);
    mbar_init(ebar + 1, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const long long first = blockIdx.x;
  if (threadIdx.x == 0) {
    if (first < A.total) stage(first, 0);
    if (first + gridDim.x < A.total) stage(first + gridDim.x, 1);
  }
  int k = 0;
  for (long long item = first; item < A.total; item += gridDim.x, ++k) {
    const int buf = k & 1;
    const It t = item_at(item);
    const PMat& M = A.mat[t.mi];
    const int jl = t.j0 + lane * CPL;
    // per-item constants in registers; a lane whose columns lie beyond n reads
    // column 0 instead (valid memory) and its results are never written
    const unsigned char* gcol = static_cast<const unsigned char*>(M.g) +
                                (jl < M.n ? jl : 0) * static_cast<int>(sizeof(Tin));
    const unsigned ldgb = static_cast<unsigned>(M.ldg * sizeof(Tin));  // < 4 GiB (host check)
    const E* es = reinterpret_cast<const E*>(ebuf + buf * A.ebuf_bytes) - t.elo;
    Tacc* z = zs + buf * kBG * LDS;
    mbar_wait(ebar + buf, (k >> 1) & 1);

    // This warp's two bins as one stream of U-entry batches (bins are padded
    // to whole batches: pads repeat the bin's last row with value 0, an L1
    // hit that adds +0), double-buffered: batch i+1's gathers are in flight
    // while batch i is consumed; ~7 instructions per entry, no predicates.
    constexpr int NBW = kBG / kSWarps;  // bins per warp: t.b0 + warp + w*kSWarps
    // per-bin entry start and batch count, indexed only with compile-time
    // indices (register-resident; dynamic lookups go through select chains)
    int es_w[NBW], nb_w[NBW];
    int nb = 0;
#pragma unroll
    for (int w = 0; w < NBW; ++w) {
      const int b = t.b0 + warp + w * kSWarps;
      const int e0 = b < A.d ? __ldg(M.ptr + b) : 0, e1 = b < A.d ? __ldg(M.ptr + b + 1) : 0;
      es_w[w] = e0;
      nb_w[w] = (e1 - e0) / U;
      nb += nb_w[w];
    }
    auto sel = [](const int (&arr)[NBW], int w) {
      int r = arr[0];
#pragma unroll
      for (int x = 1; x < NBW; ++x)
        if (w == x) r = arr[x];
      return r;
    };
    Tacc acc[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] = Tacc(0);
    auto flush = [&](int bb) {
      // z[bb][lane*CPL + c], components rotated per lane group so that the
      // CPL stores of a warp each hit 32 distinct banks
      Tacc* zr = z + bb * LDS + lane * CPL;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int cc = (c + rot) % CPL;
        Tacc v = acc[0];
#pragma unroll
        for (int q = 1; q < CPL; ++q)
          if (cc == q) v = acc[q];
        zr[cc] = v;
      }
#pragma unroll
      for (int c = 0; c < CPL; ++c) acc[c] = Tacc(0);
    };
    // load cursor (bin lb, next batch at lsrc, lleft batches left in the bin)
    int lb = 0, lleft = nb_w[0];
    const E* lsrc = es + es_w[0];
    auto load_skip = [&]() {
      while (lleft == 0 && lb < NBW - 1) {
        ++lb;
        lleft = sel(nb_w, lb);
        lsrc = es + sel(es_w, lb);
      }
    };
    load_skip();
    EW ena[U], enb[U];
    Tacc ga[U][CPL], gb[U][CPL];
    auto load = [&](EW (&en)[U], Tacc (&g)[U][CPL]) {
      const E* src = lsrc;
      lsrc += U;
      if (--lleft == 0) load_skip();
#pragma unroll
      for (int u = 0; u < U; ++u) en[u] = *reinterpret_cast<const EW*>(src + u);
#pragma unroll
      for (int u = 0; u < U; ++u)
        Vec<Tin>::load(gcol + static_cast<unsigned long long>(en[u].x * ldgb), g[u]);
    };
    // consume cursor: bin cb, cleft batches left in it; completed bins flushed
    int cb = 0, cleft = nb_w[0];
    auto consume = [&](const EW (&en)[U], const Tacc (&g)[U][CPL]) {
      while (cleft == 0 && cb < NBW - 1) {
        flush(warp + cb * kSWarps);
        ++cb;
        cleft = sel(nb_w, cb);
      }
      --cleft;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const Tacc p = EntW<Tacc>::val(en[u]);
        if constexpr (sizeof(Tacc) == 4) {
          // packed FFMA2: two IEEE fmas per instruction, same per-column chain
          const float2 pp = make_float2(p, p);
#pragma unroll
          for (int c = 0; c < CPL; c += 2) {
            const float2 r = __ffma2_rn(pp, make_float2(g[u][c], g[u][c + 1]), make_float2(acc[c], acc[c + 1]));
            acc[c] = r.x;
            acc[c + 1] = r.y;
          }
        } else {
#pragma unroll
          for (int c = 0; c < CPL; ++c) acc[c] = __fma_rn(p, g[u][c], acc[c]);
        }
      }
    };
    if constexpr (U * CPL <= 32) {  // registers for two batches: double-buffered
      if (nb > 0) load(ena, ga);
      for (int i = 0; i < nb; i += 2) {
        if (i + 1 < nb) load(enb, gb);
        consume(ena, ga);
        if (i + 1 >= nb) break;
        if (i + 2 < nb) load(ena, ga);
        consume(enb, gb);
      }
    } else {  // one (wider) batch in flight
      for (int i = 0; i < nb; ++i) {
        load(ena, ga);
        consume(ena, ga);
      }
    }
    for (; cb < NBW; ++cb) flush(warp + cb * kSWarps);  // the remaining bins
    __syncthreads();  // z[buf] complete; entry buffer `buf` free
    if (threadIdx.x == 0 && item + 2 * gridDim.x < A.total) stage(item + 2 * gridDim.x, buf);
    // Z^T[j0 + c][b0 + h*32 + lane]: 128-byte row segments per column
    for (int c = warp; c < CT; c += kSWarps) {
      const int j = t.j0 + c;
      if (j >= M.n) continue;
#pragma unroll
      for (int h = 0; h < kBG / 32; ++h)
        if (t.b0 + h * 32 + lane < A.d)
          static_cast<Tacc*>(M.zt)[static_cast<long long>(j) * M.ldz + t.b0 + h * 32 + lane] =
              z[(h * 32 + lane) * LDS + c];
    }
    // z[buf] is rewritten two items later, after the next __syncthreads
  }
}

template <typename Tin, typename Tacc>
bool spmm_impl(const std::vector<S1Job>& jobs, cudaStream_t st) {
  constexpr int CPL = Vec<Tin>::CPL;
  constexpr int ES = static_cast<int>(sizeof(typename EntW<Tacc>::E));
  constexpr int CT = 32 * CPL;
  const Pair& p0 = *jobs[0].pr;
  PArgs A{};
  A.count = static_cast<int>(jobs.size());
  A.d = p0.d;
  A.ngroups = ceil_div(p0.d, kBG);
  long long total = 0;
  for (size_t i = 0; i < jobs.size(); ++i) {
    const S1Job& J = jobs[i];
    const Pair& pr = *J.pr;
    // 16-byte row segments: G aligned, columns and leading dimension in whole vectors
    if (reinterpret_cast<uintptr_t>(J.g) % 16 || pr.n % CPL || J.ldg % CPL) return false;
    if (static_cast<unsigned long long>(pr.m) * J.ldg * sizeof(Tin) >= (1ull << 32)) return false;
    PMat& M = A.mat[i];
    M.g = J.g;
    M.ldg = J.ldg;
    const Projector::PadTable& pt = pr.p->csc_padded();
    M.ptr = pt.ptr.as<int>();
    M.ent = pt.ent.p;
    M.zt = J.zt;
    M.ldz = pr.ldz();
    M.n = pr.n;
    M.ntiles = ceil_div(pr.n, CT);
    total += static_cast<long long>(M.ntiles) * A.ngroups;
    M.item_end = total;
  }
  A.total = total;
  if (total == 0) return true;
  // entry buffer: the largest 32-bin CSC range of any matrix (+16 B alignment slack)
  int emax = 0;
  for (const S1Job& J : jobs) {
    const std::vector<int32_t>& ptr = J.pr->p->csc_padded().h_ptr;
    for (int b0 = 0; b0 < p0.d; b0 += kBG)
      emax = std::max(emax, ptr[std::min(b0 + kBG, p0.d)] - ptr[b0]);
  }
  A.ebuf_bytes = round_up16(emax * ES + 16);
  const int smem = 2 * kBG * (CT + 1) * static_cast<int>(sizeof(Tacc)) + 2 * A.ebuf_bytes + 16;
  if (smem > 227 * 1024) return false;
  // U = pad unit (fp32); fp64 keeps half the loads in flight (register budget)
  auto kern = k_compress_spmm<Tin, Tacc, sizeof(Tacc) == 4 ? Projector::kPadU : Projector::kPadU / 2>;
  LSP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid = static_cast<int>(std::min<long long>(total, kSCtas * sm_budget(kBudgetCompress)));
  kern<<<grid, kSThreads, smem, st>>>(A);
  after_launch("compress_spmm");
  return true;
}

}  // namespace

// Gather-form stage 1 (fp32 accumulation, fp32/bf16 G); false when the group
// is not eligible.  The default stage 1 for fp32 accumulation: measured on
// B200 at or below the fixed-slot kernel for every BASELINE config (C4 fp32
// 13.46 vs 13.57 ms per step of compress, C4 bf16 9.7 vs 12.6, C3 3.1 vs
// 3.6, C2 2.7 vs 3.7).  LSP_COMPRESS_SPMM=0 falls back to the slot kernel.
bool launch_compress_spmm_group(const std::vector<S1Job>& jobs, lsp_dtype gdt, cudaStream_t st) {
  if (jobs.empty()) return false;
  const char* gen = std::getenv("LSP_COMPRESS_GENERIC");
  if (gen && gen[0] == '1') return false;
  const Pair& p0 = *jobs[0].pr;
  const char* env = std::getenv("LSP_COMPRESS_SPMM");
  if (env && env[0] == '0') return false;
  if (p0.compute == LSP_F64) return gdt == LSP_F64 && spmm_impl<double, double>(jobs, st);
  if (p0.compute != LSP_F32 || (gdt != LSP_F32 && gdt != LSP_BF16)) return false;
  return gdt == LSP_F32 ? spmm_impl<float, float>(jobs, st) : spmm_impl<bf16, float>(jobs, st);
}

}  // namespace lspb
