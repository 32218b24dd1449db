// Compress: S = P^T G Q  (reference: proj/src/projector.cpp:119-168).
//
// Two stages, both written for HBM-bound streaming on sm_100a:
//
//  stage 1  Z^T = G^T P  (n x d).  One CTA owns a band of 32 columns of G and
//           every subspace bin (32 bins per warp, accumulators in registers:
//           lane = column, register = bin).  G is streamed ONCE, row chunk by
//           row chunk, through a cp.async double buffer; the chunk-major CSC
//           table of P says which tile rows feed which bin, so every G element
//           is read from HBM once and from shared memory k times (conflict-
//           free: a warp reads one 32-wide tile row).  No atomics, fixed
//           summation order -> bitwise deterministic.
//  stage 2  S^T[b][:] = sum_{j in CSC_Q(b)} q_jb Z^T[j][:]  -- coalesced row
//           gathers of the L2-resident Z^T (k_gather).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "adam_math.cuh"
#include "core.cuh"

namespace lspb {

namespace {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Load rows [row0, row0+bm) x cols [j0, j0+32) of G into a bm x 32 tile.
// Rows >= m are skipped (never referenced); columns >= n are zero-filled.
template <typename Tin, int NT>
__device__ __forceinline__ void load_tile(Tin* tile, const Tin* __restrict__ g, long long ldg,
                                          int m, int n, int row0, int j0, int bm, bool vec) {
  constexpr int kPer16 = 16 / sizeof(Tin);       // elements per 16 B
  constexpr int kPieces = 32 / kPer16;           // 16 B pieces per tile row
  const int tid = threadIdx.x;
  const int rows = min(bm, m - row0);
  if (vec) {
#pragma unroll 4
    for (int p = tid; p < rows * kPieces; p += NT) {
      const int row = p / kPieces, piece = p % kPieces;
      const int gc = j0 + piece * kPer16;
      const int valid = min(kPer16, n - gc);
      const Tin* src = g + static_cast<long long>(row0 + row) * ldg + (valid > 0 ? gc : 0);
      cp_async16(tile + row * 32 + piece * kPer16, src, valid > 0 ? valid * (int)sizeof(Tin) : 0);
    }
  } else {
    for (int p = tid; p < rows * 32; p += NT) {
      const int row = p >> 5, col = p & 31;
      const int gc = j0 + col;
      tile[p] = gc < n ? g[static_cast<long long>(row0 + row) * ldg + gc] : Tin(0.0f);
    }
  }
}

// One stage-1 job (matrix) of a grouped launch.
struct S1Mat {
  const void* g;
  long long ldg;
  int m, n;
  const int* split;
  const void* ent;
  int nchunks;
  void* zt;
  int ldz;
  int band_end;  // exclusive prefix of bands over the group
  int vec;
};
struct S1Args {
  S1Mat mat[kMaxGroup];
  int count;
  int d;
  int r;
  int bm;           // rows per chunk (the chunk tables were built for it)
  int tile_bytes;   // per-stage G tile bytes (16-aligned)
  int ent_bytes;    // per-stage entry bytes (16-aligned)
};

// One CTA = one band of 32 columns of one matrix x (WARPS*32) bins.  Per row
// chunk, the G tile AND the chunk's CSC(P) entries are staged into shared
// memory by cp.async (double buffered), so the inner loop has no global loads.
template <typename Tin, typename Tacc, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) k_compress_stage1(const __grid_constant__ S1Args A) {
  using Ent = typename EntryOf<Tacc>::type;
  constexpr int NT = WARPS * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int stage_bytes = A.tile_bytes + A.ent_bytes;
  // which matrix / band (uniform scan over <= kMaxGroup entries)
  int mi = 0;
  while (mi + 1 < A.count && static_cast<int>(blockIdx.x) >= A.mat[mi].band_end) ++mi;
  const S1Mat& M = A.mat[mi];
  const int band = blockIdx.x - (mi ? A.mat[mi - 1].band_end : 0);
  const Tin* __restrict__ g = static_cast<const Tin*>(M.g);
  const Ent* __restrict__ ent = static_cast<const Ent*>(M.ent);
  const int* __restrict__ split = M.split;
  const int d = A.d, m = M.m, n = M.n, bm = A.bm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j0 = band * 32;
  const int bin0 = blockIdx.y * NT + warp * 32;
  const int my_bin = bin0 + lane;
  const bool vec16 = M.vec != 0;

  auto stage = [&](int c, int buf) {
    unsigned char* base = smem_raw + buf * stage_bytes;
    load_tile<Tin, NT>(reinterpret_cast<Tin*>(base), g, M.ldg, m, n, c * bm, j0, bm, vec16);
    // the chunk's (even-padded) entries are contiguous in the table
    const int e0 = __ldg(split + static_cast<long long>(c) * d);
    const int e1 = __ldg(split + static_cast<long long>(c + 1) * d);
    const int bytes = (e1 - e0) * static_cast<int>(sizeof(Ent));
    const char* src = reinterpret_cast<const char*>(ent + e0);
    char* dst = reinterpret_cast<char*>(base + A.tile_bytes);
    for (int p = threadIdx.x * 16; p < bytes; p += NT * 16)
      cp_async16(dst + p, src + p, min(16, bytes - p));
  };

  Tacc acc[32];
#pragma unroll
  for (int b = 0; b < 32; ++b) acc[b] = Tacc(0);

  stage(0, 0);
  cp_async_commit();
  for (int c = 0; c < M.nchunks; ++c) {
    // Chunk c+1 goes to the other buffer; the barrier below the wait also
    // guarantees every warp has finished reading it (chunk c-1).
    cp_async_wait<0>();
    __syncthreads();
    if (c + 1 < M.nchunks) stage(c + 1, (c + 1) & 1);
    cp_async_commit();
    const unsigned char* base = smem_raw + (c & 1) * stage_bytes;
    const unsigned char* tb = base + lane * sizeof(Tin);  // + entry byte offset = G[row][lane]
    // Entries of (chunk c, bin) are contiguous, even-padded, and bins follow
    // each other, so bin b's range is [end(b-1), end(b)).
    const long long sbase = static_cast<long long>(c) * d;
    const int cbeg = __ldg(split + sbase);
    const Ent* E = reinterpret_cast<const Ent*>(base + A.tile_bytes) - cbeg;
    int e = __ldg(split + sbase + min(bin0, d));
    const int my_end = __ldg(split + sbase + min(my_bin + 1, d));
    if constexpr (std::is_same<Tin, float>::value && std::is_same<Tacc, float>::value) {
      // Two entries per 16-byte load; bra.uni keeps the warp-uniform loop free
      // of divergence bookkeeping.
      const unsigned e_base = smem_u32(base + A.tile_bytes) - static_cast<unsigned>(cbeg) * 8u;
      const unsigned t_lane = smem_u32(tb);
      unsigned ep = e_base + static_cast<unsigned>(e) * 8u;
      // software pipeline: the current pair {o0, v0, o1, v1} is always preloaded
      // (the stage has 16 bytes of slack, so preloading past the end is safe)
      unsigned o0, w0, o1, w1;
      asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(o0), "=r"(w0), "=r"(o1), "=r"(w1) : "r"(ep));
#pragma unroll
      for (int b = 0; b < 32; ++b) {
        unsigned ep_end = e_base + static_cast<unsigned>(__shfl_sync(0xffffffffu, my_end, b)) * 8u;
        float a = acc[b];
        asm volatile(
            "{\n\t.reg .pred p;\n\t.reg .b32 a0, a1;\n\t.reg .f32 v0, v1, g0, g1;\n"
            "LSPS1_L%=:\n\t"
            "setp.ge.u32 p, %1, %2;\n\t"
            "@p bra.uni LSPS1_E%=;\n\t"
            "add.u32 a0, %3, %7;\n\t"
            "add.u32 a1, %5, %7;\n\t"
            "mov.b32 v0, %4;\n\t"
            "mov.b32 v1, %6;\n\t"
            "ld.shared.f32 g0, [a0];\n\t"
            "ld.shared.f32 g1, [a1];\n\t"
            "add.u32 %1, %1, 16;\n\t"
            "ld.shared.v4.b32 {%3, %4, %5, %6}, [%1];\n\t"
            "fma.rn.f32 %0, v0, g0, %0;\n\t"
            "fma.rn.f32 %0, v1, g1, %0;\n\t"
            "bra.uni LSPS1_L%=;\n"
            "LSPS1_E%=:\n\t}"
            : "+f"(a), "+r"(ep), "+r"(ep_end), "+r"(o0), "+r"(w0), "+r"(o1), "+r"(w1)
            : "r"(t_lane)
            : "memory");
        acc[b] = a;
      }
    } else {
#pragma unroll
      for (int b = 0; b < 32; ++b) {
        const int end = __shfl_sync(0xffffffffu, my_end, b);
        Tacc a = acc[b];
#pragma unroll 1
        for (; e < end; e += 2) {  // segments are even-padded
          const Ent e0 = E[e], e1 = E[e + 1];
          const Tacc g0 = cvt<Tacc>(*reinterpret_cast<const Tin*>(tb + e0.off));
          const Tacc g1 = cvt<Tacc>(*reinterpret_cast<const Tin*>(tb + e1.off));
          a = fma(e0.val, g0, a);
          a = fma(e1.val, g1, a);
        }
        acc[b] = a;
      }
    }
  }
  const int j = j0 + lane;
  if (j < n) {
    Tacc* dst = static_cast<Tacc*>(M.zt) + static_cast<long long>(j) * M.ldz + bin0;
    if (bin0 + 32 <= M.ldz && (M.ldz % 4) == 0 && sizeof(Tacc) == 4) {
#pragma unroll
      for (int b = 0; b < 32; b += 4)
        *reinterpret_cast<float4*>(dst + b) =
            make_float4((float)acc[b], (float)acc[b + 1], (float)acc[b + 2], (float)acc[b + 3]);
    } else {
#pragma unroll
      for (int b = 0; b < 32; ++b)
        if (bin0 + b < M.ldz) dst[b] = acc[b];
    }
  }
}

template <typename Tin, typename Tacc, int WARPS>
void stage1_impl(const std::vector<S1Job>& jobs, int d, cudaStream_t st) {
  using Ent = typename EntryOf<Tacc>::type;
  const int r = jobs[0].pr->p->r;
  // Per-stage budget: ~100 KB (two stages fit the 227 KB of an SM) for the
  // 32-warp kernel, half that for smaller CTAs so several fit per SM.
  const int budget = (WARPS >= 16 ? 100 * 1024 : 48 * 1024) - d * static_cast<int>(sizeof(Ent));
  const int row_bytes = 32 * static_cast<int>(sizeof(Tin)) + r * static_cast<int>(sizeof(Ent));
  const int bm = std::max(32, (budget / row_bytes) / 32 * 32);
  S1Args A{};
  A.count = static_cast<int>(jobs.size());
  A.d = d;
  A.r = r;
  A.bm = bm;
  A.tile_bytes = static_cast<int>(round_up(static_cast<long long>(bm) * 32 * sizeof(Tin), 16));
  // a chunk holds bm*r entries plus at most one even-padding entry per bin
  A.ent_bytes = static_cast<int>(round_up(static_cast<long long>(bm * r + d) * sizeof(Ent), 16) + 16);
  int bands = 0;
  for (size_t i = 0; i < jobs.size(); ++i) {
    const S1Job& J = jobs[i];
    require(J.pr->p->r == r, "compress group: projectors must share r");
    const ChunkTable& ct = J.pr->p->chunk_table(bm, static_cast<int>(sizeof(Tin)));
    S1Mat& M = A.mat[i];
    M.g = J.g, M.ldg = J.ldg, M.m = J.pr->m, M.n = J.pr->n;
    M.split = ct.split.as<int>(), M.ent = ct.ent.p, M.nchunks = ct.nchunks;
    M.zt = J.zt, M.ldz = J.pr->ldz();
    bands += ceil_div(M.n, 32);
    M.band_end = bands;
    M.vec = (reinterpret_cast<uintptr_t>(J.g) % 16 == 0) &&
            ((J.ldg * static_cast<long long>(sizeof(Tin))) % 16 == 0);
  }
  if (bands == 0) return;
  dim3 grid(bands, ceil_div(d, WARPS * 32));
  const int smem = 2 * (A.tile_bytes + A.ent_bytes);
  auto kern = k_compress_stage1<Tin, Tacc, WARPS>;
  LSP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<grid, WARPS * 32, smem, st>>>(A);
  after_launch("compress_stage1");
}

}  // namespace

// Z^T_i = G_i^T P_i for every job of a group (same d, r, compute and G dtype).
void launch_compress_stage1_group(const std::vector<S1Job>& jobs, lsp_dtype gdt,
                                  cudaStream_t st) {
  if (jobs.empty()) return;
  require(jobs.size() <= static_cast<size_t>(kMaxGroup), "group too large");
  if (launch_compress_spmm_group(jobs, gdt, st)) return;
  if (launch_compress_slots_group(jobs, gdt, st)) return;
  const Pair& p0 = *jobs[0].pr;
  LSP_DISPATCH_ACC(p0.compute, Tacc, {
    LSP_DISPATCH_STORAGE(gdt, Tin, {
      const int need = ceil_div(p0.d, 32);  // warps needed to cover every bin once
      constexpr int kMaxWarps = sizeof(Tacc) == 8 ? 16 : 32;
      if constexpr (kMaxWarps == 32) {
        if (need > 16) {
          stage1_impl<Tin, Tacc, 32>(jobs, p0.d, st);
          break;
        }
      }
      if (need > 8)
        stage1_impl<Tin, Tacc, 16>(jobs, p0.d, st);
      else if (need > 4)
        stage1_impl<Tin, Tacc, 8>(jobs, p0.d, st);
      else
        stage1_impl<Tin, Tacc, 4>(jobs, p0.d, st);
    })
  })
}

void launch_compress_stage1(const Pair& pr, const void* g, long long ldg, lsp_dtype gdt,
                            void* zt, cudaStream_t st) {
  std::vector<S1Job> jobs{S1Job{&pr, g, ldg, zt}};
  launch_compress_stage1_group(jobs, gdt, st);
}

// ---------------------------------------------------------------------------
// Row gather: out[r][:] = beta*in[r][:] + alpha * sum_t val[t] * src[idx[t]][:]
// One warp per output row; lanes stride the columns 32 at a time, 8 columns in
// flight per lane.  Optional deterministic per-block sum of squares of the
// result (for Frobenius norms).
// ---------------------------------------------------------------------------
namespace {

constexpr int kGatherWarps = 8;
constexpr int kGatherUnroll = 8;

template <typename Tsrc, typename Tdst, typename Tacc>
__global__ void __launch_bounds__(kGatherWarps * 32)
    k_gather(int R, int c, const int* __restrict__ ptr, int k, const int* __restrict__ idx,
             const Tacc* __restrict__ val, const Tsrc* __restrict__ src, long long lds,
             const Tdst* in, long long ldi, Tdst* out, long long ldo, Tacc alpha, Tacc beta,
             double* __restrict__ partials) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double ss = 0.0;
  for (int r = blockIdx.x * kGatherWarps + warp; r < R; r += gridDim.x * kGatherWarps) {
    const int e0 = ptr ? ptr[r] : r * k;
    const int e1 = ptr ? ptr[r + 1] : e0 + k;
    for (int c0 = 0; c0 < c; c0 += 32 * kGatherUnroll) {
      Tacc acc[kGatherUnroll];
#pragma unroll
      for (int u = 0; u < kGatherUnroll; ++u) acc[u] = Tacc(0);
      for (int e = e0; e < e1; ++e) {
        const Tacc v = val[e];
        const Tsrc* s = src + static_cast<long long>(idx[e]) * lds;
#pragma unroll
        for (int u = 0; u < kGatherUnroll; ++u) {
          const int col = c0 + u * 32 + lane;
          if (col < c) acc[u] = fma(v, cvt<Tacc>(s[col]), acc[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < kGatherUnroll; ++u) {
        const int col = c0 + u * 32 + lane;
        if (col >= c) continue;
        Tacc res = alpha * acc[u];
        if (in && beta != Tacc(0))
          res = fma(beta, cvt<Tacc>(in[static_cast<long long>(r) * ldi + col]), res);
        if (out) out[static_cast<long long>(r) * ldo + col] = cvt<Tdst>(res);
        if (partials) ss += static_cast<double>(res) * static_cast<double>(res);
      }
    }
  }
  if (partials) {
    __shared__ double red[kGatherWarps];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kGatherWarps; ++w) t += red[w];
      partials[blockIdx.x] = t;
    }
  }
}

// fp64 fast form (no partials; c, lds, ldo, ldi even; 16-byte aligned rows):
// one warp per (column pass of 128 doubles, output row), passes outermost so
// the warps in flight cover every row for a few column passes (the source
// rows of those columns come from HBM once, then L2).  Lane = 2 adjacent
// columns per 64-column chunk (16-byte loads, 512 bytes per warp
// instruction); entries in groups of 4 with all 8 loads of a group in flight,
// 64 registers so four 8-warp blocks share an SM (C3-shape fit: 4 chunks at
// ~100 registers 4.76 s, 2 chunks 4.27 s, 1 chunk at 6 blocks 5.84 s).
// Per column the FMA chain runs over the entries in order, exactly as
// k_gather, so results are bitwise equal.
constexpr int kGvChunks = 2;
// nb > 1: a batch of independent gathers through the same projector, operand
// b at src + b*sbs, in + b*ibs, out + b*obs (one launch for every target of a fit).
__global__ void __launch_bounds__(kGatherWarps * 32, 4)
    k_gather_f64v(int R, int c, int npass, const int* __restrict__ ptr, int k,
                  const int* __restrict__ idx, const double* __restrict__ val,
                  const double* __restrict__ src_base, long long lds, const double* in_base, long long ldi,
                  double* out_base, long long ldo, double alpha, double beta, int nb, long long sbs,
                  long long ibs, long long obs) {
  const int lane = threadIdx.x & 31;
  const long long per = static_cast<long long>(R) * npass;
  const long long tasks = per * nb;
  for (long long t = static_cast<long long>(blockIdx.x) * kGatherWarps + (threadIdx.x >> 5); t < tasks;
       t += static_cast<long long>(gridDim.x) * kGatherWarps) {
    const int bi = static_cast<int>(t / per);
    const long long tb = t - bi * per;
    const double* __restrict__ src = src_base + bi * sbs;
    const double* in = in_base ? in_base + bi * ibs : nullptr;
    double* out = out_base + bi * obs;
    const int pass = static_cast<int>(tb / R), r = static_cast<int>(tb - static_cast<long long>(pass) * R);
    const int e0 = ptr ? __ldg(ptr + r) : r * k;
    const int e1 = ptr ? __ldg(ptr + r + 1) : e0 + k;
    const int c0 = pass * (64 * kGvChunks) + 2 * lane;
    bool ok[kGvChunks];
#pragma unroll
    for (int q = 0; q < kGvChunks; ++q) ok[q] = c0 + 64 * q < c;
    double2 acc[kGvChunks];
#pragma unroll
    for (int q = 0; q < kGvChunks; ++q) acc[q] = make_double2(0.0, 0.0);
    for (int e = e0; e < e1; e += 4) {
      double v[4];
      double2 s[4][kGvChunks];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool eu = e + u < e1;
        v[u] = eu ? __ldg(val + e + u) : 0.0;
        const double* row = src + static_cast<long long>(eu ? __ldg(idx + e + u) : 0) * lds + c0;
#pragma unroll
        for (int q = 0; q < kGvChunks; ++q)
          s[u][q] = (eu && ok[q]) ? __ldg(reinterpret_cast<const double2*>(row + 64 * q))
                                  : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (e + u < e1) {
#pragma unroll
          for (int q = 0; q < kGvChunks; ++q) {
            acc[q].x = fma(v[u], s[u][q].x, acc[q].x);
            acc[q].y = fma(v[u], s[u][q].y, acc[q].y);
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kGvChunks; ++q) {
      if (!ok[q]) continue;
      const int col = c0 + 64 * q;
      double2 res = make_double2(alpha * acc[q].x, alpha * acc[q].y);
      if (in && beta != 0.0) {
        const double2 x = *reinterpret_cast<const double2*>(in + static_cast<long long>(r) * ldi + col);
        res.x = fma(beta, x.x, res.x);
        res.y = fma(beta, x.y, res.y);
      }
      *reinterpret_cast<double2*>(out + static_cast<long long>(r) * ldo + col) = res;
    }
  }
}

}  // namespace

void launch_gather_f64_batch(int R, int c, const int* ptr, int k, const int* idx, const double* val,
                             const double* src, long long lds, long long sbs, const double* in,
                             long long ldi, long long ibs, double* out, long long ldo, long long obs,
                             int nb, double alpha, double beta, cudaStream_t st) {
  if (R <= 0 || c <= 0 || nb <= 0) return;
  require(c % 2 == 0 && lds % 2 == 0 && ldo % 2 == 0 && sbs % 2 == 0 && obs % 2 == 0 &&
              (!in || (ldi % 2 == 0 && ibs % 2 == 0)) &&
              reinterpret_cast<uintptr_t>(src) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0 &&
              (!in || reinterpret_cast<uintptr_t>(in) % 16 == 0),
          "gather_f64: 16-byte aligned rows of an even width required");
  const int npass = ceil_div(c, 64 * kGvChunks);
  const long long tasks = static_cast<long long>(R) * npass * nb;
  const int grid = static_cast<int>(std::min<long long>(ceil_div(tasks, kGatherWarps), 16LL * num_sms()));
  k_gather_f64v<<<grid, kGatherWarps * 32, 0, st>>>(R, c, npass, ptr, k, idx, val, src, lds, in, ldi, out,
                                                     ldo, alpha, beta, nb, sbs, ibs, obs);
  after_launch("gather_f64v");
}

void launch_gather(int R, int c, const int* ptr, int k, const int* idx, const void* val,
                   lsp_dtype acc, const void* src, long long lds, lsp_dtype src_dt,
                   const void* in, long long ldi, void* out, long long ldo, lsp_dtype out_dt,
                   double alpha, double beta, DevBuf* partials, int* nparts, cudaStream_t st) {
  if (R <= 0 || c <= 0) {
    if (nparts) *nparts = 0;
    return;
  }
  auto al16 = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
  if (acc == LSP_F64 && src_dt == LSP_F64 && out_dt == LSP_F64 && !partials && out &&
      c % 2 == 0 && lds % 2 == 0 && ldo % 2 == 0 && al16(src) && al16(out) &&
      (!in || beta == 0.0 || (ldi % 2 == 0 && al16(in)))) {
    if (nparts) *nparts = 0;
    launch_gather_f64_batch(R, c, ptr, k, idx, static_cast<const double*>(val),
                            static_cast<const double*>(src), lds, 0, (in && beta != 0.0) ? static_cast<const double*>(in) : nullptr,
                            ldi, 0, static_cast<double*>(out), ldo, 0, 1, alpha, beta, st);
    return;
  }
  const int grid = std::min(ceil_div(R, kGatherWarps), 8 * num_sms());
  if (nparts) *nparts = grid;
  if (partials) partials->ensure(static_cast<size_t>(grid) * sizeof(double));
  double* parts = partials ? partials->as<double>() : nullptr;
  LSP_DISPATCH_ACC(acc, Tacc, {
    LSP_DISPATCH_STORAGE(src_dt, Tsrc, {
      LSP_DISPATCH_STORAGE(out_dt, Tdst, {
        k_gather<Tsrc, Tdst, Tacc><<<grid, kGatherWarps * 32, 0, st>>>(
            R, c, ptr, k, idx, static_cast<const Tacc*>(val), static_cast<const Tsrc*>(src), lds,
            static_cast<const Tdst*>(in), ldi, static_cast<Tdst*>(out), ldo,
            static_cast<Tacc>(alpha), static_cast<Tacc>(beta), parts);
      })
    })
  })
  after_launch("gather");
}

// ---------------------------------------------------------------------------
// Tiled transpose dst[c][r] = src[r][c] (32x32 tiles through padded smem).
// ---------------------------------------------------------------------------
namespace {
template <typename T>
__global__ void k_transpose(int rows, int cols, const T* __restrict__ src, long long lds,
                            T* __restrict__ dst, long long ldd, long long sbs, long long dbs) {
  __shared__ T tile[32][33];
  src += blockIdx.z * sbs;  // batch (gridDim.z operands at fixed strides)
  dst += blockIdx.z * dbs;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int r = by + y, c = bx + threadIdx.x;
    if (r < rows && c < cols) tile[y][threadIdx.x] = src[static_cast<long long>(r) * lds + c];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int c = bx + y, r = by + threadIdx.x;
    if (r < rows && c < cols) dst[static_cast<long long>(c) * ldd + r] = tile[threadIdx.x][y];
  }
}
}  // namespace

void launch_transpose(int rows, int cols, const void* src, long long lds, void* dst,
                      long long ldd, lsp_dtype dt, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  dim3 grid(ceil_div(cols, 32), ceil_div(rows, 32)), block(32, 8);
  LSP_DISPATCH_STORAGE(dt, T, {
    k_transpose<T><<<grid, block, 0, st>>>(rows, cols, static_cast<const T*>(src), lds,
                                           static_cast<T*>(dst), ldd, 0, 0);
  })
  after_launch("transpose");
}

void launch_transpose_batch(int rows, int cols, const double* src, long long lds, long long sbs,
                            double* dst, long long ldd, long long dbs, int nb, cudaStream_t st) {
  if (rows <= 0 || cols <= 0 || nb <= 0) return;
  dim3 grid(ceil_div(cols, 32), ceil_div(rows, 32), nb), block(32, 8);
  k_transpose<double><<<grid, block, 0, st>>>(rows, cols, src, lds, dst, ldd, sbs, dbs);
  after_launch("transpose");
}

// ---------------------------------------------------------------------------
// Stage 2 (grouped, fp32): S^T_i[b][:] = sum_{t in CSC(Q_i)[b]} q_t Z^T_i[j_t][:].
// One CTA per (subspace row b, matrix); a thread owns 4 consecutive columns;
// four entries' rows are in flight per thread (L2-bound gathers of 4 KB rows).
// Non-finite results latch `flag` (reference NumericError, subspace_opt.cpp:38).
// ---------------------------------------------------------------------------
namespace {

struct S2Mat {
  const int* ptr;
  const int* row;
  const float* val;
  const float* zt;
  int ldz;
  float* s_t;
};
struct S2Args {
  S2Mat mat[kMaxGroup];
  int count;
  int d;
  int* flag;
};

constexpr int kS2Threads = 128;
constexpr int kS2V = 2;  // float4 column chunks per thread (d = 1024: the whole row)

// One CTA = one row b of S^T for one matrix: S^T[b][:] = sum over the CSC
// entries e of Q's column b (ascending row order) of q_e * Z^T[row_e][:].
// Each thread owns kS2V float4 chunks of the row, so every entry's index and
// value loads serve 8 columns and 2*4 Z^T loads are in flight per batch.
//
// k_stage2_adam_f4: the layer's subspace Adam fused into the epilogue (a single-rank step
// has no S exchange between stage 2 and Adam).  Each thread runs adam_elem on
// the S^T elements it just produced, reading the current moment pair and
// writing the other one (ping-pong, Adam::cur); the last CTA to finish flips
// the pair and advances the step counter only if no CTA of the launch latched
// a non-finite S -- the same skip semantics as k_adam's early return.  Every
// value is computed by the same operations as stage 2 followed by k_adam, so
// the results are bitwise those of the unfused pair.
// Measured (C4 fp32, ncu launch times per layer): 81.7 us vs 51.8 (stage 2)
// + 34.8 (k_adam); the moments are prefetched by cp.async at CTA start (a
// plain epilogue load made the fused kernel slower than the pair), and more
// S^T rows per CTA (fewer done-counter atomics) measured slower (2: +0.3 ms,
// 4: +1.0 ms per C4 step).
constexpr int kS2AdamMinBlocks = 8;  // 128-thread CTAs per SM the fused kernel is register-bounded for
struct S2Adam {
  long long off[kMaxGroup];  // element offset of A.mat[i]'s block in the layer state
  float *m0, *v0, *m1, *v1, *delta;
  int* cur;
  const double2* table;
  long long cap;
  double db1, db2;
  float b1, omb1, b2, omb2, eps;
  long long* step;
  unsigned* done;
};

__global__ void __launch_bounds__(kS2Threads) k_stage2_f4(const __grid_constant__ S2Args A) {
  const S2Mat& M = A.mat[blockIdx.y];
  const int b = blockIdx.x, d = A.d;
  const int e0 = __ldg(M.ptr + b), e1 = __ldg(M.ptr + b + 1);
  bool bad = false;
  for (int a_base = 4 * threadIdx.x; a_base < d; a_base += 4 * kS2Threads * kS2V) {
    float4 acc[kS2V];
    bool ok[kS2V];
#pragma unroll
    for (int c = 0; c < kS2V; ++c) {
      acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      ok[c] = a_base + c * 4 * kS2Threads < d;
    }
    int e = e0;
    for (; e + 4 <= e1; e += 4) {
      float4 z[4][kS2V];
      float q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        q[u] = __ldg(M.val + e + u);
        const float* zr = M.zt + static_cast<long long>(__ldg(M.row + e + u)) * M.ldz + a_base;
#pragma unroll
        for (int c = 0; c < kS2V; ++c)
          z[u][c] = ok[c] ? __ldg(reinterpret_cast<const float4*>(zr + c * 4 * kS2Threads))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < kS2V; ++c) {
          acc[c].x = fmaf(q[u], z[u][c].x, acc[c].x);
          acc[c].y = fmaf(q[u], z[u][c].y, acc[c].y);
          acc[c].z = fmaf(q[u], z[u][c].z, acc[c].z);
          acc[c].w = fmaf(q[u], z[u][c].w, acc[c].w);
        }
    }
    for (; e < e1; ++e) {
      const float q = __ldg(M.val + e);
      const float* zr = M.zt + static_cast<long long>(__ldg(M.row + e)) * M.ldz + a_base;
#pragma unroll
      for (int c = 0; c < kS2V; ++c) {
        if (!ok[c]) continue;
        const float4 z = __ldg(reinterpret_cast<const float4*>(zr + c * 4 * kS2Threads));
        acc[c].x = fmaf(q, z.x, acc[c].x);
        acc[c].y = fmaf(q, z.y, acc[c].y);
        acc[c].z = fmaf(q, z.z, acc[c].z);
        acc[c].w = fmaf(q, z.w, acc[c].w);
      }
    }
#pragma unroll
    for (int c = 0; c < kS2V; ++c) {
      if (!ok[c]) continue;
      bad |= !(isfinite(acc[c].x) && isfinite(acc[c].y) && isfinite(acc[c].z) && isfinite(acc[c].w));
      *reinterpret_cast<float4*>(M.s_t + static_cast<long long>(b) * d + a_base + c * 4 * kS2Threads) = acc[c];
    }
  }
  if (A.flag && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(A.flag, 1);
}

template <int NT>
__global__ void __launch_bounds__(NT, kS2AdamMinBlocks * 128 / NT)
    k_stage2_adam_f4(const __grid_constant__ S2Args A, const __grid_constant__ S2Adam K) {
  const S2Mat& M = A.mat[blockIdx.y];
  const int b = blockIdx.x, d = A.d;
  const int e0 = __ldg(M.ptr + b), e1 = __ldg(M.ptr + b + 1);
  bool bad = false;
  // the CTA's current moments, staged by cp.async while the gathers run
  __shared__ __align__(16) float4 mv_s[2 * kS2V * NT];
  // read before this CTA counts itself done: the last CTA's flip comes after
  const long long t = *K.step + 1;
  const int which = *K.cur;
  double2 c;
  if (t <= K.cap) {
    c = K.table[t - 1];
  } else {
    c.x = 1.0 - pow(K.db1, static_cast<double>(t));
    c.y = 1.0 - pow(K.db2, static_cast<double>(t));
  }
  const float c1 = static_cast<float>(c.x), c2 = static_cast<float>(c.y);
  for (int a_base = 4 * threadIdx.x; a_base < d; a_base += 4 * NT * kS2V) {
    {
      const long long i0 = K.off[blockIdx.y] + static_cast<long long>(b) * d + a_base;
      const float* mi = which ? K.m1 : K.m0;
      const float* vi = which ? K.v1 : K.v0;
#pragma unroll
      for (int c = 0; c < kS2V; ++c) {
        const bool in = a_base + c * 4 * NT < d;
        const long long i = i0 + c * 4 * NT;
        cp_async16(&mv_s[(2 * c) * NT + threadIdx.x], in ? mi + i : mi, in ? 16 : 0);
        cp_async16(&mv_s[(2 * c + 1) * NT + threadIdx.x], in ? vi + i : vi, in ? 16 : 0);
      }
      asm volatile("cp.async.commit_group;\n" ::);
    }
    float4 acc[kS2V];
    bool ok[kS2V];
#pragma unroll
    for (int c = 0; c < kS2V; ++c) {
      acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      ok[c] = a_base + c * 4 * NT < d;
    }
    int e = e0;
    for (; e + 4 <= e1; e += 4) {
      float4 z[4][kS2V];
      float q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        q[u] = __ldg(M.val + e + u);
        const float* zr = M.zt + static_cast<long long>(__ldg(M.row + e + u)) * M.ldz + a_base;
#pragma unroll
        for (int c = 0; c < kS2V; ++c)
          z[u][c] = ok[c] ? __ldg(reinterpret_cast<const float4*>(zr + c * 4 * NT))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < kS2V; ++c) {
          acc[c].x = fmaf(q[u], z[u][c].x, acc[c].x);
          acc[c].y = fmaf(q[u], z[u][c].y, acc[c].y);
          acc[c].z = fmaf(q[u], z[u][c].z, acc[c].z);
          acc[c].w = fmaf(q[u], z[u][c].w, acc[c].w);
        }
    }
    for (; e < e1; ++e) {
      const float q = __ldg(M.val + e);
      const float* zr = M.zt + static_cast<long long>(__ldg(M.row + e)) * M.ldz + a_base;
#pragma unroll
      for (int c = 0; c < kS2V; ++c) {
        if (!ok[c]) continue;
        const float4 z = __ldg(reinterpret_cast<const float4*>(zr + c * 4 * NT));
        acc[c].x = fmaf(q, z.x, acc[c].x);
        acc[c].y = fmaf(q, z.y, acc[c].y);
        acc[c].z = fmaf(q, z.z, acc[c].z);
        acc[c].w = fmaf(q, z.w, acc[c].w);
      }
    }
#pragma unroll
    for (int c = 0; c < kS2V; ++c) {
      if (!ok[c]) continue;
      bad |= !(isfinite(acc[c].x) && isfinite(acc[c].y) && isfinite(acc[c].z) && isfinite(acc[c].w));
      const long long el = static_cast<long long>(b) * d + a_base + c * 4 * NT;
      *reinterpret_cast<float4*>(M.s_t + el) = acc[c];
      {
        const long long i = K.off[blockIdx.y] + el;
        asm volatile("cp.async.wait_all;\n" ::: "memory");  // own copies only
        float4 mv = mv_s[(2 * c) * NT + threadIdx.x];
        float4 vv = mv_s[(2 * c + 1) * NT + threadIdx.x];
        float4 dv;
        dv.x = adam_elem(acc[c].x, mv.x, vv.x, K.b1, K.omb1, K.b2, K.omb2, c1, c2, K.eps);
        dv.y = adam_elem(acc[c].y, mv.y, vv.y, K.b1, K.omb1, K.b2, K.omb2, c1, c2, K.eps);
        dv.z = adam_elem(acc[c].z, mv.z, vv.z, K.b1, K.omb1, K.b2, K.omb2, c1, c2, K.eps);
        dv.w = adam_elem(acc[c].w, mv.w, vv.w, K.b1, K.omb1, K.b2, K.omb2, c1, c2, K.eps);
        *reinterpret_cast<float4*>((which ? K.m0 : K.m1) + i) = mv;
        *reinterpret_cast<float4*>((which ? K.v0 : K.v1) + i) = vv;
        *reinterpret_cast<float4*>(K.delta + i) = dv;
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(A.flag, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();  // this CTA's latch and moments before its done count
    if (atomicAdd(K.done, 1u) == gridDim.x * gridDim.y - 1) {
      if (atomicOr(A.flag, 0) == 0) {  // every CTA latched before counting itself
        *K.cur = 1 - which;
        *K.step = t;
      }
      *K.done = 0u;
      __threadfence();
    }
  }
}

// fp64 twin of k_stage2_f4 (the reference's precision): 16-byte double2 chunks,
// kS2V2 per thread (d = 1024: the whole row), the same per-element fma chain in
// CSC entry order, the non-finite latch fused.
struct S2MatD {
  const int* ptr;
  const int* row;
  const double* val;
  const double* zt;
  int ldz;
  double* s_t;
};
struct S2ArgsD {
  S2MatD mat[kMaxGroup];
  int count;
  int d;
  int* flag;
};
constexpr int kS2V2 = 4;
__global__ void __launch_bounds__(kS2Threads) k_stage2_d2(const __grid_constant__ S2ArgsD A) {
  const S2MatD& M = A.mat[blockIdx.y];
  const int b = blockIdx.x, d = A.d;
  const int e0 = __ldg(M.ptr + b), e1 = __ldg(M.ptr + b + 1);
  bool bad = false;
  for (int a_base = 2 * threadIdx.x; a_base < d; a_base += 2 * kS2Threads * kS2V2) {
    double2 acc[kS2V2];
    bool ok[kS2V2];
#pragma unroll
    for (int c = 0; c < kS2V2; ++c) {
      acc[c] = make_double2(0.0, 0.0);
      ok[c] = a_base + c * 2 * kS2Threads < d;
    }
    int e = e0;
    for (; e + 2 <= e1; e += 2) {
      double2 z[2][kS2V2];
      double q[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        q[u] = __ldg(M.val + e + u);
        const double* zr = M.zt + static_cast<long long>(__ldg(M.row + e + u)) * M.ldz + a_base;
#pragma unroll
        for (int c = 0; c < kS2V2; ++c)
          z[u][c] = ok[c] ? __ldg(reinterpret_cast<const double2*>(zr + c * 2 * kS2Threads))
                          : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int c = 0; c < kS2V2; ++c) {
          acc[c].x = fma(q[u], z[u][c].x, acc[c].x);
          acc[c].y = fma(q[u], z[u][c].y, acc[c].y);
        }
    }
    for (; e < e1; ++e) {
      const double q = __ldg(M.val + e);
      const double* zr = M.zt + static_cast<long long>(__ldg(M.row + e)) * M.ldz + a_base;
#pragma unroll
      for (int c = 0; c < kS2V2; ++c) {
        if (!ok[c]) continue;
        const double2 z = __ldg(reinterpret_cast<const double2*>(zr + c * 2 * kS2Threads));
        acc[c].x = fma(q, z.x, acc[c].x);
        acc[c].y = fma(q, z.y, acc[c].y);
      }
    }
#pragma unroll
    for (int c = 0; c < kS2V2; ++c) {
      if (!ok[c]) continue;
      bad |= !(isfinite(acc[c].x) && isfinite(acc[c].y));
      *reinterpret_cast<double2*>(M.s_t + static_cast<long long>(b) * d + a_base + c * 2 * kS2Threads) = acc[c];
    }
  }
  if (A.flag && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(A.flag, 1);
}

}  // namespace

void launch_stage2_group(const std::vector<S1Job>& jobs, int* flag, cudaStream_t st) {
  if (jobs.empty()) return;
  const Pair& p0 = *jobs[0].pr;
  const int d = p0.d;
  bool fast = p0.compute == LSP_F32 && d % 4 == 0;
  for (const S1Job& J : jobs)
    fast = fast && J.pr->ldz() % 4 == 0 && reinterpret_cast<uintptr_t>(J.zt) % 16 == 0 &&
           reinterpret_cast<uintptr_t>(J.s_t) % 16 == 0;
  if (fast) {
    S2Args A{};
    A.count = static_cast<int>(jobs.size());
    A.d = d;
    A.flag = flag;
    // matrices in reverse order: stage 1 wrote the last matrices' Z^T most
    // recently, so those reads are the likeliest L2 hits (LSP_STAGE2_REVERSE=0: forward)
    const char* rev_env = std::getenv("LSP_STAGE2_REVERSE");
    const bool rev = !(rev_env && rev_env[0] == '0');
    for (size_t i = 0; i < jobs.size(); ++i) {
      const size_t ji = rev ? jobs.size() - 1 - i : i;
      const Projector& Q = *jobs[ji].pr->q;
      A.mat[i] = S2Mat{Q.csc_ptr.as<int>(), Q.csc_row.as<int>(), Q.csc_val.as<float>(),
                       static_cast<const float*>(jobs[ji].zt), jobs[ji].pr->ldz(),
                       static_cast<float*>(jobs[ji].s_t)};
    }
    k_stage2_f4<<<dim3(d, A.count), kS2Threads, 0, st>>>(A);
    after_launch("stage2");
    return;
  }
  bool fast64 = p0.compute == LSP_F64 && d % 2 == 0;
  for (const S1Job& J : jobs)
    fast64 = fast64 && J.pr->ldz() % 2 == 0 && reinterpret_cast<uintptr_t>(J.zt) % 16 == 0 &&
             reinterpret_cast<uintptr_t>(J.s_t) % 16 == 0;
  if (fast64) {
    S2ArgsD A{};
    A.count = static_cast<int>(jobs.size());
    A.d = d;
    A.flag = flag;
    for (size_t i = 0; i < jobs.size(); ++i) {  // reverse: the last-written Z^T first
      const size_t ji = jobs.size() - 1 - i;
      const Projector& Q = *jobs[ji].pr->q;
      A.mat[i] = S2MatD{Q.csc_ptr.as<int>(), Q.csc_row.as<int>(), Q.csc_val.as<double>(),
                        static_cast<const double*>(jobs[ji].zt), jobs[ji].pr->ldz(),
                        static_cast<double*>(jobs[ji].s_t)};
    }
    k_stage2_d2<<<dim3(d, A.count), kS2Threads, 0, st>>>(A);
    after_launch("stage2_d2");
    return;
  }
  for (const S1Job& J : jobs) {
    const Projector& Q = *J.pr->q;
    launch_gather(d, d, Q.csc_ptr.as<int>(), 0, Q.csc_row.as<int>(), Q.csc_val.p, p0.compute,
                  J.zt, J.pr->ldz(), p0.compute, nullptr, 0, J.s_t, d, p0.compute, 1.0, 0.0,
                  nullptr, nullptr, st);
    if (flag) launch_check_finite(static_cast<size_t>(d) * d, J.s_t, p0.compute, flag, st);
  }
}

bool launch_stage2_adam_group(const std::vector<S1Job>& jobs, const void* s_base, Adam& a,
                              void* delta, int* flag, cudaStream_t st) {
  if (jobs.empty() || !flag || !a.cur.p || a.compute != LSP_F32) return false;
  if (const char* e = std::getenv("LSP_FUSE_ADAM"))
    if (e[0] == '0') return false;
  const Pair& p0 = *jobs[0].pr;
  const int d = p0.d;
  bool ok = p0.compute == LSP_F32 && d % 4 == 0 && a.cols == d &&
            (reinterpret_cast<uintptr_t>(delta) | reinterpret_cast<uintptr_t>(a.m.p) |
             reinterpret_cast<uintptr_t>(a.v.p) | reinterpret_cast<uintptr_t>(a.m2.p) |
             reinterpret_cast<uintptr_t>(a.v2.p)) % 16 == 0;
  for (const S1Job& J : jobs)
    ok = ok && J.pr->ldz() % 4 == 0 && reinterpret_cast<uintptr_t>(J.zt) % 16 == 0 &&
         reinterpret_cast<uintptr_t>(J.s_t) % 16 == 0;
  if (!ok) return false;
  S2Args A{};
  A.count = static_cast<int>(jobs.size());
  A.d = d;
  A.flag = flag;
  S2Adam K{};
  const char* rev_env = std::getenv("LSP_STAGE2_REVERSE");
  const bool rev = !(rev_env && rev_env[0] == '0');
  for (size_t i = 0; i < jobs.size(); ++i) {
    const size_t ji = rev ? jobs.size() - 1 - i : i;
    const Projector& Q = *jobs[ji].pr->q;
    A.mat[i] = S2Mat{Q.csc_ptr.as<int>(), Q.csc_row.as<int>(), Q.csc_val.as<float>(),
                     static_cast<const float*>(jobs[ji].zt), jobs[ji].pr->ldz(),
                     static_cast<float*>(jobs[ji].s_t)};
    const long long off = (static_cast<const char*>(jobs[ji].s_t) - static_cast<const char*>(s_base)) /
                          static_cast<long long>(sizeof(float));
    if (off < 0 || off + static_cast<long long>(d) * d > static_cast<long long>(a.count())) return false;
    K.off[i] = off;
  }
  K.m0 = a.m.as<float>();
  K.v0 = a.v.as<float>();
  K.m1 = a.m2.as<float>();
  K.v1 = a.v2.as<float>();
  K.delta = static_cast<float*>(delta);
  K.cur = a.cur.as<int>();
  K.table = correction_table(a.beta1, a.beta2, &K.cap);
  K.db1 = a.beta1;
  K.db2 = a.beta2;
  K.b1 = static_cast<float>(a.beta1);
  K.omb1 = static_cast<float>(1.0 - a.beta1);
  K.b2 = static_cast<float>(a.beta2);
  K.omb2 = static_cast<float>(1.0 - a.beta2);
  K.eps = static_cast<float>(a.eps);
  K.step = a.dstep.as<long long>();
  K.done = a.done.as<unsigned>();
  // threads per S^T row: 8 columns each, whole warps, at most kS2Threads (narrow
  // d: no idle warps, more CTAs per SM; C2 d = 512: 64 threads)
  const int nt = std::min(kS2Threads, std::max(32, static_cast<int>(round_up(ceil_div(d, 8), 32))));
  if (nt == 32)
    k_stage2_adam_f4<32><<<dim3(d, A.count), 32, 0, st>>>(A, K);
  else if (nt == 64)
    k_stage2_adam_f4<64><<<dim3(d, A.count), 64, 0, st>>>(A, K);
  else if (nt == 96)
    k_stage2_adam_f4<96><<<dim3(d, A.count), 96, 0, st>>>(A, K);
  else
    k_stage2_adam_f4<kS2Threads><<<dim3(d, A.count), kS2Threads, 0, st>>>(A, K);
  after_launch("stage2_adam");
  return true;
}

// S^T = Q^T (G^T P) for every job: grouped stage 1 into each job's zt, grouped stage 2.
void compress_group_T(const std::vector<S1Job>& jobs, lsp_dtype gdt, int* flag,
                      cudaStream_t st) {
  launch_compress_stage1_group(jobs, gdt, st);
  launch_stage2_group(jobs, flag, st);
}

// S^T = Q^T (G^T P) for one pair: stage 1 into pr.zt, stage 2 into s_t (d x d, ld d).
void compress_T(Pair& pr, const void* g, long long ldg, lsp_dtype gdt, void* s_t,
                cudaStream_t st, int* flag) {
  const size_t vs = dtype_size(pr.compute);
  pr.zt.ensure(static_cast<size_t>(pr.n) * pr.ldz() * vs);
  std::vector<S1Job> jobs{S1Job{&pr, g, ldg, pr.zt.p, s_t}};
  compress_group_T(jobs, gdt, flag, st);
}

}  // namespace lspb
