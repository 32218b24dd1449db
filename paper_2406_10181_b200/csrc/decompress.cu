// Fused decompress-and-apply: out = beta*in + alpha * P delta Q^T
// (reference: left_mul/rightT_mul proj/src/projector.cpp:105-117,148-161,
//  decompress :170-175, apply proj/src/trainer.cpp:190).
//
// Persistent, HBM-streaming design (one CTA per SM, ~190 KB of shared memory):
//   * W is cut into column bands of BN columns; the work list is the
//     band-major sequence of (band, 64-row block) tiles, split evenly over the
//     CTAs (stream-K style), so every SM gets the same number of bytes.
//   * Y_band[a][jj] = sum_l q(j,l) * delta^T[pos_q(j,l)][a] (all a, the BN
//     columns of the band) lives in shared memory (d x (BN+1), padded); it is
//     rebuilt from the L2-resident delta^T only when a CTA enters a new band.
//   * W tiles (64 rows x BN) and the matching CSR entries of P stream through
//     a 6-stage cp.async ring, so ~40 KB of W is always in flight per SM
//     independent of registers, and the first stages are in flight while
//     Y_band is being built.
//   * Each W row: k conflict-free gathers Y_band[pos_p(i,l)][:], one
//     read-modify-write of W[i][band].  W is read and written exactly once.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "core.cuh"

namespace lspb {

namespace {

constexpr int kDecThreads = 512;
constexpr int kDecWarps = kDecThreads / 32;
constexpr int kRows = 64;     // W rows per ring stage
constexpr int kStages = 6;    // ring depth

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__host__ __device__ constexpr int align16(int b) { return (b + 15) & ~15; }

template <typename Tw, typename Tacc, int BN>
struct Layout {
  int d, r;
  __host__ __device__ int y_bytes() const { return align16(d * (BN + 1) * (int)sizeof(Tacc)); }
  __host__ __device__ int w_bytes() const { return align16(kRows * BN * (int)sizeof(Tw)); }
  __host__ __device__ int pos_bytes() const { return align16(kRows * r * 4); }
  __host__ __device__ int val_bytes() const { return align16(kRows * r * (int)sizeof(Tacc)); }
  __host__ __device__ int stage_bytes() const { return w_bytes() + pos_bytes() + val_bytes(); }
  __host__ __device__ int total() const { return y_bytes() + kStages * stage_bytes(); }
};

struct DecMat {
  int m, n;
  const int* ppos;
  const void* pval;
  const int* qpos;
  const void* qval;
  const void* dT;      // d x d, ld d
  const void* in;
  long long ldi;
  void* out;
  long long ldo;
  int row_blocks;      // ceil(m / kRows)
  int nbands;          // ceil(n / BN)
  long long tile_end;  // exclusive prefix of (band, row block) tiles over the group
  int vec;             // 16-byte cp.async legal for this matrix's W / P arrays
};
struct DecArgs {
  DecMat mat[kMaxGroup];
  int count;
  int d, r;
  long long total;     // all tiles of the group
  double alpha, beta;
  int use_in;          // beta != 0 and every matrix has an input
  const int* skip;
  double* partials;
};

// Position in the group's (matrix, band, row block) tile list, advanced one
// tile at a time (no divisions in the loop).
struct Cursor {
  int mi, band, rb;
};

__device__ __forceinline__ Cursor cursor_at(const DecArgs& A, long long t) {
  int i = 0;
  while (i + 1 < A.count && t >= A.mat[i].tile_end) ++i;
  const long long lt = t - (i ? A.mat[i - 1].tile_end : 0);
  return Cursor{i, static_cast<int>(lt / A.mat[i].row_blocks),
                static_cast<int>(lt % A.mat[i].row_blocks)};
}

__device__ __forceinline__ void advance(const DecArgs& A, Cursor& c) {
  if (++c.rb == A.mat[c.mi].row_blocks) {
    c.rb = 0;
    if (++c.band == A.mat[c.mi].nbands) {
      c.band = 0;
      ++c.mi;
    }
  }
}

// KR: nonzeros per projector row known at compile time (0 = runtime A.r).
template <typename Tw, typename Tacc, int BN, int KR, bool SUMSQ>
__global__ void __launch_bounds__(kDecThreads, 1) k_decompress_band(const __grid_constant__ DecArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (A.skip && *A.skip) return;
  const int r = KR > 0 ? KR : A.r;
  const Layout<Tw, Tacc, BN> L{A.d, r};
  constexpr int LDY = BN + 1;
  Tacc* Y = reinterpret_cast<Tacc*>(smem_raw);
  unsigned char* ring = smem_raw + L.y_bytes();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = A.d;
  const Tacc alpha = static_cast<Tacc>(A.alpha), beta = static_cast<Tacc>(A.beta);
  const bool use_in = A.use_in != 0;

  // this CTA's contiguous share of the (matrix, band, row block) tile list
  const long long t_begin = A.total * blockIdx.x / gridDim.x;
  const long long t_end = A.total * (blockIdx.x + 1) / gridDim.x;
  const int ntiles = static_cast<int>(t_end - t_begin);
  if (ntiles <= 0) return;

  // W piece this thread copies in every stage (fixed row / 16-byte column piece)
  constexpr int EPP = 16 / sizeof(Tw);
  constexpr int PPR = BN / EPP > 0 ? BN / EPP : 1;
  constexpr int kPieces = kRows * PPR;
  const int my_row = tid / PPR, my_pc = tid % PPR;

  // ---- producer -------------------------------------------------------------
  Cursor ic = cursor_at(A, t_begin);
  auto issue = [&](int s) {
    if (s < ntiles) {
      const DecMat& M = A.mat[ic.mi];
      const int r0 = ic.rb * kRows, j0 = ic.band * BN;
      const int nrows = min(kRows, M.m - r0);
      unsigned char* st = ring + (s % kStages) * L.stage_bytes();
      Tw* wt = reinterpret_cast<Tw*>(st);
      int* ps = reinterpret_cast<int*>(st + L.w_bytes());
      Tacc* vs = reinterpret_cast<Tacc*>(st + L.w_bytes() + L.pos_bytes());
      const Tw* in = static_cast<const Tw*>(M.in);
      if (M.vec) {
        if (use_in) {
#pragma unroll
          for (int p = 0; p < kPieces; p += kDecThreads) {
            const int row = my_row + p / PPR;
            if (p + tid < kPieces && row < nrows) {
              const int col = j0 + my_pc * EPP;
              const int valid = max(0, min(EPP, M.n - col));
              const Tw* src = in + static_cast<long long>(r0 + row) * M.ldi + (valid ? col : 0);
              cp_async16(wt + row * BN + my_pc * EPP, src, valid * static_cast<int>(sizeof(Tw)));
            }
          }
        }
        const int pbytes = nrows * r * 4, vbytes = nrows * r * static_cast<int>(sizeof(Tacc));
        const char* psrc = reinterpret_cast<const char*>(M.ppos + static_cast<long long>(r0) * r);
        const char* vsrc = reinterpret_cast<const char*>(static_cast<const Tacc*>(M.pval) +
                                                         static_cast<long long>(r0) * r);
        for (int p = tid * 16; p < pbytes; p += kDecThreads * 16)
          cp_async16(reinterpret_cast<char*>(ps) + p, psrc + p, min(16, pbytes - p));
        for (int p = tid * 16; p < vbytes; p += kDecThreads * 16)
          cp_async16(reinterpret_cast<char*>(vs) + p, vsrc + p, min(16, vbytes - p));
      } else {
        if (use_in)
          for (int p = tid; p < nrows * BN; p += kDecThreads) {
            const int row = p / BN, c = p % BN, col = j0 + c;
            wt[p] = col < M.n ? in[static_cast<long long>(r0 + row) * M.ldi + col] : Tw(0.0f);
          }
        const Tacc* pval = static_cast<const Tacc*>(M.pval);
        for (int p = tid; p < nrows * r; p += kDecThreads) {
          ps[p] = M.ppos[static_cast<long long>(r0) * r + p];
          vs[p] = pval[static_cast<long long>(r0) * r + p];
        }
      }
      advance(A, ic);
    }
    cp_async_commit();  // always commit: keeps the group count uniform
  };

  // ---- Y_band for (matrix, band) -----------------------------------------------
  auto build_y = [&](const DecMat& M, int band) {
    const Tacc* qval = static_cast<const Tacc*>(M.qval);
    const Tacc* dT = static_cast<const Tacc*>(M.dT);
    const int j0 = band * BN;
    for (int jj = warp; jj < BN; jj += kDecWarps) {
      const int j = j0 + jj;
      for (int a0 = 0; a0 < d; a0 += 32 * 32) {
        Tacc y[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) y[t] = Tacc(0);
        if (j < M.n) {
          for (int l = 0; l < r; ++l) {
            const int b = __ldg(M.qpos + static_cast<long long>(j) * r + l);
            const Tacc q = __ldg(qval + static_cast<long long>(j) * r + l);
            const Tacc* row = dT + static_cast<long long>(b) * d + a0 + lane;
#pragma unroll
            for (int t = 0; t < 32; ++t)
              if (a0 + lane + 32 * t < d) y[t] = fma(q, row[32 * t], y[t]);
          }
        }
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const int a = a0 + lane + 32 * t;
          if (a < d) Y[a * LDY + jj] = y[t];
        }
      }
    }
  };

  // ---- consumer -----------------------------------------------------------------
  constexpr int RPW = 32 / BN;  // rows per warp instruction
  const int jj = lane % BN, rsub = lane / BN;
  double ss = 0.0;

  for (int s = 0; s < kStages - 1; ++s) issue(s);
  Cursor cc = cursor_at(A, t_begin);
  int cur_band = -1, cur_mat = -1;
  for (int s = 0; s < ntiles; ++s, advance(A, cc)) {
    const DecMat& M = A.mat[cc.mi];
    if (cc.band != cur_band || cc.mi != cur_mat) {
      __syncthreads();  // everyone is done with the previous Y_band
      build_y(M, cc.band);
      cur_band = cc.band;
      cur_mat = cc.mi;
    }
    cp_async_wait<kStages - 2>();
    __syncthreads();  // stage s visible to all; stage s-1 fully consumed
    issue(s + kStages - 1);
    const unsigned char* st = ring + (s % kStages) * L.stage_bytes();
    const Tw* wt = reinterpret_cast<const Tw*>(st);
    const int* ps = reinterpret_cast<const int*>(st + L.w_bytes());
    const Tacc* vs = reinterpret_cast<const Tacc*>(st + L.w_bytes() + L.pos_bytes());
    const int r0 = cc.rb * kRows;
    const int nrows = min(kRows, M.m - r0);
    const int j = cc.band * BN + jj;
    const bool col_ok = j < M.n;
    Tw* out = static_cast<Tw*>(M.out);
    const long long ldo = M.ldo;
    Tw* orow = out ? out + static_cast<long long>(r0) * ldo + j : nullptr;
#pragma unroll 2
    for (int q = warp * RPW + rsub; q < nrows; q += kDecWarps * RPW) {
      Tacc acc = Tacc(0);
      if constexpr (KR == 4 && sizeof(Tacc) == 4) {
        const int4 pp = *reinterpret_cast<const int4*>(ps + q * 4);
        const float4 vv = *reinterpret_cast<const float4*>(vs + q * 4);
        acc = fma(vv.x, Y[pp.x * LDY + jj], acc);
        acc = fma(vv.y, Y[pp.y * LDY + jj], acc);
        acc = fma(vv.z, Y[pp.z * LDY + jj], acc);
        acc = fma(vv.w, Y[pp.w * LDY + jj], acc);
      } else {
#pragma unroll
        for (int l = 0; l < (KR > 0 ? KR : 1); ++l) {
          if (KR > 0 || l < r) acc = fma(vs[q * r + l], Y[ps[q * r + l] * LDY + jj], acc);
        }
        if constexpr (KR == 0) {
          for (int l = 1; l < r; ++l) acc = fma(vs[q * r + l], Y[ps[q * r + l] * LDY + jj], acc);
        }
      }
      if (!col_ok) continue;
      Tacc res = alpha * acc;
      if (use_in) res = fma(beta, cvt<Tacc>(wt[q * BN + jj]), res);
      if (orow) orow[q * ldo] = cvt<Tw>(res);
      if constexpr (SUMSQ) {
        const double rv = orow ? static_cast<double>(cvt<Tacc>(cvt<Tw>(res)))
                               : static_cast<double>(res);
        ss += rv * rv;
      }
    }
  }
  cp_async_wait<0>();
  if constexpr (SUMSQ) {
    __shared__ double red[kDecWarps];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    __syncthreads();
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kDecWarps; ++w) t += red[w];
      A.partials[blockIdx.x] = t;
    }
  }
}

template <typename Tw, typename Tacc, int BN, int KR, bool SUMSQ>
void decompress_impl(const std::vector<DecJob>& jobs, double alpha, double beta,
                     const int* skip, DevBuf* partials, int* nparts, cudaStream_t st) {
  const Pair& p0 = *jobs[0].pr;
  const Layout<Tw, Tacc, BN> L{p0.d, p0.p->r};
  const int smem = L.total();
  auto kern = k_decompress_band<Tw, Tacc, BN, KR, SUMSQ>;
  LSP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  DecArgs A{};
  A.count = static_cast<int>(jobs.size());
  A.d = p0.d, A.r = p0.p->r;
  A.alpha = alpha, A.beta = beta;
  long long total = 0;
  for (size_t i = 0; i < jobs.size(); ++i) {
    const DecJob& J = jobs[i];
    const Pair& pr = *J.pr;
    DecMat& M = A.mat[i];
    M.m = pr.m, M.n = pr.n;
    M.ppos = pr.p->pos.as<int>(), M.pval = pr.p->val.p;
    M.qpos = pr.q->pos.as<int>(), M.qval = pr.q->val.p;
    M.dT = J.delta_t;
    M.in = J.in, M.ldi = J.ldi, M.out = J.out, M.ldo = J.ldo;
    M.row_blocks = ceil_div(pr.m, kRows);
    M.nbands = ceil_div(pr.n, BN);
    total += static_cast<long long>(M.nbands) * M.row_blocks;
    M.tile_end = total;
    const bool w_ok = J.in == nullptr ||
                      (reinterpret_cast<uintptr_t>(J.in) % 16 == 0 &&
                       (J.ldi * static_cast<long long>(sizeof(Tw))) % 16 == 0);
    M.vec = (w_ok && reinterpret_cast<uintptr_t>(pr.p->pos.p) % 16 == 0 &&
             reinterpret_cast<uintptr_t>(pr.p->val.p) % 16 == 0 &&
             (BN * sizeof(Tw)) % 16 == 0) ? 1 : 0;
  }
  A.total = total;
  A.skip = skip;
  A.use_in = beta != 0.0;
  for (const DecJob& J : jobs) A.use_in = A.use_in && J.in != nullptr;
  int per_sm = 0;
  LSP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDecThreads, smem));
  per_sm = std::max(per_sm, 1);
  const int grid = static_cast<int>(std::min<long long>(total, 1LL * per_sm * sm_budget(kBudgetUpdate)));
  if (nparts) *nparts = grid;
  if (SUMSQ) partials->ensure(static_cast<size_t>(grid) * sizeof(double));
  A.partials = SUMSQ ? partials->as<double>() : nullptr;
  if (grid <= 0) return;
  kern<<<grid, kDecThreads, smem, st>>>(A);
  after_launch("decompress_band");
}

}  // namespace

// LSP_DECOMPRESS_GENERIC=1 forces the cp.async kernel (tests cover both paths).
static bool force_generic() {
  const char* e = std::getenv("LSP_DECOMPRESS_GENERIC");
  return e && e[0] == '1';
}

void launch_decompress_group(const std::vector<DecJob>& jobs, lsp_dtype dt, double alpha,
                             double beta, const int* skip_flag, DevBuf* partials, int* nparts,
                             cudaStream_t st) {
  if (nparts) *nparts = 0;
  if (jobs.empty()) return;
  require(jobs.size() <= static_cast<size_t>(kMaxGroup), "group too large");
  const Pair& p0 = *jobs[0].pr;
  for (const DecJob& J : jobs)
    require(J.pr->d == p0.d && J.pr->p->r == p0.p->r && J.pr->compute == p0.compute,
            "decompress group: matrices must share d, r and compute dtype");
  std::vector<DecJob> rest;
  if (!partials && !force_generic()) {
    // fast paths per matrix (Y precompute / row orientation); the others below
    std::vector<DecJob> fast;
    for (const DecJob& J : jobs)
      (decompress_fast_eligible(J, dt, beta) ? fast : rest).push_back(J);
    if (!fast.empty()) launch_decompress_group_y(fast, dt, alpha, beta, skip_flag, st);
    if (rest.empty()) return;
  }
  const std::vector<DecJob>& jobs_left = rest.empty() ? jobs : rest;
  if (!partials && !force_generic() &&
      launch_decompress_group_tma(jobs_left, dt, alpha, beta, skip_flag, st))
    return;
  LSP_DISPATCH_ACC(p0.compute, Tacc, {
    LSP_DISPATCH_STORAGE(dt, Tw, {
      constexpr int kBudget = 220 * 1024;
      const int r = p0.p->r, d = p0.d;
      auto run = [&](auto bn) {
        constexpr int BN = decltype(bn)::value;
        if (partials) {
          decompress_impl<Tw, Tacc, BN, 0, true>(jobs_left, alpha, beta, skip_flag, partials, nparts, st);
        } else if (r == 4) {
          decompress_impl<Tw, Tacc, BN, 4, false>(jobs_left, alpha, beta, skip_flag, partials, nparts, st);
        } else {
          decompress_impl<Tw, Tacc, BN, 0, false>(jobs_left, alpha, beta, skip_flag, partials, nparts, st);
        }
      };
      if (Layout<Tw, Tacc, 32>{d, r}.total() <= kBudget)
        run(std::integral_constant<int, 32>{});
      else if (Layout<Tw, Tacc, 16>{d, r}.total() <= kBudget)
        run(std::integral_constant<int, 16>{});
      else if (Layout<Tw, Tacc, 8>{d, r}.total() <= kBudget)
        run(std::integral_constant<int, 8>{});
      else if (Layout<Tw, Tacc, 4>{d, r}.total() <= kBudget)
        run(std::integral_constant<int, 4>{});
      else
        fail(LSP_EINVAL, "decompress: subspace width too large for the band kernel");
    })
  })
}

void launch_decompress(const Pair& pr, const void* delta_t, const void* in, long long ldi,
                       void* out, long long ldo, lsp_dtype dt, double alpha, double beta,
                       const int* skip_flag, DevBuf* partials, int* nparts, cudaStream_t st) {
  if (pr.m <= 0 || pr.n <= 0) {
    if (nparts) *nparts = 0;
    return;
  }
  std::vector<DecJob> jobs{DecJob{&pr, delta_t, in, ldi, out, ldo}};
  launch_decompress_group(jobs, dt, alpha, beta, skip_flag, partials, nparts, st);
}

}  // namespace lspb
