// Decompress-and-apply in fp64 (the reference's precision): W = beta*W +
// alpha * P Delta Q^T for fp64 W, projectors and Delta (reference:
// decompress, proj/src/projector.cpp:170-175; apply, proj/src/trainer.cpp:190).
//
// The fp64 twin of the fp32 Y path (apply.cu), same two kernels per group:
//   1. k_build_y64: Y = Delta Q^T into band blocks Yb[band][a][16] (16 fp64
//      columns = 128-byte rows, so a band block is d x 128 B, 128 KB at
//      d = 1024).  A CTA = (band, 128-row chunk of a); lane = 2 consecutive a,
//      so each gather of a Delta^T row segment is one coalesced 256-byte
//      LDG.128 from L2; staged in shared memory (16-byte granules XOR-swizzled
//      by row) and written with coalesced 16-byte stores.
//   2. k_apply_y64: persistent, one CTA per SM; warp 0 streams 64-row x
//      16-column W tiles (8 KB, 2-D TMA) and the tile rows' P entries through
//      an mbarrier ring, warp 1 bulk-copies the unit's Y block, 16 consumer
//      warps in 2 groups take alternate tiles; each lane owns 2 adjacent
//      columns (16-byte Y gathers, W loads and stores).
// Per element: acc = v0 * Y[p0]; acc = fma(v_l, Y[p_l], acc); res = alpha*acc;
// res = fma(beta, w, res), and Y[a][j] = fma chain over Q's row j from 0 -- the
// order of the in-kernel-build kernel (decompress_tma.cu), so the two fp64
// paths are bitwise equal.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "core.cuh"
#include "tma.cuh"

namespace lspb {

namespace {

constexpr int kBN = 16;               // band width (fp64 columns)
constexpr int kTR = 64;               // W rows per ring tile (8 KB)
constexpr int kYRows = 128;           // a-rows per build CTA
constexpr int kNC64 = 16;             // consumer warps
constexpr int kNG64 = 2;              // consumer groups
constexpr int kThreads64 = (kNC64 + 2) * 32;
constexpr int kMaxStages64 = 16;
constexpr int kYChunk64 = 16 * 1024;
constexpr int kSmemMax64 = 227 * 1024;

// ---------------------------------------------------------------------------
// Y build
// ---------------------------------------------------------------------------
struct YMat64 {
  const int* qpos;
  const double* qval;
  const double* dT;  // Delta^T: element (a, b) of Delta at b*d + a
  double* yb;
  int n, nbands;
  long long task_end;
};
struct YArgs64 {
  YMat64 mat[kMaxGroup];
  int count, d, ablocks;
  long long total;
  const int* skip;
};

template <int KR>
__global__ void __launch_bounds__(256) k_build_y64(const __grid_constant__ YArgs64 A) {
  __shared__ __align__(16) double tile[kYRows * kBN];  // 16 KB
  if (A.skip && *A.skip) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long task = blockIdx.x;  // (matrix, band, a-chunk), a-chunk fastest
  int mi = 0;
  while (mi + 1 < A.count && task >= A.mat[mi].task_end) ++mi;
  const YMat64& M = A.mat[mi];
  const int lt = static_cast<int>(task - (mi ? A.mat[mi - 1].task_end : 0));
  const int band = lt / A.ablocks;
  const int sb = lt - band * A.ablocks;
  const int d = A.d;
  const int cg = warp & 3, ab = warp >> 2;  // 4 column groups of 4 x 2 a-halves of 64
  const int al = ab * 64 + 2 * lane;        // first of this lane's 2 rows within the chunk
  const int a = sb * kYRows + al;
  const bool a_ok = a < d;  // d even (host check)
  double y[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    y[t][0] = y[t][1] = 0.0;
    const int j = band * kBN + cg * 4 + t;
    if (j < M.n) {
#pragma unroll
      for (int e = 0; e < KR; ++e) {
        const int b = __ldg(M.qpos + static_cast<long long>(j) * KR + e);
        const double q = __ldg(M.qval + static_cast<long long>(j) * KR + e);
        double2 x = make_double2(0.0, 0.0);
        if (a_ok) x = __ldg(reinterpret_cast<const double2*>(M.dT + static_cast<long long>(b) * d + a));
        y[t][0] = fma(q, x.x, y[t][0]);
        y[t][1] = fma(q, x.y, y[t][1]);
      }
    }
  }
  // stage: row al + c, granules 2*cg + h (2 doubles each) of the row's 8,
  // physical granule = g ^ ((row >> 1) & 7): the 8 lanes of a store phase hit
  // 8 distinct bank groups
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int row = al + c;
    const int key = (row >> 1) & 7;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int g = (2 * cg + h) ^ key;
      *reinterpret_cast<double2*>(tile + row * kBN + 2 * g) = make_double2(y[2 * h][c], y[2 * h + 1][c]);
    }
  }
  __syncthreads();
  const int rows = min(kYRows, d - sb * kYRows);
  const unsigned long long pol_last = policy_evict_last();
  double* out = M.yb + (static_cast<long long>(band) * d + sb * kYRows) * kBN;
  for (int gi = threadIdx.x; gi < rows * (kBN / 2); gi += blockDim.x) {
    const int row = gi >> 3, g = gi & 7;
    const double2 v = *reinterpret_cast<const double2*>(tile + row * kBN + 2 * (g ^ ((row >> 1) & 7)));
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(out + 2 * gi), "d"(v.x),
                 "d"(v.y), "l"(pol_last)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// streaming apply
// ---------------------------------------------------------------------------
struct alignas(64) AMat64 {
  CUtensorMap tmap;        // W (input) tile map: box kBN x kTR
  const int* ppos_scaled;  // P positions * kBN * 8: byte offsets of Y rows
  const double* pval;
  const double* yb;
  double* out;
  long long ldo;
  int m, n, row_blocks, nbands, rps;
  long long unit_end;
};
struct AArgs64 {
  AMat64 mat[kMaxGroup];
  int count, d, stages, stage_bytes, y_bytes, p_bytes;
  long long units;
  double alpha, beta;
  const int* skip;
};

struct Unit64 {
  int mi, band, rb0, rb1;
};
__device__ __forceinline__ Unit64 unit64_at(const AArgs64& A, long long u) {
  int i = 0;
  while (i + 1 < A.count && u >= A.mat[i].unit_end) ++i;
  const AMat64& M = A.mat[i];
  const long long lt = u - (i ? A.mat[i - 1].unit_end : 0);
  const int seg = static_cast<int>(lt / M.nbands);
  const int rb0 = seg * M.rps;
  return Unit64{i, static_cast<int>(lt % M.nbands), rb0, min(M.row_blocks, rb0 + M.rps)};
}

__device__ __forceinline__ double2 lds_d2(unsigned addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ int lds_i(unsigned addr) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ double lds_d1(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void st_d2(double* a, double2 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(a), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_d1(double* a, double v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(a), "d"(v), "l"(pol) : "memory");
}

template <int KR, bool USE_IN>
__global__ void __launch_bounds__(kThreads64, 1) k_apply_y64(const __grid_constant__ AArgs64 A) {
  constexpr int LPR = kBN / 2;  // lanes per W row (2 columns each)
  constexpr int RPW = 32 / LPR;  // rows per warp instruction
  constexpr int WB = kTR * kBN * 8;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  if (A.skip && *A.skip) return;
  unsigned char* ring = smem_raw + A.y_bytes;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(ring + A.stages * A.stage_bytes);
  unsigned long long* empty = full + A.stages;
  unsigned long long* yfull = empty + A.stages;
  unsigned long long* yempty = yfull + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int S = A.stages;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kNC64 / kNG64);
    }
    mbar_init(yfull, 1);
    mbar_init(yempty, kNC64);
    fence_mbar_init();
  }
  __syncthreads();
  const long long u_first = blockIdx.x, u_step = gridDim.x;
  if (u_first >= A.units) return;

  if (warp == 0) {  // W / P-entry producer
    if (lane == 0) {
      const unsigned long long pol = policy_evict_first();
      int st = 0, rnd = 0;
      for (long long u = u_first; u < A.units; u += u_step) {
        const Unit64 U = unit64_at(A, u);
        const AMat64& M = A.mat[U.mi];
        for (int rb = U.rb0; rb < U.rb1; ++rb, (++st == S) ? (st = 0, ++rnd) : 0) {
          if (rnd > 0) mbar_wait(empty + st, (rnd - 1) & 1);
          const int r0 = rb * kTR;
          const int nrows = min(kTR, M.m - r0);
          unsigned char* base = ring + st * A.stage_bytes;
          // odd row counts with KR = 2: the 16-byte bulk granule (arrays carry slack)
          const unsigned pb = (static_cast<unsigned>(nrows) * KR * 4u + 15u) & ~15u;
          const unsigned vb = static_cast<unsigned>(nrows) * KR * 8u;
          mbar_arrive_expect_tx(full + st, (USE_IN ? WB : 0) + pb + vb);
          if (USE_IN) tma_load_2d(base, &M.tmap, U.band * kBN, r0, full + st, pol);
          bulk_load(base + WB, M.ppos_scaled + static_cast<long long>(r0) * KR, pb, full + st);
          bulk_load(base + WB + A.p_bytes, M.pval + static_cast<long long>(r0) * KR, vb, full + st);
        }
      }
    }
    return;
  }
  if (warp == 1) {  // Y block producer
    if (lane == 0) {
      int k = 0;
      for (long long u = u_first; u < A.units; u += u_step, ++k) {
        const Unit64 U = unit64_at(A, u);
        if (k > 0) mbar_wait(yempty, (k - 1) & 1);
        mbar_arrive_expect_tx(yfull, static_cast<unsigned>(A.y_bytes));
        const unsigned char* src =
            reinterpret_cast<const unsigned char*>(A.mat[U.mi].yb + static_cast<long long>(U.band) * A.d * kBN);
        for (int off = 0; off < A.y_bytes; off += kYChunk64)
          bulk_load(smem_raw + off, src + off, min(kYChunk64, A.y_bytes - off), yfull);
      }
    }
    return;
  }

  // consumers
  constexpr int WPG = kNC64 / kNG64;
  constexpr int kq = WPG * RPW;        // row step between a lane's rows
  constexpr int RPT = kTR / kq;        // rows per lane per tile
  const int cw = warp - 2;
  const int grp = cw / WPG, gw = cw % WPG;
  const double alpha = A.alpha, beta = A.beta;
  const int jj = (lane % LPR) * 2, rsub = lane / LPR;
  const int q0 = gw * RPW + rsub;
  const unsigned y_lane = smem_addr(smem_raw) + jj * 8u;
  const unsigned ring_s = smem_addr(ring);
  const unsigned long long pol_first = policy_evict_first();
  int s = 0, k = 0, st = 0, rnd = 0;
  for (long long u = u_first; u < A.units; u += u_step, ++k) {
    const Unit64 U = unit64_at(A, u);
    const AMat64& M = A.mat[U.mi];
    const int j = U.band * kBN + jj;
    const bool col_ok = j < M.n, pair_ok = j + 2 <= M.n;
    double* const ocol = M.out + j;
    const long long ldo = M.ldo;
    mbar_wait(yfull, k & 1);
    for (int rb = U.rb0; rb < U.rb1; ++rb, ++s, (++st == S) ? (st = 0, ++rnd) : 0) {
      if (s % kNG64 != grp) continue;
      const int r0 = rb * kTR;
      const int nrows = min(kTR, M.m - r0);
      mbar_wait(full + st, rnd & 1);
      const unsigned base = ring_s + st * A.stage_bytes;
      const unsigned wq = base + (q0 * kBN + jj) * 8u;
      const unsigned pq = base + WB + q0 * KR * 4u;
      const unsigned vq = base + WB + A.p_bytes + q0 * KR * 8u;
      auto row = [&](int v) {
        double2 acc;
#pragma unroll
        for (int l = 0; l < KR; ++l) {
          const int p = lds_i(pq + (v * kq * KR + l) * 4u);
          const double vv = lds_d1(vq + (v * kq * KR + l) * 8u);
          const double2 yv = lds_d2(y_lane + p);
          if (l == 0) {
            acc.x = vv * yv.x;
            acc.y = vv * yv.y;
          } else {
            acc.x = fma(vv, yv.x, acc.x);
            acc.y = fma(vv, yv.y, acc.y);
          }
        }
        acc.x = alpha * acc.x;
        acc.y = alpha * acc.y;
        if (USE_IN) {
          const double2 w = lds_d2(wq + v * kq * kBN * 8u);
          acc.x = fma(beta, w.x, acc.x);
          acc.y = fma(beta, w.y, acc.y);
        }
        return acc;
      };
      if (col_ok) {
        double* const orow = ocol + static_cast<long long>(r0 + q0) * ldo;
        if (pair_ok && nrows == kTR) {
#pragma unroll
          for (int v = 0; v < RPT; ++v) st_d2(orow + static_cast<long long>(v) * kq * ldo, row(v), pol_first);
        } else {
#pragma unroll 1
          for (int v = 0; v < RPT && q0 + v * kq < nrows; ++v) {
            const double2 x = row(v);
            double* o = orow + static_cast<long long>(v) * kq * ldo;
            if (pair_ok) {
              st_d2(o, x, pol_first);
            } else {
              st_d1(o, x.x, pol_first);  // the last (odd) column of n
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
    }
    if (lane == 0) mbar_arrive(yempty);
  }
}

template <int KR>
void build_y64_impl(const std::vector<DecJob>& jobs_in, const int* skip, cudaStream_t st) {
  // reverse matrix order: the apply's first Y blocks are the last written (L2)
  const std::vector<DecJob> jobs(jobs_in.rbegin(), jobs_in.rend());
  YArgs64 A{};
  A.count = static_cast<int>(jobs.size());
  A.d = jobs[0].pr->d;
  A.ablocks = ceil_div(A.d, kYRows);
  A.skip = skip;
  long long total = 0;
  for (size_t i = 0; i < jobs.size(); ++i) {
    const Pair& pr = *jobs[i].pr;
    YMat64& M = A.mat[i];
    M.qpos = pr.q->pos.as<int>();
    M.qval = pr.q->val.as<double>();
    M.dT = static_cast<const double*>(jobs[i].delta_t);
    M.yb = pr.yb.as<double>();
    M.n = pr.n;
    M.nbands = ceil_div(pr.n, kBN);
    total += static_cast<long long>(M.nbands) * A.ablocks;
    M.task_end = total;
  }
  A.total = total;
  if (total == 0) return;
  k_build_y64<KR><<<static_cast<unsigned>(total), 256, 0, st>>>(A);
  after_launch("build_y64");
}

template <int KR>
bool apply_y64_impl(const std::vector<DecJob>& jobs, double alpha, double beta, const int* skip,
                    cudaStream_t st) {
  const Pair& p0 = *jobs[0].pr;
  const bool use_in = beta != 0.0;
  AArgs64 A{};
  A.count = static_cast<int>(jobs.size());
  A.d = p0.d;
  A.alpha = alpha;
  A.beta = beta;
  A.skip = skip;
  A.y_bytes = p0.d * kBN * 8;
  A.p_bytes = static_cast<int>(round_up(kTR * KR * 4, 16));
  A.stage_bytes = static_cast<int>(round_up(kTR * kBN * 8 + A.p_bytes + kTR * KR * 8, 128));
  const int bar_bytes = (2 * kMaxStages64 + 2) * 8;
  A.stages = std::min(kMaxStages64, (kSmemMax64 - A.y_bytes - bar_bytes) / A.stage_bytes);
  A.stages -= A.stages % kNG64;  // each stage belongs to one consumer group
  if (A.stages < kNG64) return false;
  const int smem = A.y_bytes + A.stages * A.stage_bytes + bar_bytes;
  auto kern = use_in ? k_apply_y64<KR, true> : k_apply_y64<KR, false>;
  LSP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid_max = sm_budget(kBudgetUpdate);
  long long tiles = 0;
  for (const DecJob& J : jobs) tiles += static_cast<long long>(ceil_div(J.pr->n, kBN)) * ceil_div(J.pr->m, kTR);
  const long long cap = std::max<long long>(8, tiles / grid_max / 4);
  long long units = 0;
  for (size_t i = 0; i < jobs.size(); ++i) {
    const DecJob& J = jobs[i];
    const Pair& pr = *J.pr;
    AMat64& M = A.mat[i];
    if (use_in && !cached_tmap(&M.tmap, J.in, LSP_F64, pr.m, pr.n, J.ldi, kBN, kTR)) return false;
    M.ppos_scaled = pr.p->scaled_pos(kBN * 8);
    M.pval = pr.p->val.as<double>();
    M.yb = pr.yb.as<double>();
    M.out = static_cast<double*>(J.out);
    M.ldo = J.ldo;
    M.m = pr.m, M.n = pr.n;
    M.row_blocks = ceil_div(pr.m, kTR);
    M.nbands = ceil_div(pr.n, kBN);
    const int segs = static_cast<int>(ceil_div(static_cast<long long>(M.row_blocks), cap));
    M.rps = ceil_div(M.row_blocks, segs);
    units += static_cast<long long>(M.nbands) * ceil_div(M.row_blocks, M.rps);
    M.unit_end = units;
  }
  A.units = units;
  if (units == 0) return true;
  const int grid = static_cast<int>(std::min<long long>(units, grid_max));
  kern<<<grid, kThreads64, smem, st>>>(A);
  after_launch("apply_y64");
  return true;
}

template <int KR>
bool run64(const std::vector<DecJob>& jobs, double alpha, double beta, const int* skip, cudaStream_t st,
           int phase) {
  for (const DecJob& J : jobs)
    J.pr->yb_ensure(static_cast<size_t>(ceil_div(J.pr->n, kBN)) * J.pr->d * kBN * sizeof(double));
  if (phase & kPhaseBuild) build_y64_impl<KR>(jobs, skip, st);
  if (phase & kPhaseApply)
    require(apply_y64_impl<KR>(jobs, alpha, beta, skip, st), "apply_y64: launch configuration rejected");
  return true;
}

}  // namespace

// Per-matrix eligibility of the fp64 Y path.
bool y64_eligible(const DecJob& J, lsp_dtype dt, double beta) {
  const Pair& pr = *J.pr;
  if (pr.compute != LSP_F64 || dt != LSP_F64) return false;
  const int r = pr.p->r;
  if ((r != 2 && r != 4 && r != 8) || pr.q->r != r) return false;
  if (pr.d % 2 || pr.d * kBN * 8 > 160 * 1024) return false;
  if (reinterpret_cast<uintptr_t>(J.delta_t) % 16) return false;  // 16-byte Delta^T loads
  if (J.ldo % 2 || reinterpret_cast<uintptr_t>(J.out) % 16) return false;  // 16-byte stores
  if (beta != 0.0 && (J.in == nullptr || reinterpret_cast<uintptr_t>(J.in) % 16 || J.ldi % 2)) return false;
  const char* band = std::getenv("LSP_DECOMPRESS_BAND");
  return !(band && band[0] == '1');
}

// The fp64 group (every job y64_eligible, shared d and r): Y build and / or apply.
void launch_y64_group(const std::vector<DecJob>& jobs, double alpha, double beta, const int* skip,
                      cudaStream_t st, int phase) {
  const int r = jobs[0].pr->p->r, d = jobs[0].pr->d;
  for (const DecJob& J : jobs)
    require(J.pr->p->r == r && J.pr->d == d, "decompress group: matrices must share d and r");
  if (r == 4) run64<4>(jobs, alpha, beta, skip, st, phase);
  else if (r == 8) run64<8>(jobs, alpha, beta, skip, st, phase);
  else run64<2>(jobs, alpha, beta, skip, st, phase);
}

}  // namespace lspb
