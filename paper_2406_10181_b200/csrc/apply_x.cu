// Fused decompress-and-apply, ROW orientation, for fp32 W with n > m
// (opt-in: LSP_APPLY_ROWS=1; see apply_x_eligible for the measurement)
// (reference: left_mul proj/src/projector.cpp:105-117, rightT_mul :148-161,
//  decompress :170-175, apply W -= lr * decompress proj/src/trainer.cpp:190):
//
//   out = beta * in + alpha * (P Delta) Q^T
//
// The column orientation (apply.cu) keeps Y = Delta Q^T for a 32-column band
// resident and streams W in 128-byte-wide row pieces, which caps a B200 at
// ~4.8 TB/s (tools/micro/stream_rmw.cu: 128-byte column bands); 512-byte
// rows reach 5.8-6.5 TB/s.  Here the resident operand is X = P Delta for a
// band of 32 ROWS (32 x d), so W tiles can be as wide as we like:
//
// 1. k_build_x: X = P Delta (m x d) from row gathers of the row-major Delta
//    (a transpose of the stored Delta^T), stored with row pitch d + 1 so that
//    32 lanes = 32 rows reading the same column hit 32 different banks (one
//    address add per gather).  For the n > m matrices X is smaller than Y
//    (m x d vs d x n).
// 2. k_apply_x: persistent, one CTA per SM; units = (matrix, 32-row band,
//    column segment), dealt round-robin in (matrix, band, segment) order.
//    Warp 0 streams W tiles of 32 rows x 128 columns (four 32x32 2-D TMA boxes
//    with the 128-byte swizzle: 512-byte rows) plus the tile columns' CSR
//    entries of Q; warp 1 bulk-copies the band's X block (32 x d) into shared
//    memory per unit; 16 consumer warps in 2 groups take alternate tiles.
//    Lane = row: per 4-column chunk one conflict-free 16-byte read of W (the
//    swizzle spreads 8 rows over 8 bank groups), 16 conflict-free X gathers
//    X[row][pos_q(j,l)], the result written back in place; the group
//    then TMA-stores the tile (W read and written exactly once).
//
// Arithmetic: x(i,b) = sum_k p(i,k) Delta[pos_p(i,k)][b] (CSR order), then
// w(i,j) = beta*w + alpha*sum_l q(j,l) x(i,pos_q(j,l)): the same products as
// the column form in the other association ((P Delta) Q^T vs P (Delta Q^T)),
// so results agree with it to rounding, not bitwise.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "core.cuh"
#include "tma.cuh"

namespace lspb {

namespace {

constexpr int kXR = 32;                 // W rows per band (= lanes)
constexpr int kXBoxes = 4;              // 32-column boxes per tile
constexpr int kXCols = 32 * kXBoxes;    // tile columns (512-byte rows)
constexpr int kXNC = 16;                // consumer warps
constexpr int kXNG = 2;                 // consumer groups (alternate tiles)
constexpr int kXWPG = kXNC / kXNG;      // warps per group
constexpr int kXThreads = (kXNC + 2) * 32;
constexpr int kXMaxD = 1024;            // X block = 32 x d fp32 <= 128 KB
constexpr int kXChunk = 16 * 1024;      // bulk-copy granule of the X block
constexpr int kXSmemMax = 227 * 1024;

// ---------------------------------------------------------------------------
// X build
// ---------------------------------------------------------------------------
struct BXMat {
  const int* ppos;
  const float* pval;
  const float* drow;  // Delta, row-major d x d
  float* xs;          // X, m_pad x d, row-swizzled
  int m, m_pad;
  long long row_end;  // cumulative m_pad
};
struct BXArgs {
  BXMat mat[kMaxGroup];
  int count, d;
  long long rows;
  const int* skip;
};

// one warp = one row i of X; lane covers b = 128*s + 4*lane .. +3
template <int KR>
__global__ void __launch_bounds__(256) k_build_x(const __grid_constant__ BXArgs A) {
  if (A.skip && *A.skip) return;
  const int lane = threadIdx.x & 31;
  const long long r = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (r >= A.rows) return;
  int mi = 0;
  while (mi + 1 < A.count && r >= A.mat[mi].row_end) ++mi;
  const BXMat& M = A.mat[mi];
  const int i = static_cast<int>(r - (mi ? A.mat[mi - 1].row_end : 0));
  const int d = A.d;
  float* xrow = M.xs + static_cast<long long>(i) * (d + 1);  // pitch d + 1
  if (i >= M.m) {  // padding rows of the last band
    for (int b = lane; b <= d; b += 32) xrow[b] = 0.0f;
    return;
  }
  int p[KR];
  float v[KR];
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    p[k] = __ldg(M.ppos + static_cast<long long>(i) * KR + k);
    v[k] = __ldg(M.pval + static_cast<long long>(i) * KR + k);
  }
  for (int b0 = 4 * lane; b0 < d; b0 += 128) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(M.drow + static_cast<long long>(p[k]) * d + b0));
      acc[0] = fmaf(v[k], x.x, acc[0]);
      acc[1] = fmaf(v[k], x.y, acc[1]);
      acc[2] = fmaf(v[k], x.z, acc[2]);
      acc[3] = fmaf(v[k], x.w, acc[3]);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) xrow[b0 + c] = acc[c];
  }
  if (lane == 0) xrow[d] = 0.0f;  // the pad column
}

// ---------------------------------------------------------------------------
// streaming apply
// ---------------------------------------------------------------------------
struct alignas(64) XMat {
  CUtensorMap tmap;  // W, box 32 x 32, 128-byte swizzle (load and store)
  const int* qpos;
  const float* qval;
  const float* xs;
  int m, n, nbands, ntiles, tps;  // tps: column tiles per unit (segment)
  long long unit_end;
};
struct XArgs {
  XMat mat[kMaxGroup];
  int count, d, stages, stage_bytes, xb_bytes, e_bytes;
  long long units;
  double alpha, beta;
  const int* skip;
};

struct XUnit {
  int mi, band, t0, t1;
};
__device__ __forceinline__ XUnit xunit_at(const XArgs& A, long long u) {
  int i = 0;
  while (i + 1 < A.count && u >= A.mat[i].unit_end) ++i;
  const XMat& M = A.mat[i];
  const long long lt = u - (i ? A.mat[i - 1].unit_end : 0);
  const int segs = (M.ntiles + M.tps - 1) / M.tps;
  const int seg = static_cast<int>(lt % segs);
  return XUnit{i, static_cast<int>(lt / segs), seg * M.tps, min(M.ntiles, (seg + 1) * M.tps)};
}

__device__ __forceinline__ float4 ldsx4(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ int4 ldsi4(unsigned a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float ldsx(unsigned a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void stsx4(unsigned a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

template <int KR, bool USE_IN>
__global__ void __launch_bounds__(kXThreads, 1) k_apply_x(const __grid_constant__ XArgs A) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  if (A.skip && *A.skip) return;
  // the 128-byte swizzle repeats every 1024 bytes: align the layout explicitly
  unsigned char* smem_raw = smem_dyn + ((1024u - (smem_addr(smem_dyn) & 1023u)) & 1023u);
  unsigned char* ring = smem_raw + ((A.xb_bytes + 1023) & ~1023);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(ring + A.stages * A.stage_bytes);
  unsigned long long* empty = full + A.stages;
  unsigned long long* xfull = empty + A.stages;
  unsigned long long* xempty = xfull + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int S = A.stages;
  constexpr int kBoxBytes = 32 * kXR * 4;  // 4 KB
  constexpr int kWBytes = kXBoxes * kBoxBytes;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);  // the group's storer, after the tile's TMA store read it
    }
    mbar_init(xfull, 1);
    mbar_init(xempty, kXNC);
    fence_mbar_init();
  }
  __syncthreads();
  if (blockIdx.x >= A.units) return;

  if (warp == 0) {
    // ---------------- W / Q-entry producer ----------------
    if (lane == 0) {
      const unsigned long long pol = policy_evict_first();
      int s = 0;
      for (long long u = blockIdx.x; u < A.units; u += gridDim.x) {
        const XUnit U = xunit_at(A, u);
        const XMat& M = A.mat[U.mi];
        for (int ct = U.t0; ct < U.t1; ++ct, ++s) {
          const int st = s % S;
          if (s >= S) mbar_wait(empty + st, ((s / S) - 1) & 1);
          unsigned char* base = ring + st * A.stage_bytes;
          const int j0 = ct * kXCols;
          const int ncols = min(kXCols, M.n - j0);
          const unsigned eb = static_cast<unsigned>(ncols) * KR * 4u;
          mbar_arrive_expect_tx(full + st, (USE_IN ? kWBytes : 0) + 2u * eb);
          if (USE_IN)
            for (int b = 0; b < kXBoxes; ++b)
              tma_load_2d(base + b * kBoxBytes, &M.tmap, j0 + 32 * b, U.band * kXR, full + st, pol);
          bulk_load(base + kWBytes, M.qpos + static_cast<long long>(j0) * KR, eb, full + st);
          bulk_load(base + kWBytes + A.e_bytes, M.qval + static_cast<long long>(j0) * KR, eb,
                    full + st);
        }
      }
    }
    return;
  }
  if (warp == 1) {
    // ---------------- X block producer (one bulk copy per unit) ----------------
    if (lane == 0) {
      int k = 0;
      for (long long u = blockIdx.x; u < A.units; u += gridDim.x, ++k) {
        const XUnit U = xunit_at(A, u);
        if (k > 0) mbar_wait(xempty, (k - 1) & 1);
        mbar_arrive_expect_tx(xfull, static_cast<unsigned>(A.xb_bytes));
        const unsigned char* src = reinterpret_cast<const unsigned char*>(
            A.mat[U.mi].xs + static_cast<long long>(U.band) * kXR * (A.d + 1));
        for (int off = 0; off < A.xb_bytes; off += kXChunk)
          bulk_load(smem_raw + off, src + off, min(kXChunk, A.xb_bytes - off), xfull);
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int cw = warp - 2;
  const int grp = cw / kXWPG, gw = cw % kXWPG;
  const float alpha = static_cast<float>(A.alpha), beta = static_cast<float>(A.beta);
  // X block row pitch d + 1 floats: lane = row reading column b hits bank (lane + b) % 32
  const unsigned xs_lane = smem_addr(smem_raw) + static_cast<unsigned>(lane * (A.d + 1)) * 4u;
  const unsigned ring_s = smem_addr(ring);
  int s = 0, k = 0;
  for (long long u = blockIdx.x; u < A.units; u += gridDim.x, ++k) {
    const XUnit U = xunit_at(A, u);
    const XMat& M = A.mat[U.mi];
    mbar_wait(xfull, k & 1);
    for (int ct = U.t0; ct < U.t1; ++ct, ++s) {
      if (s % kXNG != grp) continue;
      const int st = s % S;
      mbar_wait(full + st, (s / S) & 1);
      const unsigned base = ring_s + st * A.stage_bytes;
      const unsigned qp = base + kWBytes, qv = base + kWBytes + A.e_bytes;
      const int ncols = min(kXCols, M.n - ct * kXCols);
      // chunk ch = 4 columns: box ch / 8, 16-byte chunk ch % 8 of the row
      auto tile = [&](auto full_tile) {
        constexpr bool FULL = decltype(full_tile)::value;
#pragma unroll
        for (int h = 0; h < kXBoxes * 8 / kXWPG; ++h) {
          const int ch = gw + h * kXWPG;
          const int bx = ch >> 3, c = ch & 7;
          const unsigned waddr = base + bx * kBoxBytes + lane * 128 + ((c ^ (lane & 7)) << 4);
          float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
          if (USE_IN) w = ldsx4(waddr);
          float r[4];
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const int jl = ch * 4 + cc;  // column within the tile
            float acc = 0.0f;
#pragma unroll
            for (int l = 0; l < KR; l += 4) {
              int4 pp = ldsi4(qp + (jl * KR + l) * 4u);
              float4 vv = ldsx4(qv + (jl * KR + l) * 4u);
              if (!FULL && jl >= ncols) {
                // columns beyond n (last tile): entries forced to (0, 0) --
                // reads X[row][0] times 0; the TMA store clips them
                pp = make_int4(0, 0, 0, 0);
                vv = make_float4(0.f, 0.f, 0.f, 0.f);
              }
              const float x0 = ldsx(xs_lane + (pp.x << 2));
              const float x1 = ldsx(xs_lane + (pp.y << 2));
              const float x2 = ldsx(xs_lane + (pp.z << 2));
              const float x3 = ldsx(xs_lane + (pp.w << 2));
              acc = l == 0 ? vv.x * x0 : fmaf(vv.x, x0, acc);
              acc = fmaf(vv.y, x1, acc);
              acc = fmaf(vv.z, x2, acc);
              acc = fmaf(vv.w, x3, acc);
            }
            r[cc] = alpha * acc;
          }
          if (USE_IN) {
            r[0] = fmaf(beta, w.x, r[0]);
            r[1] = fmaf(beta, w.y, r[1]);
            r[2] = fmaf(beta, w.z, r[2]);
            r[3] = fmaf(beta, w.w, r[3]);
          }
          stsx4(waddr, make_float4(r[0], r[1], r[2], r[3]));
        }
      };
      if (ncols == kXCols)
        tile(std::true_type{});  // straight-line, no per-column selects
      else
        tile(std::false_type{});
      fence_proxy_async_smem();                // generic-proxy writes -> TMA store
      named_barrier_sync(2 + grp, kXWPG * 32);  // the group's whole tile written
      if (gw == 0 && lane == 0) {
        for (int b = 0; b < kXBoxes; ++b)
          if (32 * b < ncols)
            tma_store_2d(&M.tmap, ct * kXCols + 32 * b, U.band * kXR,
                         ring + st * A.stage_bytes + b * kBoxBytes);
        bulk_commit();
        bulk_wait_read0();  // shared memory read by the store: the stage is free
        mbar_arrive(empty + st);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(xempty);  // this unit's X block may be replaced
  }
  if (gw == 0 && lane == 0) bulk_wait0();  // stores complete before exit
}

template <int KR>
void build_x_impl(const std::vector<DecJob>& jobs, const int* skip, cudaStream_t st) {
  const Pair& p0 = *jobs[0].pr;
  const int d = p0.d;
  BXArgs A{};
  A.count = static_cast<int>(jobs.size());
  A.d = d;
  A.skip = skip;
  long long rows = 0;
  for (size_t i = 0; i < jobs.size(); ++i) {
    const Pair& pr = *jobs[i].pr;
    // Delta (row-major) from the stored Delta^T
    launch_transpose(d, d, jobs[i].delta_t, d, pr.drow.p, d, LSP_F32, st);
    BXMat& M = A.mat[i];
    M.ppos = pr.p->pos.as<int>();
    M.pval = pr.p->val.as<float>();
    M.drow = pr.drow.as<float>();
    M.xs = pr.xs.as<float>();
    M.m = pr.m;
    M.m_pad = static_cast<int>(round_up(pr.m, kXR));
    rows += M.m_pad;
    M.row_end = rows;
  }
  A.rows = rows;
  k_build_x<KR><<<static_cast<unsigned>((rows + 7) / 8), 256, 0, st>>>(A);
  after_launch("build_x");
}

template <int KR>
bool apply_x_impl(const std::vector<DecJob>& jobs, double alpha, double beta, const int* skip,
                  cudaStream_t st) {
  const Pair& p0 = *jobs[0].pr;
  const bool use_in = beta != 0.0;
  XArgs A{};
  A.count = static_cast<int>(jobs.size());
  A.d = p0.d;
  A.alpha = alpha;
  A.beta = beta;
  A.skip = skip;
  A.xb_bytes = kXR * (p0.d + 1) * 4;  // multiple of 16: one bulk copy stream
  A.e_bytes = kXCols * KR * 4;
  A.stage_bytes = static_cast<int>(round_up(kXBoxes * 32 * kXR * 4 + 2 * A.e_bytes, 1024));
  const int bar_bytes = (2 * 8 + 2) * 8;
  const int xb_al = static_cast<int>(round_up(A.xb_bytes, 1024));
  A.stages = std::min(8, (kXSmemMax - 1024 - xb_al - bar_bytes) / A.stage_bytes);
  A.stages -= A.stages % kXNG;  // one group per stage (see apply.cu, stage parity)
  if (A.stages < 3) return false;
  const int grid_max = sm_budget(kBudgetUpdate);
  long long tiles = 0;
  for (const DecJob& J : jobs)
    tiles += static_cast<long long>(ceil_div(J.pr->m, kXR)) * ceil_div(J.pr->n, kXCols);
  // units of at most ~1/6 of a CTA's share, so the round-robin deal stays balanced
  const long long cap = std::max<long long>(4, tiles / grid_max / 6);
  long long units = 0;
  for (size_t i = 0; i < jobs.size(); ++i) {
    const DecJob& J = jobs[i];
    const Pair& pr = *J.pr;
    XMat& M = A.mat[i];
    if (!cached_tmap(&M.tmap, J.out, LSP_F32, pr.m, pr.n, J.ldo, 32, kXR, /*swz128=*/true))
      return false;
    M.qpos = pr.q->pos.as<int>();
    M.qval = pr.q->val.as<float>();
    M.xs = pr.xs.as<float>();
    M.m = pr.m, M.n = pr.n;
    M.nbands = ceil_div(pr.m, kXR);
    M.ntiles = ceil_div(pr.n, kXCols);
    const int segs = static_cast<int>(ceil_div(M.ntiles, cap));
    M.tps = ceil_div(M.ntiles, segs);
    units += static_cast<long long>(M.nbands) * ceil_div(M.ntiles, M.tps);
    M.unit_end = units;
  }
  A.units = units;
  if (units == 0) return true;
  const int smem = 1024 + xb_al + A.stages * A.stage_bytes + bar_bytes;
  auto kern = use_in ? k_apply_x<KR, true> : k_apply_x<KR, false>;
  LSP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid = static_cast<int>(std::min<long long>(units, grid_max));
  kern<<<grid, kXThreads, smem, st>>>(A);
  after_launch("apply_x");
  return true;
}

}  // namespace

// Is this matrix served by the row orientation?  Opt-in (LSP_APPLY_ROWS=1):
// measured on B200 for the C4 gate/up matrices it runs at 4.2 TB/s (164 us
// for two 4096 x 11008 fp32 matrices, latency-bound on the per-unit X block
// and the group store barrier), below the column form's 4.65 TB/s, so the
// column form stays the default.  Conditions: fp32 everything, n > m,
// d <= 1024 and a multiple of 32, r in {4, 8}, W in place or output only,
// 16-byte aligned rows.
bool apply_x_eligible(const DecJob& J, lsp_dtype dt, double beta) {
  const char* env = std::getenv("LSP_APPLY_ROWS");
  const bool off = !(env && env[0] == '1');
  const Pair& pr = *J.pr;
  if (off || dt != LSP_F32 || pr.compute != LSP_F32) return false;
  if (!(pr.n > pr.m) || pr.d > kXMaxD || pr.d % 32 || pr.p->r % 4 || pr.q->r != pr.p->r) return false;
  if (pr.p->r != 4 && pr.p->r != 8) return false;
  if (beta != 0.0 && J.in != J.out) return false;
  if (reinterpret_cast<uintptr_t>(J.out) % 16 || (J.ldo * 4) % 16) return false;
  return true;
}

// phase: kPhaseBuild (Delta transpose + X build), kPhaseApply, or both.
void launch_apply_x(const std::vector<DecJob>& jobs, double alpha, double beta,
                    const int* skip_flag, cudaStream_t st, int phase) {
  if (jobs.empty()) return;
  const int r = jobs[0].pr->p->r;
  for (const DecJob& J : jobs) {
    const Pair& pr = *J.pr;
    pr.xs_ensure(static_cast<size_t>(round_up(pr.m, kXR)) * (pr.d + 1) * sizeof(float),
                 static_cast<size_t>(pr.d) * pr.d * sizeof(float));
  }
  if (phase & kPhaseBuild) r == 4 ? build_x_impl<4>(jobs, skip_flag, st) : build_x_impl<8>(jobs, skip_flag, st);
  if (phase & kPhaseApply) {
    const bool ok = r == 4 ? apply_x_impl<4>(jobs, alpha, beta, skip_flag, st)
                           : apply_x_impl<8>(jobs, alpha, beta, skip_flag, st);
    require(ok, "apply_x: launch configuration rejected");
  }
}

}  // namespace lspb
