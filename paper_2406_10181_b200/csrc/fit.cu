// Projector fit (Eq. 3) and optimizer-state transfer, on the device in fp64.
//
// Reference: fit_loss / fit_gradient / fit  proj/src/projector.cpp:189-315,
//            projector_gram / reproject_state proj/src/subspace_opt.cpp:59-101.
//
// The reference materialises the m x n bias B = P S Q^T - G and dense m x d,
// n x d products (O((m+n) d^2) per target, 19.7 s at 2048x5504, d=1024).  Here
// every product is factored through the sparse projectors, so nothing larger
// than max(m,n) x d is formed and no dense d^3 GEMM is needed:
//   S   = P^T G Q                          (compress, stage 1 + 2)
//   A1  = Gp S = P^T (P S)                 (two row gathers)
//   V   = Q A1^T = (A1 Q^T)^T
//   D   = Gp S Gq - 2 S ,  D^T = Q^T V - 2 S^T
//   |B|^2 = |P S Q^T - G|^2 evaluated directly by the decompress kernel in
//           sum-of-squares mode (no m x n write, no cancellation)
//   dL/dP(i,a) = 2/T [ (P A2)[i,:] . S[a,:]  + X[i,:] . D[a,:] ],  A2 = S Gq, X = G Q
//   dL/dQ(j,b) = 2/T [ V[j,:] . S^T[b,:]     + Z^T[j,:] . D^T[b,:] ], Z^T = G^T P
// (derivation in DESIGN.md).  Everything runs in fp64 on shadow fp64 copies of
// the projectors; the fitted values are written back to the pair at the end.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "core.cuh"
#include "host_projector.h"

struct lsp_projector_s : lspb::Projector {};
struct lsp_pair_s : lspb::Pair {};
struct lsp_adam_s : lspb::Adam {};

namespace lspb {
extern thread_local std::string g_last_error;

namespace {

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
constexpr int kRedBlocks = 512;

// Deterministic per-block partial dot products <a, b> over `cnt` elements.
__global__ void k_dot(long long cnt, const double* __restrict__ a, const double* __restrict__ b,
                      double* __restrict__ partials) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt;
       i += (long long)gridDim.x * blockDim.x)
    s = fma(a[i], b[i], s);
  __shared__ double red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 256; ++i) t += red[i];
    partials[blockIdx.x] = t;
  }
}

// grad[r*k + l] += scale * ( A1[r,:].B1[pos[r*k+l],:] + A2[r,:].B2[pos[r*k+l],:] )
// One warp per row r; lanes take 2 adjacent columns per 64-column chunk
// (16-byte loads when d is even; ld = d); the k entries' dot products
// share the row's A1/A2 loads.
__global__ void k_sddmm(int R, int k, int d, const int* __restrict__ pos,
                        const double* __restrict__ A1, const double* __restrict__ B1,
                        const double* __restrict__ A2, const double* __restrict__ B2, int ld,
                        double scale, double* __restrict__ grad) {
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  for (int r = blockIdx.x * warps + (threadIdx.x >> 5); r < R; r += gridDim.x * warps) {
    const double* a1 = A1 + static_cast<long long>(r) * ld;
    const double* a2 = A2 + static_cast<long long>(r) * ld;
    for (int l0 = 0; l0 < k; l0 += 4) {
      const int nl = min(4, k - l0);
      const double* b1[4];
      const double* b2[4];
      double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const int b = l < nl ? __ldg(pos + static_cast<long long>(r) * k + l0 + l) : 0;
        b1[l] = B1 + static_cast<long long>(b) * ld;
        b2[l] = B2 + static_cast<long long>(b) * ld;
      }
      if (d & 1) {  // odd widths: scalar columns
        for (int c = lane; c < d; c += 32) {
#pragma unroll
          for (int l = 0; l < 4; ++l)
            if (l < nl) s[l] = fma(a1[c], b1[l][c], fma(a2[c], b2[l][c], s[l]));
        }
      } else
      for (int c = 2 * lane; c < d; c += 64) {
        const double2 x1 = __ldg(reinterpret_cast<const double2*>(a1 + c));
        const double2 x2 = __ldg(reinterpret_cast<const double2*>(a2 + c));
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          if (l >= nl) continue;
          const double2 y1 = __ldg(reinterpret_cast<const double2*>(b1[l] + c));
          const double2 y2 = __ldg(reinterpret_cast<const double2*>(b2[l] + c));
          s[l] = fma(x1.x, y1.x, fma(x2.x, y2.x, s[l]));
          s[l] = fma(x1.y, y1.y, fma(x2.y, y2.y, s[l]));
        }
      }
#pragma unroll
      for (int l = 0; l < 4; ++l) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s[l] += __shfl_xor_sync(0xffffffffu, s[l], o);
        if (lane == 0 && l < nl) grad[static_cast<long long>(r) * k + l0 + l] += scale * s[l];
      }
    }
  }
}

// Fused trial prologue, one 32 x 32 tile per block, gridDim.z = target:
//   S^T(t) = s0 - t s1 + t^2 s2 (s1 == nullptr: S^T = s0 as given, not rewritten)
// written to sT, its transpose to s, and per-block partial sums of |S|^2 in
// fixed order (partials[z][block]).  Replaces a separate polynomial, transpose
// and dot-product pass.
__global__ void k_poly_tile(int d, long long dd, const double* s0, const double* __restrict__ s1,
                            const double* __restrict__ s2, double t, double* sT,
                            double* __restrict__ s, double* __restrict__ partials) {  // s0 may alias sT
  __shared__ double tile[32][33];
  __shared__ double red[256];
  const long long off = static_cast<long long>(blockIdx.z) * dd;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;  // column / row of S^T
  double ss = 0.0;
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int r = by + y, c = bx + threadIdx.x;
    double v = 0.0;
    if (r < d && c < d) {
      const long long i = off + static_cast<long long>(r) * d + c;
      if (s1) {
        v = fma(t * t, s2[i], fma(-t, s1[i], s0[i]));
        sT[i] = v;
      } else {
        v = s0[i];
      }
      ss = fma(v, v, ss);
    }
    tile[y][threadIdx.x] = v;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int r = bx + y, c = by + threadIdx.x;  // S[r][c] = S^T[c][r]
    if (r < d && c < d) s[off + static_cast<long long>(r) * d + c] = tile[threadIdx.x][y];
  }
  const int tid = threadIdx.y * 32 + threadIdx.x;
  red[tid] = ss;
  __syncthreads();
  if (tid == 0) {
    double x = 0.0;
    for (int i = 0; i < 256; ++i) x += red[i];
    partials[static_cast<long long>(blockIdx.z) * gridDim.x * gridDim.y + blockIdx.y * gridDim.x + blockIdx.x] = x;
  }
}

// <Gp S, S Gq> = <Q A1^T, Q S^T> (A1 = Gp S): per row j of Q, u = sum_l q_jl
// A1^T[pos_jl] and w = sum_l q_jl S^T[pos_jl] (row gathers of the L2-resident
// d x d operands, never written) and u . w; one warp per row, gridDim.y =
// target, per-block partials in fixed order (partials[y][block]).  Replaces the
// n x d intermediate Q S^T, its CSC gather and a dot-product pass.
constexpr int kQdWarps = 8;
__global__ void __launch_bounds__(kQdWarps * 32)
    k_qdot(int d, int n, int k, long long dd, const int* __restrict__ pos, const double* __restrict__ val,
           const double* __restrict__ a1t, const double* __restrict__ st, double* __restrict__ partials) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long off = static_cast<long long>(blockIdx.y) * dd;
  double acc = 0.0;
  for (int j = blockIdx.x * kQdWarps + warp; j < n; j += gridDim.x * kQdWarps) {
    const int* pj = pos + static_cast<long long>(j) * k;
    const double* vj = val + static_cast<long long>(j) * k;
    if ((d & 1) == 0) {
      for (int c = 2 * lane; c < d; c += 64) {
        double2 u = make_double2(0.0, 0.0), w = make_double2(0.0, 0.0);
        for (int l = 0; l < k; ++l) {
          const long long row = off + static_cast<long long>(__ldg(pj + l)) * d + c;
          const double q = __ldg(vj + l);
          const double2 x = __ldg(reinterpret_cast<const double2*>(a1t + row));
          const double2 y = __ldg(reinterpret_cast<const double2*>(st + row));
          u.x = fma(q, x.x, u.x), u.y = fma(q, x.y, u.y);
          w.x = fma(q, y.x, w.x), w.y = fma(q, y.y, w.y);
        }
        acc = fma(u.x, w.x, fma(u.y, w.y, acc));
      }
    } else {
      for (int c = lane; c < d; c += 32) {
        double u = 0.0, w = 0.0;
        for (int l = 0; l < k; ++l) {
          const long long row = off + static_cast<long long>(__ldg(pj + l)) * d + c;
          const double q = __ldg(vj + l);
          u = fma(q, a1t[row], u);
          w = fma(q, st[row], w);
        }
        acc = fma(u, w, acc);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double red[kQdWarps];
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0;
    for (int i = 0; i < kQdWarps; ++i) x += red[i];
    partials[static_cast<long long>(blockIdx.y) * gridDim.x + blockIdx.x] = x;
  }
}
constexpr int kQdBlocks = 296;  // per target

// out (da x db, row-major) = A^T B for two projectors over the same rows, in
// the reference's summation order (rows ascending per output entry,
// subspace_opt.cpp:59-70), without contraction so fp64 results match it.
template <typename Ta, typename Tb>
__global__ void k_gram(int da, int db, int rb, const int* __restrict__ a_csc_ptr,
                       const int* __restrict__ a_csc_row, const Ta* __restrict__ a_csc_val,
                       const int* __restrict__ b_pos, const Tb* __restrict__ b_val,
                       double* __restrict__ out) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < da; x += gridDim.x * blockDim.x) {
    double* orow = out + static_cast<long long>(x) * db;
    for (int t = a_csc_ptr[x]; t < a_csc_ptr[x + 1]; ++t) {
      const int i = a_csc_row[t];
      const double va = static_cast<double>(a_csc_val[t]);
      for (int kb = 0; kb < rb; ++kb) {
        const long long e = static_cast<long long>(i) * rb + kb;
        const int y = b_pos[e];
        orow[y] = __dadd_rn(orow[y], __dmul_rn(va, static_cast<double>(b_val[e])));
      }
    }
  }
}

// fp64 GEMM C = A (MxK) * B (KxN), row-major, on the FP64 tensor cores
// (mma.sync m8n8k4 f64 -> DMMA): 64 x 64 block tiles (256 CTAs at d = 1024),
// K staged 16 at a time through shared memory with the next slice prefetched
// into registers, 4 warps of 32 x 32 (4 x 4 MMA tiles of 8 x 8: 8 fragment
// loads per 16 MMAs).  Used only by reproject_state's d^3
// transfer products (the one dense contraction on the path);
// zero-filled edges handle any M, N, K.
constexpr int kMT = 64, kNT = 64, kKT = 16, kGW = 4;  // 4 warps of 32 x 32
__global__ void __launch_bounds__(kGW * 32) k_dgemm(int M, int N, int K, const double* __restrict__ A,
                                               const double* __restrict__ B, double* __restrict__ C) {
  __shared__ double As[kMT][kKT + 1];
  __shared__ double Bs[kKT][kNT + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;  // 2 x 2 warps, warp tile 32 x 32
  const int row0 = blockIdx.y * kMT, col0 = blockIdx.x * kNT;
  const int g = lane >> 2, q = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  double ra[kMT * kKT / (kGW * 32)], rb[kKT * kNT / (kGW * 32)];  // next K slice, in registers
  auto fetch = [&](int k0) {
#pragma unroll
    for (int i = 0; i < kMT * kKT / (kGW * 32); ++i) {
      const int t = tid + kGW * 32 * i, r = t / kKT, c = t % kKT;
      ra[i] = (row0 + r < M && k0 + c < K) ? A[static_cast<long long>(row0 + r) * K + k0 + c] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < kKT * kNT / (kGW * 32); ++i) {
      const int t = tid + kGW * 32 * i, r = t / kNT, c = t % kNT;
      rb[i] = (k0 + r < K && col0 + c < N) ? B[static_cast<long long>(k0 + r) * N + col0 + c] : 0.0;
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int i = 0; i < kMT * kKT / (kGW * 32); ++i) {
      const int t = tid + kGW * 32 * i;
      As[t / kKT][t % kKT] = ra[i];
    }
#pragma unroll
    for (int i = 0; i < kKT * kNT / (kGW * 32); ++i) {
      const int t = tid + kGW * 32 * i;
      Bs[t / kNT][t % kNT] = rb[i];
    }
  };
  fetch(0);
  stash();
  __syncthreads();
  for (int k0 = 0; k0 < K; k0 += kKT) {
    if (k0 + kKT < K) fetch(k0 + kKT);  // global loads of the next slice overlap the MMAs
#pragma unroll
    for (int kk = 0; kk < kKT; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) a[mt] = As[wm * 32 + mt * 8 + g][kk + q];   // A: row g, k q
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) b[nt] = Bs[kk + q][wn * 32 + nt * 8 + g];   // B: k q, col g
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
              : "=d"(acc[mt][nt][0]), "=d"(acc[mt][nt][1])
              : "d"(a[mt]), "d"(b[nt]), "d"(acc[mt][nt][0]), "d"(acc[mt][nt][1]));
    }
    __syncthreads();  // the slice is consumed
    if (k0 + kKT < K) {
      stash();
      __syncthreads();
    }
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int r = row0 + wm * 32 + mt * 8 + g, c = col0 + wn * 32 + nt * 8 + 2 * q;  // D: row g, cols 2q, 2q+1
      if (r < M && c < N) C[static_cast<long long>(r) * N + c] = acc[mt][nt][0];
      if (r < M && c + 1 < N) C[static_cast<long long>(r) * N + c + 1] = acc[mt][nt][1];
    }
}

__global__ void k_square(long long cnt, double* __restrict__ x) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = x[i] * x[i];
}
__global__ void k_clamp0(long long cnt, double* __restrict__ x) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt;
       i += (long long)gridDim.x * blockDim.x)
    if (x[i] < 0.0) x[i] = 0.0;
}

int egrid(long long cnt) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>((cnt + 255) / 256, 4096)));
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
double dot_sync(const double* a, const double* b, long long cnt, DevBuf& parts, cudaStream_t st) {
  parts.ensure(kRedBlocks * sizeof(double));
  k_dot<<<kRedBlocks, 256, 0, st>>>(cnt, a, b, parts.as<double>());
  after_launch("dot");
  return reduce_partials_sync(parts.as<double>(), kRedBlocks, st);
}

void dgemm(int M, int N, int K, const double* A, const double* B, double* C, cudaStream_t st) {
  dim3 grid(ceil_div(N, kNT), ceil_div(M, kMT));
  k_dgemm<<<grid, kGW * 32, 0, st>>>(M, N, K, A, B, C);
  after_launch("dgemm");
}

// out = alpha * (rows of src gathered by the CSR of P) [+ beta*in]
void csr_gather(const Projector& P, const double* src, int c, double* out,
                cudaStream_t st, double beta = 0.0, const double* in = nullptr) {
  launch_gather(P.n_rows, c, nullptr, P.r, P.pos.as<int>(), P.val.p, LSP_F64, src, c, LSP_F64,
                in, c, out, c, LSP_F64, 1.0, beta, nullptr, nullptr, st);
}
void csc_gather(const Projector& P, const double* src, int c, double* out,
                cudaStream_t st, double beta = 0.0, const double* in = nullptr) {
  launch_gather(P.d, c, P.csc_ptr.as<int>(), 0, P.csc_row.as<int>(), P.csc_val.p, LSP_F64, src,
                c, LSP_F64, in, c, out, c, LSP_F64, 1.0, beta, nullptr, nullptr, st);
}

std::unique_ptr<lsp_projector_s> shadow64(const Projector& P, const std::vector<double>& vals) {
  auto S = std::make_unique<lsp_projector_s>();
  S->n_rows = P.n_rows;
  S->d = P.d;
  S->r = P.r;
  S->compute = LSP_F64;
  S->h_pos = P.h_pos;
  S->h_val = vals;
  S->h_csc_ptr = P.h_csc_ptr;
  S->h_csc_rows = P.h_csc_rows;
  S->h_csc_perm = P.h_csc_perm;
  const size_t nnz = P.nnz();
  auto up = [](DevBuf& b, const void* src, size_t bytes) {
    b.ensure(std::max<size_t>(bytes, 16));
    if (bytes) LSP_CUDA(cudaMemcpy(b.p, src, bytes, cudaMemcpyHostToDevice));
  };
  up(S->pos, S->h_pos.data(), nnz * 4);
  up(S->csc_ptr, S->h_csc_ptr.data(), S->h_csc_ptr.size() * 4);
  up(S->csc_row, S->h_csc_rows.data(), nnz * 4);
  up(S->csc_perm, S->h_csc_perm.data(), nnz * 4);
  S->csc_val.ensure(std::max<size_t>(nnz * 8, 16));
  up(S->val, vals.data(), nnz * 8);
  launch_refresh_values(*S, nullptr);
  return S;
}

void set_values64(Projector& S, const std::vector<double>& vals, cudaStream_t st) {
  S.h_val = vals;
  LSP_CUDA(cudaMemcpyAsync(S.val.p, vals.data(), vals.size() * 8, cudaMemcpyHostToDevice, st));
  launch_refresh_values(S, st);
}

// The fit engine: fp64 shadows of (P, Q), the targets and their transposes.
struct FitEngine {
  Pair& orig;
  int m, n, d, r, T;
  cudaStream_t st;
  std::unique_ptr<lsp_projector_s> P, Q, Pd, Qd;  // Pd, Qd: the descent direction's values
  // per target (contiguous, target-major): S^T(t) = s0T - t s1T + t^2 s2T, and the
  // batched loss intermediates
  DevBuf s0T, s1T, s2T, bsT, bs, bu, ba1, ba2T;
  DevBuf zt_all;  // per target Z^T = G^T P of the last gradient (reused by prepare_line)
  DevBuf dgp, dgq;  // gradient accumulators (values layout)
  std::vector<DevBuf> g, gT;  // fp64 targets and transposes
  std::vector<double> gnorm2;
  DevBuf sT, s, u, a1, a1T, v, dT, dd, qs, a2T, a2, w1, x, xT, z, zt, zdt, parts, lparts;

  FitEngine(Pair& pr, const void* const* targets, int t, long long ld, lsp_dtype dt,
            cudaStream_t stream)
      : orig(pr), m(pr.m), n(pr.n), d(pr.d), r(pr.p->r), T(t), st(stream) {
    require(t >= 1, "fit: empty target corpus");
    require(pr.p->r == pr.q->r, "fit: P and Q must have the same nonzeros per row");
    require(ld >= n, "fit: target leading dimension smaller than columns");
    P = shadow64(*pr.p, pr.p->h_val);
    Q = shadow64(*pr.q, pr.q->h_val);
    Pd = shadow64(*pr.p, pr.p->h_val);
    Qd = shadow64(*pr.q, pr.q->h_val);
    const size_t mn = static_cast<size_t>(m) * n;
    g.resize(t);
    gT.resize(t);
    gnorm2.resize(t);
    for (int i = 0; i < t; ++i) {
      require(targets[i] != nullptr, "fit: null target");
      g[i].ensure(mn * 8);
      gT[i].ensure(mn * 8);
      // dense fp64 copy (handles ld and dtype), then its transpose
      launch_convert2d(m, n, targets[i], ld, dt, g[i].p, n, LSP_F64, st);
      launch_transpose(m, n, g[i].p, n, gT[i].p, m, LSP_F64, st);
      gnorm2[i] = dot_sync(g[i].as<double>(), g[i].as<double>(), static_cast<long long>(mn), parts, st);
    }
    const size_t dd2 = static_cast<size_t>(d) * d * 8;
    for (DevBuf* b : {&sT, &s, &a1, &a1T, &dT, &dd, &a2T, &a2}) b->ensure(dd2);
    const size_t ms = static_cast<size_t>(m) * d * 8, ns = static_cast<size_t>(n) * d * 8;
    u.ensure(ms);
    w1.ensure(ms);
    x.ensure(ms);
    xT.ensure(ms);
    v.ensure(ns);
    qs.ensure(ns);
    zt.ensure(ns);
    z.ensure(ns);
  }

  void set_values(const std::vector<double>& pv, const std::vector<double>& qv) {
    set_values64(*P, pv, st);
    set_values64(*Q, qv, st);
  }

  // S^T = (P^T G_i Q)^T through row gathers: Z = P^T G_i (d x n, CSC of P),
  // Z^T (n x d) by a transpose, S^T = Q^T Z^T (CSC of Q).  Per output entry the
  // sums run over the CSC rows in ascending order, as stage 1 / stage 2 do.
  void compress(int i, double* ztp, double* sTp) {
    csc_gather(*P, g[i].as<double>(), n, z.as<double>(), st);      // Z   (d x n)
    launch_transpose(d, n, z.p, n, ztp, d, LSP_F64, st);           // Z^T (n x d)
    csc_gather(*Q, ztp, d, sTp, st);                               // S^T (d x d)
  }

  // Line search along (P, Q) - t (dP, dQ): the trial values are the current
  // ones minus t times the gradient, and S is bilinear in (P, Q), so
  //   S(t) = S0 - t S1 + t^2 S2,  S0 = P^T G Q,  S1 = dP^T G Q + P^T G dQ,
  //   S2 = dP^T G dQ
  // per target, computed once per GD step (two passes over G instead of one
  // per trial); a trial then costs only the d-wide gathers of bias2_from_bsT.
  // Requires the gradient at (pv, qv) just before: its Z0^T and S0^T (zt_all,
  // s0T) are reused, so a GD step makes one extra pass over each G (Zd).
  void prepare_line(const std::vector<double>& pv, const std::vector<double>& qv,
                    const std::vector<double>& gp, const std::vector<double>& gq) {
    set_values(pv, qv);
    set_values64(*Pd, gp, st);
    set_values64(*Qd, gq, st);
    const size_t dd = static_cast<size_t>(d) * d, nd = static_cast<size_t>(n) * d;
    for (DevBuf* b : {&s1T, &s2T}) b->ensure(T * dd * 8);
    zdt.ensure(nd * 8);
    for (int i = 0; i < T; ++i) {
      const double* z0t = zt_all.as<double>() + i * nd;
      double* s1 = s1T.as<double>() + i * dd;
      double* s2 = s2T.as<double>() + i * dd;
      csc_gather(*Pd, g[i].as<double>(), n, z.as<double>(), st);     // Zd  = dP^T G
      launch_transpose(d, n, z.p, n, zdt.p, d, LSP_F64, st);
      csc_gather(*Q, zdt.as<double>(), d, s1, st);                    // (dP^T G Q)^T
      csc_gather(*Qd, z0t, d, s1, st, 1.0, s1);                       // + (P^T G dQ)^T
      csc_gather(*Qd, zdt.as<double>(), d, s2, st);                   // S2^T
    }
  }

  // |b_i|^2 = |P S Q^T - G_i|^2 = |G_i|^2 - 2 |S|^2 + <Gp S, S Gq>  (S = P^T G_i Q,
  // so <P S Q^T, G_i> = |S|^2 and |P S Q^T|^2 = <Gp S Gq, S>), for every target
  // from S^T in bsT (T x d x d): one batched launch per product, the two d x d
  // dot products' partials of target i in lparts slot i (no host sync)
  // batch of T row gathers through projector X (CSR rows when csr, else CSC
  // bins) from src + i*sbs into out + i*obs; odd widths go target by target
  // through the generic gather
  void gather_batch(const Projector& X, bool csr, const double* src, long long sbs, double* out,
                    long long obs) {
    const int R = csr ? X.n_rows : X.d;
    const int* ptr = csr ? nullptr : X.csc_ptr.as<int>();
    const int k = csr ? X.r : 0;
    const int* idx = csr ? X.pos.as<int>() : X.csc_row.as<int>();
    const double* val = csr ? X.val.as<double>() : X.csc_val.as<double>();
    if (d % 2 == 0) {
      launch_gather_f64_batch(R, d, ptr, k, idx, val, src, d, sbs, nullptr, 0, 0, out, d, obs, T, 1.0, 0.0, st);
      return;
    }
    for (int i = 0; i < T; ++i)
      launch_gather(R, d, ptr, k, idx, val, LSP_F64, src + i * sbs, d, LSP_F64, nullptr, 0, out + i * obs, d,
                    LSP_F64, 1.0, 0.0, nullptr, nullptr, st);
  }

  void bias2_from_bsT(double line_t) {
    const size_t dd = static_cast<size_t>(d) * d, md = static_cast<size_t>(m) * d;
    bs.ensure(T * dd * 8), ba1.ensure(T * dd * 8), ba2T.ensure(T * dd * 8);
    bu.ensure(T * md * 8);
    const int tiles = ceil_div(d, 32);
    const size_t np = static_cast<size_t>(tiles) * tiles;
    lparts.ensure(T * (np + kQdBlocks) * sizeof(double));
    double* ss_parts = lparts.as<double>();
    double* ag_parts = lparts.as<double>() + T * np;
    const dim3 tg(tiles, tiles, T), tb(32, 8);
    // S^T (polynomial, or as compressed), its transpose S and |S|^2
    k_poly_tile<<<tg, tb, 0, st>>>(d, static_cast<long long>(dd), line_t >= 0.0 ? s0T.as<double>() : bsT.as<double>(),
                                   line_t >= 0.0 ? s1T.as<double>() : nullptr,
                                   line_t >= 0.0 ? s2T.as<double>() : nullptr, line_t, bsT.as<double>(),
                                   bs.as<double>(), ss_parts);
    after_launch("poly_tile");
    gather_batch(*P, true, bs.as<double>(), dd, bu.as<double>(), md);      // U    = P S
    gather_batch(*P, false, bu.as<double>(), md, ba1.as<double>(), dd);    // A1   = Gp S
    double* a1t = ba2T.as<double>();                                      // (buffer reuse)
    launch_transpose_batch(d, d, ba1.as<double>(), d, dd, a1t, d, dd, T, st);  // A1^T
    k_qdot<<<dim3(kQdBlocks, T), kQdWarps * 32, 0, st>>>(d, n, Q->r, static_cast<long long>(dd),
                                                          Q->pos.as<int>(), Q->val.as<double>(), a1t,
                                                          bsT.as<double>(), ag_parts);
    after_launch("qdot");
  }

  // all targets' |b_i|^2 with one synchronisation (clamped at 0: the identity
  // can round below zero for an exactly representable target); line_t >= 0:
  // S^T from the prepared line-search polynomial instead of a pass over G
  std::vector<double> bias2_all(double line_t = -1.0) {
    const size_t dd = static_cast<size_t>(d) * d;
    bsT.ensure(T * dd * 8);
    if (line_t < 0.0)
      for (int i = 0; i < T; ++i) compress(i, zt.as<double>(), bsT.as<double>() + i * dd);
    bias2_from_bsT(line_t);
    const int tiles = ceil_div(d, 32);
    const size_t np = static_cast<size_t>(tiles) * tiles;
    std::vector<double> h(T * (np + kQdBlocks));
    LSP_CUDA(cudaMemcpyAsync(h.data(), lparts.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    LSP_CUDA(cudaStreamSynchronize(st));
    std::vector<double> out(T);
    for (int i = 0; i < T; ++i) {
      double ss = 0.0, ag = 0.0;
      for (size_t b = 0; b < np; ++b) ss += h[i * np + b];
      for (int b = 0; b < kQdBlocks; ++b) ag += h[T * np + static_cast<size_t>(i) * kQdBlocks + b];
      out[i] = std::max(0.0, gnorm2[i] - 2.0 * ss + ag);
    }
    return out;
  }

  // Gradient chain for target i: S^T, Z^T, A1, V, D^T.
  void chain(int i, double* ztp, double* sTp) {
    compress(i, ztp, sTp);
    launch_transpose(d, d, sTp, d, s.p, d, LSP_F64, st);
    csr_gather(*P, s.as<double>(), d, u.as<double>(), st);         // U  = P S     (m x d)
    csc_gather(*P, u.as<double>(), d, a1.as<double>(), st);        // A1 = P^T U   (d x d)
    launch_transpose(d, d, a1.p, d, a1T.p, d, LSP_F64, st);
    csr_gather(*Q, a1T.as<double>(), d, v.as<double>(), st);       // V  = Q A1^T  (n x d)
    csc_gather(*Q, v.as<double>(), d, dT.as<double>(), st, -2.0, sTp);            // D^T
  }

  // loss = mean_t |b_t|^2 + reg ; rel = mean over nonzero targets of |b_t|/|G_t|
  void loss(const std::vector<double>& pv, const std::vector<double>& qv,
            const lsp_fit_config& cfg, double* loss_out, double* rel_out, double line_t = -1.0) {
    set_values(pv, qv);
    double sum = 0.0, rel = 0.0;
    int counted = 0;
    const std::vector<double> all = bias2_all(line_t);
    for (int i = 0; i < T; ++i) {
      const double b2 = all[i];
      sum += b2;
      if (gnorm2[i] > 0.0) {
        rel += std::sqrt(b2) / std::sqrt(gnorm2[i]);
        ++counted;
      }
    }
    *loss_out = sum / T + reg_term(pv, qv, cfg);
    if (rel_out) *rel_out = counted ? rel / counted : 0.0;
  }

  static double reg_term(const std::vector<double>& pv, const std::vector<double>& qv,
                         const lsp_fit_config& cfg) {
    if (cfg.reg_beta == 0.0) return 0.0;
    double ps = 0.0, qs2 = 0.0;
    for (double x : pv) ps += x * x;
    for (double x : qv) qs2 += x * x;
    if (cfg.reg_kind == LSP_REG_SQUARED) return cfg.reg_beta * (ps + qs2);
    return cfg.reg_beta * (std::sqrt(ps) + std::sqrt(qs2));
  }

  void gradient(const std::vector<double>& pv, const std::vector<double>& qv,
                const lsp_fit_config& cfg, std::vector<double>& gp, std::vector<double>& gq) {
    set_values(pv, qv);
    // members: a cudaMalloc / cudaFree pair per call cost up to ~8 ms per GD step
    // once the allocator had served earlier fits' multi-GB buffers
    dgp.ensure(std::max<size_t>(pv.size() * 8, 16));
    dgq.ensure(std::max<size_t>(qv.size() * 8, 16));
    LSP_CUDA(cudaMemsetAsync(dgp.p, 0, pv.size() * 8, st));
    LSP_CUDA(cudaMemsetAsync(dgq.p, 0, qv.size() * 8, st));
    const double scale = 2.0 / T;
    const size_t ddd = static_cast<size_t>(d) * d, nd = static_cast<size_t>(n) * d;
    s0T.ensure(T * ddd * 8);
    zt_all.ensure(T * nd * 8);
    for (int i = 0; i < T; ++i) {
      double* sTp = s0T.as<double>() + i * ddd;
      double* ztp = zt_all.as<double>() + i * nd;
      chain(i, ztp, sTp);                                           // S^T, Z^T, A1, V, D^T
      launch_transpose(d, d, dT.p, d, dd.p, d, LSP_F64, st);        // D
      csc_gather(*Q, gT[i].as<double>(), m, xT.as<double>(), st);  // X^T = Q^T G^T (d x m)
      launch_transpose(d, m, xT.p, m, x.p, d, LSP_F64, st);         // X = G Q    (m x d)
      csr_gather(*Q, sTp, d, qs.as<double>(), st);                  // Q S^T    (n x d)
      csc_gather(*Q, qs.as<double>(), d, a2T.as<double>(), st);     // A2^T = Gq S^T
      launch_transpose(d, d, a2T.p, d, a2.p, d, LSP_F64, st);       // A2 = S Gq
      csr_gather(*P, a2.as<double>(), d, w1.as<double>(), st);      // W1 = P A2 (m x d)
      k_sddmm<<<egrid(static_cast<long long>(m) * 32), 256, 0, st>>>(
          m, r, d, P->pos.as<int>(), w1.as<double>(), s.as<double>(), x.as<double>(), dd.as<double>(), d,
          scale, dgp.as<double>());
      after_launch("sddmm_p");
      k_sddmm<<<egrid(static_cast<long long>(n) * 32), 256, 0, st>>>(
          n, r, d, Q->pos.as<int>(), v.as<double>(), sTp, ztp, dT.as<double>(), d,
          scale, dgq.as<double>());
      after_launch("sddmm_q");
    }
    gp.resize(pv.size());
    gq.resize(qv.size());
    LSP_CUDA(cudaMemcpyAsync(gp.data(), dgp.p, gp.size() * 8, cudaMemcpyDeviceToHost, st));
    LSP_CUDA(cudaMemcpyAsync(gq.data(), dgq.p, gq.size() * 8, cudaMemcpyDeviceToHost, st));
    LSP_CUDA(cudaStreamSynchronize(st));
    // regulariser gradient (projector.cpp:34-54)
    if (cfg.reg_beta != 0.0) {
      if (cfg.reg_kind == LSP_REG_SQUARED) {
        for (size_t i = 0; i < gp.size(); ++i) gp[i] += 2.0 * cfg.reg_beta * pv[i];
        for (size_t i = 0; i < gq.size(); ++i) gq[i] += 2.0 * cfg.reg_beta * qv[i];
      } else {
        double pn = 0.0, qn = 0.0;
        for (double x2 : pv) pn += x2 * x2;
        for (double x2 : qv) qn += x2 * x2;
        pn = std::sqrt(pn);
        qn = std::sqrt(qn);
        if (pn > 0.0)
          for (size_t i = 0; i < gp.size(); ++i) gp[i] += cfg.reg_beta * pv[i] / pn;
        if (qn > 0.0)
          for (size_t i = 0; i < gq.size(); ++i) gq[i] += cfg.reg_beta * qv[i] / qn;
      }
    }
  }
};

lsp_fit_config cfg_or_default(const lsp_fit_config* cfg) {
  return cfg ? *cfg : lsp_fit_config_default();
}

template <typename F>
int guard_fit(F&& f) {
  try {
    f();
    return LSP_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return LSP_EINVAL;
  }
}

}  // namespace
}  // namespace lspb

using namespace lspb;

extern "C" {

int lsp_fit_loss(lsp_pair_t pair, const void* const* targets, int t, int64_t ld, lsp_dtype dtype,
                 const lsp_fit_config* cfg, double* loss, lsp_stream_t stream) {
  return guard_fit([&] {
    require(pair && targets && loss, "fit_loss: null argument");
    const lsp_fit_config c = cfg_or_default(cfg);
    FitEngine fe(*pair, targets, t, ld, dtype, as_stream(stream));
    fe.loss(pair->p->h_val, pair->q->h_val, c, loss, nullptr);
  });
}

int lsp_fit_gradient(lsp_pair_t pair, const void* const* targets, int t, int64_t ld,
                     lsp_dtype dtype, const lsp_fit_config* cfg, double* grad_p, double* grad_q,
                     lsp_stream_t stream) {
  return guard_fit([&] {
    require(pair && targets && grad_p && grad_q, "fit_gradient: null argument");
    const lsp_fit_config c = cfg_or_default(cfg);
    FitEngine fe(*pair, targets, t, ld, dtype, as_stream(stream));
    std::vector<double> gp, gq;
    fe.gradient(pair->p->h_val, pair->q->h_val, c, gp, gq);
    std::copy(gp.begin(), gp.end(), grad_p);
    std::copy(gq.begin(), gq.end(), grad_q);
  });
}

// fit: gradient descent on the values with a <=40-halving backtracking line
// search, stopping on mean relative bias <= alpha (projector.cpp:253-315).
int lsp_fit(lsp_pair_t pair, const void* const* targets, int t, int64_t ld, lsp_dtype dtype,
            const lsp_fit_config* cfg, lsp_fit_report* report, double* loss_curve, int max_curve,
            lsp_stream_t stream) {
  return guard_fit([&] {
    require(pair && targets && report, "fit: null argument");
    require(t >= 1, "fit: empty target corpus");
    const lsp_fit_config c = cfg_or_default(cfg);
    if (c.alpha <= 0.0 || c.alpha > 1.0) fail(LSP_EINVAL, "fit: alpha must be in (0, 1]");
    if (c.max_steps < 1) fail(LSP_EINVAL, "fit: max_steps must be >= 1");
    if (c.step_size <= 0.0) fail(LSP_EINVAL, "fit: step_size must be positive");
    FitEngine fe(*pair, targets, t, ld, dtype, as_stream(stream));
    std::vector<double> pv = pair->p->h_val, qv = pair->q->h_val;
    const int budget = std::min(c.max_steps, c.timeout_steps);
    const auto t_start = std::chrono::steady_clock::now();
    int trials = 0;
    const char* trace_env = std::getenv("LSP_FIT_TRACE");
    const bool trace = trace_env && trace_env[0] == '1';
    auto t_phase = t_start;
    double t_grad = 0.0, t_prep = 0.0, t_trial = 0.0, t_other = 0.0;
    *report = lsp_fit_report{};
    int ncurve = 0;
    auto push = [&](double l) {
      if (loss_curve && ncurve < max_curve) loss_curve[ncurve] = l;
      ++ncurve;
    };
    double loss = 0.0, rel = 0.0;
    fe.loss(pv, qv, c, &loss, &rel);
    if (!std::isfinite(loss)) fail(LSP_ENUMERIC, "fit: non-finite loss at initialization");
    push(loss);
    bool success = rel <= c.alpha, stalled = false;
    std::vector<double> gp, gq, tp(pv.size()), tq(qv.size());
    for (int step = 0; step < budget && !success; ++step) {
      auto tick = [&](double& acc) {  // LSP_FIT_TRACE phase timing (synchronises)
        if (!trace) return;
        LSP_CUDA(cudaStreamSynchronize(fe.st));
        const auto now = std::chrono::steady_clock::now();
        acc += std::chrono::duration<double>(now - t_phase).count();
        t_phase = now;
      };
      tick(t_other);
      fe.gradient(pv, qv, c, gp, gq);
      tick(t_grad);
      fe.prepare_line(pv, qv, gp, gq);
      tick(t_prep);
      double trial_step = c.step_size;
      bool accepted = false;
      for (int halving = 0; halving < 40; ++halving) {
        ++trials;
        for (size_t i = 0; i < pv.size(); ++i) tp[i] = pv[i] - trial_step * gp[i];
        for (size_t i = 0; i < qv.size(); ++i) tq[i] = qv[i] - trial_step * gq[i];
        double tl = 0.0, trel = 0.0;
        fe.loss(tp, tq, c, &tl, &trel, trial_step);
        tick(t_trial);
        if (std::isfinite(tl) && tl < loss) {
          pv.swap(tp);
          qv.swap(tq);
          loss = tl;
          rel = trel;
          accepted = true;
          break;
        }
        trial_step *= 0.5;
      }
      if (!accepted) {
        stalled = true;
        break;
      }
      ++report->steps;
      push(loss);
      success = rel <= c.alpha;
    }
    if (trace)
      std::fprintf(stderr,
                   "lsp_fit: %d x %d, T=%d: %d steps, %d loss evaluations, %.3f s (gradient %.3f, "
                   "line prep %.3f, trials %.3f, other %.3f)\n",
                   fe.m, fe.n, t, report->steps, trials + 1,
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count(), t_grad,
                   t_prep, t_trial, t_other);
    report->final_rel_bias = rel;
    report->success = success ? 1 : 0;
    report->stalled = stalled ? 1 : 0;
    report->timed_out = (!success && !stalled) ? 1 : 0;
    report->n_loss = ncurve;
    // write the fitted values back (positions are frozen)
    pair->p->h_val = pv;
    pair->q->h_val = qv;
    pair->p->upload_values();
    pair->q->upload_values();
  });
}

int lsp_projector_gram(lsp_projector_t a, lsp_projector_t b, double* out, lsp_stream_t stream) {
  return guard_fit([&] {
    require(a && b && out, "projector_gram: null argument");
    if (a->n_rows != b->n_rows) fail(LSP_EINVAL, "projector_gram: row spaces differ");
    cudaStream_t st = as_stream(stream);
    LSP_CUDA(cudaMemsetAsync(out, 0, static_cast<size_t>(a->d) * b->d * 8, st));
    LSP_DISPATCH_ACC(a->compute, Ta, {
      LSP_DISPATCH_ACC(b->compute, Tb, {
        k_gram<Ta, Tb><<<ceil_div(a->d, 128), 128, 0, st>>>(
            a->d, b->d, b->r, a->csc_ptr.as<int>(), a->csc_row.as<int>(), a->csc_val.as<Ta>(),
            b->pos.as<int>(), b->val.as<Tb>(), out);
      })
    })
    after_launch("gram");
  });
}

int lsp_reproject_state(lsp_adam_t st, lsp_pair_t old_pair, lsp_pair_t new_pair,
                        lsp_transfer_kind kind, lsp_stream_t stream) {
  return guard_fit([&] {
    require(st && old_pair && new_pair, "reproject_state: null argument");
    if (old_pair->d != new_pair->d) fail(LSP_EINVAL, "reproject_state: subspace widths differ");
    if (old_pair->m != new_pair->m || old_pair->n != new_pair->n)
      fail(LSP_EINVAL, "reproject_state: weight dims differ");
    if (st->rows != old_pair->d || st->cols != old_pair->d)
      fail(LSP_EINVAL, "reproject_state: state dims do not match pair");
    cudaStream_t s = as_stream(stream);
    const int d = old_pair->d;
    const size_t dd = static_cast<size_t>(d) * d;
    DevBuf tp, tq, tp2, tq2, mm, vv, tmp;
    for (DevBuf* b : {&tp, &tq, &tp2, &tq2, &mm, &vv, &tmp}) b->ensure(dd * 8);
    int rc = lsp_projector_gram(static_cast<lsp_projector_t>(new_pair->p),
                                static_cast<lsp_projector_t>(old_pair->p), tp.as<double>(), stream);
    if (rc) fail(rc, g_last_error);
    rc = lsp_projector_gram(static_cast<lsp_projector_t>(old_pair->q),
                            static_cast<lsp_projector_t>(new_pair->q), tq.as<double>(), stream);
    if (rc) fail(rc, g_last_error);
    // moments -> fp64 row layout
    auto to_row64 = [&](const DevBuf& src, DevBuf& dst) {
      launch_convert(dd, src.p, st->compute, tmp.p, LSP_F64, s);
      if (st->layout == LSP_LAYOUT_T)
        launch_transpose(d, d, tmp.p, d, dst.p, d, LSP_F64, s);
      else
        LSP_CUDA(cudaMemcpyAsync(dst.p, tmp.p, dd * 8, cudaMemcpyDeviceToDevice, s));
    };
    auto from_row64 = [&](DevBuf& src, DevBuf& dst) {
      const void* p = src.p;
      if (st->layout == LSP_LAYOUT_T) {
        launch_transpose(d, d, src.p, d, tmp.p, d, LSP_F64, s);
        p = tmp.p;
      }
      launch_convert(dd, p, LSP_F64, dst.p, st->compute, s);
    };
    to_row64(st->m, mm);
    to_row64(st->v, vv);
    if (kind == LSP_TRANSFER_ENTRYWISE) {
      LSP_CUDA(cudaMemcpyAsync(tp2.p, tp.p, dd * 8, cudaMemcpyDeviceToDevice, s));
      LSP_CUDA(cudaMemcpyAsync(tq2.p, tq.p, dd * 8, cudaMemcpyDeviceToDevice, s));
      k_square<<<egrid(dd), 256, 0, s>>>(dd, tp2.as<double>());
      after_launch("square");
      k_square<<<egrid(dd), 256, 0, s>>>(dd, tq2.as<double>());
      after_launch("square");
    } else {
      dgemm(d, d, d, tp.as<double>(), tp.as<double>(), tp2.as<double>(), s);
      dgemm(d, d, d, tq.as<double>(), tq.as<double>(), tq2.as<double>(), s);
    }
    DevBuf t1;
    t1.ensure(dd * 8);
    dgemm(d, d, d, tp.as<double>(), mm.as<double>(), t1.as<double>(), s);
    dgemm(d, d, d, t1.as<double>(), tq.as<double>(), mm.as<double>(), s);
    dgemm(d, d, d, tp2.as<double>(), vv.as<double>(), t1.as<double>(), s);
    dgemm(d, d, d, t1.as<double>(), tq2.as<double>(), vv.as<double>(), s);
    k_clamp0<<<egrid(dd), 256, 0, s>>>(dd, vv.as<double>());
    after_launch("clamp0");
    from_row64(mm, st->m);
    from_row64(vv, st->v);
    LSP_CUDA(cudaStreamSynchronize(s));
  });
}

}  // extern "C"
