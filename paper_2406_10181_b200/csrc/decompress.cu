// Fused decompress-and-apply: out = beta*in + alpha * P delta Q^T
// (reference: left_mul/rightT_mul proj/src/projector.cpp:105-117,148-161,
//  decompress :170-175, apply proj/src/trainer.cpp:190).
//
// One CTA owns a band of BN columns of W (and a range of rows):
//  phase 1  Y_band[a][jj] = sum_l q(j,l) * delta^T[pos_q(j,l)][a]  for all a,
//           built in shared memory from coalesced rows of the L2-resident
//           delta^T (d x (BN+1) floats, padded against bank conflicts);
//  phase 2  every W row i of the range: k conflict-free row gathers
//           Y_band[pos_p(i,l)][:] and ONE read-modify-write of W[i][band].
// W is read and written exactly once; delta never leaves L2.
#include <algorithm>
#include <cmath>
#include <memory>
#include <mutex>
#include <vector>

#include "core.cuh"

namespace lspb {

namespace {

constexpr int kDecThreads = 512;
constexpr int kDecUnroll = 4;

template <typename Tw, typename Tacc, int BN>
__global__ void __launch_bounds__(kDecThreads)
    k_decompress_band(int m, int n, int d, int r, const int* __restrict__ ppos,
                      const Tacc* __restrict__ pval, const int* __restrict__ qpos,
                      const Tacc* __restrict__ qval, const Tacc* __restrict__ dT, int ldd,
                      const Tw* in, long long ldi, Tw* out, long long ldo, Tacc alpha, Tacc beta,
                      int nbands, int rows_per_unit, const int* __restrict__ skip,
                      double* __restrict__ partials) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Tacc* Y = reinterpret_cast<Tacc*>(smem_raw);  // [d][BN+1]
  constexpr int LDY = BN + 1;
  if (skip && *skip) return;
  const int band = blockIdx.x % nbands, rs = blockIdx.x / nbands;
  const int j0 = band * BN;
  const int i_begin = rs * rows_per_unit;
  const int i_end = min(m, i_begin + rows_per_unit);
  const int tid = threadIdx.x;

  // ---- phase 1: Y_band ----------------------------------------------------
  for (int jj = 0; jj < BN; ++jj) {
    const int j = j0 + jj;
    if (j >= n) {
      for (int a = tid; a < d; a += kDecThreads) Y[a * LDY + jj] = Tacc(0);
      continue;
    }
    for (int a = tid; a < d; a += kDecThreads) {
      Tacc y = Tacc(0);
      for (int l = 0; l < r; ++l) {
        const int b = qpos[static_cast<long long>(j) * r + l];
        y = fma(qval[static_cast<long long>(j) * r + l], dT[static_cast<long long>(b) * ldd + a], y);
      }
      Y[a * LDY + jj] = y;
    }
  }
  __syncthreads();

  // ---- phase 2: stream W rows ----------------------------------------------
  constexpr int RPW = 32 / BN;  // rows per warp per iteration
  const int lane = tid & 31, warp = tid >> 5;
  const int jj = lane % BN, rsub = lane / BN;
  const int j = j0 + jj;
  const bool col_ok = j < n;
  const int stride = (kDecThreads / 32) * RPW;
  double ss = 0.0;
  const bool use_in = in != nullptr && beta != Tacc(0);
  for (int i0 = i_begin + warp * RPW + rsub; i0 < i_end; i0 += stride * kDecUnroll) {
    Tw wv[kDecUnroll];
#pragma unroll
    for (int u = 0; u < kDecUnroll; ++u) {
      const int i = i0 + u * stride;
      if (use_in && col_ok && i < i_end) wv[u] = in[static_cast<long long>(i) * ldi + j];
    }
#pragma unroll
    for (int u = 0; u < kDecUnroll; ++u) {
      const int i = i0 + u * stride;
      if (i >= i_end) break;
      Tacc acc = Tacc(0);
      for (int l = 0; l < r; ++l) {
        const long long e = static_cast<long long>(i) * r + l;
        acc = fma(pval[e], Y[ppos[e] * LDY + jj], acc);
      }
      if (!col_ok) continue;
      Tacc res = alpha * acc;
      if (use_in) res = fma(beta, cvt<Tacc>(wv[u]), res);
      if (out) out[static_cast<long long>(i) * ldo + j] = cvt<Tw>(res);
      if (partials) {
        const double rv = static_cast<double>(cvt<Tacc>(cvt<Tw>(res)));
        ss += out ? rv * rv : static_cast<double>(res) * static_cast<double>(res);
      }
    }
  }
  if (partials) {
    __shared__ double red[kDecThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kDecThreads / 32; ++w) t += red[w];
      partials[blockIdx.x] = t;
    }
  }
}

template <typename Tw, typename Tacc, int BN>
void decompress_impl(const Pair& pr, const Tacc* dT, const Tw* in, long long ldi, Tw* out,
                     long long ldo, double alpha, double beta, const int* skip,
                     DevBuf* partials, int* nparts, cudaStream_t st) {
  const int smem = pr.d * (BN + 1) * static_cast<int>(sizeof(Tacc));
  auto kern = k_decompress_band<Tw, Tacc, BN>;
  LSP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int nbands = ceil_div(pr.n, BN);
  const int per_sm = std::max(1, std::min(4, (220 * 1024) / std::max(smem, 1)));
  const int target = 2 * per_sm * num_sms();
  const int max_split = std::max(1, ceil_div(pr.m, 64));
  const int rsplit = std::max(1, std::min(max_split, ceil_div(target, nbands)));
  const int rows_per_unit = ceil_div(pr.m, rsplit);
  const int units = nbands * ceil_div(pr.m, rows_per_unit);
  if (nparts) *nparts = units;
  if (partials) partials->ensure(static_cast<size_t>(units) * sizeof(double));
  double* parts = partials ? partials->as<double>() : nullptr;
  kern<<<units, kDecThreads, smem, st>>>(pr.m, pr.n, pr.d, pr.p->r, pr.p->pos.as<int>(),
                                         pr.p->val.as<Tacc>(), pr.q->pos.as<int>(),
                                         pr.q->val.as<Tacc>(), dT, pr.d, in, ldi, out, ldo,
                                         static_cast<Tacc>(alpha), static_cast<Tacc>(beta),
                                         nbands, rows_per_unit, skip, parts);
  after_launch("decompress_band");
}

}  // namespace

void launch_decompress(const Pair& pr, const void* delta_t, const void* in, long long ldi,
                       void* out, long long ldo, lsp_dtype dt, double alpha, double beta,
                       const int* skip_flag, DevBuf* partials, int* nparts, cudaStream_t st) {
  LSP_DISPATCH_ACC(pr.compute, Tacc, {
    LSP_DISPATCH_STORAGE(dt, Tw, {
      const size_t budget = 200 * 1024;
      const size_t row = static_cast<size_t>(pr.d) * sizeof(Tacc);
      const Tacc* dT = static_cast<const Tacc*>(delta_t);
      const Tw* pin = static_cast<const Tw*>(in);
      Tw* pout = static_cast<Tw*>(out);
      if (row * 33 <= budget)
        decompress_impl<Tw, Tacc, 32>(pr, dT, pin, ldi, pout, ldo, alpha, beta, skip_flag, partials, nparts, st);
      else if (row * 17 <= budget)
        decompress_impl<Tw, Tacc, 16>(pr, dT, pin, ldi, pout, ldo, alpha, beta, skip_flag, partials, nparts, st);
      else if (row * 9 <= budget)
        decompress_impl<Tw, Tacc, 8>(pr, dT, pin, ldi, pout, ldo, alpha, beta, skip_flag, partials, nparts, st);
      else if (row * 5 <= budget)
        decompress_impl<Tw, Tacc, 4>(pr, dT, pin, ldi, pout, ldo, alpha, beta, skip_flag, partials, nparts, st);
      else
        fail(LSP_EINVAL, "decompress: subspace width too large for the band kernel");
    })
  })
}

// ---------------------------------------------------------------------------
// Subspace Adam (proj/src/subspace_opt.cpp:35-57).  Elementwise, no
// contraction (explicit _rn ops) so the fp64 path rounds exactly like the
// reference: m = b1*m + (1-b1)*g; v = b2*v + (1-b2)*g*g;
// delta = (m / c1) / (sqrt(v / c2) + eps).
// ---------------------------------------------------------------------------
namespace {

__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float div_(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float sqrt_(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ double sqrt_(double a) { return __dsqrt_rn(a); }

// Advances the device step counter (unless a non-finite gradient is latched)
// and publishes (1 - b1^t, 1 - b2^t).  The corrections come from a host table
// computed with std::pow, exactly as the reference does (subspace_opt.cpp:44-45).
__global__ void k_adam_prep(const int* __restrict__ skip, long long* __restrict__ step,
                            const double2* __restrict__ table, long long cap, double b1,
                            double b2, double* __restrict__ corr) {
  if (skip && *skip) return;
  const long long t = *step + 1;
  *step = t;
  double2 c;
  if (t <= cap) {
    c = table[t - 1];
  } else {
    c.x = 1.0 - pow(b1, static_cast<double>(t));
    c.y = 1.0 - pow(b2, static_cast<double>(t));
  }
  corr[0] = c.x;
  corr[1] = c.y;
}

template <typename T>
__global__ void k_adam(long long cnt, const T* __restrict__ g, T* __restrict__ m,
                       T* __restrict__ v, T* __restrict__ delta, T b1, T omb1, T b2, T omb2,
                       const double* __restrict__ corr, T eps, const int* __restrict__ skip) {
  if (skip && *skip) return;
  const T c1 = static_cast<T>(corr[0]), c2 = static_cast<T>(corr[1]);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt;
       i += (long long)gridDim.x * blockDim.x) {
    const T gi = g[i];
    const T mi = add_(mul_(b1, m[i]), mul_(omb1, gi));
    const T vi = add_(mul_(b2, v[i]), mul_(mul_(omb2, gi), gi));
    m[i] = mi;
    v[i] = vi;
    delta[i] = div_(div_(mi, c1), add_(sqrt_(div_(vi, c2)), eps));
  }
}

__device__ __forceinline__ bool finite_val(float v) { return isfinite(v); }
__device__ __forceinline__ bool finite_val(double v) { return isfinite(v); }
__device__ __forceinline__ bool finite_val(bf16 v) { return isfinite(__bfloat162float(v)); }

template <typename T>
__global__ void k_check_finite(long long cnt, const T* __restrict__ x, int* flag) {
  bool bad = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt;
       i += (long long)gridDim.x * blockDim.x)
    bad |= !finite_val(x[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

template <typename Ts, typename Td>
__global__ void k_convert(long long cnt, const Ts* __restrict__ s, Td* __restrict__ d) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt;
       i += (long long)gridDim.x * blockDim.x)
    d[i] = cvt<Td>(cvt<double>(s[i]));
}

template <typename Ts, typename Td>
__global__ void k_convert2d(int rows, int cols, const Ts* __restrict__ s, long long lds,
                            Td* __restrict__ d, long long ldd) {
  const long long cnt = static_cast<long long>(rows) * cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / cols, c = i % cols;
    d[r * ldd + c] = cvt<Td>(cvt<double>(s[r * lds + c]));
  }
}

__global__ void k_reduce_partials(const double* __restrict__ p, int n, double* out) {
  // single block, fixed order -> deterministic
  __shared__ double red[256];
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) t += p[i];
  red[threadIdx.x] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < 256; ++i) s += red[i];
    *out = s;
  }
}

template <typename T>
__global__ void k_gather_values(long long cnt, const int* __restrict__ perm,
                                const T* __restrict__ src, T* __restrict__ dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[perm[i]];
}
template <typename E, typename T>
__global__ void k_gather_entry_values(long long cnt, const int* __restrict__ perm,
                                      const T* __restrict__ src, E* __restrict__ dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt;
       i += (long long)gridDim.x * blockDim.x)
    dst[i].val = src[perm[i]];
}

int grid_for(long long cnt) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>((cnt + 255) / 256, 16LL * num_sms())));
}

}  // namespace

// Bias-correction tables shared by every state with the same betas.
static const double2* correction_table(double b1, double b2, long long* cap) {
  struct Entry {
    double b1, b2;
    DevBuf buf;
  };
  static std::mutex mu;
  static std::vector<std::unique_ptr<Entry>> cache;
  constexpr long long kCap = 1LL << 17;
  std::lock_guard<std::mutex> lock(mu);
  *cap = kCap;
  for (auto& e : cache)
    if (e->b1 == b1 && e->b2 == b2) return e->buf.as<double2>();
  auto e = std::make_unique<Entry>();
  e->b1 = b1;
  e->b2 = b2;
  std::vector<double2> h(kCap);
  for (long long t = 1; t <= kCap; ++t)
    h[t - 1] = make_double2(1.0 - std::pow(b1, static_cast<double>(t)),
                            1.0 - std::pow(b2, static_cast<double>(t)));
  e->buf.ensure(kCap * sizeof(double2));
  LSP_CUDA(cudaMemcpy(e->buf.p, h.data(), kCap * sizeof(double2), cudaMemcpyHostToDevice));
  cache.push_back(std::move(e));
  return cache.back()->buf.as<double2>();
}

void launch_adam(Adam& a, const void* grad, void* delta, const int* skip_flag, cudaStream_t st) {
  long long cap = 0;
  const double2* table = correction_table(a.beta1, a.beta2, &cap);
  k_adam_prep<<<1, 1, 0, st>>>(skip_flag, a.dstep.as<long long>(), table, cap, a.beta1, a.beta2,
                               a.corr.as<double>());
  after_launch("adam_prep");
  const long long cnt = static_cast<long long>(a.count());
  LSP_DISPATCH_ACC(a.compute, T, {
    k_adam<T><<<grid_for(cnt), 256, 0, st>>>(cnt, static_cast<const T*>(grad), a.m.as<T>(),
                                             a.v.as<T>(), static_cast<T*>(delta), (T)a.beta1,
                                             (T)(1.0 - a.beta1), (T)a.beta2, (T)(1.0 - a.beta2),
                                             a.corr.as<double>(), (T)a.eps, skip_flag);
  })
  after_launch("adam");
}

void launch_check_finite(size_t cnt, const void* x, lsp_dtype dt, int* flag, cudaStream_t st) {
  LSP_DISPATCH_STORAGE(dt, T, {
    k_check_finite<T><<<grid_for(cnt), 256, 0, st>>>(static_cast<long long>(cnt),
                                                     static_cast<const T*>(x), flag);
  })
  after_launch("check_finite");
}

void launch_convert(size_t cnt, const void* src, lsp_dtype sdt, void* dst, lsp_dtype ddt,
                    cudaStream_t st) {
  LSP_DISPATCH_STORAGE(sdt, Ts, {
    LSP_DISPATCH_STORAGE(ddt, Td, {
      k_convert<Ts, Td><<<grid_for(cnt), 256, 0, st>>>(static_cast<long long>(cnt),
                                                       static_cast<const Ts*>(src),
                                                       static_cast<Td*>(dst));
    })
  })
  after_launch("convert");
}

void launch_convert2d(int rows, int cols, const void* src, long long lds, lsp_dtype sdt,
                      void* dst, long long ldd, lsp_dtype ddt, cudaStream_t st) {
  const long long cnt = static_cast<long long>(rows) * cols;
  if (cnt <= 0) return;
  LSP_DISPATCH_STORAGE(sdt, Ts, {
    LSP_DISPATCH_STORAGE(ddt, Td, {
      k_convert2d<Ts, Td><<<grid_for(cnt), 256, 0, st>>>(rows, cols, static_cast<const Ts*>(src),
                                                         lds, static_cast<Td*>(dst), ldd);
    })
  })
  after_launch("convert2d");
}

double reduce_partials_sync(const double* partials, int n, cudaStream_t st) {
  static thread_local DevBuf out;
  out.ensure(sizeof(double));
  k_reduce_partials<<<1, 256, 0, st>>>(partials, n, out.as<double>());
  after_launch("reduce_partials");
  double h = 0.0;
  LSP_CUDA(cudaMemcpyAsync(&h, out.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  LSP_CUDA(cudaStreamSynchronize(st));
  return h;
}

void launch_refresh_values(const Projector& p, cudaStream_t st) {
  const long long nnz = static_cast<long long>(p.nnz());
  LSP_DISPATCH_ACC(p.compute, T, {
    k_gather_values<T><<<grid_for(nnz), 256, 0, st>>>(nnz, p.csc_perm.as<int>(), p.val.as<T>(),
                                                      p.csc_val.as<T>());
    after_launch("refresh_csc");
    for (const auto& ct : p.chunks) {
      using E = typename EntryOf<T>::type;
      k_gather_entry_values<E, T><<<grid_for(nnz), 256, 0, st>>>(nnz, ct->perm.as<int>(),
                                                                 p.val.as<T>(), ct->ent.as<E>());
      after_launch("refresh_chunks");
    }
  })
}

// delta given in `layout` -> pointer to delta^T (d x d, ld d) on the device.
const void* delta_as_T(Pair& pr, const void* s, lsp_layout layout, cudaStream_t st) {
  if (layout == LSP_LAYOUT_T) return s;
  pr.d_t.ensure(static_cast<size_t>(pr.d) * pr.d * dtype_size(pr.compute));
  launch_transpose(pr.d, pr.d, s, pr.d, pr.d_t.p, pr.d, pr.compute, st);
  return pr.d_t.p;
}

}  // namespace lspb
