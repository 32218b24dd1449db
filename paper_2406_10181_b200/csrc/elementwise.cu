// Elementwise / bookkeeping kernels: subspace Adam, non-finite checks, dtype
// conversion, deterministic reductions and projector value refresh.
#include <algorithm>
#include <cmath>
#include <memory>
#include <mutex>
#include <vector>

#include "adam_math.cuh"
#include "core.cuh"

namespace lspb {

// ---------------------------------------------------------------------------
// Subspace Adam (proj/src/subspace_opt.cpp:35-57): the element update is
// adam_elem (adam_math.cuh), no contraction.
// ---------------------------------------------------------------------------
namespace {

// Subspace Adam.  Every block reads the step counter, computes the bias
// corrections (1 - b1^t, 1 - b2^t) from a host table filled with std::pow,
// exactly like the reference (subspace_opt.cpp:44-45), and the last block to
// finish advances the counter -- so a captured CUDA graph replays correctly.
//
// kChecked (layer state with ping-pong moments): the finiteness check of the
// gradient is fused in -- every block reads the current moment pair, writes
// the other one, and latches the flag on a non-finite gradient element; the
// last block flips the pair and advances the step only when the flag is clear
// (k_check_finite + k_adam in one pass, the same outcome).
template <typename T, bool kChecked>
__global__ void k_adam(long long cnt, const T* __restrict__ g, T* m, T* v, T* __restrict__ delta,
                       T b1, T omb1, T b2, T omb2, const double2* __restrict__ table,
                       long long cap, double db1, double db2, T eps,
                       long long* __restrict__ step, unsigned* __restrict__ done, int* skip,
                       T* m1, T* v1, int* __restrict__ cur) {
  if (!kChecked && skip && *skip) return;  // uniform over the grid: nobody touches the counter
  const int which = cur ? *cur : 0;
  // ping-pong moments (layer state): the current pair is (m1, v1) when *cur
  T* mi = which ? m1 : m;
  T* vi = which ? v1 : v;
  T* mo = kChecked ? (which ? m : m1) : mi;  // unchecked: in place
  T* vo = kChecked ? (which ? v : v1) : vi;
  const long long t = *step + 1;
  double2 c;
  if (t <= cap) {
    c = table[t - 1];
  } else {
    c.x = 1.0 - pow(db1, static_cast<double>(t));
    c.y = 1.0 - pow(db2, static_cast<double>(t));
  }
  const T c1 = static_cast<T>(c.x), c2 = static_cast<T>(c.y);
  bool bad = false;
  auto one = [&](T gi, T& mv, T& vv) {  // returns delta; updates the moments in place
    if constexpr (kChecked) bad |= !isfinite(gi);
    return adam_elem(gi, mv, vv, b1, omb1, b2, omb2, c1, c2, eps);
  };
  long long i0 = 0;
  if constexpr (sizeof(T) == 4) {
    // 16-byte vector path (all of a layer's blocks are 16-byte aligned, cnt % 4 == 0)
    if ((cnt & 3) == 0 && ((reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(mi) |
                            reinterpret_cast<uintptr_t>(vi) | reinterpret_cast<uintptr_t>(mo) |
                            reinterpret_cast<uintptr_t>(vo) | reinterpret_cast<uintptr_t>(delta)) & 15) == 0) {
      const long long n4 = cnt >> 2;
      for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
           i += (long long)gridDim.x * blockDim.x) {
        const float4 gv = reinterpret_cast<const float4*>(g)[i];
        float4 mv = reinterpret_cast<const float4*>(mi)[i];
        float4 vv = reinterpret_cast<const float4*>(vi)[i];
        float4 dv;
        dv.x = one(gv.x, mv.x, vv.x);
        dv.y = one(gv.y, mv.y, vv.y);
        dv.z = one(gv.z, mv.z, vv.z);
        dv.w = one(gv.w, mv.w, vv.w);
        reinterpret_cast<float4*>(mo)[i] = mv;
        reinterpret_cast<float4*>(vo)[i] = vv;
        reinterpret_cast<float4*>(delta)[i] = dv;
      }
      i0 = cnt;
    }
  }
  for (long long i = i0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt;
       i += (long long)gridDim.x * blockDim.x) {
    T mv = mi[i], vv = vi[i];
    delta[i] = one(g[i], mv, vv);
    mo[i] = mv;
    vo[i] = vv;
  }
  if constexpr (kChecked) {
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(skip, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();  // (checked: this block's latch and moments before its done count)
    if (atomicAdd(done, 1u) == gridDim.x - 1) {  // every block has read *step
      if (!kChecked || atomicOr(skip, 0) == 0) {
        if (kChecked) *cur = 1 - which;
        *step = t;
      }
      *done = 0u;
      __threadfence();
    }
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
    if (perm[i] >= 0) dst[i].val = src[perm[i]];
}

int grid_for(long long cnt) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>((cnt + 255) / 256, 16LL * num_sms())));
}

}  // namespace

// Bias-correction tables shared by every state with the same betas.
const double2* correction_table(double b1, double b2, long long* cap) {
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

void launch_adam(Adam& a, const void* grad, void* delta, const int* skip_flag, cudaStream_t st,
                 bool checked) {
  long long cap = 0;
  const double2* table = correction_table(a.beta1, a.beta2, &cap);
  const long long cnt = static_cast<long long>(a.count());
  int* flag = const_cast<int*>(skip_flag);
  if (checked) require(flag && a.cur.p, "adam: the checked update needs a flag and ping-pong moments");
  LSP_DISPATCH_ACC(a.compute, T, {
    auto kern = checked ? k_adam<T, true> : k_adam<T, false>;
    kern<<<grid_for(cnt), 256, 0, st>>>(
        cnt, static_cast<const T*>(grad), a.m.as<T>(), a.v.as<T>(), static_cast<T*>(delta),
        (T)a.beta1, (T)(1.0 - a.beta1), (T)a.beta2, (T)(1.0 - a.beta2), table, cap, a.beta1,
        a.beta2, (T)a.eps, a.dstep.as<long long>(), a.done.as<unsigned>(), flag,
        a.m2.as<T>(), a.v2.as<T>(), a.cur.as<int>());
  })
  after_launch(checked ? "adam_checked" : "adam");
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
      k_gather_entry_values<E, T><<<grid_for(ct->count), 256, 0, st>>>(ct->count, ct->perm.as<int>(),
                                                                 p.val.as<T>(), ct->ent.as<E>());
      after_launch("refresh_chunks");
    }
    if (p.csc_pad && p.csc_pad->count) {
      using E = typename EntryOf<T>::type;
      k_gather_entry_values<E, T><<<grid_for(p.csc_pad->count), 256, 0, st>>>(
          p.csc_pad->count, p.csc_pad->perm.as<int>(), p.val.as<T>(), p.csc_pad->ent.as<E>());
      after_launch("refresh_csc_padded");
    }
    if constexpr (sizeof(T) == 4) {
      if (p.csc_ent.p && nnz) {
        k_gather_entry_values<EntryF, T><<<grid_for(nnz), 256, 0, st>>>(
            nnz, p.csc_perm.as<int>(), p.val.as<T>(), p.csc_ent.as<EntryF>());
        after_launch("refresh_csc_entries");
      }
      for (const auto& t : p.slot_tables) {
        k_gather_entry_values<EntryF, T><<<grid_for(t->nslots), 256, 0, st>>>(
            t->nslots, t->perm.as<int>(), p.val.as<T>(), t->slots.as<EntryF>());
        after_launch("refresh_slots");
        if (t->novf) {
          k_gather_entry_values<EntryF, T><<<grid_for(t->novf), 256, 0, st>>>(
              t->novf, t->ovf_perm.as<int>(), p.val.as<T>(), t->ovf.as<EntryF>());
          after_launch("refresh_overflow");
        }
      }
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
