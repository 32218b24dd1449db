// Per-layer schedule unit (north-star subsystem 5): the matrices of one
// transformer layer stepped together with ONE grouped launch per stage,
//   compress (stage 1 + stage 2)  ->  [caller all-reduces S]  ->  Adam  ->  apply,
// which is the body of the reference's per-layer loop (proj/src/trainer.cpp:186-198)
// for all linear layers of a block at once.  The S^T, delta^T and moment
// buffers of the layer are contiguous, so a data-parallel caller all-reduces
// the whole layer with one collective.
#include <cstdlib>
#include <cstring>
#include <vector>

#include "core.cuh"

struct lsp_pair_s : lspb::Pair {};

namespace lspb {
extern thread_local std::string g_last_error;
}

struct lsp_layer_s {
  int count = 0, d = 0, r = 0;
  lsp_dtype compute = LSP_F32;
  std::vector<lsp_pair_s*> pairs;
  lspb::Adam adam;            // (count*d) x d moments, per-matrix S^T blocks stacked
  lspb::DevBuf s_t, d_t, zt;  // S^T, delta^T (count*d*d each), Z^T workspace
  std::vector<size_t> zt_off;
  struct Bind {
    const void* g = nullptr;
    long long ldg = 0;
    lsp_dtype gdt = LSP_F32;
    void* w = nullptr;
    long long ldw = 0;
    lsp_dtype wdt = LSP_F32;
  };
  std::vector<Bind> binds;
  bool prepared = false;  // Y of the split apply built (lsp_layer_apply_prepare)

  size_t dd() const { return static_cast<size_t>(d) * d; }
  size_t vs() const { return lspb::dtype_size(compute); }
  char* s_block(int i) const { return s_t.as<char>() + i * dd() * vs(); }
  char* d_block(int i) const { return d_t.as<char>() + i * dd() * vs(); }
};

using namespace lspb;

namespace {

template <typename F>
int guard_layer(F&& f) {
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

void check_bound(const lsp_layer_s& L) {
  for (int i = 0; i < L.count; ++i) {
    require(L.binds[i].g && L.binds[i].w, "layer: matrix " + std::to_string(i) + " not bound");
    require(L.binds[i].gdt == L.binds[0].gdt && L.binds[i].wdt == L.binds[0].wdt,
            "layer: all matrices of a layer must share G and W dtypes");
  }
}

std::vector<S1Job> compress_jobs(lsp_layer_s& L) {
  check_bound(L);
  std::vector<S1Job> jobs;
  for (int i = 0; i < L.count; ++i)
    jobs.push_back(S1Job{L.pairs[i], L.binds[i].g, L.binds[i].ldg,
                         L.zt.as<char>() + L.zt_off[i], L.s_block(i)});
  return jobs;
}

void layer_compress(lsp_layer_s& L, cudaStream_t st) {
  compress_group_T(compress_jobs(L), L.binds[0].gdt, L.adam.flag.as<int>(), st);
}

void layer_adam(lsp_layer_s& L, bool check, cudaStream_t st) {
  int* flag = L.adam.flag.as<int>();
  const char* e = std::getenv("LSP_FUSE_ADAM");
  if (check && !(e && e[0] == '0')) {  // the check fused into Adam (ping-pong moments)
    launch_adam(L.adam, L.s_t.p, L.d_t.p, flag, st, true);
    return;
  }
  if (check) launch_check_finite(L.count * L.dd(), L.s_t.p, L.compute, flag, st);
  launch_adam(L.adam, L.s_t.p, L.d_t.p, flag, st);
}

// Stage 2 and Adam of a layer with no S exchange between them (single rank):
// one fused launch when eligible (k_stage2_f4<true>), else the unfused pair.
void layer_stage2_adam(lsp_layer_s& L, cudaStream_t st) {
  const std::vector<S1Job> jobs = compress_jobs(L);
  int* flag = L.adam.flag.as<int>();
  if (launch_stage2_adam_group(jobs, L.s_t.p, L.adam, L.d_t.p, flag, st)) return;
  launch_stage2_group(jobs, flag, st);
  launch_adam(L.adam, L.s_t.p, L.d_t.p, flag, st);
}

void layer_compress_adam(lsp_layer_s& L, cudaStream_t st) {
  launch_compress_stage1_group(compress_jobs(L), L.binds[0].gdt, st);
  layer_stage2_adam(L, st);
}

void layer_apply(lsp_layer_s& L, double lr, cudaStream_t st) {
  check_bound(L);
  int* flag = L.adam.flag.as<int>();
  std::vector<DecJob> jobs;
  for (int i = 0; i < L.count; ++i)
    jobs.push_back(DecJob{L.pairs[i], L.d_block(i), L.binds[i].w, L.binds[i].ldw, L.binds[i].w,
                          L.binds[i].ldw});
  launch_decompress_group(jobs, L.binds[0].wdt, -lr, 1.0, flag, nullptr, nullptr, st);
}

std::vector<DecJob> apply_jobs(lsp_layer_s& L) {
  std::vector<DecJob> jobs;
  for (int i = 0; i < L.count; ++i)
    jobs.push_back(DecJob{L.pairs[i], L.d_block(i), L.binds[i].w, L.binds[i].ldw, L.binds[i].w,
                          L.binds[i].ldw});
  return jobs;
}

// The fast-path matrices of the layer (Y precompute / row orientation).
std::vector<DecJob> fast_jobs(lsp_layer_s& L, std::vector<DecJob>* rest) {
  std::vector<DecJob> fast;
  const char* gen = std::getenv("LSP_DECOMPRESS_GENERIC");
  const bool generic = gen && gen[0] == '1';
  for (const DecJob& J : apply_jobs(L))
    (!generic && decompress_fast_eligible(J, L.binds[0].wdt, 1.0) ? fast : *rest).push_back(J);
  return fast;
}

void layer_apply_prepare(lsp_layer_s& L, cudaStream_t st) {
  check_bound(L);
  std::vector<DecJob> rest;
  const std::vector<DecJob> fast = fast_jobs(L, &rest);
  L.prepared = !fast.empty() && launch_decompress_group_y(fast, L.binds[0].wdt, -1.0, 1.0,
                                                          L.adam.flag.as<int>(), st, kPhaseBuild);
}

void layer_apply_finish(lsp_layer_s& L, double lr, cudaStream_t st) {
  check_bound(L);
  if (!L.prepared) {
    layer_apply(L, lr, st);
    return;
  }
  L.prepared = false;
  std::vector<DecJob> rest;
  const std::vector<DecJob> fast = fast_jobs(L, &rest);
  require(launch_decompress_group_y(fast, L.binds[0].wdt, -lr, 1.0, L.adam.flag.as<int>(), st,
                                    kPhaseApply),
          "layer_apply_finish: apply rejected after the Y build");
  if (!rest.empty())
    launch_decompress_group(rest, L.binds[0].wdt, -lr, 1.0, L.adam.flag.as<int>(), nullptr,
                            nullptr, st);
}

void layer_update(lsp_layer_s& L, double lr, bool check, cudaStream_t st) {
  check_bound(L);
  layer_adam(L, check, st);
  layer_apply(L, lr, st);
}

}  // namespace

namespace lspb {
void layer_s_view(lsp_layer_s* L, void** buf, long long* count, lsp_dtype* dt, int** flag) {
  *buf = L->s_t.p;
  *count = static_cast<long long>(L->count * L->dd());
  *dt = L->compute;
  *flag = L->adam.flag.as<int>();
}
}  // namespace lspb

extern "C" {

int lsp_layer_create(int count, const lsp_pair_t* pairs, double beta1, double beta2, double eps,
                     lsp_layer_t* out) {
  return guard_layer([&] {
    require(out && pairs, "layer_create: null argument");
    require(count >= 1 && count <= kMaxGroup, "layer_create: 1 <= count <= 16 matrices");
    if (beta1 <= 0.0 || beta1 >= 1.0 || beta2 <= 0.0 || beta2 >= 1.0)
      fail(LSP_EINVAL, "make_opt_state: betas must lie in (0, 1)");
    if (eps <= 0.0) fail(LSP_EINVAL, "make_opt_state: eps must be positive");
    auto L = std::make_unique<lsp_layer_s>();
    L->count = count;
    for (int i = 0; i < count; ++i) {
      require(pairs[i] != nullptr, "layer_create: null pair");
      L->pairs.push_back(pairs[i]);
    }
    const Pair& p0 = *pairs[0];
    L->d = p0.d;
    L->r = p0.p->r;
    L->compute = p0.compute;
    size_t zt_bytes = 0;
    for (int i = 0; i < count; ++i) {
      const Pair& p = *pairs[i];
      require(p.d == L->d && p.p->r == L->r && p.q->r == L->r && p.compute == L->compute,
              "layer_create: pairs must share d, r and compute dtype");
      L->zt_off.push_back(zt_bytes);
      zt_bytes += round_up(static_cast<size_t>(p.n) * p.ldz() * L->vs(), 256);
    }
    L->zt.ensure(std::max<size_t>(zt_bytes, 256));
    L->s_t.ensure(count * L->dd() * L->vs());
    L->d_t.ensure(count * L->dd() * L->vs());
    LSP_CUDA(cudaMemset(L->s_t.p, 0, count * L->dd() * L->vs()));
    Adam& a = L->adam;
    a.rows = count * L->d;
    a.cols = L->d;
    a.beta1 = beta1;
    a.beta2 = beta2;
    a.eps = eps;
    a.compute = L->compute;
    a.layout = LSP_LAYOUT_T;
    const size_t bytes = a.count() * L->vs();
    a.m.ensure(bytes);
    a.v.ensure(bytes);
    a.flag.ensure(sizeof(int));
    a.dstep.ensure(sizeof(long long));
    a.done.ensure(sizeof(unsigned));
    a.m2.ensure(bytes);  // ping-pong pair of the fused stage-2 + Adam (Adam::cur)
    a.v2.ensure(bytes);
    a.cur.ensure(sizeof(int));
    LSP_CUDA(cudaMemset(a.m.p, 0, bytes));
    LSP_CUDA(cudaMemset(a.v.p, 0, bytes));
    LSP_CUDA(cudaMemset(a.m2.p, 0, bytes));
    LSP_CUDA(cudaMemset(a.v2.p, 0, bytes));
    LSP_CUDA(cudaMemset(a.cur.p, 0, sizeof(int)));
    LSP_CUDA(cudaMemset(a.flag.p, 0, sizeof(int)));
    LSP_CUDA(cudaMemset(a.dstep.p, 0, sizeof(long long)));
    LSP_CUDA(cudaMemset(a.done.p, 0, sizeof(unsigned)));
    L->binds.resize(count);
    *out = L.release();
  });
}

int lsp_layer_destroy(lsp_layer_t layer) {
  return guard_layer([&] { delete layer; });
}

int lsp_layer_bind(lsp_layer_t L, int idx, const void* g, int64_t ldg, lsp_dtype g_dtype,
                   void* w, int64_t ldw, lsp_dtype w_dtype) {
  return guard_layer([&] {
    require(L != nullptr, "layer_bind: null layer");
    require(idx >= 0 && idx < L->count, "layer_bind: index out of range");
    const Pair& p = *L->pairs[idx];
    require(ldg >= p.n && ldw >= p.n, "layer_bind: leading dimension smaller than columns");
    dtype_size(g_dtype);
    dtype_size(w_dtype);
    L->binds[idx] = lsp_layer_s::Bind{g, ldg, g_dtype, w, ldw, w_dtype};
  });
}

int lsp_layer_s_buffer(lsp_layer_t L, void** s_t, int64_t* count) {
  return guard_layer([&] {
    require(L && s_t, "layer_s_buffer: null argument");
    *s_t = L->s_t.p;
    if (count) *count = static_cast<int64_t>(L->count * L->dd());
  });
}

int lsp_layer_compress(lsp_layer_t L, lsp_stream_t stream) {
  return guard_layer([&] {
    require(L != nullptr, "layer_compress: null layer");
    layer_compress(*L, as_stream(stream));
  });
}

int lsp_layer_compress_prepare(lsp_layer_t L, lsp_stream_t stream) {
  return guard_layer([&] {
    require(L != nullptr, "layer_compress_prepare: null layer");
    launch_compress_stage1_group(compress_jobs(*L), L->binds[0].gdt, as_stream(stream));
  });
}

int lsp_layer_compress_finish(lsp_layer_t L, lsp_stream_t stream) {
  return guard_layer([&] {
    require(L != nullptr, "layer_compress_finish: null layer");
    launch_stage2_group(compress_jobs(*L), L->adam.flag.as<int>(), as_stream(stream));
  });
}

int lsp_layer_compress_adam(lsp_layer_t L, lsp_stream_t stream) {
  return guard_layer([&] {
    require(L != nullptr, "layer_compress_adam: null layer");
    layer_compress_adam(*L, as_stream(stream));
  });
}

int lsp_layer_compress_finish_adam(lsp_layer_t L, lsp_stream_t stream) {
  return guard_layer([&] {
    require(L != nullptr, "layer_compress_finish_adam: null layer");
    layer_stage2_adam(*L, as_stream(stream));
  });
}

int lsp_layer_update(lsp_layer_t L, double lr, int check_finite, lsp_stream_t stream) {
  return guard_layer([&] {
    require(L != nullptr, "layer_update: null layer");
    layer_update(*L, lr, check_finite != 0, as_stream(stream));
  });
}

int lsp_layer_adam(lsp_layer_t L, int check_finite, lsp_stream_t stream) {
  return guard_layer([&] {
    require(L != nullptr, "layer_adam: null layer");
    layer_adam(*L, check_finite != 0, as_stream(stream));
  });
}

int lsp_layer_apply(lsp_layer_t L, double lr, lsp_stream_t stream) {
  return guard_layer([&] {
    require(L != nullptr, "layer_apply: null layer");
    layer_apply(*L, lr, as_stream(stream));
  });
}

int lsp_layer_apply_prepare(lsp_layer_t L, lsp_stream_t stream) {
  return guard_layer([&] {
    require(L != nullptr, "layer_apply_prepare: null layer");
    layer_apply_prepare(*L, as_stream(stream));
  });
}

int lsp_layer_apply_finish(lsp_layer_t L, double lr, lsp_stream_t stream) {
  return guard_layer([&] {
    require(L != nullptr, "layer_apply_finish: null layer");
    layer_apply_finish(*L, lr, as_stream(stream));
  });
}

int lsp_layer_step(lsp_layer_t L, double lr, lsp_stream_t stream) {
  return guard_layer([&] {
    require(L != nullptr, "layer_step: null layer");
    layer_compress_adam(*L, as_stream(stream));  // one rank: Adam in the stage-2 epilogue
    layer_apply(*L, lr, as_stream(stream));
  });
}

int lsp_layer_check(lsp_layer_t L, lsp_stream_t stream) {
  return guard_layer([&] {
    require(L != nullptr, "layer_check: null layer");
    int h = 0;
    cudaStream_t st = as_stream(stream);
    LSP_CUDA(cudaMemcpyAsync(&h, L->adam.flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    LSP_CUDA(cudaStreamSynchronize(st));
    if (h) {
      LSP_CUDA(cudaMemset(L->adam.flag.p, 0, sizeof(int)));
      fail(LSP_ENUMERIC, "adam_step: non-finite gradient");
    }
  });
}

int lsp_layer_adam_get(lsp_layer_t L, int idx, double* m, double* v, int64_t* step,
                       lsp_layout layout) {
  return guard_layer([&] {
    require(L != nullptr, "layer_adam_get: null layer");
    require(idx >= 0 && idx < L->count, "layer_adam_get: index out of range");
    LSP_CUDA(cudaDeviceSynchronize());
    const int d = L->d;
    auto fetch = [&](const DevBuf& b, double* out) {
      if (!out) return;
      LSP_DISPATCH_ACC(L->compute, T, {
        std::vector<T> tmp(L->dd());
        LSP_CUDA(cudaMemcpy(tmp.data(), b.as<char>() + idx * L->dd() * sizeof(T),
                            L->dd() * sizeof(T), cudaMemcpyDeviceToHost));
        for (int a = 0; a < d; ++a)
          for (int c = 0; c < d; ++c) {  // stored T: element (a, c) at c*d + a
            const double x = static_cast<double>(tmp[static_cast<size_t>(c) * d + a]);
            out[layout == LSP_LAYOUT_ROW ? static_cast<size_t>(a) * d + c
                                         : static_cast<size_t>(c) * d + a] = x;
          }
      })
    };
    int cur = 0;
    LSP_CUDA(cudaMemcpy(&cur, L->adam.cur.p, sizeof(int), cudaMemcpyDeviceToHost));
    fetch(cur ? L->adam.m2 : L->adam.m, m);
    fetch(cur ? L->adam.v2 : L->adam.v, v);
    if (step) {
      long long h = 0;
      LSP_CUDA(cudaMemcpy(&h, L->adam.dstep.p, sizeof(h), cudaMemcpyDeviceToHost));
      *step = h;
    }
  });
}

}  // extern "C"
