// extern "C" boundary (include/lsp_b200.h): argument validation with the
// reference's error semantics, handle management, and orchestration of the
// device kernels.  No compute happens on the host except index generation.
#include <algorithm>
#include <cmath>
#include <limits>
#include <cstring>
#include <string>

#include "core.cuh"
#include "host_projector.h"

struct lsp_projector_s : lspb::Projector {};
struct lsp_pair_s : lspb::Pair {};
struct lsp_adam_s : lspb::Adam {};

namespace lspb {

std::atomic<uint64_t> g_launches{0};
thread_local std::string g_last_error;

size_t dtype_size(lsp_dtype t) {
  switch (t) {
    case LSP_F64: return 8;
    case LSP_F32: return 4;
    case LSP_BF16: return 2;
  }
  fail(LSP_EINVAL, "unknown dtype");
}

bool trace_launches() {
  static const bool on = [] {
    const char* e = std::getenv("LSP_TRACE");
    return e && e[0] == '1';
  }();
  return on;
}

int num_sms() {
  static int sms = [] {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
    return v > 0 ? v : 148;
  }();
  return sms;
}

std::atomic<int> g_budget[2] = {{0}, {0}};

// lsp_schedule_set_partition: persistent grids sized for the partition while a
// partitioned step is enqueued (host side, one thread)
void budget_exchange(int compress_sms, int update_sms, int* old_compress, int* old_update) {
  const int c = g_budget[0].exchange(compress_sms), u = g_budget[1].exchange(update_sms);
  if (old_compress) *old_compress = c;
  if (old_update) *old_update = u;
}

int sm_budget(int phase) {
  const int b = g_budget[phase].load(std::memory_order_relaxed);
  return b > 0 ? std::min(b, num_sms()) : num_sms();
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return LSP_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_last_error = "host allocation failed";
    return LSP_ENOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return LSP_EINVAL;
  }
}

// ---- Projector ---------------------------------------------------------------
static void upload(DevBuf& b, const void* src, size_t bytes) {
  b.ensure(bytes + 16);  // 16 bytes of slack: 16-byte vector/bulk reads may round up past the end
  if (bytes) LSP_CUDA(cudaMemcpy(b.p, src, bytes, cudaMemcpyHostToDevice));
  // zero the slack: a vector read that rounds past the end sees position 0 / value 0
  LSP_CUDA(cudaMemset(static_cast<char*>(b.p) + bytes, 0, b.bytes - bytes));
}

template <typename T>
static std::vector<T> cast_values(const std::vector<double>& v) {
  return std::vector<T>(v.begin(), v.end());
}

void Projector::upload_values() {
  LSP_DISPATCH_ACC(compute, T, {
    auto cv = cast_values<T>(h_val);
    upload(val, cv.data(), cv.size() * sizeof(T));
  })
  launch_refresh_values(*this, nullptr);
  LSP_CUDA(cudaDeviceSynchronize());
}

void Projector::refresh_values(cudaStream_t st) { launch_refresh_values(*this, st); }

const ChunkTable& Projector::chunk_table(int bm, int esize) {
  for (auto& c : chunks)
    if (c->bm == bm && c->esize == esize) return *c;
  auto ct = std::make_unique<ChunkTable>();
  ct->bm = bm;
  ct->esize = esize;
  ct->nchunks = ceil_div(n_rows, bm);
  std::vector<int32_t> split, rows, perm;
  build_chunks(n_rows, d, bm, h_csc_ptr, h_csc_rows, h_csc_perm, split, rows, perm);
  upload(ct->split, split.data(), split.size() * sizeof(int32_t));
  upload(ct->perm, perm.data(), perm.size() * sizeof(int32_t));
  ct->count = static_cast<long long>(perm.size());
  LSP_DISPATCH_ACC(compute, T, {
    using E = typename EntryOf<T>::type;
    std::vector<E> ent(rows.size());
    for (size_t t = 0; t < rows.size(); ++t) {
      ent[t] = E{};
      ent[t].off = rows[t] * 32 * esize;
      ent[t].val = perm[t] >= 0 ? static_cast<T>(h_val[perm[t]]) : T(0);
    }
    upload(ct->ent, ent.data(), ent.size() * sizeof(E));
  })
  chunks.push_back(std::move(ct));
  return *chunks.back();
}

const SlotTable& Projector::slot_table(int bm, int row_bytes, int K, int bpw) {
  for (auto& t : slot_tables)
    if (t->bm == bm && t->row_bytes == row_bytes && t->K == K && t->bpw == bpw) return *t;
  require(K >= 2 && K % 2 == 0 && bpw >= 1 && 32 % bpw == 0, "slot table: bad K / bins per warp");
  auto t = std::make_unique<SlotTable>();
  t->bm = bm, t->row_bytes = row_bytes, t->K = K, t->bpw = bpw;
  t->nchunks = ceil_div(n_rows, bm);
  t->dpad = static_cast<int>(round_up(d, 32));
  SlotHost h;
  build_slots(n_rows, d, bm, K, bpw, h_csc_ptr, h_csc_rows, h_csc_perm, h);
  t->nslots = static_cast<long long>(h.slot_row.size());
  t->novf = static_cast<long long>(h.ovf_row.size());
  const int zero = slot_zero_off(bm, row_bytes);
  require(static_cast<long long>(zero) < (1LL << 27), "slot table: tile too large");
  std::vector<EntryF> sl(h.slot_row.size()), ov(h.ovf_row.size());
  for (size_t i = 0; i < sl.size(); ++i) {
    const int row = h.slot_row[i];
    sl[i].off = row < 0 ? zero : row * row_bytes;
    sl[i].val = row < 0 ? 0.0f : static_cast<float>(h_val[h.slot_perm[i]]);
  }
  for (size_t i = 0; i < ov.size(); ++i) {
    ov[i].off = (h.ovf_row[i] * row_bytes) | (h.ovf_bin[i] << 27);
    ov[i].val = static_cast<float>(h_val[h.ovf_perm[i]]);
  }
  upload(t->slots, sl.data(), sl.size() * sizeof(EntryF));
  upload(t->perm, h.slot_perm.data(), h.slot_perm.size() * sizeof(int32_t));
  upload(t->ovf_split, h.ovf_split.data(), h.ovf_split.size() * sizeof(int32_t));
  upload(t->ovf, ov.data(), ov.size() * sizeof(EntryF));
  upload(t->ovf_perm, h.ovf_perm.data(), h.ovf_perm.size() * sizeof(int32_t));
  slot_tables.push_back(std::move(t));
  return *slot_tables.back();
}

long long Projector::overflow(int K, int bm) {
  for (auto& e : ovf_counts)
    if (e.first == std::make_pair(K, bm)) return e.second;
  const long long v = count_overflow(n_rows, d, bm, K, h_csc_ptr, h_csc_rows);
  ovf_counts.emplace_back(std::make_pair(K, bm), v);
  return v;
}

const int* Projector::scaled_pos(int scale) {
  for (auto& e : scaled)
    if (e.first == scale) return e.second->as<int>();
  std::vector<int32_t> sp(h_pos.size());
  for (size_t i = 0; i < sp.size(); ++i) sp[i] = h_pos[i] * scale;
  auto buf = std::make_unique<DevBuf>();
  upload(*buf, sp.data(), sp.size() * sizeof(int32_t));
  scaled.emplace_back(scale, std::move(buf));
  return scaled.back().second->as<int>();
}

const EntryF* Projector::csc_entries() {
  require(compute == LSP_F32, "csc_entries: fp32 projectors only");
  if (!csc_ent.p) {
    std::vector<EntryF> e(nnz() + 2);  // +16 B: 16-byte bulk copies may read past the end
    for (size_t k = 0; k < nnz(); ++k) {
      e[k].off = h_csc_rows[k];
      e[k].val = 0.0f;
    }
    upload(csc_ent, e.data(), e.size() * sizeof(EntryF));
    launch_refresh_values(*this, nullptr);  // values from the device CSR array
    LSP_CUDA(cudaDeviceSynchronize());
  }
  return csc_ent.as<EntryF>();
}

const Projector::PadTable& Projector::csc_padded() {
  if (!csc_pad) {
    auto t = std::make_unique<PadTable>();
    t->h_ptr.assign(d + 1, 0);
    std::vector<int32_t> rows, perm;
    for (int b = 0; b < d; ++b) {
      const int k0 = h_csc_ptr[b], k1 = h_csc_ptr[b + 1];
      for (int k = k0; k < k1; ++k) {
        rows.push_back(h_csc_rows[k]);
        perm.push_back(h_csc_perm[k]);
      }
      const int cnt = k1 - k0, padded = (cnt + kPadU - 1) / kPadU * kPadU;
      for (int k = cnt; k < padded; ++k) {
        rows.push_back(h_csc_rows[k1 - 1]);
        perm.push_back(-1);
      }
      t->h_ptr[b + 1] = static_cast<int32_t>(rows.size());
    }
    t->count = static_cast<long long>(rows.size());
    upload(t->ptr, t->h_ptr.data(), t->h_ptr.size() * sizeof(int32_t));
    LSP_DISPATCH_ACC(compute, T, {
      using E = typename EntryOf<T>::type;
      std::vector<E> e(rows.size());
      for (size_t k = 0; k < rows.size(); ++k) {
        e[k] = E{};
        e[k].off = rows[k];
        e[k].val = perm[k] >= 0 ? static_cast<T>(h_val[perm[k]]) : T(0);
      }
      upload(t->ent, e.data(), std::max<size_t>(e.size(), 1) * sizeof(E));
    })
    upload(t->perm, perm.data(), std::max<size_t>(perm.size(), 1) * sizeof(int32_t));
    csc_pad = std::move(t);
    launch_refresh_values(*this, nullptr);  // current device values
    LSP_CUDA(cudaDeviceSynchronize());
  }
  return *csc_pad;
}

int* Pair::flag_ptr() {
  if (!flag.p) {
    flag.ensure(sizeof(int));
    LSP_CUDA(cudaMemset(flag.p, 0, sizeof(int)));
  }
  return flag.as<int>();
}

static lsp_projector_s* make_projector(int n_rows, int d, int r, const int32_t* pos,
                                 const double* val, lsp_dtype compute) {
  require(compute == LSP_F32 || compute == LSP_F64, "projector compute dtype must be F32 or F64");
  require(pos && val, "projector: null arrays");
  validate_projector(n_rows, d, r, pos, val, LSP_EINVAL);
  auto P = std::make_unique<lsp_projector_s>();
  P->n_rows = n_rows;
  P->d = d;
  P->r = r;
  P->compute = compute;
  const size_t nnz = P->nnz();
  P->h_pos.assign(pos, pos + nnz);
  P->h_val.assign(val, val + nnz);
  build_csc(n_rows, d, r, pos, P->h_csc_ptr, P->h_csc_rows, P->h_csc_perm);
  upload(P->pos, pos, nnz * sizeof(int32_t));
  upload(P->csc_ptr, P->h_csc_ptr.data(), P->h_csc_ptr.size() * sizeof(int32_t));
  upload(P->csc_row, P->h_csc_rows.data(), nnz * sizeof(int32_t));
  upload(P->csc_perm, P->h_csc_perm.data(), nnz * sizeof(int32_t));
  P->csc_val.ensure(std::max<size_t>(nnz * P->vsize(), 16));
  P->upload_values();
  return P.release();
}

double sumsq_sync(Pair& pr, int rows, int cols, const void* x, long long ld, lsp_dtype dt,
                  cudaStream_t st) {
  // gather with zero entries per row and beta = 1: the result is x itself,
  // whose squares the kernel sums deterministically.
  int np = 0;
  launch_gather(rows, cols, nullptr, 0, nullptr, nullptr, pr.compute, x, ld, dt, x, ld, nullptr,
                0, dt, 0.0, 1.0, &pr.red, &np, st);
  return reduce_partials_sync(pr.red.as<double>(), np, st);
}

}  // namespace lspb

using namespace lspb;

static void check_ld(long long ld, int cols, const char* what) {
  if (ld < cols) fail(LSP_EINVAL, std::string(what) + ": leading dimension smaller than columns");
}

template <typename T>
static void moments_to_host(const Adam& a, const DevBuf& b, double* out, lsp_layout layout) {
  std::vector<T> tmp(a.count());
  LSP_CUDA(cudaMemcpy(tmp.data(), b.p, tmp.size() * sizeof(T), cudaMemcpyDeviceToHost));
  const bool tr = layout != a.layout;
  // stored layout: ROW -> [r][c] at r*cols+c ; T -> [r][c] at c*rows+r
  for (int r = 0; r < a.rows; ++r)
    for (int c = 0; c < a.cols; ++c) {
      const size_t src = a.layout == LSP_LAYOUT_ROW ? static_cast<size_t>(r) * a.cols + c
                                                    : static_cast<size_t>(c) * a.rows + r;
      const size_t dst = (tr ? layout : a.layout) == LSP_LAYOUT_ROW
                             ? static_cast<size_t>(r) * a.cols + c
                             : static_cast<size_t>(c) * a.rows + r;
      out[dst] = static_cast<double>(tmp[src]);
    }
}

template <typename T>
static void moments_from_host(const Adam& a, DevBuf& b, const double* in, lsp_layout layout) {
  std::vector<T> tmp(a.count());
  for (int r = 0; r < a.rows; ++r)
    for (int c = 0; c < a.cols; ++c) {
      const size_t src = layout == LSP_LAYOUT_ROW ? static_cast<size_t>(r) * a.cols + c
                                                  : static_cast<size_t>(c) * a.rows + r;
      const size_t dst = a.layout == LSP_LAYOUT_ROW ? static_cast<size_t>(r) * a.cols + c
                                                    : static_cast<size_t>(c) * a.rows + r;
      tmp[dst] = static_cast<T>(in[src]);
    }
  LSP_CUDA(cudaMemcpy(b.p, tmp.data(), tmp.size() * sizeof(T), cudaMemcpyHostToDevice));
}

extern "C" {

const char* lsp_last_error(void) { return g_last_error.c_str(); }
int lsp_version(void) { return LSP_B200_VERSION; }
uint64_t lsp_launch_count(void) { return g_launches.load(); }

int lsp_set_sm_budget(int compress_sms, int update_sms) {
  return guard([&] {
    if (compress_sms < 0 || update_sms < 0) fail(LSP_EINVAL, "lsp_set_sm_budget: negative budget");
    g_budget[0].store(compress_sms);
    g_budget[1].store(update_sms);
  });
}

int lsp_device_count(int* count) {
  return guard([&] {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *count = c;
  });
}

lsp_fit_config lsp_fit_config_default(void) {
  lsp_fit_config c;
  c.alpha = 0.1;
  c.reg_beta = 0.0;
  c.step_size = 1e-2;
  c.max_steps = 500;
  c.timeout_steps = 500;
  c.seed = 0;
  c.reg_kind = LSP_REG_SQUARED;
  return c;
}

uint64_t lsp_derive_seed(uint64_t master, uint64_t tag, uint64_t index) {
  return derive_seed(master, tag, index);
}

int lsp_init_sparse(int n_rows, int d, int r, uint64_t seed, int32_t* pos, double* val) {
  return guard([&] { init_sparse(n_rows, d, r, seed, pos, val); });
}

int lsp_identity_pattern(int n_rows, int32_t* pos, double* val) {
  return guard([&] {
    require(n_rows >= 1, "identity_pattern: n_rows must be >= 1");
    for (int i = 0; i < n_rows; ++i) {
      pos[i] = i;
      val[i] = 1.0;
    }
  });
}

int lsp_save_projector(int n_rows, int d, int r, const int32_t* pos, const double* val,
                       char* buf, int64_t cap, int64_t* needed) {
  return guard([&] {
    const std::string s = save_projector_text(n_rows, d, r, pos, val);
    if (needed) *needed = static_cast<int64_t>(s.size()) + 1;
    if (buf && cap > 0) {
      const size_t nc = std::min<size_t>(static_cast<size_t>(cap - 1), s.size());
      std::memcpy(buf, s.data(), nc);
      buf[nc] = '\0';
    }
  });
}

int lsp_load_projector(const char* text, int64_t len, int* n_rows, int* d, int* r,
                       int32_t* pos, double* val) {
  return guard([&] {
    require(text != nullptr, "load_projector: null text");
    const std::string s(text, len >= 0 ? static_cast<size_t>(len) : std::strlen(text));
    load_projector_text(s, n_rows, d, r, pos, val);
  });
}

int lsp_subsample_size(double gamma_bound, double chernoff_beta, int m, int n, int total_steps,
                       double delta, int64_t* out) {
  return guard([&] { *out = subsample_size(gamma_bound, chernoff_beta, m, n, total_steps, delta); });
}

// ---- projectors / pairs --------------------------------------------------------
int lsp_projector_create(int n_rows, int d, int r, const int32_t* pos, const double* val,
                         lsp_dtype compute, lsp_projector_t* out) {
  return guard([&] {
    *out = make_projector(n_rows, d, r, pos, val, compute);
  });
}

int lsp_projector_set_values(lsp_projector_t p, const double* val) {
  return guard([&] {
    require(p && val, "projector_set_values: null argument");
    validate_projector(p->n_rows, p->d, p->r, p->h_pos.data(), val, LSP_EINVAL);
    p->h_val.assign(val, val + p->nnz());
    p->upload_values();
  });
}

int lsp_projector_get(lsp_projector_t p, int32_t* pos, double* val) {
  return guard([&] {
    require(p != nullptr, "projector_get: null handle");
    if (pos) std::copy(p->h_pos.begin(), p->h_pos.end(), pos);
    if (val) {
      LSP_DISPATCH_ACC(p->compute, T, {
        std::vector<T> tmp(p->nnz());
        LSP_CUDA(cudaMemcpy(tmp.data(), p->val.p, tmp.size() * sizeof(T), cudaMemcpyDeviceToHost));
        if (p->compute == LSP_F64)
          std::copy(tmp.begin(), tmp.end(), val);
        else  // fp32 device copy: report the exact host values the caller gave
          std::copy(p->h_val.begin(), p->h_val.end(), val);
      })
    }
  });
}

int lsp_projector_shape(lsp_projector_t p, int* n_rows, int* d, int* r) {
  return guard([&] {
    require(p != nullptr, "projector_shape: null handle");
    if (n_rows) *n_rows = p->n_rows;
    if (d) *d = p->d;
    if (r) *r = p->r;
  });
}

int lsp_projector_destroy(lsp_projector_t p) {
  return guard([&] { delete p; });
}

int lsp_pair_create(lsp_projector_t p, lsp_projector_t q, lsp_pair_t* out) {
  return guard([&] {
    require(p && q && out, "pair_create: null argument");
    if (p->d != q->d) fail(LSP_EINVAL, "projector pair: P.d != Q.d");
    require(p->compute == q->compute, "pair_create: P and Q compute dtypes differ");
    auto* pr = new lsp_pair_s();
    pr->p = p;
    pr->q = q;
    pr->m = p->n_rows;
    pr->n = q->n_rows;
    pr->d = p->d;
    pr->compute = p->compute;
    *out = pr;
  });
}

int lsp_pair_destroy(lsp_pair_t pair) {
  return guard([&] { delete pair; });
}

int lsp_projector_mul(lsp_projector_t p, int op, int free_dim, const void* x, int64_t ldx,
                      void* out, int64_t ldo, lsp_stream_t stream) {
  return guard([&] {
    require(p && x && out, "projector_mul: null argument");
    require(free_dim >= 0, "projector_mul: negative dimension");
    cudaStream_t st = as_stream(stream);
    const Projector& P = *p;
    const lsp_dtype dt = P.compute;
    const size_t vs = dtype_size(dt);
    if (free_dim == 0) return;
    switch (op) {
      case LSP_LEFT:  // rows of x gathered by the CSR of P
        check_ld(ldx, free_dim, "left_mul");
        check_ld(ldo, free_dim, "left_mul");
        launch_gather(P.n_rows, free_dim, nullptr, P.r, P.pos.as<int>(), P.val.p, dt, x, ldx,
                      dt, nullptr, 0, out, ldo, dt, 1.0, 0.0, nullptr, nullptr, st);
        break;
      case LSP_LEFT_T:  // rows of x gathered by the CSC of P
        check_ld(ldx, free_dim, "leftT_mul");
        check_ld(ldo, free_dim, "leftT_mul");
        launch_gather(P.d, free_dim, P.csc_ptr.as<int>(), 0, P.csc_row.as<int>(), P.csc_val.p,
                      dt, x, ldx, dt, nullptr, 0, out, ldo, dt, 1.0, 0.0, nullptr, nullptr, st);
        break;
      case LSP_RIGHT:
      case LSP_RIGHT_T: {
        // x P = (P^T x^T)^T ;  x P^T = (P x^T)^T
        const bool right = op == LSP_RIGHT;
        const int in_cols = right ? P.n_rows : P.d;
        const int out_cols = right ? P.d : P.n_rows;
        check_ld(ldx, in_cols, "right_mul");
        check_ld(ldo, out_cols, "right_mul");
        DevBuf xt, yt;
        xt.ensure(static_cast<size_t>(in_cols) * free_dim * vs);
        yt.ensure(static_cast<size_t>(out_cols) * free_dim * vs);
        launch_transpose(free_dim, in_cols, x, ldx, xt.p, free_dim, dt, st);
        if (right)
          launch_gather(P.d, free_dim, P.csc_ptr.as<int>(), 0, P.csc_row.as<int>(), P.csc_val.p,
                        dt, xt.p, free_dim, dt, nullptr, 0, yt.p, free_dim, dt, 1.0, 0.0,
                        nullptr, nullptr, st);
        else
          launch_gather(P.n_rows, free_dim, nullptr, P.r, P.pos.as<int>(), P.val.p, dt, xt.p,
                        free_dim, dt, nullptr, 0, yt.p, free_dim, dt, 1.0, 0.0, nullptr, nullptr,
                        st);
        launch_transpose(out_cols, free_dim, yt.p, free_dim, out, ldo, dt, st);
        LSP_CUDA(cudaStreamSynchronize(st));  // temporaries die here
        break;
      }
      default:
        fail(LSP_EINVAL, "projector_mul: unknown op");
    }
  });
}

// ---- hot path ------------------------------------------------------------------

int lsp_compress(lsp_pair_t pair, const void* g, int64_t ldg, lsp_dtype g_dtype, void* s,
                 lsp_layout s_layout, lsp_stream_t stream) {
  return guard([&] {
    require(pair && g && s, "compress: null argument");
    check_ld(ldg, pair->n, "compress");
    cudaStream_t st = as_stream(stream);
    if (s_layout == LSP_LAYOUT_T) {
      compress_T(*pair, g, ldg, g_dtype, s, st);
    } else {
      pair->s_t.ensure(static_cast<size_t>(pair->d) * pair->d * dtype_size(pair->compute));
      compress_T(*pair, g, ldg, g_dtype, pair->s_t.p, st);
      launch_transpose(pair->d, pair->d, pair->s_t.p, pair->d, s, pair->d, pair->compute, st);
    }
  });
}

int lsp_decompress(lsp_pair_t pair, const void* s, lsp_layout s_layout, void* out, int64_t ldo,
                   lsp_dtype out_dtype, lsp_stream_t stream) {
  return guard([&] {
    require(pair && s && out, "decompress: null argument");
    check_ld(ldo, pair->n, "decompress");
    cudaStream_t st = as_stream(stream);
    const void* dT = delta_as_T(*pair, s, s_layout, st);
    launch_decompress(*pair, dT, nullptr, 0, out, ldo, out_dtype, 1.0, 0.0, nullptr, nullptr,
                      nullptr, st);
  });
}

int lsp_decompress_apply(lsp_pair_t pair, const void* delta, lsp_layout delta_layout, double lr,
                         void* w, int64_t ldw, lsp_dtype w_dtype, lsp_stream_t stream) {
  return guard([&] {
    require(pair && delta && w, "decompress_apply: null argument");
    check_ld(ldw, pair->n, "decompress_apply");
    cudaStream_t st = as_stream(stream);
    const void* dT = delta_as_T(*pair, delta, delta_layout, st);
    launch_decompress(*pair, dT, w, ldw, w, ldw, w_dtype, -lr, 1.0, nullptr, nullptr, nullptr,
                      st);
  });
}

int lsp_estimation_bias(lsp_pair_t pair, const void* sigma, int64_t lds, lsp_dtype dtype,
                        void* out, int64_t ldo, lsp_stream_t stream) {
  return guard([&] {
    require(pair && sigma && out, "estimation_bias: null argument");
    check_ld(lds, pair->n, "estimation_bias");
    check_ld(ldo, pair->n, "estimation_bias");
    cudaStream_t st = as_stream(stream);
    pair->s_t.ensure(static_cast<size_t>(pair->d) * pair->d * dtype_size(pair->compute));
    compress_T(*pair, sigma, lds, dtype, pair->s_t.p, st);
    launch_decompress(*pair, pair->s_t.p, sigma, lds, out, ldo, dtype, 1.0, -1.0, nullptr,
                      nullptr, nullptr, st);
  });
}

int lsp_relative_bias(lsp_pair_t pair, const void* sigma, int64_t lds, lsp_dtype dtype,
                      double* out, lsp_stream_t stream) {
  return guard([&] {
    require(pair && sigma && out, "relative_bias: null argument");
    check_ld(lds, pair->n, "relative_bias");
    cudaStream_t st = as_stream(stream);
    const double den = std::sqrt(sumsq_sync(*pair, pair->m, pair->n, sigma, lds, dtype, st));
    if (den == 0.0) fail(LSP_EINVAL, "relative_bias: zero sigma");
    pair->s_t.ensure(static_cast<size_t>(pair->d) * pair->d * dtype_size(pair->compute));
    compress_T(*pair, sigma, lds, dtype, pair->s_t.p, st);
    int np = 0;
    launch_decompress(*pair, pair->s_t.p, sigma, lds, nullptr, 0, dtype, 1.0, -1.0, nullptr,
                      &pair->red, &np, st);
    const double num = std::sqrt(reduce_partials_sync(pair->red.as<double>(), np, st));
    *out = num / den;
  });
}

// ---- Adam ------------------------------------------------------------------------
int lsp_adam_create(int rows, int cols, double beta1, double beta2, double eps,
                    lsp_dtype compute, lsp_layout layout, lsp_adam_t* out) {
  return guard([&] {
    if (rows < 1 || cols < 1) fail(LSP_EINVAL, "make_opt_state: dims must be >= 1");
    if (beta1 <= 0.0 || beta1 >= 1.0 || beta2 <= 0.0 || beta2 >= 1.0)
      fail(LSP_EINVAL, "make_opt_state: betas must lie in (0, 1)");
    if (eps <= 0.0) fail(LSP_EINVAL, "make_opt_state: eps must be positive");
    require(compute == LSP_F32 || compute == LSP_F64, "adam: compute dtype must be F32 or F64");
    auto* a = new lsp_adam_s();
    a->rows = rows;
    a->cols = cols;
    a->beta1 = beta1;
    a->beta2 = beta2;
    a->eps = eps;
    a->compute = compute;
    a->layout = layout;
    const size_t bytes = a->count() * dtype_size(compute);
    try {
      a->m.ensure(bytes);
      a->v.ensure(bytes);
      a->flag.ensure(sizeof(int));
      a->dstep.ensure(sizeof(long long));
      a->done.ensure(sizeof(unsigned));
      LSP_CUDA(cudaMemset(a->done.p, 0, sizeof(unsigned)));
      LSP_CUDA(cudaMemset(a->m.p, 0, bytes));
      LSP_CUDA(cudaMemset(a->v.p, 0, bytes));
      LSP_CUDA(cudaMemset(a->flag.p, 0, sizeof(int)));
      LSP_CUDA(cudaMemset(a->dstep.p, 0, sizeof(long long)));
    } catch (...) {
      delete a;
      throw;
    }
    *out = a;
  });
}

int lsp_adam_destroy(lsp_adam_t st) {
  return guard([&] { delete st; });
}

int lsp_adam_step(lsp_adam_t a, const void* grad, void* delta, lsp_stream_t stream) {
  return guard([&] {
    require(a && grad && delta, "adam_step: null argument");
    cudaStream_t st = as_stream(stream);
    // Reference semantics: a non-finite gradient throws before any state
    // change (subspace_opt.cpp:38) -> check first, skip the update if latched.
    launch_check_finite(a->count(), grad, a->compute, a->flag.as<int>(), st);
    launch_adam(*a, grad, delta, a->flag.as<int>(), st);
  });
}

int lsp_adam_check(lsp_adam_t a, lsp_stream_t stream) {
  int rc = guard([&] {
    require(a != nullptr, "adam_check: null handle");
    int h = 0;
    cudaStream_t st = as_stream(stream);
    LSP_CUDA(cudaMemcpyAsync(&h, a->flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    LSP_CUDA(cudaStreamSynchronize(st));
    if (h) {
      LSP_CUDA(cudaMemset(a->flag.p, 0, sizeof(int)));
      fail(LSP_ENUMERIC, "adam_step: non-finite gradient");
    }
  });
  return rc;
}

int lsp_adam_get(lsp_adam_t a, double* m, double* v, int64_t* step, lsp_layout layout) {
  return guard([&] {
    require(a != nullptr, "adam_get: null handle");
    LSP_CUDA(cudaDeviceSynchronize());
    LSP_DISPATCH_ACC(a->compute, T, {
      if (m) moments_to_host<T>(*a, a->m, m, layout);
      if (v) moments_to_host<T>(*a, a->v, v, layout);
    })
    if (step) {
      long long h = 0;
      LSP_CUDA(cudaMemcpy(&h, a->dstep.p, sizeof(h), cudaMemcpyDeviceToHost));
      *step = h;
    }
  });
}

int lsp_adam_set(lsp_adam_t a, const double* m, const double* v, int64_t step,
                 lsp_layout layout) {
  return guard([&] {
    require(a != nullptr, "adam_set: null handle");
    LSP_CUDA(cudaDeviceSynchronize());
    LSP_DISPATCH_ACC(a->compute, T, {
      if (m) moments_from_host<T>(*a, a->m, m, layout);
      if (v) moments_from_host<T>(*a, a->v, v, layout);
    })
    const long long h = step;
    LSP_CUDA(cudaMemcpy(a->dstep.p, &h, sizeof(h), cudaMemcpyHostToDevice));
  });
}

int lsp_adam_info(lsp_adam_t a, int* rows, int* cols, double* beta1, double* beta2,
                  double* eps) {
  return guard([&] {
    require(a != nullptr, "adam_info: null handle");
    if (rows) *rows = a->rows;
    if (cols) *cols = a->cols;
    if (beta1) *beta1 = a->beta1;
    if (beta2) *beta2 = a->beta2;
    if (eps) *eps = a->eps;
  });
}

// ---- fused per-matrix step -----------------------------------------------------
static void check_step_args(lsp_pair_t pair, lsp_adam_t a) {
  require(pair && a, "step: null handle");
  require(a->rows == pair->d && a->cols == pair->d, "adam_step: grad dims do not match state");
  require(a->layout == LSP_LAYOUT_T, "step: the Adam state must use LSP_LAYOUT_T");
  require(a->compute == pair->compute, "step: Adam and pair compute dtypes differ");
}

static void update_impl(Pair& pr, Adam& a, const void* s_t, void* w, long long ldw,
                        lsp_dtype w_dtype, double lr, cudaStream_t st, bool check) {
  pr.d_t.ensure(static_cast<size_t>(pr.d) * pr.d * dtype_size(pr.compute));
  // non-finite S -> skip Adam and the apply (NumericError semantics)
  if (check) launch_check_finite(a.count(), s_t, a.compute, a.flag.as<int>(), st);
  launch_adam(a, s_t, pr.d_t.p, a.flag.as<int>(), st);
  launch_decompress(pr, pr.d_t.p, w, ldw, w, ldw, w_dtype, -lr, 1.0, a.flag.as<int>(), nullptr,
                    nullptr, st);
}

int lsp_step(lsp_pair_t pair, lsp_adam_t a, const void* g, int64_t ldg, lsp_dtype g_dtype,
             void* w, int64_t ldw, lsp_dtype w_dtype, double lr, void* s_out,
             lsp_stream_t stream) {
  return guard([&] {
    check_step_args(pair, a);
    require(g && w, "step: null argument");
    check_ld(ldg, pair->n, "step");
    check_ld(ldw, pair->n, "step");
    cudaStream_t st = as_stream(stream);
    void* s_t = s_out;
    if (!s_t) {
      pair->s_t.ensure(static_cast<size_t>(pair->d) * pair->d * dtype_size(pair->compute));
      s_t = pair->s_t.p;
    }
    // stage 2 latches the non-finite flag while writing S, so no extra check pass
    compress_T(*pair, g, ldg, g_dtype, s_t, st, a->flag.as<int>());
    update_impl(*pair, *a, s_t, w, ldw, w_dtype, lr, st, false);
  });
}

int lsp_update(lsp_pair_t pair, lsp_adam_t a, const void* s_t, void* w, int64_t ldw,
               lsp_dtype w_dtype, double lr, lsp_stream_t stream) {
  return guard([&] {
    check_step_args(pair, a);
    require(s_t && w, "update: null argument");
    check_ld(ldw, pair->n, "update");
    update_impl(*pair, *a, s_t, w, ldw, w_dtype, lr, as_stream(stream), true);
  });
}

}  // extern "C"

// ---- bias-gated projector refresh (proj/src/trainer.cpp:74-112) -----------------
extern "C" {

int lsp_maybe_update(lsp_pair_t pair, lsp_adam_t st, const void* grad_sub, int64_t ld,
                     lsp_dtype dtype, const void* const* extra, int n_extra, int r,
                     double alpha, const lsp_fit_config* fit_cfg, lsp_transfer_kind transfer,
                     uint64_t reinit_seed, lsp_projector_t* new_p, lsp_projector_t* new_q,
                     lsp_pair_t* new_pair, lsp_maybe_update_result* res, lsp_stream_t stream) {
  lsp_projector_t np = nullptr, nq = nullptr;
  lsp_pair_t npair = nullptr;
  const int rc = guard([&] {
    require(pair && st && grad_sub && fit_cfg && new_p && new_q && new_pair && res,
            "maybe_update: null argument");
    require(n_extra >= 0 && (n_extra == 0 || extra), "maybe_update: bad extra targets");
    check_ld(ld, pair->n, "maybe_update");
    *new_p = nullptr, *new_q = nullptr, *new_pair = nullptr;
    cudaStream_t s = as_stream(stream);
    const double nan = std::numeric_limits<double>::quiet_NaN();
    *res = lsp_maybe_update_result{0, 0, 0, 0, 0.0, 0.0};
    // trainer.cpp:82-87: a zero gradient skips the check
    if (sumsq_sync(*pair, pair->m, pair->n, grad_sub, ld, dtype, s) == 0.0) {
      res->skipped_zero_grad = 1;
      res->bias_before = res->bias_after = nan;
      return;
    }
    auto call = [](int code) {
      if (code != LSP_OK) fail(code, g_last_error);
    };
    call(lsp_relative_bias(pair, grad_sub, ld, dtype, &res->bias_before, stream));
    res->bias_after = res->bias_before;
    if (res->bias_before <= alpha) return;  // trainer.cpp:88
    // trainer.cpp:90-93: fresh pair from the refresh seed
    const lspb::Projector& op = *pair->p;
    const lspb::Projector& oq = *pair->q;
    std::vector<int32_t> pp(static_cast<size_t>(op.n_rows) * r), qp(static_cast<size_t>(oq.n_rows) * r);
    std::vector<double> pv(pp.size()), qv(qp.size());
    call(lsp_init_sparse(op.n_rows, op.d, r, lsp_derive_seed(reinit_seed, 1, 0), pp.data(), pv.data()));
    call(lsp_init_sparse(oq.n_rows, oq.d, r, lsp_derive_seed(reinit_seed, 2, 0), qp.data(), qv.data()));
    call(lsp_projector_create(op.n_rows, op.d, r, pp.data(), pv.data(), op.compute, &np));
    call(lsp_projector_create(oq.n_rows, oq.d, r, qp.data(), qv.data(), oq.compute, &nq));
    call(lsp_pair_create(np, nq, &npair));
    // trainer.cpp:95-103: fit on grad_sub plus the non-zero extra targets
    std::vector<const void*> targets{grad_sub};
    for (int i = 0; i < n_extra; ++i) {
      require(extra[i] != nullptr, "maybe_update: null extra target");
      if (sumsq_sync(*pair, pair->m, pair->n, extra[i], ld, dtype, s) > 0.0) targets.push_back(extra[i]);
    }
    lsp_fit_config cfg = *fit_cfg;
    cfg.seed = lsp_derive_seed(reinit_seed, 3, 0);
    lsp_fit_report rep{};
    call(lsp_fit(npair, targets.data(), static_cast<int>(targets.size()), ld, dtype, &cfg, &rep,
                 nullptr, 0, stream));
    // trainer.cpp:105-110: state transfer, report, bias on the new pair
    call(lsp_reproject_state(st, pair, npair, transfer, stream));
    res->refreshed = 1;
    res->fit_timed_out = (rep.timed_out || rep.stalled) ? 1 : 0;
    res->fit_steps = rep.steps;
    call(lsp_relative_bias(npair, grad_sub, ld, dtype, &res->bias_after, stream));
    *new_p = np, *new_q = nq, *new_pair = npair;
  });
  if (rc != LSP_OK) {  // nothing half-built escapes
    if (npair) lsp_pair_destroy(npair);
    if (np) lsp_projector_destroy(np);
    if (nq) lsp_projector_destroy(nq);
  }
  return rc;
}

}  // extern "C"
