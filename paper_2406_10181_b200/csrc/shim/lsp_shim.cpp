// C++ drop-in implementation (include/lsp_b200/lsp.hpp) over the C-ABI.
// Device work goes through liblsp_b200.so in fp64; this file only moves
// lsp::Matrix values to and from the device and maps status codes to the
// reference's exception types.
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <istream>
#include <memory>
#include <ostream>
#include <sstream>

#include "lsp_b200.h"
#include "lsp_b200/lsp.hpp"

namespace lsp {
namespace {

[[noreturn]] void raise(int rc) {
  const std::string msg = lsp_last_error();
  switch (rc) {
    case LSP_EINVAL: throw std::invalid_argument(msg);
    case LSP_ENUMERIC: throw NumericError(msg);
    case LSP_EIO: throw IoError(msg);
    default: throw std::runtime_error("lsp_b200: " + msg);
  }
}
void ck(int rc) {
  if (rc != LSP_OK) raise(rc);
}
void cuda_ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Device copy of a host matrix (fp64).
struct DevMat {
  double* p = nullptr;
  int rows = 0, cols = 0;
  DevMat(int r, int c) : rows(r), cols(c) {
    const size_t n = std::max<size_t>(static_cast<size_t>(r) * c, 1);
    cuda_ck(cudaMalloc(&p, n * sizeof(double)), "cudaMalloc");
  }
  explicit DevMat(const Matrix& m) : DevMat(m.rows(), m.cols()) {
    if (m.size())
      cuda_ck(cudaMemcpy(p, m.data(), m.size() * sizeof(double), cudaMemcpyHostToDevice), "h2d");
  }
  DevMat(const DevMat&) = delete;
  ~DevMat() { cudaFree(p); }
  Matrix host() const {
    Matrix m(rows, cols);
    cuda_ck(cudaDeviceSynchronize(), "sync");
    if (m.size())
      cuda_ck(cudaMemcpy(m.data(), p, m.size() * sizeof(double), cudaMemcpyDeviceToHost), "d2h");
    return m;
  }
  int64_t ld() const { return std::max(cols, 1); }
};

struct DevProj {
  lsp_projector_t h = nullptr;
  explicit DevProj(const SparseProjector& sp) {
    if (sp.n_rows < 1 || sp.r < 1 || sp.r > sp.d)
      throw std::invalid_argument("projector: invalid dimensions");
    static_assert(sizeof(int) == sizeof(int32_t), "int must be 32-bit");
    ck(lsp_projector_create(sp.n_rows, sp.d, sp.r,
                            reinterpret_cast<const int32_t*>(sp.positions.data()),
                            sp.values.data(), LSP_F64, &h));
  }
  DevProj(const DevProj&) = delete;
  ~DevProj() { lsp_projector_destroy(h); }
};

struct DevPair {
  DevProj p, q;
  lsp_pair_t h = nullptr;
  explicit DevPair(const ProjectorPair& pr) : p(pr.p), q(pr.q) { ck(lsp_pair_create(p.h, q.h, &h)); }
  DevPair(const DevPair&) = delete;
  ~DevPair() { lsp_pair_destroy(h); }
};

void check_pair(const ProjectorPair& pair) {
  if (pair.p.d != pair.q.d) throw std::invalid_argument("projector pair: P.d != Q.d");
}

void check_targets(const ProjectorPair& pair, const std::vector<Matrix>& targets) {
  if (targets.empty()) throw std::invalid_argument("fit: empty target corpus");
  for (const Matrix& g : targets)
    if (g.rows() != pair.p.n_rows || g.cols() != pair.q.n_rows)
      throw std::invalid_argument("fit: target dims do not match projector pair");
}

lsp_fit_config to_c(const FitConfig& c) {
  lsp_fit_config o = lsp_fit_config_default();
  o.alpha = c.alpha;
  o.reg_beta = c.reg_beta;
  o.step_size = c.step_size;
  o.max_steps = c.max_steps;
  o.timeout_steps = c.timeout_steps;
  o.seed = c.seed;
  o.reg_kind = c.reg_kind == RegKind::kSquared ? LSP_REG_SQUARED : LSP_REG_UNSQUARED;
  return o;
}

struct DevTargets {
  std::vector<std::unique_ptr<DevMat>> mats;
  std::vector<const void*> ptrs;
  explicit DevTargets(const std::vector<Matrix>& t) {
    for (const Matrix& g : t) {
      mats.push_back(std::make_unique<DevMat>(g));
      ptrs.push_back(mats.back()->p);
    }
  }
};

Matrix mul(const SparseProjector& sp, int op, int free_dim, const Matrix& x, int out_rows,
           int out_cols) {
  if (out_rows == 0 || out_cols == 0) return Matrix(out_rows, out_cols);
  DevProj p(sp);
  DevMat dx(x), out(out_rows, out_cols);
  ck(lsp_projector_mul(p.h, op, free_dim, dx.p, dx.ld(), out.p, out.ld(), nullptr));
  return out.host();
}

}  // namespace

// ---- common ------------------------------------------------------------------
uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
uint64_t derive_seed(uint64_t master, uint64_t tag, uint64_t index) {
  return lsp_derive_seed(master, tag, index);
}

// ---- Matrix (host carrier) ------------------------------------------------------
Matrix::Matrix(int rows, int cols, double fill) : r_(rows), c_(cols) {
  if (rows < 0 || cols < 0) throw std::invalid_argument("Matrix: negative dimension");
  v_.assign(static_cast<size_t>(rows) * cols, fill);
}
Matrix::Matrix(int rows, int cols, std::vector<double> data) : r_(rows), c_(cols), v_(std::move(data)) {
  if (rows < 0 || cols < 0) throw std::invalid_argument("Matrix: negative dimension");
  if (v_.size() != static_cast<size_t>(rows) * cols)
    throw std::invalid_argument("Matrix: data length does not match rows*cols");
}
Matrix Matrix::identity(int n) {
  Matrix m(n, n);
  for (int i = 0; i < n; ++i) m(i, i) = 1.0;
  return m;
}
bool Matrix::all_finite() const {
  return std::all_of(v_.begin(), v_.end(), [](double x) { return std::isfinite(x); });
}
Matrix Matrix::transposed() const {
  Matrix t(c_, r_);
  for (int i = 0; i < r_; ++i)
    for (int j = 0; j < c_; ++j) t(j, i) = (*this)(i, j);
  return t;
}
Matrix& Matrix::operator+=(const Matrix& o) {
  if (!same_shape(o)) throw std::invalid_argument("Matrix+=: shape mismatch");
  for (size_t i = 0; i < v_.size(); ++i) v_[i] += o.v_[i];
  return *this;
}
Matrix& Matrix::operator-=(const Matrix& o) {
  if (!same_shape(o)) throw std::invalid_argument("Matrix-=: shape mismatch");
  for (size_t i = 0; i < v_.size(); ++i) v_[i] -= o.v_[i];
  return *this;
}
Matrix& Matrix::operator*=(double s) {
  for (double& x : v_) x *= s;
  return *this;
}
Matrix matmul(const Matrix& a, const Matrix& b) {
  if (a.cols() != b.rows()) throw std::invalid_argument("matmul: inner dimensions differ");
  Matrix out(a.rows(), b.cols());
  for (int i = 0; i < a.rows(); ++i)
    for (int k = 0; k < a.cols(); ++k) {
      const double x = a(i, k);
      if (x == 0.0) continue;
      for (int j = 0; j < b.cols(); ++j) out(i, j) += x * b(k, j);
    }
  return out;
}
double frobenius_norm(const Matrix& a) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a.data()[i] * a.data()[i];
  return std::sqrt(s);
}
double frobenius_distance(const Matrix& a, const Matrix& b) {
  if (!a.same_shape(b)) throw std::invalid_argument("frobenius_distance: shape mismatch");
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    const double d = a.data()[i] - b.data()[i];
    s += d * d;
  }
  return std::sqrt(s);
}
std::string format_double(double v) {
  char buf[32];
  auto res = std::to_chars(buf, buf + sizeof(buf), v);
  if (res.ec != std::errc()) throw NumericError("format_double: conversion failed");
  return std::string(buf, res.ptr);
}
void save_csv(const Matrix& m, std::ostream& out) {
  for (int i = 0; i < m.rows(); ++i) {
    for (int j = 0; j < m.cols(); ++j) out << (j ? "," : "") << format_double(m(i, j));
    out << '\n';
  }
}
Matrix load_csv(std::istream& in) {
  std::vector<double> data;
  int rows = 0, cols = -1;
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    int nc = 0;
    const char* p = line.data();
    const char* end = p + line.size();
    while (p < end) {
      double v;
      auto res = std::from_chars(p, end, v);
      if (res.ec != std::errc()) throw IoError("load_csv: bad number");
      data.push_back(v);
      ++nc;
      p = res.ptr;
      if (p < end) {
        if (*p != ',') throw IoError("load_csv: expected ','");
        ++p;
      }
    }
    if (cols >= 0 && nc != cols) throw IoError("load_csv: ragged rows");
    cols = nc;
    ++rows;
  }
  return Matrix(rows, std::max(cols, 0), std::move(data));
}

// ---- Rng (host) -----------------------------------------------------------------
double Rng::next_unit() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
uint64_t Rng::uniform_int(uint64_t n) {
  const uint64_t cap = UINT64_MAX - UINT64_MAX % n;
  for (;;) {
    const uint64_t x = gen_();
    if (x < cap) return x % n;
  }
}
double Rng::normal() {
  if (has_spare_) {
    has_spare_ = false;
    return spare_;
  }
  double u1 = next_unit();
  while (u1 <= 0.0) u1 = next_unit();
  const double u2 = next_unit();
  const double rad = std::sqrt(-2.0 * std::log(u1)), th = 6.283185307179586476925286766559 * u2;
  spare_ = rad * std::sin(th);
  has_spare_ = true;
  return rad * std::cos(th);
}
std::vector<int> Rng::sample_without_replacement(int n, int k) {
  std::vector<int> pool(n);
  for (int i = 0; i < n; ++i) pool[i] = i;
  for (int i = 0; i < k; ++i)
    std::swap(pool[i], pool[i + static_cast<int>(uniform_int(static_cast<uint64_t>(n - i)))]);
  pool.resize(k);
  std::sort(pool.begin(), pool.end());
  return pool;
}

// ---- projectors -------------------------------------------------------------------
SparseProjector init_sparse(int n_rows, int d, int r, std::uint64_t seed) {
  SparseProjector p;
  p.n_rows = n_rows;
  p.d = d;
  p.r = r;
  const size_t cnt = (n_rows > 0 && r > 0) ? static_cast<size_t>(n_rows) * r : 0;
  p.positions.resize(std::max<size_t>(cnt, 1));
  p.values.resize(std::max<size_t>(cnt, 1));
  ck(lsp_init_sparse(n_rows, d, r, seed, reinterpret_cast<int32_t*>(p.positions.data()),
                     p.values.data()));
  p.positions.resize(cnt);
  p.values.resize(cnt);
  return p;
}
SparseProjector identity_pattern(int n_rows) {
  SparseProjector p;
  p.n_rows = n_rows;
  p.d = n_rows;
  p.r = 1;
  p.positions.resize(n_rows);
  p.values.assign(n_rows, 1.0);
  for (int i = 0; i < n_rows; ++i) p.positions[i] = i;
  return p;
}
Matrix to_dense(const SparseProjector& p) {
  Matrix m(p.n_rows, p.d);
  for (int i = 0; i < p.n_rows; ++i)
    for (int k = 0; k < p.r; ++k) m(i, p.pos(i, k)) = p.val(i, k);
  return m;
}

Matrix left_mul(const SparseProjector& p, const Matrix& y) {
  if (y.rows() != p.d) throw std::invalid_argument("left_mul: y.rows != d");
  return mul(p, LSP_LEFT, y.cols(), y, p.n_rows, y.cols());
}
Matrix leftT_mul(const SparseProjector& p, const Matrix& x) {
  if (x.rows() != p.n_rows) throw std::invalid_argument("leftT_mul: x.rows != n_rows");
  return mul(p, LSP_LEFT_T, x.cols(), x, p.d, x.cols());
}
Matrix right_mul(const Matrix& x, const SparseProjector& q) {
  if (x.cols() != q.n_rows) throw std::invalid_argument("right_mul: x.cols != n_rows");
  return mul(q, LSP_RIGHT, x.rows(), x, x.rows(), q.d);
}
Matrix rightT_mul(const Matrix& x, const SparseProjector& q) {
  if (x.cols() != q.d) throw std::invalid_argument("rightT_mul: x.cols != d");
  return mul(q, LSP_RIGHT_T, x.rows(), x, x.rows(), q.n_rows);
}

Matrix compress(const ProjectorPair& pair, const Matrix& g) {
  check_pair(pair);
  if (g.rows() != pair.p.n_rows || g.cols() != pair.q.n_rows)
    throw std::invalid_argument("compress: g dims do not match pair");
  DevPair dp(pair);
  DevMat dg(g), s(pair.p.d, pair.q.d);
  ck(lsp_compress(dp.h, dg.p, dg.ld(), LSP_F64, s.p, LSP_LAYOUT_ROW, nullptr));
  return s.host();
}
Matrix decompress(const ProjectorPair& pair, const Matrix& s) {
  check_pair(pair);
  if (s.rows() != pair.p.d || s.cols() != pair.q.d)
    throw std::invalid_argument("decompress: s is not d x d");
  DevPair dp(pair);
  DevMat ds(s), out(pair.p.n_rows, pair.q.n_rows);
  ck(lsp_decompress(dp.h, ds.p, LSP_LAYOUT_ROW, out.p, out.ld(), LSP_F64, nullptr));
  return out.host();
}
Matrix estimation_bias(const ProjectorPair& pair, const Matrix& sigma) {
  check_pair(pair);
  if (sigma.rows() != pair.p.n_rows || sigma.cols() != pair.q.n_rows)
    throw std::invalid_argument("compress: g dims do not match pair");
  DevPair dp(pair);
  DevMat ds(sigma), out(sigma.rows(), sigma.cols());
  ck(lsp_estimation_bias(dp.h, ds.p, ds.ld(), LSP_F64, out.p, out.ld(), nullptr));
  return out.host();
}
double relative_bias(const ProjectorPair& pair, const Matrix& sigma) {
  check_pair(pair);
  if (sigma.rows() != pair.p.n_rows || sigma.cols() != pair.q.n_rows)
    throw std::invalid_argument("compress: g dims do not match pair");
  DevPair dp(pair);
  DevMat ds(sigma);
  double out = 0.0;
  ck(lsp_relative_bias(dp.h, ds.p, ds.ld(), LSP_F64, &out, nullptr));
  return out;
}

double fit_loss(const ProjectorPair& pair, const std::vector<Matrix>& targets,
                const FitConfig& cfg) {
  check_targets(pair, targets);
  DevPair dp(pair);
  DevTargets dt(targets);
  const lsp_fit_config c = to_c(cfg);
  double out = 0.0;
  ck(lsp_fit_loss(dp.h, dt.ptrs.data(), static_cast<int>(dt.ptrs.size()), pair.q.n_rows,
                  LSP_F64, &c, &out, nullptr));
  return out;
}
FitGradient fit_gradient(const ProjectorPair& pair, const std::vector<Matrix>& targets,
                         const FitConfig& cfg) {
  check_targets(pair, targets);
  DevPair dp(pair);
  DevTargets dt(targets);
  const lsp_fit_config c = to_c(cfg);
  FitGradient g;
  g.wrt_p.resize(pair.p.values.size());
  g.wrt_q.resize(pair.q.values.size());
  ck(lsp_fit_gradient(dp.h, dt.ptrs.data(), static_cast<int>(dt.ptrs.size()), pair.q.n_rows,
                      LSP_F64, &c, g.wrt_p.data(), g.wrt_q.data(), nullptr));
  return g;
}
std::pair<ProjectorPair, FitReport> fit(const ProjectorPair& pair0,
                                        const std::vector<Matrix>& targets,
                                        const FitConfig& cfg) {
  check_pair(pair0);
  check_targets(pair0, targets);
  DevPair dp(pair0);
  DevTargets dt(targets);
  const lsp_fit_config c = to_c(cfg);
  lsp_fit_report rep{};
  const int cap = std::max(1, std::min(cfg.max_steps, cfg.timeout_steps) + 1);
  std::vector<double> curve(cap);
  ck(lsp_fit(dp.h, dt.ptrs.data(), static_cast<int>(dt.ptrs.size()), pair0.q.n_rows, LSP_F64,
             &c, &rep, curve.data(), cap, nullptr));
  ProjectorPair out = pair0;
  ck(lsp_projector_get(dp.p.h, nullptr, out.p.values.data()));
  ck(lsp_projector_get(dp.q.h, nullptr, out.q.values.data()));
  FitReport r;
  curve.resize(std::min(rep.n_loss, cap));
  r.loss_curve = std::move(curve);
  r.final_rel_bias = rep.final_rel_bias;
  r.success = rep.success != 0;
  r.timed_out = rep.timed_out != 0;
  r.stalled = rep.stalled != 0;
  r.steps = rep.steps;
  return {out, r};
}

void save_projector(const SparseProjector& p, std::ostream& out) {
  int64_t need = 0;
  ck(lsp_save_projector(p.n_rows, p.d, p.r, reinterpret_cast<const int32_t*>(p.positions.data()),
                        p.values.data(), nullptr, 0, &need));
  std::string buf(static_cast<size_t>(need), '\0');
  ck(lsp_save_projector(p.n_rows, p.d, p.r, reinterpret_cast<const int32_t*>(p.positions.data()),
                        p.values.data(), buf.data(), need, &need));
  out << buf.c_str();
}
SparseProjector load_projector(std::istream& in) {
  // Whitespace-token based like the reference (proj/src/projector.cpp:329-354):
  // consume the three header tokens, then exactly n_rows * 2r value tokens,
  // whatever the line breaks; the C-ABI parser validates them.
  std::string h0, h1, h2;
  if (!(in >> h0 >> h1 >> h2)) throw IoError("load_projector: bad header");
  std::string text = h0 + ' ' + h1 + ' ' + h2 + '\n';
  int n_rows = 0, d = 0, r = 0;
  int rc = lsp_load_projector(text.c_str(), static_cast<int64_t>(text.size()), &n_rows, &d, &r,
                              nullptr, nullptr);
  if (rc) raise(rc);
  const long long tokens = 2LL * n_rows * r;
  std::string tok;
  for (long long t = 0; t < tokens && (in >> tok); ++t) {
    text += tok;
    text += ((t + 1) % (2 * r) == 0) ? '\n' : ' ';
  }
  SparseProjector p;
  p.n_rows = n_rows;
  p.d = d;
  p.r = r;
  p.positions.resize(static_cast<size_t>(n_rows) * r);
  p.values.resize(static_cast<size_t>(n_rows) * r);
  ck(lsp_load_projector(text.c_str(), static_cast<int64_t>(text.size()), &n_rows, &d, &r,
                        reinterpret_cast<int32_t*>(p.positions.data()), p.values.data()));
  return p;
}

// ---- subspace optimizer ----------------------------------------------------------
SubspaceOptState make_opt_state(int d, double beta1, double beta2, double eps) {
  return make_opt_state(d, d, beta1, beta2, eps);
}
SubspaceOptState make_opt_state(int rows, int cols, double beta1, double beta2, double eps) {
  if (rows < 1 || cols < 1) throw std::invalid_argument("make_opt_state: dims must be >= 1");
  if (beta1 <= 0.0 || beta1 >= 1.0 || beta2 <= 0.0 || beta2 >= 1.0)
    throw std::invalid_argument("make_opt_state: betas must lie in (0, 1)");
  if (eps <= 0.0) throw std::invalid_argument("make_opt_state: eps must be positive");
  SubspaceOptState s;
  s.m = Matrix(rows, cols);
  s.v = Matrix(rows, cols);
  s.beta1 = beta1;
  s.beta2 = beta2;
  s.eps = eps;
  return s;
}

namespace {
struct DevAdam {
  lsp_adam_t h = nullptr;
  explicit DevAdam(const SubspaceOptState& s) {
    ck(lsp_adam_create(s.m.rows(), s.m.cols(), s.beta1, s.beta2, s.eps, LSP_F64, LSP_LAYOUT_ROW,
                       &h));
    ck(lsp_adam_set(h, s.m.data(), s.v.data(), s.step, LSP_LAYOUT_ROW));
  }
  DevAdam(const DevAdam&) = delete;
  ~DevAdam() { lsp_adam_destroy(h); }
  void read(SubspaceOptState& s) const {
    int64_t step = 0;
    ck(lsp_adam_get(h, s.m.data(), s.v.data(), &step, LSP_LAYOUT_ROW));
    s.step = step;
  }
};
}  // namespace

AdamResult adam_step(const SubspaceOptState& state, const Matrix& grad) {
  if (!grad.same_shape(state.m)) throw std::invalid_argument("adam_step: grad dims do not match state");
  DevAdam a(state);
  DevMat g(grad), delta(grad.rows(), grad.cols());
  ck(lsp_adam_step(a.h, g.p, delta.p, nullptr));
  ck(lsp_adam_check(a.h, nullptr));  // NumericError before any state change
  AdamResult out;
  out.state = state;
  a.read(out.state);
  out.delta = delta.host();
  return out;
}

Matrix projector_gram(const SparseProjector& a, const SparseProjector& b) {
  if (a.n_rows != b.n_rows) throw std::invalid_argument("projector_gram: row spaces differ");
  DevProj da(a), db(b);
  DevMat out(a.d, b.d);
  ck(lsp_projector_gram(da.h, db.h, out.p, nullptr));
  return out.host();
}

SubspaceOptState reproject_state(const SubspaceOptState& state, const ProjectorPair& old_pair,
                                 const ProjectorPair& new_pair, TransferKind kind) {
  if (old_pair.p.d != new_pair.p.d || old_pair.q.d != new_pair.q.d)
    throw std::invalid_argument("reproject_state: subspace widths differ");
  if (old_pair.p.n_rows != new_pair.p.n_rows || old_pair.q.n_rows != new_pair.q.n_rows)
    throw std::invalid_argument("reproject_state: weight dims differ");
  if (state.m.rows() != old_pair.p.d || state.m.cols() != old_pair.q.d)
    throw std::invalid_argument("reproject_state: state dims do not match pair");
  DevPair op(old_pair), np(new_pair);
  DevAdam a(state);
  ck(lsp_reproject_state(a.h, op.h, np.h,
                         kind == TransferKind::kEntrywiseSquare ? LSP_TRANSFER_ENTRYWISE
                                                                : LSP_TRANSFER_MATRIX,
                         nullptr));
  SubspaceOptState out = state;
  a.read(out);
  return out;
}

void save_opt_state(const SubspaceOptState& s, std::ostream& out) {
  out << s.step << ' ' << format_double(s.beta1) << ' ' << format_double(s.beta2) << ' '
      << format_double(s.eps) << ' ' << s.m.rows() << ' ' << s.m.cols() << '\n';
  save_csv(s.m, out);
  save_csv(s.v, out);
}
SubspaceOptState load_opt_state(std::istream& in) {
  std::string header;
  if (!std::getline(in, header)) throw IoError("load_opt_state: missing header");
  std::istringstream h(header);
  SubspaceOptState s;
  int rows = 0, cols = 0;
  if (!(h >> s.step >> s.beta1 >> s.beta2 >> s.eps >> rows >> cols))
    throw IoError("load_opt_state: bad header");
  if (rows < 1 || cols < 1) throw IoError("load_opt_state: bad dimensions");
  auto block = [&](const char* what) {
    std::string text, line;
    for (int i = 0; i < rows; ++i) {
      if (!std::getline(in, line)) throw IoError(std::string("load_opt_state: truncated ") + what);
      text += line + "\n";
    }
    std::istringstream ts(text);
    return load_csv(ts);
  };
  s.m = block("M");
  s.v = block("V");
  if (s.m.rows() != rows || s.m.cols() != cols || !s.m.same_shape(s.v))
    throw IoError("load_opt_state: matrix dims disagree with header");
  for (size_t i = 0; i < s.v.size(); ++i)
    if (s.v.data()[i] < 0.0) throw IoError("load_opt_state: negative second moment");
  return s;
}

}  // namespace lsp
