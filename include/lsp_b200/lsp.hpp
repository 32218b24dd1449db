// lsp_b200/lsp.hpp -- C++ drop-in for the reference's hot-path API.
//
// A reference caller written against lspkit's headers (proj/include/lsp/*.hpp)
// compiles unchanged against include/lsp/*.hpp (thin forwarders to this file)
// and links liblsp_b200_cxx.so instead of lsp_core.  The types keep the
// reference's value semantics (host lsp::Matrix in, fresh lsp::Matrix out);
// every projector product, the subspace Adam step, the fit and the state
// transfer run on the GPU through the C-ABI (include/lsp_b200.h) in fp64, and
// errors surface as the reference's exception types.
//
// Host-only pieces (Matrix arithmetic, Rng, text I/O) exist because callers
// and tests use them as the carrier and to build inputs; they are not on the
// device path.
#pragma once

#include <cstddef>
#include <cstdint>
#include <iosfwd>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace lsp {

// ---- errors (reference: proj/include/lsp/common.hpp:13-31) -----------------
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

uint64_t mix64(uint64_t x);
uint64_t derive_seed(uint64_t master, uint64_t tag, uint64_t index = 0);

// ---- dense carrier (reference: proj/include/lsp/matrix.hpp:15-55) ----------
class Matrix {
 public:
  Matrix() = default;
  Matrix(int rows, int cols) : Matrix(rows, cols, 0.0) {}
  Matrix(int rows, int cols, double fill);
  Matrix(int rows, int cols, std::vector<double> data);
  static Matrix identity(int n);

  int rows() const { return r_; }
  int cols() const { return c_; }
  std::size_t size() const { return v_.size(); }
  double& operator()(int i, int j) { return v_[static_cast<std::size_t>(i) * c_ + j]; }
  double operator()(int i, int j) const { return v_[static_cast<std::size_t>(i) * c_ + j]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double* row(int i) { return v_.data() + static_cast<std::size_t>(i) * c_; }
  const double* row(int i) const { return v_.data() + static_cast<std::size_t>(i) * c_; }
  bool same_shape(const Matrix& o) const { return r_ == o.r_ && c_ == o.c_; }
  bool all_finite() const;
  Matrix transposed() const;

  Matrix& operator+=(const Matrix& o);
  Matrix& operator-=(const Matrix& o);
  Matrix& operator*=(double s);
  friend Matrix operator+(Matrix a, const Matrix& b) { return a += b; }
  friend Matrix operator-(Matrix a, const Matrix& b) { return a -= b; }
  friend Matrix operator*(Matrix a, double s) { return a *= s; }
  friend Matrix operator*(double s, Matrix a) { return a *= s; }

 private:
  int r_ = 0, c_ = 0;
  std::vector<double> v_;
};

Matrix matmul(const Matrix& a, const Matrix& b);
double frobenius_norm(const Matrix& a);
double frobenius_distance(const Matrix& a, const Matrix& b);
std::string format_double(double v);
void save_csv(const Matrix& m, std::ostream& out);
Matrix load_csv(std::istream& in);

// ---- RNG (reference: proj/include/lsp/rng.hpp:18-85); same streams ---------
class Rng {
 public:
  explicit Rng(uint64_t seed) : gen_(seed) {}
  uint64_t next_u64() { return gen_(); }
  double next_unit();
  uint64_t uniform_int(uint64_t n);
  double normal();
  double normal(double mean, double stddev) { return mean + stddev * normal(); }
  std::vector<int> sample_without_replacement(int n, int k);
  template <typename T>
  void shuffle(std::vector<T>& v) {
    for (std::size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[uniform_int(i)]);
  }

 private:
  std::mt19937_64 gen_;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

// ---- projectors (reference: proj/include/lsp/projector.hpp) ----------------
struct SparseProjector {
  int n_rows = 0;
  int d = 0;
  int r = 0;
  std::vector<int> positions;
  std::vector<double> values;
  int pos(int row, int slot) const { return positions[static_cast<std::size_t>(row) * r + slot]; }
  double val(int row, int slot) const { return values[static_cast<std::size_t>(row) * r + slot]; }
  double& val(int row, int slot) { return values[static_cast<std::size_t>(row) * r + slot]; }
};

struct ProjectorPair {
  SparseProjector p;
  SparseProjector q;
  std::int64_t birth_step = 0;
};

enum class RegKind { kSquared, kUnsquared };

struct FitConfig {
  double alpha = 0.1;
  double reg_beta = 0.0;
  double step_size = 1e-2;
  int max_steps = 500;
  int timeout_steps = 500;
  std::uint64_t seed = 0;
  RegKind reg_kind = RegKind::kSquared;
};

struct FitReport {
  std::vector<double> loss_curve;
  double final_rel_bias = 0.0;
  bool success = false;
  bool timed_out = false;
  bool stalled = false;
  int steps = 0;
};

struct FitGradient {
  std::vector<double> wrt_p;
  std::vector<double> wrt_q;
};

SparseProjector init_sparse(int n_rows, int d, int r, std::uint64_t seed);
SparseProjector identity_pattern(int n_rows);
Matrix to_dense(const SparseProjector& p);

Matrix left_mul(const SparseProjector& p, const Matrix& y);
Matrix leftT_mul(const SparseProjector& p, const Matrix& x);
Matrix right_mul(const Matrix& x, const SparseProjector& q);
Matrix rightT_mul(const Matrix& x, const SparseProjector& q);

Matrix compress(const ProjectorPair& pair, const Matrix& g);
Matrix decompress(const ProjectorPair& pair, const Matrix& s);
Matrix estimation_bias(const ProjectorPair& pair, const Matrix& sigma);
double relative_bias(const ProjectorPair& pair, const Matrix& sigma);

double fit_loss(const ProjectorPair& pair, const std::vector<Matrix>& targets,
                const FitConfig& cfg);
FitGradient fit_gradient(const ProjectorPair& pair, const std::vector<Matrix>& targets,
                         const FitConfig& cfg);
std::pair<ProjectorPair, FitReport> fit(const ProjectorPair& pair0,
                                        const std::vector<Matrix>& targets,
                                        const FitConfig& cfg);

void save_projector(const SparseProjector& p, std::ostream& out);
SparseProjector load_projector(std::istream& in);

// ---- subspace optimizer (reference: proj/include/lsp/subspace_opt.hpp) -----
struct SubspaceOptState {
  Matrix m;
  Matrix v;
  std::int64_t step = 0;
  double beta1 = 0.9;
  double beta2 = 0.999;
  double eps = 1e-8;
};

SubspaceOptState make_opt_state(int d, double beta1 = 0.9, double beta2 = 0.999,
                                double eps = 1e-8);
SubspaceOptState make_opt_state(int rows, int cols, double beta1, double beta2, double eps);

struct AdamResult {
  SubspaceOptState state;
  Matrix delta;
};
AdamResult adam_step(const SubspaceOptState& state, const Matrix& grad);

enum class TransferKind { kEntrywiseSquare, kMatrixSquare };
SubspaceOptState reproject_state(const SubspaceOptState& state, const ProjectorPair& old_pair,
                                 const ProjectorPair& new_pair,
                                 TransferKind kind = TransferKind::kEntrywiseSquare);
Matrix projector_gram(const SparseProjector& a, const SparseProjector& b);

void save_opt_state(const SubspaceOptState& s, std::ostream& out);
SubspaceOptState load_opt_state(std::istream& in);

}  // namespace lsp
