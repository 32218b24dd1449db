// Host-side projector construction and text I/O.
//
// Index generation must be bit-exact with the reference:
//   engine      std::mt19937_64 (standard-specified)           rng.hpp:18-20
//   integers    rejection sampling below UINT64_MAX - MAX % n   rng.hpp:30-37
//   positions   partial Fisher-Yates over [0,d), then ascending rng.hpp:60-70
//   values      Box-Muller N(0, 1/r), one spare cached          rng.hpp:40-55
//   per row: all r positions first, then r values              projector.cpp:76-83
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstring>
#include <numeric>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "host_projector.h"

namespace lspb {

uint64_t derive_seed(uint64_t master, uint64_t tag, uint64_t index) {
  auto mix = [](uint64_t x) {  // SplitMix64 finaliser, common.hpp:34-40
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
  };
  return mix(mix(master ^ mix(tag)) ^ index);
}

namespace {

class ProjectorRng {
 public:
  explicit ProjectorRng(uint64_t seed) : eng_(seed) {}

  uint64_t below(uint64_t n) {
    const uint64_t cap = UINT64_MAX - UINT64_MAX % n;
    for (;;) {
      const uint64_t x = eng_();
      if (x < cap) return x % n;
    }
  }

  double gaussian() {
    if (cached_) {
      cached_ = false;
      return cache_;
    }
    double u1 = unit();
    while (u1 <= 0.0) u1 = unit();
    const double u2 = unit();
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double th = 6.283185307179586476925286766559 * u2;
    cache_ = rad * std::sin(th);
    cached_ = true;
    return rad * std::cos(th);
  }

 private:
  double unit() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  std::mt19937_64 eng_;
  bool cached_ = false;
  double cache_ = 0.0;
};

}  // namespace

void init_sparse(int n_rows, int d, int r, uint64_t seed, int32_t* pos, double* val) {
  if (n_rows < 1 || r < 1 || r > d)
    fail(LSP_EINVAL, "init_sparse: need n_rows >= 1 and 1 <= r <= d");
  ProjectorRng rng(seed);
  const double sd = 1.0 / std::sqrt(static_cast<double>(r));
  std::vector<int32_t> pool(static_cast<size_t>(d));
  for (int row = 0; row < n_rows; ++row) {
    std::iota(pool.begin(), pool.end(), 0);
    for (int i = 0; i < r; ++i) {
      const int j = i + static_cast<int>(rng.below(static_cast<uint64_t>(d - i)));
      std::swap(pool[i], pool[j]);
    }
    int32_t* prow = pos + static_cast<size_t>(row) * r;
    std::copy(pool.begin(), pool.begin() + r, prow);
    std::sort(prow, prow + r);
    double* vrow = val + static_cast<size_t>(row) * r;
    for (int k = 0; k < r; ++k) vrow[k] = 0.0 + sd * rng.gaussian();
  }
}

void validate_projector(int n_rows, int d, int r, const int32_t* pos, const double* val,
                        int code) {
  if (n_rows < 1 || r < 1 || r > d) fail(code, "projector: invalid dimensions");
  for (int row = 0; row < n_rows; ++row)
    for (int k = 0; k < r; ++k) {
      const size_t i = static_cast<size_t>(row) * r + k;
      if (pos[i] < 0 || pos[i] >= d) fail(code, "projector: bad position");
      if (k > 0 && pos[i - 1] >= pos[i]) fail(code, "projector: positions not strictly ascending");
      if (!std::isfinite(val[i])) fail(code, "projector: non-finite value");
    }
}

static std::string shortest(double v) {
  char buf[32];
  auto res = std::to_chars(buf, buf + sizeof(buf), v);
  if (res.ec != std::errc()) fail(LSP_ENUMERIC, "format_double: conversion failed");
  return std::string(buf, res.ptr);
}

std::string save_projector_text(int n_rows, int d, int r, const int32_t* pos,
                                const double* val) {
  std::string out = std::to_string(n_rows) + ' ' + std::to_string(d) + ' ' + std::to_string(r) + '\n';
  for (int row = 0; row < n_rows; ++row) {
    const size_t base = static_cast<size_t>(row) * r;
    for (int k = 0; k < r; ++k) {
      if (k) out += ' ';
      out += std::to_string(pos[base + k]);
    }
    for (int k = 0; k < r; ++k) {
      out += ' ';
      out += shortest(val[base + k]);
    }
    out += '\n';
  }
  return out;
}

void load_projector_text(const std::string& text, int* n_rows, int* d, int* r, int32_t* pos,
                         double* val) {
  std::istringstream in(text);
  int nr = 0, dd = 0, rr = 0;
  if (!(in >> nr >> dd >> rr)) fail(LSP_EIO, "load_projector: bad header");
  if (nr < 1 || rr < 1 || rr > dd) fail(LSP_EIO, "load_projector: invalid dimensions in header");
  *n_rows = nr;
  *d = dd;
  *r = rr;
  if (!pos) return;
  for (int row = 0; row < nr; ++row) {
    const size_t base = static_cast<size_t>(row) * rr;
    for (int k = 0; k < rr; ++k) {
      int v;
      if (!(in >> v) || v < 0 || v >= dd) fail(LSP_EIO, "load_projector: bad position");
      if (k > 0 && pos[base + k - 1] >= v)
        fail(LSP_EIO, "load_projector: positions not strictly ascending");
      pos[base + k] = v;
    }
    for (int k = 0; k < rr; ++k) {
      double v;
      if (!(in >> v)) fail(LSP_EIO, "load_projector: bad value");
      if (!std::isfinite(v)) fail(LSP_EIO, "load_projector: non-finite value");
      val[base + k] = v;
    }
  }
}

int64_t subsample_size(double gamma, double beta, int m, int n, int total_steps,
                       double delta) {
  if (gamma <= 0.0 || beta <= 0.0 || m < 1 || n < 1 || total_steps < 1)
    fail(LSP_EINVAL, "subsample_size: inputs must be positive");
  if (delta <= 0.0 || delta >= 1.0) fail(LSP_EINVAL, "subsample_size: delta must be in (0, 1)");
  const double lead = 8.0 * gamma * gamma / (3.0 * beta * beta);
  const double raw = lead * std::log(static_cast<double>(m + n) * static_cast<double>(total_steps) / delta);
  if (raw >= 9.0e18) return 9000000000000000000LL;
  return static_cast<int64_t>(std::ceil(raw));
}

// CSC (column-major, rows ascending within a column) of a CSR projector.
void build_csc(int n_rows, int d, int r, const int32_t* pos, std::vector<int32_t>& ptr,
               std::vector<int32_t>& rows, std::vector<int32_t>& perm) {
  const size_t nnz = static_cast<size_t>(n_rows) * r;
  ptr.assign(static_cast<size_t>(d) + 1, 0);
  for (size_t i = 0; i < nnz; ++i) ptr[pos[i] + 1]++;
  for (int a = 0; a < d; ++a) ptr[a + 1] += ptr[a];
  std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
  rows.resize(nnz);
  perm.resize(nnz);
  for (int row = 0; row < n_rows; ++row)
    for (int k = 0; k < r; ++k) {
      const size_t i = static_cast<size_t>(row) * r + k;
      const int32_t t = fill[pos[i]]++;
      rows[t] = row;
      perm[t] = static_cast<int32_t>(i);
    }
}

// Chunk-major entry table for the compress stage-1 kernel: entries ordered by
// (row chunk of `bm` rows, column, row).  split[c*d + a] is the first entry of
// (chunk c, column a); split[nchunks*d] = total.  row_in_chunk = row - c*bm.
// Every (chunk, column) segment is padded to an EVEN length with a dummy
// entry (row 0 of the chunk, value 0, perm -1) so the kernel consumes two
// entries per 16-byte shared-memory load with no remainder branch.
void build_chunks(int n_rows, int d, int bm, const std::vector<int32_t>& csc_ptr,
                  const std::vector<int32_t>& csc_rows, const std::vector<int32_t>& csc_perm,
                  std::vector<int32_t>& split, std::vector<int32_t>& row_in_chunk,
                  std::vector<int32_t>& perm) {
  const int nchunks = ceil_div(n_rows, bm);
  const size_t nnz = csc_rows.size();
  split.assign(static_cast<size_t>(nchunks) * d + 1, 0);
  row_in_chunk.clear();
  perm.clear();
  row_in_chunk.reserve(nnz + nnz / 4 + d);
  perm.reserve(nnz + nnz / 4 + d);
  // cursor[a] walks column a's (row-sorted) entries chunk by chunk
  std::vector<int32_t> cursor(csc_ptr.begin(), csc_ptr.end() - 1);
  for (int c = 0; c < nchunks; ++c) {
    const int lim = (c + 1) * bm;
    for (int a = 0; a < d; ++a) {
      split[static_cast<size_t>(c) * d + a] = static_cast<int32_t>(perm.size());
      int32_t& cu = cursor[a];
      int cnt = 0;
      while (cu < csc_ptr[a + 1] && csc_rows[cu] < lim) {
        row_in_chunk.push_back(csc_rows[cu] - c * bm);
        perm.push_back(csc_perm[cu]);
        ++cu;
        ++cnt;
      }
      if (cnt & 1) {  // pad to even
        row_in_chunk.push_back(0);
        perm.push_back(-1);
      }
    }
  }
  split[static_cast<size_t>(nchunks) * d] = static_cast<int32_t>(perm.size());
}

void build_slots(int n_rows, int d, int bm, int K, int bpw, const std::vector<int32_t>& csc_ptr,
                 const std::vector<int32_t>& csc_rows, const std::vector<int32_t>& csc_perm,
                 SlotHost& out) {
  const int nchunks = ceil_div(n_rows, bm);
  const int dpad = static_cast<int>(round_up(d, 32));
  const int nw = dpad / bpw;
  const size_t nslots = static_cast<size_t>(nchunks) * dpad * K;
  out.slot_row.assign(nslots, -1);
  out.slot_perm.assign(nslots, -1);
  out.ovf_split.assign(static_cast<size_t>(nchunks) * nw + 1, 0);
  out.ovf_row.clear();
  out.ovf_bin.clear();
  out.ovf_perm.clear();
  std::vector<int32_t> cursor(csc_ptr.begin(), csc_ptr.end() - 1);
  for (int c = 0; c < nchunks; ++c) {
    const int lim = (c + 1) * bm;
    for (int a = 0; a < dpad; ++a) {
      if (a % bpw == 0)
        out.ovf_split[static_cast<size_t>(c) * nw + a / bpw] = static_cast<int32_t>(out.ovf_row.size());
      if (a >= d) continue;
      int32_t& cu = cursor[a];
      int t = 0;
      for (; cu < csc_ptr[a + 1] && csc_rows[cu] < lim; ++cu, ++t) {
        if (t < K) {
          const size_t s = (static_cast<size_t>(c) * dpad + a) * K + t;
          out.slot_row[s] = csc_rows[cu] - c * bm;
          out.slot_perm[s] = csc_perm[cu];
        } else {
          out.ovf_row.push_back(csc_rows[cu] - c * bm);
          out.ovf_bin.push_back(a % bpw);
          out.ovf_perm.push_back(csc_perm[cu]);
        }
      }
    }
  }
  out.ovf_split.back() = static_cast<int32_t>(out.ovf_row.size());
}

long long count_overflow(int n_rows, int d, int bm, int K, const std::vector<int32_t>& csc_ptr,
                         const std::vector<int32_t>& csc_rows) {
  long long ovf = 0;
  for (int a = 0; a < d; ++a) {
    int chunk = -1, t = 0;
    for (int e = csc_ptr[a]; e < csc_ptr[a + 1]; ++e) {
      const int c = csc_rows[e] / bm;
      if (c != chunk) chunk = c, t = 0;
      if (++t > K) ++ovf;
    }
  }
  (void)n_rows;
  return ovf;
}

}  // namespace lspb
