// Internal handle types and kernel launchers.
#pragma once

#include <memory>
#include <vector>

#include "common.cuh"

namespace lspb {

// Owning device allocation (move-only).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr, o.bytes = 0; }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  // Grow-only reallocation (contents are not preserved).
  void ensure(size_t n) {
    if (n <= bytes) return;
    release();
    LSP_CUDA(cudaMalloc(&p, n));
    bytes = n;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Entry of the chunk-major stage-1 table: byte offset of the entry's row in
// the shared-memory G tile (row_in_chunk * 32 * sizeof(Tin)) and value.
struct __align__(8) EntryF {
  int32_t off;
  float val;
};
struct __align__(16) EntryD {
  int32_t off;
  int32_t pad;
  double val;
};
template <typename Tacc>
struct EntryOf;
template <>
struct EntryOf<float> {
  using type = EntryF;
};
template <>
struct EntryOf<double> {
  using type = EntryD;
};

struct ChunkTable {
  int bm = 0;
  int esize = 0;  // sizeof(Tin) the byte offsets were scaled for
  int nchunks = 0;
  long long count = 0;  // entries incl. even-length padding
  DevBuf split;  // int32 [nchunks*d + 1]
  DevBuf ent;    // EntryF / EntryD [nnz]
  DevBuf perm;   // int32 [count] -> CSR index (-1 for padding), for value refresh
};

// Fixed-slot stage-1 table (see build_slots): K slots per (chunk, bin), an
// overflow list per (chunk, 32-bin group).  Padding slots point at the zero
// row that follows the bm-row G tile in shared memory.
struct SlotTable {
  int bm = 0, row_bytes = 0, K = 0, bpw = 0, nchunks = 0, dpad = 0;
  long long nslots = 0, novf = 0;
  DevBuf slots;      // EntryF [nchunks][dpad][K]: off = tile byte offset, val
  DevBuf perm;       // int32 [nslots] -> CSR index (-1: padding)
  DevBuf ovf_split;  // int32 [nchunks*dpad/bpw + 1]
  DevBuf ovf;        // EntryF [novf]: off | (bin % bpw) << 27, val
  DevBuf ovf_perm;   // int32 [novf]
};
// Byte offset of the zero row (= bytes of a bm-row tile, 128-aligned).
inline int slot_zero_off(int bm, int row_bytes) {
  return static_cast<int>(round_up(static_cast<long long>(bm) * row_bytes, 128));
}

// Device-resident SparseProjector (proj/include/lsp/projector.hpp:18-30) in
// CSR (row-major positions/values, the reference layout) and CSC orientation.
struct Projector {
  int n_rows = 0, d = 0, r = 0;
  lsp_dtype compute = LSP_F32;
  std::vector<int32_t> h_pos;
  std::vector<double> h_val;
  std::vector<int32_t> h_csc_ptr, h_csc_rows, h_csc_perm;
  DevBuf pos, val;                           // CSR: int32 / compute [n_rows*r]
  DevBuf csc_ptr, csc_row, csc_val, csc_perm;  // CSC: [d+1], [nnz], [nnz], [nnz]
  std::vector<std::unique_ptr<ChunkTable>> chunks;
  std::vector<std::unique_ptr<SlotTable>> slot_tables;
  std::vector<std::pair<std::pair<int, int>, long long>> ovf_counts;  // (K, bm) -> overflow

  size_t nnz() const { return static_cast<size_t>(n_rows) * r; }
  size_t vsize() const { return dtype_size(compute); }
  const ChunkTable& chunk_table(int bm, int esize);
  const SlotTable& slot_table(int bm, int row_bytes, int K, int bpw);
  long long overflow(int K, int bm);
  // CSR positions multiplied by `scale` (cached per scale), for kernels that
  // index shared-memory rows by byte offset.
  const int* scaled_pos(int scale);
  // CSC entries packed as {row, value} (fp32 compute only), built on first use
  // and kept current by refresh_values.
  const EntryF* csc_entries();
  DevBuf csc_ent;
  // CSC entries with every bin padded to a multiple of kPadU entries (pads:
  // the bin's last row, value 0, perm -1) for the gather-form compress;
  // EntryF for fp32 projectors, EntryD for fp64.
  static constexpr int kPadU = 8;
  struct PadTable {
    DevBuf ptr, ent, perm;
    long long count = 0;
    std::vector<int32_t> h_ptr;
  };
  std::unique_ptr<PadTable> csc_pad;
  const PadTable& csc_padded();
  std::vector<std::pair<int, std::unique_ptr<DevBuf>>> scaled;
  // Re-derive CSC and chunk-table values from the CSR values on the device.
  void refresh_values(cudaStream_t st);
  void upload_values();  // h_val -> device CSR values, then refresh
};

struct Pair {
  Projector* p = nullptr;
  Projector* q = nullptr;
  int m = 0, n = 0, d = 0;
  lsp_dtype compute = LSP_F32;
  DevBuf zt;    // n x ldz, compute   (stage-1 output Z^T = G^T P)
  DevBuf s_t;   // d x d,  compute    (S^T)
  DevBuf d_t;   // d x d,  compute    (delta^T or transposed input)
  DevBuf red;   // double partial sums
  DevBuf flag;  // int
  mutable DevBuf yb;  // float [nbands][d][BN]: Y = delta Q^T, band-blocked (apply.cu)
  void yb_ensure(size_t bytes) const { yb.ensure(bytes); }
  mutable DevBuf xs, drow;  // X = P delta (row-swizzled) and delta row-major (apply_x.cu)
  void xs_ensure(size_t xbytes, size_t dbytes) const {
    xs.ensure(xbytes);
    drow.ensure(dbytes);
  }
  int ldz() const { return static_cast<int>(round_up(d, 4)); }
  int* flag_ptr();
};

struct Adam {
  int rows = 0, cols = 0;
  double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
  lsp_dtype compute = LSP_F32;
  lsp_layout layout = LSP_LAYOUT_T;
  DevBuf m, v;
  DevBuf flag;   // int: latched non-finite gradient
  DevBuf dstep;  // int64: step counter, advanced on the device (graph-replay safe)
  DevBuf done;   // unsigned: blocks finished in the current Adam launch
  // Ping-pong moments (layer state only; empty otherwise): int `cur` on the
  // device selects (m, v) or (m2, v2).  k_adam updates the current pair in
  // place; the stage-2 + Adam kernel writes the other pair and its last block
  // flips `cur` only when the layer's S was finite, so a skipped step leaves
  // the moments untouched exactly like k_adam's early return.
  DevBuf m2, v2, cur;
  size_t count() const { return static_cast<size_t>(rows) * cols; }
};

constexpr int kMaxGroup = 16;  // matrices per grouped launch (one layer)

// One matrix of a grouped compress.
struct S1Job {
  const Pair* pr;
  const void* g;
  long long ldg;
  void* zt;   // n x ldz workspace (compute dtype)
  void* s_t;  // d x d output S^T (compute dtype)
};

// One matrix of a grouped decompress: out = beta*in + alpha * P delta Q^T.
struct DecJob {
  const Pair* pr;
  const void* delta_t;  // d x d, ld d
  const void* in;
  long long ldi;
  void* out;
  long long ldo;
};

// ---- launchers (templated kernels live in the .cu files) -------------------
// Z^T = G^T P (n x ldz) with the chunked register-accumulator kernel.
void launch_compress_stage1(const Pair& pr, const void* g, long long ldg, lsp_dtype gdt,
                            void* zt, cudaStream_t st);
void launch_compress_stage1_group(const std::vector<S1Job>& jobs, lsp_dtype gdt,
                                  cudaStream_t st);
// Fixed-slot TMA variant (compress_slots.cu); false if the group is not eligible.
bool launch_compress_slots_group(const std::vector<S1Job>& jobs, lsp_dtype gdt, cudaStream_t st);
// Gather-form kernel (compress_spmm.cu); false if the group is not eligible.
bool launch_compress_spmm_group(const std::vector<S1Job>& jobs, lsp_dtype gdt, cudaStream_t st);
void launch_stage2_group(const std::vector<S1Job>& jobs, int* flag, cudaStream_t st);
void compress_group_T(const std::vector<S1Job>& jobs, lsp_dtype gdt, int* flag,
                      cudaStream_t st);
// out[r][:] = beta*in[r][:] + alpha * sum_t val[t] * src[idx[t]][:]
// Rows' entries are [ptr[r], ptr[r+1]) when ptr != nullptr, else [r*k, r*k+k).
void launch_gather(int R, int c, const int* ptr, int k, const int* idx, const void* val,
                   lsp_dtype acc, const void* src, long long lds, lsp_dtype src_dt,
                   const void* in, long long ldi, void* out, long long ldo, lsp_dtype out_dt,
                   double alpha, double beta, DevBuf* partials, int* nparts, cudaStream_t st);
// fp64 batch of row gathers through one projector (operand b at base + b * stride)
void launch_gather_f64_batch(int R, int c, const int* ptr, int k, const int* idx, const double* val,
                             const double* src, long long lds, long long sbs, const double* in,
                             long long ldi, long long ibs, double* out, long long ldo, long long obs,
                             int nb, double alpha, double beta, cudaStream_t st);
void launch_transpose_batch(int rows, int cols, const double* src, long long lds, long long sbs,
                            double* dst, long long ldd, long long dbs, int nb, cudaStream_t st);
void launch_transpose(int rows, int cols, const void* src, long long lds, void* dst,
                      long long ldd, lsp_dtype dt, cudaStream_t st);
// Fused decompress: out = beta*in + alpha * P (delta) Q^T, delta given as delta^T.
void launch_decompress(const Pair& pr, const void* delta_t, const void* in, long long ldi,
                       void* out, long long ldo, lsp_dtype dt, double alpha, double beta,
                       const int* skip_flag, DevBuf* partials, int* nparts, cudaStream_t st);
// TMA/mbarrier fast path; returns false when the shapes or pointers do not allow it.
bool launch_decompress_group_tma(const std::vector<DecJob>& jobs, lsp_dtype dt, double alpha,
                                 double beta, const int* skip_flag, cudaStream_t st);
// Y-precompute + streaming apply (apply.cu); false when not eligible.  phase:
// both kernels, only the Y build, or only the apply (after a Y build of the
// same group on the same stream).
constexpr int kPhaseBuild = 1, kPhaseApply = 2, kPhaseBoth = 3;
// Does this matrix go through launch_decompress_group_y (row or column form)?
bool decompress_fast_eligible(const DecJob& J, lsp_dtype dt, double beta);
// fp64 Y path (apply_f64.cu): per-matrix eligibility, and the group launch.
bool y64_eligible(const DecJob& J, lsp_dtype dt, double beta);
void launch_y64_group(const std::vector<DecJob>& jobs, double alpha, double beta, const int* skip,
                      cudaStream_t st, int phase);
// Row-orientation apply (apply_x.cu) for n > m matrices.
bool apply_x_eligible(const DecJob& J, lsp_dtype dt, double beta);
void launch_apply_x(const std::vector<DecJob>& jobs, double alpha, double beta,
                    const int* skip_flag, cudaStream_t st, int phase);
bool launch_decompress_group_y(const std::vector<DecJob>& jobs, lsp_dtype dt, double alpha,
                               double beta, const int* skip_flag, cudaStream_t st,
                               int phase = kPhaseBoth);
void launch_decompress_group(const std::vector<DecJob>& jobs, lsp_dtype dt, double alpha,
                             double beta, const int* skip_flag, DevBuf* partials, int* nparts,
                             cudaStream_t st);
// checked: fused finiteness check of `grad` (ping-pong state only, see Adam::cur)
void launch_adam(Adam& a, const void* grad, void* delta, const int* skip_flag, cudaStream_t st,
                 bool checked = false);
const double2* correction_table(double b1, double b2, long long* cap);
// Stage 2 with the layer's Adam fused into its epilogue (fp32, ping-pong
// moments); false (nothing launched) when the group is not eligible.
bool launch_stage2_adam_group(const std::vector<S1Job>& jobs, const void* s_base, Adam& a,
                              void* delta, int* flag, cudaStream_t st);
void launch_check_finite(size_t cnt, const void* x, lsp_dtype dt, int* flag, cudaStream_t st);
void launch_convert(size_t cnt, const void* src, lsp_dtype sdt, void* dst, lsp_dtype ddt,
                    cudaStream_t st);
void launch_convert2d(int rows, int cols, const void* src, long long lds, lsp_dtype sdt,
                      void* dst, long long ldd, lsp_dtype ddt, cudaStream_t st);
// deterministic sum of `n` doubles on device -> host value (synchronous)
double reduce_partials_sync(const double* partials, int n, cudaStream_t st);
double sumsq_sync(Pair& pr, int rows, int cols, const void* x, long long ld, lsp_dtype dt,
                  cudaStream_t st);
void launch_refresh_values(const Projector& p, cudaStream_t st);

// High-level building blocks used by the C-ABI.
void compress_T(Pair& pr, const void* g, long long ldg, lsp_dtype gdt, void* s_t,
                cudaStream_t st, int* flag = nullptr);
const void* delta_as_T(Pair& pr, const void* s, lsp_layout layout, cudaStream_t st);

}  // namespace lspb
