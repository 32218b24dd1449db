// Fused decompress-and-apply, TMA + mbarrier producer/consumer version (the
// fast path of launch_decompress_group; decompress.cu keeps the generic
// cp.async kernel for shapes TMA cannot describe).
//
//   warp 16, one lane : producer.  Per (matrix, band, 128-row block) tile it
//                       waits for the stage to be empty, then issues ONE 2-D
//                       TMA load of the W tile (32 cols x 128 rows, evict-first
//                       L2 policy) and two 1-D bulk copies of the tile rows'
//                       CSR entries of P, all completing on the stage's
//                       "full" mbarrier.
//   warps 0..15        : consumers.  Wait on "full", apply 8 rows each
//                       (4 conflict-free Y_band gathers + 1 FMA with W per
//                       element), store W, arrive on "empty".  A named barrier
//                       among the consumers guards the Y_band rebuild when the
//                       CTA moves to a new band.
// No block-wide barrier inside the streaming loop; 4 stages x 16 KB of W are
// in flight per SM.  Persistent, stream-K split of the tile list as in
// decompress.cu.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "core.cuh"
#include "tma.cuh"

namespace lspb {

bool encode_tmap_2d(CUtensorMap* map, const void* base, lsp_dtype dt, long long rows,
                    long long cols, long long ld_elems, int box_cols, int box_rows, bool swz128) {
  static PFN_cuTensorMapEncodeTiled encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }();
  if (!encode) return false;
  const size_t es = dtype_size(dt);
  if (reinterpret_cast<uintptr_t>(base) % 16 || (ld_elems * es) % 16) return false;
  CUtensorMapDataType t = dt == LSP_F64   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                          : dt == LSP_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                          : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_elems * es)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  const CUresult rc = encode(map, t, 2, const_cast<void*>(base), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE,
                             swz128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return rc == CUDA_SUCCESS;
}

namespace {
struct MapKey {
  const void* p;
  long long rows, cols, ld;
  int dt, bc, br, swz;
  bool operator<(const MapKey& o) const {
    return std::tie(p, rows, cols, ld, dt, bc, br, swz) <
           std::tie(o.p, o.rows, o.cols, o.ld, o.dt, o.bc, o.br, o.swz);
  }
};

}  // namespace

bool cached_tmap(CUtensorMap* out, const void* base, lsp_dtype dt, long long rows, long long cols,
                 long long ld, int bc, int br, bool swz128) {
  static std::mutex mu;
  static std::map<MapKey, CUtensorMap> cache;
  const MapKey k{base, rows, cols, ld, static_cast<int>(dt), bc, br, swz128 ? 1 : 0};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(k);
  if (it != cache.end()) {
    *out = it->second;
    return true;
  }
  if (!encode_tmap_2d(out, base, dt, rows, cols, ld, bc, br, swz128)) return false;
  if (cache.size() > 4096) cache.clear();
  cache.emplace(k, *out);
  return true;
}

namespace {

constexpr int kTRows = 128;   // W rows per stage
constexpr int kTStages = 4;   // ring depth
constexpr int kConsumers = 16;
constexpr int kTThreads = (kConsumers + 1) * 32;
constexpr int kKR = 4;        // nonzeros per projector row handled by this path

struct alignas(64) TMat {
  CUtensorMap tmap;  // W (input) tile map: box BN x kTRows
  int m, n;
  const int* ppos_scaled;  // P positions * (BN+1) * sizeof(Tacc): Y_band row byte offsets
  const void* pval;
  const int* qpos;
  const void* qval;
  const void* dT;
  void* out;
  long long ldo;
  int row_blocks, nbands;
  long long tile_end;
};
struct TArgs {
  TMat mat[kMaxGroup];
  int count, d;
  long long total;
  double alpha, beta;
  const int* skip;
};

__device__ __forceinline__ float lds_f(unsigned addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ double lds_d(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

struct TCursor {
  int mi, band, rb;
};
__device__ __forceinline__ TCursor tcursor_at(const TArgs& A, long long t) {
  int i = 0;
  while (i + 1 < A.count && t >= A.mat[i].tile_end) ++i;
  const long long lt = t - (i ? A.mat[i - 1].tile_end : 0);
  return TCursor{i, static_cast<int>(lt / A.mat[i].row_blocks),
                 static_cast<int>(lt % A.mat[i].row_blocks)};
}
__device__ __forceinline__ void tadvance(const TArgs& A, TCursor& c) {
  if (++c.rb == A.mat[c.mi].row_blocks) {
    c.rb = 0;
    if (++c.band == A.mat[c.mi].nbands) {
      c.band = 0;
      ++c.mi;
    }
  }
}

template <typename Tw, typename Tacc, int BN>
struct TLayout {
  int d;
  __host__ __device__ int y_bytes() const { return (d * (BN + 1) * (int)sizeof(Tacc) + 127) & ~127; }
  static constexpr int w_bytes() { return kTRows * BN * (int)sizeof(Tw); }
  static constexpr int pos_bytes() { return kTRows * kKR * 4; }
  static constexpr int val_bytes() { return kTRows * kKR * (int)sizeof(Tacc); }
  static constexpr int stage_bytes() { return (w_bytes() + pos_bytes() + val_bytes() + 127) & ~127; }
  __host__ __device__ int bar_offset() const { return y_bytes() + kTStages * stage_bytes(); }
  __host__ __device__ int total() const { return bar_offset() + 2 * kTStages * 8; }
};

template <typename Tw, typename Tacc, int BN, bool USE_IN>
__global__ void __launch_bounds__(kTThreads, 1) k_decompress_tma(const __grid_constant__ TArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  if (A.skip && *A.skip) return;
  const TLayout<Tw, Tacc, BN> L{A.d};
  constexpr int LDY = BN + 1;
  Tacc* Y = reinterpret_cast<Tacc*>(smem_raw);
  unsigned char* ring = smem_raw + L.y_bytes();
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem_raw + L.bar_offset());
  unsigned long long* empty = full + kTStages;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = A.d;

  const long long t_begin = A.total * blockIdx.x / gridDim.x;
  const long long t_end = A.total * (blockIdx.x + 1) / gridDim.x;
  const int ntiles = static_cast<int>(t_end - t_begin);

  if (tid == 0) {
    for (int s = 0; s < kTStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kConsumers);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (ntiles <= 0) return;

  if (warp == kConsumers) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const unsigned long long pol = policy_evict_first();
      TCursor c = tcursor_at(A, t_begin);
      for (int s = 0; s < ntiles; ++s, tadvance(A, c)) {
        const int st = s % kTStages;
        if (s >= kTStages) mbar_wait(empty + st, ((s / kTStages) - 1) & 1);
        const TMat& M = A.mat[c.mi];
        const int r0 = c.rb * kTRows;
        const int nrows = min(kTRows, M.m - r0);
        unsigned char* base = ring + st * L.stage_bytes();
        const unsigned pbytes = nrows * kKR * 4, vbytes = nrows * kKR * sizeof(Tacc);
        mbar_arrive_expect_tx(full + st, (USE_IN ? L.w_bytes() : 0) + pbytes + vbytes);
        if (USE_IN) tma_load_2d(base, &M.tmap, c.band * BN, r0, full + st, pol);
        bulk_load(base + L.w_bytes(), M.ppos_scaled + static_cast<long long>(r0) * kKR, pbytes,
                  full + st);
        bulk_load(base + L.w_bytes() + L.pos_bytes(),
                  static_cast<const Tacc*>(M.pval) + static_cast<long long>(r0) * kKR, vbytes,
                  full + st);
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const Tacc alpha = static_cast<Tacc>(A.alpha), beta = static_cast<Tacc>(A.beta);
  auto build_y = [&](const TMat& M, int band) {
    const Tacc* qval = static_cast<const Tacc*>(M.qval);
    const Tacc* dT = static_cast<const Tacc*>(M.dT);
    const int j0 = band * BN;
    for (int jj = warp; jj < BN; jj += kConsumers) {
      const int j = j0 + jj;
      for (int a0 = 0; a0 < d; a0 += 32 * 32) {
        Tacc y[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) y[t] = Tacc(0);
        if (j < M.n) {
#pragma unroll
          for (int l = 0; l < kKR; ++l) {
            const int b = __ldg(M.qpos + static_cast<long long>(j) * kKR + l);
            const Tacc q = __ldg(qval + static_cast<long long>(j) * kKR + l);
            const Tacc* row = dT + static_cast<long long>(b) * d + a0 + lane;
#pragma unroll
            for (int t = 0; t < 32; ++t)
              if (a0 + lane + 32 * t < d) y[t] = fma(q, row[32 * t], y[t]);
          }
        }
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const int a = a0 + lane + 32 * t;
          if (a < d) Y[a * LDY + jj] = y[t];
        }
      }
    }
  };

  constexpr int RPW = 32 / BN;                    // rows per warp instruction
  constexpr int kIters = kTRows / (kConsumers * RPW);
  const int jj = lane % BN, rsub = lane / BN;
  // byte address of Y_band[0][jj]; rows of Y_band are LDY*sizeof(Tacc) bytes apart
  const unsigned y_lane = smem_addr(Y) + jj * static_cast<unsigned>(sizeof(Tacc));
  TCursor c = tcursor_at(A, t_begin);
  int cur_band = -1, cur_mat = -1;
  for (int s = 0; s < ntiles; ++s, tadvance(A, c)) {
    const TMat& M = A.mat[c.mi];
    if (c.band != cur_band || c.mi != cur_mat) {
      named_barrier_sync(1, kConsumers * 32);  // all consumers done with the old Y_band
      build_y(M, c.band);
      named_barrier_sync(1, kConsumers * 32);
      cur_band = c.band;
      cur_mat = c.mi;
    }
    const int st = s % kTStages;
    const int r0 = c.rb * kTRows;
    const int nrows = min(kTRows, M.m - r0);
    const int j = c.band * BN + jj;
    const long long ldo = M.ldo;
    Tw* const out = static_cast<Tw*>(M.out);
    const bool col_ok = j < M.n;
    mbar_wait(full + st, (s / kTStages) & 1);
    const unsigned char* base = ring + st * L.stage_bytes();
    const Tw* wt = reinterpret_cast<const Tw*>(base);
    // P entries of the tile, already scaled to Y_band row byte offsets
    const int* ps = reinterpret_cast<const int*>(base + L.w_bytes());
    const Tacc* vs = reinterpret_cast<const Tacc*>(base + L.w_bytes() + L.pos_bytes());
    if (col_ok) {
      const int q0 = warp * RPW + rsub;
      Tw* orow = out + static_cast<long long>(r0 + q0) * ldo + j;
      const long long ostep = static_cast<long long>(kConsumers * RPW) * ldo;
      auto row = [&](int q, Tw* o) {
        const int4 pp = *reinterpret_cast<const int4*>(ps + q * kKR);
        Tacc acc;
        if constexpr (sizeof(Tacc) == 4) {
          const float4 vv = *reinterpret_cast<const float4*>(vs + q * kKR);
          acc = vv.x * lds_f(y_lane + pp.x);
          acc = fma(vv.y, lds_f(y_lane + pp.y), acc);
          acc = fma(vv.z, lds_f(y_lane + pp.z), acc);
          acc = fma(vv.w, lds_f(y_lane + pp.w), acc);
        } else {
          acc = vs[q * kKR] * lds_d(y_lane + pp.x);
          acc = fma(vs[q * kKR + 1], lds_d(y_lane + pp.y), acc);
          acc = fma(vs[q * kKR + 2], lds_d(y_lane + pp.z), acc);
          acc = fma(vs[q * kKR + 3], lds_d(y_lane + pp.w), acc);
        }
        Tacc res = alpha * acc;
        if (USE_IN) res = fma(beta, cvt<Tacc>(wt[q * BN + jj]), res);
        *o = cvt<Tw>(res);
      };
      if (nrows == kTRows) {
#pragma unroll
        for (int u = 0; u < kIters; ++u) row(q0 + u * kConsumers * RPW, orow + u * ostep);
      } else {
#pragma unroll 1
        for (int u = 0; u < kIters; ++u) {
          const int q = q0 + u * kConsumers * RPW;
          if (q < nrows) row(q, orow + u * ostep);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);
  }
}

template <typename Tw, typename Tacc, int BN>
bool tma_impl(const std::vector<DecJob>& jobs, double alpha, double beta, const int* skip,
              cudaStream_t st) {
  const Pair& p0 = *jobs[0].pr;
  const TLayout<Tw, Tacc, BN> L{p0.d};
  if (L.total() > 227 * 1024) return false;
  const bool use_in = beta != 0.0;
  TArgs A{};
  A.count = static_cast<int>(jobs.size());
  A.d = p0.d;
  A.alpha = alpha;
  A.beta = beta;
  A.skip = skip;
  long long total = 0;
  for (size_t i = 0; i < jobs.size(); ++i) {
    const DecJob& J = jobs[i];
    const Pair& pr = *J.pr;
    if (pr.p->r != kKR || pr.q->r != kKR) return false;
    if (use_in && J.in == nullptr) return false;
    if (reinterpret_cast<uintptr_t>(pr.p->val.p) % 16) return false;
    TMat& M = A.mat[i];
    if (use_in && !cached_tmap(&M.tmap, J.in, std::is_same<Tw, double>::value  ? LSP_F64
                                              : std::is_same<Tw, float>::value ? LSP_F32
                                                                               : LSP_BF16,
                               pr.m, pr.n, J.ldi, BN, kTRows))
      return false;
    M.m = pr.m, M.n = pr.n;
    M.ppos_scaled = pr.p->scaled_pos((BN + 1) * static_cast<int>(sizeof(Tacc)));
    M.pval = pr.p->val.p;
    M.qpos = pr.q->pos.as<int>(), M.qval = pr.q->val.p;
    M.dT = J.delta_t;
    M.out = J.out, M.ldo = J.ldo;
    M.row_blocks = ceil_div(pr.m, kTRows);
    M.nbands = ceil_div(pr.n, BN);
    total += static_cast<long long>(M.nbands) * M.row_blocks;
    M.tile_end = total;
  }
  A.total = total;
  if (total == 0) return true;
  const int smem = L.total();
  auto kern = use_in ? k_decompress_tma<Tw, Tacc, BN, true> : k_decompress_tma<Tw, Tacc, BN, false>;
  LSP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid = static_cast<int>(std::min<long long>(total, sm_budget(kBudgetUpdate)));
  kern<<<grid, kTThreads, smem, st>>>(A);
  after_launch("decompress_tma");
  return true;
}

}  // namespace

bool launch_decompress_group_tma(const std::vector<DecJob>& jobs, lsp_dtype dt, double alpha,
                                 double beta, const int* skip_flag, cudaStream_t st) {
  if (jobs.empty() || jobs.size() > static_cast<size_t>(kMaxGroup)) return false;
  const Pair& p0 = *jobs[0].pr;
  bool ok = false;
  LSP_DISPATCH_ACC(p0.compute, Tacc, {
    LSP_DISPATCH_STORAGE(dt, Tw, {
      const TLayout<Tw, Tacc, 32> L32{p0.d};
      const TLayout<Tw, Tacc, 16> L16{p0.d};
      if (L32.total() <= 227 * 1024)
        ok = tma_impl<Tw, Tacc, 32>(jobs, alpha, beta, skip_flag, st);
      else if (L16.total() <= 227 * 1024)
        ok = tma_impl<Tw, Tacc, 16>(jobs, alpha, beta, skip_flag, st);
    })
  })
  return ok;
}

}  // namespace lspb
