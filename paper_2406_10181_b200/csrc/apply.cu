// Fused decompress-and-apply, two-kernel form for fp32 accumulation
// (reference: rightT_mul proj/src/projector.cpp:148-161, left_mul :105-117,
//  decompress :170-175, apply W -= lr * decompress proj/src/trainer.cpp:190):
//
//   out = beta * in + alpha * P (Delta Q^T)
//
// 1. k_build_y: Y = Delta Q^T (d x n) is computed ONCE per matrix into a
//    band-blocked workspace Yb[band][a][jj] (BN columns per band, so every
//    band is one contiguous d x BN block).  Y[a][j] = sum_l q(j,l) *
//    Delta^T[pos_q(j,l)][a]: row gathers of the L2-resident Delta^T, 128-byte
//    coalesced per warp, the l-sum in the reference's order.
// 2. k_apply_y: persistent streaming kernel, one CTA per SM, stream-K split
//    of the (matrix, band, row-block) tile list.  Warp 0 streams W tiles (2-D
//    TMA, evict-first) and the tile rows' CSR entries of P (bulk copies)
//    through an S-stage mbarrier ring; warp 1 bulk-copies the band's Y block
//    into shared memory whenever the CTA enters a new band (no arithmetic,
//    no block-wide barrier); 16 consumer warps do, per W element, k
//    conflict-free shared-memory gathers Y[pos_p(i,l)][jj] and one
//    read-modify-write of W.  W is read and written exactly once.
//
// Compared with building Y_band inside the apply kernel (decompress_tma.cu),
// the per-band cost drops from r*BN row gathers of Delta^T (512 KB of L2
// traffic plus the FMAs, during which the W stream stalls) to one 128 KB bulk
// copy that overlaps the ring.  Arithmetic and summation order are unchanged,
// so results are bitwise those of the other decompress kernels.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "core.cuh"
#include "tma.cuh"

#ifndef LSP_APPLY_TILE_F32
#define LSP_APPLY_TILE_F32 8192
#endif

namespace lspb {

namespace {

constexpr int kYMaxBytes = 160 * 1024;  // Y block of one band in shared memory
constexpr int kSmemMax = 227 * 1024;
constexpr int kNC = 16;                 // consumer warps
constexpr int kNG = 2;                  // consumer groups
constexpr int kAThreads = (kNC + 2) * 32;
constexpr int kMaxStages = 16;
constexpr int kYChunk = 16 * 1024;      // bulk-copy granule for the Y block
// W bytes per ring tile (BN x TR elements): smaller fp32 tiles keep more of the
// ring in flight while two tiles are being consumed (C4 apply 10.1 ms per step
// with 8 KB vs 10.4 with 16 KB); bf16 measured faster with 16 KB (6.8 vs 7.2).
template <typename Tw>
constexpr int tile_bytes() { return sizeof(Tw) == 4 ? LSP_APPLY_TILE_F32 : 16384; }


// A projector row's (or column's) KR entries, read with the widest vectors KR
// allows (KR in {2, 4, 8}); order is the reference's l = 0 .. KR-1.
template <int KR>
struct Ent {
  int p[KR];
  float v[KR];
};
template <int KR>
__device__ __forceinline__ Ent<KR> ent_ldg(const int* pp, const float* vp) {
  Ent<KR> e;
  if constexpr (KR == 2) {
    const int2 a = __ldg(reinterpret_cast<const int2*>(pp));
    const float2 b = __ldg(reinterpret_cast<const float2*>(vp));
    e.p[0] = a.x, e.p[1] = a.y, e.v[0] = b.x, e.v[1] = b.y;
  } else {
#pragma unroll
    for (int l = 0; l < KR; l += 4) {
      const int4 a = __ldg(reinterpret_cast<const int4*>(pp + l));
      const float4 b = __ldg(reinterpret_cast<const float4*>(vp + l));
      e.p[l] = a.x, e.p[l + 1] = a.y, e.p[l + 2] = a.z, e.p[l + 3] = a.w;
      e.v[l] = b.x, e.v[l + 1] = b.y, e.v[l + 2] = b.z, e.v[l + 3] = b.w;
    }
  }
  return e;
}
template <int KR>
__device__ __forceinline__ Ent<KR> ent_gen(const int* pp, const float* vp) {  // shared via generic
  Ent<KR> e;
  if constexpr (KR == 2) {
    const int2 a = *reinterpret_cast<const int2*>(pp);
    const float2 b = *reinterpret_cast<const float2*>(vp);
    e.p[0] = a.x, e.p[1] = a.y, e.v[0] = b.x, e.v[1] = b.y;
  } else {
#pragma unroll
    for (int l = 0; l < KR; l += 4) {
      const int4 a = *reinterpret_cast<const int4*>(pp + l);
      const float4 b = *reinterpret_cast<const float4*>(vp + l);
      e.p[l] = a.x, e.p[l + 1] = a.y, e.p[l + 2] = a.z, e.p[l + 3] = a.w;
      e.v[l] = b.x, e.v[l + 1] = b.y, e.v[l + 2] = b.z, e.v[l + 3] = b.w;
    }
  }
  return e;
}

// ---------------------------------------------------------------------------
// Y build
// ---------------------------------------------------------------------------
struct YMat {
  const int* qpos;
  const float* qval;
  const float* dT;  // Delta^T: element (a, b) of Delta at b*d + a
  float* yb;
  int n, nbands;
  long long task_end;
};
struct YArgs {
  YMat mat[kMaxGroup];
  int count, d, ablocks;
  long long total;
  const int* skip;
};

// One warp = one (matrix, band, 64-row block of a).  Lane owns a0+lane and
// a0+32+lane; the band's BN columns are unrolled into registers so every
// output row segment (BN floats) is written with contiguous 16-byte stores.
template <int BN, int KR>
__global__ void __launch_bounds__(256) k_build_y(const __grid_constant__ YArgs A) {
  if (A.skip && *A.skip) return;
  const int lane = threadIdx.x & 31;
  const long long task = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (task >= A.total) return;
  int mi = 0;
  while (mi + 1 < A.count && task >= A.mat[mi].task_end) ++mi;
  const YMat& M = A.mat[mi];
  const long long lt = task - (mi ? A.mat[mi - 1].task_end : 0);
  const int band = static_cast<int>(lt / A.ablocks);
  const int a0 = static_cast<int>(lt % A.ablocks) * 64;
  const int d = A.d;
  const int a_lo = a0 + lane, a_hi = a0 + 32 + lane;
  const bool ok_lo = a_lo < d, ok_hi = a_hi < d;
  float y0[BN], y1[BN];
#pragma unroll
  for (int jj = 0; jj < BN; ++jj) {
    y0[jj] = 0.0f;
    y1[jj] = 0.0f;
    const int j = band * BN + jj;
    if (j < M.n) {
      const Ent<KR> en = ent_ldg<KR>(M.qpos + static_cast<long long>(j) * KR,
                                     M.qval + static_cast<long long>(j) * KR);
      const int* p = en.p;
      const float* q = en.v;
#pragma unroll
      for (int l = 0; l < KR; ++l) {
        const float* row = M.dT + static_cast<long long>(p[l]) * d;
        if (ok_lo) y0[jj] = fmaf(q[l], __ldg(row + a_lo), y0[jj]);
        if (ok_hi) y1[jj] = fmaf(q[l], __ldg(row + a_hi), y1[jj]);
      }
    }
  }
  float* base = M.yb + static_cast<long long>(band) * d * BN;
  if (ok_lo) {
    float4* o = reinterpret_cast<float4*>(base + static_cast<long long>(a_lo) * BN);
#pragma unroll
    for (int t = 0; t < BN / 4; ++t)
      o[t] = make_float4(y0[4 * t], y0[4 * t + 1], y0[4 * t + 2], y0[4 * t + 3]);
  }
  if (ok_hi) {
    float4* o = reinterpret_cast<float4*>(base + static_cast<long long>(a_hi) * BN);
#pragma unroll
    for (int t = 0; t < BN / 4; ++t)
      o[t] = make_float4(y1[4 * t], y1[4 * t + 1], y1[4 * t + 2], y1[4 * t + 3]);
  }
}

// Shared-memory form (d <= kDsMaxD): a CTA stages the 32 columns a0..a0+31 of
// Delta (= rows of Delta^T restricted to a0..a0+31, d x 128 B) once and
// computes Yb[band][a0 + lane][0..BN) for a contiguous range of bands with
// conflict-free shared-memory gathers (lane = a).  Work units are (matrix,
// a-block, chunk of kYBands bands), dealt as contiguous ranges so a CTA
// re-stages Delta only when its (matrix, a-block) changes.
constexpr int kYBands = 16;
constexpr int kYWarps = 16;
constexpr int kDsMaxD = 1536;

struct Y2Args {
  YMat mat[kMaxGroup];
  int count, d, ablocks, tbuf;  // tbuf: transposed write-out (BN == 32, smem permitting)
  long long units;  // mat[i].task_end: cumulative units
  const int* skip;
};

template <int BN, int KR>
__global__ void __launch_bounds__(kYWarps * 32, 1) k_build_y_smem(const __grid_constant__ Y2Args A) {
  constexpr int NQ = BN * KR / 4;          // int4 (and float4) entry chunks per band
  constexpr int NE = (NQ + 31) / 32;       // per lane
  extern __shared__ __align__(16) float ds[];  // [d][32], then per-warp entry areas
  if (A.skip && *A.skip) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = A.d;
  int4* epos = reinterpret_cast<int4*>(ds + d * 32) + warp * 2 * NQ;  // [NQ] pos, then [NQ] val
  const long long u_begin = A.units * blockIdx.x / gridDim.x;
  const long long u_end = A.units * (blockIdx.x + 1) / gridDim.x;
  struct UInfo {
    int mi, ab, chunk, band_end;
  };
  auto decode = [&](long long u) {
    int mi = 0;
    while (mi + 1 < A.count && u >= A.mat[mi].task_end) ++mi;
    const YMat& M = A.mat[mi];
    const long long lt = u - (mi ? A.mat[mi - 1].task_end : 0);
    const int nchunks = (M.nbands + kYBands - 1) / kYBands;
    const int chunk = static_cast<int>(lt % nchunks);
    return UInfo{mi, static_cast<int>(lt / nchunks), chunk, min(M.nbands, (chunk + 1) * kYBands)};
  };
  // the band's BN*KR (pos, val) pairs are contiguous in the CSR arrays of Q
  auto fetch = [&](int mi, int band, int band_end, int4 (&pr)[NE], float4 (&vr)[NE]) {
    const YMat& F = A.mat[mi];
    const long long qlim = static_cast<long long>(F.n) * KR;
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int t = lane + 32 * e;
      const long long off = static_cast<long long>(band) * BN * KR + 4LL * t;
      pr[e] = make_int4(0, 0, 0, 0);
      vr[e] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < NQ && band < band_end && off < qlim) {
        pr[e] = __ldg(reinterpret_cast<const int4*>(F.qpos + off));
        vr[e] = __ldg(reinterpret_cast<const float4*>(F.qval + off));
      }
    }
  };
  int4 pr[NE];
  float4 vr[NE];
  if (u_begin < u_end) {
    const UInfo f = decode(u_begin);
    fetch(f.mi, f.chunk * kYBands + warp, f.band_end, pr, vr);
  }
  int cur_mi = -1, cur_ab = -1;
  for (long long u = u_begin; u < u_end; ++u) {
    const UInfo U = decode(u);
    const YMat& M = A.mat[U.mi];
    const int a0 = U.ab * 32;
    if (U.mi != cur_mi || U.ab != cur_ab) {
      __syncthreads();  // previous block fully consumed
      // ds[b][t] = Delta^T[b][a0 + t]  (zero beyond d); 8 loads in flight per thread
      for (int i0 = threadIdx.x; i0 < d * 8; i0 += 8 * blockDim.x) {
        float4 v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int idx = i0 + e * blockDim.x;
          const int b = idx >> 3, q = (idx & 7) * 4;
          v[e] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (idx < d * 8) {
            const float* src = M.dT + static_cast<long long>(b) * d + a0 + q;
            if (a0 + q + 3 < d) {
              v[e] = __ldg(reinterpret_cast<const float4*>(src));
            } else {
              if (a0 + q < d) v[e].x = src[0];
              if (a0 + q + 1 < d) v[e].y = src[1];
              if (a0 + q + 2 < d) v[e].z = src[2];
            }
          }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int idx = i0 + e * blockDim.x;
          if (idx < d * 8) *reinterpret_cast<float4*>(ds + (idx >> 3) * 32 + (idx & 7) * 4) = v[e];
        }
      }
      __syncthreads();
      cur_mi = U.mi;
      cur_ab = U.ab;
    }
    const int a = a0 + lane;
    const int band0 = U.chunk * kYBands + warp;
    if (band0 >= U.band_end && u + 1 < u_end) {  // no band here: entries for the next unit
      const UInfo f = decode(u + 1);
      fetch(f.mi, f.chunk * kYBands + warp, f.band_end, pr, vr);
    }
    for (int band = band0; band < U.band_end; band += kYWarps) {
      __syncwarp();
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const int t = lane + 32 * e;
        if (t < NQ) {
          epos[t] = pr[e];
          reinterpret_cast<float4*>(epos + NQ)[t] = vr[e];
        }
      }
      __syncwarp();
      // next band's entries in flight while this one is computed (possibly in
      // the next unit of this CTA's range)
      if (band + kYWarps < U.band_end) {
        fetch(U.mi, band + kYWarps, U.band_end, pr, vr);
      } else if (u + 1 < u_end) {
        const UInfo f = decode(u + 1);
        fetch(f.mi, f.chunk * kYBands + warp, f.band_end, pr, vr);
      }
      const int* sp = reinterpret_cast<const int*>(epos);
      const float* sv = reinterpret_cast<const float*>(epos + NQ);
      float y[BN];
#pragma unroll
      for (int jj = 0; jj < BN; ++jj) {
        // columns beyond n have zero entries (fetch), so y stays 0: no branch,
        // the BN column chains interleave freely
        y[jj] = 0.0f;
        const Ent<KR> en = ent_gen<KR>(sp + jj * KR, sv + jj * KR);
#pragma unroll
        for (int l = 0; l < KR; ++l) y[jj] = fmaf(en.v[l], ds[en.p[l] * 32 + lane], y[jj]);
      }
      if (A.tbuf) {
        // transposed write-out through a per-warp 32 x 33 buffer: every store
        // is one 128-byte row segment Yb[band][a0 + rr][0..31]
        float* tb = ds + d * 32 + kYWarps * 2 * NQ * 4 + warp * 32 * 33;
        __syncwarp();
#pragma unroll
        for (int jj = 0; jj < BN; ++jj) tb[lane * 33 + jj] = y[jj];
        __syncwarp();
        float* o = M.yb + (static_cast<long long>(band) * d + a0) * BN;
        const int rows = min(32, d - a0);
        for (int rr = 0; rr < rows; ++rr) o[rr * BN + lane] = tb[rr * 33 + lane];
      } else if (a < d) {
        float4* o = reinterpret_cast<float4*>(M.yb + (static_cast<long long>(band) * d + a) * BN);
#pragma unroll
        for (int t = 0; t < BN / 4; ++t)
          o[t] = make_float4(y[4 * t], y[4 * t + 1], y[4 * t + 2], y[4 * t + 3]);
      }
    }
  }
}

// Vector form (no shared memory): one warp = (matrix, band, 128-row block of
// a, 8 of the band's columns).  Lane owns a = a0 + 4*lane .. +3 and reads
// Delta^T[pos][a..a+3] with one 16-byte load (512 B per warp instruction, L2
// hits: Delta^T is 4 MiB); per (column, entry) that is ONE memory instruction
// for 4 outputs, against 1.5 shared-memory instructions per output in
// k_build_y_smem (MIO-throttle bound).  Q entries are warp-uniform loads.
constexpr int kYVJ = 8;  // band columns per warp task
template <int BN, int KR>
__global__ void __launch_bounds__(256) k_build_y_vec(const __grid_constant__ YArgs A) {
  if (A.skip && *A.skip) return;
  const int lane = threadIdx.x & 31;
  const long long task = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (task >= A.total) return;
  int mi = 0;
  while (mi + 1 < A.count && task >= A.mat[mi].task_end) ++mi;
  const YMat& M = A.mat[mi];
  // task order: (band, column group, a-block), a-block fastest: the warps of
  // one band share its Q entries in L1.  32-bit decode (< 2^31 tasks per matrix)
  const int lt = static_cast<int>(task - (mi ? A.mat[mi - 1].task_end : 0));
  const int rest = lt / A.ablocks;
  const int ab = lt - rest * A.ablocks;
  constexpr int NG = BN / kYVJ;
  const int band = rest / NG;
  const int cg = rest - band * NG;
  const int d = A.d;
  const int a = ab * 128 + 4 * lane;
  const bool a_ok = a < d;  // d % 4 == 0 (host check)
  float y[kYVJ][4];
#pragma unroll
  for (int t = 0; t < kYVJ; ++t) {
    y[t][0] = y[t][1] = y[t][2] = y[t][3] = 0.0f;
    const int j = band * BN + cg * kYVJ + t;
    if (j < M.n) {
      const Ent<KR> en = ent_ldg<KR>(M.qpos + static_cast<long long>(j) * KR,
                                     M.qval + static_cast<long long>(j) * KR);
#pragma unroll
      for (int e = 0; e < KR; ++e) {
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (a_ok) x = __ldg(reinterpret_cast<const float4*>(M.dT + static_cast<long long>(en.p[e]) * d + a));
        y[t][0] = fmaf(en.v[e], x.x, y[t][0]);
        y[t][1] = fmaf(en.v[e], x.y, y[t][1]);
        y[t][2] = fmaf(en.v[e], x.z, y[t][2]);
        y[t][3] = fmaf(en.v[e], x.w, y[t][3]);
      }
    }
  }
  if (!a_ok) return;
  const unsigned long long pol_last = policy_evict_last();
  float* base = M.yb + (static_cast<long long>(band) * d + a) * BN + cg * kYVJ;
#pragma unroll
  for (int c = 0; c < 4; ++c) {  // row a + c of the band block: kYVJ contiguous floats
    float4* o = reinterpret_cast<float4*>(base + c * BN);
#pragma unroll
    for (int t = 0; t < kYVJ; t += 4)  // evict-last: the apply reads Y right after
      st_hint_f4(reinterpret_cast<float*>(o + t / 4),
                 make_float4(y[t][c], y[t + 1][c], y[t + 2][c], y[t + 3][c]), pol_last);
  }
}


// Tiled form of k_build_y_vec for BN = 32 (the default Y build): one CTA = 8
// warps = (matrix, band, 256-row super-block of a); warp w computes column
// group w % 4 (8 of the band's 32 columns) for a-block w / 4 (128 rows) with
// exactly k_build_y_vec's loads and FMA order (so Y is bitwise the same), then
// stages its 128 x 8 outputs in a shared-memory copy of the CTA's output chunk
// Yb[band][a0 .. a0+255][0 .. 31] -- which is ONE contiguous 32 KB span of
// the workspace -- and the CTA writes the chunk out with 512-byte coalesced
// stores.  Stage-in granules are 16 bytes, XOR-swizzled by bits 2..4 of the
// row so the 8 lanes of a store phase hit 8 distinct bank groups; the
// write-out reads whole 128-byte rows (conflict-free).  k_build_y_vec wrote
// 32-byte row pieces straight from the lanes: 8x the L1 store wavefronts.
constexpr int kYTRows = 256;
template <int KR>
__global__ void __launch_bounds__(256) k_build_y_tile(const __grid_constant__ YArgs A) {
  constexpr int BN = 32;
  __shared__ __align__(16) float tile[kYTRows * BN];  // 32 KB
  if (A.skip && *A.skip) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long task = blockIdx.x;  // (matrix, band, super-block), super-block fastest
  int mi = 0;
  while (mi + 1 < A.count && task >= A.mat[mi].task_end) ++mi;
  const YMat& M = A.mat[mi];
  const int lt = static_cast<int>(task - (mi ? A.mat[mi - 1].task_end : 0));
  const int band = lt / A.ablocks;   // A.ablocks = super-blocks per band here
  const int sb = lt - band * A.ablocks;
  const int d = A.d;
  const int cg = warp & 3, ab = warp >> 2;
  const int al = ab * 128 + 4 * lane;  // first of this lane's 4 rows within the chunk
  const int a = sb * kYTRows + al;
  const bool a_ok = a < d;  // d % 4 == 0 (host check)
  float y[kYVJ][4];
#pragma unroll
  for (int t = 0; t < kYVJ; ++t) {
    y[t][0] = y[t][1] = y[t][2] = y[t][3] = 0.0f;
    const int j = band * BN + cg * kYVJ + t;
    if (j < M.n) {
      const Ent<KR> en = ent_ldg<KR>(M.qpos + static_cast<long long>(j) * KR,
                                     M.qval + static_cast<long long>(j) * KR);
#pragma unroll
      for (int e = 0; e < KR; ++e) {
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (a_ok) x = __ldg(reinterpret_cast<const float4*>(M.dT + static_cast<long long>(en.p[e]) * d + a));
        y[t][0] = fmaf(en.v[e], x.x, y[t][0]);
        y[t][1] = fmaf(en.v[e], x.y, y[t][1]);
        y[t][2] = fmaf(en.v[e], x.z, y[t][2]);
        y[t][3] = fmaf(en.v[e], x.w, y[t][3]);
      }
    }
  }
  // stage: row al + c, granules 2*cg + h (4 floats each) of the row's 8,
  // physical granule = g ^ ((row >> 2) & 7)
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int row = al + c;
    const int key = (row >> 2) & 7;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int g = (2 * cg + h) ^ key;
      *reinterpret_cast<float4*>(tile + row * BN + 4 * g) =
          make_float4(y[4 * h][c], y[4 * h + 1][c], y[4 * h + 2][c], y[4 * h + 3][c]);
    }
  }
  __syncthreads();
  // write-out: rows a0 .. a0 + rows - 1 of the band block are contiguous
  const int rows = min(kYTRows, d - sb * kYTRows);
  const unsigned long long pol_last = policy_evict_last();
  float* out = M.yb + (static_cast<long long>(band) * d + sb * kYTRows) * BN;
  for (int gi = threadIdx.x; gi < rows * (BN / 4); gi += blockDim.x) {
    const int row = gi >> 3, g = gi & 7;
    const float4 v = *reinterpret_cast<const float4*>(tile + row * BN + 4 * (g ^ ((row >> 2) & 7)));
    st_hint_f4(out + 4 * gi, v, pol_last);  // evict-last: the apply reads Y right after
  }
}


// ---------------------------------------------------------------------------
// streaming apply
// ---------------------------------------------------------------------------
struct alignas(64) AMat {
  CUtensorMap tmap;        // W (input) tile map: box BN x TR
  const int* ppos_scaled;  // P positions * BN * 4: byte offsets of Y rows
  const float* pval;
  const float* yb;
  void* out;
  long long ldo;
  int m, n, row_blocks, nbands, rps;  // rps: row blocks per unit (row segment)
  int nbu;  // units per row segment: nbands, or band pairs for the cluster-pair kernel
  long long unit_end;
};
struct AArgs {
  AMat mat[kMaxGroup];
  int count, d, stages, stage_bytes, y_bytes, w_bytes, e_bytes, pf;
  long long units;
  double alpha, beta;
  const int* skip;
};

// A unit = (matrix, row segment, band): the band's Y block is loaded once per
// unit.  Units are ordered (matrix, segment, band) and dealt round-robin to
// the CTAs, so the units in flight at any moment are ADJACENT bands of the
// same rows: together they read and write contiguous row spans of W (DRAM
// page locality), while each CTA still walks down its own band.
struct Unit {
  int mi, band, rb0, rb1;
};
__device__ __forceinline__ Unit unit_at(const AArgs& A, long long u) {
  int i = 0;
  while (i + 1 < A.count && u >= A.mat[i].unit_end) ++i;
  const AMat& M = A.mat[i];
  const long long lt = u - (i ? A.mat[i - 1].unit_end : 0);
  const int seg = static_cast<int>(lt / M.nbu);
  const int rb0 = seg * M.rps;
  return Unit{i, static_cast<int>(lt % M.nbu), rb0, min(M.row_blocks, rb0 + M.rps)};
}

__device__ __forceinline__ float lds_f32(unsigned addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ int2 lds_v2i(unsigned addr) {
  int2 v;
  asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ float2 lds_v2f(unsigned addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ int4 lds_v4i(unsigned addr) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ float4 lds_v4f(unsigned addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
template <int N>
struct FV {
  float v[N];
};
template <int N>
__device__ __forceinline__ FV<N> lds_yv(unsigned addr) {
  FV<N> r;
  if constexpr (N == 2) {
    const float2 t = lds_v2f(addr);
    r.v[0] = t.x, r.v[1] = t.y;
  } else {
    const float4 t = lds_v4f(addr);
    r.v[0] = t.x, r.v[1] = t.y, r.v[2] = t.z, r.v[3] = t.w;
  }
  return r;
}
template <typename Tw, int N>
__device__ __forceinline__ FV<N> lds_wv(unsigned addr) {
  FV<N> r;
  if constexpr (std::is_same<Tw, float>::value) {
    r = lds_yv<N>(addr);
  } else if constexpr (N == 2) {
    unsigned h;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(h) : "r"(addr));
    r.v[0] = __uint_as_float(h << 16), r.v[1] = __uint_as_float(h & 0xffff0000u);
  } else {
    unsigned h0, h1;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(h0), "=r"(h1) : "r"(addr));
    r.v[0] = __uint_as_float(h0 << 16), r.v[1] = __uint_as_float(h0 & 0xffff0000u);
    r.v[2] = __uint_as_float(h1 << 16), r.v[3] = __uint_as_float(h1 & 0xffff0000u);
  }
  return r;
}
template <int N>
__device__ __forceinline__ void st_hintv(float* a, const FV<N>& x, unsigned long long pol) {
  if constexpr (N == 2) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;\n" ::"l"(a), "f"(x.v[0]),
                 "f"(x.v[1]), "l"(pol)
                 : "memory");
  } else {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;\n" ::"l"(a),
                 "f"(x.v[0]), "f"(x.v[1]), "f"(x.v[2]), "f"(x.v[3]), "l"(pol)
                 : "memory");
  }
}
template <int N>
__device__ __forceinline__ void st_hintv(bf16* a, const FV<N>& x, unsigned long long pol) {
  const __nv_bfloat162 h0 = __floats2bfloat162_rn(x.v[0], x.v[1]);
  if constexpr (N == 2) {
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;\n" ::"l"(a),
                 "r"(*reinterpret_cast<const unsigned*>(&h0)), "l"(pol)
                 : "memory");
  } else {
    const __nv_bfloat162 h1 = __floats2bfloat162_rn(x.v[2], x.v[3]);
    asm volatile("st.global.L2::cache_hint.v2.b32 [%0], {%1, %2}, %3;\n" ::"l"(a),
                 "r"(*reinterpret_cast<const unsigned*>(&h0)),
                 "r"(*reinterpret_cast<const unsigned*>(&h1)), "l"(pol)
                 : "memory");
  }
}
template <typename Tw>
__device__ __forceinline__ float lds_w(unsigned addr) {
  if constexpr (std::is_same<Tw, float>::value) {
    return lds_f32(addr);
  } else {
    unsigned short h;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(addr));
    return __uint_as_float(static_cast<unsigned>(h) << 16);
  }
}

// PAIR (opt-in): 2-CTA clusters own pairs of adjacent bands; CTA k of the
// pair streams band 2u+k.  The leader's producer issues both W boxes of a
// tile back to back (one 2*BN-column row span of W per request pair, the
// access pattern tools/micro/stream_rmw.cu ring4 measured faster), each
// multicast to its CTA alone, and the tile's P entries multicast to both;
// consumers free a stage with a remote arrive on the leader's empty barrier.
// CPL = 2 / 4: each lane owns CPL adjacent columns (8- / 16-byte Y gathers, W
// loads and stores of CPL elements), cutting the consumer instructions per
// element; per-element arithmetic unchanged, so results are bitwise equal to
// CPL = 1.
template <typename Tw, int BN, int KR, bool USE_IN, bool PAIR, int CPL>
__global__ void __launch_bounds__(kAThreads, 1) k_apply_y(const __grid_constant__ AArgs A) {
  constexpr int TRW = tile_bytes<Tw>() / static_cast<int>(sizeof(Tw)) / BN;
  constexpr int TR = TRW < 256 ? TRW : 256;  // W rows per tile (16 KB of W; <= 256 TMA box rows)
  constexpr int LPR = BN / CPL;        // lanes per W row
  constexpr int RPW = 32 / LPR;        // rows per warp instruction
  extern __shared__ __align__(128) unsigned char smem_raw[];
  if (A.skip && *A.skip) return;
  // consumer warps form kNG groups; group g takes tiles g, g+kNG, ... so kNG
  // tiles are consumed concurrently (a tile's latency is not serialised)
  unsigned char* ring = smem_raw + A.y_bytes;
  unsigned long long* full =
      reinterpret_cast<unsigned long long*>(ring + A.stages * A.stage_bytes);
  unsigned long long* empty = full + A.stages;
  unsigned long long* yfull = empty + A.stages;
  unsigned long long* yempty = yfull + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int S = A.stages;

  unsigned crank = 0;
  if constexpr (PAIR) crank = cluster_ctarank();
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, (PAIR ? 2 : 1) * (kNC / kNG));
    }
    mbar_init(yfull, 1);
    mbar_init(yempty, kNC);
    fence_mbar_init();
  }
  if constexpr (PAIR) {
    cluster_sync_all();  // peers' barriers initialised before any remote arrive
  } else {
    __syncthreads();
  }
  // unit sequence of this CTA (of its cluster for PAIR: both CTAs walk it)
  const long long u_first = PAIR ? blockIdx.x / 2 : blockIdx.x;
  const long long u_step = PAIR ? gridDim.x / 2 : gridDim.x;
  if (u_first >= A.units) return;  // PAIR grids never have idle clusters

  if (warp == 0) {
    // ---------------- W / P-entry producer ----------------
    if (lane == 0) {
      const unsigned long long pol = policy_evict_first();
      int st = 0, rnd = 0;  // ring stage of the current tile and its wrap count
      for (long long u = u_first; u < A.units; u += u_step) {
        const Unit U = unit_at(A, u);
        const AMat& M = A.mat[U.mi];
        if constexpr (PAIR) {
          for (int rb = U.rb0; rb < U.rb1; ++rb, (++st == S) ? (st = 0, ++rnd) : 0) {
            if (rnd > 0) {
              // leader: both CTAs consumed the stage; everyone: own previous
              // phase complete before re-arming it
              if (crank == 0) mbar_wait(empty + st, (rnd - 1) & 1);
              mbar_wait(full + st, (rnd - 1) & 1);
            }
            const int r0 = rb * TR;
            const int nrows = min(TR, M.m - r0);
            unsigned char* base = ring + st * A.stage_bytes;
            const unsigned eb = (static_cast<unsigned>(nrows) * KR * 4u + 15u) & ~15u;
            mbar_arrive_expect_tx(full + st, A.w_bytes + 2u * eb);
            if (crank == 0) {
              tma_load_2d_mc(base, &M.tmap, (2 * U.band) * BN, r0, full + st, 1, pol);
              tma_load_2d_mc(base, &M.tmap, (2 * U.band + 1) * BN, r0, full + st, 2, pol);
              bulk_load_mc(base + A.w_bytes, M.ppos_scaled + static_cast<long long>(r0) * KR, eb,
                           full + st, 3);
              bulk_load_mc(base + A.w_bytes + A.e_bytes, M.pval + static_cast<long long>(r0) * KR,
                           eb, full + st, 3);
            }
          }
          continue;
        }
        if (USE_IN && A.pf > S)  // fill the L2 prefetch window beyond the ring
          for (int rb = U.rb0 + S; rb < min(U.rb1, U.rb0 + A.pf); ++rb)
            tma_prefetch_2d(&M.tmap, U.band * BN, rb * TR);
        for (int rb = U.rb0; rb < U.rb1; ++rb, (++st == S) ? (st = 0, ++rnd) : 0) {
          if (USE_IN && A.pf > S && rb + A.pf < U.rb1)
            tma_prefetch_2d(&M.tmap, U.band * BN, (rb + A.pf) * TR);
          if (rnd > 0) mbar_wait(empty + st, (rnd - 1) & 1);
          const int r0 = rb * TR;
          const int nrows = min(TR, M.m - r0);
          unsigned char* base = ring + st * A.stage_bytes;
          // odd row counts with KR = 2: round up to the 16-byte bulk-copy
          // granule (the projector arrays carry 16 bytes of slack)
          const unsigned eb = (static_cast<unsigned>(nrows) * KR * 4u + 15u) & ~15u;
          mbar_arrive_expect_tx(full + st, (USE_IN ? A.w_bytes : 0) + 2u * eb);
          if (USE_IN) tma_load_2d(base, &M.tmap, U.band * BN, r0, full + st, pol);
          bulk_load(base + A.w_bytes, M.ppos_scaled + static_cast<long long>(r0) * KR, eb,
                    full + st);
          bulk_load(base + A.w_bytes + A.e_bytes, M.pval + static_cast<long long>(r0) * KR, eb,
                    full + st);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- Y block producer (one bulk copy per unit) ----------------
    if (lane == 0) {
      int k = 0;
      for (long long u = u_first; u < A.units; u += u_step, ++k) {
        const Unit U = unit_at(A, u);
        const int band = PAIR ? 2 * U.band + static_cast<int>(crank) : U.band;
        if (k > 0) mbar_wait(yempty, (k - 1) & 1);
        if (PAIR && band >= A.mat[U.mi].nbands) {  // odd band count: no Y, no stores
          mbar_arrive(yfull);
          continue;
        }
        mbar_arrive_expect_tx(yfull, static_cast<unsigned>(A.y_bytes));
        const unsigned char* src = reinterpret_cast<const unsigned char*>(
            A.mat[U.mi].yb + static_cast<long long>(band) * A.d * BN);
        for (int off = 0; off < A.y_bytes; off += kYChunk)
          bulk_load(smem_raw + off, src + off, min(kYChunk, A.y_bytes - off), yfull);
      }
    }
  } else {

  // ---------------- consumers ----------------
  constexpr int WPG = kNC / kNG;          // warps per consumer group
  constexpr int RPT = TR / (WPG * RPW);   // rows per lane per tile
  const int cw = warp - 2;
  const int grp = cw / WPG, gw = cw % WPG;
  const float alpha = static_cast<float>(A.alpha), beta = static_cast<float>(A.beta);
  const int jj = (lane % LPR) * CPL, rsub = lane / LPR;
  const int q0 = gw * RPW + rsub;  // this lane's first row in a tile; rows q0 + v*WPG*RPW
  const unsigned y_lane = smem_addr(smem_raw) + jj * 4u;
  const unsigned ring_s = smem_addr(ring);
  // W is written once and not re-read: evict-first keeps the Y blocks in L2
  const unsigned long long pol_first = policy_evict_first();
  int s = 0, k = 0, st = 0, rnd = 0;  // tile counter, unit counter, stage, wrap count
  for (long long u = u_first; u < A.units; u += u_step, ++k) {
    const Unit U = unit_at(A, u);
    const AMat& M = A.mat[U.mi];
    const int band = PAIR ? 2 * U.band + static_cast<int>(crank) : U.band;
    const int j = band * BN + jj;
    const bool col_ok = j < M.n;
    const bool group_ok = j + CPL <= M.n;  // all CPL columns of the lane in range
    Tw* const ocol = static_cast<Tw*>(M.out) + j;  // element offsets below fit in 32 bits
    const int ldo = static_cast<int>(M.ldo);
    mbar_wait(yfull, k & 1);
    for (int rb = U.rb0; rb < U.rb1; ++rb, ++s, (++st == S) ? (st = 0, ++rnd) : 0) {
      if (s % kNG != grp) continue;
      const int r0 = rb * TR;
      const int nrows = min(TR, M.m - r0);
      mbar_wait(full + st, rnd & 1);
      const unsigned base = ring_s + st * A.stage_bytes;
      const unsigned wq = base + (q0 * BN + jj) * static_cast<unsigned>(sizeof(Tw));
      const unsigned pq = base + A.w_bytes + q0 * KR * 4u;
      const unsigned vq = base + A.w_bytes + A.e_bytes + q0 * KR * 4u;
      constexpr int kq = WPG * RPW;  // row step between a lane's rows
      auto row = [&](int v) {
        int pp[KR];
        float vv[KR];
        if constexpr (KR == 2) {
          const int2 a = lds_v2i(pq + v * kq * KR * 4u);
          const float2 b = lds_v2f(vq + v * kq * KR * 4u);
          pp[0] = a.x, pp[1] = a.y, vv[0] = b.x, vv[1] = b.y;
        } else {
#pragma unroll
          for (int l = 0; l < KR; l += 4) {
            const int4 a = lds_v4i(pq + (v * kq * KR + l) * 4u);
            const float4 b = lds_v4f(vq + (v * kq * KR + l) * 4u);
            pp[l] = a.x, pp[l + 1] = a.y, pp[l + 2] = a.z, pp[l + 3] = a.w;
            vv[l] = b.x, vv[l + 1] = b.y, vv[l + 2] = b.z, vv[l + 3] = b.w;
          }
        }
        if constexpr (CPL == 1) {
          float acc = vv[0] * lds_f32(y_lane + pp[0]);
#pragma unroll
          for (int l = 1; l < KR; ++l) acc = fmaf(vv[l], lds_f32(y_lane + pp[l]), acc);
          float res = alpha * acc;
          if (USE_IN) res = fmaf(beta, lds_w<Tw>(wq + v * kq * BN * static_cast<unsigned>(sizeof(Tw))), res);
          return cvt<Tw>(res);
        } else {
          // packed FMUL2 / FFMA2 (two IEEE operations per instruction, same
          // per-column order as CPL = 1)
          FV<CPL> acc = lds_yv<CPL>(y_lane + pp[0]);
          auto pairs = [&](auto&& op) {
#pragma unroll
            for (int c = 0; c < CPL; c += 2) {
              const float2 r = op(c, make_float2(acc.v[c], acc.v[c + 1]));
              acc.v[c] = r.x;
              acc.v[c + 1] = r.y;
            }
          };
          pairs([&](int, float2 a) { return __fmul2_rn(make_float2(vv[0], vv[0]), a); });
#pragma unroll
          for (int l = 1; l < KR; ++l) {
            const FV<CPL> y = lds_yv<CPL>(y_lane + pp[l]);
            pairs([&](int c, float2 a) {
              return __ffma2_rn(make_float2(vv[l], vv[l]), make_float2(y.v[c], y.v[c + 1]), a);
            });
          }
          pairs([&](int, float2 a) { return __fmul2_rn(make_float2(alpha, alpha), a); });
          if (USE_IN) {
            const FV<CPL> w = lds_wv<Tw, CPL>(wq + v * kq * BN * static_cast<unsigned>(sizeof(Tw)));
            pairs([&](int c, float2 a) {
              return __ffma2_rn(make_float2(beta, beta), make_float2(w.v[c], w.v[c + 1]), a);
            });
          }
          return acc;
        }
      };
      if (col_ok) {
        Tw* const orow = ocol + static_cast<long long>(r0 + q0) * ldo;
        if constexpr (CPL == 1) {
          if (nrows == TR) {  // straight-line: rows interleave freely
            const int stride = kq * ldo;
#pragma unroll
            for (int v = 0; v < RPT; ++v) st_hint(orow + v * stride, row(v), pol_first);
          } else {
#pragma unroll 1
            for (int v = 0; v < RPT && q0 + v * kq < nrows; ++v)
              st_hint(orow + static_cast<long long>(v) * kq * ldo, row(v), pol_first);
          }
        } else if (group_ok) {
          if (nrows == TR) {
            const int stride = kq * ldo;
#pragma unroll
            for (int v = 0; v < RPT; ++v) st_hintv<CPL>(orow + v * stride, row(v), pol_first);
          } else {
#pragma unroll 1
            for (int v = 0; v < RPT && q0 + v * kq < nrows; ++v)
              st_hintv<CPL>(orow + static_cast<long long>(v) * kq * ldo, row(v), pol_first);
          }
        } else {  // the last columns of n: the valid ones only
#pragma unroll 1
          for (int v = 0; v < RPT && q0 + v * kq < nrows; ++v) {
            const FV<CPL> x = row(v);
#pragma unroll
            for (int c = 0; c < CPL; ++c)
              if (j + c < M.n) st_hint(orow + static_cast<long long>(v) * kq * ldo + c, cvt<Tw>(x.v[c]), pol_first);
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR) {
          mbar_arrive_cluster(empty + st, 0);
        } else {
          mbar_arrive(empty + st);
        }
      }
    }
    if (lane == 0) mbar_arrive(yempty);  // this unit's Y block may be replaced
  }
  }  // consumers
  if constexpr (PAIR) {
    __syncwarp();
    cluster_sync_all();  // no CTA exits while its peer may still signal it
  }
}

template <int BN, int KR>
void build_y_impl(const std::vector<DecJob>& jobs_in, const int* skip, cudaStream_t st) {
  // Build the group's Y blocks in reverse matrix order: the apply walks the
  // matrices forward, so the blocks it needs first are the ones written last
  // (evict-last) and still L2-resident when a layer's Y exceeds the L2.
  // LSP_BUILD_Y_REVERSE=0 keeps the forward order (results are identical).
  const char* rev_env = std::getenv("LSP_BUILD_Y_REVERSE");
  const bool rev = !(rev_env && rev_env[0] == '0');
  const std::vector<DecJob> jobs = rev ? std::vector<DecJob>(jobs_in.rbegin(), jobs_in.rend()) : jobs_in;
  const Pair& p0 = *jobs[0].pr;
  const char* env = std::getenv("LSP_BUILD_Y_GLOBAL");
  // the shared-memory build stages Delta^T rows with 16-byte loads: d % 4 == 0
  const bool use_smem = p0.d <= kDsMaxD && p0.d % 4 == 0 && !(env && env[0] == '1');
  YArgs A{};
  Y2Args B{};
  A.count = B.count = static_cast<int>(jobs.size());
  A.d = B.d = p0.d;
  A.ablocks = ceil_div(p0.d, 64);
  B.ablocks = ceil_div(p0.d, 32);
  A.skip = B.skip = skip;
  long long total = 0, units = 0;
  for (size_t i = 0; i < jobs.size(); ++i) {
    const Pair& pr = *jobs[i].pr;
    YMat M{};
    M.qpos = pr.q->pos.as<int>();
    M.qval = pr.q->val.as<float>();
    M.dT = static_cast<const float*>(jobs[i].delta_t);
    M.yb = pr.yb.as<float>();
    M.n = pr.n;
    M.nbands = ceil_div(pr.n, BN);
    total += static_cast<long long>(M.nbands) * A.ablocks;
    units += static_cast<long long>(ceil_div(M.nbands, kYBands)) * B.ablocks;
    M.task_end = total;
    A.mat[i] = M;
    M.task_end = units;
    B.mat[i] = M;
  }
  A.total = total;
  B.units = units;
  if (total == 0) return;
  const char* vec_env = std::getenv("LSP_BUILD_Y_VEC");
  const char* tile_env = std::getenv("LSP_BUILD_Y_TILE");
  if constexpr (BN == 32) {
    if (p0.d % 4 == 0 && !(vec_env && vec_env[0] == '0') && !(tile_env && tile_env[0] == '0')) {
      YArgs V = A;
      V.ablocks = ceil_div(p0.d, kYTRows);  // super-blocks per band
      long long tv = 0;
      for (int i = 0; i < V.count; ++i) {
        tv += static_cast<long long>(V.mat[i].nbands) * V.ablocks;
        V.mat[i].task_end = tv;
      }
      V.total = tv;
      k_build_y_tile<KR><<<static_cast<unsigned>(tv), 256, 0, st>>>(V);
      after_launch("build_y_tile");
      return;
    }
  }
  if (p0.d % 4 == 0 && BN % kYVJ == 0 && !(vec_env && vec_env[0] == '0')) {
    YArgs V = A;
    V.ablocks = ceil_div(p0.d, 128);
    long long tv = 0;
    for (int i = 0; i < V.count; ++i) {
      tv += static_cast<long long>(V.mat[i].nbands) * (BN / kYVJ) * V.ablocks;
      V.mat[i].task_end = tv;
    }
    V.total = tv;
    k_build_y_vec<BN, KR><<<static_cast<unsigned>((tv + 7) / 8), 256, 0, st>>>(V);
    after_launch("build_y_vec");
    return;
  }
  if (use_smem) {
    int smem = p0.d * 32 * static_cast<int>(sizeof(float)) + kYWarps * 2 * BN * KR * 4;
    const int tbytes = kYWarps * 32 * 33 * static_cast<int>(sizeof(float));
    B.tbuf = BN == 32 && smem + tbytes <= 227 * 1024;
    if (B.tbuf) smem += tbytes;
    auto kern = k_build_y_smem<BN, KR>;
    LSP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int grid = static_cast<int>(std::min<long long>(units, sm_budget(kBudgetUpdate)));
    kern<<<grid, kYWarps * 32, smem, st>>>(B);
    after_launch("build_y_smem");
    return;
  }
  k_build_y<BN, KR><<<static_cast<unsigned>((total + 7) / 8), 256, 0, st>>>(A);
  after_launch("build_y");
}

template <typename Tw, int BN, int KR>
bool apply_impl(const std::vector<DecJob>& jobs, double alpha, double beta, const int* skip,
                cudaStream_t st) {
  constexpr int TRW = tile_bytes<Tw>() / static_cast<int>(sizeof(Tw)) / BN;
  constexpr int TR = TRW < 256 ? TRW : 256;
  const Pair& p0 = *jobs[0].pr;
  const bool use_in = beta != 0.0;
  AArgs A{};
  A.count = static_cast<int>(jobs.size());
  A.d = p0.d;
  A.alpha = alpha;
  A.beta = beta;
  A.skip = skip;
  A.y_bytes = p0.d * BN * 4;
  A.w_bytes = TR * BN * static_cast<int>(sizeof(Tw));
  A.e_bytes = TR * KR * 4;
  A.stage_bytes = static_cast<int>(round_up(A.w_bytes + 2 * A.e_bytes, 128));
  const int bar_bytes = (2 * kMaxStages + 2) * 8;
  A.stages = std::min(kMaxStages, (kSmemMax - A.y_bytes - bar_bytes) / A.stage_bytes);
  if (const char* e = std::getenv("LSP_APPLY_STAGES")) A.stages = std::min(A.stages, std::atoi(e));
  // Group g consumes tiles g, g + kNG, ...: with a stage count that is a
  // multiple of kNG each stage belongs to one group, so a group's waits on a
  // stage's full barrier are one phase apart.  With an odd count the groups
  // share stages, and a fast group can be two phases ahead of a stage whose
  // parity then matches an older completed phase (it would read stale data).
  A.stages -= A.stages % kNG;
  if (A.stages < kNG) return false;
  A.pf = 0;  // L2 prefetch distance in tiles (0: off)
  if (const char* e = std::getenv("LSP_APPLY_PF")) A.pf = std::atoi(e);
  const char* pair_env = std::getenv("LSP_APPLY_PAIR");
  const bool pair = use_in && pair_env && pair_env[0] == '1';
  const int smem = A.y_bytes + A.stages * A.stage_bytes + bar_bytes;
  // columns per lane: 4 by default (2 or 1 when rows are not 4-element
  // aligned).  Measured on B200, apply ms per step at CPL 1 / 2 / 4: C4
  // 11.4 / 10.6 / 10.4, C4-bf16 9.5 / 7.5 / 6.8, C3 2.2 / 1.8 / 1.6.
  // LSP_APPLY_CPL=1|2|4 overrides.
  const char* cpl_env = std::getenv("LSP_APPLY_CPL");
  int cpl = cpl_env ? std::atoi(cpl_env) : 4;
  if (cpl != 1 && cpl != 2 && cpl != 4) cpl = 4;
  for (const DecJob& J : jobs)
    while (cpl > 1 && (J.ldo % cpl != 0 || reinterpret_cast<uintptr_t>(J.out) % (cpl * sizeof(Tw)) != 0))
      cpl /= 2;
  void (*kern)(AArgs);
  if (pair) {
    kern = cpl == 4 ? k_apply_y<Tw, BN, KR, true, true, 4>
                    : (cpl == 2 ? k_apply_y<Tw, BN, KR, true, true, 2> : k_apply_y<Tw, BN, KR, true, true, 1>);
  } else if (use_in) {
    kern = cpl == 4 ? k_apply_y<Tw, BN, KR, true, false, 4>
                    : (cpl == 2 ? k_apply_y<Tw, BN, KR, true, false, 2> : k_apply_y<Tw, BN, KR, true, false, 1>);
  } else {
    kern = cpl == 4 ? k_apply_y<Tw, BN, KR, false, false, 4>
                    : (cpl == 2 ? k_apply_y<Tw, BN, KR, false, false, 2> : k_apply_y<Tw, BN, KR, false, false, 1>);
  }
  LSP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  int grid_max = sm_budget(kBudgetUpdate);
  if (pair) {  // grid_max counts clusters: as many 2-CTA clusters as fit at once
    cfg.blockDim = dim3(kAThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(grid_max / 2 * 2);
    int ncl = 0;
    LSP_CUDA(cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg));
    if (ncl < 1) return false;
    grid_max = std::min(ncl, grid_max / 2);
  }
  long long tiles = 0;
  for (const DecJob& J : jobs)
    tiles += static_cast<long long>(ceil_div(ceil_div(J.pr->n, BN), pair ? 2 : 1)) *
             ceil_div(J.pr->m, TR);
  // unit (row segment of a band) at most ~1/4 of a CTA's share, so the
  // round-robin deal stays balanced; env LSP_APPLY_SEG overrides (rows blocks)
  long long cap = std::max<long long>(8, tiles / grid_max / 4);
  if (const char* e = std::getenv("LSP_APPLY_SEG")) cap = std::max(1, std::atoi(e));
  long long units = 0;
  for (size_t i = 0; i < jobs.size(); ++i) {
    const DecJob& J = jobs[i];
    const Pair& pr = *J.pr;
    AMat& M = A.mat[i];
    if (use_in && !cached_tmap(&M.tmap, J.in, std::is_same<Tw, float>::value ? LSP_F32 : LSP_BF16,
                               pr.m, pr.n, J.ldi, BN, TR))
      return false;
    M.ppos_scaled = pr.p->scaled_pos(BN * 4);
    M.pval = pr.p->val.as<float>();
    M.yb = pr.yb.as<float>();
    M.out = J.out;
    M.ldo = J.ldo;
    M.m = pr.m, M.n = pr.n;
    M.row_blocks = ceil_div(pr.m, TR);
    M.nbands = ceil_div(pr.n, BN);
    M.nbu = pair ? ceil_div(M.nbands, 2) : M.nbands;
    const int segs = ceil_div(M.row_blocks, cap);
    M.rps = ceil_div(M.row_blocks, segs);
    units += static_cast<long long>(M.nbu) * ceil_div(M.row_blocks, M.rps);
    M.unit_end = units;
  }
  A.units = units;
  if (units == 0) return true;
  const int grid = static_cast<int>(std::min<long long>(units, grid_max));
  if (pair) {
    cfg.gridDim = dim3(2 * grid);
    LSP_CUDA(cudaLaunchKernelEx(&cfg, kern, A));
    after_launch("apply_y_pair");
    return true;
  }
  kern<<<grid, kAThreads, smem, st>>>(A);
  after_launch("apply_y");
  return true;
}

template <int BN, int KR>
bool run_bn(const std::vector<DecJob>& jobs, lsp_dtype dt, double alpha, double beta,
            const int* skip, cudaStream_t st, int phase) {
  for (const DecJob& J : jobs) {
    const Pair& pr = *J.pr;
    J.pr->yb_ensure(static_cast<size_t>(ceil_div(pr.n, BN)) * pr.d * BN * sizeof(float));
  }
  // check eligibility of the apply before enqueueing the Y build
  for (const DecJob& J : jobs)  // 32-bit element offsets into W
    if (static_cast<long long>(J.pr->m) * J.ldo >= (1LL << 31)) return false;
  if (beta != 0.0)
    for (const DecJob& J : jobs) {
      if (J.in == nullptr) return false;
      const size_t es = dtype_size(dt);
      if (reinterpret_cast<uintptr_t>(J.in) % 16 || (J.ldi * es) % 16) return false;
    }
  if (phase != kPhaseBoth) {  // split form: the whole group, build or apply
    if (phase == kPhaseBuild) build_y_impl<BN, KR>(jobs, skip, st);
    if (phase == kPhaseApply) {
      const bool ok = dt == LSP_F32 ? apply_impl<float, BN, KR>(jobs, alpha, beta, skip, st)
                                    : apply_impl<bf16, BN, KR>(jobs, alpha, beta, skip, st);
      require(ok, "apply_y: launch configuration rejected after the Y build");
    }
    return true;
  }
  // Y build + apply per subgroup of at most LSP_APPLY_YB_MB of Y blocks
  // (default: the whole group -- measured faster than L2-sized subgroups)
  size_t budget = ~size_t(0);
  if (const char* e = std::getenv("LSP_APPLY_YB_MB")) budget = static_cast<size_t>(std::atoi(e)) << 20;
  size_t i = 0;
  while (i < jobs.size()) {
    size_t j = i, bytes = 0;
    while (j < jobs.size()) {
      const Pair& pr = *jobs[j].pr;
      const size_t b = static_cast<size_t>(ceil_div(pr.n, BN)) * pr.d * BN * sizeof(float);
      if (j > i && bytes + b > budget) break;
      bytes += b;
      ++j;
    }
    const std::vector<DecJob> sub(jobs.begin() + i, jobs.begin() + j);
    build_y_impl<BN, KR>(sub, skip, st);
    const bool ok = dt == LSP_F32 ? apply_impl<float, BN, KR>(sub, alpha, beta, skip, st)
                                  : apply_impl<bf16, BN, KR>(sub, alpha, beta, skip, st);
    require(ok, "apply_y: launch configuration rejected after the Y build");
    i = j;
  }
  return true;
}

}  // namespace

// Fast path of launch_decompress_group for fp32 accumulation, W in fp32 or
// bf16, r in {4, 8}; false (nothing enqueued) when not eligible.
// Per-matrix eligibility of the Y path (column orientation).
static bool y_eligible(const DecJob& J, lsp_dtype dt, double beta) {
  const Pair& pr = *J.pr;
  if (pr.compute != LSP_F32 || (dt != LSP_F32 && dt != LSP_BF16)) return false;
  const int r = pr.p->r;
  if ((r != 2 && r != 4 && r != 8) || pr.q->r != r) return false;
  if (pr.d * 8 * 4 > kYMaxBytes) return false;
  if (static_cast<long long>(pr.m) * J.ldo >= (1LL << 31)) return false;  // 32-bit offsets
  // the Y builds read delta^T with 16-byte vector loads
  if (reinterpret_cast<uintptr_t>(J.delta_t) % 16) return false;
  if (beta != 0.0) {
    const size_t es = dtype_size(dt);
    if (J.in == nullptr || reinterpret_cast<uintptr_t>(J.in) % 16 || (J.ldi * es) % 16) return false;
  }
  const char* band = std::getenv("LSP_DECOMPRESS_BAND");
  return !(band && band[0] == '1');
}

bool decompress_fast_eligible(const DecJob& J, lsp_dtype dt, double beta) {
  return apply_x_eligible(J, dt, beta) || y_eligible(J, dt, beta) || y64_eligible(J, dt, beta);
}

bool launch_decompress_group_y(const std::vector<DecJob>& all_jobs, lsp_dtype dt, double alpha,
                               double beta, const int* skip_flag, cudaStream_t st, int phase) {
  if (all_jobs.empty() || all_jobs.size() > static_cast<size_t>(kMaxGroup)) return false;
  for (const DecJob& J : all_jobs)
    if (!decompress_fast_eligible(J, dt, beta)) return false;
  if (all_jobs[0].pr->compute == LSP_F64) {  // fp64 twin of the Y path (apply_f64.cu)
    launch_y64_group(all_jobs, alpha, beta, skip_flag, st, phase);
    return true;
  }
  // n > m matrices go to the row orientation (apply_x.cu), the rest here;
  // every matrix's path depends only on the matrix, never on its group
  std::vector<DecJob> jobs, xjobs;
  for (const DecJob& J : all_jobs) (apply_x_eligible(J, dt, beta) ? xjobs : jobs).push_back(J);
  if (!jobs.empty()) {
    const Pair& p0 = *jobs[0].pr;
    const int r = p0.p->r, d = p0.d;
    for (const DecJob& J : jobs)
      require(J.pr->p->r == r && J.pr->d == d, "decompress group: matrices must share d and r");
    auto pick = [&](auto bn) -> bool {
      constexpr int BN = decltype(bn)::value;
      return r == 4   ? run_bn<BN, 4>(jobs, dt, alpha, beta, skip_flag, st, phase)
             : r == 8 ? run_bn<BN, 8>(jobs, dt, alpha, beta, skip_flag, st, phase)
                      : run_bn<BN, 2>(jobs, dt, alpha, beta, skip_flag, st, phase);
    };
    const char* bn_env = std::getenv("LSP_APPLY_BN");
    const int bn_max = bn_env ? std::atoi(bn_env) : 32;
    bool ok = false;
    if (bn_max >= 32 && d * 32 * 4 <= kYMaxBytes)
      ok = pick(std::integral_constant<int, 32>{});
    else if (d * 16 * 4 <= kYMaxBytes)
      ok = pick(std::integral_constant<int, 16>{});
    else
      ok = pick(std::integral_constant<int, 8>{});
    require(ok, "decompress: Y path rejected an eligible group");
  }
  if (!xjobs.empty()) launch_apply_x(xjobs, alpha, beta, skip_flag, st, phase);
  return true;
}

}  // namespace lspb
