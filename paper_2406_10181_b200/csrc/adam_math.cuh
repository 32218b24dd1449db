// Subspace Adam element update (proj/src/subspace_opt.cpp:35-57), shared by the
// standalone Adam kernel (elementwise.cu) and the stage-2 + Adam kernel
// (compress.cu).  Elementwise, no contraction (explicit _rn ops) so the fp64
// path rounds exactly like the reference:
//   m = b1*m + (1-b1)*g;  v = b2*v + (1-b2)*g*g;  delta = (m / c1) / (sqrt(v / c2) + eps).
#pragma once

namespace lspb {

__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float div_(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float sqrt_(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ double sqrt_(double a) { return __dsqrt_rn(a); }

// Returns delta; updates the moments in place.
template <typename T>
__device__ __forceinline__ T adam_elem(T g, T& m, T& v, T b1, T omb1, T b2, T omb2, T c1, T c2,
                                       T eps) {
  const T mi = add_(mul_(b1, m), mul_(omb1, g));
  const T vi = add_(mul_(b2, v), mul_(mul_(omb2, g), g));
  m = mi;
  v = vi;
  return div_(div_(mi, c1), add_(sqrt_(div_(vi, c2)), eps));
}

}  // namespace lspb
