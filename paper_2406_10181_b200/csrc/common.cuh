// Shared host/device helpers for the B200-native LSP projector path.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "lsp_b200.h"

namespace lspb {

using bf16 = __nv_bfloat16;

// Host-side error carrying an lsp_status; converted at the C-ABI boundary.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void require(bool ok, const std::string& msg) {
  if (!ok) fail(LSP_EINVAL, msg);
}

#define LSP_CUDA(x)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess)                                                            \
      throw ::lspb::Error(e_ == cudaErrorMemoryAllocation ? LSP_ENOMEM : LSP_ECUDA,   \
                          std::string(#x) + ": " + cudaGetErrorString(e_));           \
  } while (0)

extern std::atomic<uint64_t> g_launches;
// Call after every kernel launch: surfaces launch errors and counts launches.
// LSP_TRACE=1 prints every launch's name to stderr (debugging aid).
bool trace_launches();
inline void after_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(LSP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (trace_launches()) fprintf(stderr, "[lsp] launch %s\n", what);
}

inline cudaStream_t as_stream(lsp_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }
inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }
inline long long round_up(long long a, long long b) { return (a + b - 1) / b * b; }

size_t dtype_size(lsp_dtype t);
int num_sms();
// SMs a persistent grid of the given phase may size for (lsp_set_sm_budget)
enum { kBudgetCompress = 0, kBudgetUpdate = 1 };
int sm_budget(int phase);

#ifdef __CUDACC__
// ---------------------------------------------------------------------------
// Device conversions between storage types (double / float / bf16) and the
// accumulator type (double or float).
// ---------------------------------------------------------------------------

template <typename To, typename From>
struct Cvt {
  __device__ __forceinline__ static To f(From v) { return static_cast<To>(v); }
};
template <>
struct Cvt<float, bf16> {
  __device__ __forceinline__ static float f(bf16 v) { return __bfloat162float(v); }
};
template <>
struct Cvt<double, bf16> {
  __device__ __forceinline__ static double f(bf16 v) { return (double)__bfloat162float(v); }
};
template <>
struct Cvt<bf16, float> {
  __device__ __forceinline__ static bf16 f(float v) { return __float2bfloat16_rn(v); }
};
template <>
struct Cvt<bf16, double> {
  __device__ __forceinline__ static bf16 f(double v) { return __double2bfloat16(v); }
};
template <typename To, typename From>
__device__ __forceinline__ To cvt(From v) {
  return Cvt<To, From>::f(v);
}


#endif  // __CUDACC__

// Dispatch a runtime dtype to a C++ type.
#define LSP_DISPATCH_STORAGE(DT, T, ...)                      \
  switch (DT) {                                               \
    case LSP_F64: { using T = double; __VA_ARGS__; break; }   \
    case LSP_F32: { using T = float; __VA_ARGS__; break; }    \
    case LSP_BF16: { using T = ::lspb::bf16; __VA_ARGS__; break; } \
    default: ::lspb::fail(LSP_EINVAL, "unknown dtype");        \
  }
#define LSP_DISPATCH_ACC(DT, T, ...)                                         \
  switch (DT) {                                                              \
    case LSP_F64: { using T = double; __VA_ARGS__; break; }                  \
    case LSP_F32: { using T = float; __VA_ARGS__; break; }                   \
    default: ::lspb::fail(LSP_EINVAL, "compute dtype must be F32 or F64");   \
  }

}  // namespace lspb
