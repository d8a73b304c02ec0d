// Shared device helpers for libs2v (sm_100a).  Compiled with -fmad=false:
// every fused multiply-add in this library is an explicit fma(), every other
// a*b+c is rounded twice, matching the reference's numpy/OpenBLAS order.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/s2v.h"

namespace s2v {

void set_error(const std::string &msg);
int fail(int code, const char *fmt, ...);

#define S2V_CUDA_CHECK(expr)                                                      \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess)                                                        \
      return ::s2v::fail(S2V_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,    \
                         cudaGetErrorString(_e));                                 \
  } while (0)

#define S2V_LAUNCH_CHECK() S2V_CUDA_CHECK(cudaGetLastError())

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kNumSMs = 148;

// np.maximum(x, 0): NaN propagates, -0 stays -0 (a >= b ? a : b).
template <class T>
__device__ __forceinline__ T relu(T x) {
  return (x >= T(0) || x != x) ? x : T(0);
}

__device__ __forceinline__ float fmaT(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fmaT(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float addT(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double addT(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float mulT(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mulT(double a, double b) { return __dmul_rn(a, b); }

// Selection key: score (order-preserving 64-bit image, -0 == +0, NaN above
// +inf for argmax semantics) then lowest node id.  fp32 scores widen to fp64
// exactly, so one key type serves both dtypes.
struct Key {
  uint64_t s;    // orderable(score); 0 = "no key"
  uint64_t inv;  // ~node, so that larger is better on ties
};

__device__ __forceinline__ uint64_t orderable(double d) {
  if (d != d) return ~0ull;
  uint64_t b = (d == 0.0) ? 0ull : (uint64_t)__double_as_longlong(d);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ bool key_gt(const Key &a, const Key &b) {
  return a.s > b.s || (a.s == b.s && a.inv > b.inv);
}

__device__ __forceinline__ Key make_key(double s, int64_t node) {
  return Key{orderable(s), ~(uint64_t)node};
}

__device__ __forceinline__ Key null_key() { return Key{0ull, 0ull}; }

__device__ __forceinline__ Key shfl_key(const Key &k, int src) {
  Key r;
  r.s = __shfl_sync(0xffffffffu, k.s, src);
  r.inv = __shfl_sync(0xffffffffu, k.inv, src);
  return r;
}

__device__ __forceinline__ Key shfl_xor_key(const Key &k, int m) {
  Key r;
  r.s = __shfl_xor_sync(0xffffffffu, k.s, m);
  r.inv = __shfl_xor_sync(0xffffffffu, k.inv, m);
  return r;
}

}  // namespace s2v
