// common.cuh -- shared internals of librnn.so (status plumbing, warp helpers).
// Product code only: nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/rnn.h"

// Measurement probes (clock64 phase timers, event counters read through the
// rnn_internal_*_stats hooks) are compiled in only for measurement builds (-DRNN_PROBES);
// the production library carries none of them.
#ifdef RNN_PROBES
#define RNN_PROBE(...) __VA_ARGS__
#else
#define RNN_PROBE(...)
#endif

namespace rnn {

// --------------------------------------------------------------------------------------
// error plumbing: thread-local detail string, status codes, CUDA-call checks
// --------------------------------------------------------------------------------------
void set_error(const char* fmt, ...);
void clear_error();

#define RNN_FAIL(code, ...)          \
  do {                               \
    ::rnn::set_error(__VA_ARGS__);   \
    return (code);                   \
  } while (0)

#define RNN_REQUIRE(cond, code, ...)        \
  do {                                      \
    if (!(cond)) RNN_FAIL(code, __VA_ARGS__); \
  } while (0)

#define RNN_CUDA(call)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      RNN_FAIL(RNN_ERR_CUDA, "%s failed at %s:%d: %s", #call, __FILE__, __LINE__,           \
               cudaGetErrorString(e_));                                                   \
  } while (0)

#define RNN_LAUNCH_CHECK()                                                                \
  do {                                                                                    \
    cudaError_t e_ = cudaGetLastError();                                                  \
    if (e_ != cudaSuccess)                                                                \
      RNN_FAIL(RNN_ERR_CUDA, "kernel launch failed at %s:%d: %s", __FILE__, __LINE__,       \
               cudaGetErrorString(e_));                                                   \
  } while (0)

#define RNN_TRY(expr)                    \
  do {                                   \
    rnn_status s_ = (expr);              \
    if (s_ != RNN_OK) return s_;         \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// --------------------------------------------------------------------------------------
// workspace carving: a bump allocator over a caller-provided buffer (256-byte aligned)
// --------------------------------------------------------------------------------------
struct Carve {
  char* base;
  size_t used = 0;
  explicit Carve(void* b) : base(static_cast<char*>(b)) {}
  template <class T>
  T* take(size_t n) {
    used = (used + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + used) : nullptr;
    used += n * sizeof(T);
    return p;
  }
};

// --------------------------------------------------------------------------------------
// device helpers
// --------------------------------------------------------------------------------------
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ float4 ld_f4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
// L2-coherent load (bypasses L1) for data written earlier in the same launch
__device__ __forceinline__ float4 ld_f4_cg(const float* p) {
  return __ldcg(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ void st_f4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

__device__ __forceinline__ float4 f4_zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ float4 f4_fma(float a, float4 x, float4 acc) {
  acc.x = fmaf(a, x.x, acc.x); acc.y = fmaf(a, x.y, acc.y);
  acc.z = fmaf(a, x.z, acc.z); acc.w = fmaf(a, x.w, acc.w);
  return acc;
}
__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 f4_mul(float4 a, float4 b) {
  return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
}
__device__ __forceinline__ float4 f4_scale(float a, float4 b) {
  return make_float4(a * b.x, a * b.y, a * b.z, a * b.w);
}
__device__ __forceinline__ float f4_dot(float4 a, float4 b) {
  return a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
}
__device__ __forceinline__ float4 f4_shfl_xor(float4 v, int m) {
  v.x = __shfl_xor_sync(FULL, v.x, m); v.y = __shfl_xor_sync(FULL, v.y, m);
  v.z = __shfl_xor_sync(FULL, v.z, m); v.w = __shfl_xor_sync(FULL, v.w, m);
  return v;
}

// first index i in [lo, hi) with a[i] > x (a ascending); hi if none
template <class T>
__device__ __forceinline__ int64_t upper_bound_dev(const T* a, int64_t lo, int64_t hi, T x) {
  while (lo < hi) {
    int64_t mid = lo + ((hi - lo) >> 1);
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}
// first index i in [lo, hi) with a[i] >= x
template <class T>
__device__ __forceinline__ int64_t lower_bound_dev(const T* a, int64_t lo, int64_t hi, T x) {
  while (lo < hi) {
    int64_t mid = lo + ((hi - lo) >> 1);
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__device__ __forceinline__ int64_t ceil_div_dev(int64_t a, int64_t b) { return (a + b - 1) / b; }

// --------------------------------------------------------------------------------------
// internal primitives (scan_sort.cu)
// --------------------------------------------------------------------------------------
// exclusive prefix sum of in[n] (int64) into out[n+1]; out[n] = total.  in may equal out.
size_t scan_workspace_bytes(int64_t n);
rnn_status exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* ws,
                              cudaStream_t st);
// stable LSD radix sort of (key, value) pairs on the low `bits` bits of the keys.
// keys/vals are sorted in place (ping-pong through alt buffers in ws).
size_t radix_sort_workspace_bytes(int64_t n);
rnn_status radix_sort_u64(uint64_t* keys, int32_t* vals, int64_t n, int bits, void* ws,
                          cudaStream_t st);
rnn_status radix_sort_u32(uint32_t* keys, int32_t* vals, int64_t n, int bits, void* ws,
                          cudaStream_t st);

}  // namespace rnn
