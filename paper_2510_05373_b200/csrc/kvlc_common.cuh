// Shared host/device helpers for libkvlinc (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <cmath>

#include "../../include/kvlinc.h"

namespace kvlc {

// ---- error plumbing (thread-local message, reference ValueError wording) ----
void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);
int check_launch(const char* what);
bool device_ok();

#define KVLC_REQUIRE(cond, ...)                        \
  do {                                                 \
    if (!(cond)) return ::kvlc::fail(KVLC_EINVAL, __VA_ARGS__); \
  } while (0)

#define KVLC_CUDA(expr)                                                        \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess)                                                     \
      return ::kvlc::fail(KVLC_ECUDA, "CUDA error %s at %s:%d",                \
                          cudaGetErrorString(_e), __FILE__, __LINE__);         \
  } while (0)

#define KVLC_NEED_DEVICE()                                                     \
  do {                                                                         \
    if (!::kvlc::device_ok())                                                  \
      return ::kvlc::fail(KVLC_ENODEV,                                         \
                          "no sm_100 CUDA device: libkvlinc has no CPU path"); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
void note_cache_write(const kvlc_cache* c);  // kvlc_api.cu: the next decode of `c` waits fully
bool take_cache_write(const kvlc_cache* c);  // true (and cleared) if `c` was marked

// Fragment-native code words (kvlc_flush.cu pack_k_word / pack_v_word) are stored rotated
// left by 2 bits: code (byte q, bit pair j) sits at bit (8 q + 2 j + 2) mod 32, so the
// decode's fp16 operands (x & (0x000C000C << 2 j), and the same on x rotated right by 8)
// are c 4^(j+1) 2^-24 rather than c 4^j 2^-24.  The smallest subnormals (c 2^-24) lost
// low-order product bits in the tensor core (rows of j = 0 carried a -8e-6 bias in the
// output at 131k tokens, 17x the j = 1 rows; tools/decode_err_diag.py).
__device__ __forceinline__ uint32_t frag_store(uint32_t w) { return __funnelshift_l(w, w, 2); }
__device__ __forceinline__ uint32_t frag_load(uint32_t w) { return __funnelshift_r(w, w, 2); }

inline int lane_bits(int bits) { return bits == 2 ? 2 : (bits == 8 ? 8 : 4); }
inline int lanes_per_word(int bits) { return 32 / lane_bits(bits); }
inline bool valid_bits(int bits) { return bits == 2 || bits == 3 || bits == 4 || bits == 8; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline bool pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Carves a caller workspace into aligned sub-buffers.
struct Arena {
  char* base;
  size_t cap, off = 0;
  Arena(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <typename T>
  T* take(size_t n) {
    size_t need = align_up(n * sizeof(T));
    if (base == nullptr || off + need > cap) return nullptr;
    T* p = reinterpret_cast<T*>(base + off);
    off += need;
    return p;
  }
};

// ---- device helpers ----
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// The reference's code decision (quantize.py:131-134 / 202-207):
//   scale = (max - min) / top;  code = clip(rint((x - min) / scale), 0, top)
// in float64 with IEEE division (no reciprocal) and half-to-even rint.
__device__ __forceinline__ uint32_t code_of(double x, double mn, double scale, int top) {
  if (!(scale > 0.0)) return 0u;
  double q = rint(__ddiv_rn(__dsub_rn(x, mn), scale));
  q = fmin(fmax(q, 0.0), (double)top);
  return (uint32_t)q;
}

}  // namespace kvlc
