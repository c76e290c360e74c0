// Shared device helpers for the cerdot kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "cerdot.h"

namespace cerdot {

// ---------------------------------------------------------------- errors
void set_error(const std::string &msg);
int fail(int status, const std::string &msg);
int cuda_fail(cudaError_t err, const char *where);

#define CERDOT_CUDA_CHECK(expr)                               \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return ::cerdot::cuda_fail(_e, #expr); \
  } while (0)

#define CERDOT_LAUNCH_CHECK() CERDOT_CUDA_CHECK(cudaGetLastError())

// ---------------------------------------------------------------- value keys
// A float64 value is keyed by an order-preserving u64 so integer compares give
// np.sort's order: -0.0 and +0.0 share the key of +0.0 (np.unique compares
// values), every NaN shares one key above +inf (np.unique equal_nan).
// Key 0 is the image of bit pattern 0xFFFF...F (a NaN), which canonicalises
// away, so 0 marks an empty hash slot.
constexpr uint64_t kEmptyKey = 0ull;

__host__ __device__ __forceinline__ uint64_t canon_bits(double v) {
  if (v != v) return 0x7ff8000000000000ull;
  if (v == 0.0) return 0ull;
#ifdef __CUDA_ARCH__
  return static_cast<uint64_t>(__double_as_longlong(v));
#else
  uint64_t b;
  __builtin_memcpy(&b, &v, 8);
  return b;
#endif
}

__host__ __device__ __forceinline__ uint64_t order_key(uint64_t bits) {
  return (bits >> 63) ? ~bits : (bits | 0x8000000000000000ull);
}

__host__ __device__ __forceinline__ uint64_t value_key(double v) { return order_key(canon_bits(v)); }

__host__ __device__ __forceinline__ double key_value(uint64_t key) {
  uint64_t bits = (key >> 63) ? (key & 0x7fffffffffffffffull) : ~key;
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(bits));
#else
  double v;
  __builtin_memcpy(&v, &bits, 8);
  return v;
#endif
}

__host__ __device__ __forceinline__ uint32_t hash_key(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return static_cast<uint32_t>(k);
}

template <typename T>
__device__ __forceinline__ double as_double(T v) {
  return static_cast<double>(v);
}

// ---------------------------------------------------------------- index widths
__device__ __forceinline__ uint32_t load_index(const void *p, int bits, int64_t i) {
  switch (bits) {
    case 8:
      return __ldg(static_cast<const uint8_t *>(p) + i);
    case 16:
      return __ldg(static_cast<const uint16_t *>(p) + i);
    default:
      return __ldg(static_cast<const uint32_t *>(p) + i);
  }
}

__device__ __forceinline__ void store_index(void *p, int bits, int64_t i, uint64_t v) {
  switch (bits) {
    case 8:
      static_cast<uint8_t *>(p)[i] = static_cast<uint8_t>(v);
      break;
    case 16:
      static_cast<uint16_t *>(p)[i] = static_cast<uint16_t>(v);
      break;
    default:
      static_cast<uint32_t *>(p)[i] = static_cast<uint32_t>(v);
      break;
  }
}

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

int num_sms();

}  // namespace cerdot
