// LEMX container -> device encoding (lemt io.py:177-278 layout).  The host reads the file and checks
// the header; the payload crosses the bus once (raw, packed at the declared widths) and this kernel
// scatters it into the encoding's arena: the index arrays keep their widths (byte copies into the
// 256 B-aligned slots) and omega is widened from its element format (f64 / f32 / f16 / i8) to f64.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"
#include "encode.cuh"

namespace cerdot {

namespace {

struct Spans {
  int64_t src[4], dst[4], bytes[4];
  int count;
};

__global__ void k_lemx_unpack(const unsigned char *__restrict__ payload, Spans sp, int element_bits, int64_t k,
                              int64_t omega_src, double *__restrict__ omega, unsigned char *__restrict__ arena) {
  const int which = blockIdx.y;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  if (which < sp.count) {  // an index array: 16 bytes per thread per step
    const unsigned char *src = payload + sp.src[which];
    unsigned char *dst = arena + sp.dst[which];
    const int64_t nb = sp.bytes[which];
    for (int64_t b = tid * 16; b < nb; b += stride * 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (b + j < nb) dst[b + j] = src[b + j];
    }
    return;
  }
  const int eb = element_bits / 8;  // omega: widen to f64
  for (int64_t i = tid; i < k; i += stride) {
    const unsigned char *p = payload + omega_src + i * eb;
    double v = 0.0;
    if (element_bits == 64) {
      unsigned long long u = 0;
      for (int j = 0; j < 8; ++j) u |= static_cast<unsigned long long>(p[j]) << (8 * j);
      v = __longlong_as_double(static_cast<long long>(u));
    } else if (element_bits == 32) {
      unsigned int u = 0;
      for (int j = 0; j < 4; ++j) u |= static_cast<unsigned int>(p[j]) << (8 * j);
      v = static_cast<double>(__uint_as_float(u));
    } else if (element_bits == 16) {
      const unsigned short u = static_cast<unsigned short>(p[0] | (p[1] << 8));
      v = static_cast<double>(__half2float(__ushort_as_half(u)));
    } else {
      v = static_cast<double>(static_cast<signed char>(p[0]));
    }
    omega[i] = v;
  }
}

}  // namespace

int lemx_unpack(const void *payload, int element_bits, int64_t k, int64_t omega_src, double *omega,
                const int64_t *spans, int count, void *arena, cudaStream_t st) {
  if (count < 0 || count > 4) return fail(CERDOT_E_VALUE, "lemx_unpack: 0-4 index arrays");
  if (element_bits != 8 && element_bits != 16 && element_bits != 32 && element_bits != 64)
    return fail(CERDOT_E_VALUE, "lemx_unpack: element_bits must be 8, 16, 32 or 64");
  Spans sp{};
  sp.count = count;
  int64_t most = k;
  for (int i = 0; i < count; ++i) {
    sp.src[i] = spans[3 * i];
    sp.dst[i] = spans[3 * i + 1];
    sp.bytes[i] = spans[3 * i + 2];
    most = std::max<int64_t>(most, ceil_div(sp.bytes[i], 16));
  }
  const int gx = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(most, 256), int64_t(num_sms()) * 4)));
  k_lemx_unpack<<<dim3(gx, count + 1), 256, 0, st>>>(static_cast<const unsigned char *>(payload), sp, element_bits, k,
                                                     omega_src, omega, static_cast<unsigned char *>(arena));
  CERDOT_LAUNCH_CHECK();
  return CERDOT_OK;
}

}  // namespace cerdot
