// Synthetic inputs for the benchmark and the parity tests: numpy's Generator(PCG64).choice(K, p=pmf)
// reproduced bit for bit on the device, so the 32768^2 layer (W =
// levels[default_rng(seed).choice(K, size=(m, n), p=pmf)]) is drawn in milliseconds instead of a host
// minute and is THE seeded numpy matrix, not a statistical stand-in.
//
// numpy (PCG64, XSL-RR 128/64):   state <- state * MULT + inc  (mod 2^128);  out = rotr64(hi ^ lo, state >> 122)
//   random()  = (next64 >> 11) * 2^-53
//   choice(K, p) = searchsorted(cdf, random(), side='right'),  cdf = cumsum(p) / cumsum(p)[-1]
// Element i of the draw is the output of the state advanced i + 1 steps from the generator's state.
// Lane l of a warp draws elements base + l + 32 j: one jump of 32 steps (A32 * state + C32) per draw,
// writes coalesced.  A thread reaches its first element with the O(log i) LCG jump-ahead.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace cerdot {

namespace {

struct U128 {
  uint64_t lo, hi;
};

__host__ __device__ __forceinline__ U128 mul128(U128 a, U128 b) {
#ifdef __CUDA_ARCH__
  const uint64_t lo = a.lo * b.lo;
  const uint64_t hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
#else
  const unsigned __int128 p = static_cast<unsigned __int128>(a.lo) * b.lo;
  const uint64_t lo = static_cast<uint64_t>(p);
  const uint64_t hi = static_cast<uint64_t>(p >> 64) + a.hi * b.lo + a.lo * b.hi;
#endif
  return {lo, hi};
}

__host__ __device__ __forceinline__ U128 add128(U128 a, U128 b) {
  const uint64_t lo = a.lo + b.lo;
  return {lo, a.hi + b.hi + (lo < a.lo ? 1ull : 0ull)};
}

constexpr U128 kMult{0x4385DF649FCCF645ull, 0x2360ED051FC65DA4ull};

// Jump parameters of `delta` LCG steps: state' = mult * state + plus (the PCG paper's advance).
__host__ __device__ __forceinline__ void jump(U128 inc, uint64_t delta, U128 &mult, U128 &plus) {
  U128 am{1, 0}, ap{0, 0}, cm = kMult, cp = inc;
  while (delta) {
    if (delta & 1) {
      am = mul128(am, cm);
      ap = add128(mul128(ap, cm), cp);
    }
    cp = mul128(add128(cm, U128{1, 0}), cp);
    cm = mul128(cm, cm);
    delta >>= 1;
  }
  mult = am;
  plus = ap;
}

__device__ __forceinline__ uint64_t xsl_rr(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = static_cast<unsigned>(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

constexpr int kSynthThreads = 256;
constexpr int kPerLane = 64;  // draws per lane

__global__ void __launch_bounds__(kSynthThreads) k_choice(U128 s0, U128 inc, uint64_t offset, const double *cdf_g,
                                                          const float *levels_g, int k, int64_t count,
                                                          float *__restrict__ out) {
  extern __shared__ unsigned char sm[];
  double *cdf = reinterpret_cast<double *>(sm);
  float *lv = reinterpret_cast<float *>(cdf + k);
  for (int i = threadIdx.x; i < k; i += kSynthThreads) {
    cdf[i] = cdf_g[i];
    lv[i] = levels_g[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * kSynthThreads + threadIdx.x) >> 5;
  const int64_t base = warp * 32 * kPerLane;
  if (base >= count) return;
  U128 m, p;
  jump(inc, offset + static_cast<uint64_t>(base + lane) + 1u, m, p);
  U128 s = add128(mul128(m, s0), p);
  U128 m32, p32;
  jump(inc, 32, m32, p32);
  for (int j = 0; j < kPerLane; ++j) {
    const int64_t e = base + lane + 32 * j;
    if (e >= count) break;
    const double u = static_cast<double>(xsl_rr(s) >> 11) * (1.0 / 9007199254740992.0);
    int lo = 0, hi = k;  // first index with cdf[idx] > u  (searchsorted side='right')
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cdf[mid] <= u) lo = mid + 1; else hi = mid;
    }
    out[e] = lv[min(lo, k - 1)];
    s = add128(mul128(m32, s), p32);
  }
}

}  // namespace

int synth_choice(const uint64_t *state, const uint64_t *inc, uint64_t offset, const double *cdf, const float *levels,
                 int32_t k, int64_t count, float *out, cudaStream_t st) {
  if (k <= 0 || k > 4096) return fail(CERDOT_E_VALUE, "synth: 1 <= k <= 4096");
  if (count <= 0) return CERDOT_OK;
  const int64_t per_block = static_cast<int64_t>(kSynthThreads) * kPerLane;
  const int64_t grid = ceil_div(count, per_block);
  if (grid > 2147483647) return fail(CERDOT_E_VALUE, "synth: count too large");
  const size_t smem = static_cast<size_t>(k) * (sizeof(double) + sizeof(float));
  k_choice<<<static_cast<unsigned>(grid), kSynthThreads, smem, st>>>(U128{state[0], state[1]}, U128{inc[0], inc[1]},
                                                                     offset, cdf, levels, k, count, out);
  CERDOT_LAUNCH_CHECK();
  return CERDOT_OK;
}

}  // namespace cerdot
