// Device/host helpers shared by the dot-product translation units (dot.cu, dot_stream.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"
#include "tileview.cuh"

namespace cerdot {

struct DotArgs {
  const double *omega;
  const void *col;
  const void *op;
  const void *rp;
  const void *oi;
  int rp_bits, oi_bits;
  int64_t m, n, k;
  int mode;  // position of the background in omega (CER: 0)
  double bg;
  const double *colsum;  // batch doubles when bg != 0
  int64_t segs;          // segment count (omegaPtr has segs + 1 entries)
  int64_t nnz;           // entries (len(colI))
  int64_t max_row_nnz, max_row_segs;
  const uint32_t *re;  // optional row_entry index (m+1): re[r] = op[rp[r]]
  int dbg;  // CERDOT_TRACE: print per-CTA phase timestamps (debug only)
  // fused output exchange (cerdot_dot_peers): every y element is also stored at ypeer_off + i of each
  // peer's output buffer (NVLink P2P stores); npeer = 0 for a plain dot
  float *const *ypeer;
  int npeer;
  int64_t ypeer_off;
};

// The one-row-per-warp mat-vec (dot_row.cu).
bool matvec_row_fits(const DotArgs &a, size_t col_bytes);
int matvec_row(const DotArgs &a, bool cser, int col_bits, int op_bits, const float *x, float *y, cudaStream_t st);

// The long-row mat-vec (dot_stream.cu).
bool matvec_stream_fits(int64_t k, int64_t n, int op_bits, int oi_bits);
int matvec_stream(const DotArgs &a, bool cser, int col_bits, int op_bits, const float *x, float *y, cudaStream_t st);

namespace {

constexpr int kMatvecThreads = 512;
constexpr int kMatvecWarps = kMatvecThreads / 32;
constexpr int kSmemValues = 4096;             // omega entries cached in smem
constexpr int kMaxSmemBytes = 227 * 1024;
constexpr size_t kHalfSmemBytes = 112 * 1024;  // two CTAs per SM (228 KB minus 1 KB reserved each)


// y[i] = v, and the same element of every peer's output (the row-sharded all-gather, fused).
__device__ __forceinline__ void put_y(const DotArgs &a, float *y, int64_t i, float v) {
  y[i] = v;
  for (int p = 0; p < a.npeer; ++p) a.ypeer[p][a.ypeer_off + i] = v;
}

// Raise a kernel's dynamic shared-memory limit once per kernel (and device) -- the host call costs ~us.
template <typename K>
int allow_max_smem(K kern) {
  static std::mutex mu;
  static std::set<std::pair<const void *, int>> done;
  int dev = 0;
  CERDOT_CUDA_CHECK(cudaGetDevice(&dev));
  const auto key = std::make_pair(reinterpret_cast<const void *>(kern), dev);
  {
    std::lock_guard<std::mutex> lock(mu);
    if (done.count(key)) return CERDOT_OK;
  }
  CERDOT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  std::lock_guard<std::mutex> lock(mu);
  done.insert(key);
  return CERDOT_OK;
}

// Resident CTAs per SM of a kernel at `threads` threads (no dynamic shared memory), cached per kernel
// and device.  (Keyed by the kernel's address: every k_matmat_flat instance has the same C++ type.)
template <typename K>
int blocks_per_sm(K kern, int threads, int *out) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, int> cache;
  int dev = 0;
  CERDOT_CUDA_CHECK(cudaGetDevice(&dev));
  const auto key = std::make_pair(reinterpret_cast<const void *>(kern), dev);
  {
    std::lock_guard<std::mutex> lock(mu);
    const auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return CERDOT_OK;
    }
  }
  int n = 0;
  CERDOT_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, 0));
  std::lock_guard<std::mutex> lock(mu);
  cache[key] = n;
  *out = n;
  return CERDOT_OK;
}

template <typename T>
__device__ __forceinline__ uint32_t ld_idx(const T *p, int64_t i) {
  return __ldg(p + i);
}

// 16-byte vector of indices -> unpacked u32 lanes
template <typename ColT>
struct ColVec;
template <>
struct ColVec<uint8_t> {
  static constexpr int kPer = 16;
  __device__ static void unpack(const uint4 &v, uint32_t *out) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int b = 0; b < 4; ++b) out[4 * i + b] = (w[i] >> (8 * b)) & 0xffu;
  }
};
template <>
struct ColVec<uint16_t> {
  static constexpr int kPer = 8;
  __device__ static void unpack(const uint4 &v, uint32_t *out) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      out[2 * i] = w[i] & 0xffffu;
      out[2 * i + 1] = w[i] >> 16;
    }
  }
};
template <>
struct ColVec<uint32_t> {
  static constexpr int kPer = 4;
  __device__ static void unpack(const uint4 &v, uint32_t *out) {
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
  }
};

__device__ __forceinline__ uint4 ld_stream(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// TMA-engine prefetch of a contiguous global range into L2 (no registers, no smem).
__device__ __forceinline__ void bulk_prefetch_l2(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

constexpr int kFifoDepth = 4;

__device__ __forceinline__ void cp_async4(void *smem_dst, const void *gmem_src) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int kEPL = 32;                      // entries per lane per window
constexpr uint32_t kWin = 32 * kEPL;          // entries per window

// Window-local prefix table of a warp: entry position p (lane p/32, item j=p%32) lives at
// (j/4)*128 + lane*4 + j%4 so each lane writes its 32 prefixes as eight conflict-free 16 B stores.
__device__ __forceinline__ uint32_t ppos(uint32_t p) { return ((p & 31u) >> 2) * 128u + (p >> 5) * 4u + (p & 3u); }

// Gather x for one lane's 32 window entries (MASKED: only entries in [e0, e1)), build the lane's
// running prefix sums and store them to the warp's prefix table; returns the lane total.
template <typename ColT, bool XSMEM, bool MASKED>
__device__ __forceinline__ float gather_prefix(const uint4 *raw_v, uint32_t w0, uint32_t e0, uint32_t e1,
                                               const float *__restrict__ xs, const float *__restrict__ x, float *pre,
                                               int lane) {
  using CV = ColVec<ColT>;
  constexpr int NV = kEPL / CV::kPer;
  const uint32_t p0 = w0 + lane * kEPL;
  uint32_t vmask = 0xffffffffu;
  if (MASKED) {
    const uint32_t jlo = e0 > p0 ? min(e0 - p0, 32u) : 0u;
    const uint32_t jhi = e1 > p0 ? min(e1 - p0, 32u) : 0u;
    vmask = (jhi >= 32u ? 0xffffffffu : ((1u << jhi) - 1u)) & ~(jlo >= 32u ? 0xffffffffu : ((1u << jlo) - 1u));
  }
  float run = 0.f;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    uint32_t c[CV::kPer];
    CV::unpack(raw_v[v], c);
#pragma unroll
    for (int q = 0; q < CV::kPer / 4; ++q) {
      float o[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int j = v * CV::kPer + q * 4 + t;
        float g;
        if (MASKED) {
          g = 0.f;
          if ((vmask >> j) & 1u) g = XSMEM ? xs[c[q * 4 + t]] : __ldg(x + c[q * 4 + t]);
        } else {
          g = XSMEM ? xs[c[q * 4 + t]] : __ldg(x + c[q * 4 + t]);
        }
        run += g;
        o[t] = run;
      }
      const int jq = (v * CV::kPer + q * 4) >> 2;
      *reinterpret_cast<float4 *>(pre + jq * 128 + lane * 4) = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
  return run;
}



}  // namespace
}  // namespace cerdot
