// CER / CSER dot product on sm_100a, fp32.
//
// Reference: lemt kernels.py:283-301 (_dot_segmented) evaluated in float64:
//   y[r] = sum_seg (omega[seg] - bg) * (sum_{i in seg} x[colI[i]])  (+ bg * sum(x) if bg != 0)
// Summation order here (stated for the 1e-5 parity bar):
//   * inner per-segment sums: sequential fp32 in colI order,
//   * one fp32 fma per non-empty segment into a per-lane row accumulator,
//   * lanes combined by a fixed xor-butterfly (deterministic),
//   * background correction: sum(x) in fp64 (fixed tree), bg * sum in fp64,
//     added to the fp32 row sum in fp64 and rounded once.
// The segment value is (float)(omega[k] - bg) computed in fp64 per segment.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "common.cuh"
#include "encode.cuh"

namespace cerdot {

namespace {

struct DotArgs {
  const double *omega;
  const void *col;
  const void *op;
  const void *rp;
  const void *oi;
  int rp_bits, oi_bits;
  int64_t m, n;
  double bg;
  const double *colsum;  // batch doubles when bg != 0
};

template <typename T>
__device__ __forceinline__ uint32_t ld_idx(const T *p, int64_t i) {
  return __ldg(p + i);
}

__device__ __forceinline__ float seg_value(const DotArgs &a, bool cser, int64_t s, int64_t s0) {
  const int64_t k = cser ? static_cast<int64_t>(load_index(a.oi, a.oi_bits, s)) : (s - s0 + 1);
  return static_cast<float>(__ldg(a.omega + k) - a.bg);
}

// Mat-vec: warp per row, lanes stride over the row's segments.
template <typename ColT, typename PtrT, bool CSER>
__global__ void __launch_bounds__(256) k_dot_vec(DotArgs a, const float *__restrict__ x, float *__restrict__ y) {
  const ColT *col = static_cast<const ColT *>(a.col);
  const PtrT *op = static_cast<const PtrT *>(a.op);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < a.m; row += nwarps) {
    const int64_t s0 = load_index(a.rp, a.rp_bits, row), s1 = load_index(a.rp, a.rp_bits, row + 1);
    float acc = 0.f;
    for (int64_t s = s0 + lane; s < s1; s += 32) {
      const int64_t e0 = ld_idx(op, s), e1 = ld_idx(op, s + 1);
      if (e1 > e0) {
        float sum = 0.f;
        for (int64_t i = e0; i < e1; ++i) sum += __ldg(x + ld_idx(col, i));
        acc = fmaf(seg_value(a, CSER, s, s0), sum, acc);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) y[row] = a.bg != 0.0 ? static_cast<float>(static_cast<double>(acc) + a.bg * a.colsum[0]) : acc;
  }
}

// Mat-mat: warp per row, lanes across V-wide column groups of the batch.
template <typename ColT, typename PtrT, bool CSER, int V>
__global__ void __launch_bounds__(256) k_dot_mat(DotArgs a, const float *__restrict__ x, int64_t ldx, int64_t batch,
                                                 float *__restrict__ y, int64_t ldy) {
  const ColT *col = static_cast<const ColT *>(a.col);
  const PtrT *op = static_cast<const PtrT *>(a.op);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < a.m; row += nwarps) {
    const int64_t s0 = load_index(a.rp, a.rp_bits, row), s1 = load_index(a.rp, a.rp_bits, row + 1);
    for (int64_t c0 = 0; c0 < batch; c0 += 32 * V) {
      const int64_t cb = c0 + lane * V;
      const bool full = cb + V <= batch;
      float acc[V];
#pragma unroll
      for (int j = 0; j < V; ++j) acc[j] = 0.f;
      for (int64_t s = s0; s < s1; ++s) {
        const int64_t e0 = ld_idx(op, s), e1 = ld_idx(op, s + 1);
        if (e1 <= e0) continue;
        float sum[V];
#pragma unroll
        for (int j = 0; j < V; ++j) sum[j] = 0.f;
        for (int64_t i = e0; i < e1; ++i) {
          const float *xr = x + static_cast<int64_t>(ld_idx(col, i)) * ldx + cb;
          if (V == 4 && full) {
            const float4 v = __ldg(reinterpret_cast<const float4 *>(xr));
            sum[0] += v.x; sum[1] += v.y; sum[2] += v.z; sum[V - 1] += v.w;
          } else if (V == 2 && full) {
            const float2 v = __ldg(reinterpret_cast<const float2 *>(xr));
            sum[0] += v.x; sum[V - 1] += v.y;
          } else {
#pragma unroll
            for (int j = 0; j < V; ++j)
              if (cb + j < batch) sum[j] += __ldg(xr + j);
          }
        }
        const float v = seg_value(a, CSER, s, s0);
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = fmaf(v, sum[j], acc[j]);
      }
      float *yr = y + row * ldy;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int64_t c = cb + j;
        if (c < batch)
          yr[c] = a.bg != 0.0 ? static_cast<float>(static_cast<double>(acc[j]) + a.bg * a.colsum[c]) : acc[j];
      }
    }
  }
}

// Column sums of x (n x batch, row stride ldx) in fp64, fixed reduction order.
__global__ void __launch_bounds__(256) k_colsum(const float *__restrict__ x, int64_t n, int64_t ldx, int64_t batch,
                                                double *__restrict__ out) {
  __shared__ double part[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * 32 + tx;
  double s = 0.0;
  if (c < batch)
    for (int64_t r = ty; r < n; r += 8) s += static_cast<double>(__ldg(x + r * ldx + c));
  part[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && c < batch) {
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += part[j][tx];
    out[c] = t;
  }
}

// Mat-vec column sum: one CTA tree reduction.
__global__ void __launch_bounds__(1024) k_vecsum(const float *__restrict__ x, int64_t n, double *__restrict__ out) {
  __shared__ double part[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += static_cast<double>(__ldg(x + i));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = part[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) out[0] = s;
  }
}

template <typename ColT, typename PtrT, bool CSER>
int launch_dot(const DotArgs &a, const float *x, int64_t ldx, int64_t batch, float *y, int64_t ldy, cudaStream_t st) {
  const int64_t warps_per_block = 8;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(a.m, warps_per_block),
                                                                           static_cast<int64_t>(num_sms()) * 64)));
  if (batch == 1) {
    k_dot_vec<ColT, PtrT, CSER><<<grid, 256, 0, st>>>(a, x, y);
  } else {
    const bool al4 = (ldx % 4 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0);
    const bool al2 = (ldx % 2 == 0) && (reinterpret_cast<uintptr_t>(x) % 8 == 0);
    if (batch >= 128 && al4)
      k_dot_mat<ColT, PtrT, CSER, 4><<<grid, 256, 0, st>>>(a, x, ldx, batch, y, ldy);
    else if (batch >= 64 && al2)
      k_dot_mat<ColT, PtrT, CSER, 2><<<grid, 256, 0, st>>>(a, x, ldx, batch, y, ldy);
    else
      k_dot_mat<ColT, PtrT, CSER, 1><<<grid, 256, 0, st>>>(a, x, ldx, batch, y, ldy);
  }
  CERDOT_LAUNCH_CHECK();
  return CERDOT_OK;
}

template <typename ColT, bool CSER>
int by_ptr(const DotArgs &a, int op_bits, const float *x, int64_t ldx, int64_t batch, float *y, int64_t ldy,
           cudaStream_t st) {
  switch (op_bits) {
    case 8: return launch_dot<ColT, uint8_t, CSER>(a, x, ldx, batch, y, ldy, st);
    case 16: return launch_dot<ColT, uint16_t, CSER>(a, x, ldx, batch, y, ldy, st);
    default: return launch_dot<ColT, uint32_t, CSER>(a, x, ldx, batch, y, ldy, st);
  }
}

template <bool CSER>
int by_col(const DotArgs &a, int col_bits, int op_bits, const float *x, int64_t ldx, int64_t batch, float *y,
           int64_t ldy, cudaStream_t st) {
  switch (col_bits) {
    case 8: return by_ptr<uint8_t, CSER>(a, op_bits, x, ldx, batch, y, ldy, st);
    case 16: return by_ptr<uint16_t, CSER>(a, op_bits, x, ldx, batch, y, ldy, st);
    default: return by_ptr<uint32_t, CSER>(a, op_bits, x, ldx, batch, y, ldy, st);
  }
}

}  // namespace

int dot(const cerdot_matrix *mat, const float *x, int64_t ldx, int64_t batch, float *y, int64_t ldy, void *workspace,
        size_t workspace_bytes, cudaStream_t st) {
  const bool cser = mat->kind == CERDOT_CSER;
  DotArgs a{};
  a.omega = mat->omega;
  a.col = mat->col_index;
  a.op = mat->omega_ptr;
  a.rp = mat->row_ptr;
  a.oi = mat->omega_index;
  a.rp_bits = mat->row_ptr_bits;
  a.oi_bits = mat->omega_index_bits;
  a.m = mat->m;
  a.n = mat->n;
  a.bg = mat->background;
  if (a.m == 0 || batch == 0) return CERDOT_OK;
  if (a.bg != 0.0) {
    if (workspace == nullptr || workspace_bytes < sizeof(double) * static_cast<size_t>(batch))
      return fail(CERDOT_E_WORKSPACE, "dot workspace too small for the background column sums");
    double *cs = static_cast<double *>(workspace);
    if (batch == 1)
      k_vecsum<<<1, 1024, 0, st>>>(x, a.n, cs);
    else
      k_colsum<<<static_cast<int>(ceil_div(batch, 32)), 256, 0, st>>>(x, a.n, ldx, batch, cs);
    CERDOT_LAUNCH_CHECK();
    a.colsum = cs;
  }
  return cser ? by_col<true>(a, mat->col_bits, mat->omega_ptr_bits, x, ldx, batch, y, ldy, st)
              : by_col<false>(a, mat->col_bits, mat->omega_ptr_bits, x, ldx, batch, y, ldy, st);
}

}  // namespace cerdot
