// CER / CSER mat-vec (batch 1) when every row fits one 1024-entry window: the row kernel (k_matvec_row).
//
// Reference: lemt kernels.py:283-301 (_dot_segmented):
//   y[r] = sum_seg (omega[seg] - bg) * (sum_{i in seg} x[colI[i]])  (+ bg * sum(x) when bg != 0)
//
// The window kernel (k_matvec, dot.cu) carries machinery for rows of any length (a window generator three
// windows ahead, a cp.async segment ring, TMA L2 prefetch of the streams): ~1030 warp instructions per
// AlexNet-fc6 row, of which about half is that machinery, issued between the first index load and the
// colI loads it gates.  With <= 1017 entries per row none of it is needed: a warp reads its row bounds,
// issues the whole row's colI (four 16 B loads per lane) and its segment ends at once, waits for x, and
// runs the window kernel's single-window arithmetic unchanged -- so its results are bitwise those of
// k_matvec (tests/test_gpu_parity.py::test_row_kernel_bitwise_equals_window_kernel):
//   * 32 gathers per lane from the x copy in shared memory, fp32 lane-local prefixes to the warp's prefix
//     table, lane totals scanned in fp64 and kept as fp32 (hi, lo) pairs;
//   * lane i of batch t takes segment 32 t + i: sum = G(end) - G(start - 1), the start's lane-local
//     prefix being the previous segment's end value (shuffled); one fp32 fma per segment;
//   * xor butterfly per row.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"
#include "dotk.cuh"

namespace cerdot {

namespace {

constexpr int kRowNT = 896;  // 28 warps per SM: a 4096-row layer has at most one row per warp on 148 SMs

constexpr uint32_t kRowStage = 1024;  // results a CTA can stage for the fused exchange's coalesced peer stores

struct RowSmem {
  uint32_t bar, wv, pre, off, ystage, xs, total;
};
__host__ __device__ __forceinline__ RowSmem row_layout(int64_t k, int64_t n, uint32_t warps) {
  RowSmem L{};
  uint32_t o = 0;
  auto take = [&](uint32_t bytes) {
    const uint32_t r = o;
    o += (bytes + 15u) & ~15u;
    return r;
  };
  L.bar = take(16u);
  L.wv = take(static_cast<uint32_t>(k) * 4u);
  L.pre = take(warps * kWin * 4u);
  L.off = take(warps * 32u * 8u);
  L.ystage = take(kRowStage * 4u);
  L.xs = take(static_cast<uint32_t>(n) * 4u);
  L.total = o;
  return L;
}

template <typename ColT, typename PtrT, bool CSER, bool PEERS>
__global__ void __launch_bounds__(kRowNT, 1) k_matvec_row(DotArgs a, const float *__restrict__ x,
                                                          float *__restrict__ y) {
  constexpr int kWarps = kRowNT / 32;
  using CV = ColVec<ColT>;
  constexpr int NV = kEPL / CV::kPer;
  constexpr uint32_t kAlign = CV::kPer;
  constexpr uint32_t kFull = 0xffffffffu;
  constexpr int kPre = 4;  // segment batches whose bounds are loaded with the row (128 segments)
  extern __shared__ __align__(16) unsigned char smem[];
  const RowSmem L = row_layout(a.k, a.n, kWarps);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float *wv = reinterpret_cast<float *>(smem + L.wv);
  float *pre = reinterpret_cast<float *>(smem + L.pre) + wid * kWin;
  float2 *off = reinterpret_cast<float2 *>(smem + L.off) + wid * 32;
  float *xs = reinterpret_cast<float *>(smem + L.xs);
  uint64_t *xbar = reinterpret_cast<uint64_t *>(smem + L.bar), *wbar = xbar + 1;
  const ColT *col = static_cast<const ColT *>(a.col);
  const PtrT *op = static_cast<const PtrT *>(a.op);
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kWarps;
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kWarps + wid;
  const uint32_t R0 = static_cast<uint32_t>(gw * a.m / nw), R1 = static_cast<uint32_t>((gw + 1) * a.m / nw);
  pdl_launch_dependents();
  const bool x_async = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const uint32_t x_tma = x_async ? static_cast<uint32_t>(a.n * 4) & ~15u : 0u;
  if (threadIdx.x == 0) {
    mbar_init(xbar, 1);           // x: thread 0's arrive + the TMA bytes
    mbar_init(wbar, blockDim.x);  // value table: every thread arrives once its share is stored
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // ---- the first row's index loads, all in flight before anything waits: bounds (lanes 0-3), then colI
  // and the segment ends, which depend only on the bounds
  auto bounds = [&](uint32_t r, uint32_t &e0, uint32_t &e1, uint32_t &s0, uint32_t &s1) {
    uint32_t v = 0;
    if (lane < 2) v = a.re ? __ldg(a.re + r + lane) : ld_idx(op, load_index(a.rp, a.rp_bits, r + lane));
    else if (lane < 4) v = load_index(a.rp, a.rp_bits, r + lane - 2);
    e0 = __shfl_sync(kFull, v, 0);
    e1 = __shfl_sync(kFull, v, 1);
    s0 = __shfl_sync(kFull, v, 2);
    s1 = __shfl_sync(kFull, v, 3);
  };
  uint32_t e0 = 0, e1 = 0, s0 = 0, s1 = 0;
  uint4 raw[NV];
  uint32_t pen[kPre], pk[kPre];
  auto row_loads = [&](uint32_t r) {
    bounds(r, e0, e1, s0, s1);
    const uint32_t w0 = e0 & ~(kAlign - 1u);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const uint32_t vp = w0 + lane * kEPL + v * CV::kPer;
      raw[v] = vp < e1 ? ld_stream(col + vp) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int i = 0; i < kPre; ++i) {
      const uint32_t sidx = s0 + lane + 32u * i;
      pen[i] = sidx < s1 ? ld_idx(op, sidx + 1) : 0u;
      pk[i] = sidx < s1 ? (CSER ? load_index(a.oi, a.oi_bits, sidx) : sidx - s0 + 1u) : 0u;
    }
  };
  if (R0 < R1) row_loads(R0);

  // ---- x: one TMA bulk copy once the producer grid is done (thread 0); the value table by all threads
  if (x_async) {
    if (threadIdx.x == 0) {
      pdl_wait();
      for (int64_t i = x_tma >> 2; i < a.n; ++i) xs[i] = __ldg(x + i);
      mbar_expect_tx(xbar, x_tma);
      constexpr uint32_t kChunk = 32768;
      for (uint32_t o = 0; o < x_tma; o += kChunk)
        bulk_g2s(reinterpret_cast<unsigned char *>(xs) + o, reinterpret_cast<const unsigned char *>(x) + o,
                 min(kChunk, x_tma - o), xbar);
    }
  } else {  // misaligned x: cooperative staging
    pdl_wait();
    for (int64_t i = threadIdx.x; i < a.n; i += kRowNT) xs[i] = __ldg(x + i);
    __syncthreads();
    if (threadIdx.x == 0) mbar_expect_tx(xbar, 0u);
  }
  for (int i = threadIdx.x; i < a.k; i += kRowNT) wv[i] = static_cast<float>(__ldg(a.omega + i) - a.bg);
  mbar_arrive(wbar);
  pdl_wait();  // y may be read or written by the producer grid
  bool ready = false;
  const float y_empty = a.bg != 0.0 ? static_cast<float>(a.bg * a.colsum[0]) : 0.f;
  // Row-sharded exchange (peers): the CTA's rows are contiguous, so their results are staged in shared
  // memory and written to y and to every peer's buffer as coalesced stores at the end (one 4-byte NVLink
  // store per row per peer otherwise).  Without peers a result is stored as soon as its row is done.
  const uint32_t cta_r0 = static_cast<uint32_t>(static_cast<uint64_t>(blockIdx.x) * kWarps * a.m / nw);
  const uint32_t cta_r1 = static_cast<uint32_t>((static_cast<uint64_t>(blockIdx.x) + 1) * kWarps * a.m / nw);
  const bool staged = PEERS && cta_r1 - cta_r0 <= kRowStage;  // (a separate instance: the plain one keeps its registers)
  float *ystage = reinterpret_cast<float *>(smem + L.ystage);
  auto emit = [&](uint32_t row, float v) {
    if (staged) ystage[row - cta_r0] = v;
    else put_y(a, y, row, v);
  };

  for (uint32_t r = R0; r < R1; ++r) {
    if (r != R0) row_loads(r);
    if (e1 <= e0) {  // empty row
      if (lane == 0) emit(r, y_empty);
      continue;
    }
    const uint32_t w0 = e0 & ~(kAlign - 1u), wn = w0 + kWin;
    if (!ready) {
      mbar_wait(xbar, 0);
      mbar_wait(wbar, 0);
      ready = true;
    }
    const float run = (w0 >= e0 && wn <= e1) ? gather_prefix<ColT, true, false>(raw, w0, e0, e1, xs, x, pre, lane)
                                             : gather_prefix<ColT, true, true>(raw, w0, e0, e1, xs, x, pre, lane);
    // lane offsets: exclusive scan of the lane totals in fp64, kept as an fp32 pair (dot.cu, k_matvec)
    double incl = run;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double t = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += t;
    }
    {
      const double up = __shfl_up_sync(kFull, incl, 1);
      const double excl = lane ? up : 0.0;
      const float hi = static_cast<float>(excl);
      off[lane] = make_float2(hi, static_cast<float>(excl - static_cast<double>(hi)));
    }
    __syncwarp();
    float acc = 0.f;
    uint32_t e_prev = e0;  // end of the previous segment
    float p_prev = 0.f;    // its lane-local prefix
    auto seg = [&](uint32_t en, uint32_t k, bool valid) {
      const bool has = valid && en > w0;
      const float pe = has ? pre[ppos(en - 1u - w0)] : 0.f;
      uint32_t st = __shfl_up_sync(kFull, en, 1);
      float ps = __shfl_up_sync(kFull, pe, 1);
      if (lane == 0) {
        st = e_prev;
        ps = p_prev;
      }
      e_prev = __shfl_sync(kFull, en, 31);
      p_prev = __shfl_sync(kFull, pe, 31);
      if (valid && en > st) {
        const float2 oe = off[(en - 1u - w0) >> 5];
        float hi = oe.x, lo = oe.y + pe;
        if (st > w0) {
          const float2 os = off[(st - 1u - w0) >> 5];
          hi -= os.x;
          lo -= os.y + ps;
        }
        acc = fmaf(wv[k], hi + lo, acc);
      }
    };
#pragma unroll
    for (int i = 0; i < kPre; ++i) seg(pen[i], pk[i], s0 + lane + 32u * i < s1);
    for (uint32_t base = s0 + 32u * kPre; base < s1; base += 32) {  // rows with more than 128 segments
      const uint32_t sidx = base + lane;
      const bool valid = sidx < s1;
      const uint32_t en = valid ? ld_idx(op, sidx + 1) : 0u;
      const uint32_t k = valid ? (CSER ? load_index(a.oi, a.oi_bits, sidx) : sidx - s0 + 1u) : 0u;
      seg(en, k, valid);
    }
    __syncwarp();  // the tables are rewritten by the next row
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if (lane == 0) emit(r, a.bg != 0.0 ? static_cast<float>(static_cast<double>(acc) + a.bg * a.colsum[0]) : acc);
  }
  if (staged) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < cta_r1 - cta_r0; i += kRowNT) put_y(a, y, cta_r0 + i, ystage[i]);
  }
  if (threadIdx.x == 0 && !ready) mbar_wait(xbar, 0);  // no CTA exits with the bulk copy in flight
}

template <typename ColT, typename PtrT, bool CSER>
int launch_row(const DotArgs &a, const float *x, float *y, cudaStream_t st) {
  const size_t smem = row_layout(a.k, a.n, kRowNT / 32).total;
  auto kern = a.npeer > 0 ? k_matvec_row<ColT, PtrT, CSER, true> : k_matvec_row<ColT, PtrT, CSER, false>;
  if (int rc_ = allow_max_smem(kern)) return rc_;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(num_sms(), a.m)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kRowNT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CERDOT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, a, x, y));
  return CERDOT_OK;
}

template <typename ColT, bool CSER>
int by_ptr(const DotArgs &a, int op_bits, const float *x, float *y, cudaStream_t st) {
  switch (op_bits) {
    case 8: return launch_row<ColT, uint8_t, CSER>(a, x, y, st);
    case 16: return launch_row<ColT, uint16_t, CSER>(a, x, y, st);
    default: return launch_row<ColT, uint32_t, CSER>(a, x, y, st);
  }
}

template <bool CSER>
int by_col(const DotArgs &a, int col_bits, int op_bits, const float *x, float *y, cudaStream_t st) {
  switch (col_bits) {
    case 8: return by_ptr<uint8_t, CSER>(a, op_bits, x, y, st);
    case 16: return by_ptr<uint16_t, CSER>(a, op_bits, x, y, st);
    default: return by_ptr<uint32_t, CSER>(a, op_bits, x, y, st);
  }
}

}  // namespace

// Every row inside one window from its 16 B-aligned start, the tables and x in shared memory.
bool matvec_row_fits(const DotArgs &a, size_t col_bytes) {
  const int64_t align = 16 / static_cast<int64_t>(col_bytes);
  if (a.k < 1 || a.k > kSmemValues || a.max_row_nnz <= 0 || a.max_row_nnz > static_cast<int64_t>(kWin) - (align - 1))
    return false;
  if (a.nnz >= (int64_t(1) << 32) - 4096 || a.m >= (int64_t(1) << 31)) return false;
  return row_layout(a.k, a.n, kRowNT / 32).total <= static_cast<uint32_t>(kMaxSmemBytes);
}

int matvec_row(const DotArgs &a, bool cser, int col_bits, int op_bits, const float *x, float *y, cudaStream_t st) {
  return cser ? by_col<true>(a, col_bits, op_bits, x, y, st) : by_col<false>(a, col_bits, op_bits, x, y, st);
}

}  // namespace cerdot
