// Mat-mat (batch > 1) over a column-tiled view of the encoding, X tiles staged in shared memory by TMA.
//
// Reference: lemt kernels.py:283-301 (_dot_segmented with a matrix right-hand side) over
// _segmented_sums (kernels.py:117-125): Y[r, :] = sum_seg (omega[seg] - bg) * sum_{i in seg} X[colI[i], :].
//
// Why a view.  The gather of one X row serves 32*V batch columns when lane l of a warp reads columns
// [32*V*cb + V*l, +V) of it: one 128*V B access, conflict-free, if the X row sits in shared memory.  X
// (n x B) does not fit in shared memory, so X is cut into tiles of NT rows (the matrix's columns) and
// every segment is split at the tile boundaries (colI is ascending inside a segment, formats.py:220, so
// a segment's entries in tile t are one contiguous run: a "fragment").  The view lists, tile by tile and
// row by row, every entry as one 8-byte record {column inside the tile | its row | row-end and
// fragment-end flags, the segment's value omega[k] - bg in fp32}, in the encoding's (rank, column) order:
//
//   tile_ptr[t*m + r]   start of row r's records in tile t (tile-major; tile_ptr[T*m] = nnz)
//   tile_rec[p]         .x = col - t*NT (bits 0-8) | (row & 0xfff) << 9 | bit 30: last record of its
//                       (row, tile) list | bit 31: last entry of its fragment;  .y = float bits of v
//
// It is derived from colI / omegaPtr / rowPtr / omegaI once per encoding (k_tv_count, a scan, k_tv_fill)
// and cached by the caller, like the rowEntry index; the format itself is unchanged.
//
// Kernel (k_matmat_tv).  CTA = (block of RB rows, 32*V batch columns, one of S shares of the X tiles), 16
// warps, one CTA per SM; with S > 1 a CTA writes a partial product and k_tv_reduce adds the S partials in
// split order:
//   * TMA (cp.async.bulk.tensor.2d, one elected thread) streams X tiles (NT rows x 32V columns,
//     zero-filled past n and B) into a double buffer; the last warp to finish a tile re-arms its buffer;
//   * warp w owns a contiguous range of the CTA's rows balanced by entries (rowEntry prefix), so its
//     records for tile t are one contiguous stream; 32 records at a time are loaded lane-parallel (the
//     next chunk -- possibly the next tile's first -- is prefetched) and broadcast from shared memory;
//   * per entry: one V-wide shared load of the X row, V adds into the fragment's running sums; at a
//     fragment end one fma per column with the segment value (one multiply per fragment);
//   * at a record with the row-end flag the warp adds its accumulators into the row's slot of a shared y
//     tile (the row is named by the record: no row-pointer walk; each row owned by one warp: no atomics,
//     fixed order); the epilogue adds bg * colsum(X) (fp64) and stores y (and to peers).
// Summation order (the 1e-5 bar): per (row, column) fragments in (tile, rank, column) order, sequential
// fp32 sums inside a fragment, one fp32 fma per fragment, tile partials added in tile order.
// Deterministic: no floating-point atomics.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"
#include "tileview.cuh"

namespace cerdot {

namespace {

constexpr int kTvThreads = 512;
constexpr int kTvWarps = kTvThreads / 32;
constexpr uint32_t kTvMaxStages = 6;
constexpr int32_t kTileRows = 128;      // X rows per tile (NT) of dense-ish layers
constexpr int32_t kTileRowsWide = 256;  // ... of sparse wide layers (longer (row, tile) lists)
constexpr uint32_t kFragEnd = 0x80000000u;  // record .x bit 31: last entry of its segment fragment
constexpr uint32_t kRowEnd = 0x40000000u;   // bit 30: last record of its (row, tile) list
constexpr uint32_t kColMask = 0x1ffu;       // bits 0-8: X row inside the tile (NT = the sentinel zero row)
constexpr uint32_t kRowShift = 9;           // bits 9-20: the matrix row, low 12 bits
constexpr uint32_t kRowMask = 0xfffu;
constexpr int kCountWarps = 8;
constexpr int kScanThreads = 1024;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
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
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

template <typename T>
__device__ __forceinline__ uint32_t ldi(const T *p, int64_t i) {
  return __ldg(p + i);
}

// ---------------------------------------------------------------------------------------------- view build
// Per (row, tile) entry counts, written tile-major.  Warp per row, per-warp shared histogram.
template <typename ColT>
__global__ void __launch_bounds__(kCountWarps * 32) k_tv_count(const ColT *__restrict__ col,
                                                               const uint32_t *__restrict__ re, int64_t m,
                                                               uint32_t nt, uint32_t tiles,
                                                               uint32_t *__restrict__ cnt) {
  extern __shared__ uint32_t hist_all[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t *hist = hist_all + wid * tiles;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kCountWarps;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * kCountWarps + wid; r < m; r += nwarps) {
    for (uint32_t t = lane; t < tiles; t += 32) hist[t] = 0;
    __syncwarp();
    const uint32_t e0 = __ldg(re + r), e1 = __ldg(re + r + 1);
    for (uint32_t e = e0 + lane; e < e1; e += 32) atomicAdd(hist + ldi(col, e) / nt, 1u);
    __syncwarp();
    for (uint32_t t = lane; t < tiles; t += 32) cnt[static_cast<int64_t>(t) * m + r] = hist[t];
    __syncwarp();
  }
}

// Exclusive scan of n u32 counts in place (three passes; totals fit u32 because nnz < 2^32).
__global__ void __launch_bounds__(kScanThreads) k_scan_part(const uint32_t *__restrict__ v, int64_t n,
                                                            int64_t per_cta, uint32_t *__restrict__ sums) {
  __shared__ uint32_t red[32];
  const int64_t b0 = static_cast<int64_t>(blockIdx.x) * per_cta, b1 = min64(n, b0 + per_cta);
  uint32_t s = 0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += kScanThreads) s += v[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = red[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) sums[blockIdx.x] = s;
  }
}

__device__ __forceinline__ uint32_t block_exscan(uint32_t v, uint32_t *sh, uint32_t *total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  if (lane == 31) sh[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < static_cast<int>(blockDim.x >> 5) ? sh[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= d) wi += t;
    }
    sh[lane] = wi - w;
    if (lane == 31) sh[32] = wi;
  }
  __syncthreads();
  const uint32_t r = sh[wid] + incl - v;
  *total = sh[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_top(uint32_t *__restrict__ sums, int nparts) {
  __shared__ uint32_t sh[33];
  uint32_t carry = 0;
  for (int base = 0; base < nparts; base += kScanThreads) {
    const int i = base + threadIdx.x;
    const uint32_t v = i < nparts ? sums[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exscan(v, sh, &tot);
    if (i < nparts) sums[i] = carry + ex;
    carry += tot;
  }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_apply(uint32_t *__restrict__ v, int64_t n, int64_t per_cta,
                                                             const uint32_t *__restrict__ sums, uint32_t total_out) {
  __shared__ uint32_t sh[33];
  const int64_t b0 = static_cast<int64_t>(blockIdx.x) * per_cta, b1 = min64(n, b0 + per_cta);
  uint32_t carry = sums[blockIdx.x];
  for (int64_t base = b0; base < b1; base += kScanThreads) {
    const int64_t i = base + threadIdx.x;
    const uint32_t x = i < b1 ? v[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exscan(x, sh, &tot);
    if (i < b1) v[i] = carry + ex;
    carry += tot;
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) v[n] = total_out;
}

// Records: warp per row, segment by segment in the encoding's order; a stable per-tile cursor scatter.
template <typename ColT, typename PtrT, bool CSER>
__global__ void __launch_bounds__(kCountWarps * 32) k_tv_fill(const ColT *__restrict__ col,
                                                              const PtrT *__restrict__ op, const void *rp,
                                                              int rp_bits, const void *oi, int oi_bits,
                                                              const double *__restrict__ omega, double bg, int64_t m,
                                                              uint32_t nt, uint32_t tiles,
                                                              const uint32_t *__restrict__ tptr,
                                                              uint2 *__restrict__ rec) {
  extern __shared__ uint32_t cur_all[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t *cur = cur_all + wid * tiles;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kCountWarps;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * kCountWarps + wid; r < m; r += nwarps) {
    for (uint32_t t = lane; t < tiles; t += 32) cur[t] = tptr[static_cast<int64_t>(t) * m + r];
    __syncwarp();
    const uint32_t s0 = load_index(rp, rp_bits, r), s1 = load_index(rp, rp_bits, r + 1);
    for (uint32_t s = s0; s < s1; ++s) {
      const uint32_t st = ldi(op, s), en = ldi(op, s + 1);
      if (en <= st) continue;
      const uint32_t k = CSER ? load_index(oi, oi_bits, s) : s - s0 + 1;
      const float v = static_cast<float>(__ldg(omega + k) - bg);
      for (uint32_t base = st; base < en; base += 32) {
        const uint32_t e = base + lane;
        const bool valid = e < en;
        const uint32_t c = valid ? ldi(col, e) : 0u;
        const uint32_t t = valid ? c / nt : 0xffffffffu;
        const uint32_t cn = (e + 1 < en) ? ldi(col, e + 1) : 0xffffffffu;
        const bool last = valid && (cn == 0xffffffffu || cn / nt != t);
        const unsigned peers = __match_any_sync(0xffffffffu, t);
        uint32_t pos = 0;
        if (valid) pos = cur[t] + __popc(peers & lt);
        __syncwarp();
        if (valid && (peers & lt) == 0) cur[t] += __popc(peers);
        __syncwarp();
        if (valid) {
          const bool row_end = pos + 1u == __ldg(tptr + static_cast<int64_t>(t) * m + r + 1);
          rec[pos] = make_uint2((c - t * nt) | ((static_cast<uint32_t>(r) & kRowMask) << kRowShift) |
                                    (row_end ? kRowEnd : 0u) | (last ? kFragEnd : 0u),
                                __float_as_uint(v));
        }
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------------------------- mat-mat
struct TvArgs {
  const uint32_t *tptr;
  const uint2 *rec;
  const uint32_t *re;
  int64_t m, batch;
  uint32_t nt, tiles, rb, box_rows, stages;
  uint32_t tper;   // X tiles per CTA (gridDim.z CTAs split the tiles of one row block)
  float *part;     // tile-split partial products, [gridDim.z][m][ldp]; null: the CTA writes y itself
  int64_t ldp;
  double bg;
  const double *colsum;
  float *const *ypeer;
  int npeer;
  int64_t ypeer_off;
};

struct TvSmem {
  uint32_t xs, xs_stride, ys, wb, es, bar, cnt, total;
};

__host__ __device__ __forceinline__ TvSmem tv_layout(uint32_t nt, uint32_t cb, uint32_t rb, uint32_t stages) {
  TvSmem L{};
  uint32_t o = 0;
  auto take = [&](uint32_t bytes, uint32_t align) {
    o = (o + align - 1) / align * align;
    const uint32_t r = o;
    o += bytes;
    return r;
  };
  L.xs_stride = ((nt + 1) * cb * 4 + 127) / 128 * 128;  // one tile + the zero row (sentinel records)
  L.xs = take(stages * L.xs_stride, 128);
  L.ys = take(rb * cb * 4, 16);
  L.wb = take(kTvWarps * 32 * 8, 16);  // per-warp broadcast buffer: 32 records
  L.es = take((rb + 1) * 4, 16);
  L.bar = take(kTvMaxStages * 8, 8);
  L.cnt = take(kTvMaxStages * 4, 4);
  L.total = o;
  return L;
}

template <int V>
struct XV {
  float v[V];
};
template <int V>
__device__ __forceinline__ XV<V> lds_x(const unsigned char *p) {
  XV<V> r;
  if (V == 4) {
    const float4 t = *reinterpret_cast<const float4 *>(p);
    r.v[0] = t.x; r.v[1 % V] = t.y; r.v[2 % V] = t.z; r.v[3 % V] = t.w;
  } else if (V == 2) {
    const float2 t = *reinterpret_cast<const float2 *>(p);
    r.v[0] = t.x; r.v[1 % V] = t.y;
  } else {
    r.v[0] = *reinterpret_cast<const float *>(p);
  }
  return r;
}

// FRAG = true: sum the entries of each fragment, one multiply per fragment (the paper's sum-then-multiply,
// segments split at tile boundaries).  FRAG = false: the segment value is folded into each entry's fused
// multiply-add (an FFMA issues at the rate of an FADD on the CUDA cores, so this drops the fragment
// bookkeeping -- a warp-divergent branch per entry -- at no extra arithmetic cost).  Both sum in fp32 in
// the view's order; both are checked against the oracle.
template <int V, bool FRAG>
__global__ void __launch_bounds__(kTvThreads, 1) k_matmat_tv(const __grid_constant__ CUtensorMap xmap, TvArgs a,
                                                             float *__restrict__ y, int64_t ldy) {
  constexpr int CB = 32 * V;
  extern __shared__ __align__(128) unsigned char smem[];
  const TvSmem L = tv_layout(a.nt, CB, a.rb, a.stages);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float *ys = reinterpret_cast<float *>(smem + L.ys);
  uint2 *wb = reinterpret_cast<uint2 *>(smem + L.wb) + wid * 32;  // per-warp broadcast of 32 records
  uint32_t *es = reinterpret_cast<uint32_t *>(smem + L.es);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + L.bar);
  uint32_t *done_cnt = reinterpret_cast<uint32_t *>(smem + L.cnt);
  const uint32_t m = static_cast<uint32_t>(a.m);
  const uint32_t R0 = blockIdx.x * a.rb, R1 = min(m, R0 + a.rb);
  const int cb0 = static_cast<int>(blockIdx.y) * CB;
  const uint32_t nrow = R1 > R0 ? R1 - R0 : 0u;
  const uint32_t nboxes = a.nt / a.box_rows;
  const uint32_t tile_bytes = a.nt * CB * 4;
  const uint32_t S = a.stages;
  const uint32_t t_lo = blockIdx.z * a.tper, t_hi = min(a.tiles, t_lo + a.tper);  // this CTA's X tiles

  // ---- prologue: barriers, zero y tile and sentinel rows, entry prefix of the CTA's rows
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < S; ++i) {
      mbar_init(full + i, 1);
      done_cnt[i] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (uint32_t i = threadIdx.x; i < nrow * CB; i += kTvThreads) ys[i] = 0.f;
  for (uint32_t i = threadIdx.x; i < S * CB; i += kTvThreads)
    reinterpret_cast<float *>(smem + L.xs + (i / CB) * L.xs_stride)[a.nt * CB + (i % CB)] = 0.f;
  for (uint32_t i = threadIdx.x; i <= nrow; i += kTvThreads) es[i] = __ldg(a.re + R0 + i);
  __syncthreads();
  auto issue = [&](uint32_t t) {  // TMA of X tile t (rows t*NT.., columns cb0..) into buffer (t - t_lo) % S
    uint64_t *bar = full + ((t - t_lo) % S);
    float *dst = reinterpret_cast<float *>(smem + L.xs + ((t - t_lo) % S) * L.xs_stride);
    mbar_expect_tx(bar, tile_bytes);
    for (uint32_t bx = 0; bx < nboxes; ++bx)
      tma_load_2d(dst + bx * a.box_rows * CB, &xmap, cb0, static_cast<int>(t * a.nt + bx * a.box_rows), bar);
  };
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
    for (uint32_t t = t_lo; t < t_lo + S && t < t_hi; ++t) issue(t);
  }
  // ---- this warp's rows [ra, rb): contiguous, balanced by entries (first row whose prefix >= target)
  uint32_t ra, rb;
  {
    const uint32_t tot = es[nrow] - es[0];
    auto split = [&](uint32_t w) -> uint32_t {
      if (w == 0) return 0u;
      if (w >= kTvWarps) return nrow;
      const uint32_t target = es[0] + static_cast<uint32_t>((static_cast<uint64_t>(tot) * w) / kTvWarps);
      uint32_t lo = 0, hi = nrow;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (es[mid] < target) lo = mid + 1; else hi = mid;
      }
      return lo;
    };
    ra = split(wid);
    rb = max(ra, split(wid + 1));
  }
  const uint32_t nr = rb - ra;
  const uint32_t gra = R0 + ra;
  // the warp's record range in tile t: tile_ptr at its first and one-past-last row (lanes 0 and 1),
  // prefetched three tiles ahead; the rows themselves are named by the records (row bits, row-end flag)
  auto load_rp = [&](uint32_t t) -> uint32_t {
    return (t < t_hi && lane < 2) ? __ldg(a.tptr + static_cast<int64_t>(t) * m + gra + (lane ? nr : 0u)) : 0u;
  };
  const uint2 sentinel = make_uint2(a.nt, 0u);  // the zero row, no flags
  auto load_chunk = [&](uint32_t start, uint32_t end) -> uint2 {
    return (start + lane < end) ? __ldg(a.rec + start + lane) : sentinel;
  };
  // prefetch pipeline: the range three tiles ahead, the first record chunk two tiles ahead (a warp
  // holds only a few dozen records per tile, so the tile boundary is where L2 latency would show)
  uint32_t rp_c = load_rp(t_lo), rp_n = load_rp(t_lo + 1), rp_nn = load_rp(t_lo + 2);
  auto range = [&](uint32_t reg, uint32_t &b, uint32_t &e) {
    b = __shfl_sync(0xffffffffu, reg, 0);
    e = __shfl_sync(0xffffffffu, reg, 1);
  };
  uint32_t P, Pe, Pn, Pne;
  range(rp_c, P, Pe);
  range(rp_n, Pn, Pne);
  uint2 first = load_chunk(P, Pe);
  uint2 first_n = load_chunk(Pn, Pne);
  const uint32_t lane_off = static_cast<uint32_t>(lane) * V * 4;
  float *yl = ys + lane * V;  // this lane's columns of the CTA's y tile
  const uint32_t r0low = R0 & kRowMask;

  for (uint32_t t = t_lo; t < t_hi; ++t) {
    const uint32_t bsel = (t - t_lo) % S;
    const uint32_t rp_n3 = load_rp(t + 3);
    uint32_t Pnn, Pnne;
    range(rp_nn, Pnn, Pnne);
    const uint2 first_nn = load_chunk(Pnn, Pnne);
    mbar_wait(full + bsel, ((t - t_lo) / S) & 1);
    const unsigned char *xb = smem + L.xs + bsel * L.xs_stride + lane_off;
    uint2 cur = first;
    float acc[V], run[V];
#pragma unroll
    for (int q = 0; q < V; ++q) acc[q] = run[q] = 0.f;
    auto row_flush = [&](uint32_t recx) {  // the record closes its row's list in this tile
      float *yr = yl + (((recx >> kRowShift) - r0low) & kRowMask) * CB;
#pragma unroll
      for (int q = 0; q < V; ++q) {
        yr[q] += acc[q];
        acc[q] = 0.f;
      }
    };
    for (uint32_t p = P; p < Pe; p += 32) {
      const uint2 nxt = (p + 32 < Pe) ? load_chunk(p + 32, Pe) : sentinel;
      const unsigned emask = FRAG ? __ballot_sync(0xffffffffu, (cur.x & kFragEnd) != 0u) : 0u;
      const unsigned rmask = __ballot_sync(0xffffffffu, (cur.x & kRowEnd) != 0u);
      // broadcast buffer: the X row's byte offset inside the tile buffer (flags and row bits stay in cur.x)
      wb[lane] = make_uint2((cur.x & kColMask) * (CB * 4), cur.y);
      __syncwarp();
      const uint32_t cnt = min(32u, Pe - p);
      for (uint32_t g = 0; g < cnt; g += 8) {
        uint32_t off[8];
        float vv[8];
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          const uint4 q2 = *reinterpret_cast<const uint4 *>(wb + g + j);  // two records, one broadcast
          off[j] = q2.x;
          vv[j] = __uint_as_float(q2.y);
          off[j + 1] = q2.z;
          vv[j + 1] = __uint_as_float(q2.w);
        }
        XV<V> xv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) xv[j] = lds_x<V>(xb + off[j]);
        const unsigned rg = (rmask >> g) & 0xffu;
        if (FRAG) {
          const unsigned eg = (emask >> g) & 0xffu;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int q = 0; q < V; ++q) run[q] += xv[j].v[q];
            if (eg & (1u << j)) {  // fragment end: one multiply per fragment
#pragma unroll
              for (int q = 0; q < V; ++q) {
                acc[q] = fmaf(vv[j], run[q], acc[q]);
                run[q] = 0.f;
              }
              if (rg & (1u << j)) row_flush(__shfl_sync(0xffffffffu, cur.x, g + j));  // a list ends with a fragment end
            }
          }
        } else if (rg == 0u) {  // no row boundary inside these 8 entries
#pragma unroll
          for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int q = 0; q < V; ++q) acc[q] = fmaf(vv[j], xv[j].v[q], acc[q]);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int q = 0; q < V; ++q) acc[q] = fmaf(vv[j], xv[j].v[q], acc[q]);
            if (rg & (1u << j)) row_flush(__shfl_sync(0xffffffffu, cur.x, g + j));
          }
        }
      }
      __syncwarp();
      cur = nxt;
    }
    first = first_n;
    first_n = first_nn;
    P = Pn; Pe = Pne;
    Pn = Pnn; Pne = Pnne;
    rp_nn = rp_n3;
    // release buffer bsel: the last warp to finish tile t re-arms it with tile t + S
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      const uint32_t old = atomicAdd(done_cnt + bsel, 1u);
      if (old == kTvWarps - 1) {
        atomicExch(done_cnt + bsel, 0u);
        if (t + S < t_hi) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(t + S);
        }
      }
    }
  }
  __syncthreads();
  // ---- epilogue: y = y tile (+ bg * colsum), coalesced rows of CB columns
  if (a.part != nullptr) {  // tile split: this CTA's partial product; k_tv_reduce adds the splits in order
    float *pz = a.part + (static_cast<int64_t>(blockIdx.z) * a.m + R0) * a.ldp + cb0;
    for (uint32_t i = threadIdx.x; i < nrow * CB; i += kTvThreads) pz[static_cast<int64_t>(i / CB) * a.ldp + (i % CB)] = ys[i];
    return;
  }
  const int64_t ncols = min64(CB, a.batch - cb0);
  for (uint32_t i = threadIdx.x; i < nrow * CB; i += kTvThreads) {
    const uint32_t rr = i / CB, cc = i % CB;
    if (static_cast<int64_t>(cc) >= ncols) continue;
    const int64_t c = cb0 + cc;
    float v = ys[i];
    if (a.bg != 0.0) v = static_cast<float>(static_cast<double>(v) + a.bg * a.colsum[c]);
    const int64_t off = static_cast<int64_t>(R0 + rr) * ldy + c;
    y[off] = v;
    for (int pp = 0; pp < a.npeer; ++pp) a.ypeer[pp][a.ypeer_off + off] = v;
  }
}

// y = sum over the tile splits (in split order: deterministic) + bg * colsum.
__global__ void __launch_bounds__(256) k_tv_reduce(const float *__restrict__ part, int64_t ldp, uint32_t splits,
                                                   int64_t m, int64_t batch, double bg, const double *__restrict__ colsum,
                                                   float *__restrict__ y, int64_t ldy, float *const *ypeer, int npeer,
                                                   int64_t ypeer_off) {
  const int64_t total = m * batch;
  if (npeer == 0 && (batch & 3) == 0 && (ldp & 3) == 0 && (ldy & 3) == 0 &&
      ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(part)) & 15) == 0) {  // four columns per thread
    const int64_t q = batch >> 2;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m * q;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const int64_t r = i / q, c = (i - r * q) << 2;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      for (uint32_t z = 0; z < splits; ++z) {
        const float4 p = *reinterpret_cast<const float4 *>(part + (static_cast<int64_t>(z) * m + r) * ldp + c);
        v.x += p.x; v.y += p.y; v.z += p.z; v.w += p.w;
      }
      if (bg != 0.0) {
        v.x = static_cast<float>(static_cast<double>(v.x) + bg * colsum[c]);
        v.y = static_cast<float>(static_cast<double>(v.y) + bg * colsum[c + 1]);
        v.z = static_cast<float>(static_cast<double>(v.z) + bg * colsum[c + 2]);
        v.w = static_cast<float>(static_cast<double>(v.w) + bg * colsum[c + 3]);
      }
      *reinterpret_cast<float4 *>(y + r * ldy + c) = v;
    }
    return;
  }
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / batch, c = i - r * batch;
    float v = 0.f;
    for (uint32_t z = 0; z < splits; ++z) v += part[(static_cast<int64_t>(z) * m + r) * ldp + c];
    if (bg != 0.0) v = static_cast<float>(static_cast<double>(v) + bg * colsum[c]);
    const int64_t off = r * ldy + c;
    y[off] = v;
    for (int pp = 0; pp < npeer; ++pp) ypeer[pp][ypeer_off + off] = v;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static std::once_flag once;
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int allow_smem_once(const void *kern) {
  static std::mutex mu;
  static std::set<std::pair<const void *, int>> done;
  int dev = 0;
  CERDOT_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({kern, dev})) return CERDOT_OK;
  CERDOT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  done.insert({kern, dev});
  return CERDOT_OK;
}

constexpr uint32_t kYBudget = 80 * 1024;    // the CTA's y tile

}  // namespace

// Launch geometry of the tiled mat-mat for V (columns per lane): CTAs in whole waves of one per SM,
// rows per CTA within the y-tile budget.
struct TvGeom {
  int64_t col_blocks, row_blocks, rb;
};
TvGeom tv_geom(int64_t m, int64_t batch, int V, int64_t splits = 1) {
  const int64_t CB = 32 * V;
  TvGeom g{};
  g.col_blocks = ceil_div(batch, CB);
  const int64_t rb_max = kYBudget / (CB * 4);
  const int64_t sms = num_sms();
  for (int64_t waves = 1;; ++waves) {
    g.row_blocks = std::max<int64_t>(1, sms * waves / (g.col_blocks * splits));
    g.rb = ceil_div(m, g.row_blocks);
    if (g.rb <= rb_max || waves > 4096) break;
  }
  g.rb = std::max<int64_t>(1, std::min<int64_t>(g.rb, rb_max));
  g.row_blocks = ceil_div(m, g.rb);
  return g;
}

// Columns per lane: the V with the smallest modelled time per SM, max of (a) shared-memory wavefronts
// (V per X-row gather + 1/2 per record broadcast + the X tile fills), (b) issue slots (~10 + V
// instructions per entry per warp, 4 per clock) and (c) the X tile fills through L2 (~6 KB/clk chip-wide,
// B300_MICROARCH.md "LTS throughput cap").  Low X reuse (few rows per CTA, long X) favours narrow
// column blocks; high reuse favours wide ones.
int tile_view_v(int64_t m, int64_t n, int64_t nnz, int64_t batch, int32_t nt) {
  const double sms = num_sms();
  double best = 1e300;
  int bv = 1;
  for (int V : {1, 2, 4}) {
    if (V > 1 && batch <= 16 * V) continue;  // more than half the lanes idle
    // two X stages and a y tile of at least 64 rows must fit
    if (V > 1 && tv_layout(nt, 32 * V, 64, 2).total > 227u * 1024u) continue;
    const TvGeom g = tv_geom(m, batch, V);
    const double ctas = static_cast<double>(g.row_blocks * g.col_blocks);
    const double fill_bytes = ctas * static_cast<double>(n) * 32.0 * V * 4.0;
    const double lsu = static_cast<double>(nnz) * g.col_blocks * (V + 0.5) + fill_bytes / 128.0;
    const double issue = static_cast<double>(nnz) * g.col_blocks * (10.0 + V) / 4.0;
    const double per_sm = std::max(lsu, issue) / std::min(ctas, sms);
    const double l2 = fill_bytes / 6000.0;
    const double t = std::max(per_sm, l2);
    if (t < best * 0.98) {
      best = t;
      bv = V;
    }
  }
  return bv;
}

// Tile splits: CTAs per row block that share its X tiles (gridDim.z).  A sparse wide layer leaves a warp
// only a handful of entries per (row, tile) list when one CTA walks every tile of a few rows; splitting
// the tiles over S CTAs gives each CTA S times the rows (longer per-tile record streams, 1/S of X through
// its shared memory) at the price of S partial products added by k_tv_reduce.
int tile_view_splits(const cerdot_matrix *a, int64_t batch, int V) {
  const int forced = kernel_path(CERDOT_PATH_MATMAT_SPLIT);
  const int32_t nt = a->tile_rows > 0 ? a->tile_rows : kTileRows;
  const int64_t tiles = tile_view_tiles(a->n, nt);
  int s = 1;
  if (forced > 0) {
    s = forced;
  } else {
    // entries per warp per tile at one split; aim for >= 96 (three record chunks), within 8 splits
    const TvGeom g = tv_geom(a->m, batch, V);
    const double per_warp_tile = static_cast<double>(a->nnz) / static_cast<double>(a->m) * nt /
                                 static_cast<double>(a->n) * static_cast<double>(g.rb) / kTvWarps;
    while (s < 8 && per_warp_tile * s < 96.0) s *= 2;
  }
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(s, tiles)));
}

size_t tile_view_dot_workspace_bytes(const cerdot_matrix *a, int64_t batch) {
  if (a->tile_ptr == nullptr || a->tile_rows <= 0 || batch <= 1) return 0;
  const int V = tile_view_v(a->m, a->n, a->nnz, batch, a->tile_rows);
  const int s = tile_view_splits(a, batch, V);
  if (s <= 1) return 0;
  const int64_t ldp = ceil_div(batch, 32 * V) * 32 * V;
  return sizeof(float) * static_cast<size_t>(s) * static_cast<size_t>(a->m) * static_cast<size_t>(ldp);
}

int32_t tile_view_rows(const cerdot_matrix *a, int64_t batch) {
  if (batch <= 1 || a->nnz >= (int64_t(1) << 32) || a->m >= (int64_t(1) << 31) || a->n >= (int64_t(1) << 31))
    return 0;
  const int path = kernel_path(CERDOT_PATH_MATMAT);
  const int force_nt = kernel_path(CERDOT_PATH_MATMAT_TILE);
  if (path == 3 || path == 4) return force_nt ? force_nt : kTileRows;  // forced
  if (path != 0) return 0;
  // Automatic choice, measured on B200 (tools/mm_tiled_time.py, tools/mm_split_time.py): the tiled kernel
  // pays a fixed cost per (row, tile) list (the y-tile update), so it needs enough entries per list:
  //   * >= 24 per 128-row tile (ResNet conv ~70, the 32768^2 layer ~38): 128-row tiles;
  //   * 8..24 (AlexNet fc6 ~12) at >= 48 columns: 256-row tiles with the tiles split over CTAs
  //     (AlexNet fc6 B=64: 58 us vs 79 us flat);
  //   * below that (VGG fc6 ~5: 145 us tiled vs 143 us flat) the flat L2-gather kernel stays.
  const double per_list = static_cast<double>(a->nnz) / static_cast<double>(a->m) * kTileRows / static_cast<double>(a->n);
  if (per_list >= 24.0) return kTileRows;
  if (per_list >= 8.0 && batch >= 48) return kTileRowsWide;
  return 0;
}

int64_t tile_view_tiles(int64_t n, int32_t nt) { return nt > 0 ? ceil_div(n, nt) : 0; }

size_t tile_view_workspace_bytes(int64_t m, int64_t n, int32_t nt) {
  const int64_t cnt = tile_view_tiles(n, nt) * m;
  const int64_t per = 64 * kScanThreads;
  return sizeof(uint32_t) * static_cast<size_t>(ceil_div(std::max<int64_t>(cnt, 1), per) + 1);
}

int tile_view_build(const cerdot_matrix *a, int32_t nt, uint32_t *tptr, void *rec_v, void *workspace,
                    size_t workspace_bytes, cudaStream_t st) {
  if (nt <= 0 || (nt % 32) != 0) return fail(CERDOT_E_VALUE, "tile rows must be a positive multiple of 32");
  if (a->row_entry == nullptr) return fail(CERDOT_E_VALUE, "the tile view needs the row_entry index");
  if (a->nnz >= (int64_t(1) << 32)) return fail(CERDOT_E_VALUE, "the tile view needs nnz < 2^32");
  const int64_t tiles = tile_view_tiles(a->n, nt);
  if (tiles > 4096) return fail(CERDOT_E_VALUE, "too many column tiles");
  if (workspace_bytes < tile_view_workspace_bytes(a->m, a->n, nt))
    return fail(CERDOT_E_WORKSPACE, "tile view workspace too small");
  const int64_t m = a->m;
  const int64_t count = tiles * m;
  uint2 *rec = static_cast<uint2 *>(rec_v);
  const size_t hsmem = sizeof(uint32_t) * kCountWarps * static_cast<size_t>(tiles);
  if (hsmem > 227 * 1024) return fail(CERDOT_E_VALUE, "too many column tiles");
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, kCountWarps), num_sms() * 16)));
  if (m == 0) {
    CERDOT_CUDA_CHECK(cudaMemsetAsync(tptr, 0, sizeof(uint32_t) * (count + 1), st));
    return CERDOT_OK;
  }
  // counts
  switch (a->col_bits) {
    case 8: {
      auto k = k_tv_count<uint8_t>;
      CERDOT_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      k<<<grid, kCountWarps * 32, hsmem, st>>>(static_cast<const uint8_t *>(a->col_index), a->row_entry, m, nt,
                                              static_cast<uint32_t>(tiles), tptr);
      break;
    }
    case 16: {
      auto k = k_tv_count<uint16_t>;
      CERDOT_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      k<<<grid, kCountWarps * 32, hsmem, st>>>(static_cast<const uint16_t *>(a->col_index), a->row_entry, m, nt,
                                               static_cast<uint32_t>(tiles), tptr);
      break;
    }
    default: {
      auto k = k_tv_count<uint32_t>;
      CERDOT_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      k<<<grid, kCountWarps * 32, hsmem, st>>>(static_cast<const uint32_t *>(a->col_index), a->row_entry, m, nt,
                                               static_cast<uint32_t>(tiles), tptr);
    }
  }
  CERDOT_LAUNCH_CHECK();
  // scan
  const int64_t per = 64 * kScanThreads;
  const int nparts = static_cast<int>(ceil_div(count, per));
  uint32_t *sums = static_cast<uint32_t *>(workspace);
  k_scan_part<<<nparts, kScanThreads, 0, st>>>(tptr, count, per, sums);
  k_scan_top<<<1, kScanThreads, 0, st>>>(sums, nparts);
  k_scan_apply<<<nparts, kScanThreads, 0, st>>>(tptr, count, per, sums, static_cast<uint32_t>(a->nnz));
  CERDOT_LAUNCH_CHECK();
  // records
  const bool cser = a->kind == CERDOT_CSER;
  auto fill = [&](auto kern, const auto *col, const auto *op) -> int {
    CERDOT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    kern<<<grid, kCountWarps * 32, hsmem, st>>>(col, op, a->row_ptr, a->row_ptr_bits, a->omega_index,
                                                a->omega_index_bits, a->omega, a->background, m, nt,
                                                static_cast<uint32_t>(tiles), tptr, rec);
    CERDOT_LAUNCH_CHECK();
    return CERDOT_OK;
  };
  auto by_op = [&](auto ctag) -> int {
    using ColT = decltype(ctag);
    const ColT *col = static_cast<const ColT *>(a->col_index);
    switch (a->omega_ptr_bits) {
      case 8: {
        const uint8_t *op = static_cast<const uint8_t *>(a->omega_ptr);
        return cser ? fill(k_tv_fill<ColT, uint8_t, true>, col, op) : fill(k_tv_fill<ColT, uint8_t, false>, col, op);
      }
      case 16: {
        const uint16_t *op = static_cast<const uint16_t *>(a->omega_ptr);
        return cser ? fill(k_tv_fill<ColT, uint16_t, true>, col, op) : fill(k_tv_fill<ColT, uint16_t, false>, col, op);
      }
      default: {
        const uint32_t *op = static_cast<const uint32_t *>(a->omega_ptr);
        return cser ? fill(k_tv_fill<ColT, uint32_t, true>, col, op) : fill(k_tv_fill<ColT, uint32_t, false>, col, op);
      }
    }
  };
  switch (a->col_bits) {
    case 8: return by_op(uint8_t{});
    case 16: return by_op(uint16_t{});
    default: return by_op(uint32_t{});
  }
}

// Returns CERDOT_OK with *used = false when the tiled path does not apply (the caller falls back).
int matmat_tiled(const cerdot_matrix *mat, const float *x, int64_t ldx, int64_t batch, float *y, int64_t ldy,
                 const double *colsum, float *const *peers, int npeers, int64_t peer_offset, void *workspace,
                 size_t workspace_bytes, cudaStream_t st, bool *used) {
  *used = false;
  if (mat->tile_ptr == nullptr || mat->tile_rec == nullptr || mat->tile_rows <= 0 || mat->row_entry == nullptr)
    return CERDOT_OK;
  if (batch <= 1 || (ldx % 4) != 0 || (reinterpret_cast<uintptr_t>(x) & 15) != 0) return CERDOT_OK;
  if (mat->m >= (int64_t(1) << 31) || mat->n >= (int64_t(1) << 31)) return CERDOT_OK;
  auto enc = tensor_map_encoder();
  if (enc == nullptr) return CERDOT_OK;
  const uint32_t nt = static_cast<uint32_t>(mat->tile_rows);
  if (nt != static_cast<uint32_t>(kTileRows) && nt != static_cast<uint32_t>(kTileRowsWide)) return CERDOT_OK;
  const int V = tile_view_v(mat->m, mat->n, mat->nnz, batch, mat->tile_rows);
  const uint32_t CB = 32u * V;
  int splits = tile_view_splits(mat, batch, V);
  const int64_t ldp = ceil_div(batch, CB) * CB;
  if (splits > 1 && (workspace == nullptr ||
                     workspace_bytes < sizeof(float) * static_cast<size_t>(splits) * mat->m * static_cast<size_t>(ldp)))
    splits = 1;  // no room for the partial products: one CTA per row block walks every tile
  const TvGeom g = tv_geom(mat->m, batch, V, splits);
  if (g.col_blocks > 65535 || g.row_blocks > 2147483647) return CERDOT_OK;
  const int64_t rb = g.rb, row_blocks = g.row_blocks, col_blocks = g.col_blocks;
  const uint32_t box_rows = std::min<uint32_t>(nt, 256u);
  if (nt % box_rows) return CERDOT_OK;

  CUtensorMap map;
  const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(batch), static_cast<cuuint64_t>(mat->n)};
  const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(ldx) * 4};
  const cuuint32_t box[2] = {CB, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(x), gdim, gstride, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return CERDOT_OK;

  TvArgs a{};
  a.tptr = mat->tile_ptr;
  a.rec = static_cast<const uint2 *>(mat->tile_rec);
  a.re = mat->row_entry;
  a.m = mat->m;
  a.batch = batch;
  a.nt = nt;
  a.tiles = static_cast<uint32_t>(tile_view_tiles(mat->n, nt));
  a.tper = static_cast<uint32_t>(ceil_div(a.tiles, splits));
  a.part = splits > 1 ? static_cast<float *>(workspace) : nullptr;
  a.ldp = ldp;
  a.rb = static_cast<uint32_t>(rb);
  a.box_rows = box_rows;
  // as many X stages (2..4) as fit next to the y tile
  a.stages = kTvMaxStages;
  while (a.stages > 2 && tv_layout(nt, CB, a.rb, a.stages).total > 227u * 1024u) --a.stages;
  a.bg = mat->background;
  a.colsum = colsum;
  a.ypeer = peers;
  a.npeer = peers ? npeers : 0;
  a.ypeer_off = peer_offset;
  const size_t smem = tv_layout(nt, CB, a.rb, a.stages).total;
  if (smem > 227u * 1024u) return CERDOT_OK;
  const dim3 grid(static_cast<unsigned>(row_blocks), static_cast<unsigned>(col_blocks), static_cast<unsigned>(splits));
  // per-entry fma (default) or sum-then-multiply per fragment (CERDOT_PATH_MATMAT = 4)
  const bool frag = kernel_path(CERDOT_PATH_MATMAT) == 4;
  auto go = [&](auto kern) -> int {
    if (int rc = allow_smem_once(reinterpret_cast<const void *>(kern))) return rc;
    kern<<<grid, kTvThreads, smem, st>>>(map, a, y, ldy);
    return CERDOT_OK;
  };
  int rc = CERDOT_OK;
  switch (V) {
    case 1: rc = frag ? go(k_matmat_tv<1, true>) : go(k_matmat_tv<1, false>); break;
    case 2: rc = frag ? go(k_matmat_tv<2, true>) : go(k_matmat_tv<2, false>); break;
    default: rc = frag ? go(k_matmat_tv<4, true>) : go(k_matmat_tv<4, false>);
  }
  if (rc) return rc;
  CERDOT_LAUNCH_CHECK();
  if (splits > 1) {
    const int rgrid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(mat->m * batch, 1024), num_sms() * 8)));
    k_tv_reduce<<<rgrid, 256, 0, st>>>(a.part, ldp, static_cast<uint32_t>(splits), mat->m, batch, a.bg, colsum, y, ldy,
                                        a.ypeer, a.npeer, a.ypeer_off);
    CERDOT_LAUNCH_CHECK();
  }
  *used = true;
  return CERDOT_OK;
}

}  // namespace cerdot
