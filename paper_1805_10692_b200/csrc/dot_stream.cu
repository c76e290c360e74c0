// CER / CSER mat-vec (batch 1) for long rows: the stream kernel (k_matvec_stream).
//
// Reference: lemt kernels.py:283-301 (_dot_segmented):
//   y[r] = sum_seg (omega[seg] - bg) * (sum_{i in seg} x[colI[i]])  (+ bg * sum(x) when bg != 0)
//
// The long-row kernel it replaces (k_matvec_run, dot.cu) was bound by the shared-memory pipe (93%): next
// to the x gathers (~27 wavefronts per 256-entry window) it paid a cp.async colI ring (~14), a window
// prefix table (8 stores + ~4 lookups) and a 5-step warp scan.  This kernel keeps only the gathers:
//   * colI goes global -> registers (16 B per lane per window), D windows in flight in a statically
//     indexed register ring; a warp's rows are contiguous in colI, so the ring is one linear stream and a
//     window that straddles a row boundary is simply walked once per row;
//   * segment bounds (omegaPtr, omegaI) are one linear stream per warp too, copied 8 batches of 32 ahead
//     into a per-warp ring by cp.async; row bounds are held lane-parallel and read by shuffle (a pending
//     row-bound load shared a scoreboard with the colI ring: profiles/r02_stream_notes.txt);
//   * segments never meet across lanes: a lane sums its 8 entries fragment by fragment (a fragment = the
//     part of a segment inside one lane) and multiplies each fragment once by its segment's value,
//     sum_seg v * S(seg) = sum_fragments v * S(fragment).  Up to four segment starts in a window are
//     broadcast one by one from the lanes that hold the segments (one shuffle, one value read, an
//     in-register prefix select each); more starts (a row's segment-dense tail) are marked in a 256-slot
//     per-warp flag table with the segment's value slot, and every lane walks the 8 flags of its entries
//     in order.  The value in force at a lane's first entry is warp-uniform state (the few-starts path)
//     or comes from the nearest flagged lane below (one shuffle);
//   * windows in which no segment starts touch neither the table nor the shuffle unit: eight gathers,
//     eight adds, one fma.
// 28 warps per SM at <= 72 registers, two windows in flight.  The kernel is bound by instruction issue
// (~195 per window at 0.80 per scheduler per cycle), not by the shared-memory pipe.
// Summation order (stated for the 1e-5 bar): fp32 fragment sums in colI order, one fp32 fma per fragment
// into a per-lane accumulator, lanes combined by an xor butterfly per row.  Deterministic.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"
#include "dotk.cuh"

namespace cerdot {

namespace {

constexpr uint32_t kStreamWin = 256;   // entries per window, 8 per lane
constexpr uint32_t kSegRing = 256;     // segment bounds held per warp (8 batches of 32)

// Dynamic shared memory: x first (so a gather is one scaled-index load), then the value table, the
// per-warp flag tables and segment-bound rings, the x barrier.
struct StreamSmem {
  uint32_t wv, flag, opr, oir, yb, bar, total;
};
__host__ __device__ __forceinline__ StreamSmem stream_layout(int64_t k, int64_t n, uint32_t warps, uint32_t flag_bytes,
                                                             uint32_t op_bytes, uint32_t oi_bytes) {
  StreamSmem L{};
  uint32_t o = (static_cast<uint32_t>(n) * 4u + 15u) & ~15u;
  auto take = [&](uint32_t bytes) {
    const uint32_t r = o;
    o += (bytes + 15u) & ~15u;
    return r;
  };
  L.wv = take(static_cast<uint32_t>(k) * 4u);
  L.flag = take(warps * kStreamWin * flag_bytes);
  L.opr = take(warps * kSegRing * op_bytes);
  L.oir = take(warps * kSegRing * oi_bytes);
  L.yb = take(warps * 128u);  // 32 results per warp, written out together
  L.bar = take(16u);
  L.total = o;
  return L;
}

// Shared-space accesses by 32-bit address (keeps the table bases in registers: no generic-pointer math)
__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
template <typename T>
__device__ __forceinline__ uint32_t lds_idx(uint32_t addr) {
  uint32_t v;
  if constexpr (sizeof(T) == 1)
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  else if constexpr (sizeof(T) == 2)
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
  else
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ void cp_async16(uint32_t smem_dst, const void *gmem_src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_dst), "l"(gmem_src), "r"(src_bytes)
               : "memory");
}

// One lane's 8 column indices of a window, as loaded (2 / 4 / 8 words for u8 / u16 / u32 colI).
template <typename ColT>
struct Win {
  static constexpr int NW = 2 * sizeof(ColT);
  uint32_t w[NW];
};

__device__ __forceinline__ uint2 ld_stream8(const void *p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

// entries [pos, pos + 8) of colI; pieces at or past lim (the readable end, 16 B rounded) read as 0
template <typename ColT>
__device__ __forceinline__ void win_load(Win<ColT> &q, const ColT *col, uint32_t pos, uint32_t lim) {
  if constexpr (sizeof(ColT) == 1) {
    uint2 v = make_uint2(0u, 0u);
    if (pos < lim) v = ld_stream8(col + pos);
    q.w[0] = v.x; q.w[1] = v.y;
  } else if constexpr (sizeof(ColT) == 2) {
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (pos < lim) v = ld_stream(col + pos);
    q.w[0] = v.x; q.w[1] = v.y; q.w[2] = v.z; q.w[3] = v.w;
  } else {
    uint4 v0 = make_uint4(0u, 0u, 0u, 0u), v1 = v0;
    if (pos < lim) v0 = ld_stream(col + pos);
    if (pos + 4 < lim) v1 = ld_stream(col + pos + 4);
    q.w[0] = v0.x; q.w[1] = v0.y; q.w[2] = v0.z; q.w[3] = v0.w;
    q.w[4] = v1.x; q.w[5] = v1.y; q.w[6] = v1.z; q.w[7] = v1.w;
  }
}

__device__ __forceinline__ uint32_t mad4(uint32_t c, uint32_t base) {  // base + 4 * c as one multiply-add
  uint32_t r;
  asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(r) : "r"(c), "r"(base));
  return r;
}

// shared-memory addresses of the 8 gathered x entries: base + 4 * column
template <typename ColT>
__device__ __forceinline__ void win_addrs(const Win<ColT> &q, uint32_t base, uint32_t c[8]) {
  if constexpr (sizeof(ColT) == 1) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      c[b] = mad4((q.w[0] >> (8 * b)) & 0xffu, base);
      c[4 + b] = mad4((q.w[1] >> (8 * b)) & 0xffu, base);
    }
  } else if constexpr (sizeof(ColT) == 2) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      c[2 * i] = mad4(q.w[i] & 0xffffu, base);
      c[2 * i + 1] = mad4(q.w[i] >> 16, base);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = mad4(q.w[i], base);
  }
}

// A lane's 8 flags (value slots; 0 = no segment starts at this entry).
template <typename FlagT>
struct Flags;
template <>
struct Flags<uint8_t> {
  uint2 f;
  // a = shared address of the lane's 8 flags
  __device__ __forceinline__ void load(uint32_t a) { asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(f.x), "=r"(f.y) : "r"(a)); }
  __device__ __forceinline__ bool any() const { return (f.x | f.y) != 0u; }
  __device__ __forceinline__ static void clear(uint32_t a) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %1};" ::"r"(a), "r"(0u) : "memory");
  }
  __device__ __forceinline__ static void set(uint32_t table, uint32_t pos, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(table + pos), "r"(v) : "memory");
  }
  // bit i set <=> entry i of the lane is flagged
  __device__ __forceinline__ uint32_t mask() const {
    auto nib = [](uint32_t w) -> uint32_t {
      const uint32_t nz = (((w & 0x7f7f7f7fu) + 0x7f7f7f7fu) | w) & 0x80808080u;  // bit 7 of each non-zero byte
      return ((nz >> 7) * 0x01020408u) >> 24;                                     // -> bits 0..3
    };
    return nib(f.x) | (nib(f.y) << 4);
  }
  __device__ __forceinline__ uint32_t at(uint32_t b) const { return __byte_perm(f.x, f.y, b) & 0xffu; }
};
template <>
struct Flags<uint16_t> {
  uint4 f;
  __device__ __forceinline__ void load(uint32_t a) {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(f.x), "=r"(f.y), "=r"(f.z), "=r"(f.w) : "r"(a));
  }
  __device__ __forceinline__ bool any() const { return (f.x | f.y | f.z | f.w) != 0u; }
  __device__ __forceinline__ static void clear(uint32_t a) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(a), "r"(0u) : "memory");
  }
  __device__ __forceinline__ static void set(uint32_t table, uint32_t pos, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(table + 2u * pos), "r"(v) : "memory");
  }
  __device__ __forceinline__ uint32_t mask() const {
    auto two = [](uint32_t w) -> uint32_t {
      const uint32_t nz = (((w & 0x7fff7fffu) + 0x7fff7fffu) | w) & 0x80008000u;  // bit 15 of each non-zero half
      return ((nz >> 15) | (nz >> 30)) & 3u;
    };
    return two(f.x) | (two(f.y) << 2) | (two(f.z) << 4) | (two(f.w) << 6);
  }
  __device__ __forceinline__ uint32_t at(uint32_t b) const {
    const uint32_t lo = (b & 2u) ? f.y : f.x, hi = (b & 2u) ? f.w : f.z;
    const uint32_t w = (b & 4u) ? hi : lo;
    return (b & 1u) ? (w >> 16) : (w & 0xffffu);
  }
};

// exclusive in-lane prefix at entry b (0..7) of the inclusive prefixes g[0..7], by a select tree
__device__ __forceinline__ float prefix_before(const float g[8], uint32_t b) {
  const bool b0 = b & 1u, b1 = b & 2u, b2 = b & 4u;
  const float t0 = b0 ? g[0] : 0.f, t1 = b0 ? g[2] : g[1], t2 = b0 ? g[4] : g[3], t3 = b0 ? g[6] : g[5];
  const float u0 = b1 ? t1 : t0, u1 = b1 ? t3 : t2;
  return b2 ? u1 : u0;
}

// inclusive-prefix value G(t) of a lane: the sum of its first t entries, t clamped to [0, 8]
__device__ __forceinline__ float prefix_at(const float g[8], int t) {
  const int tt = max(t, 0);
  const float lo = prefix_before(g, static_cast<uint32_t>(tt) & 7u);
  return tt >= 8 ? g[7] : lo;
}

template <typename ColT, typename PtrT, bool CSER, typename FlagT, int D, int NT, bool PEERS>
__global__ void __launch_bounds__(NT, 1) k_matvec_stream(DotArgs a, const float *__restrict__ x,
                                                         float *__restrict__ y) {
  constexpr int kWarps = NT / 32;
  constexpr uint32_t kAlign = 16 / sizeof(ColT) < 8 ? 16 / sizeof(ColT) : 8;  // entries per 16 B piece, <= 8
  constexpr uint32_t kFull = 0xffffffffu;
  constexpr int kUni = 4;  // up to this many segment starts in a window are broadcast one by one
  constexpr int kAhead = kSegRing / 32;  // batches of segment bounds in flight
  extern __shared__ __align__(16) float xs[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(xs);
  const uint32_t oib = CSER ? static_cast<uint32_t>(a.oi_bits) / 8u : 0u;
  const StreamSmem L = stream_layout(a.k, a.n, kWarps, sizeof(FlagT), sizeof(PtrT), oib);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float *wv = reinterpret_cast<float *>(smem + L.wv);
  // 32-bit shared addresses of the tables (kept in registers)
  const uint32_t xs_s = smem_u32(xs), wv_s = xs_s + L.wv;
  const uint32_t flag_s = xs_s + L.flag + wid * kStreamWin * static_cast<uint32_t>(sizeof(FlagT));  // the warp's table
  const uint32_t myflag_s = flag_s + 8u * lane * static_cast<uint32_t>(sizeof(FlagT));                // the lane's 8 flags
  const uint32_t opr_s = xs_s + L.opr + wid * kSegRing * static_cast<uint32_t>(sizeof(PtrT));
  const uint32_t oir_s = xs_s + L.oir + wid * kSegRing * oib;
  uint64_t *xbar = reinterpret_cast<uint64_t *>(smem + L.bar);
  const ColT *col = static_cast<const ColT *>(a.col);
  const PtrT *op = static_cast<const PtrT *>(a.op);
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kWarps;
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kWarps + wid;
  const uint32_t R0 = static_cast<uint32_t>(gw * a.m / nw), R1 = static_cast<uint32_t>((gw + 1) * a.m / nw);
  pdl_launch_dependents();
  const bool x_async = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const uint32_t x_tma = x_async ? static_cast<uint32_t>(a.n * 4) & ~15u : 0u;
  if (threadIdx.x == 0) {
    mbar_init(xbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // x: one TMA bulk copy once the producer grid is done; the unaligned tail by thread 0
  if (threadIdx.x == 0) {
    pdl_wait();
    for (int64_t i = x_tma >> 2; i < a.n; ++i) xs[i] = __ldg(x + i);
    mbar_expect_tx(xbar, x_tma);
    constexpr uint32_t kChunk = 32768;
    for (uint32_t o = 0; o < x_tma; o += kChunk)
      bulk_g2s(reinterpret_cast<unsigned char *>(xs) + o, reinterpret_cast<const unsigned char *>(x) + o,
               min(kChunk, x_tma - o), xbar);
  }

  // row bounds: entries E(r), segments S(r) = rowPtr[r]; the warp's rows are contiguous in both streams
  auto row_e = [&](uint32_t r) -> uint32_t {
    return a.re ? __ldg(a.re + r) : ld_idx(op, load_index(a.rp, a.rp_bits, r));
  };
  auto row_s = [&](uint32_t r) -> uint32_t { return load_index(a.rp, a.rp_bits, r); };
  const bool have_rows = R0 < R1;
  const uint32_t e_beg = have_rows ? row_e(R0) : 0u, e_end = have_rows ? row_e(R1) : 0u;
  const uint32_t s_beg = have_rows ? row_s(R0) : 0u, s_end = have_rows ? row_s(R1) : 0u;

  // colI stream: windows of 256 entries from W0 (16 B aligned), D in flight in registers
  const uint32_t W0 = e_beg & ~(kAlign - 1u);
  const uint32_t e_lim = (e_end + kAlign - 1u) & ~(kAlign - 1u);
  Win<ColT> q[D];
#pragma unroll
  for (int u = 0; u < D; ++u) win_load(q[u], col, W0 + kStreamWin * u + 8u * lane, e_lim);

  // Segment-bound stream: batches of 32 consecutive segments from S0 (aligned down to 16), copied into
  // the warp's ring kAhead batches ahead (cp.async, one group per batch): omegaPtr by lanes 0-7, omegaI by
  // lanes 8-15.  Chunks wholly past the arrays (or the warp's last segment) are zero-filled.
  const uint32_t S0 = s_beg & ~15u;
  const uint32_t op_count = static_cast<uint32_t>(a.segs) + 1u, oi_count = static_cast<uint32_t>(a.segs);
  auto seg_issue = [&](uint32_t b) {  // batch b of the stream -> ring slot b % kAhead
    const uint32_t first = S0 + 32u * b;
    if (first <= s_end) {
      constexpr uint32_t kOpPer = 16u / sizeof(PtrT);  // values per 16 B
      const uint32_t j = static_cast<uint32_t>(lane);
      if (j < 32u / kOpPer) {
        const uint32_t s = first + j * kOpPer;
        cp_async16(opr_s + ((32u * b + j * kOpPer) & (kSegRing - 1u)) * static_cast<uint32_t>(sizeof(PtrT)),
                   op + (s < op_count ? s : 0u), s < op_count ? 16u : 0u);
      }
      if (CSER) {
        const uint32_t per = 16u / oib, jj = j - 8u;
        if (j >= 8u && jj < 32u / per) {
          const uint32_t s = first + jj * per;
          cp_async16(oir_s + ((32u * b + jj * per) & (kSegRing - 1u)) * oib,
                     static_cast<const unsigned char *>(a.oi) + static_cast<size_t>(s < oi_count ? s : 0u) * oib,
                     s < oi_count ? 16u : 0u);
        }
      }
    }
    cp_async_commit();
  };
#pragma unroll 1
  for (int b = 0; b < kAhead; ++b) seg_issue(b);

  // value slots: slot(i) = i + 1 below the background's position, i above it (never the background
  // itself), so slots run 1..k-1 and fit the flag type; slot 0 = no flag
  const uint32_t mode = static_cast<uint32_t>(a.mode);
  for (int i = threadIdx.x; i < a.k; i += NT) {
    if (static_cast<uint32_t>(i) != mode)
      wv[static_cast<uint32_t>(i) < mode ? i + 1 : i] = static_cast<float>(__ldg(a.omega + i) - a.bg);
  }
  if (threadIdx.x == 0) wv[0] = 0.f;
  Flags<FlagT>::clear(myflag_s);

  // current batch: lane j holds segment sb + j of the stream (first entry st, end en, omegaI value oiv)
  uint32_t sb = S0, st = 0, en = 0, nb = 0, kp8 = 0;  // kp8 = the segment's value slot << 8 (current row)
  uint32_t r = R0, e0 = 0, e1 = e_beg, s0 = 0, s1 = s_beg;
  auto slot_update = [&](uint32_t idx) { kp8 = (idx < mode ? idx + 1u : idx) << 8; };
  auto seg_take = [&]() {  // read batch nb from the ring (it and the next batch's first bound have landed)
    cp_async_wait<kAhead - 2>();
    __syncwarp();
    const uint32_t pos = 32u * nb + lane;
    st = lds_idx<PtrT>(opr_s + (pos & (kSegRing - 1u)) * static_cast<uint32_t>(sizeof(PtrT)));
    en = lds_idx<PtrT>(opr_s + ((pos + 1u) & (kSegRing - 1u)) * static_cast<uint32_t>(sizeof(PtrT)));
    sb = S0 + 32u * nb;
    if (CSER) {
      const uint32_t pa = oir_s + (pos & (kSegRing - 1u)) * oib;
      slot_update(oib == 1 ? lds_idx<uint8_t>(pa) : (oib == 2 ? lds_idx<uint16_t>(pa) : lds_idx<uint32_t>(pa)));
    } else {
      slot_update(sb + lane - s0 + 1u);
    }
    __syncwarp();
    seg_issue(nb + kAhead);
    ++nb;
  };
  uint32_t jdone = s_beg - S0;  // lanes of the first batch that belong to rows before R0
  float acc = 0.f, vcur = 0.f;
  const double bgy = a.bg != 0.0 ? a.bg * a.colsum[0] : 0.0;
  // Row bounds are held lane-parallel, 32 rows per group (lane j: row cg + j), and read by shuffle: no
  // global load stays pending across windows (a pending row-bound load shared a scoreboard with the
  // colI ring's loads and stalled the ring: profiles/r02_stream_notes.txt).
  uint32_t cg = R0, cgE = 0, cgS = 0;
  auto group_load = [&]() {
    const uint32_t rr = cg + lane;
    cgE = rr <= R1 ? row_e(rr) : 0u;
    cgS = rr <= R1 ? row_s(rr) : 0u;
  };
  if (have_rows) group_load();
  // Results leave the warp 32 rows at a time: lane j keeps y of the warp's row R0 + 32 g + j, and a full
  // group (or the warp's last rows) is written as one coalesced store -- to y and, for the row-sharded
  // exchange, to every peer's buffer (one 128 B NVLink store per 32 rows instead of 32 single-lane ones).
  // (the 32 slots live in shared memory: a register held across the walk cost the CSER instance 6%; and
  // the kernel without peers is its own instance that stores each result directly: the buffering cost it
  // 1.5% on one GPU)
  auto emit = [&](uint32_t row, float v) {
    if (!PEERS) {
      if (lane == 0) put_y(a, y, row, v);
      return;
    }
    float *yb = reinterpret_cast<float *>(smem + L.yb) + wid * 32;
    const uint32_t j = (row - R0) & 31u;
    if (lane == 0) yb[j] = v;
    if (j == 31u || row + 1 == R1) {
      __syncwarp();
      if (static_cast<uint32_t>(lane) <= j) put_y(a, y, row - j + lane, yb[lane]);
      __syncwarp();
    }
  };
  // position the walk at the first non-empty row at or after r (empty rows are written here)
  auto row_init = [&]() {
    while (r < R1) {
      if (r + 1 - cg >= 32u) {
        cg = r + 1;
        group_load();
      }
      e0 = e1;
      s0 = s1;
      e1 = __shfl_sync(kFull, cgE, static_cast<int>(r + 1 - cg));
      s1 = __shfl_sync(kFull, cgS, static_cast<int>(r + 1 - cg));
      if (e1 > e0) {
        acc = 0.f;
        vcur = 0.f;
        if (!CSER) slot_update(sb + lane - s0 + 1u);
        return;
      }
      emit(r, static_cast<float>(bgy));
      ++r;
    }
  };
  __syncthreads();  // value table, cleared flags
  if (have_rows) seg_take();
  row_init();
  bool x_ready = false;

  for (uint32_t wb = W0; wb < e_end; wb += kStreamWin * D) {
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const uint32_t wbu = wb + kStreamWin * u;
      if (wbu >= e_end) break;
      const uint32_t wend = wbu + kStreamWin, p0 = wbu + 8u * lane;
      uint32_t c[8];
      win_addrs<ColT>(q[u], xs_s, c);
      win_load(q[u], col, p0 + kStreamWin * D, e_lim);
      if (!x_ready) {
        mbar_wait(xbar, 0);
        x_ready = true;
      }
      // every row that meets this window (rows are contiguous in colI)
      while (r < R1 && e0 < wend) {
        float g[8], run = 0.f;
        if (e0 <= wbu && e1 >= wend) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            run += lds_f32(c[i]);
            g[i] = run;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t p = p0 + i;
            if (p >= e0 && p < e1) run += lds_f32(c[i]);
            g[i] = run;
          }
        }
        // Segments of this row whose first entry lies in this window, batch by batch.  Invariant: every
        // entry before the last start handled so far is accounted; gp = the lane's prefix at that start,
        // vcur (warp-uniform) = the value in force from it on.  Lanes below jdone are done (earlier
        // windows or rows); a lane past the row's last segment never starts.
        float gp = 0.f;
        while (true) {
          const uint32_t s = sb + lane;
          const uint32_t cnt = static_cast<uint32_t>(__popc(__ballot_sync(kFull, s < s1 && st < wend)));
          const bool mine = static_cast<uint32_t>(lane) >= jdone && static_cast<uint32_t>(lane) < cnt && en > st;
          uint32_t mm = __ballot_sync(kFull, mine);
          const int nstart = __popc(mm);
          if (nstart > kUni) {
            // many starts: through the flag table
            if (mine) Flags<FlagT>::set(flag_s, (st - wbu) & (kStreamWin - 1u), kp8 >> 8);
            __syncwarp();
            Flags<FlagT> fl;
            fl.load(myflag_s);
            if (fl.any()) Flags<FlagT>::clear(myflag_s);
            const uint32_t F = __ballot_sync(kFull, fl.any());
            // walk the lane's 8 entries in order (static positions: no prefix select, no per-flag loop; a
            // segment-dense row tail holds several flags per lane)
            float ghead = 0.f, glast = 0.f, vlast = 0.f, accl = 0.f;
            bool have = false;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
              const uint32_t slot = fl.at(b);
              if (slot != 0u) {
                const float gb = b ? g[b - 1] : 0.f;
                if (have)
                  accl = fmaf(vlast, gb - glast, accl);
                else
                  ghead = gb;
                have = true;
                vlast = lds_f32(wv_s + 4u * slot);
                glast = gb;
              }
            }
            const uint32_t below = F & ((1u << lane) - 1u);
            const bool above = ((F >> lane) >> 1) != 0u;
            const float vs = __shfl_sync(kFull, vlast, below ? 31 - __clz(static_cast<int>(below)) : lane);
            const float vin = below ? vs : vcur;
            if (have) {
              acc = fmaf(vin, ghead - gp, acc) + accl;
              gp = glast;
              if (above) {
                acc = fmaf(vlast, g[7] - glast, acc);
                gp = g[7];
              }
            } else if (above) {
              acc = fmaf(vin, g[7] - gp, acc);
              gp = g[7];
            }
            vcur = __shfl_sync(kFull, vlast, 31 - __clz(static_cast<int>(F | 1u)));
            __syncwarp();  // flags cleared before the next pass writes them
          } else if (nstart > 0) {
            // few starts: each one broadcast from the lane that holds the segment
            const uint32_t pk = ((st - wbu) & (kStreamWin - 1u)) | kp8;
            do {
              const uint32_t uu = __shfl_sync(kFull, pk, __ffs(static_cast<int>(mm)) - 1);
              mm &= mm - 1u;
              const float gt = prefix_at(g, static_cast<int>(uu & 255u) - 8 * lane);
              acc = fmaf(vcur, gt - gp, acc);
              gp = gt;
              vcur = lds_f32(wv_s + ((uu >> 8) << 2));
            } while (mm != 0u);
          }
          jdone = cnt;
          if (cnt == 32u && sb + 32u < s1) {  // batch used up inside this window: the next 32 segments
            seg_take();
            jdone = 0;
            continue;
          }
          break;
        }
        acc = fmaf(vcur, g[7] - gp, acc);
        if (e1 > wend) break;
        // the row ends in this window
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        emit(r, a.bg != 0.0 ? static_cast<float>(static_cast<double>(acc) + bgy) : acc);
        ++r;
        row_init();
      }
    }
  }
  if (!x_ready) mbar_wait(xbar, 0);  // no CTA exits with a bulk copy in flight
  cp_async_wait<0>();
}

template <typename ColT, typename PtrT, bool CSER, typename FlagT, int NT>
int launch_stream(const DotArgs &a, const float *x, float *y, cudaStream_t st) {
  constexpr int D = (sizeof(ColT) == 4 || NT > 768) ? 2 : 3;
  const size_t smem = stream_layout(a.k, a.n, NT / 32, sizeof(FlagT), sizeof(PtrT), CSER ? a.oi_bits / 8 : 0).total;
  auto kern = a.npeer > 0 ? k_matvec_stream<ColT, PtrT, CSER, FlagT, D, NT, true>
                          : k_matvec_stream<ColT, PtrT, CSER, FlagT, D, NT, false>;
  if (int rc_ = allow_max_smem(kern)) return rc_;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(num_sms(), ceil_div(a.m, NT / 32))));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
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

template <typename ColT, typename PtrT, bool CSER>
int by_flag(const DotArgs &a, const float *x, float *y, cudaStream_t st) {
  // 28 warps at <= 72 registers with two colI windows in flight (measured on the 32768^2 layer: CER 296 us,
  // CSER 284 us; 24 warps with three windows 309 / 316 us; 32 warps at 64 registers 296 / 330 us -- the CSER
  // instance then spills a ring slot, i.e. waits for the load it just issued).  CERDOT_PATH_MATVEC_NT = 768
  // pins the 24-warp variant (A/B).
  if (kernel_path(CERDOT_PATH_MATVEC_NT) == 768)
    return a.k <= 256 ? launch_stream<ColT, PtrT, CSER, uint8_t, 768>(a, x, y, st)
                      : launch_stream<ColT, PtrT, CSER, uint16_t, 768>(a, x, y, st);
  return a.k <= 256 ? launch_stream<ColT, PtrT, CSER, uint8_t, 896>(a, x, y, st)
                    : launch_stream<ColT, PtrT, CSER, uint16_t, 896>(a, x, y, st);
}

template <typename ColT, bool CSER>
int by_ptr(const DotArgs &a, int op_bits, const float *x, float *y, cudaStream_t st) {
  switch (op_bits) {
    case 8: return by_flag<ColT, uint8_t, CSER>(a, x, y, st);
    case 16: return by_flag<ColT, uint16_t, CSER>(a, x, y, st);
    default: return by_flag<ColT, uint32_t, CSER>(a, x, y, st);
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

bool matvec_stream_fits(int64_t k, int64_t n, int op_bits, int oi_bits) {
  if (k > kSmemValues || k < 1) return false;
  return stream_layout(k, n, 896 / 32, k <= 256 ? 1 : 2, op_bits / 8, oi_bits / 8).total <=
         static_cast<uint32_t>(kMaxSmemBytes);
}

int matvec_stream(const DotArgs &a, bool cser, int col_bits, int op_bits, const float *x, float *y, cudaStream_t st) {
  return cser ? by_col<true>(a, col_bits, op_bits, x, y, st) : by_col<false>(a, col_bits, op_bits, x, y, st);
}

}  // namespace cerdot
