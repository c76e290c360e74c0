// CER / CSER dot product on sm_100a, fp32, no tensor cores.
//
// Reference: lemt kernels.py:283-301 (_dot_segmented), float64:
//   y[r] = sum_seg (omega[seg] - bg) * (sum_{i in seg} x[colI[i]])  (+ bg * sum(x) when bg != 0)
//
// Mat-vec (batch 1) — k_matvec, HBM-bound:
//   * persistent CTAs stage x in shared memory once (random gathers from smem
//     cost ~3.5 bank-cycles per 32 lanes; from L1 they cost one wavefront per
//     distinct 128 B line, ~9x more), plus the per-element segment values
//     (float)(omega[k] - bg);
//   * a warp walks one row in windows of 32 x EPL entries: every lane loads EPL
//     consecutive colI entries with 16 B vector loads (coalesced stream), the
//     next window is prefetched into registers;
//   * the row's segment starts (omegaPtr) are registered lane-parallel into a
//     per-warp slot table (slot = entry position -> element index k), so each
//     lane knows where segments begin inside its run;
//   * each lane sums its run segment by segment; a segment that ends inside the
//     lane is multiplied there; pieces that cross lanes are joined by a warp
//     segmented scan (fixed Hillis-Steele order) and multiplied once at the
//     lane where the segment closes; the open segment carries across windows.
//     Every non-empty segment is multiplied exactly once (kernels.py:296).
// Mat-mat (batch > 1) — k_matmat, gather-bound (L2 -> SM):
//   * a warp owns (row, 32*V batch columns); 32 entries at a time are loaded
//     lane-parallel with their segment heads, then walked with V-wide vector
//     loads of the X rows, eight in flight; one fma per segment per column.
//
// Summation order (the 1e-5 parity bar): fp32 segment sums
// in colI order within a lane, lane pieces joined left-to-right by the scan;
// one fp32 fma per segment into per-lane row accumulators; lanes combined by
// an xor butterfly.  Background correction: sum(x) in fp64 (fixed tree),
// bg*sum in fp64, added to the fp32 row sum in fp64, rounded once.
// Deterministic: no floating-point atomics, fixed reduction order.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <map>
#include <set>
#include <utility>
#include <string>

#include "common.cuh"
#include "dotk.cuh"
#include "encode.cuh"
#include "tileview.cuh"

namespace cerdot {

namespace {


// Shared-memory carve-up of k_matvec (byte offsets; all 16 B aligned).
struct MatvecSmem {
  uint32_t bar, wv, pre, off, ring_op, ring_oi, xs, total;
};
__host__ __device__ __forceinline__ MatvecSmem matvec_layout(int64_t k, int64_t n_smem, uint32_t warps, uint32_t depth,
                                                             uint32_t oi_bytes) {
  MatvecSmem L{};
  uint32_t o = 0;
  auto take = [&](uint32_t bytes) {
    const uint32_t r = o;
    o += (bytes + 15u) & ~15u;
    return r;
  };
  L.bar = take(16u);
  L.wv = take(static_cast<uint32_t>(min64(k, kSmemValues)) * 4u);
  L.pre = take(warps * kWin * 4u);
  L.off = take(warps * 32u * 8u);  // per-warp lane offsets, (hi, lo) fp32 pairs
  L.ring_op = take(warps * depth * 128u);
  L.ring_oi = take(warps * depth * 32u * oi_bytes);
  L.xs = take(static_cast<uint32_t>(n_smem) * 4u);
  L.total = o;
  return L;
}

template <typename ColT, typename PtrT, bool CSER, bool XSMEM, int NT, int NBUF, int MINB, int D>
__global__ void __launch_bounds__(NT, MINB) k_matvec(DotArgs a, const float *__restrict__ x, float *__restrict__ y) {
  constexpr int kWarps = NT / 32;
  using CV = ColVec<ColT>;
  constexpr uint32_t W = kWin;
  constexpr int NV = kEPL / CV::kPer;
  constexpr uint32_t kAlign = CV::kPer;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t oib = CSER ? static_cast<uint32_t>(a.oi_bits / 8) : 1u;
  MatvecSmem L = matvec_layout(a.k, XSMEM ? a.n : 0, kWarps, D, oib);
  float *wv = reinterpret_cast<float *>(smem + L.wv);
  float *pre = reinterpret_cast<float *>(smem + L.pre) + wid * W;
  float2 *off = reinterpret_cast<float2 *>(smem + L.off) + wid * 32;
  unsigned char *ring_op = smem + L.ring_op + wid * D * 128;
  unsigned char *ring_oi = smem + L.ring_oi + wid * D * 32 * oib;
  float *xs = reinterpret_cast<float *>(smem + L.xs);
  const ColT *col = static_cast<const ColT *>(a.col);
  const PtrT *op = static_cast<const PtrT *>(a.op);
  const uint32_t m = static_cast<uint32_t>(a.m);
  const uint64_t nw_total = static_cast<uint64_t>(gridDim.x) * kWarps;
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kWarps + wid;
  const uint32_t R0 = static_cast<uint32_t>(gw * m / nw_total), R1 = static_cast<uint32_t>((gw + 1) * m / nw_total);
  pdl_launch_dependents();  // the next grid may start its own index prologue as our CTAs retire
  // x staging: one TMA bulk copy (16 B-aligned part of x) issued at kernel start by thread 0 once the
  // producer grid has finished, so it overlaps every warp's index chain below; the unaligned tail and
  // the omega table are staged by all threads after their own chain.
  uint64_t *xbar = reinterpret_cast<uint64_t *>(smem + L.bar), *wbar = xbar + 1;
  const bool x_async = XSMEM && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const uint32_t x_tma_bytes = x_async ? static_cast<uint32_t>(a.n * 4) & ~15u : 0u;
  if (threadIdx.x == 0) {
    mbar_init(xbar, 1);           // x: thread 0's arrive + the TMA bytes
    mbar_init(wbar, blockDim.x);  // omega table: every thread arrives once its share is stored
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (x_async && threadIdx.x == 0) {
    pdl_wait();
    for (int64_t i = x_tma_bytes >> 2; i < a.n; ++i) xs[i] = __ldg(x + i);  // <= 3 unaligned tail values
    mbar_expect_tx(xbar, x_tma_bytes);
    constexpr uint32_t kChunk = 32768;
    for (uint32_t o = 0; o < x_tma_bytes; o += kChunk)
      bulk_g2s(reinterpret_cast<unsigned char *>(xs) + o, reinterpret_cast<const unsigned char *>(x) + o,
               min(kChunk, x_tma_bytes - o), xbar);
  }
  const int kv = static_cast<int>(min64(a.k, kSmemValues));
  const double wd0 = static_cast<int>(threadIdx.x) < kv ? __ldg(a.omega + threadIdx.x) : 0.0;
#ifdef CERDOT_TRACE_KERNELS
  unsigned long long tr[9] = {gtimer(), 0, 0, 0, 0, 0, 0, 0, 0};
#define CERDOT_TR(i, dep) \
  if (a.dbg && tr[i] == 0) tr[i] = gtimer() + (dep)
#else
#define CERDOT_TR(i, dep)
#endif

  // ------------------------------------------------------------ row groups (31 rows per lane-register group)
  uint32_t gG = R0, g_rp = 0, g_ep = 0;
  auto load_group = [&](uint32_t g) {
    gG = g;
    const uint32_t idx = g + lane;
    g_rp = 0;
    g_ep = 0;
    if (idx <= R1 && R0 < R1) {
      g_rp = load_index(a.rp, a.rp_bits, idx);
      g_ep = a.re ? __ldg(a.re + idx) : ld_idx(op, g_rp);  // row_entry: no rowPtr -> omegaPtr dependence
    }
  };
  load_group(R0);
  const uint32_t s_beg = __shfl_sync(0xffffffffu, g_rp, 0);
  const uint32_t s_end = R0 < R1 ? load_index(a.rp, a.rp_bits, R1) : s_beg;
  const uint32_t e_beg = __shfl_sync(0xffffffffu, g_ep, 0);
  const uint32_t e_end = R0 < R1 ? (a.re ? __ldg(a.re + R1) : ld_idx(op, s_end)) : e_beg;

  // ------------------------------------------------------------ L2 stream prefetch (TMA engine)
  constexpr uint32_t kChunkE = 4096 / sizeof(ColT), kAheadE = 24576 / sizeof(ColT);
  constexpr uint32_t kChunkS = 4096 / sizeof(PtrT), kAheadS = 8192 / sizeof(PtrT);
  uint32_t pf_e = e_beg & ~(16u / sizeof(ColT) - 1u), pf_s = s_beg & ~(16u / sizeof(PtrT) - 1u);
  auto stream_prefetch = [&](uint32_t e_pos, uint32_t s_pos) {
    if (lane == 0) {
      while (pf_e < e_end && pf_e < e_pos + kAheadE) {
        const uint32_t ne = min(kChunkE, (e_end - pf_e + 15u) & ~15u);
        bulk_prefetch_l2(col + pf_e, ne * sizeof(ColT));
        pf_e += ne;
      }
      while (pf_s < s_end && pf_s < s_pos + kAheadS) {
        const uint32_t ns = min(kChunkS, (s_end - pf_s + 15u) & ~15u);
        bulk_prefetch_l2(op + pf_s, ns * sizeof(PtrT));
        pf_s += ns;
      }
    }
  };
  stream_prefetch(pf_e, pf_s);

  // ------------------------------------------------------------ segment FIFO: smem ring filled by cp.async
  // batch t holds omegaPtr[fb + 32t .. +32) (raw PtrT) and omegaI of the same segments (CSER)
  const uint32_t fb = s_beg & ~31u;
  uint32_t ft = 0;                      // batch being consumed
  auto fifo_issue = [&](uint32_t tt) {
    const uint32_t base = fb + 32u * tt;
    const int slot = static_cast<int>(tt % D);
    constexpr uint32_t per = 4u / sizeof(PtrT) ? 4u / sizeof(PtrT) : 1u;  // entries per 4 B chunk
    const uint32_t nchunks = 32u / per;
    if (static_cast<uint32_t>(lane) < nchunks) {
      const uint32_t e = base + lane * per;
      if (e <= static_cast<uint32_t>(a.segs) && base <= s_end)
        cp_async4(ring_op + slot * 128 + lane * 4, op + e);
    }
    if (CSER) {
      // omegaI entries per 4 B chunk and chunks per 32 segments, by shifts (a runtime integer division
      // here cost ~20 instructions per batch per warp: the CSER kernel executed 19% more instructions)
      const uint32_t ob_bytes = a.oi_bits >> 3;
      const uint32_t osh = ob_bytes == 1 ? 0u : (ob_bytes == 2 ? 1u : 2u);
      const uint32_t per_oi = 4u >> osh, nch = 8u << osh;
      if (static_cast<uint32_t>(lane) < nch) {
        const uint32_t e = base + lane * per_oi;
        if (e < static_cast<uint32_t>(a.segs) && base < s_end)
          cp_async4(ring_oi + slot * 32 * ob_bytes + lane * 4, static_cast<const unsigned char *>(a.oi) + e * ob_bytes);
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int i = 0; i < D; ++i) fifo_issue(i);
  auto fifo_shift = [&]() {
    fifo_issue(ft + D);
    ++ft;
  };
  // the ring is a circular buffer of D*32 consecutive segments: segment s sits at (s - fb) % (32 D)
  // inside its batch's 128 B slot (entries of PtrT / omegaI width)
  auto ring_ptr = [&](uint32_t s) -> uint32_t {
    const uint32_t r = (s - fb) % (32u * D);
    return reinterpret_cast<const PtrT *>(ring_op + (r >> 5) * 128)[r & 31u];
  };
  auto ring_oi_val = [&](uint32_t s) -> int {
    const uint32_t r = (s - fb) % (32u * D);
    const unsigned char *slot = ring_oi + (r >> 5) * 32u * oib;
    switch (a.oi_bits) {
      case 8: return slot[r & 31u];
      case 16: return reinterpret_cast<const uint16_t *>(slot)[r & 31u];
      default: return static_cast<int>(reinterpret_cast<const uint32_t *>(slot)[r & 31u]);
    }
  };

  // ------------------------------------------------------------ window generator (runs 3 windows ahead)
  struct Win {
    uint32_t row, w0, s0, s1, e0, e1;
  };
  uint32_t g_row = R0, g_w0 = 0;
  auto row_meta = [&](uint32_t r, Win &w) {
    w.row = r;
    w.s0 = __shfl_sync(0xffffffffu, g_rp, static_cast<int>(r - gG));
    w.s1 = __shfl_sync(0xffffffffu, g_rp, static_cast<int>(r - gG + 1));
    w.e0 = __shfl_sync(0xffffffffu, g_ep, static_cast<int>(r - gG));
    w.e1 = __shfl_sync(0xffffffffu, g_ep, static_cast<int>(r - gG + 1));
  };
  Win gcur;  // metadata of the generator's current row
  auto seek_row = [&](uint32_t r) {  // first non-empty row >= r (rows of entries; empty rows are emitted by the consumer)
    for (; r < R1; ++r) {
      if (r >= gG + 31) load_group(r);
      row_meta(r, gcur);
      if (gcur.e1 > gcur.e0) break;
    }
    g_row = r;
    g_w0 = r < R1 ? (gcur.e0 & ~(kAlign - 1)) : 0u;
  };
  seek_row(R0);
  auto gen = [&](Win &w, uint4 *buf) {
    w = gcur;
    w.row = g_row;
    w.w0 = g_w0;
    if (g_row >= R1) return;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const uint32_t vp = g_w0 + lane * kEPL + v * CV::kPer;
      buf[v] = vp < gcur.e1 ? ld_stream(col + vp) : make_uint4(0u, 0u, 0u, 0u);
    }
    if (g_w0 + W < gcur.e1) g_w0 += W;
    else seek_row(g_row + 1);
  };
  Win ma, mb, mc;
  uint4 A[NV], B[NV], C[NV];
  gen(ma, A);
  if (NBUF > 1) {
    gen(mb, B);
    gen(mc, C);
  }
  CERDOT_TR(1, A[0].x & 0u);  // forces the prologue loads to complete for the timestamp

  // ------------------------------------------------------------ wait for the producer of x
  pdl_wait();
  CERDOT_TR(2, 0u);
  if (static_cast<int>(threadIdx.x) < kv) wv[threadIdx.x] = static_cast<float>(wd0 - a.bg);
  for (int i = threadIdx.x + blockDim.x; i < kv; i += blockDim.x) wv[i] = static_cast<float>(__ldg(a.omega + i) - a.bg);
  mbar_arrive(wbar);  // no CTA-wide barrier: each warp waits for x / the omega table only when it needs them
  if (XSMEM && !x_async) {  // misaligned x: cooperative staging
    for (int64_t i = threadIdx.x; i < a.n; i += blockDim.x) xs[i] = __ldg(x + i);
    __syncthreads();
  }
  bool x_ready = !x_async, w_ready = false;
  const float y_empty = a.bg != 0.0 ? static_cast<float>(a.bg * a.colsum[0]) : 0.f;

  // ------------------------------------------------------------ consumer
  uint32_t next_emit = R0;  // first row whose y is not written yet
  float acc = 0.f, carry = 0.f;
  uint32_t sc = 0;
  auto emit_empty = [&](uint32_t upto) {
    for (uint32_t r = next_emit + lane; r < upto; r += 32) put_y(a, y, r, y_empty);
    next_emit = max(next_emit, upto);
  };
  auto process = [&](const uint4 *cur, const Win &w) {
    if (w.w0 == (w.e0 & ~(kAlign - 1))) {  // first window of the row
      emit_empty(w.row);
      acc = 0.f;
      carry = 0.f;
      sc = w.s0;
      while (sc >= fb + 32u * (ft + 1)) fifo_shift();
    }
    const uint32_t w0 = w.w0, wn = w0 + W;
    stream_prefetch(w0, fb + 32u * ft);
    // whole row in this window: issue its first 128 segment bounds (and omegaI) now, so the loads are
    // in flight during the gather below (they do not depend on x)
    const bool single = w.w0 == (w.e0 & ~(kAlign - 1)) && wn >= w.e1;
    constexpr int kPre = NBUF > 1 ? 1 : 4;  // register budget: the 3-buffer variant keeps one prefetch batch
    uint32_t pen[kPre];
    if (single) {
#pragma unroll
      for (int i = 0; i < kPre; ++i) {
        const uint32_t sidx = w.s0 + lane + 32u * i;
        pen[i] = sidx < w.s1 ? __ldg(op + sidx + 1) : 0u;
      }
      // CSER omegaI of the same segments: prefetched into L1 now (no registers held across the gather,
      // where they would spill and stall on the load), read after it
      if (CSER) {
        const uint32_t ob = a.oi_bits / 8;
        const uintptr_t lo = reinterpret_cast<uintptr_t>(a.oi) + w.s0 * ob;
        const uintptr_t hi = reinterpret_cast<uintptr_t>(a.oi) + min(w.s1, w.s0 + 32u * kPre) * ob;
        const uintptr_t line = (lo & ~uintptr_t(127)) + static_cast<uintptr_t>(lane) * 128u;
        if (line < hi) asm volatile("prefetch.global.L1 [%0];" ::"l"(line));
      }
    }
    if (!x_ready) {
      mbar_wait(xbar, 0);
      x_ready = true;
      CERDOT_TR(3, 0u);
    }
    const float run = (w0 >= w.e0 && wn <= w.e1)
                          ? gather_prefix<ColT, XSMEM, false>(cur, w0, w.e0, w.e1, xs, x, pre, lane)
                          : gather_prefix<ColT, XSMEM, true>(cur, w0, w.e0, w.e1, xs, x, pre, lane);
    // Lane offsets (exclusive scan of the lane totals), scanned in fp64 and kept as an fp32 pair
    // hi + lo.  A segment sum is a difference of window-global prefixes G; with all-positive x a plain
    // fp32 offset (a sum of up to ~1000 entries) cancels against a segment of a few entries and its
    // rounding dominates (measured: 1.8e-5 on AlexNet fc6 with x = |N(0,1)|).  With the pair, the hi
    // parts of two nearby prefixes subtract exactly (Sterbenz) and only the fp32 lane-local prefixes
    // (<= 32 entries) round; per-segment arithmetic stays fp32 (an fp64 G cost 11-21% of the call).
    double incl = run;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t;
    }
    {
      const double up = __shfl_up_sync(0xffffffffu, incl, 1);  // every lane takes part in the shuffle
      const double excl = lane ? up : 0.0;
      const float hi = static_cast<float>(excl);
      off[lane] = make_float2(hi, static_cast<float>(excl - static_cast<double>(hi)));
    }
    __syncwarp();
    CERDOT_TR(5, static_cast<uint32_t>(incl) & 0u);
    // window-global inclusive prefix at window position p as (hi, lo + lane-local prefix)
    struct GP {
      float hi, lo;
    };
    auto G = [&](uint32_t p) -> GP {
      const float2 o = off[p >> 5];
      return GP{o.x, o.y + pre[ppos(p)]};
    };
    if (!w_ready) {
      mbar_wait(wbar, 0);
      w_ready = true;
    }
    if (single) {
      // ---- the whole row is in this window: lane i of a batch takes segment s0 + 32t + i, reads the
      // window prefix at its end and gets its start value (the previous segment's end) by shuffle
      uint32_t e_prev = w.e0;  // end of the previous segment
      float p_prev = 0.f;      // its lane-local prefix (entries before e0 were masked to 0)
      // segment [st, en): G(en - 1) - G(st - 1), G = lane offset (hi, lo) + lane-local prefix; the lane-local
      // prefix at st - 1 is the previous segment's end value (shuffled), the offsets come from the
      // 32-entry table (one random prefix-table read per segment)
      auto seg = [&](uint32_t en, int k, bool valid) {
        const bool has = valid && en > w0;
        const float pe = has ? pre[ppos(en - 1u - w0)] : 0.f;
        uint32_t st = __shfl_up_sync(0xffffffffu, en, 1);
        float ps = __shfl_up_sync(0xffffffffu, pe, 1);
        if (lane == 0) {
          st = e_prev;
          ps = p_prev;
        }
        e_prev = __shfl_sync(0xffffffffu, en, 31);
        p_prev = __shfl_sync(0xffffffffu, pe, 31);
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
      for (int i = 0; i < kPre; ++i) {
        const uint32_t sidx = w.s0 + lane + 32u * i;
        const int k = sidx < w.s1 ? (CSER ? static_cast<int>(load_index(a.oi, a.oi_bits, sidx))
                                          : static_cast<int>(sidx - w.s0 + 1))
                                  : 0;
        seg(pen[i], k, sidx < w.s1);
      }
      for (uint32_t base = w.s0 + 32u * kPre; base < w.s1; base += 32) {  // rows with > 32 kPre segments
        const uint32_t sidx = base + lane;
        const bool valid = sidx < w.s1;
        const uint32_t en = valid ? static_cast<uint32_t>(__ldg(op + sidx + 1)) : 0u;
        const int k = valid ? (CSER ? static_cast<int>(load_index(a.oi, a.oi_bits, sidx))
                                    : static_cast<int>(sidx - w.s0 + 1))
                            : 0;
        seg(en, k, valid);
      }
      sc = w.s1;
    } else
    // ---- segments overlapping this window: one lane per segment
    for (;;) {
      cp_async_wait<D - 2>();  // batches ft and ft+1 hold segments [sc, sc + 32]
      __syncwarp();
      const uint32_t s = sc + lane;
      const uint32_t st = ring_ptr(s);
      const uint32_t en = ring_ptr(s + 1);
      const bool take = s < w.s1 && st < wn;
      const bool done = take && en <= wn;
      const bool live = take && en > st;
      float total = 0.f;
      if (live) {
        const uint32_t lo = st > w0 ? st - w0 : 0u;
        const uint32_t b = (en < wn ? en - w0 : W) - 1u;
        const float pb = pre[ppos(b)];
        if (lo == 0u) {
          const float2 ob = off[b >> 5];
          total = ob.x + (ob.y + pb);
          if (st < w0) total = carry + total;  // the segment continued from the previous window
        } else {
          const uint32_t a0 = lo - 1u;
          const float pa = pre[ppos(a0)];
          if ((a0 >> 5) == (b >> 5)) {
            total = pb - pa;
          } else {
            const float2 ob = off[b >> 5], oa = off[a0 >> 5];
            total = (ob.x - oa.x) + ((ob.y + pb) - (oa.y + pa));
          }
        }
        if (done) acc = fmaf(wv[CSER ? ring_oi_val(s) : static_cast<int>(s - w.s0 + 1)], total, acc);
      }
      const unsigned done_m = __ballot_sync(0xffffffffu, done);
      const unsigned open_m = __ballot_sync(0xffffffffu, live && !done);
      if (open_m) carry = __shfl_sync(0xffffffffu, total, __ffs(open_m) - 1);
      const int ndone = __popc(done_m);
      sc += ndone;
      while (sc >= fb + 32u * (ft + 1)) fifo_shift();
      if (ndone < 32) break;
    }
    __syncwarp();
    CERDOT_TR(6, __float_as_uint(acc) & 0u);
    if (wn >= w.e1) {  // last window of the row
      float r = acc;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
      if (lane == 0) put_y(a, y, w.row, a.bg != 0.0 ? static_cast<float>(static_cast<double>(r) + a.bg * a.colsum[0]) : r);
      next_emit = w.row + 1;
#ifdef CERDOT_TRACE_KERNELS
      if (a.dbg) tr[7] = gtimer();
#endif
    }
  };
  if (NBUF > 1) {  // three windows in flight, statically rolled (no register moves)
    for (;;) {
      if (ma.row >= R1) break;
      process(A, ma);
      gen(ma, A);
      if (mb.row >= R1) break;
      process(B, mb);
      gen(mb, B);
      if (mc.row >= R1) break;
      process(C, mc);
      gen(mc, C);
    }
  } else {
    while (ma.row < R1) {
      process(A, ma);
      gen(ma, A);
    }
  }
  emit_empty(R1);
  cp_async_wait<0>();
#ifdef CERDOT_TRACE_KERNELS
  if (a.dbg) tr[8] = gtimer();
#endif
  if (x_async && threadIdx.x == 0) mbar_wait(xbar, 0);  // the CTA must not retire with the x copy in flight
#ifdef CERDOT_TRACE_KERNELS
  if (a.dbg && lane == 0 && (blockIdx.x % 37) == 0 && (wid == 0 || wid == kWarps - 1)) {
    tr[4] = gtimer();
    printf("TRACE cta %d warp %d rows %u start %llu prologue %llu wait %llu staged %llu end %llu gath %llu seg %llu "
           "rowdone %llu drained %llu\n",
           blockIdx.x, wid, R1 - R0, tr[0], tr[1], tr[2], tr[3], tr[4], tr[5], tr[6], tr[7], tr[8]);
  }
#endif
}

// ---------------------------------------------------------------------------------------------
// Mat-vec, CTA-tile pipeline (rows that fit a tile): a persistent CTA owns a block of rows, groups
// them into tiles of whole rows (<= kTileE entries, <= kTileS segments) and streams each tile's
// colI / omegaPtr / omegaI ranges into double-buffered shared memory with TMA bulk copies
// (cp.async.bulk + mbarrier).  Per tile, all threads: (A) gather x from smem and build per-thread
// prefix sums, (B) a block scan of thread totals, (C) warp-per-row segment sums as hierarchical
// prefix differences (thread / warp / tile levels, so no long-prefix cancellation), one fma per
// segment, warp reduction per row.
constexpr int kTileNT = 768;  // 24 warps: a 12288-entry tile holds four ResNet-conv rows (one tile per CTA; 512 threads
                                // and 8192 entries needed two tiles for 46% of the CTAs: 7.8 / 8.2 -> 7.2 / 7.8 us)
constexpr int kTileWarps = kTileNT / 32;
constexpr int kTileEPT = 16;                                  // entries per thread (>= 16 B of u8 colI)
constexpr uint32_t kTileCap = kTileNT * kTileEPT;            // aligned entry slots (12288)
constexpr uint32_t kTileE = kTileCap - 32;                   // entries per tile (16 B alignment slack)
constexpr uint32_t kTileS = 2048;                             // segments per tile
constexpr uint32_t kTileRows = 1024;                          // rows staged per row group

struct TileSmem {
  uint32_t xs, wv, rp, ep, trow, stage, stage_bytes, col_off, op_off, oi_off, pre, tex, tinc, wex, winc, bar, total;
};
__host__ __device__ __forceinline__ TileSmem tile_layout(int64_t k, int64_t n, int col_bytes, int ptr_bytes,
                                                         int oi_bytes) {
  TileSmem L{};
  uint32_t o = 0;
  auto take = [&](uint32_t b) {
    const uint32_t r = o;
    o += (b + 15u) & ~15u;
    return r;
  };
  L.bar = take(2 * 8);
  L.xs = take(static_cast<uint32_t>(n) * 4u);
  L.wv = take(static_cast<uint32_t>(min64(k, kSmemValues)) * 4u);
  L.rp = take((kTileRows + 1) * 4u);
  L.ep = take((kTileRows + 1) * 4u);
  L.trow = take((kTileRows + 2) * 4u);
  L.col_off = 0;
  L.op_off = (kTileCap * col_bytes + 15u) & ~15u;
  L.oi_off = L.op_off + (((kTileS + 1) * ptr_bytes + 32u + 15u) & ~15u);
  L.stage_bytes = L.oi_off + ((kTileS * oi_bytes + 32u + 15u) & ~15u);
  L.stage = take(2 * L.stage_bytes);
  L.pre = take(kTileCap * 4u);
  L.tex = take(kTileNT * 4u);
  L.tinc = take(kTileNT * 4u);
  L.wex = take(kTileWarps * 4u);
  L.winc = take(kTileWarps * 4u);
  L.total = o;
  return L;
}

// prefix-table slot of aligned entry q (thread q/EPT, item j=q%EPT): (j/4)*NT*4 + thread*4 + j%4
__device__ __forceinline__ uint32_t tpos(uint32_t q) {
  return ((q % kTileEPT) >> 2) * (kTileNT * 4u) + (q / kTileEPT) * 4u + (q & 3u);
}

template <typename ColT, typename PtrT, bool CSER>
__global__ void __launch_bounds__(kTileNT, 1) k_matvec_tile(DotArgs a, const float *__restrict__ x,
                                                            float *__restrict__ y) {
  using CV = ColVec<ColT>;
  constexpr int NVT = kTileEPT / CV::kPer;  // 16 B vectors per thread per tile
  extern __shared__ __align__(16) unsigned char smem[];
  const int oib = CSER ? a.oi_bits / 8 : 1;
  const TileSmem L = tile_layout(a.k, a.n, sizeof(ColT), sizeof(PtrT), oib);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + L.bar);
  float *xs = reinterpret_cast<float *>(smem + L.xs);
  float *wv = reinterpret_cast<float *>(smem + L.wv);
  uint32_t *rp_s = reinterpret_cast<uint32_t *>(smem + L.rp);
  uint32_t *ep_s = reinterpret_cast<uint32_t *>(smem + L.ep);
  uint32_t *trow = reinterpret_cast<uint32_t *>(smem + L.trow);
  float *pre = reinterpret_cast<float *>(smem + L.pre);
  float *tex = reinterpret_cast<float *>(smem + L.tex);
  float *tinc = reinterpret_cast<float *>(smem + L.tinc);
  float *wex = reinterpret_cast<float *>(smem + L.wex);
  float *winc = reinterpret_cast<float *>(smem + L.winc);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const ColT *col = static_cast<const ColT *>(a.col);
  const PtrT *op = static_cast<const PtrT *>(a.op);
  const unsigned char *oi = static_cast<const unsigned char *>(a.oi);
  const uint32_t m = static_cast<uint32_t>(a.m);
  const uint32_t R0 = static_cast<uint32_t>(static_cast<uint64_t>(blockIdx.x) * m / gridDim.x);
  const uint32_t R1 = static_cast<uint32_t>(static_cast<uint64_t>(blockIdx.x + 1) * m / gridDim.x);
  pdl_launch_dependents();
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t issued = 0, consumed = 0;  // tiles issued / consumed by this CTA (stage = u % 2)
  bool staged_x = false;
  float y_empty = 0.f;

  // TMA issue of one tile (rows [ta, tb) of the current group) into stage u % 2
  auto issue = [&](uint32_t ta, uint32_t tb, uint32_t u) {
    unsigned char *st = smem + L.stage + (u & 1u) * L.stage_bytes;
    const uint32_t Sa = rp_s[ta], Sb = rp_s[tb], Ea = ep_s[ta], Eb = ep_s[tb];
    const uintptr_t c0 = reinterpret_cast<uintptr_t>(col + Ea) & ~uintptr_t(15);
    const uintptr_t c1 = (reinterpret_cast<uintptr_t>(col + Eb) + 15) & ~uintptr_t(15);
    const uintptr_t o0 = reinterpret_cast<uintptr_t>(op + Sa) & ~uintptr_t(15);
    const uintptr_t o1 = (reinterpret_cast<uintptr_t>(op + Sb + 1) + 15) & ~uintptr_t(15);
    uintptr_t i0 = 0, i1 = 0;
    if (CSER && Sb > Sa) {
      i0 = reinterpret_cast<uintptr_t>(oi + static_cast<size_t>(Sa) * oib) & ~uintptr_t(15);
      i1 = (reinterpret_cast<uintptr_t>(oi + static_cast<size_t>(Sb) * oib) + 15) & ~uintptr_t(15);
    }
    const uint32_t nc = Eb > Ea ? static_cast<uint32_t>(c1 - c0) : 0u;
    const uint32_t no = static_cast<uint32_t>(o1 - o0), ni = static_cast<uint32_t>(i1 - i0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&bar[u & 1u], nc + no + ni);
    if (nc) bulk_g2s(st + L.col_off, reinterpret_cast<const void *>(c0), nc, &bar[u & 1u]);
    bulk_g2s(st + L.op_off, reinterpret_cast<const void *>(o0), no, &bar[u & 1u]);
    if (ni) bulk_g2s(st + L.oi_off, reinterpret_cast<const void *>(i0), ni, &bar[u & 1u]);
  };

  for (uint32_t g0 = R0; g0 < R1; g0 += kTileRows) {
    const uint32_t g1 = min(R1, g0 + kTileRows), ng = g1 - g0;
    __syncthreads();  // previous group's tiles fully consumed
    for (uint32_t i = tid; i <= ng; i += kTileNT) {
      rp_s[i] = load_index(a.rp, a.rp_bits, g0 + i);
      if (a.re) ep_s[i] = __ldg(a.re + g0 + i);  // row_entry: both loads in flight together
    }
    __syncthreads();
    if (!a.re) {
      for (uint32_t i = tid; i <= ng; i += kTileNT) ep_s[i] = ld_idx(op, rp_s[i]);
      __syncthreads();
    }
    if (tid == 0) {  // greedy tiles of whole rows
      uint32_t nt = 0, r = 0;
      trow[0] = 0;
      while (r < ng) {
        uint32_t e = r + 1;
        while (e < ng && ep_s[e + 1] - ep_s[r] <= kTileE && rp_s[e + 1] - rp_s[r] <= kTileS) ++e;
        trow[++nt] = e;
        r = e;
      }
      trow[kTileRows + 1] = nt;
      for (uint32_t t = 0; t < 2 && t < nt; ++t) issue(trow[t], trow[t + 1], issued++);
    }
    if (!staged_x) {  // x is the only input produced by an earlier grid
      pdl_wait();
      const int kv = static_cast<int>(min64(a.k, kSmemValues));
      for (int i = tid; i < kv; i += kTileNT) wv[i] = static_cast<float>(__ldg(a.omega + i) - a.bg);
      const int64_t n4 = a.n >> 2;
      if ((reinterpret_cast<uintptr_t>(x) & 15) == 0) {
        const float4 *x4 = reinterpret_cast<const float4 *>(x);
        float4 *xs4 = reinterpret_cast<float4 *>(xs);
        for (int64_t i = tid; i < n4; i += kTileNT) xs4[i] = __ldg(x4 + i);
        for (int64_t i = (n4 << 2) + tid; i < a.n; i += kTileNT) xs[i] = __ldg(x + i);
      } else {
        for (int64_t i = tid; i < a.n; i += kTileNT) xs[i] = __ldg(x + i);
      }
      y_empty = a.bg != 0.0 ? static_cast<float>(a.bg * a.colsum[0]) : 0.f;
      staged_x = true;
    }
    __syncthreads();
    const uint32_t nt = trow[kTileRows + 1];
    for (uint32_t t = 0; t < nt; ++t) {
      const uint32_t u = consumed++;
      const uint32_t ta = trow[t], tb = trow[t + 1];
      const uint32_t Sa = rp_s[ta], Ea = ep_s[ta], Eb = ep_s[tb];
      mbar_wait(&bar[u & 1u], (u >> 1) & 1u);
      const unsigned char *st = smem + L.stage + (u & 1u) * L.stage_bytes;
      const uint32_t ebase = static_cast<uint32_t>(
          ((reinterpret_cast<uintptr_t>(col + Ea) & ~uintptr_t(15)) - reinterpret_cast<uintptr_t>(col)) / sizeof(ColT));
      const uint32_t sbase = static_cast<uint32_t>(
          ((reinterpret_cast<uintptr_t>(op + Sa) & ~uintptr_t(15)) - reinterpret_cast<uintptr_t>(op)) / sizeof(PtrT));
      const uint32_t ibase = CSER ? static_cast<uint32_t>(((reinterpret_cast<uintptr_t>(oi + static_cast<size_t>(Sa) * oib) &
                                                             ~uintptr_t(15)) - reinterpret_cast<uintptr_t>(oi)) / oib)
                                  : 0u;
      const ColT *cst = reinterpret_cast<const ColT *>(st + L.col_off);
      const PtrT *ost = reinterpret_cast<const PtrT *>(st + L.op_off);
      const unsigned char *ist = st + L.oi_off;
      // ---- (A) gather + per-thread prefix of this thread's 16 aligned entry slots
      float run = 0.f;
      {
        const uint32_t q0 = tid * kTileEPT;  // aligned-relative slot
        const uint32_t g0e = ebase + q0;      // global entry of slot q0
        if (g0e < Eb) {
          float o[kTileEPT];
#pragma unroll
          for (int v = 0; v < NVT; ++v) {
            uint32_t c[CV::kPer];
            CV::unpack(reinterpret_cast<const uint4 *>(cst)[tid * NVT + v], c);
#pragma unroll
            for (int i = 0; i < CV::kPer; ++i) {
              const uint32_t ge = g0e + v * CV::kPer + i;
              float g = 0.f;
              if (ge >= Ea && ge < Eb) g = xs[c[i]];
              run += g;
              o[v * CV::kPer + i] = run;
            }
          }
#pragma unroll
          for (int q = 0; q < kTileEPT / 4; ++q)
            *reinterpret_cast<float4 *>(pre + q * (kTileNT * 4) + tid * 4) =
                make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        }
      }
      // ---- (B) block scan of thread totals
      float incl = run;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const float v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
      }
      tinc[tid] = incl;
      tex[tid] = incl - run;
      if (lane == 31) winc[wid] = incl;  // warp total
      __syncthreads();
      if (wid == 0) {
        const float wt = lane < kTileWarps ? winc[lane] : 0.f;
        float wi = wt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const float v = __shfl_up_sync(0xffffffffu, wi, d);
          if (lane >= d) wi += v;
        }
        if (lane < kTileWarps) wex[lane] = wi - wt;
      }
      __syncthreads();
      // sum of aligned slots [lo, hi), lo < hi
      auto range_sum = [&](uint32_t lo, uint32_t hi) -> float {
        const uint32_t tl = lo / kTileEPT, th = (hi - 1) / kTileEPT;
        const float pl = (lo % kTileEPT) ? pre[tpos(lo - 1)] : 0.f;
        const float ph = pre[tpos(hi - 1)];
        if (tl == th) return ph - pl;
        const float tl_tot = tinc[tl] - tex[tl];
        const uint32_t wl = tl >> 5, wh = th >> 5;
        if (wl == wh) return ((tl_tot - pl) + (tex[th] - tinc[tl])) + ph;
        const float mid = (wl + 1 < wh) ? (wex[wh] - wex[wl + 1]) : 0.f;  // whole warps in between
        return (((tl_tot - pl) + (winc[wl] - tinc[tl])) + mid + tex[th]) + ph;
      };
      // ---- (C) warp per row: one lane per segment, one fma per segment
      for (uint32_t r = ta + wid; r < tb; r += kTileWarps) {
        const uint32_t s0 = rp_s[r], s1 = rp_s[r + 1];
        float acc = 0.f;
        for (uint32_t s = s0 + lane; s < s1; s += 32) {
          const uint32_t stt = ost[s - sbase], enn = ost[s + 1 - sbase];
          if (enn > stt) {
            int k;
            if (CSER) {
              const uint32_t ii = s - ibase;
              k = oib == 1 ? ist[ii] : (oib == 2 ? reinterpret_cast<const uint16_t *>(ist)[ii]
                                                  : static_cast<int>(reinterpret_cast<const uint32_t *>(ist)[ii]));
            } else {
              k = static_cast<int>(s - s0 + 1);
            }
            acc = fmaf(wv[k], range_sum(stt - ebase, enn - ebase), acc);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0)
          put_y(a, y, g0 + r, s1 > s0 ? (a.bg != 0.0 ? static_cast<float>(static_cast<double>(acc) + a.bg * a.colsum[0]) : acc)
                              : y_empty);
      }
      __syncthreads();  // stage (u % 2), the prefix table and scans are free again
      if (tid == 0 && t + 2 < nt) issue(trow[t + 2], trow[t + 3], issued++);
    }
  }
}

template <typename ColT, typename PtrT, bool CSER>
int launch_matvec_tile(const DotArgs &a, const float *x, float *y, cudaStream_t st) {
  const TileSmem L = tile_layout(a.k, a.n, sizeof(ColT), sizeof(PtrT), CSER ? a.oi_bits / 8 : 1);
  auto kern = k_matvec_tile<ColT, PtrT, CSER>;
  if (int rc_ = allow_max_smem(kern)) return rc_;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(num_sms(), a.m)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTileNT);
  cfg.dynamicSmemBytes = L.total;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CERDOT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, a, x, y));
  return CERDOT_OK;
}

// ---------------------------------------------------------------------------------------------------
// Mat-vec for long rows (k_matvec_run): 32 warps per SM, 256-entry windows.
//
// The window kernel above holds a 1024-entry window per warp (32 colI registers per lane, a 4 KB prefix
// table per warp), which caps it at 16 warps and 128 registers when x is large -- on the 32768^2 layer
// (x = 128 KB) ncu shows it latency-bound: 0.31 issued warps per scheduler, 40% of the shared-memory
// pipe.  This kernel keeps the same arithmetic (window-local fp32 prefix differences, one fma per
// segment) with a quarter of the state, so a CTA runs 1024 threads at <= 64 registers:
//   * lane l owns entries [wb + 8l, wb + 8l + 8) of the window: one 16 B colI load (u16), the next
//     window's load in flight; 8 gathers from the x copy in shared memory; an in-lane running sum,
//     lane offsets by a 5-step warp scan; the window prefix G stored to a 1 KB per-warp table;
//   * segments are held lane-parallel, 32 at a time (lane j: segment sb + j, its start, end and value);
//     all segments that close inside the window are finished in one pass: sum = G(end) - G(start - 1),
//     or carry + G(end) for the segment open at the window start; the next 32 bounds are prefetched;
//   * per-lane fp32 accumulators, one xor butterfly per row.
// Rows are split evenly over all warps of the grid (one CTA per SM).
constexpr int kRunNT = 1024;
constexpr uint32_t kRunWin = 256;
constexpr uint32_t kRunRingBytes = 2048;  // per warp: colI windows in flight (4 x 512 B for u16)

template <typename ColT>
struct RunRing {
  static constexpr uint32_t kSlot = kRunWin * sizeof(ColT);     // bytes per window
  static constexpr uint32_t kDepth = kRunRingBytes / kSlot;      // windows in flight (8 / 4 / 2)
  static constexpr uint32_t kAlign = 16 / sizeof(ColT);           // window starts are 16 B aligned
  static constexpr uint32_t kLane = 8 * sizeof(ColT);             // bytes per lane per window
};

// async copy of one lane's colI bytes into its ring slot; bytes past the warp's range are zero-filled
template <uint32_t N>
__device__ __forceinline__ void cp_async_lane(void *dst, const void *src, uint32_t valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  if (N == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid) : "memory");
}

struct RunSmem {
  uint32_t bar, wv, pre, ring, xs, total;
};
__host__ __device__ __forceinline__ RunSmem run_layout(int64_t k, int64_t n, uint32_t warps, uint32_t depth) {
  RunSmem L{};
  uint32_t o = 0;
  auto take = [&](uint32_t bytes) {
    const uint32_t r = o;
    o += (bytes + 15u) & ~15u;
    return r;
  };
  (void)depth;
  L.bar = take(16u);  // x barrier
  L.wv = take(static_cast<uint32_t>(k) * 4u);
  L.pre = take(warps * kRunWin * 4u);
  L.ring = take(warps * kRunRingBytes);
  L.xs = take(static_cast<uint32_t>(n) * 4u);
  L.total = o;
  return L;
}

// a lane's 8 column indices of the window held in the ring slot
template <typename ColT>
__device__ __forceinline__ void ring_cols8(const unsigned char *slot, int lane, uint32_t c[8]);
template <>
__device__ __forceinline__ void ring_cols8<uint8_t>(const unsigned char *slot, int lane, uint32_t c[8]) {
  const uint2 v = *reinterpret_cast<const uint2 *>(slot + 8 * lane);
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    c[b] = (v.x >> (8 * b)) & 0xffu;
    c[4 + b] = (v.y >> (8 * b)) & 0xffu;
  }
}
template <>
__device__ __forceinline__ void ring_cols8<uint16_t>(const unsigned char *slot, int lane, uint32_t c[8]) {
  ColVec<uint16_t>::unpack(*reinterpret_cast<const uint4 *>(slot + 16 * lane), c);
}
template <>
__device__ __forceinline__ void ring_cols8<uint32_t>(const unsigned char *slot, int lane, uint32_t c[8]) {
  const uint4 v0 = *reinterpret_cast<const uint4 *>(slot + 32 * lane);
  const uint4 v1 = *reinterpret_cast<const uint4 *>(slot + 32 * lane + 16);
  c[0] = v0.x; c[1] = v0.y; c[2] = v0.z; c[3] = v0.w;
  c[4] = v1.x; c[5] = v1.y; c[6] = v1.z; c[7] = v1.w;
}

template <typename ColT, typename PtrT, bool CSER>
__global__ void __launch_bounds__(kRunNT, 1) k_matvec_run(DotArgs a, const float *__restrict__ x,
                                                          float *__restrict__ y) {
  using RR = RunRing<ColT>;
  constexpr int kWarps = kRunNT / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  const RunSmem L = run_layout(a.k, a.n, kWarps, RR::kDepth);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float *wv = reinterpret_cast<float *>(smem + L.wv);
  float *pre = reinterpret_cast<float *>(smem + L.pre) + wid * kRunWin;
  unsigned char *ring = smem + L.ring + wid * kRunRingBytes;
  float *xs = reinterpret_cast<float *>(smem + L.xs);
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
  for (int i = threadIdx.x; i < a.k; i += kRunNT) wv[i] = static_cast<float>(__ldg(a.omega + i) - a.bg);

  // row entry bounds E(r), 32 rows per lane-parallel group (separate groups for producer and consumer)
  auto row_e = [&](uint32_t r) -> uint32_t {
    return a.re ? __ldg(a.re + r) : ld_idx(op, load_index(a.rp, a.rp_bits, r));
  };
  const uint32_t e_end = R0 < R1 ? row_e(R1) : 0u;  // end of this warp's colI range
  uint32_t pg = R0, pgE = (R0 + lane <= R1 && R0 < R1) ? row_e(R0 + lane) : 0u;
  uint32_t cg = pg, cgE = pgE;
  auto group_e = [&](uint32_t r, uint32_t &g, uint32_t &gE) -> uint32_t {  // E(r), r in [R0, R1]
    if (r - g >= 32u) {
      g = r;
      gE = (r + lane <= R1) ? row_e(r + lane) : 0u;
    }
    return __shfl_sync(0xffffffffu, gE, static_cast<int>(r - g));
  };

  // colI producer: windows of every non-empty row of the warp in order, kDepth in flight; each lane
  // copies (cp.async) and later reads back only its own bytes, so no cross-lane synchronisation
  uint32_t pr = R0, pwb = 0, pe1 = 0, pk = 0;
  bool pdone = R0 >= R1;
  auto prod_row = [&]() {  // position the producer at the first window of row pr (skipping empty rows)
    while (pr < R1) {
      const uint32_t e0 = group_e(pr, pg, pgE), e1 = group_e(pr + 1, pg, pgE);
      if (e1 > e0) {
        pwb = e0 & ~(RR::kAlign - 1u);
        pe1 = e1;
        return;
      }
      ++pr;
    }
    pdone = true;
  };
  const uint32_t e_lim = (e_end + RR::kAlign - 1u) & ~(RR::kAlign - 1u);  // readable (16 B rounded)
  auto produce = [&]() {
    if (!pdone) {
      const uint32_t slot = pk % RR::kDepth, pos = pwb + 8u * lane;
      const uint32_t valid = pos < e_lim ? RR::kLane : 0u;
      unsigned char *dst = ring + slot * RR::kSlot + lane * RR::kLane;
      const ColT *src = col + (pos < e_lim ? pos : pwb);
      if (RR::kLane == 32) {
        cp_async_lane<16>(dst, src, valid);
        cp_async_lane<16>(dst + 16, src + 4, valid);
      } else {
        cp_async_lane<RR::kLane>(dst, src, valid);
      }
    }
    cp_async_commit();  // one group per window (empty past the end) keeps wait_group counting exact
    if (pdone) return;
    ++pk;
    pwb += kRunWin;
    if (pwb >= pe1) {
      ++pr;
      prod_row();
    }
  };
  if (!pdone) prod_row();
  for (uint32_t d = 0; d < RR::kDepth; ++d) produce();
  uint32_t ck = 0;  // windows consumed
  __syncthreads();  // value table (x is waited on per warp below)
  bool x_ready = false;

  for (uint32_t r = R0; r < R1; ++r) {
    const uint32_t e0 = group_e(r, cg, cgE), e1 = group_e(r + 1, cg, cgE);
    float acc = 0.f;
    if (e1 > e0) {
      const uint32_t s0 = load_index(a.rp, a.rp_bits, r), s1 = load_index(a.rp, a.rp_bits, r + 1);
      // segment batch: lane j holds segment sb + j (start st, end en, value v); invalid lanes never close
      uint32_t sb = s0, st, en, nst, nen, nk;
      auto fetch = [&](uint32_t b, uint32_t &fst, uint32_t &fen, uint32_t &fk) {
        const uint32_t s = b + lane;
        fst = s < s1 ? ld_idx(op, s) : 0xffffffffu;
        fen = s < s1 ? ld_idx(op, s + 1) : 0xffffffffu;
        fk = s < s1 ? (CSER ? load_index(a.oi, a.oi_bits, s) : s - s0 + 1) : 0u;
      };
      uint32_t k0;
      fetch(sb, st, en, k0);
      fetch(sb + 32, nst, nen, nk);
      if (!x_ready) {
        mbar_wait(xbar, 0);
        x_ready = true;
      }
      float v = wv[k0];
      uint32_t jdone = 0;
      float carry = 0.f;
      for (uint32_t wb = e0 & ~(RR::kAlign - 1u); wb < e1; wb += kRunWin) {
        const uint32_t slot = ck % RR::kDepth;
        cp_async_wait<RR::kDepth - 1>();
        uint32_t c[8];
        ring_cols8<ColT>(ring + slot * RR::kSlot, lane, c);
        ++ck;
        produce();
        // gather + in-lane running sum (entries outside [e0, e1) count as 0)
        const uint32_t p0 = wb + 8 * lane;
        float g[8], run = 0.f;
        if (p0 >= e0 && p0 + 8 <= e1) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            run += xs[c[i]];
            g[i] = run;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t p = p0 + i;
            if (p >= e0 && p < e1) run += xs[c[i]];
            g[i] = run;
          }
        }
        float incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const float off = incl - run;
#pragma unroll
        for (int i = 0; i < 8; ++i) g[i] += off;
        *reinterpret_cast<float4 *>(pre + lane * 8) = make_float4(g[0], g[1], g[2], g[3]);
        *reinterpret_cast<float4 *>(pre + lane * 8 + 4) = make_float4(g[4], g[5], g[6], g[7]);
        const float T = __shfl_sync(0xffffffffu, g[7], 31);  // window total, as stored at slot 255
        __syncwarp();
        // segments closing in this window (one pass per batch of 32)
        const uint32_t wend = wb + kRunWin;
        bool any = false;
        float glast = 0.f;
        while (true) {
          const uint32_t closed = __ballot_sync(0xffffffffu, en <= wend);
          const int cnt = __popc(closed);
          const bool mine = lane >= static_cast<int>(jdone) && lane < cnt && en > st;
          float ge = 0.f;
          if (mine) {
            ge = pre[en - 1 - wb];
            const float gs = st > wb ? pre[st - 1 - wb] : -carry;
            acc = fmaf(v, ge - gs, acc);
          }
          const uint32_t hit = __ballot_sync(0xffffffffu, mine);
          const float gl = __shfl_sync(0xffffffffu, ge, 31 - __clz(hit | 1u));
          if (hit) {
            glast = gl;
            any = true;
          }
          if (cnt == 32 && sb + 32 < s1) {  // batch exhausted inside this window: next 32 segments
            sb += 32;
            st = nst;
            en = nen;
            v = wv[nk];
            fetch(sb + 32, nst, nen, nk);
            jdone = 0;
            continue;
          }
          jdone = static_cast<uint32_t>(cnt);
          break;
        }
        carry = any ? T - glast : carry + T;
        __syncwarp();  // the prefix table is rewritten by the next window
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) put_y(a, y, r, a.bg != 0.0 ? static_cast<float>(static_cast<double>(acc) + a.bg * a.colsum[0]) : acc);
  }
  if (!x_ready) mbar_wait(xbar, 0);  // no CTA exits with a bulk copy in flight
  cp_async_wait<0>();
}

template <typename ColT, typename PtrT, bool CSER>
int launch_matvec_run(const DotArgs &a, const float *x, float *y, cudaStream_t st) {
  const size_t smem = run_layout(a.k, a.n, kRunNT / 32, RunRing<ColT>::kDepth).total;
  auto kern = k_matvec_run<ColT, PtrT, CSER>;
  if (int rc_ = allow_max_smem(kern)) return rc_;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(num_sms(), ceil_div(a.m, kRunNT / 32))));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kRunNT);
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

// Generic mat-vec for alphabets beyond the u16 slot table: warp per row, lanes over segments.
template <typename ColT, typename PtrT, bool CSER>
__global__ void __launch_bounds__(256) k_matvec_generic(DotArgs a, const float *__restrict__ x,
                                                        float *__restrict__ y) {
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
        const int64_t k = CSER ? static_cast<int64_t>(load_index(a.oi, a.oi_bits, s)) : (s - s0 + 1);
        acc = fmaf(static_cast<float>(__ldg(a.omega + k) - a.bg), sum, acc);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) put_y(a, y, row, a.bg != 0.0 ? static_cast<float>(static_cast<double>(acc) + a.bg * a.colsum[0]) : acc);
  }
}

template <int V>
struct XVec {
  float v[V];
};

template <int V>
__device__ __forceinline__ XVec<V> ld_x(const float *p, int64_t cb, int64_t batch) {
  XVec<V> r;
  if (V == 4 && cb + 4 <= batch) {
    const float4 t = __ldg(reinterpret_cast<const float4 *>(p));
    r.v[0] = t.x; r.v[1] = t.y; r.v[2] = t.z; r.v[V - 1] = t.w;
  } else if (V == 2 && cb + 2 <= batch) {
    const float2 t = __ldg(reinterpret_cast<const float2 *>(p));
    r.v[0] = t.x; r.v[V - 1] = t.y;
  } else {
#pragma unroll
    for (int j = 0; j < V; ++j) r.v[j] = (cb + j < batch) ? __ldg(p + j) : 0.f;
  }
  return r;
}

// Mat-mat: warp per (row, 32*V batch columns).  The row's colI entries are walked as one
// contiguous stream (32-entry chunks loaded lane-parallel, the next chunk prefetched); segments are
// iterated at warp level (bounds and omegaI loaded 32 at a time), so an entry costs one shuffle, one
// V-wide vector load of its X row and V adds, eight loads in flight; one fma per segment per column.
template <typename ColT, typename PtrT, bool CSER, int V>
__global__ void __launch_bounds__(256, (V == 4 ? 4 : 1)) k_matmat(DotArgs a, const float *__restrict__ x, int64_t ldx, int64_t batch,
                                                float *__restrict__ y, int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const ColT *col = static_cast<const ColT *>(a.col);
  const PtrT *op = static_cast<const PtrT *>(a.op);
  const int64_t chunks = ceil_div(batch, 32 * V);
  const int64_t units = a.m * chunks;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < units; u += nwarps) {
    const int64_t row = u / chunks, cb = (u - row * chunks) * 32 * V + lane * V;
    const uint32_t s0 = load_index(a.rp, a.rp_bits, row), s1 = load_index(a.rp, a.rp_bits, row + 1);
    float acc[V];
#pragma unroll
    for (int q = 0; q < V; ++q) acc[q] = 0.f;
    if (s1 > s0) {
      const float *xb = x + cb;                       // this lane's columns
      const bool full = cb + V <= batch;              // lanes past the batch end take the guarded path
      const int nval = static_cast<int>(max64(0, min64(V, batch - cb)));
      const uint32_t ldx32 = static_cast<uint32_t>(ldx);
      const uint32_t e0 = ld_idx(op, s0), e1 = ld_idx(op, s1);
      // colI stream: cur holds entries [ch, ch + 32), nxt the following 32
      uint32_t ch = e0;
      uint32_t cur = (ch + lane < e1) ? ld_idx(col, ch + lane) : 0u;
      uint32_t nxt = (ch + 32 + lane < e1) ? ld_idx(col, ch + 32 + lane) : 0u;
      for (uint32_t sb = s0; sb < s1; sb += 32) {
        // bounds / element of segments sb .. sb+31 (lane l: segment sb + l)
        const uint32_t my_s = sb + lane;
        const uint32_t my_st = my_s < s1 ? ld_idx(op, my_s) : 0u;
        const uint32_t my_en = my_s < s1 ? ld_idx(op, my_s + 1) : 0u;
        int my_k = 0;
        if (my_s < s1) my_k = CSER ? static_cast<int>(load_index(a.oi, a.oi_bits, my_s)) : static_cast<int>(my_s - s0 + 1);
        const float my_v = my_s < s1 ? static_cast<float>(__ldg(a.omega + my_k) - a.bg) : 0.f;
        const int nseg = static_cast<int>(min64(32, s1 - sb));
        for (int t = 0; t < nseg; ++t) {
          uint32_t e = __shfl_sync(0xffffffffu, my_st, t);
          const uint32_t en = __shfl_sync(0xffffffffu, my_en, t);
          if (en <= e) continue;
          float sum[V];
#pragma unroll
          for (int q = 0; q < V; ++q) sum[q] = 0.f;
          while (e < en) {
            uint32_t j = e - ch;
            if (j >= 32u) {  // advance the colI stream
              ch += 32;
              cur = nxt;
              nxt = (ch + 32 + lane < e1) ? ld_idx(col, ch + 32 + lane) : 0u;
              continue;
            }
            const uint32_t here = min(en - e, 32u - j);
            for (uint32_t t0 = 0; t0 < here; t0 += 8) {
              XVec<V> xv[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const uint32_t c = __shfl_sync(0xffffffffu, cur, (j + t0 + i) & 31u);
                if (t0 + i < here) {
                  const float *p = xb + static_cast<size_t>(c) * ldx32;
                  if (full) {
                    if (V == 4) {
                      const float4 t4 = __ldg(reinterpret_cast<const float4 *>(p));
                      xv[i].v[0] = t4.x; xv[i].v[1] = t4.y; xv[i].v[2] = t4.z; xv[i].v[V - 1] = t4.w;
                    } else if (V == 2) {
                      const float2 t2 = __ldg(reinterpret_cast<const float2 *>(p));
                      xv[i].v[0] = t2.x; xv[i].v[V - 1] = t2.y;
                    } else {
                      xv[i].v[0] = __ldg(p);
                    }
                  } else {
#pragma unroll
                    for (int q = 0; q < V; ++q) xv[i].v[q] = q < nval ? __ldg(p + q) : 0.f;
                  }
                }
              }
#pragma unroll
              for (int i = 0; i < 8; ++i)
                if (t0 + i < here) {
#pragma unroll
                  for (int q = 0; q < V; ++q) sum[q] += xv[i].v[q];
                }
            }
            e += here;
          }
          const float v = __shfl_sync(0xffffffffu, my_v, t);
#pragma unroll
          for (int q = 0; q < V; ++q) acc[q] = fmaf(v, sum[q], acc[q]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int64_t c = cb + q;
      if (c < batch)
        put_y(a, y, row * ldy + c,
              a.bg != 0.0 ? static_cast<float>(static_cast<double>(acc[q]) + a.bg * a.colsum[c]) : acc[q]);
    }
  }
}

// Mat-mat, flat entry stream (k_matmat_flat): warp per (row, 32*V batch columns), as k_matmat, but the
// row's entries are walked 32 at a time without regard to segment boundaries: the 32 column indices of
// a chunk sit one per lane, the segments ending inside the chunk are turned into a 32-bit mask
// (redux.or over the lane-parallel segment bounds) and their values into a per-warp 32-slot table, so
// each entry costs one shuffle, one V-wide X-row load, V adds and a bit test, with eight loads in flight.
// ncu on k_matmat (AlexNet fc6, B = 64): 44 instructions per entry, issue-bound; this walk is ~10.
// Per column the arithmetic is k_matmat's exactly (sequential fp32 segment sums in colI order, one
// fma per non-empty segment): the two kernels agree bitwise.
template <int V>
__device__ __forceinline__ void ld_xrow(const float *p, bool full, int nval, float *out) {
  if (full) {
    if (V == 4) {
      const float4 t = __ldg(reinterpret_cast<const float4 *>(p));
      out[0] = t.x; out[1 % V] = t.y; out[2 % V] = t.z; out[3 % V] = t.w;
    } else if (V == 2) {
      const float2 t = __ldg(reinterpret_cast<const float2 *>(p));
      out[0] = t.x; out[1 % V] = t.y;
    } else {
      out[0] = __ldg(p);
    }
  } else {
#pragma unroll
    for (int q = 0; q < V; ++q) out[q] = q < nval ? __ldg(p + q) : 0.f;
  }
}

template <typename ColT, typename PtrT, bool CSER, int V, int D>
__global__ void __launch_bounds__(256) k_matmat_flat(DotArgs a, const float *__restrict__ x,
                                                                      int64_t ldx, int64_t batch,
                                                                      float *__restrict__ y, int64_t ldy) {
  __shared__ float vtab_all[8][32];
  __shared__ uint32_t cbuf_all[8][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float *vtab = vtab_all[wid];
  const uint32_t *cbuf = cbuf_all[wid];
  const ColT *col = static_cast<const ColT *>(a.col);
  const PtrT *op = static_cast<const PtrT *>(a.op);
  const int64_t chunks = ceil_div(batch, 32 * V);
  const int64_t units = a.m * chunks;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < units; u += nwarps) {
    const int64_t row = u / chunks, cb = (u - row * chunks) * 32 * V + lane * V;
    const uint32_t s0 = load_index(a.rp, a.rp_bits, row), s1 = load_index(a.rp, a.rp_bits, row + 1);
    float acc[V];
#pragma unroll
    for (int q = 0; q < V; ++q) acc[q] = 0.f;
    if (s1 > s0) {
      const float *xb = x + cb;
      const bool full = cb + V <= batch;
      const bool all_full = __all_sync(0xffffffffu, full);  // no per-load guard (B a multiple of 32 V)
      const int nval = static_cast<int>(max64(0, min64(V, batch - cb)));
      const uint32_t ldx_b = static_cast<uint32_t>(ldx) * 4u;  // X row stride in bytes
      // X row c of this lane's columns: one IMAD.WIDE from a 32-bit index
      auto xrow = [&](uint32_t c) {
        return reinterpret_cast<const float *>(reinterpret_cast<const char *>(xb) + static_cast<uint64_t>(c) * ldx_b);
      };
      const uint32_t e0 = a.re ? __ldg(a.re + row) : ld_idx(op, s0);
      const uint32_t e1 = a.re ? __ldg(a.re + row + 1) : ld_idx(op, s1);
      // segment batch (lane j: segment sb + j) with the next batch prefetched
      auto fetch = [&](uint32_t b, uint32_t &fst, uint32_t &fen, float &fv) {
        const uint32_t s = b + lane;
        fst = s < s1 ? ld_idx(op, s) : 0xffffffffu;
        fen = s < s1 ? ld_idx(op, s + 1) : 0xffffffffu;
        fv = 0.f;
        if (s < s1) {
          const uint32_t k = CSER ? load_index(a.oi, a.oi_bits, s) : s - s0 + 1;
          fv = static_cast<float>(__ldg(a.omega + k) - a.bg);
        }
      };
      uint32_t sb = s0, st, en, nst, nen;
      float v, nv;
      fetch(sb, st, en, v);
      fetch(sb + 32, nst, nen, nv);
      float s[V];
#pragma unroll
      for (int q = 0; q < V; ++q) s[q] = 0.f;
      uint32_t cur = (e0 + lane < e1) ? ld_idx(col, e0 + lane) : 0u;
      for (uint32_t ch = e0; ch < e1; ch += 32) {
        const uint32_t nxt = (ch + 32 + lane < e1) ? ld_idx(col, ch + 32 + lane) : 0u;
        const uint32_t cend = min(ch + 32, e1);
        // segments ending in [ch, cend): mask of their last entries, values into vtab
        uint32_t mask = 0;
        while (true) {
          const bool ends_here = en > st && en - 1 >= ch && en - 1 < cend;
          if (ends_here) vtab[en - 1 - ch] = v;
          mask |= __reduce_or_sync(0xffffffffu, ends_here ? 1u << (en - 1 - ch) : 0u);
          // batch exhausted before the chunk end: next 32 segments (their ends may fall in this chunk)
          const bool need = __shfl_sync(0xffffffffu, en, 31) < cend && sb + 32 < s1;
          if (!need) break;
          sb += 32;
          st = nst;
          en = nen;
          v = nv;
          fetch(sb + 32, nst, nen, nv);
        }
        cbuf_all[wid][lane] = cur;  // the chunk's column indices, read back as broadcasts
        __syncwarp();
        const uint32_t cnt = cend - ch;
        // D X-row loads in flight
        if (cnt == 32) {
#pragma unroll
          for (int i0 = 0; i0 < 32; i0 += D) {
            float xv[D][V];
            if (all_full) {
#pragma unroll
              for (int i = 0; i < D; ++i) ld_xrow<V>(xrow(cbuf[i0 + i]), true, V, xv[i]);
            } else {
#pragma unroll
              for (int i = 0; i < D; ++i) ld_xrow<V>(xrow(cbuf[i0 + i]), full, nval, xv[i]);
            }
#pragma unroll
            for (int i = 0; i < D; ++i) {
#pragma unroll
              for (int q = 0; q < V; ++q) s[q] += xv[i][q];
              if ((mask >> (i0 + i)) & 1u) {
                const float vv = vtab[i0 + i];
#pragma unroll
                for (int q = 0; q < V; ++q) {
                  acc[q] = fmaf(vv, s[q], acc[q]);
                  s[q] = 0.f;
                }
              }
            }
          }
        } else {  // the row's last, partial chunk
          for (uint32_t i0 = 0; i0 < cnt; i0 += D) {
            float xv[D][V];
#pragma unroll
            for (int i = 0; i < D; ++i)
              if (i0 + i < cnt) ld_xrow<V>(xrow(cbuf[(i0 + i) & 31u]), full, nval, xv[i]);
#pragma unroll
            for (int i = 0; i < D; ++i) {
              if (i0 + i < cnt) {
#pragma unroll
                for (int q = 0; q < V; ++q) s[q] += xv[i][q];
                if ((mask >> (i0 + i)) & 1u) {
                  const float vv = vtab[i0 + i];
#pragma unroll
                  for (int q = 0; q < V; ++q) {
                    acc[q] = fmaf(vv, s[q], acc[q]);
                    s[q] = 0.f;
                  }
                }
              }
            }
          }
        }
        __syncwarp();  // vtab and cbuf are rewritten for the next chunk
        cur = nxt;
      }
    }
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int64_t c = cb + q;
      if (c < batch)
        put_y(a, y, row * ldy + c,
              a.bg != 0.0 ? static_cast<float>(static_cast<double>(acc[q]) + a.bg * a.colsum[c]) : acc[q]);
    }
  }
}

// Column sums of x (n x batch, row stride ldx) in fp64, fixed reduction order, in two passes:
// k_colsum_part sums row range s (of kColsumSplit) of 32 columns per CTA (8 strided partials in flight,
// combined in order), k_colsum_fin adds the kColsumSplit partials in order.  (One CTA per 32 columns
// was 49 CTAs for the ResNet conv layer at B = 1568: ~0.1 ms of a ~0.9 ms call with X cold.)
constexpr int kColsumSplit = 16;

__global__ void __launch_bounds__(256) k_colsum_part(const float *__restrict__ x, int64_t n, int64_t ldx,
                                                     int64_t batch, double *__restrict__ part_out) {
  __shared__ double part[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * 32 + tx;
  const int64_t r0 = blockIdx.y * n / kColsumSplit, r1 = (blockIdx.y + 1) * n / kColsumSplit;
  double s = 0.0;
  if (c < batch) {
    constexpr int kU = 16;
    int64_t r = r0 + ty;
    for (; r + 8 * (kU - 1) < r1; r += 8 * kU) {
      float v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = __ldg(x + (r + 8 * u) * ldx + c);
#pragma unroll
      for (int u = 0; u < kU; ++u) s += static_cast<double>(v[u]);
    }
    for (; r < r1; r += 8) s += static_cast<double>(__ldg(x + r * ldx + c));
  }
  part[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && c < batch) {
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += part[j][tx];
    part_out[blockIdx.y * batch + c] = t;
  }
}

__global__ void __launch_bounds__(256) k_colsum_fin(const double *__restrict__ part, int64_t batch,
                                                    double *__restrict__ out) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= batch) return;
  double t = 0.0;
#pragma unroll
  for (int s = 0; s < kColsumSplit; ++s) t += part[s * batch + c];
  out[c] = t;
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

size_t matvec_smem(int64_t k, int64_t n, bool xsmem, uint32_t warps, uint32_t depth, uint32_t oib) {
  return matvec_layout(k, xsmem ? n : 0, warps, depth, oib).total;
}

template <typename ColT, typename PtrT, bool CSER, bool XSMEM, int NT, int NBUF, int MINB, int D>
int launch_matvec(const DotArgs &a, const float *x, float *y, cudaStream_t st) {
  const uint32_t oib = CSER ? static_cast<uint32_t>(a.oi_bits / 8) : 1u;
  const size_t smem = matvec_smem(a.k, a.n, XSMEM, NT / 32, D, oib);
  auto kern = k_matvec<ColT, PtrT, CSER, XSMEM, NT, NBUF, MINB, D>;
  if (int rc_ = allow_max_smem(kern)) return rc_;
  // every SM gets a CTA; rows are split fractionally over all warps (R0 = gw*m/warps)
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(num_sms(), a.m)));
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
int launch_dot(const DotArgs &a, const float *x, int64_t ldx, int64_t batch, float *y, int64_t ldy, cudaStream_t st) {
  if (batch == 1 && (a.m >= (int64_t(1) << 31) || a.k > kSmemValues)) {
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(a.m, 8), int64_t(num_sms()) * 16)));
    k_matvec_generic<ColT, PtrT, CSER><<<grid, 256, 0, st>>>(a, x, y);
    CERDOT_LAUNCH_CHECK();
    return CERDOT_OK;
  }
  if (batch == 1) {
    // rows that fit a tile (known from the encoding's row statistics): CTA-tile TMA pipeline
    const int force_path = kernel_path(CERDOT_PATH_MATVEC);
    const bool tile_ok = a.max_row_nnz > 0 && a.max_row_nnz <= kTileE && a.max_row_segs <= kTileS &&
                         a.k <= kSmemValues &&
                         tile_layout(a.k, a.n, sizeof(ColT), sizeof(PtrT), CSER ? a.oi_bits / 8 : 1).total <=
                             static_cast<uint32_t>(kMaxSmemBytes);
    // measured on B200: the tile pipeline wins when there are fewer rows than warps in the window kernel
    // (ResNet conv 512 rows: 8.2 vs 13+ us); with >= 1 row per warp the window kernel wins (AlexNet, VGG)
    const bool few_rows = a.m < int64_t(num_sms()) * 16;
    // long rows (>= 4096 entries on average, the 32768^2 layer: 9829): the 32-warp run kernel
    // (431 -> 314 us there); at ~1000-entry rows (AlexNet, VGG fc6) the window kernel is 0-30% faster
    const bool long_rows = a.nnz >= int64_t(4096) * a.m;
    // one short row per warp (AlexNet fc6: 4096 rows of <= 1017 entries over 148 x 28 warps): the row kernel
    const bool short_rows = a.max_row_nnz > 0 && matvec_row_fits(a, sizeof(ColT));
    // (measured: AlexNet fc6 CER 7.26 -> 6.57 us, CSER 8.26 -> 6.91 us vs the window kernel; the 512 x 1024
    // oracle layer 3.21 us vs 3.49 us for the tile pipeline)
    const int want = force_path ? force_path : (short_rows ? 5 : (few_rows ? 2 : (long_rows ? 4 : 1)));
    if (want == 5 && short_rows) return matvec_row(a, CSER, 8 * sizeof(ColT), 8 * sizeof(PtrT), x, y, st);
    if (tile_ok && want == 2) return launch_matvec_tile<ColT, PtrT, CSER>(a, x, y, st);
    // the stream kernel (dot_stream.cu): colI through registers, fragment sums, no prefix table
    if (want == 4 && a.nnz < (int64_t(1) << 32) - 65536 && matvec_stream_fits(a.k, a.n, 8 * sizeof(PtrT), CSER ? a.oi_bits : 0))
      return matvec_stream(a, CSER, 8 * sizeof(ColT), 8 * sizeof(PtrT), x, y, st);
    if ((want == 3 || want == 4) && run_layout(a.k, a.n, kRunNT / 32, RunRing<ColT>::kDepth).total <= static_cast<uint32_t>(kMaxSmemBytes))
      return launch_matvec_run<ColT, PtrT, CSER>(a, x, y, st);
    // Prefer the co-resident variant (16 warps, <= 64 regs, <= half the SM's shared memory): two
    // consecutive calls' CTAs then share an SM and, with programmatic dependent launch, the next call's
    // index prologue (rowPtr -> omegaPtr -> colI latency chain) overlaps this call's work.
    const uint32_t oib = CSER ? static_cast<uint32_t>(a.oi_bits / 8) : 1u;
    // (measured: AlexNet-fc6 12.5 us co-resident vs 10.6 us exclusive -- the post-wait chain dominates,
    // so the co-resident variant is opt-in: CERDOT_PATH_MATVEC_NT = 1)
    const int want_nt = kernel_path(CERDOT_PATH_MATVEC_NT);
    if (want_nt == 1 && matvec_smem(a.k, a.n, true, 16, 3, oib) <= kHalfSmemBytes)
      return launch_matvec<ColT, PtrT, CSER, true, 512, 1, 2, 3>(a, x, y, st);
    // 28 warps per SM (896 threads, <= 72 regs) when x and the per-warp tables fit: enough warps that
    // each holds at most one row of a 4096-row layer (a second row would run serially)
    const bool wide = (want_nt == 896 || want_nt == 0) && matvec_smem(a.k, a.n, true, 28, 4, oib) <= kMaxSmemBytes &&
                      a.m > int64_t(num_sms()) * 16;
    if (wide) return launch_matvec<ColT, PtrT, CSER, true, 896, 1, 1, 4>(a, x, y, st);
    // large x (VGG fc6: 100 KB): the same 28 warps with a 2-deep segment ring still fit
    const bool wide2 = (want_nt == 896 || want_nt == 0) && matvec_smem(a.k, a.n, true, 28, 2, oib) <= kMaxSmemBytes &&
                       a.m > int64_t(num_sms()) * 16;
    if (wide2) return launch_matvec<ColT, PtrT, CSER, true, 896, 1, 1, 2>(a, x, y, st);
    const bool xsmem = matvec_smem(a.k, a.n, true, 16, 4, oib) <= static_cast<size_t>(kMaxSmemBytes);
    // u32 colI windows are 32 registers each: one window buffer (three would spill)
    constexpr int kNbuf = sizeof(ColT) == 4 ? 1 : 3;
    return xsmem ? launch_matvec<ColT, PtrT, CSER, true, 512, kNbuf, 1, 4>(a, x, y, st)
                 : launch_matvec<ColT, PtrT, CSER, false, 512, kNbuf, 1, 4>(a, x, y, st);
  }
  const bool al4 = (ldx % 4 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0);
  const bool al2 = (ldx % 2 == 0) && (reinterpret_cast<uintptr_t>(x) % 8 == 0);
  const int V = (batch > 64 && al4) ? 4 : ((batch > 32 && al2) ? 2 : 1);
  const int64_t units = a.m * ceil_div(batch, 32 * V);
  if (kernel_path(CERDOT_PATH_MATMAT) != 2) {
    // flat entry stream (default); one resident wave of CTAs (occupancy API), units round-robin over warps
    auto go = [&](auto kern) -> int {
      int per_sm = 0;
      if (int rc_ = blocks_per_sm(kern, 256, &per_sm)) return rc_;
      const int grid = static_cast<int>(std::max<int64_t>(
          1, std::min<int64_t>(ceil_div(units, 8), int64_t(num_sms()) * std::max(per_sm, 1))));
      kern<<<grid, 256, 0, st>>>(a, x, ldx, batch, y, ldy);
      CERDOT_LAUNCH_CHECK();
      return CERDOT_OK;
    };
    // 8 X-row loads in flight for every V (measured: V = 4 at D = 4 runs 3 CTAs per SM instead of 2
    // but is slower on all of VGG fc6 B=128, ResNet conv B=1568 and 32768^2 B=256)
    // V = 2 at 16 loads in flight (AlexNet fc6 B=64: 97 -> 80 us); V = 1 stays at 8 (16 is 9% slower at
    // B=32).  CERDOT_PATH_MATMAT_DEPTH forces 8 / 16 for V <= 2 (A/B only).
    const int fd = kernel_path(CERDOT_PATH_MATMAT_DEPTH);
    if (V == 4) return go(k_matmat_flat<ColT, PtrT, CSER, 4, 8>);
    if (V == 2)
      return (fd ? fd : 16) == 16 ? go(k_matmat_flat<ColT, PtrT, CSER, 2, 16>)
                                        : go(k_matmat_flat<ColT, PtrT, CSER, 2, 8>);
    return (fd ? fd : 8) == 16 ? go(k_matmat_flat<ColT, PtrT, CSER, 1, 16>)
                                     : go(k_matmat_flat<ColT, PtrT, CSER, 1, 8>);
  }
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(units, 8),
                                                                           int64_t(num_sms()) * 8)));
  if (V == 4)
    k_matmat<ColT, PtrT, CSER, 4><<<grid, 256, 0, st>>>(a, x, ldx, batch, y, ldy);
  else if (V == 2)
    k_matmat<ColT, PtrT, CSER, 2><<<grid, 256, 0, st>>>(a, x, ldx, batch, y, ldy);
  else
    k_matmat<ColT, PtrT, CSER, 1><<<grid, 256, 0, st>>>(a, x, ldx, batch, y, ldy);
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

template <typename PtrT>
__global__ void __launch_bounds__(256) k_row_entries(const void *rp, int rp_bits, const PtrT *__restrict__ op,
                                                     int64_t m, uint32_t *__restrict__ out) {
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r <= m;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[r] = static_cast<uint32_t>(op[load_index(rp, rp_bits, r)]);
}

}  // namespace

int row_entries(const cerdot_matrix *mat, uint32_t *out, cudaStream_t st) {
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(mat->m + 1, 256), num_sms() * 8)));
  switch (mat->omega_ptr_bits) {
    case 8:
      k_row_entries<<<grid, 256, 0, st>>>(mat->row_ptr, mat->row_ptr_bits, static_cast<const uint8_t *>(mat->omega_ptr),
                                          mat->m, out);
      break;
    case 16:
      k_row_entries<<<grid, 256, 0, st>>>(mat->row_ptr, mat->row_ptr_bits,
                                          static_cast<const uint16_t *>(mat->omega_ptr), mat->m, out);
      break;
    default:
      k_row_entries<<<grid, 256, 0, st>>>(mat->row_ptr, mat->row_ptr_bits,
                                          static_cast<const uint32_t *>(mat->omega_ptr), mat->m, out);
  }
  CERDOT_LAUNCH_CHECK();
  return CERDOT_OK;
}

int dot(const cerdot_matrix *mat, const float *x, int64_t ldx, int64_t batch, float *y, int64_t ldy, void *workspace,
        size_t workspace_bytes, cudaStream_t st, float *const *peers, int npeers, int64_t peer_offset) {
  const bool cser = mat->kind == CERDOT_CSER;
  DotArgs a{};
  a.ypeer = peers;
  a.npeer = peers ? npeers : 0;
  a.ypeer_off = peer_offset;
  a.omega = mat->omega;
  a.col = mat->col_index;
  a.op = mat->omega_ptr;
  a.rp = mat->row_ptr;
  a.oi = mat->omega_index;
  a.rp_bits = mat->row_ptr_bits;
  a.oi_bits = mat->omega_index_bits;
  a.m = mat->m;
  a.n = mat->n;
  a.k = mat->k;
  a.mode = cser ? mat->mode_index : 0;
  a.bg = mat->background;
  a.segs = mat->segments;
  a.max_row_nnz = mat->max_row_nnz;
  a.nnz = mat->nnz;
  a.dbg = kernel_path(CERDOT_PATH_TRACE) ? 1 : 0;
  a.max_row_segs = mat->max_row_segments;
  a.re = mat->row_entry;
  if (a.m == 0 || batch == 0) return CERDOT_OK;
  if (a.bg != 0.0) {
    if (workspace == nullptr || workspace_bytes < sizeof(double) * static_cast<size_t>(batch))
      return fail(CERDOT_E_WORKSPACE, "dot workspace too small for the background column sums");
    double *cs = static_cast<double *>(workspace);
    if (batch == 1) {
      k_vecsum<<<1, 1024, 0, st>>>(x, a.n, cs);
    } else {
      if (workspace_bytes < sizeof(double) * static_cast<size_t>(batch) * (1 + kColsumSplit))
        return fail(CERDOT_E_WORKSPACE, "dot workspace too small for the background column sums");
      k_colsum_part<<<dim3(static_cast<unsigned>(ceil_div(batch, 32)), kColsumSplit), 256, 0, st>>>(
          x, a.n, ldx, batch, cs + batch);
      k_colsum_fin<<<static_cast<unsigned>(ceil_div(batch, 256)), 256, 0, st>>>(cs + batch, batch, cs);
    }
    CERDOT_LAUNCH_CHECK();
    a.colsum = cs;
  }
  // batch > 1: the TMA-staged mat-mat over the column-tiled view when the matrix carries one
  const int mm = kernel_path(CERDOT_PATH_MATMAT);
  if (batch > 1 && (mm == 0 || mm == 3 || mm == 4)) {
    bool used = false;
    // workspace past the (256 B aligned) column sums: the tile-split partial products
    const size_t cs = a.bg != 0.0 ? ((sizeof(double) * static_cast<size_t>(batch) * (1 + kColsumSplit) + 255) & ~size_t(255)) : 0;
    void *pws = (workspace != nullptr && workspace_bytes > cs) ? static_cast<char *>(workspace) + cs : nullptr;
    if (int rc = matmat_tiled(mat, x, ldx, batch, y, ldy, a.colsum, peers, a.npeer, peer_offset, pws,
                              pws ? workspace_bytes - cs : 0, st, &used))
      return rc;
    if (used) return CERDOT_OK;
  }
  return cser ? by_col<true>(a, mat->col_bits, mat->omega_ptr_bits, x, ldx, batch, y, ldy, st)
              : by_col<false>(a, mat->col_bits, mat->omega_ptr_bits, x, ldx, batch, y, ldy, st);
}

}  // namespace cerdot
