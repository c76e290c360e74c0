// Dense -> CER / CSER conversion on sm_100a (bit-exact with lemt.formats).
//
// Reference: lemt formats.py:193-295.  The reference sorts every element
// (np.unique + lexsort over (row, rank, col)); here the work is split into
// streaming passes that each read the matrix (or its 1-2 byte rank grid) once:
//
//   k_value_hist    value histogram: per-CTA shared-memory hash table with
//                   warp-aggregated (match.any) counting, merged into a small
//                   global table                         (formats.py:195)
//   k_alphabet      one CTA: (count desc, value asc) order, background moved
//                   or prepended, value-ascending positions for CSER, and the
//                   value -> rank lookup table            (formats.py:196-208, 269-271)
//   k_row_count     CTA per row: rank of every element (rank grid), per-row
//                   non-background count, last present rank, present count
//                                                         (formats.py:218-223, 238-240, 274-278)
//   k_scan_rows     exclusive scans -> entry offsets, CER/CSER row pointers
//                                                         (formats.py:246-247, 283-284)
//   k_row_fill      CTA per row: per-rank block scan -> omegaPtr (+ omegaI),
//                   then a stable per-warp-slab counting scatter of the
//                   columns into colI: (row, rank, col) order without a sort
//                                                         (formats.py:220-221, 241-247, 273-283)
//
// Alphabets larger than CERDOT_FAST_K take the sort-based path in encode_sort.cu (the plan then asks
// for a larger workspace with CERDOT_E_WORKSPACE).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "common.cuh"
#include "encode.cuh"

namespace cerdot {

namespace {

constexpr int kLocalCap = 2048;        // per-CTA hash slots in k_value_hist
constexpr int kLocalProbe = 64;        // probes before spilling to the global table
constexpr int kGlobalCap = 8192;       // global hash slots (<= 25% load at the fast limit)
constexpr int kFastDistinct = CERDOT_FAST_K - 1;  // room for a prepended background
constexpr int kRowThreads = 256;
constexpr int kRowWarps = kRowThreads / 32;

struct Ctrl {
  unsigned int distinct;     // distinct keys inserted in the global table
  unsigned int overflow;     // alphabet exceeds the on-chip path
  unsigned int pos_zero;     // a +0.0 was seen
  unsigned int neg_zero;     // a -0.0 was seen
  unsigned int k;            // final alphabet size
  unsigned int rcap;         // rank table capacity (power of two)
  int mode_index;            // CSER background position
  int pad;
  double background;         // omega[0]
  unsigned long long max_stat[3];  // largest per-row nnz, CER segments, CSER segments
  unsigned long long totals[3];    // nnz, CER segments, CSER segments (= the scans' last entries)
};

struct FastWs {
  unsigned long long *gkey;   // kGlobalCap
  unsigned long long *gcnt;   // kGlobalCap
  double *omega_freq;         // CERDOT_FAST_K
  uint32_t *to_vpos;          // CERDOT_FAST_K
  unsigned long long *rkey;   // 2 * CERDOT_FAST_K
  uint32_t *rrank;            // 2 * CERDOT_FAST_K
  Ctrl *ctrl;
  uint64_t *row_stat;         // 3*m: nnz, last, present
  uint64_t *scan;             // 3*(m+1): entry offset, CER row ptr, CSER row ptr
  void *ranks;                // m*n rank grid (u8 if k <= 256 else u16)
  size_t bytes;
};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

FastWs carve(void *base, int64_t m, int64_t n) {
  FastWs w{};
  char *p = static_cast<char *>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    void *r = p ? p + off : nullptr;
    off = align_up(off + bytes, 256);
    return r;
  };
  w.gkey = static_cast<unsigned long long *>(take(sizeof(unsigned long long) * kGlobalCap));
  w.gcnt = static_cast<unsigned long long *>(take(sizeof(unsigned long long) * kGlobalCap));
  w.omega_freq = static_cast<double *>(take(sizeof(double) * CERDOT_FAST_K));
  w.to_vpos = static_cast<uint32_t *>(take(sizeof(uint32_t) * CERDOT_FAST_K));
  w.rkey = static_cast<unsigned long long *>(take(sizeof(unsigned long long) * 2 * CERDOT_FAST_K));
  w.rrank = static_cast<uint32_t *>(take(sizeof(uint32_t) * 2 * CERDOT_FAST_K));
  w.ctrl = static_cast<Ctrl *>(take(sizeof(Ctrl)));
  w.row_stat = static_cast<uint64_t *>(take(sizeof(uint64_t) * 3 * m));
  w.scan = static_cast<uint64_t *>(take(sizeof(uint64_t) * 3 * (m + 1)));
  w.ranks = take(static_cast<size_t>(m) * n * 2);
  w.bytes = off;
  return w;
}

// ---------------------------------------------------------------- hashing
__device__ __forceinline__ bool global_insert(unsigned long long *gkey, unsigned long long *gcnt, Ctrl *ctrl,
                                              unsigned long long key, unsigned long long cnt) {
  uint32_t h = hash_key(key) & (kGlobalCap - 1);
  for (int probe = 0; probe < kGlobalCap; ++probe) {
    unsigned long long cur = gkey[h];
    if (cur == kEmptyKey) {
      if (ctrl->distinct >= kFastDistinct) {
        atomicOr(&ctrl->overflow, 1u);
        return false;
      }
      cur = atomicCAS(&gkey[h], kEmptyKey, key);
      if (cur == kEmptyKey) {
        if (atomicAdd(&ctrl->distinct, 1u) >= kFastDistinct) atomicOr(&ctrl->overflow, 1u);
        cur = key;
      }
    }
    if (cur == key) {
      atomicAdd(&gcnt[h], cnt);
      return true;
    }
    h = (h + 1) & (kGlobalCap - 1);
  }
  atomicOr(&ctrl->overflow, 1u);
  return false;
}

template <typename T, int V>
struct VecLoad;
template <>
struct VecLoad<float, 4> {
  __device__ static void load(const float *p, double (&out)[4]) {
    float4 v = __ldg(reinterpret_cast<const float4 *>(p));
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
  }
};
template <>
struct VecLoad<double, 2> {
  __device__ static void load(const double *p, double (&out)[2]) {
    double2 v = __ldg(reinterpret_cast<const double2 *>(p));
    out[0] = v.x; out[1] = v.y;
  }
};

// V elements per lane per step; V > 1 requires a contiguous, 16B-aligned matrix.
// Counting: low-entropy matrices are dominated by one value (the background-to-be: 40-96% of the
// elements in the BASELINE configs), so every thread counts the CTA's "hot" key -- the most frequent
// key among the first 32 elements of the matrix -- in a register and sends only the other elements to
// the shared-memory hash (atomics on ~4-60% of the elements, no warp-wide match per element).  The hot
// guess only affects speed: its count is added like any other key's at the end.
template <typename T, int V>
__global__ void __launch_bounds__(256) k_value_hist(const T *__restrict__ w, int64_t m, int64_t n, int64_t ldw,
                                                    FastWs ws) {
  __shared__ unsigned long long skey[kLocalCap];
  __shared__ unsigned int scnt[kLocalCap];
  __shared__ unsigned long long hot_sh;
  __shared__ unsigned int hot_total;
  for (int i = threadIdx.x; i < kLocalCap; i += blockDim.x) {
    skey[i] = kEmptyKey;
    scnt[i] = 0;
  }
  const int lane = threadIdx.x & 31;
  const int64_t total = m * n;
  const bool contig = (ldw == n);
  if (threadIdx.x < 32) {  // hot key: the mode of the first 32 elements (ties: lowest lane)
    const int64_t e = lane;
    unsigned long long kk = kEmptyKey;
    if (e < total) {
      const int64_t r = contig ? 0 : e / n;
      kk = value_key(as_double(__ldg(w + (contig ? e : r * ldw + (e - r * n)))));
    }
    const unsigned int peers = __match_any_sync(0xffffffffu, kk);
    const unsigned int c = kk == kEmptyKey ? 0u : static_cast<unsigned int>(__popc(peers));
    unsigned int best = (c << 5) | (31u - lane);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    const unsigned long long hk = __shfl_sync(0xffffffffu, kk, 31 - static_cast<int>(best & 31u));
    if (lane == 0) {
      hot_sh = hk;
      hot_total = 0;
    }
  }
  __syncthreads();
  const unsigned long long hot = hot_sh;
  unsigned int hot_cnt = 0;
  const int64_t nvec = ceil_div(total, V);
  const int64_t warp_id = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  unsigned int saw_pos0 = 0, saw_neg0 = 0;
  auto insert_local = [&](unsigned long long key) -> bool {  // false: the alphabet overflowed the on-chip path
    uint32_t h = hash_key(key) & (kLocalCap - 1);
    for (int probe = 0; probe < kLocalProbe; ++probe) {
      unsigned long long cur = skey[h];
      if (cur == kEmptyKey) cur = atomicCAS(&skey[h], kEmptyKey, key), cur = (cur == kEmptyKey) ? key : cur;
      if (cur == key) {
        atomicAdd(&scnt[h], 1u);
        return true;
      }
      h = (h + 1) & (kLocalCap - 1);
    }
    return global_insert(ws.gkey, ws.gcnt, ws.ctrl, key, 1ull);
  };
  bool ok = true;
  for (int64_t base = warp_id * 32; base < nvec; base += nwarps * 32) {
    const int64_t vi = base + lane;
    // the grid-stride loop holds one 16 B load per lane: bring the lines of two steps ahead into L2
    if (V > 1 && contig && (vi + 2 * nwarps * 32) * V + V <= total)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(w + (vi + 2 * nwarps * 32) * V));
    double vals[V];
    bool valid[V];
    if (V > 1 && vi * V + V <= total) {
      double tmp[V];
      if constexpr (V > 1) VecLoad<T, V>::load(w + vi * V, tmp);
#pragma unroll
      for (int j = 0; j < V; ++j) { vals[j] = tmp[j]; valid[j] = true; }
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int64_t e = vi * V + j;
        valid[j] = e < total;
        if (valid[j]) {
          int64_t addr = e;
          if (!contig) {
            const int64_t r = e / n;
            addr = r * ldw + (e - r * n);
          }
          vals[j] = as_double(__ldg(w + addr));
        } else {
          vals[j] = 0.0;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (!valid[j]) continue;
      if (vals[j] == 0.0) {
        if (__double_as_longlong(vals[j]) < 0) saw_neg0 = 1; else saw_pos0 = 1;
      }
      const unsigned long long key = value_key(vals[j]);
      if (key == hot) ++hot_cnt;
      else if (ok) ok = insert_local(key);
    }
    if (__any_sync(0xffffffffu, !ok)) break;  // overflowed: the plan switches to the sort path
  }
  if (__any_sync(0xffffffffu, saw_pos0) && lane == 0) atomicOr(&ws.ctrl->pos_zero, 1u);
  if (__any_sync(0xffffffffu, saw_neg0) && lane == 0) atomicOr(&ws.ctrl->neg_zero, 1u);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hot_cnt += __shfl_xor_sync(0xffffffffu, hot_cnt, o);
  if (lane == 0 && hot_cnt) atomicAdd(&hot_total, hot_cnt);
  __syncthreads();
  if (threadIdx.x == 0 && hot_total) global_insert(ws.gkey, ws.gcnt, ws.ctrl, hot, hot_total);
  for (int i = threadIdx.x; i < kLocalCap; i += blockDim.x)
    if (skey[i] != kEmptyKey) global_insert(ws.gkey, ws.gcnt, ws.ctrl, skey[i], scnt[i]);
}

// fp32 fast path of the histogram.  An fp32 value is keyed on chip by its 32 bits (+-0 folded to +0,
// every NaN to one NaN: np.unique's equalities), an order-preserving map of the float, so the per-element
// work is integer only; the CTA's distinct keys are converted to the 64-bit float64 keys of the global
// table (value_key) once, when merged.  Same counting scheme as k_value_hist (hot key in registers).
__device__ __forceinline__ uint32_t fkey32(uint32_t b) {
  if ((b & 0x7fffffffu) == 0u) return 0x80000000u;                               // +-0 -> key of +0
  if ((b & 0x7f800000u) == 0x7f800000u && (b & 0x007fffffu)) return 0xffffffffu;  // NaN -> above +inf
  return (b >> 31) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float fkey32_value(uint32_t k) {
  if (k == 0xffffffffu) return __int_as_float(0x7fc00000);
  return __uint_as_float((k >> 31) ? (k & 0x7fffffffu) : ~k);
}
constexpr uint32_t kEmpty32 = 0x7fffffffu;  // key of a negative NaN bit pattern: never produced by fkey32

// Shared-memory hash insert of one key (k_value_hist_f32's non-hot elements).  false: alphabet overflow.
__device__ __forceinline__ bool hist32_insert(uint32_t *skey, unsigned int *scnt, FastWs ws, uint32_t key) {
  uint32_t h = (key * 0x9E3779B1u) >> (32 - 11);  // kLocalCap = 2^11 slots
  for (int probe = 0; probe < kLocalProbe; ++probe) {
    uint32_t cur = skey[h];
    if (cur == kEmpty32) {
      cur = atomicCAS(&skey[h], kEmpty32, key);
      if (cur == kEmpty32) cur = key;
    }
    if (cur == key) {
      atomicAdd(&scnt[h], 1u);
      return true;
    }
    h = (h + 1) & (kLocalCap - 1);
  }
  return global_insert(ws.gkey, ws.gcnt, ws.ctrl, value_key(static_cast<double>(fkey32_value(key))), 1ull);
}

__global__ void __launch_bounds__(256) k_value_hist_f32(const float4 *__restrict__ w4, int64_t nvec, FastWs ws) {
  __shared__ uint32_t skey[kLocalCap];
  __shared__ unsigned int scnt[kLocalCap];
  __shared__ uint32_t hot_sh;
  __shared__ unsigned int hot_total;
  __shared__ uint32_t stage_all[8][256];  // per-warp staging of non-hot keys (8 per lane per step)
  for (int i = threadIdx.x; i < kLocalCap; i += blockDim.x) {
    skey[i] = kEmpty32;
    scnt[i] = 0;
  }
  const int lane = threadIdx.x & 31;
  uint32_t *stage = stage_all[threadIdx.x >> 5];
  if (threadIdx.x < 32) {  // hot key: the mode of the first 32 elements
    const float *w = reinterpret_cast<const float *>(w4);
    const uint32_t kk = lane < nvec * 4 ? fkey32(__float_as_uint(__ldg(w + lane))) : kEmpty32;
    const unsigned int peers = __match_any_sync(0xffffffffu, kk);
    unsigned int best = ((kk == kEmpty32 ? 0u : __popc(peers)) << 5) | (31u - lane);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    const uint32_t hk = __shfl_sync(0xffffffffu, kk, 31 - static_cast<int>(best & 31u));
    if (lane == 0) {
      hot_sh = hk;
      hot_total = 0;
    }
  }
  __syncthreads();
  const uint32_t hot = hot_sh;
  // The hot key as a test on raw bits: ((b ^ hb) & hm) == 0.  +-0 share a key (the sign is masked); a NaN
  // hot key matches one NaN pattern only (other NaNs take the staged path and merge under the same key).
  const bool hot_zero = hot == 0x80000000u;
  const uint32_t hb = hot_zero ? 0u : (hot == 0xffffffffu ? 0x7fc00000u : __float_as_uint(fkey32_value(hot)));
  const uint32_t hm = hot_zero ? 0x7fffffffu : 0xffffffffu;
  unsigned int hot_cnt = 0, saw_pos0 = 0, saw_neg0 = 0;
  uint32_t hot_or = 0u, hot_and = 0xffffffffu;  // sign bits seen among the hot elements (+-0 bookkeeping)
  bool ok = true;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < nvec; v += 2 * stride) {
    const float4 a = __ldg(w4 + v);
    const bool two = v + stride < nvec;
    const float4 b = two ? __ldg(w4 + v + stride) : a;  // no second vector: the first again, masked out below
    const uint32_t bits[8] = {__float_as_uint(a.x), __float_as_uint(a.y), __float_as_uint(a.z), __float_as_uint(a.w),
                              __float_as_uint(b.x), __float_as_uint(b.y), __float_as_uint(b.z), __float_as_uint(b.w)};
    unsigned todo = 0;  // elements that are not the hot key: the rare, staged path
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t bb = bits[j];
      if (((bb ^ hb) & hm) != 0u) {
        todo |= 1u << j;
      } else {  // (a repeated first vector marks the same signs again: harmless)
        hot_or |= bb;
        hot_and &= bb;
      }
    }
    if (!two) todo &= 0xfu;
    hot_cnt += (two ? 8u : 4u) - __popc(todo);
    // warp-cooperative insertion: the warp's non-hot elements are staged (raw bits) in shared memory and
    // inserted one per lane (a divergent per-lane loop serialised ~3 atomic chains per warp step)
    const unsigned c = __popc(todo);
    unsigned incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const unsigned total_keys = __shfl_sync(0xffffffffu, incl, 31);
    if (total_keys) {
      unsigned pos = incl - c;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (todo & (1u << j)) stage[pos++] = bits[j];
      __syncwarp();
      for (unsigned i = lane; i < total_keys; i += 32) {
        const uint32_t bb = stage[i];
        if ((bb & 0x7fffffffu) == 0u) {
          if (bb) saw_neg0 = 1; else saw_pos0 = 1;
        }
        ok = hist32_insert(skey, scnt, ws, fkey32(bb)) && ok;
      }
      __syncwarp();
    }
    if (__any_sync(0xffffffffu, !ok)) break;  // overflowed: the plan switches to the sort path
  }
  if (hot_zero && hot_cnt) {  // which zeros the hot elements were
    if (hot_or >> 31) saw_neg0 = 1;
    if (!(hot_and >> 31)) saw_pos0 = 1;
  }
  if (__any_sync(0xffffffffu, saw_pos0) && lane == 0) atomicOr(&ws.ctrl->pos_zero, 1u);
  if (__any_sync(0xffffffffu, saw_neg0) && lane == 0) atomicOr(&ws.ctrl->neg_zero, 1u);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hot_cnt += __shfl_xor_sync(0xffffffffu, hot_cnt, o);
  if (lane == 0 && hot_cnt) atomicAdd(&hot_total, hot_cnt);
  __syncthreads();
  if (threadIdx.x == 0 && hot_total)
    global_insert(ws.gkey, ws.gcnt, ws.ctrl, value_key(static_cast<double>(fkey32_value(hot))), hot_total);
  for (int i = threadIdx.x; i < kLocalCap; i += blockDim.x)
    if (skey[i] != kEmpty32)
      global_insert(ws.gkey, ws.gcnt, ws.ctrl, value_key(static_cast<double>(fkey32_value(skey[i]))), scnt[i]);
}

// One CTA: order the alphabet and build the rank lookup table.
__global__ void __launch_bounds__(1024) k_alphabet(FastWs ws, int bg_mode, double bg_value) {
  __shared__ unsigned long long key[CERDOT_FAST_K];
  __shared__ unsigned long long cnt[CERDOT_FAST_K];
  __shared__ unsigned int final_rank[CERDOT_FAST_K];  // by compacted index
  __shared__ unsigned int n_distinct;
  __shared__ int bg_pos;                              // frequency position of the background, -1 if absent
  __shared__ unsigned int k_final, rcap;
  unsigned long long *fkey = cnt;  // value keys of the final alphabet (reuses cnt after the ranking)
  Ctrl *ctrl = ws.ctrl;
  if (ctrl->overflow) return;  // the plan switches to the sort path after its one host synchronisation
  if (threadIdx.x == 0) {
    n_distinct = 0;
    bg_pos = -1;
  }
  __syncthreads();
  {  // all of this thread's slots loaded at once (8 independent loads, not 8 dependent round trips)
    constexpr int kPer = kGlobalCap / 1024;
    unsigned long long kk[kPer], cc[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      kk[j] = ws.gkey[threadIdx.x + j * 1024];
      cc[j] = ws.gcnt[threadIdx.x + j * 1024];
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j)
      if (kk[j] != kEmptyKey) {
        const unsigned int idx = atomicAdd(&n_distinct, 1u);
        key[idx] = kk[j];
        cnt[idx] = cc[j];
      }
  }
  __syncthreads();
  const int k0 = static_cast<int>(n_distinct);
  const unsigned long long bg_key_explicit = value_key(bg_value);
  // frequency position: count desc, value (key) asc -- a total order on distinct keys
  for (int i = threadIdx.x; i < k0; i += blockDim.x) {
    int r = 0;
    const unsigned long long ci = cnt[i], ki = key[i];
    for (int j = 0; j < k0; ++j) r += (cnt[j] > ci) || (cnt[j] == ci && key[j] < ki);
    final_rank[i] = r;
    if (bg_mode ? (ki == bg_key_explicit) : (r == 0)) bg_pos = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    k_final = bg_pos >= 0 ? k0 : k0 + 1;
    unsigned int c = 64;
    while (c < 2 * k_final) c <<= 1;
    rcap = c;
  }
  __syncthreads();
  const int kf = static_cast<int>(k_final);
  const int bp = bg_pos;
  // move / prepend the background (formats.py:201-205)
  for (int i = threadIdx.x; i < k0; i += blockDim.x) {
    const int r = static_cast<int>(final_rank[i]);
    final_rank[i] = bp < 0 ? r + 1 : (r == bp ? 0 : (r < bp ? r + 1 : r));
  }
  for (int s = threadIdx.x; s < static_cast<int>(rcap); s += blockDim.x) ws.rkey[s] = kEmptyKey;
  __syncthreads();
  for (int i = threadIdx.x; i < k0; i += blockDim.x) {
    const int f = static_cast<int>(final_rank[i]);
    double v = key_value(key[i]);
    if (v == 0.0) v = ctrl->pos_zero ? 0.0 : -0.0;  // np.unique keeps one zero; see DESIGN.md
    if (f == 0 && bg_mode) v = bg_value;              // the given background heads omega as given
    ws.omega_freq[f] = v;
    // rank lookup table
    uint32_t h = hash_key(key[i]) & (rcap - 1);
    while (atomicCAS(&ws.rkey[h], kEmptyKey, key[i]) != kEmptyKey) h = (h + 1) & (rcap - 1);
    ws.rrank[h] = static_cast<uint32_t>(f);
  }
  if (bp < 0 && threadIdx.x == 0) ws.omega_freq[0] = bg_value;
  __syncthreads();
  for (int f = threadIdx.x; f < kf; f += blockDim.x) fkey[f] = value_key(ws.omega_freq[f]);
  __syncthreads();
  // value-ascending position of every final element (CSER, formats.py:269-270)
  for (int f = threadIdx.x; f < kf; f += blockDim.x) {
    const unsigned long long kf_key = fkey[f];
    int pos = 0;
    for (int g = 0; g < kf; ++g) pos += fkey[g] < kf_key;
    ws.to_vpos[f] = pos;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ctrl->k = k_final;
    ctrl->rcap = rcap;
    ctrl->mode_index = static_cast<int>(ws.to_vpos[0]);
    ctrl->background = ws.omega_freq[0];
  }
}

__device__ __forceinline__ void block_reduce3(uint64_t &a, uint64_t &b, uint64_t &c, uint64_t *sh) {
  // a, b: sums; c: max.  sh holds 3*32 entries.
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c = max(c, __shfl_xor_sync(0xffffffffu, c, o));
  }
  __syncthreads();
  if (lane == 0) {
    sh[wid] = a;
    sh[32 + wid] = b;
    sh[64 + wid] = c;
  }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    a = lane < nw ? sh[lane] : 0;
    b = lane < nw ? sh[32 + lane] : 0;
    c = lane < nw ? sh[64 + lane] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
      c = max(c, __shfl_xor_sync(0xffffffffu, c, o));
    }
  }
}

// CTA per row: ranks + per-row statistics.
template <typename T, typename RankT>
__global__ void __launch_bounds__(kRowThreads) k_row_count(const T *__restrict__ w, int64_t m, int64_t n,
                                                           int64_t ldw, FastWs ws) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint64_t red[96];
  // both rank widths are launched without a host round trip; the one that does not match k exits
  if (ws.ctrl->overflow || (ws.ctrl->k <= 256) != (sizeof(RankT) == 1)) return;
  const unsigned int rcap = ws.ctrl->rcap;
  const unsigned int k = ws.ctrl->k;
  unsigned long long *rkey = reinterpret_cast<unsigned long long *>(smem);
  unsigned int *hist = reinterpret_cast<unsigned int *>(rkey + rcap);
  unsigned short *rrank = reinterpret_cast<unsigned short *>(hist + k);
  for (unsigned int s = threadIdx.x; s < rcap; s += blockDim.x) {
    rkey[s] = ws.rkey[s];
    rrank[s] = static_cast<unsigned short>(ws.rrank[s]);
  }
  RankT *ranks = static_cast<RankT *>(ws.ranks);
  const int lane = threadIdx.x & 31;
  // vector path: VC consecutive columns per thread (one 16 B load), two loads in flight, the ranks
  // stored packed, the histogram by predicated shared atomics (background rank 0 is not counted)
  constexpr int VC = sizeof(T) == 4 ? 4 : 2;
  const bool vec = (n % VC == 0) && (ldw % VC == 0) && (reinterpret_cast<uintptr_t>(w) % 16 == 0);
  auto rank_of = [&](double v) -> unsigned int {
    const unsigned long long kk = value_key(v);
    uint32_t h = hash_key(kk) & (rcap - 1);
    while (rkey[h] != kk) h = (h + 1) & (rcap - 1);
    return rrank[h];
  };
  for (int64_t row = blockIdx.x; row < m; row += gridDim.x) {
    for (unsigned int q = threadIdx.x; q < k; q += blockDim.x) hist[q] = 0;
    __syncthreads();
    const T *wr = w + row * ldw;
    RankT *rr = ranks + row * n;
    if (vec) {
#pragma unroll 2
      for (int64_t c = static_cast<int64_t>(threadIdx.x) * VC; c < n; c += static_cast<int64_t>(blockDim.x) * VC) {
        double v[VC];
        VecLoad<T, VC>::load(wr + c, v);
        unsigned int rk[VC];
#pragma unroll
        for (int j = 0; j < VC; ++j) {
          rk[j] = rank_of(v[j]);
          if (rk[j] != 0) atomicAdd(&hist[rk[j]], 1u);
        }
        if (sizeof(RankT) == 1) {
          uint32_t pk = 0;
#pragma unroll
          for (int j = 0; j < VC; ++j) pk |= (rk[j] & 0xffu) << (8 * j);
          if (VC == 4) *reinterpret_cast<uint32_t *>(rr + c) = pk;
          else *reinterpret_cast<uint16_t *>(rr + c) = static_cast<uint16_t>(pk);
        } else {
          uint64_t pk = 0;
#pragma unroll
          for (int j = 0; j < VC; ++j) pk |= static_cast<uint64_t>(rk[j] & 0xffffu) << (16 * j);
          if (VC == 4) *reinterpret_cast<uint64_t *>(rr + c) = pk;
          else *reinterpret_cast<uint32_t *>(rr + c) = static_cast<uint32_t>(pk);
        }
      }
    } else
    for (int64_t c0 = threadIdx.x - lane; c0 < n; c0 += blockDim.x) {
      const int64_t c = c0 + lane;
      unsigned int rk = 0;
      if (c < n) {
        const unsigned long long kk = value_key(as_double(__ldg(wr + c)));
        uint32_t h = hash_key(kk) & (rcap - 1);
        while (rkey[h] != kk) h = (h + 1) & (rcap - 1);
        rk = rrank[h];
        rr[c] = static_cast<RankT>(rk);
      }
      const unsigned int peers = __match_any_sync(0xffffffffu, rk);
      if (rk != 0 && lane == __ffs(peers) - 1) atomicAdd(&hist[rk], __popc(peers));
    }
    __syncthreads();
    uint64_t nnz = 0, present = 0, last = 0;
    for (unsigned int q = 1 + threadIdx.x; q < k; q += blockDim.x) {
      const unsigned int h = hist[q];
      nnz += h;
      present += h > 0;
      if (h) last = max(last, static_cast<uint64_t>(q));
    }
    block_reduce3(nnz, present, last, red);
    if (threadIdx.x == 0) {
      ws.row_stat[row] = nnz;
      ws.row_stat[m + row] = last;
      ws.row_stat[2 * m + row] = present;
    }
    __syncthreads();
  }
}

// fp32 fast path of k_row_count (contiguous rows, n % 4 == 0): elements keyed by their 32 bits (fkey32)
// against a 32-bit copy of the rank table built in shared memory from the 64-bit one, the background
// short-circuited; per element: integer key, one probe, a packed rank store, a shared atomic when it
// is not the background.
template <typename RankT>
__global__ void __launch_bounds__(kRowThreads) k_row_count_f32(const float *__restrict__ w, int64_t m, int64_t n,
                                                               int64_t ldw, FastWs ws) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint64_t red[96];
  if (ws.ctrl->overflow || (ws.ctrl->k <= 256) != (sizeof(RankT) == 1)) return;
  const unsigned int rcap = 2 * CERDOT_FAST_K;  // sparse (>= 2x the 64-bit table): ~1 probe per lookup
  const unsigned int k = ws.ctrl->k;
  uint32_t *rkey = reinterpret_cast<uint32_t *>(smem);
  unsigned int *hist = rkey + rcap;
  unsigned short *rrank = reinterpret_cast<unsigned short *>(hist + CERDOT_FAST_K);
  const int shift = 32 - __ffs(rcap) + 1;  // rcap is a power of two
  const unsigned int rcap64 = ws.ctrl->rcap;
  for (unsigned int q = threadIdx.x; q < rcap; q += blockDim.x) rkey[q] = kEmpty32;
  __syncthreads();
  uint32_t bg32 = kEmpty32;
  for (unsigned int q = threadIdx.x; q < rcap64; q += blockDim.x) {
    const unsigned long long k64 = ws.rkey[q];
    if (k64 == kEmptyKey) continue;
    const double v = key_value(k64);
    const float f = static_cast<float>(v);
    if (!(static_cast<double>(f) == v || (v != v))) continue;  // not an fp32 value: no element can match it
    const uint32_t key = fkey32(__float_as_uint(f));
    uint32_t h = (key * 0x9E3779B1u) >> shift;
    while (atomicCAS(&rkey[h], kEmpty32, key) != kEmpty32) h = (h + 1) & (rcap - 1);
    rrank[h] = static_cast<unsigned short>(ws.rrank[q]);
  }
  {
    const double bgv = ws.ctrl->background;
    const float f = static_cast<float>(bgv);
    if (static_cast<double>(f) == bgv || bgv != bgv) bg32 = fkey32(__float_as_uint(f));
  }
  RankT *ranks = static_cast<RankT *>(ws.ranks);
  (void)bg32;
  auto rank_of = [&](uint32_t key) -> unsigned int {  // every element's key is in the table
    uint32_t h = (key * 0x9E3779B1u) >> shift;
    while (rkey[h] != key) h = (h + 1) & (rcap - 1);
    return rrank[h];
  };
  for (int64_t row = blockIdx.x; row < m; row += gridDim.x) {
    for (unsigned int q = threadIdx.x; q < k; q += blockDim.x) hist[q] = 0;
    __syncthreads();
    const float4 *wr = reinterpret_cast<const float4 *>(w + row * ldw);
    RankT *rr = ranks + row * n;
    const int64_t nv = n / 4;
#pragma unroll 4
    for (int64_t c = threadIdx.x; c < nv; c += blockDim.x) {
      const float4 v = __ldg(wr + c);
      const uint32_t rk0 = rank_of(fkey32(__float_as_uint(v.x))), rk1 = rank_of(fkey32(__float_as_uint(v.y)));
      const uint32_t rk2 = rank_of(fkey32(__float_as_uint(v.z))), rk3 = rank_of(fkey32(__float_as_uint(v.w)));
      if (rk0) atomicAdd(&hist[rk0], 1u);
      if (rk1) atomicAdd(&hist[rk1], 1u);
      if (rk2) atomicAdd(&hist[rk2], 1u);
      if (rk3) atomicAdd(&hist[rk3], 1u);
      if (sizeof(RankT) == 1)
        reinterpret_cast<uint32_t *>(rr)[c] = (rk0 & 0xffu) | ((rk1 & 0xffu) << 8) | ((rk2 & 0xffu) << 16) | (rk3 << 24);
      else
        reinterpret_cast<uint2 *>(rr)[c] = make_uint2(rk0 | (rk1 << 16), rk2 | (rk3 << 16));
    }
    __syncthreads();
    uint64_t nnz = 0, present = 0, last = 0;
    for (unsigned int q = 1 + threadIdx.x; q < k; q += blockDim.x) {
      const unsigned int h = hist[q];
      nnz += h;
      present += h > 0;
      if (h) last = max(last, static_cast<uint64_t>(q));
    }
    block_reduce3(nnz, present, last, red);
    if (threadIdx.x == 0) {
      ws.row_stat[row] = nnz;
      ws.row_stat[m + row] = last;
      ws.row_stat[2 * m + row] = present;
    }
    __syncthreads();
  }
}

// One CTA of 1024 threads: three exclusive scans over m rows (m+1 outputs each).
__global__ void __launch_bounds__(1024) k_scan_rows(int64_t m, FastWs ws) {
  // thread t owns rows [t*per, (t+1)*per); its row statistics are loaded in one batch (up to 8 rows x 3
  // statistics in flight) before the block scan, then the outputs are written from registers
  __shared__ uint64_t wsum[3][32];
  __shared__ uint64_t mx_sh[3][32];
  constexpr int kBatch = 8;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int64_t per = ceil_div(m, 1024);
  const int64_t r0 = min64(m, t * per), r1 = min64(m, r0 + per);
  uint64_t s[3] = {0, 0, 0}, mx[3] = {0, 0, 0};
  for (int64_t b = r0; b < r1; b += kBatch) {
    uint64_t v[3][kBatch];
#pragma unroll
    for (int i = 0; i < kBatch; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) v[j][i] = b + i < r1 ? ws.row_stat[j * m + b + i] : 0;
#pragma unroll
    for (int i = 0; i < kBatch; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        s[j] += v[j][i];
        mx[j] = max(mx[j], v[j][i]);
      }
  }
  // block exclusive scan of the three sums; block max of the three maxima
  uint64_t incl[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    incl[j] = s[j];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t u = __shfl_up_sync(0xffffffffu, incl[j], o);
      if (lane >= o) incl[j] += u;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx[j] = max(mx[j], static_cast<uint64_t>(__shfl_xor_sync(0xffffffffu, mx[j], o)));
    if (lane == 31) wsum[j][wid] = incl[j];
    if (lane == 0) mx_sh[j][wid] = mx[j];
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      uint64_t w = wsum[j][lane], wi = w, mm = mx_sh[j][lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t u = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += u;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mm = max(mm, static_cast<uint64_t>(__shfl_xor_sync(0xffffffffu, mm, o)));
      wsum[j][lane] = wi - w;  // exclusive warp offsets
      if (lane == 31) {
        ws.scan[j * (m + 1) + m] = wi;
        ws.ctrl->totals[j] = wi;  // read back with the rest of the control block: one copy, not four
      }
      if (lane == 0) ws.ctrl->max_stat[j] = mm;
    }
  }
  __syncthreads();
  uint64_t run[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) run[j] = wsum[j][wid] + incl[j] - s[j];
  for (int64_t r = r0; r < r1; ++r)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      ws.scan[j * (m + 1) + r] = run[j];
      run[j] += ws.row_stat[j * m + r];
    }
}

// Exclusive block scan of (a, b) pairs over the CTA; returns totals too.
__device__ __forceinline__ void block_exscan2(unsigned int a, unsigned int b, unsigned int &ea, unsigned int &eb,
                                              unsigned int *sh /* 2*32 */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned int ia = a, ib = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int va = __shfl_up_sync(0xffffffffu, ia, o);
    const unsigned int vb = __shfl_up_sync(0xffffffffu, ib, o);
    if (lane >= o) { ia += va; ib += vb; }
  }
  if (lane == 31) { sh[wid] = ia; sh[32 + wid] = ib; }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    unsigned int wa = lane < nw ? sh[lane] : 0, wb = lane < nw ? sh[32 + lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned int va = __shfl_up_sync(0xffffffffu, wa, o);
      const unsigned int vb = __shfl_up_sync(0xffffffffu, wb, o);
      if (lane >= o) { wa += va; wb += vb; }
    }
    sh[lane] = wa;
    sh[32 + lane] = wb;
  }
  __syncthreads();
  const unsigned int base_a = wid ? sh[wid - 1] : 0, base_b = wid ? sh[32 + wid - 1] : 0;
  ea = base_a + ia - a;
  eb = base_b + ib - b;
  __syncthreads();
}

// CTA per row: write omegaPtr (+ omegaI for CSER) and scatter colI.
template <typename ColT, typename RankT, bool CSER>
__global__ void __launch_bounds__(kRowThreads) k_row_fill(int64_t m, int64_t n, FastWs ws, ColT *__restrict__ col,
                                                          void *omega_ptr, int op_bits, void *omega_index,
                                                          int oi_bits) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned int scan_sh[64];
  const unsigned int k = ws.ctrl->k;
  unsigned int *wc = reinterpret_cast<unsigned int *>(smem);  // [kRowWarps][k] per-warp counts -> offsets
  unsigned int *cnt = wc + kRowWarps * k;                      // [k] per-rank count
  unsigned int *excl = cnt + k;                                // [k] exclusive entry offset per rank
  unsigned int *pidx = excl + k;                               // [k] CSER: index among present ranks
  const RankT *ranks = static_cast<const RankT *>(ws.ranks);
  const uint64_t *entry_off = ws.scan;
  const uint64_t *seg_off = ws.scan + (CSER ? 2 : 1) * (m + 1);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t slab = ceil_div(ceil_div(n, kRowWarps), 32) * 32;
  const unsigned int per = static_cast<unsigned int>(ceil_div(k, kRowThreads));
  for (int64_t row = blockIdx.x; row < m; row += gridDim.x) {
    for (unsigned int q = threadIdx.x; q < kRowWarps * k; q += blockDim.x) wc[q] = 0;
    __syncthreads();
    const RankT *rr = ranks + row * n;
    const int64_t c_begin = wid * slab, c_end = min64(n, c_begin + slab);
    if (sizeof(RankT) == 1 && (slab & 3) == 0 && (n & 3) == 0) {
      // count pass, 4 ranks per lane per load, predicated shared atomics (no match.any; the counts are
      // order-free, only the scatter below needs lane order)
      for (int64_t c = c_begin + 4 * lane; c < c_end; c += 128) {
        const uint32_t pk = *reinterpret_cast<const uint32_t *>(rr + c);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const unsigned int rk = (pk >> (8 * j)) & 0xffu;
          if (rk != 0 && c + j < c_end) atomicAdd(&wc[wid * k + rk], 1u);
        }
      }
    } else {
      for (int64_t c0 = c_begin; c0 < c_end; c0 += 32) {
        const int64_t c = c0 + lane;
        const unsigned int rk = c < c_end ? rr[c] : 0u;
        const unsigned int peers = __match_any_sync(0xffffffffu, rk);
        if (rk != 0 && lane == __ffs(peers) - 1) wc[wid * k + rk] += __popc(peers);
      }
    }
    __syncthreads();
    // per rank: total count and per-warp exclusive offsets
    for (unsigned int q = threadIdx.x; q < k; q += blockDim.x) {
      unsigned int run = 0;
#pragma unroll
      for (int w2 = 0; w2 < kRowWarps; ++w2) {
        const unsigned int v = wc[w2 * k + q];
        wc[w2 * k + q] = run;
        run += v;
      }
      cnt[q] = q == 0 ? 0 : run;
    }
    __syncthreads();
    // block scan over ranks: thread t owns ranks [t*per, (t+1)*per)
    unsigned int la = 0, lb = 0;
    const unsigned int q0 = threadIdx.x * per, q1 = min(k, q0 + per);
    for (unsigned int q = q0; q < q1; ++q) { la += cnt[q]; lb += cnt[q] > 0; }
    unsigned int ea, eb;
    block_exscan2(la, lb, ea, eb, scan_sh);
    for (unsigned int q = q0; q < q1; ++q) {
      excl[q] = ea;
      pidx[q] = eb;
      ea += cnt[q];
      eb += cnt[q] > 0;
    }
    __syncthreads();
    const uint64_t e0 = entry_off[row], s0 = seg_off[row];
    const unsigned int last = static_cast<unsigned int>(ws.row_stat[m + row]);
    for (unsigned int q = 1 + threadIdx.x; q < k; q += blockDim.x) {
      const uint64_t end = e0 + excl[q] + cnt[q];
      if (CSER) {
        if (cnt[q]) {
          const uint64_t j = s0 + pidx[q];
          store_index(omega_index, oi_bits, j, ws.to_vpos[q]);
          store_index(omega_ptr, op_bits, j + 1, end);
        }
      } else if (q <= last) {
        store_index(omega_ptr, op_bits, s0 + q, end);  // segment s0 + q - 1 ends here
      }
    }
    // stable scatter: warp slabs are column-ordered, lanes ordered inside a step
    const unsigned int lt = (1u << lane) - 1u;
    for (int64_t c0 = c_begin; c0 < c_end; c0 += 32) {
      const int64_t c = c0 + lane;
      const unsigned int rk = c < c_end ? rr[c] : 0u;
      const unsigned int peers = __match_any_sync(0xffffffffu, rk);
      if (rk != 0) {
        const uint64_t pos = e0 + excl[rk] + wc[wid * k + rk] + __popc(peers & lt);
        col[pos] = static_cast<ColT>(c);
      }
      __syncwarp();
      if (rk != 0 && lane == __ffs(peers) - 1) wc[wid * k + rk] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
  }
}

// CTA per row, u8 rank grid, n a multiple of 16: a warp compacts the non-zero ranks of its column slab into
// a shared list of (column << 8 | rank) entries in column order (16 ranks per lane per load, one warp scan
// per 512 columns), so the stable scatter walks only the row's entries instead of every column.
//   CHUNKED = false (sparse rows): the whole slab is listed once, counting on the way (a 91%-zero fc layer:
//     11x fewer scatter steps; 130 -> 56 us on AlexNet fc6);
//   CHUNKED = true (any density, 2 KB of list per warp): a counting pass, then 512 columns at a time are
//     listed and scattered (the 32768^2 layer at 30%: a third of the scatter steps).
template <typename ColT, bool CSER, bool CHUNKED>
__global__ void __launch_bounds__(kRowThreads) k_row_fill_compact(int64_t m, int64_t n, FastWs ws, uint32_t cap,
                                                                  ColT *__restrict__ col, void *omega_ptr, int op_bits,
                                                                  void *omega_index, int oi_bits) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned int scan_sh[64];
  const unsigned int k = ws.ctrl->k;
  unsigned int *wc = reinterpret_cast<unsigned int *>(smem);  // [kRowWarps][k] per-warp counts -> offsets
  unsigned int *cnt = wc + kRowWarps * k;                      // [k] per-rank count
  unsigned int *excl = cnt + k;                                // [k] exclusive entry offset per rank
  unsigned int *pidx = excl + k;                               // [k] CSER: index among present ranks
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t *list = reinterpret_cast<uint32_t *>(pidx + k) + static_cast<size_t>(wid) * cap;  // the warp's entries
  const uint8_t *ranks = static_cast<const uint8_t *>(ws.ranks);
  const uint64_t *entry_off = ws.scan;
  const uint64_t *seg_off = ws.scan + (CSER ? 2 : 1) * (m + 1);
  const int64_t slab = ceil_div(ceil_div(n, kRowWarps), 512) * 512;  // whole 512-column steps per warp
  const unsigned int per = static_cast<unsigned int>(ceil_div(k, kRowThreads));
  const unsigned int lt = (1u << lane) - 1u;
  for (int64_t row = blockIdx.x; row < m; row += gridDim.x) {
    for (unsigned int q = threadIdx.x; q < kRowWarps * k; q += blockDim.x) wc[q] = 0;
    __syncthreads();
    const uint8_t *rr = ranks + row * n;
    const int64_t c_begin = wid * slab, c_end = min64(n, c_begin + slab);
    // one 512-column step: the non-zero ranks, listed from `base` in column order (LIST) and / or counted
    // per rank (COUNT); returns how many there were
    auto step = [&](int64_t c0, uint32_t base, bool do_list, bool do_count) -> uint32_t {
      const int64_t c = c0 + 16 * lane;
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (c < c_end) v = *reinterpret_cast<const uint4 *>(rr + c);  // n % 16 == 0: whole vectors
      const uint32_t wv4[4] = {v.x, v.y, v.z, v.w};
      uint32_t nib[4], mine = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t nz = (((wv4[j] & 0x7f7f7f7fu) + 0x7f7f7f7fu) | wv4[j]) & 0x80808080u;
        nib[j] = ((nz >> 7) * 0x01020408u) >> 24;  // bit b: byte b of the word is non-zero
        mine += __popc(nib[j]);
      }
      uint32_t incl = mine;
      if (do_list) {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
      }
      uint32_t at = base + incl - mine;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t mk = nib[j];
        while (mk) {
          const int b = __ffs(static_cast<int>(mk)) - 1;
          mk &= mk - 1u;
          const uint32_t rk = (wv4[j] >> (8 * b)) & 0xffu;
          if (do_list) list[at++] = (static_cast<uint32_t>(c + 4 * j + b) << 8) | rk;
          if (do_count) atomicAdd(&wc[wid * k + rk], 1u);
        }
      }
      return do_list ? __shfl_sync(0xffffffffu, incl, 31) : 0u;
    };
    // ---- count (and, for sparse rows, list the whole slab)
    uint32_t nzw = 0;
    for (int64_t c0 = c_begin; c0 < c_end; c0 += 512) nzw += step(c0, nzw, !CHUNKED, true);
    __syncthreads();
    // per rank: total count and per-warp exclusive offsets
    for (unsigned int q = threadIdx.x; q < k; q += blockDim.x) {
      unsigned int run = 0;
#pragma unroll
      for (int w2 = 0; w2 < kRowWarps; ++w2) {
        const unsigned int v = wc[w2 * k + q];
        wc[w2 * k + q] = run;
        run += v;
      }
      cnt[q] = q == 0 ? 0 : run;
    }
    __syncthreads();
    // block scan over ranks: thread t owns ranks [t*per, (t+1)*per)
    unsigned int la = 0, lb = 0;
    const unsigned int q0 = threadIdx.x * per, q1 = min(k, q0 + per);
    for (unsigned int q = q0; q < q1; ++q) { la += cnt[q]; lb += cnt[q] > 0; }
    unsigned int ea, eb;
    block_exscan2(la, lb, ea, eb, scan_sh);
    for (unsigned int q = q0; q < q1; ++q) {
      excl[q] = ea;
      pidx[q] = eb;
      ea += cnt[q];
      eb += cnt[q] > 0;
    }
    __syncthreads();
    const uint64_t e0 = entry_off[row], s0 = seg_off[row];
    const unsigned int last = static_cast<unsigned int>(ws.row_stat[m + row]);
    for (unsigned int q = 1 + threadIdx.x; q < k; q += blockDim.x) {
      const uint64_t end = e0 + excl[q] + cnt[q];
      if (CSER) {
        if (cnt[q]) {
          const uint64_t j = s0 + pidx[q];
          store_index(omega_index, oi_bits, j, ws.to_vpos[q]);
          store_index(omega_ptr, op_bits, j + 1, end);
        }
      } else if (q <= last) {
        store_index(omega_ptr, op_bits, s0 + q, end);  // segment s0 + q - 1 ends here
      }
    }
    // stable scatter over listed entries: warp lists are column-ordered, lanes ordered inside a step
    auto scatter = [&](uint32_t count) {
      for (uint32_t i0 = 0; i0 < count; i0 += 32) {
        const uint32_t e = i0 + lane < count ? list[i0 + lane] : 0u;
        const unsigned int rk = e & 0xffu;
        const unsigned int peers = __match_any_sync(0xffffffffu, rk);
        if (rk != 0) {
          const uint64_t pos = e0 + excl[rk] + wc[wid * k + rk] + __popc(peers & lt);
          col[pos] = static_cast<ColT>(e >> 8);
        }
        __syncwarp();
        if (rk != 0 && lane == __ffs(peers) - 1) wc[wid * k + rk] += __popc(peers);
        __syncwarp();
      }
    };
    if (CHUNKED) {
      for (int64_t c0 = c_begin; c0 < c_end; c0 += 512) {
        const uint32_t got = step(c0, 0u, true, false);
        __syncwarp();
        scatter(got);
      }
    } else {
      scatter(nzw);
    }
    __syncthreads();
  }
}

// Tail: omega (CER frequency order / CSER value order), rowPtr, omegaPtr[0].
__global__ void k_fill_tail(int64_t m, FastWs ws, bool cser, double *omega, void *row_ptr, int rp_bits,
                            void *omega_ptr, int op_bits) {
  const unsigned int k = ws.ctrl->k;
  const uint64_t *seg_scan = ws.scan + (cser ? 2 : 1) * (m + 1);
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = tid; i <= m; i += stride) store_index(row_ptr, rp_bits, i, seg_scan[i]);
  for (int64_t f = tid; f < k; f += stride) omega[cser ? ws.to_vpos[f] : f] = ws.omega_freq[f];
  if (tid == 0) store_index(omega_ptr, op_bits, 0, 0);
}

template <typename T>
int launch_hist(const void *w, int64_t m, int64_t n, int64_t ldw, const FastWs &ws, cudaStream_t st) {
  const int64_t total = m * n;
  constexpr int V = sizeof(T) == 4 ? 4 : 2;
  const bool vec_ok = (ldw == n) && (reinterpret_cast<uintptr_t>(w) % 16 == 0);
  if (sizeof(T) == 4 && vec_ok && total % 4 == 0) {  // fp32, contiguous: integer keys on chip
    const int64_t nvec = total / 4;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nvec, 256 * 8), num_sms() * 6)));
    k_value_hist_f32<<<grid, 256, 0, st>>>(static_cast<const float4 *>(w), nvec, ws);
    CERDOT_LAUNCH_CHECK();
    return CERDOT_OK;
  }
  const int64_t units = vec_ok ? ceil_div(total, V) : total;
  const int64_t want = ceil_div(units, 256 * 8);
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, num_sms() * 8)));
  if (vec_ok)
    k_value_hist<T, V><<<grid, 256, 0, st>>>(static_cast<const T *>(w), m, n, ldw, ws);
  else
    k_value_hist<T, 1><<<grid, 256, 0, st>>>(static_cast<const T *>(w), m, n, ldw, ws);
  CERDOT_LAUNCH_CHECK();
  return CERDOT_OK;
}

template <typename T, typename RankT>
int launch_row_count(const void *w, int64_t m, int64_t n, int64_t ldw, const FastWs &ws, cudaStream_t st) {
  if (sizeof(T) == 4 && n % 4 == 0 && ldw % 4 == 0 && reinterpret_cast<uintptr_t>(w) % 16 == 0) {
    constexpr unsigned int kRcapMax32 = 2 * CERDOT_FAST_K;
    const size_t smem32 = kRcapMax32 * (sizeof(uint32_t) + sizeof(unsigned short)) + CERDOT_FAST_K * sizeof(unsigned int) + 16;
    auto kern32 = k_row_count_f32<RankT>;
    CERDOT_CUDA_CHECK(cudaFuncSetAttribute(kern32, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem32)));
    int per_sm = 0;  // one full wave of CTAs (a partial second wave idled a third of the GPU)
    CERDOT_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern32, kRowThreads, smem32));
    const int grid32 = static_cast<int>(std::min<int64_t>(m, static_cast<int64_t>(num_sms()) * std::max(per_sm, 1)));
    kern32<<<grid32, kRowThreads, smem32, st>>>(static_cast<const float *>(w), m, n, ldw, ws);
    CERDOT_LAUNCH_CHECK();
    return CERDOT_OK;
  }
  // sized for the largest on-chip alphabet (k and the rank-table capacity are device-side values here)
  constexpr unsigned int kRcapMax = 2 * CERDOT_FAST_K;
  const size_t smem =
      kRcapMax * (sizeof(unsigned long long) + sizeof(unsigned short)) + CERDOT_FAST_K * sizeof(unsigned int) + 16;
  auto kern = k_row_count<T, RankT>;
  CERDOT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int grid = static_cast<int>(std::min<int64_t>(m, num_sms() * 8));
  kern<<<grid, kRowThreads, smem, st>>>(static_cast<const T *>(w), m, n, ldw, ws);
  CERDOT_LAUNCH_CHECK();
  return CERDOT_OK;
}

template <typename ColT, typename RankT>
int launch_fill(int64_t m, int64_t n, const FastWs &ws, unsigned int k, int64_t max_row_nnz, int64_t nnz, bool cser, void *col,
                void *op, int op_bits, void *oi, int oi_bits, cudaStream_t st) {
  const size_t smem = (kRowWarps + 3) * static_cast<size_t>(k) * sizeof(unsigned int);
  // u8 ranks, whole 16 B vectors per row, columns that fit 24 bits: the compacting kernel.  Sparse rows
  // (<= 20% non-zero) whose per-warp lists fit (sized by the longest row: a warp's slab cannot hold more)
  // are listed whole; otherwise 512 columns at a time (2 KB of list per warp).
  if (sizeof(RankT) == 1 && (n % 16) == 0 && n < (int64_t(1) << 24)) {
    const int64_t slab = ceil_div(ceil_div(n, kRowWarps), 512) * 512;
    const uint32_t cap_whole = static_cast<uint32_t>(std::min<int64_t>(slab, std::max<int64_t>(max_row_nnz, 1)));
    const bool whole = nnz <= m * n / 5 && smem + sizeof(uint32_t) * kRowWarps * static_cast<size_t>(cap_whole) <= 56 * 1024;
    const uint32_t cap = whole ? cap_whole : 512u;
    const size_t smem_c = smem + sizeof(uint32_t) * kRowWarps * static_cast<size_t>(cap);
    auto goc = [&](auto kern) -> int {
      CERDOT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_c)));
      int per_sm = 0;
      CERDOT_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRowThreads, smem_c));
      const int grid = static_cast<int>(std::min<int64_t>(m, static_cast<int64_t>(num_sms()) * std::max(per_sm, 1)));
      kern<<<grid, kRowThreads, smem_c, st>>>(m, n, ws, cap, static_cast<ColT *>(col), op, op_bits, oi, oi_bits);
      return CERDOT_OK;
    };
    int rc;
    if (whole) rc = cser ? goc(k_row_fill_compact<ColT, true, false>) : goc(k_row_fill_compact<ColT, false, false>);
    else rc = cser ? goc(k_row_fill_compact<ColT, true, true>) : goc(k_row_fill_compact<ColT, false, true>);
    if (rc) return rc;
    CERDOT_LAUNCH_CHECK();
    return CERDOT_OK;
  }
  auto go = [&](auto kern) -> int {
    CERDOT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int per_sm = 0;  // one full wave of CTAs over the rows (no partial tail wave)
    CERDOT_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRowThreads, smem));
    const int grid = static_cast<int>(std::min<int64_t>(m, static_cast<int64_t>(num_sms()) * std::max(per_sm, 1)));
    kern<<<grid, kRowThreads, smem, st>>>(m, n, ws, static_cast<ColT *>(col), op, op_bits, oi, oi_bits);
    return CERDOT_OK;
  };
  if (int rc = cser ? go(k_row_fill<ColT, RankT, true>) : go(k_row_fill<ColT, RankT, false>)) return rc;
  CERDOT_LAUNCH_CHECK();
  return CERDOT_OK;
}

}  // namespace

size_t encode_workspace_bytes(int64_t m, int64_t n) { return carve(nullptr, m, n).bytes; }

int encode_plan(const void *w, int dtype, int64_t m, int64_t n, int64_t ldw, int bg_mode, double bg_value,
                void *workspace, size_t workspace_bytes, cerdot_encode_info *info, cudaStream_t st) {
  if (m <= 0 || n <= 0)  // the reference fails on omega[0] of an empty alphabet (formats.py:199)
    return fail(CERDOT_E_INDEX, "index 0 is out of bounds for axis 0 with size 0");
  if (ldw < n) return fail(CERDOT_E_VALUE, "row stride ldw must be >= n");
  if (dtype != CERDOT_F32 && dtype != CERDOT_F64) return fail(CERDOT_E_TYPE, "w must be float32 or float64");
  const size_t need = encode_workspace_bytes(m, n);
  info->m = m;
  info->n = n;
  info->workspace_bytes = need;
  if (workspace == nullptr || workspace_bytes < need)
    return fail(CERDOT_E_WORKSPACE, "encode workspace too small: need " + std::to_string(need) + " bytes");
  FastWs ws = carve(workspace, m, n);
  // the key and count tables are adjacent in the workspace (carve): one memset
  CERDOT_CUDA_CHECK(cudaMemsetAsync(ws.gkey, 0,
                                    reinterpret_cast<char *>(ws.gcnt + kGlobalCap) - reinterpret_cast<char *>(ws.gkey), st));
  CERDOT_CUDA_CHECK(cudaMemsetAsync(ws.ctrl, 0, sizeof(Ctrl), st));
  int rc = dtype == CERDOT_F32 ? launch_hist<float>(w, m, n, ldw, ws, st) : launch_hist<double>(w, m, n, ldw, ws, st);
  if (rc) return rc;
  // alphabet, ranks, row statistics and scans are queued without host round trips (each kernel exits
  // when the histogram overflowed the on-chip path); one synchronisation at the end reads the sizes
  k_alphabet<<<1, 1024, 0, st>>>(ws, bg_mode, bg_value);
  CERDOT_LAUNCH_CHECK();
  rc = dtype == CERDOT_F32 ? launch_row_count<float, uint8_t>(w, m, n, ldw, ws, st)
                           : launch_row_count<double, uint8_t>(w, m, n, ldw, ws, st);
  if (rc) return rc;
  rc = dtype == CERDOT_F32 ? launch_row_count<float, uint16_t>(w, m, n, ldw, ws, st)
                           : launch_row_count<double, uint16_t>(w, m, n, ldw, ws, st);
  if (rc) return rc;
  k_scan_rows<<<1, 1024, 0, st>>>(m, ws);
  CERDOT_LAUNCH_CHECK();
  Ctrl ctrl{};
  CERDOT_CUDA_CHECK(cudaMemcpyAsync(&ctrl, ws.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
  CERDOT_CUDA_CHECK(cudaStreamSynchronize(st));
  const unsigned long long *totals = ctrl.totals;
  if (ctrl.overflow)  // alphabet too large for the on-chip tables: sort-based path (encode_sort.cu)
    return encode_sort_plan(w, dtype, m, n, ldw, bg_mode, bg_value, workspace, workspace_bytes, info, st);
  const unsigned int k = ctrl.k;
  info->k = k;
  info->nnz = static_cast<int64_t>(totals[0]);
  info->segments_cer = static_cast<int64_t>(totals[1]);
  info->segments_cser = static_cast<int64_t>(totals[2]);
  info->mode_index = ctrl.mode_index;
  info->background = ctrl.background;
  info->path = 0;
  info->max_row_nnz = static_cast<int64_t>(ctrl.max_stat[0]);
  info->max_row_segments_cer = static_cast<int64_t>(ctrl.max_stat[1]);
  info->max_row_segments_cser = static_cast<int64_t>(ctrl.max_stat[2]);
  return CERDOT_OK;
}

int encode_fill(const cerdot_encode_info *info, int kind, void *workspace, size_t workspace_bytes, double *omega,
                void *col, int col_bits, void *op, int op_bits, void *rp, int rp_bits, void *oi, int oi_bits,
                cudaStream_t st) {
  const int64_t m = info->m, n = info->n;
  if (info->path == 1)
    return encode_sort_fill(info, kind, workspace, workspace_bytes, omega, col, col_bits, op, op_bits, rp, rp_bits, oi,
                            oi_bits, st);
  if (workspace == nullptr || workspace_bytes < encode_workspace_bytes(m, n))
    return fail(CERDOT_E_WORKSPACE, "encode workspace too small");
  FastWs ws = carve(workspace, m, n);
  const bool cser = kind == CERDOT_CSER;
  const unsigned int k = static_cast<unsigned int>(info->k);
  int rc;
  auto by_col = [&](auto rank_tag) -> int {
    using RankT = decltype(rank_tag);
    switch (col_bits) {
      case 8: return launch_fill<uint8_t, RankT>(m, n, ws, k, info->max_row_nnz, info->nnz, cser, col, op, op_bits, oi, oi_bits, st);
      case 16: return launch_fill<uint16_t, RankT>(m, n, ws, k, info->max_row_nnz, info->nnz, cser, col, op, op_bits, oi, oi_bits, st);
      default: return launch_fill<uint32_t, RankT>(m, n, ws, k, info->max_row_nnz, info->nnz, cser, col, op, op_bits, oi, oi_bits, st);
    }
  };
  rc = k <= 256 ? by_col(uint8_t{}) : by_col(uint16_t{});
  if (rc) return rc;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(m + 1, 256), num_sms() * 4)));
  k_fill_tail<<<grid, 256, 0, st>>>(m, ws, cser, omega, rp, rp_bits, op, op_bits);
  CERDOT_LAUNCH_CHECK();
  return CERDOT_OK;
}

}  // namespace cerdot
