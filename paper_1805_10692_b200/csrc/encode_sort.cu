// Sort-based dense -> CER / CSER conversion for alphabets larger than the on-chip tables
// (more than CERDOT_FAST_K - 1 distinct values).  Same semantics as encode.cu, bit-exact with
// lemt formats.py:193-295; it follows the reference's own structure (sort, unique, lexsort) with
// device radix sorts (CUB) over order-preserving value keys and (row*K + rank, col) pairs.
//
//   keys     value key of every element                      (formats.py:195 np.unique)
//   sort+RLE distinct values (ascending) + counts
//   sort     stable by ~count -> frequency order (count desc, value asc)   (formats.py:196)
//   ranks    background moved / prepended; value positions for CSER        (formats.py:198-208, 269-271)
//   pairs    non-background elements keyed row*K + rank, value col; stable sort -> (row, rank, col)
//                                                                           (formats.py:218-221)
//   RLE      (row, rank) runs = CSER segments; CER segments = runs scattered to rank slots, empty
//            padding filled by a max-scan of the (non-decreasing) segment ends (formats.py:238-247)
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cub/cub.cuh>
#include <string>

#include "common.cuh"
#include "encode.cuh"

namespace cerdot {

namespace {

struct GenCtrl {
  unsigned int nrun, npair, nnz, pos_zero, neg_zero, k, absent;
  int bg_pos;  // frequency position of the background among distinct values, -1 if absent
  int mode_index;
  int pad;
  unsigned long long max_stat[3];
};

struct GenWs {
  uint64_t *k0, *k1, *uniq, *pair_key, *pair_end, *row_stat, *scan;
  uint32_t *v0, *v1, *cnt, *rank_of_u, *to_vpos, *pair_cnt;
  double *omega_freq;
  GenCtrl *ctrl;
  void *tmp;
  size_t tmp_bytes, bytes;
};

size_t align256(size_t v) { return (v + 255) / 256 * 256; }

size_t cub_tmp_bytes(int64_t N) {
  size_t b = 0, t = 0;
  const int n = static_cast<int>(N);
  cub::DeviceRadixSort::SortKeys(nullptr, t, static_cast<uint64_t *>(nullptr), static_cast<uint64_t *>(nullptr), n);
  b = std::max(b, t);
  cub::DeviceRadixSort::SortPairs(nullptr, t, static_cast<uint64_t *>(nullptr), static_cast<uint64_t *>(nullptr),
                                  static_cast<uint32_t *>(nullptr), static_cast<uint32_t *>(nullptr), n);
  b = std::max(b, t);
  cub::DeviceRunLengthEncode::Encode(nullptr, t, static_cast<uint64_t *>(nullptr), static_cast<uint64_t *>(nullptr),
                                     static_cast<uint32_t *>(nullptr), static_cast<uint32_t *>(nullptr), n);
  b = std::max(b, t);
  cub::DeviceScan::InclusiveSum(nullptr, t, static_cast<uint64_t *>(nullptr), static_cast<uint64_t *>(nullptr), n);
  b = std::max(b, t);
  // CER max-scan runs over S_cer + 1 <= 2^31 items of 8/16/32 bits: bound it at the largest count
  const int big = 0x7fffffff;
  cub::DeviceScan::InclusiveScan(nullptr, t, static_cast<uint32_t *>(nullptr), static_cast<uint32_t *>(nullptr),
                                 cub::Max(), big);
  b = std::max(b, t);
  cub::DeviceScan::InclusiveScan(nullptr, t, static_cast<uint16_t *>(nullptr), static_cast<uint16_t *>(nullptr),
                                 cub::Max(), big);
  b = std::max(b, t);
  cub::DeviceScan::InclusiveScan(nullptr, t, static_cast<uint8_t *>(nullptr), static_cast<uint8_t *>(nullptr),
                                 cub::Max(), big);
  b = std::max(b, t);
  return b;
}

GenWs gen_carve(void *base, int64_t m, int64_t n) {
  GenWs w{};
  const int64_t N = m * n;
  char *p = static_cast<char *>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    void *r = p ? p + off : nullptr;
    off = align256(off + bytes);
    return r;
  };
  w.k0 = static_cast<uint64_t *>(take(8 * N));
  w.k1 = static_cast<uint64_t *>(take(8 * N));
  w.uniq = static_cast<uint64_t *>(take(8 * N));
  w.pair_key = static_cast<uint64_t *>(take(8 * N));
  w.pair_end = static_cast<uint64_t *>(take(8 * N));
  w.row_stat = static_cast<uint64_t *>(take(8 * 3 * m));
  w.scan = static_cast<uint64_t *>(take(8 * 3 * (m + 1)));
  w.v0 = static_cast<uint32_t *>(take(4 * N));
  w.v1 = static_cast<uint32_t *>(take(4 * N));
  w.cnt = static_cast<uint32_t *>(take(4 * N));
  w.rank_of_u = static_cast<uint32_t *>(take(4 * N));
  w.to_vpos = static_cast<uint32_t *>(take(4 * (N + 1)));
  w.pair_cnt = static_cast<uint32_t *>(take(4 * N));
  w.omega_freq = static_cast<double *>(take(8 * (N + 1)));
  w.ctrl = static_cast<GenCtrl *>(take(sizeof(GenCtrl)));
  w.tmp_bytes = cub_tmp_bytes(N);
  w.tmp = take(w.tmp_bytes);
  w.bytes = off;
  return w;
}

__device__ __forceinline__ uint32_t lower_bound_u64(const uint64_t *a, uint32_t n, uint64_t key) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <typename T>
__global__ void k_gen_keys(const T *__restrict__ w, int64_t m, int64_t n, int64_t ldw, GenWs ws) {
  const int64_t N = m * n;
  unsigned int p0 = 0, n0 = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / n, c = i - r * n;
    const double v = static_cast<double>(w[r * ldw + c]);
    ws.k0[i] = value_key(v);
    if (v == 0.0) {
      if (__double_as_longlong(v) < 0) n0 = 1; else p0 = 1;
    }
  }
  if (p0) atomicOr(&ws.ctrl->pos_zero, 1u);
  if (n0) atomicOr(&ws.ctrl->neg_zero, 1u);
}

__global__ void k_gen_negcount(GenWs ws) {
  const uint32_t k0 = ws.ctrl->nrun;
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < k0; u += gridDim.x * blockDim.x) {
    ws.k0[u] = static_cast<uint64_t>(~ws.cnt[u]);  // ascending ~count == count descending
    ws.v0[u] = u;
  }
}

// v1[f] = distinct index at frequency position f  ->  v0[u] = frequency position of u
__global__ void k_gen_freqpos(GenWs ws) {
  const uint32_t k0 = ws.ctrl->nrun;
  for (uint32_t f = blockIdx.x * blockDim.x + threadIdx.x; f < k0; f += gridDim.x * blockDim.x) ws.v0[ws.v1[f]] = f;
}

__global__ void k_gen_background(GenWs ws, int bg_mode, double bg_value) {
  const uint32_t k0 = ws.ctrl->nrun;
  int pos = 0;
  if (bg_mode) {
    const uint64_t key = value_key(bg_value);
    const uint32_t u = lower_bound_u64(ws.uniq, k0, key);
    pos = (u < k0 && ws.uniq[u] == key) ? static_cast<int>(ws.v0[u]) : -1;
  }
  ws.ctrl->bg_pos = pos;
  ws.ctrl->absent = pos < 0;
  ws.ctrl->k = k0 + (pos < 0 ? 1u : 0u);
}

__global__ void k_gen_ranks(GenWs ws, int bg_mode, double bg_value) {
  const uint32_t k0 = ws.ctrl->nrun;
  const int p = ws.ctrl->bg_pos;
  const uint64_t bg_key = value_key(bg_value);
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < k0; u += gridDim.x * blockDim.x) {
    const int f = static_cast<int>(ws.v0[u]);
    const uint32_t r = p < 0 ? f + 1 : (f == p ? 0 : (f < p ? f + 1 : f));
    ws.rank_of_u[u] = r;
    double v = key_value(ws.uniq[u]);
    if (v == 0.0) v = ws.ctrl->pos_zero ? 0.0 : -0.0;  // np.unique keeps one zero
    if (r == 0 && bg_mode) v = bg_value;               // an explicit background heads omega as given
    ws.omega_freq[r] = v;
    ws.to_vpos[r] = u + ((p < 0 && bg_key < ws.uniq[u]) ? 1u : 0u);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && p < 0) {
    ws.omega_freq[0] = bg_value;
    ws.to_vpos[0] = lower_bound_u64(ws.uniq, k0, bg_key);
  }
}

__global__ void k_gen_mode(GenWs ws) { ws.ctrl->mode_index = static_cast<int>(ws.to_vpos[0]); }

template <typename T>
__global__ void k_gen_pairs(const T *__restrict__ w, int64_t m, int64_t n, int64_t ldw, GenWs ws) {
  const int64_t N = m * n;
  const uint32_t k0 = ws.ctrl->nrun;
  const uint64_t K = ws.ctrl->k;
  unsigned int local = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / n, c = i - r * n;
    const uint64_t key = value_key(static_cast<double>(w[r * ldw + c]));
    const uint32_t rank = ws.rank_of_u[lower_bound_u64(ws.uniq, k0, key)];
    if (rank) {
      ws.k0[i] = static_cast<uint64_t>(r) * K + rank;
      ws.v0[i] = static_cast<uint32_t>(c);
      ++local;
    } else {
      ws.k0[i] = ~0ull;
      ws.v0[i] = 0u;
    }
  }
  atomicAdd(&ws.ctrl->nnz, local);
}

__global__ void k_gen_widen(GenWs ws) {
  const uint32_t np = ws.ctrl->npair;
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x)
    ws.pair_end[p] = ws.pair_cnt[p];
}

__global__ void k_gen_rowstats(GenWs ws, int64_t m) {
  const uint32_t np = ws.ctrl->npair;
  const uint64_t K = ws.ctrl->k;
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x) {
    const uint64_t key = ws.pair_key[p];
    const uint64_t r = key / K, rank = key - r * K;
    atomicAdd(reinterpret_cast<unsigned long long *>(&ws.row_stat[r]), static_cast<unsigned long long>(ws.pair_cnt[p]));
    atomicMax(reinterpret_cast<unsigned long long *>(&ws.row_stat[m + r]), static_cast<unsigned long long>(rank));
    atomicAdd(reinterpret_cast<unsigned long long *>(&ws.row_stat[2 * m + r]), 1ull);
  }
}

// three exclusive scans over the rows + largest per-row values (one CTA; tiny next to the sorts)
__global__ void __launch_bounds__(1024) k_gen_scan_rows(int64_t m, GenWs ws) {
  __shared__ uint64_t part[3][1024];
  const int t = threadIdx.x;
  const int64_t per = ceil_div(m, 1024);
  const int64_t r0 = min64(m, t * per), r1 = min64(m, r0 + per);
  uint64_t s[3] = {0, 0, 0}, mx[3] = {0, 0, 0};
  for (int64_t r = r0; r < r1; ++r)
    for (int j = 0; j < 3; ++j) {
      s[j] += ws.row_stat[j * m + r];
      mx[j] = max(mx[j], ws.row_stat[j * m + r]);
    }
  for (int j = 0; j < 3; ++j) {
    part[j][t] = s[j];
    atomicMax(&ws.ctrl->max_stat[j], static_cast<unsigned long long>(mx[j]));
  }
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    uint64_t v[3];
    for (int j = 0; j < 3; ++j) v[j] = t >= o ? part[j][t - o] : 0;
    __syncthreads();
    for (int j = 0; j < 3; ++j) part[j][t] += v[j];
    __syncthreads();
  }
  uint64_t run[3];
  for (int j = 0; j < 3; ++j) run[j] = part[j][t] - s[j];
  for (int64_t r = r0; r < r1; ++r)
    for (int j = 0; j < 3; ++j) {
      ws.scan[j * (m + 1) + r] = run[j];
      run[j] += ws.row_stat[j * m + r];
    }
  if (t == 1023)
    for (int j = 0; j < 3; ++j) ws.scan[j * (m + 1) + m] = part[j][1023];
}

__global__ void k_gen_fill_col(GenWs ws, void *col, int col_bits) {
  const uint32_t nnz = ws.ctrl->nnz;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += gridDim.x * blockDim.x)
    store_index(col, col_bits, i, ws.v1[i]);
}

__global__ void k_gen_fill_segments(GenWs ws, int64_t m, bool cser, void *op, int op_bits, void *oi, int oi_bits) {
  const uint32_t np = ws.ctrl->npair;
  const uint64_t K = ws.ctrl->k;
  const uint64_t *rp_cer = ws.scan + (m + 1);
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x) {
    const uint64_t key = ws.pair_key[p];
    const uint64_t r = key / K, rank = key - r * K;
    if (cser) {
      store_index(oi, oi_bits, p, ws.to_vpos[rank]);
      store_index(op, op_bits, p + 1, ws.pair_end[p]);
    } else {
      store_index(op, op_bits, rp_cer[r] + rank, ws.pair_end[p]);  // segment rp_cer[r] + rank - 1 ends here
    }
  }
}

__global__ void k_gen_fill_tail(int64_t m, GenWs ws, bool cser, double *omega, void *row_ptr, int rp_bits) {
  const uint32_t k = ws.ctrl->k;
  const uint64_t *seg_scan = ws.scan + (cser ? 2 : 1) * (m + 1);
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = tid; i <= m; i += stride) store_index(row_ptr, rp_bits, i, seg_scan[i]);
  for (int64_t f = tid; f < k; f += stride) omega[cser ? ws.to_vpos[f] : f] = ws.omega_freq[f];
}

int grid_for(int64_t items) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(items, 256), int64_t(num_sms()) * 16)));
}

template <typename T>
int launch_keys(const void *w, int64_t m, int64_t n, int64_t ldw, const GenWs &ws, cudaStream_t st, bool pairs) {
  if (pairs)
    k_gen_pairs<T><<<grid_for(m * n), 256, 0, st>>>(static_cast<const T *>(w), m, n, ldw, ws);
  else
    k_gen_keys<T><<<grid_for(m * n), 256, 0, st>>>(static_cast<const T *>(w), m, n, ldw, ws);
  CERDOT_LAUNCH_CHECK();
  return CERDOT_OK;
}

template <typename U>
int max_scan_inplace(U *buf, int64_t items, const GenWs &ws, cudaStream_t st) {
  size_t tb = ws.tmp_bytes;
  CERDOT_CUDA_CHECK(cub::DeviceScan::InclusiveScan(ws.tmp, tb, buf, buf, cub::Max(), static_cast<int>(items), st));
  return CERDOT_OK;
}

int bits_for(uint64_t v) {
  int b = 1;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

}  // namespace

size_t encode_sort_workspace_bytes(int64_t m, int64_t n) { return gen_carve(nullptr, m, n).bytes; }

int encode_sort_plan(const void *w, int dtype, int64_t m, int64_t n, int64_t ldw, int bg_mode, double bg_value,
                     void *workspace, size_t workspace_bytes, cerdot_encode_info *info, cudaStream_t st) {
  const int64_t N = m * n;
  if (N >= (int64_t(1) << 31)) return fail(CERDOT_E_UNSUPPORTED, "sort path: matrix has >= 2^31 elements");
  const size_t need = encode_sort_workspace_bytes(m, n);
  info->workspace_bytes = need;
  info->path = 1;
  if (workspace == nullptr || workspace_bytes < need)
    return fail(CERDOT_E_WORKSPACE, "large alphabet: the sort-based conversion needs " + std::to_string(need) +
                                        " bytes of workspace");
  GenWs ws = gen_carve(workspace, m, n);
  CERDOT_CUDA_CHECK(cudaMemsetAsync(ws.ctrl, 0, sizeof(GenCtrl), st));
  CERDOT_CUDA_CHECK(cudaMemsetAsync(ws.row_stat, 0, sizeof(uint64_t) * 3 * m, st));
  int rc = dtype == CERDOT_F32 ? launch_keys<float>(w, m, n, ldw, ws, st, false)
                               : launch_keys<double>(w, m, n, ldw, ws, st, false);
  if (rc) return rc;
  size_t tb = ws.tmp_bytes;
  const int ni = static_cast<int>(N);
  CERDOT_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(ws.tmp, tb, ws.k0, ws.k1, ni, 0, 64, st));
  tb = ws.tmp_bytes;
  CERDOT_CUDA_CHECK(cub::DeviceRunLengthEncode::Encode(ws.tmp, tb, ws.k1, ws.uniq, ws.cnt, &ws.ctrl->nrun, ni, st));
  GenCtrl h{};
  CERDOT_CUDA_CHECK(cudaMemcpyAsync(&h, ws.ctrl, sizeof(GenCtrl), cudaMemcpyDeviceToHost, st));
  CERDOT_CUDA_CHECK(cudaStreamSynchronize(st));
  const int k0 = static_cast<int>(h.nrun);
  k_gen_negcount<<<grid_for(k0), 256, 0, st>>>(ws);
  CERDOT_LAUNCH_CHECK();
  tb = ws.tmp_bytes;
  CERDOT_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(ws.tmp, tb, ws.k0, ws.k1, ws.v0, ws.v1, k0, 0, 32, st));
  k_gen_freqpos<<<grid_for(k0), 256, 0, st>>>(ws);
  k_gen_background<<<1, 1, 0, st>>>(ws, bg_mode, bg_value);
  k_gen_ranks<<<grid_for(k0), 256, 0, st>>>(ws, bg_mode, bg_value);
  k_gen_mode<<<1, 1, 0, st>>>(ws);
  CERDOT_LAUNCH_CHECK();
  rc = dtype == CERDOT_F32 ? launch_keys<float>(w, m, n, ldw, ws, st, true)
                           : launch_keys<double>(w, m, n, ldw, ws, st, true);
  if (rc) return rc;
  CERDOT_CUDA_CHECK(cudaMemcpyAsync(&h, ws.ctrl, sizeof(GenCtrl), cudaMemcpyDeviceToHost, st));
  CERDOT_CUDA_CHECK(cudaStreamSynchronize(st));
  const int end_bit = std::min(64, bits_for(static_cast<uint64_t>(m) * h.k) + 1);
  tb = ws.tmp_bytes;
  // bits above end_bit are only set in the background sentinel ~0, which therefore still sorts last
  CERDOT_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(ws.tmp, tb, ws.k0, ws.k1, ws.v0, ws.v1, ni, 0, 64, st));
  (void)end_bit;
  const int nnz = static_cast<int>(h.nnz);
  tb = ws.tmp_bytes;
  CERDOT_CUDA_CHECK(
      cub::DeviceRunLengthEncode::Encode(ws.tmp, tb, ws.k1, ws.pair_key, ws.pair_cnt, &ws.ctrl->npair, nnz, st));
  CERDOT_CUDA_CHECK(cudaMemcpyAsync(&h, ws.ctrl, sizeof(GenCtrl), cudaMemcpyDeviceToHost, st));
  CERDOT_CUDA_CHECK(cudaStreamSynchronize(st));
  const int np = static_cast<int>(h.npair);
  k_gen_widen<<<grid_for(np), 256, 0, st>>>(ws);
  CERDOT_LAUNCH_CHECK();
  if (np > 0) {
    tb = ws.tmp_bytes;
    CERDOT_CUDA_CHECK(cub::DeviceScan::InclusiveSum(ws.tmp, tb, ws.pair_end, ws.pair_end, np, st));
  }
  k_gen_rowstats<<<grid_for(np), 256, 0, st>>>(ws, m);
  k_gen_scan_rows<<<1, 1024, 0, st>>>(m, ws);
  CERDOT_LAUNCH_CHECK();
  uint64_t totals[3];
  for (int j = 0; j < 3; ++j)
    CERDOT_CUDA_CHECK(
        cudaMemcpyAsync(&totals[j], ws.scan + j * (m + 1) + m, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  CERDOT_CUDA_CHECK(cudaMemcpyAsync(&h, ws.ctrl, sizeof(GenCtrl), cudaMemcpyDeviceToHost, st));
  double bg = 0.0;
  CERDOT_CUDA_CHECK(cudaMemcpyAsync(&bg, ws.omega_freq, sizeof(double), cudaMemcpyDeviceToHost, st));
  CERDOT_CUDA_CHECK(cudaStreamSynchronize(st));
  info->k = h.k;
  info->nnz = static_cast<int64_t>(totals[0]);
  info->segments_cer = static_cast<int64_t>(totals[1]);
  info->segments_cser = static_cast<int64_t>(totals[2]);
  info->mode_index = h.mode_index;
  info->background = bg;
  info->max_row_nnz = static_cast<int64_t>(h.max_stat[0]);
  info->max_row_segments_cer = static_cast<int64_t>(h.max_stat[1]);
  info->max_row_segments_cser = static_cast<int64_t>(h.max_stat[2]);
  if (info->segments_cer >= (int64_t(1) << 31))
    return fail(CERDOT_E_UNSUPPORTED, "sort path: more than 2^31 CER segments");
  return CERDOT_OK;
}

int encode_sort_fill(const cerdot_encode_info *info, int kind, void *workspace, size_t workspace_bytes, double *omega,
                     void *col, int col_bits, void *op, int op_bits, void *rp, int rp_bits, void *oi, int oi_bits,
                     cudaStream_t st) {
  const int64_t m = info->m, n = info->n;
  if (workspace == nullptr || workspace_bytes < encode_sort_workspace_bytes(m, n))
    return fail(CERDOT_E_WORKSPACE, "encode workspace too small");
  GenWs ws = gen_carve(workspace, m, n);
  const bool cser = kind == CERDOT_CSER;
  const int64_t segs = cser ? info->segments_cser : info->segments_cer;
  if (info->nnz) k_gen_fill_col<<<grid_for(info->nnz), 256, 0, st>>>(ws, col, col_bits);
  if (!cser) CERDOT_CUDA_CHECK(cudaMemsetAsync(op, 0, static_cast<size_t>(segs + 1) * (op_bits / 8), st));
  k_gen_fill_segments<<<grid_for(std::max<int64_t>(1, segs)), 256, 0, st>>>(ws, m, cser, op, op_bits, oi, oi_bits);
  CERDOT_LAUNCH_CHECK();
  if (cser) {
    CERDOT_CUDA_CHECK(cudaMemsetAsync(op, 0, op_bits / 8, st));  // omegaPtr[0] = 0
  } else if (segs > 0) {  // empty padding segments take the previous end (ends are non-decreasing)
    int rc;
    switch (op_bits) {
      case 8: rc = max_scan_inplace(static_cast<uint8_t *>(op), segs + 1, ws, st); break;
      case 16: rc = max_scan_inplace(static_cast<uint16_t *>(op), segs + 1, ws, st); break;
      default: rc = max_scan_inplace(static_cast<uint32_t *>(op), segs + 1, ws, st); break;
    }
    if (rc) return rc;
  }
  k_gen_fill_tail<<<grid_for(m + 1), 256, 0, st>>>(m, ws, cser, omega, rp, rp_bits);
  CERDOT_LAUNCH_CHECK();
  return CERDOT_OK;
}

}  // namespace cerdot
