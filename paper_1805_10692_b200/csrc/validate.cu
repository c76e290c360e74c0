// Device validate / decode of CER and CSER encodings (sm_100a).
//
// Reference: lemt.formats.validate (formats.py:298-392) and decode (formats.py:395-424).  validate runs
// the reference's structural checks in its order and reports the FIRST violation; every check is a
// data-parallel pass whose violating positions are reduced with atomicMin, so the device finds the
// same (array, offset) the reference's np.nonzero(...)[0] picks.  Checks that need only the tiny
// alphabet (duplicate / unsorted omega, mode_index range) and array lengths are the host's
// (paper_1805_10692_b200/formats.py); this file covers the index arrays.
//
//   phase 1  omegaPtr / rowPtr monotone and their end values          (k_ends, k_monotone)
//   phase 2  (pointers valid) colI in range, strictly ascending inside a segment (segment-head marks),
//            unique per row (per-row 2-bit column bitmaps), CER rows <= k-1 segments and no trailing
//            empty segment, CSER omegaI in range / not the background / segments non-empty / unique
//            per row.
// A duplicate is reported as the reference does: the second occurrence (index order) of the smallest
// duplicated (row, column) key -- or (row, element) key for omegaI.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "encode.cuh"

namespace cerdot {

namespace {

constexpr unsigned long long kNone = ~0ull;
constexpr int kDupThreads = 256;

struct VState {
  unsigned long long first[CERDOT_CHECK_COUNT];  // smallest violating position per check
  unsigned long long ends[4];                    // omegaPtr[0], omegaPtr[segs], rowPtr[0], rowPtr[m]
};

__global__ void k_vinit(VState *v) {
  for (int i = threadIdx.x; i < CERDOT_CHECK_COUNT; i += blockDim.x) v->first[i] = kNone;
}

__global__ void k_ends(const void *op, int op_bits, int64_t segs, const void *rp, int rp_bits, int64_t m,
                       VState *v) {
  if (threadIdx.x == 0) {
    v->ends[0] = load_index(op, op_bits, 0);
    v->ends[1] = load_index(op, op_bits, segs);
    v->ends[2] = load_index(rp, rp_bits, 0);
    v->ends[3] = load_index(rp, rp_bits, m);
  }
}

// first i >= 1 with a[i] < a[i-1]
__global__ void k_monotone(const void *a, int bits, int64_t len, unsigned long long *slot) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x + 1; i < len;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (load_index(a, bits, i) < load_index(a, bits, i - 1)) atomicMin(slot, static_cast<unsigned long long>(i));
}

__global__ void k_mark_heads(const void *op, int op_bits, int64_t segs, int64_t nnz, unsigned char *head) {
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < segs;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t e = load_index(op, op_bits, s);
    if (e < nnz) head[e] = 1;
  }
}

// colI range and in-segment order
__global__ void k_columns(const void *col, int col_bits, int64_t nnz, int64_t n, const unsigned char *head,
                          VState *v) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nnz;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t c = load_index(col, col_bits, i);
    if (c >= n) atomicMin(&v->first[CERDOT_CHECK_COL_RANGE], static_cast<unsigned long long>(i));
    if (i > 0 && !head[i] && c <= load_index(col, col_bits, i - 1))
      atomicMin(&v->first[CERDOT_CHECK_COL_ORDER], static_cast<unsigned long long>(i));
  }
}

// Per-row duplicate keys: CTA per row (grid-stride), a 2-bit-per-key bitmap in global scratch per CTA
// (seen, repeated).  Item j of row r is position base(r) + j of `vals` (colI entries of the row, or
// omegaI of its segments); keys >= width are ignored (reported by the range checks).  Reports
// (row << 32 | second occurrence of the smallest repeated key) -- rows ordered first, like the
// reference's stable argsort of row * width + key.
__global__ void __launch_bounds__(kDupThreads) k_row_dups(const void *vals, int val_bits, const void *op, int op_bits,
                                                          const void *rp, int rp_bits, int64_t m, int64_t width,
                                                          bool entries, uint32_t *scratch, int64_t words,
                                                          unsigned long long *slot) {
  __shared__ unsigned int s_key, s_first, s_second;
  uint32_t *bm = scratch + static_cast<int64_t>(blockIdx.x) * words;
  for (int64_t r = blockIdx.x; r < m; r += gridDim.x) {
    const uint32_t s0 = load_index(rp, rp_bits, r), s1 = load_index(rp, rp_bits, r + 1);
    const uint32_t b0 = entries ? load_index(op, op_bits, s0) : s0;
    const uint32_t b1 = entries ? load_index(op, op_bits, s1) : s1;
    for (int64_t w = threadIdx.x; w < words; w += blockDim.x) bm[w] = 0u;
    if (threadIdx.x == 0) {
      s_key = 0xffffffffu;
      s_first = 0xffffffffu;
      s_second = 0xffffffffu;
    }
    __syncthreads();
    for (uint32_t j = b0 + threadIdx.x; j < b1; j += blockDim.x) {
      const uint32_t key = load_index(vals, val_bits, j);
      if (key >= width) continue;
      const uint32_t bit = 1u << (2u * (key & 15u));
      const uint32_t old = atomicOr(&bm[key >> 4], bit);
      if (old & bit) atomicOr(&bm[key >> 4], bit << 1);
    }
    __syncthreads();
    for (int64_t w = threadIdx.x; w < words; w += blockDim.x) {
      const uint32_t rep = bm[w] & 0xaaaaaaaau;
      if (rep) atomicMin(&s_key, static_cast<unsigned int>(w * 16 + (__ffs(rep) - 1) / 2));
    }
    __syncthreads();
    const uint32_t key = s_key;
    if (key != 0xffffffffu) {
      for (uint32_t j = b0 + threadIdx.x; j < b1; j += blockDim.x)
        if (load_index(vals, val_bits, j) == key) atomicMin(&s_first, j);
      __syncthreads();
      for (uint32_t j = b0 + threadIdx.x; j < b1; j += blockDim.x)
        if (j != s_first && load_index(vals, val_bits, j) == key) atomicMin(&s_second, j);
      __syncthreads();
      if (threadIdx.x == 0) atomicMin(slot, (static_cast<unsigned long long>(r) << 32) | s_second);
    }
    __syncthreads();
  }
}

// CER: rows hold <= k-1 segments; no row ends with an empty (padding) segment
__global__ void k_cer_rows(const void *op, int op_bits, const void *rp, int rp_bits, int64_t m, int64_t k,
                           VState *v) {
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < m;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t s0 = load_index(rp, rp_bits, r), s1 = load_index(rp, rp_bits, r + 1);
    if (s1 - s0 > k - 1) atomicMin(&v->first[CERDOT_CHECK_CER_ROW_SEGMENTS], static_cast<unsigned long long>(r));
    if (s1 > s0 && load_index(op, op_bits, s1) == load_index(op, op_bits, s1 - 1))
      atomicMin(&v->first[CERDOT_CHECK_CER_TRAILING_EMPTY], static_cast<unsigned long long>(s1 - 1));
  }
}

// CSER: omegaI in range and not the background; no empty segment
__global__ void k_cser_segs(const void *oi, int oi_bits, const void *op, int op_bits, int64_t segs, int64_t k,
                            int64_t mode, VState *v) {
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < segs;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t o = load_index(oi, oi_bits, s);
    if (o >= k) atomicMin(&v->first[CERDOT_CHECK_OI_RANGE], static_cast<unsigned long long>(s));
    if (o == mode) atomicMin(&v->first[CERDOT_CHECK_OI_BACKGROUND], static_cast<unsigned long long>(s));
    if (load_index(op, op_bits, s + 1) == load_index(op, op_bits, s))
      atomicMin(&v->first[CERDOT_CHECK_EMPTY_SEGMENT], static_cast<unsigned long long>(s));
  }
}

int grid_for(int64_t items) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(items, 256), int64_t(num_sms()) * 8)));
}

// decode: background fill, then each row's segments scattered (CTA per row, thread per segment)
__global__ void k_decode_fill(double *out, int64_t m, int64_t n, int64_t ldo, double bg) {
  const int64_t total = m * n;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / n;
    out[r * ldo + (i - r * n)] = bg;
  }
}

__global__ void k_decode_scatter(cerdot_matrix a, double *out, int64_t ldo) {
  const bool cser = a.kind == CERDOT_CSER;
  for (int64_t r = blockIdx.x; r < a.m; r += gridDim.x) {
    const uint32_t s0 = load_index(a.row_ptr, a.row_ptr_bits, r), s1 = load_index(a.row_ptr, a.row_ptr_bits, r + 1);
    for (uint32_t s = s0 + threadIdx.x; s < s1; s += blockDim.x) {
      const int64_t kk = cser ? static_cast<int64_t>(load_index(a.omega_index, a.omega_index_bits, s)) : (s - s0 + 1);
      const double val = a.omega[kk];
      const uint32_t e0 = load_index(a.omega_ptr, a.omega_ptr_bits, s), e1 = load_index(a.omega_ptr, a.omega_ptr_bits, s + 1);
      for (uint32_t e = e0; e < e1; ++e) out[r * ldo + load_index(a.col_index, a.col_bits, e)] = val;
    }
  }
}

// Trace counts (kernels.py:175-234 inputs) over all rows: segments, non-empty segments, entries,
// rows with segments, sum over rows of max(non-empty - 1, 0).  Thread per row; integer atomics.
__global__ void k_trace_counts(cerdot_matrix a, unsigned long long *out) {
  unsigned long long c[5] = {0, 0, 0, 0, 0};
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < a.m;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t s0 = load_index(a.row_ptr, a.row_ptr_bits, r), s1 = load_index(a.row_ptr, a.row_ptr_bits, r + 1);
    uint32_t ne = 0, prev = load_index(a.omega_ptr, a.omega_ptr_bits, s0);
    const uint32_t first = prev;
    for (uint32_t s = s0; s < s1; ++s) {
      const uint32_t nxt = load_index(a.omega_ptr, a.omega_ptr_bits, s + 1);
      ne += nxt > prev;
      prev = nxt;
    }
    c[0] += s1 - s0;
    c[1] += ne;
    c[2] += prev - first;
    c[3] += s1 > s0;
    c[4] += ne > 0 ? ne - 1 : 0;
  }
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    unsigned long long v = c[i];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(out + i, v);
  }
}

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

int64_t dup_grid(int64_t m) { return std::max<int64_t>(1, std::min<int64_t>(m, int64_t(num_sms()) * 2)); }

}  // namespace

size_t validate_workspace_bytes(const cerdot_matrix *a) {
  const int64_t width = std::max<int64_t>(a->n, a->k);
  const int64_t words = ceil_div(std::max<int64_t>(width, 1), 16);
  return align256(sizeof(VState)) + align256(static_cast<size_t>(std::max<int64_t>(a->nnz, 1))) +
         static_cast<size_t>(dup_grid(a->m)) * static_cast<size_t>(words) * 4;
}

int validate(const cerdot_matrix *a, cerdot_format_error *err, void *workspace, size_t workspace_bytes,
             cudaStream_t st) {
  if (workspace == nullptr || workspace_bytes < validate_workspace_bytes(a))
    return fail(CERDOT_E_WORKSPACE, "validate workspace too small");
  err->check = CERDOT_CHECK_NONE;
  err->offset = 0;
  err->value = 0;
  char *ws = static_cast<char *>(workspace);
  VState *dv = reinterpret_cast<VState *>(ws);
  unsigned char *head = reinterpret_cast<unsigned char *>(ws + align256(sizeof(VState)));
  uint32_t *scratch = reinterpret_cast<uint32_t *>(ws + align256(sizeof(VState)) +
                                                   align256(static_cast<size_t>(std::max<int64_t>(a->nnz, 1))));
  const int64_t segs = a->segments, m = a->m;
  VState hv;
  auto fetch = [&]() -> int {
    CERDOT_CUDA_CHECK(cudaMemcpyAsync(&hv, dv, sizeof(VState), cudaMemcpyDeviceToHost, st));
    CERDOT_CUDA_CHECK(cudaStreamSynchronize(st));
    return CERDOT_OK;
  };
  auto report = [&](int check, int64_t offset, int64_t value) {
    err->check = check;
    err->offset = offset;
    err->value = value;
    return CERDOT_OK;
  };
  // ---- phase 1: the pointer arrays
  k_vinit<<<1, 32, 0, st>>>(dv);
  k_ends<<<1, 32, 0, st>>>(a->omega_ptr, a->omega_ptr_bits, segs, a->row_ptr, a->row_ptr_bits, m, dv);
  k_monotone<<<grid_for(segs + 1), 256, 0, st>>>(a->omega_ptr, a->omega_ptr_bits, segs + 1,
                                                 &dv->first[CERDOT_CHECK_PTR_ORDER]);
  k_monotone<<<grid_for(m + 1), 256, 0, st>>>(a->row_ptr, a->row_ptr_bits, m + 1,
                                              &dv->first[CERDOT_CHECK_ROW_ORDER]);
  CERDOT_LAUNCH_CHECK();
  if (int rc = fetch()) return rc;
  if (hv.ends[0] != 0) return report(CERDOT_CHECK_PTR_START, 0, static_cast<int64_t>(hv.ends[0]));
  if (hv.first[CERDOT_CHECK_PTR_ORDER] != kNone)
    return report(CERDOT_CHECK_PTR_ORDER, static_cast<int64_t>(hv.first[CERDOT_CHECK_PTR_ORDER]), 0);
  if (static_cast<int64_t>(hv.ends[1]) != a->nnz) return report(CERDOT_CHECK_PTR_END, segs, static_cast<int64_t>(hv.ends[1]));
  if (hv.ends[2] != 0) return report(CERDOT_CHECK_ROW_START, 0, static_cast<int64_t>(hv.ends[2]));
  if (hv.first[CERDOT_CHECK_ROW_ORDER] != kNone)
    return report(CERDOT_CHECK_ROW_ORDER, static_cast<int64_t>(hv.first[CERDOT_CHECK_ROW_ORDER]), 0);
  if (static_cast<int64_t>(hv.ends[3]) != segs) return report(CERDOT_CHECK_ROW_END, m, static_cast<int64_t>(hv.ends[3]));

  // ---- phase 2: pointers are monotone from 0 to their ends, every derived index below is in range
  CERDOT_CUDA_CHECK(cudaMemsetAsync(head, 0, static_cast<size_t>(std::max<int64_t>(a->nnz, 1)), st));
  k_mark_heads<<<grid_for(segs), 256, 0, st>>>(a->omega_ptr, a->omega_ptr_bits, segs, a->nnz, head);
  k_columns<<<grid_for(a->nnz), 256, 0, st>>>(a->col_index, a->col_bits, a->nnz, a->n, head, dv);
  const int64_t g = dup_grid(m);
  k_row_dups<<<static_cast<int>(g), kDupThreads, 0, st>>>(a->col_index, a->col_bits, a->omega_ptr, a->omega_ptr_bits,
                                                          a->row_ptr, a->row_ptr_bits, m, a->n, true, scratch,
                                                          ceil_div(std::max<int64_t>(a->n, 1), 16),
                                                          &dv->first[CERDOT_CHECK_COL_DUPLICATE]);
  if (a->kind == CERDOT_CER) {
    k_cer_rows<<<grid_for(m), 256, 0, st>>>(a->omega_ptr, a->omega_ptr_bits, a->row_ptr, a->row_ptr_bits, m, a->k, dv);
  } else {
    k_cser_segs<<<grid_for(segs), 256, 0, st>>>(a->omega_index, a->omega_index_bits, a->omega_ptr, a->omega_ptr_bits,
                                                segs, a->k, a->mode_index, dv);
    k_row_dups<<<static_cast<int>(g), kDupThreads, 0, st>>>(a->omega_index, a->omega_index_bits, nullptr, 0,
                                                            a->row_ptr, a->row_ptr_bits, m, a->k, false, scratch,
                                                            ceil_div(std::max<int64_t>(a->k, 1), 16),
                                                            &dv->first[CERDOT_CHECK_OI_DUPLICATE]);
  }
  CERDOT_LAUNCH_CHECK();
  if (int rc = fetch()) return rc;
  for (int c = CERDOT_CHECK_COL_RANGE; c < CERDOT_CHECK_COUNT; ++c) {
    const unsigned long long f = hv.first[c];
    if (f == kNone) continue;
    int64_t off = static_cast<int64_t>(f), value = 0;
    if (c == CERDOT_CHECK_COL_DUPLICATE || c == CERDOT_CHECK_OI_DUPLICATE) off = static_cast<int64_t>(f & 0xffffffffull);
    if (c == CERDOT_CHECK_COL_RANGE) {
      uint32_t v32 = 0;
      const int bytes = a->col_bits / 8;
      CERDOT_CUDA_CHECK(cudaMemcpyAsync(&v32, static_cast<const char *>(a->col_index) + off * bytes, bytes,
                                        cudaMemcpyDeviceToHost, st));
      CERDOT_CUDA_CHECK(cudaStreamSynchronize(st));
      value = v32;
    }
    if (c == CERDOT_CHECK_CER_ROW_SEGMENTS) {  // offset = row + 1 (the rowPtr entry that closes the row)
      uint32_t pair[2] = {0, 0};
      const int bytes = a->row_ptr_bits / 8;
      unsigned char raw[8] = {0};
      CERDOT_CUDA_CHECK(cudaMemcpyAsync(raw, static_cast<const char *>(a->row_ptr) + off * bytes, 2 * bytes,
                                        cudaMemcpyDeviceToHost, st));
      CERDOT_CUDA_CHECK(cudaStreamSynchronize(st));
      for (int i = 0; i < 2; ++i) {
        uint32_t x = 0;
        for (int b = 0; b < bytes; ++b) x |= static_cast<uint32_t>(raw[i * bytes + b]) << (8 * b);
        pair[i] = x;
      }
      value = static_cast<int64_t>(pair[1]) - pair[0];
      off += 1;
    }
    if (c == CERDOT_CHECK_CER_TRAILING_EMPTY || c == CERDOT_CHECK_EMPTY_SEGMENT) off += 1;  // omegaPtr entry
    return report(c, off, value);
  }
  return CERDOT_OK;
}

int trace_counts(const cerdot_matrix *a, uint64_t *counts, void *workspace, cudaStream_t st) {
  unsigned long long *d = static_cast<unsigned long long *>(workspace);
  CERDOT_CUDA_CHECK(cudaMemsetAsync(d, 0, 5 * sizeof(unsigned long long), st));
  if (a->m > 0) {
    k_trace_counts<<<grid_for(a->m), 256, 0, st>>>(*a, d);
    CERDOT_LAUNCH_CHECK();
  }
  CERDOT_CUDA_CHECK(cudaMemcpyAsync(counts, d, 5 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CERDOT_CUDA_CHECK(cudaStreamSynchronize(st));
  return CERDOT_OK;
}

int decode(const cerdot_matrix *a, double *out, int64_t ldo, cudaStream_t st) {
  if (a->m == 0 || a->n == 0) return CERDOT_OK;
  k_decode_fill<<<grid_for(a->m * a->n), 256, 0, st>>>(out, a->m, a->n, ldo, a->background);
  k_decode_scatter<<<static_cast<int>(std::min<int64_t>(a->m, int64_t(num_sms()) * 8)), 128, 0, st>>>(*a, out, ldo);
  CERDOT_LAUNCH_CHECK();
  return CERDOT_OK;
}

}  // namespace cerdot
