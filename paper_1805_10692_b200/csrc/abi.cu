// extern "C" entry points of libcerdot (declared in include/cerdot.h).
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "cerdot.h"
#include "common.cuh"
#include "encode.cuh"
#include "tileview.cuh"

#include <atomic>

namespace cerdot {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int status, const std::string &msg) {
  g_last_error = msg;
  return status;
}

int cuda_fail(cudaError_t err, const char *where) {
  g_last_error = std::string("CUDA error ") + cudaGetErrorName(err) + " (" + cudaGetErrorString(err) + ") in " + where;
  return CERDOT_E_CUDA;
}

int num_sms() {
  // per-device cache (the only mutable state in the library)
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev] = v;
  }
  return cache[dev];
}

static bool valid_bits(int b) { return b == 8 || b == 16 || b == 32; }

// formats.py:66-71 — width check with the reference's messages
static int check_width(int bits, uint64_t max_value) {
  if (!valid_bits(bits)) return fail(CERDOT_E_VALUE, "index bits must be one of (8, 16, 32)");
  if (bits < 64 && (max_value >> bits) != 0)
    return fail(CERDOT_E_VALUE, "index value " + std::to_string(max_value) + " does not fit in " +
                                    std::to_string(bits) + " bits");
  return CERDOT_OK;
}

static int check_matrix(const cerdot_matrix *a, int64_t batch, const float *x, const float *y, int64_t ldx,
                        int64_t ldy) {
  if (a == nullptr) return fail(CERDOT_E_TYPE, "not an encoded matrix: NULL");
  if (a->kind != CERDOT_CER && a->kind != CERDOT_CSER)
    return fail(CERDOT_E_TYPE, "not a CER/CSER matrix: kind " + std::to_string(a->kind));
  if (!valid_bits(a->col_bits) || !valid_bits(a->omega_ptr_bits) || !valid_bits(a->row_ptr_bits) ||
      (a->kind == CERDOT_CSER && !valid_bits(a->omega_index_bits)))
    return fail(CERDOT_E_VALUE, "index bits must be one of (8, 16, 32)");
  if (batch < 0) return fail(CERDOT_E_VALUE, "batch must be >= 0");
  if (batch > 1 && (ldx < batch || ldy < batch)) return fail(CERDOT_E_VALUE, "row strides must be >= batch");
  // the mat-vec kernels read x and write y contiguously: a strided single column must be made contiguous
  if (batch == 1 && (ldx != 1 || ldy != 1)) return fail(CERDOT_E_VALUE, "batch 1 needs unit row strides");
  if (a->m > 0 && batch > 0 && (x == nullptr || y == nullptr)) return fail(CERDOT_E_VALUE, "null x or y");
  return CERDOT_OK;
}

static std::atomic<int> g_paths[CERDOT_PATH_COUNT];

int kernel_path(int op) { return (op >= 0 && op < CERDOT_PATH_COUNT) ? g_paths[op].load(std::memory_order_relaxed) : 0; }

}  // namespace cerdot

using namespace cerdot;

extern "C" {

int cerdot_abi_version(void) { return CERDOT_ABI_VERSION; }

const char *cerdot_last_error(void) { return g_last_error.c_str(); }

int32_t cerdot_index_bitwidth(int64_t max_value) {
  if (max_value < 0) {
    fail(CERDOT_E_VALUE, "index values are unsigned");
    return 0;
  }
  for (int bits : {8, 16, 32})
    if ((static_cast<uint64_t>(max_value) >> bits) == 0) return bits;
  fail(CERDOT_E_VALUE, "index value " + std::to_string(max_value) + " does not fit in 32 bits");
  return 0;
}

size_t cerdot_encode_workspace_bytes(int64_t m, int64_t n) {
  if (m <= 0 || n <= 0) return 0;
  return encode_workspace_bytes(m, n);
}

int cerdot_encode_plan(const void *w, int32_t dtype, int64_t m, int64_t n, int64_t ldw, int32_t bg_mode,
                       double bg_value, void *workspace, size_t workspace_bytes, cerdot_encode_info *info,
                       void *stream) {
  if (info == nullptr) return fail(CERDOT_E_VALUE, "info must not be NULL");
  *info = cerdot_encode_info{};
  if (m > 0 && n > 0 && w == nullptr) return fail(CERDOT_E_VALUE, "w must not be NULL");
  return encode_plan(w, dtype, m, n, ldw, bg_mode, bg_value, workspace, workspace_bytes, info,
                     static_cast<cudaStream_t>(stream));
}

int cerdot_encode_fill(const cerdot_encode_info *info, int32_t kind, void *workspace, size_t workspace_bytes,
                       double *omega, void *col_index, int32_t col_bits, void *omega_ptr, int32_t omega_ptr_bits,
                       void *row_ptr, int32_t row_ptr_bits, void *omega_index, int32_t omega_index_bits,
                       void *stream) {
  if (info == nullptr) return fail(CERDOT_E_VALUE, "info must not be NULL");
  if (kind != CERDOT_CER && kind != CERDOT_CSER) return fail(CERDOT_E_TYPE, "kind must be CER or CSER");
  const bool cser = kind == CERDOT_CSER;
  const int64_t segs = cser ? info->segments_cser : info->segments_cer;
  int rc;
  // the reference narrows in this order: colI, [omegaI], omegaPtr, rowPtr (formats.py:249-252, 286-290)
  if ((rc = check_width(col_bits, static_cast<uint64_t>(info->n > 0 ? info->n - 1 : 0)))) return rc;
  if (cser && (rc = check_width(omega_index_bits, static_cast<uint64_t>(info->k > 0 ? info->k - 1 : 0)))) return rc;
  if ((rc = check_width(omega_ptr_bits, static_cast<uint64_t>(info->nnz)))) return rc;
  if ((rc = check_width(row_ptr_bits, static_cast<uint64_t>(segs)))) return rc;
  if (omega == nullptr || omega_ptr == nullptr || row_ptr == nullptr || (info->nnz > 0 && col_index == nullptr) ||
      (cser && segs > 0 && omega_index == nullptr))
    return fail(CERDOT_E_VALUE, "null output buffer");
  return encode_fill(info, kind, workspace, workspace_bytes, omega, col_index, col_bits, omega_ptr, omega_ptr_bits,
                     row_ptr, row_ptr_bits, omega_index, omega_index_bits, static_cast<cudaStream_t>(stream));
}

static size_t align256(size_t v) { return (v + 255) / 256 * 256; }

size_t cerdot_dot_workspace_bytes(const cerdot_matrix *a, int64_t batch) {
  if (a == nullptr || batch <= 0) return 0;
  // column sums, plus 16 row-range partials per column for batch > 1 (dot.cu: kColsumSplit), 256 B
  // aligned; then the tiled mat-mat's tile-split partial products (tileview.cu)
  const size_t cs = a->background != 0.0 ? sizeof(double) * static_cast<size_t>(batch) * (batch > 1 ? 17 : 1) : 0;
  const size_t part = cerdot::tile_view_dot_workspace_bytes(a, batch);
  return part ? align256(cs) + part : cs;
}

size_t cerdot_validate_workspace_bytes(const cerdot_matrix *a) {
  return a ? cerdot::validate_workspace_bytes(a) : 0;
}

int cerdot_validate(const cerdot_matrix *a, cerdot_format_error *err, void *workspace, size_t workspace_bytes,
                    void *stream) {
  if (a == nullptr || err == nullptr) return fail(CERDOT_E_VALUE, "validate: null matrix or error record");
  if (a->m < 0 || a->n < 0 || a->k < 0 || a->nnz < 0 || a->segments < 0)
    return fail(CERDOT_E_VALUE, "validate: negative sizes");
  int rc = cerdot::validate(a, err, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
  if (rc) return rc;
  return err->check == CERDOT_CHECK_NONE ? CERDOT_OK : fail(CERDOT_E_FORMAT, "structural violation (see the error record)");
}

int cerdot_decode(const cerdot_matrix *a, double *out, int64_t ldo, void *stream) {
  if (a == nullptr || out == nullptr || ldo < a->n) return fail(CERDOT_E_VALUE, "decode: bad output");
  return cerdot::decode(a, out, ldo, static_cast<cudaStream_t>(stream));
}

int cerdot_trace_counts(const cerdot_matrix *a, uint64_t *counts, void *workspace, void *stream) {
  if (a == nullptr || counts == nullptr || workspace == nullptr) return fail(CERDOT_E_VALUE, "trace_counts: null");
  return cerdot::trace_counts(a, counts, workspace, static_cast<cudaStream_t>(stream));
}

int cerdot_lemx_unpack(const void *payload, int32_t element_bits, int64_t k, int64_t omega_offset, double *omega,
                       const int64_t *spans, int32_t count, void *arena, void *stream) {
  if (payload == nullptr || omega == nullptr || (count > 0 && (spans == nullptr || arena == nullptr)))
    return fail(CERDOT_E_VALUE, "lemx_unpack: null buffer");
  return cerdot::lemx_unpack(payload, element_bits, k, omega_offset, omega, spans, count, arena,
                             static_cast<cudaStream_t>(stream));
}

int cerdot_dot_peers(const cerdot_matrix *a, const float *x, int64_t ldx, int64_t batch, float *y, int64_t ldy,
                     float *const *peers, int32_t npeers, int64_t peer_offset, void *workspace,
                     size_t workspace_bytes, void *stream) {
  int rc = check_matrix(a, batch, x, y, ldx, ldy);
  if (rc) return rc;
  if (npeers < 0 || (npeers > 0 && peers == nullptr) || peer_offset < 0)
    return fail(CERDOT_E_VALUE, "dot_peers: need a device array of npeers >= 0 peer output pointers");
  return cerdot::dot(a, x, ldx, batch, y, ldy, workspace, workspace_bytes, static_cast<cudaStream_t>(stream), peers,
                     npeers, peer_offset);
}

int cerdot_dot(const cerdot_matrix *a, const float *x, int64_t ldx, int64_t batch, float *y, int64_t ldy,
               void *workspace, size_t workspace_bytes, void *stream) {
  int rc = check_matrix(a, batch, x, y, ldx, ldy);
  if (rc) return rc;
  return cerdot::dot(a, x, ldx, batch, y, ldy, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
}

int cerdot_dot_cer(const cerdot_matrix *a, const float *x, int64_t ldx, int64_t batch, float *y, int64_t ldy,
                   void *workspace, size_t workspace_bytes, void *stream) {
  if (a != nullptr && a->kind != CERDOT_CER) return fail(CERDOT_E_TYPE, "dot_cer needs a CER matrix");
  return cerdot_dot(a, x, ldx, batch, y, ldy, workspace, workspace_bytes, stream);
}

int cerdot_dot_cser(const cerdot_matrix *a, const float *x, int64_t ldx, int64_t batch, float *y, int64_t ldy,
                    void *workspace, size_t workspace_bytes, void *stream) {
  if (a != nullptr && a->kind != CERDOT_CSER) return fail(CERDOT_E_TYPE, "dot_cser needs a CSER matrix");
  return cerdot_dot(a, x, ldx, batch, y, ldy, workspace, workspace_bytes, stream);
}


size_t cerdot_dot_host_workspace_bytes(const cerdot_matrix *a, int64_t batch) {
  if (a == nullptr || batch <= 0) return 0;
  const size_t b = static_cast<size_t>(batch);
  return align256(static_cast<size_t>(a->n) * b * 4) + align256(static_cast<size_t>(a->m) * b * 4) +
         align256(cerdot_dot_workspace_bytes(a, batch) + 1);
}

int cerdot_dot_host(const cerdot_matrix *a, const float *x_host, int64_t ldx, int64_t batch, float *y_host,
                    int64_t ldy, void *workspace, size_t workspace_bytes, void *stream) {
  int rc = check_matrix(a, batch, x_host, y_host, ldx, ldy);
  if (rc) return rc;
  if (a->m == 0 || batch == 0) return CERDOT_OK;
  if (workspace == nullptr || workspace_bytes < cerdot_dot_host_workspace_bytes(a, batch))
    return fail(CERDOT_E_WORKSPACE, "dot_host workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t b = static_cast<size_t>(batch);
  char *base = static_cast<char *>(workspace);
  float *dx = reinterpret_cast<float *>(base);
  float *dy = reinterpret_cast<float *>(base + align256(static_cast<size_t>(a->n) * b * 4));
  char *dws = reinterpret_cast<char *>(dy) + align256(static_cast<size_t>(a->m) * b * 4);
  const size_t xrow = b * 4, yrow = b * 4;
  if (batch == 1 || ldx == batch)
    CERDOT_CUDA_CHECK(cudaMemcpyAsync(dx, x_host, static_cast<size_t>(a->n) * xrow, cudaMemcpyHostToDevice, st));
  else
    CERDOT_CUDA_CHECK(cudaMemcpy2DAsync(dx, xrow, x_host, static_cast<size_t>(ldx) * 4, xrow, a->n,
                                        cudaMemcpyHostToDevice, st));
  rc = cerdot::dot(a, dx, batch == 1 ? 1 : batch, batch, dy, batch == 1 ? 1 : batch, dws,
                   cerdot_dot_workspace_bytes(a, batch), st);
  if (rc) return rc;
  if (batch == 1 || ldy == batch)
    CERDOT_CUDA_CHECK(cudaMemcpyAsync(y_host, dy, static_cast<size_t>(a->m) * yrow, cudaMemcpyDeviceToHost, st));
  else
    CERDOT_CUDA_CHECK(cudaMemcpy2DAsync(y_host, static_cast<size_t>(ldy) * 4, dy, yrow, yrow, a->m,
                                        cudaMemcpyDeviceToHost, st));
  CERDOT_CUDA_CHECK(cudaStreamSynchronize(st));
  return CERDOT_OK;
}

static uint64_t host_index(const void *p, int bits, int64_t i) {
  switch (bits) {
    case 8: return static_cast<const uint8_t *>(p)[i];
    case 16: return static_cast<const uint16_t *>(p)[i];
    default: return static_cast<const uint32_t *>(p)[i];
  }
}

int cerdot_row_entries(const cerdot_matrix *a, uint32_t *out, void *stream) {
  int rc = check_matrix(a, 0, nullptr, nullptr, 0, 0);
  if (rc) return rc;
  if (a->nnz > static_cast<int64_t>(UINT32_MAX)) return fail(CERDOT_E_VALUE, "row_entry needs nnz < 2^32");
  if (out == nullptr) return fail(CERDOT_E_VALUE, "null row_entry output");
  if (a->m < 0) return fail(CERDOT_E_VALUE, "m must be >= 0");
  return cerdot::row_entries(a, out, static_cast<cudaStream_t>(stream));
}

int cerdot_synth_choice(const uint64_t *state, const uint64_t *inc, uint64_t offset, const double *cdf,
                        const float *levels, int32_t k, int64_t count, float *out, void *stream) {
  if (state == nullptr || inc == nullptr || cdf == nullptr || levels == nullptr || (count > 0 && out == nullptr))
    return fail(CERDOT_E_VALUE, "synth_choice: null argument");
  return cerdot::synth_choice(state, inc, offset, cdf, levels, k, count, out, static_cast<cudaStream_t>(stream));
}

int32_t cerdot_set_kernel_path(int32_t op, int32_t path) {
  if (op < 0 || op >= CERDOT_PATH_COUNT) {
    fail(CERDOT_E_VALUE, "unknown kernel-path op " + std::to_string(op));
    return -1;
  }
  return g_paths[op].exchange(path);
}

int32_t cerdot_tile_view_rows(const cerdot_matrix *a, int64_t batch) {
  if (a == nullptr || a->m <= 0 || a->n <= 0) return 0;
  return cerdot::tile_view_rows(a, batch);
}

size_t cerdot_tile_view_workspace_bytes(const cerdot_matrix *a, int32_t tile_rows) {
  if (a == nullptr || tile_rows <= 0) return 0;
  return cerdot::tile_view_workspace_bytes(a->m, a->n, tile_rows);
}

int cerdot_tile_view_build(const cerdot_matrix *a, int32_t tile_rows, uint32_t *tile_ptr, void *tile_rec,
                           void *workspace, size_t workspace_bytes, void *stream) {
  int rc = check_matrix(a, 0, nullptr, nullptr, 0, 0);
  if (rc) return rc;
  if (tile_ptr == nullptr || (a->nnz > 0 && tile_rec == nullptr)) return fail(CERDOT_E_VALUE, "null tile view buffer");
  return cerdot::tile_view_build(a, tile_rows, tile_ptr, tile_rec, workspace, workspace_bytes,
                                 static_cast<cudaStream_t>(stream));
}

int cerdot_shard_plan(const void *row_ptr, int32_t row_ptr_bits, const void *omega_ptr, int32_t omega_ptr_bits,
                      int32_t col_bits, int32_t omega_index_bits, int64_t m, int32_t parts, int64_t *bounds) {
  if (parts < 1) return fail(CERDOT_E_VALUE, "parts must be >= 1");
  if (m < 0 || bounds == nullptr || (m > 0 && (row_ptr == nullptr || omega_ptr == nullptr)))
    return fail(CERDOT_E_VALUE, "invalid shard-plan arguments");
  if (!valid_bits(row_ptr_bits) || !valid_bits(omega_ptr_bits) || !valid_bits(col_bits) ||
      (omega_index_bits != 0 && !valid_bits(omega_index_bits)))
    return fail(CERDOT_E_VALUE, "index bits must be one of (8, 16, 32)");
  // prefix of encoded bytes per row: entries*col + segments*(ptr + CSER omegaI) + row pointer
  const double seg_bytes = (omega_ptr_bits + omega_index_bits) / 8.0;
  std::vector<double> prefix(static_cast<size_t>(m) + 1, 0.0);
  for (int64_t r = 0; r < m; ++r) {
    const uint64_t s0 = host_index(row_ptr, row_ptr_bits, r), s1 = host_index(row_ptr, row_ptr_bits, r + 1);
    const uint64_t e0 = host_index(omega_ptr, omega_ptr_bits, static_cast<int64_t>(s0));
    const uint64_t e1 = host_index(omega_ptr, omega_ptr_bits, static_cast<int64_t>(s1));
    prefix[r + 1] = prefix[r] + (e1 - e0) * (col_bits / 8.0) + (s1 - s0) * seg_bytes + row_ptr_bits / 8.0;
  }
  bounds[0] = 0;
  for (int p = 1; p < parts; ++p) {
    const double target = prefix[m] * p / parts;
    int64_t lo = bounds[p - 1], hi = m;
    while (lo < hi) {  // first r with prefix[r] >= target
      const int64_t mid = (lo + hi) / 2;
      if (prefix[mid] < target) lo = mid + 1; else hi = mid;
    }
    // pick the nearer of lo-1 / lo
    if (lo > bounds[p - 1] && target - prefix[lo - 1] < prefix[lo] - target) --lo;
    bounds[p] = lo;
  }
  bounds[parts] = m;
  return CERDOT_OK;
}

}  // extern "C"
