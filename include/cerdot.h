/*
 * cerdot — B200 (sm_100a) CER/CSER conversion and dot product, C ABI.
 *
 * The reference (`lemt`, pure Python) has no FFI; its drop-in boundary is the
 * module-level Python API.  Each entry point below replaces the numpy body of
 * one reference function and is bound from Python with ctypes by
 * paper_1805_10692_b200/_native.py (see INTEGRATION.md for the binding a
 * maintainer would add to lemt itself):
 *
 *   cerdot_encode_plan / cerdot_encode_fill
 *       replace lemt.formats._frequency_alphabet + _segment_layout +
 *       encode_cer / encode_cser                (formats.py:193-295)
 *   cerdot_dot / cerdot_dot_cer / cerdot_dot_cser
 *       replace lemt.kernels._dot_segmented + dot_cer / dot_cser / dot
 *                                               (kernels.py:283-336)
 *   cerdot_index_bitwidth
 *       replaces lemt.formats.index_bitwidth     (formats.py:52-59)
 *   cerdot_shard_plan
 *       new: contiguous row blocks balanced by encoded bytes
 *   cerdot_row_entries
 *       new: derived per-row entry offsets (shortens the mat-vec start-up chain)
 *   cerdot_tile_view_rows / cerdot_tile_view_build
 *       new: derived column-tiled view feeding the TMA-staged mat-mat
 *
 * Conventions
 *   - Every pointer marked (device) is CUDA device memory on the current
 *     device; every size is in elements unless named *_bytes.
 *   - The caller allocates every buffer (sizes come from the plan); the
 *     library never allocates or frees caller memory and keeps no global
 *     mutable state besides a per-thread last-error string.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  All device
 *     work is stream-ordered.  cerdot_encode_plan synchronises `stream`
 *     (its outputs are sizes the caller needs to allocate); nothing else does.
 *   - Status codes map 1:1 onto the reference's Python exceptions:
 *       CERDOT_E_VALUE -> ValueError   (formats.py:54-71, kernels.py:106-110)
 *       CERDOT_E_TYPE  -> TypeError    (kernels.py:336)
 *       CERDOT_E_INDEX -> IndexError   (empty alphabet, formats.py:199)
 *       CERDOT_E_CUDA / CERDOT_E_UNSUPPORTED -> RuntimeError
 *     cerdot_last_error() returns the message for the calling thread.
 */
#ifndef CERDOT_H_
#define CERDOT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CERDOT_ABI_VERSION 3

typedef enum {
  CERDOT_OK = 0,
  CERDOT_E_VALUE = 1,
  CERDOT_E_TYPE = 2,
  CERDOT_E_INDEX = 3,
  CERDOT_E_CUDA = 4,
  CERDOT_E_UNSUPPORTED = 5,
  CERDOT_E_WORKSPACE = 6, /* workspace too small: info->workspace_bytes holds the need */
  CERDOT_E_FORMAT = 7     /* cerdot_validate found a structural violation (-> FormatError) */
} cerdot_status;

typedef enum { CERDOT_CER = 0, CERDOT_CSER = 1 } cerdot_kind;
typedef enum { CERDOT_F32 = 0, CERDOT_F64 = 1 } cerdot_dtype;

/* A CER or CSER matrix resident in device memory (field meaning as
 * lemt.formats.CerMatrix / CserMatrix, formats.py:105-170). */
typedef struct {
  int32_t kind;               /* cerdot_kind */
  int32_t mode_index;         /* CSER: position of the background in omega; CER: 0 */
  int64_t m, n;               /* rows, columns */
  int64_t k;                  /* alphabet size, len(omega) */
  int64_t nnz;                /* len(col_index) */
  int64_t segments;           /* len(omega_ptr) - 1 */
  const double *omega;        /* (device) k: CER frequency-major, CSER value-ascending */
  const void *col_index;      /* (device) nnz unsigned ints of col_bits.  col_index, omega_ptr and
                                 omega_index must be readable up to the next 16-byte boundary past
                                 their last entry (16 B vector loads / TMA bulk copies) */
  const void *omega_ptr;      /* (device) segments+1 unsigned ints of omega_ptr_bits */
  const void *row_ptr;        /* (device) m+1 unsigned ints of row_ptr_bits */
  const void *omega_index;    /* (device) CSER: segments unsigned ints of omega_index_bits */
  int32_t col_bits, omega_ptr_bits, row_ptr_bits, omega_index_bits; /* 8, 16 or 32 */
  double background;          /* host copy of omega[0] (CER) / omega[mode_index] (CSER) */
  int64_t max_row_nnz;        /* largest row (entries), 0 = unknown; selects the mat-vec tiling */
  int64_t max_row_segments;   /* largest row (segments), 0 = unknown */
  const uint32_t *row_entry;  /* (device, optional) m+1 entry offsets, row_entry[r] = omega_ptr[row_ptr[r]]
                                 (cerdot_row_entries); NULL = the kernels derive them.  A derived index,
                                 not part of the format: it removes one dependent DRAM load from the
                                 mat-vec's start-up chain */
  /* Optional column-tiled view for the mat-mat (batch > 1), built by cerdot_tile_view_build for
   * tile_rows = cerdot_tile_view_rows(a, batch); all three zero/NULL = no view (the mat-mat then
   * gathers X rows from L2).  A derived index, not part of the format. */
  int32_t tile_rows;          /* X rows per tile (NT) the view was built for */
  int32_t reserved0;
  const uint32_t *tile_ptr;   /* (device) T*m+1 u32, T = ceil(n/NT): tile-major row starts of the records */
  const void *tile_rec;       /* (device) nnz 8-byte records {column in tile | fragment end, fp32 value} */
} cerdot_matrix;

/* Result of phase 1 of the conversion. */
typedef struct {
  int64_t m, n;
  int64_t k;                  /* alphabet size (a prepended absent background included) */
  int64_t nnz;                /* non-background entries */
  int64_t segments_cer;       /* CER segments incl. empty padding */
  int64_t segments_cser;      /* CSER segments (present elements only) */
  int32_t mode_index;         /* CSER position of the background */
  int32_t path;               /* 0 = on-chip hash path (k <= CERDOT_FAST_K), 1 = sort path */
  double background;          /* omega[0] of the CER alphabet */
  size_t workspace_bytes;     /* bytes of workspace the plan+fill need */
  int64_t max_row_nnz;        /* largest row in entries */
  int64_t max_row_segments_cer;
  int64_t max_row_segments_cser;
} cerdot_encode_info;

#define CERDOT_FAST_K 2048

int cerdot_abi_version(void);
const char *cerdot_last_error(void);

/* Smallest of 8/16/32 holding max_value unsigned, or 0 with CERDOT_E_VALUE set
 * when max_value is negative or needs more than 32 bits (formats.py:52-59). */
int32_t cerdot_index_bitwidth(int64_t max_value);

/* Workspace bound for the on-chip path of an m x n matrix.  Call the plan with
 * at least this; the plan reports a larger need (CERDOT_E_WORKSPACE) only
 * when the alphabet is too large for the on-chip path. */
size_t cerdot_encode_workspace_bytes(int64_t m, int64_t n);

/* Phase 1: alphabet, ranks, per-row counts, sizes.
 *   w        (device) m x n values, row stride ldw elements, dtype f32 or f64
 *   bg_mode  0: background = most frequent value (ties -> smallest);
 *            1: background = bg_value (prepended when absent)  (formats.py:198-205)
 * Synchronises `stream`; fills *info.  The workspace holds the state the fill
 * reads, so do not reuse it in between. */
int cerdot_encode_plan(const void *w, int32_t dtype, int64_t m, int64_t n, int64_t ldw, int32_t bg_mode,
                       double bg_value, void *workspace, size_t workspace_bytes, cerdot_encode_info *info,
                       void *stream);

/* Phase 2: write one encoding into caller buffers sized from *info:
 *   omega k doubles; col_index nnz; omega_ptr S+1; row_ptr m+1; omega_index S (CSER)
 * with S = segments_cer / segments_cser.  Widths are 8/16/32 and must hold the
 * largest value (formats.py:66-74); CERDOT_E_VALUE otherwise. */
int cerdot_encode_fill(const cerdot_encode_info *info, int32_t kind, void *workspace, size_t workspace_bytes,
                       double *omega, void *col_index, int32_t col_bits, void *omega_ptr, int32_t omega_ptr_bits,
                       void *row_ptr, int32_t row_ptr_bits, void *omega_index, int32_t omega_index_bits,
                       void *stream);

/* Workspace the dot needs (zero unless the background is non-zero: then
 * batch doubles for the column sums of x, plus 16 x batch doubles of
 * row-range partial sums when batch > 1). */
size_t cerdot_dot_workspace_bytes(const cerdot_matrix *a, int64_t batch);

/* y (m x batch, row stride ldy) = A . x (n x batch, row stride ldx), fp32.
 * batch == 1 is the mat-vec.  Stream-ordered, no allocation, deterministic. */
int cerdot_dot(const cerdot_matrix *a, const float *x, int64_t ldx, int64_t batch, float *y, int64_t ldy,
               void *workspace, size_t workspace_bytes, void *stream);
int cerdot_dot_cer(const cerdot_matrix *a, const float *x, int64_t ldx, int64_t batch, float *y, int64_t ldy,
                   void *workspace, size_t workspace_bytes, void *stream);
int cerdot_dot_cser(const cerdot_matrix *a, const float *x, int64_t ldx, int64_t batch, float *y, int64_t ldy,
                    void *workspace, size_t workspace_bytes, void *stream);

/* Row-sharded dot with the output all-gather fused into the kernels' epilogue: this
 * rank's block y (rows of its shard) is written to `y` as by cerdot_dot and, element by element, to
 * position peer_offset + i of each of the `npeers` other ranks' full-output buffers (`peers`: a DEVICE
 * array of device pointers, e.g. the NVLink peer mappings of a symmetric-memory buffer; peer_offset =
 * the shard's first row times ldy).  The stores leave from the epilogue as each row finishes, so the
 * exchange overlaps the rest of the computation.  The caller completes it with a stream-ordered
 * cross-rank barrier (signal/wait) after the call.  npeers = 0 is cerdot_dot. */
int cerdot_dot_peers(const cerdot_matrix *a, const float *x, int64_t ldx, int64_t batch, float *y, int64_t ldy,
                     float *const *peers, int32_t npeers, int64_t peer_offset, void *workspace,
                     size_t workspace_bytes, void *stream);

/* Host-buffer convenience (the e2e path of the reference-facing API): copies x (HOST, fp32, n x batch,
 * row stride ldx; pinned for asynchronous copies) to the device, runs cerdot_dot, copies y (HOST,
 * m x batch, row stride ldy) back and synchronises `stream`.  The device workspace (size from
 * cerdot_dot_host_workspace_bytes) holds the device copies of x and y and the dot's own scratch. */
size_t cerdot_dot_host_workspace_bytes(const cerdot_matrix *a, int64_t batch);
int cerdot_dot_host(const cerdot_matrix *a, const float *x_host, int64_t ldx, int64_t batch, float *y_host,
                    int64_t ldy, void *workspace, size_t workspace_bytes, void *stream);

/* Derived index for cerdot_matrix.row_entry: out[r] = omega_ptr[row_ptr[r]] for r in [0, m], u32
 * (device, m+1).  CERDOT_E_VALUE when nnz does not fit 32 bits.  Stream-ordered. */
int cerdot_row_entries(const cerdot_matrix *a, uint32_t *out, void *stream);

/* Column-tiled view (derived index) for the TMA-staged mat-mat -- the batch > 1 path of
 * kernels.py:283-301: every segment split at the X-tile boundaries (colI is ascending inside a segment,
 * formats.py:220).  cerdot_tile_view_rows returns the tile height NT the mat-mat wants for this batch
 * (0 = the tiled path does not apply: batch 1, nnz >= 2^32).  Buffers: tile_ptr ceil(n/NT)*m+1 u32,
 * tile_rec nnz*8 bytes, workspace cerdot_tile_view_workspace_bytes.  Needs a->row_entry.
 * Stream-ordered. */
int32_t cerdot_tile_view_rows(const cerdot_matrix *a, int64_t batch);
size_t cerdot_tile_view_workspace_bytes(const cerdot_matrix *a, int32_t tile_rows);
int cerdot_tile_view_build(const cerdot_matrix *a, int32_t tile_rows, uint32_t *tile_ptr, void *tile_rec,
                           void *workspace, size_t workspace_bytes, void *stream);

/* Kernel selection override for A/B measurements and parity tests (process-wide; 0 = automatic, the
 * default).  Replaces reading environment variables on the dot path.
 *   CERDOT_PATH_MATVEC: 1 window kernel, 2 CTA-tile kernel, 3 long-row kernel (cp.async ring),
 *                       4 long-row stream kernel (register ring, fragment sums),
 *                       5 one-row-per-warp kernel (rows of at most one 1024-entry window)
 *   CERDOT_PATH_MATMAT: 1 flat L2-gather kernel, 2 per-segment kernel, 3 tiled (needs a view),
 *                       4 tiled with sum-then-multiply per segment fragment
 *   CERDOT_PATH_MATVEC_NT: 1 co-resident 16-warp window kernel, 896 the 28-warp one
 *   CERDOT_PATH_MATMAT_DEPTH: X-row loads in flight of the flat kernel (8 / 16)
 *   CERDOT_PATH_MATMAT_SPLIT: CTAs per row block sharing the X tiles of the tiled mat-mat (1, 2, 4, 8)
 *   CERDOT_PATH_MATMAT_TILE: X rows per tile of a forced tiled mat-mat (128 / 256)
 * Returns the previous value; CERDOT_E_VALUE for an unknown op. */
typedef enum {
  CERDOT_PATH_MATVEC = 0,
  CERDOT_PATH_MATMAT = 1,
  CERDOT_PATH_MATVEC_NT = 2,
  CERDOT_PATH_MATMAT_DEPTH = 3,
  CERDOT_PATH_TRACE = 4,
  CERDOT_PATH_MATMAT_SPLIT = 5,
  CERDOT_PATH_MATMAT_TILE = 6,
  CERDOT_PATH_COUNT
} cerdot_path_op;
int32_t cerdot_set_kernel_path(int32_t op, int32_t path);

/* Structural validation of an (untrusted) encoding on the device -- lemt.formats.validate
 * (formats.py:298-392) for the index arrays.  The checks run in the reference's order; the first
 * violation is written to *err (check id, offset into the named array, and the value its message
 * quotes) and CERDOT_E_FORMAT returned; CERDOT_OK when every check passes.  The alphabet checks
 * (duplicate / unsorted omega, mode_index range) and array-length checks are the caller's: the
 * matrix struct carries lengths, not arrays of other lengths.  Synchronises `stream`. */
typedef enum {
  CERDOT_CHECK_NONE = 0,
  CERDOT_CHECK_PTR_START,         /* omegaPtr[0] != 0                 ("must start at 0, found v") */
  CERDOT_CHECK_PTR_ORDER,         /* omegaPtr decreasing at offset     ("must be non-decreasing") */
  CERDOT_CHECK_PTR_END,           /* omegaPtr[segs] != nnz             ("must end at nnz, found v") */
  CERDOT_CHECK_ROW_START,         /* rowPtr[0] != 0 */
  CERDOT_CHECK_ROW_ORDER,         /* rowPtr decreasing */
  CERDOT_CHECK_ROW_END,           /* rowPtr[m] != segments */
  CERDOT_CHECK_COL_RANGE,         /* colI[offset] = v >= n */
  CERDOT_CHECK_COL_ORDER,         /* colI not strictly ascending inside a segment */
  CERDOT_CHECK_COL_DUPLICATE,     /* a column twice in one row (offset = second occurrence) */
  CERDOT_CHECK_CER_ROW_SEGMENTS,  /* rowPtr[offset]: the row holds v > k-1 segments */
  CERDOT_CHECK_CER_TRAILING_EMPTY,/* omegaPtr[offset]: a row ends with an empty segment */
  CERDOT_CHECK_OI_RANGE,          /* omegaI[offset] >= k */
  CERDOT_CHECK_OI_BACKGROUND,     /* omegaI[offset] == mode_index */
  CERDOT_CHECK_EMPTY_SEGMENT,     /* omegaPtr[offset]: CSER segment without entries */
  CERDOT_CHECK_OI_DUPLICATE,      /* an element twice in one row (offset = second occurrence) */
  CERDOT_CHECK_COUNT
} cerdot_check;

typedef struct {
  int32_t check;   /* cerdot_check */
  int64_t offset;  /* position in the array the check names */
  int64_t value;   /* the value the reference's message quotes (found start/end, column, segments) */
} cerdot_format_error;

size_t cerdot_validate_workspace_bytes(const cerdot_matrix *a);
int cerdot_validate(const cerdot_matrix *a, cerdot_format_error *err, void *workspace, size_t workspace_bytes,
                    void *stream);

/* Dense reconstruction (lemt.formats.decode, formats.py:395-424) of a VALID encoding: out (device,
 * m x n float64, row stride ldo) = background, then every segment's element at its columns.
 * Stream-ordered. */
int cerdot_decode(const cerdot_matrix *a, double *out, int64_t ldo, void *stream);

/* Inputs of the analytic OpTrace (lemt kernels.py:175-234) over all rows, counted on the device:
 * counts (HOST, 5) = segments, non-empty segments, entries, rows holding segments, and the sum over
 * rows of max(non-empty segments - 1, 0).  workspace: 64 device bytes.  Synchronises `stream`. */
int cerdot_trace_counts(const cerdot_matrix *a, uint64_t *counts, void *workspace, void *stream);

/* LEMX container loader (lemt io.py:177-278), device half: `payload` (device) holds the container's
 * array payload as read from the file (everything after the fixed header).  omega (k elements of
 * element_bits: f64 / f32 / f16 / i8, at payload offset omega_offset) is widened to f64 into `omega`;
 * each of `count` (<= 4) index arrays is copied byte for byte: spans (HOST) holds count triples
 * (payload offset, arena offset, bytes).  The host parses and checks the header.  Stream-ordered. */
int cerdot_lemx_unpack(const void *payload, int32_t element_bits, int64_t k, int64_t omega_offset, double *omega,
                       const int64_t *spans, int32_t count, void *arena, void *stream);

/* Synthetic inputs (benchmark / tests, not the format path): out[i] = levels[searchsorted(cdf, u_{offset+i},
 * side='right')] for i < count, where u_j is the j-th random() of numpy's Generator(PCG64) whose 128-bit
 * state / increment are state[0..1] / inc[0..1] (low word first, as numpy's bit_generator.state) -- i.e.
 * numpy's default_rng(seed).choice(k, size, p) bit for bit, with cdf = cumsum(p)/cumsum(p)[-1] (float64)
 * and the draw starting `offset` elements in.  cdf / levels / out are device arrays.  Stream-ordered. */
int cerdot_synth_choice(const uint64_t *state, const uint64_t *inc, uint64_t offset, const double *cdf,
                        const float *levels, int32_t k, int64_t count, float *out, void *stream);

/* Row-shard planner (host).  row_ptr / omega_ptr are HOST arrays of the
 * given widths.  Writes parts+1 row bounds (bounds[0]=0, bounds[parts]=m)
 * splitting rows into contiguous blocks of near-equal encoded bytes
 * (entries*col_bytes + segments*(ptr_bytes + omegaI bytes) + rows*row_bytes);
 * omega_index_bits = 0 for CER. */
int cerdot_shard_plan(const void *row_ptr, int32_t row_ptr_bits, const void *omega_ptr, int32_t omega_ptr_bits,
                      int32_t col_bits, int32_t omega_index_bits, int64_t m, int32_t parts, int64_t *bounds);

#ifdef __cplusplus
}
#endif

#endif /* CERDOT_H_ */
