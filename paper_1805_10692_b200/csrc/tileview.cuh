// Column-tiled view of a CER/CSER encoding and the TMA-staged mat-mat over it (tileview.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "cerdot.h"

namespace cerdot {

// X rows per tile the mat-mat wants at this batch (0: no tiled path for this matrix / batch).
int32_t tile_view_rows(const cerdot_matrix *a, int64_t batch);
int64_t tile_view_tiles(int64_t n, int32_t nt);
size_t tile_view_workspace_bytes(int64_t m, int64_t n, int32_t nt);
int tile_view_build(const cerdot_matrix *a, int32_t nt, uint32_t *tptr, void *rec, void *workspace,
                    size_t workspace_bytes, cudaStream_t st);
// Runs the tiled mat-mat when the matrix carries a usable view; *used = false otherwise (caller falls back).
int matmat_tiled(const cerdot_matrix *mat, const float *x, int64_t ldx, int64_t batch, float *y, int64_t ldy,
                 const double *colsum, float *const *peers, int npeers, int64_t peer_offset, void *workspace,
                 size_t workspace_bytes, cudaStream_t st, bool *used);
// Bytes of dot workspace the tiled mat-mat wants for its tile-split partial products (0: none).
size_t tile_view_dot_workspace_bytes(const cerdot_matrix *a, int64_t batch);

// numpy Generator(PCG64).choice on the device (synth.cu).
int synth_choice(const uint64_t *state, const uint64_t *inc, uint64_t offset, const double *cdf, const float *levels,
                 int32_t k, int64_t count, float *out, cudaStream_t st);

// Kernel-path overrides (cerdot_set_kernel_path); 0 = automatic.
int kernel_path(int op);

}  // namespace cerdot
