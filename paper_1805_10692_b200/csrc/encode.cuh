#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "cerdot.h"

namespace cerdot {

size_t encode_workspace_bytes(int64_t m, int64_t n);
int encode_plan(const void *w, int dtype, int64_t m, int64_t n, int64_t ldw, int bg_mode, double bg_value,
                void *workspace, size_t workspace_bytes, cerdot_encode_info *info, cudaStream_t st);
int encode_fill(const cerdot_encode_info *info, int kind, void *workspace, size_t workspace_bytes, double *omega,
                void *col, int col_bits, void *op, int op_bits, void *rp, int rp_bits, void *oi, int oi_bits,
                cudaStream_t st);

size_t encode_sort_workspace_bytes(int64_t m, int64_t n);
int encode_sort_plan(const void *w, int dtype, int64_t m, int64_t n, int64_t ldw, int bg_mode, double bg_value,
                     void *workspace, size_t workspace_bytes, cerdot_encode_info *info, cudaStream_t st);
int encode_sort_fill(const cerdot_encode_info *info, int kind, void *workspace, size_t workspace_bytes, double *omega,
                     void *col, int col_bits, void *op, int op_bits, void *rp, int rp_bits, void *oi, int oi_bits,
                     cudaStream_t st);

int row_entries(const cerdot_matrix *a, uint32_t *out, cudaStream_t st);
int dot(const cerdot_matrix *a, const float *x, int64_t ldx, int64_t batch, float *y, int64_t ldy, void *workspace,
        size_t workspace_bytes, cudaStream_t st, float *const *peers = nullptr, int npeers = 0,
        int64_t peer_offset = 0);

size_t validate_workspace_bytes(const cerdot_matrix *a);
int validate(const cerdot_matrix *a, cerdot_format_error *err, void *workspace, size_t workspace_bytes,
             cudaStream_t st);
int decode(const cerdot_matrix *a, double *out, int64_t ldo, cudaStream_t st);
int trace_counts(const cerdot_matrix *a, uint64_t *counts, void *workspace, cudaStream_t st);
int lemx_unpack(const void *payload, int element_bits, int64_t k, int64_t omega_src, double *omega,
                const int64_t *spans, int count, void *arena, cudaStream_t st);

}  // namespace cerdot
