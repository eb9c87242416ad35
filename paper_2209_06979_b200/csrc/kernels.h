// kernels.h -- internal launch interfaces shared by the CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace mcube {

void count_launch();

struct SpmmParams {
  int64_t M, K, N, vrows;
  int V, S, LB, RB, shuffled, batch;
  const int64_t* row_begin;
  const int64_t* row_end;
  const uint32_t* col_indices;
  const uint32_t* lhs_words;
  int64_t lhs_stride;  // words per batch item
  const uint32_t* rhs_words;
  int64_t rhs_stride;
  int32_t* out;
  int64_t out_stride;
  const double* alpha;
  double alpha_host;
  uint16_t* out_f16;
  int64_t f16_stride;
  uint32_t* status;
  int64_t stored;  // stored vectors per batch item (SR-BCRS col_indices length); 0 = unknown
  int gather_tma;  // tcgen05 path: stage gathered rows with TMA gather4 instead of cp.async
  // filled by the launcher
  int64_t ntiles, tasks;
};

struct SddmmParams {
  int64_t M, K, N, vrows, n_blocks;
  int V, LB, RB, batch;
  const uint32_t* a_words;  // M x K row-major
  int64_t a_stride;
  const uint32_t* b_words;  // K x N column-major == N x K row-major
  int64_t b_stride;
  const int64_t* row_offsets;
  const uint32_t* col_indices;
  int32_t* out;
  int64_t out_stride;
  const double* alpha;
  double alpha_host;
  uint16_t* out_f16;
  int64_t f16_stride;
  uint32_t* status;
  int splits;  // warps per vector row, chosen by the launcher
  int64_t tasks;
};

struct SddmmTcParams {
  int64_t M, N, K, vrows, n_blocks;
  int V;
  const int64_t* row_offsets;
  const uint32_t* col_indices;
  int32_t* out;
  int64_t out_stride;
  const double* alpha;
  double alpha_host;
  uint16_t* out_f16;
  int64_t f16_stride;
  uint32_t* status;
  int n_panels, n_ctiles;
  int64_t tiles;
  int debug;
};

cudaError_t launch_spmm(SpmmParams p, cudaStream_t stream);
// true when a 4-bit-width plan must keep the reference's per-nibble chunk accumulators
bool spmm_needs_nibble_chunks(const SpmmParams& p);
// the densify kernel's value staging can hold whole strides of this problem
bool densify_stride_ok(const SpmmParams& p);
// dense-tile path for moderate sparsity (dense.cu + gemm_tc.cu): densify the LHS into int8
// planes in a caller-provided workspace, then an exact tcgen05 GEMM
bool dense_spmm_eligible(const SpmmParams& p);
size_t dense_spmm_workspace(const SpmmParams& p);
cudaError_t launch_dense_spmm(SpmmParams p, void* workspace, cudaStream_t stream);
cudaError_t launch_gemm_tc(const SpmmParams& p, const int8_t* a0, const int8_t* a1, const int8_t* b0,
                           const int8_t* b1, cudaStream_t stream);
// row-segment gather path (spmm_seg.cu) for the large gather-bound problems; with a
// workspace (spmm_seg_workspace bytes) a 4-bit right-hand side is pre-transformed once
bool spmm_seg_supported(const SpmmParams& p);
cudaError_t launch_spmm_seg(const SpmmParams& p, cudaStream_t stream);
size_t spmm_seg_workspace(const SpmmParams& p);
cudaError_t launch_spmm_seg_ws(SpmmParams p, void* workspace, cudaStream_t stream);
// tcgen05 gather path (spmm_tc.cu); launch_spmm dispatches to it when supported
bool spmm_tc_supported(const SpmmParams& p);
cudaError_t launch_spmm_tc(SpmmParams p, cudaStream_t stream);
cudaError_t launch_sddmm(SddmmParams p, cudaStream_t stream);
// MC_SDDMM_PATH_* of the kernel launch_sddmm picks
int sddmm_path(const SddmmParams& p);
// dense-tile tcgen05 path (sddmm_tc.cu); launch_sddmm dispatches to it by density
bool sddmm_tc_supported(const SddmmParams& p);
cudaError_t launch_sddmm_tc(const SddmmParams& p, cudaStream_t stream);

// SR-BCRS packer (sparse_format.py:284-315)
cudaError_t launch_srbcrs_plan(const int64_t* row_offsets, int64_t vrows, int stride,
                               int64_t* row_begin, int64_t* row_end, int64_t* total,
                               cudaStream_t stream);
cudaError_t launch_srbcrs_fill(const int64_t* row_offsets, const uint32_t* col_indices,
                               int64_t vrows, int64_t n_blocks, int V, int stride,
                               const int64_t* row_begin, const int64_t* row_end,
                               int64_t stored_total, const uint32_t* values, int bits,
                               uint32_t* col_out, uint32_t* values_out, cudaStream_t stream);
cudaError_t launch_shuffle(const uint32_t* in, int64_t n, uint32_t* out, cudaStream_t stream);

}  // namespace mcube
