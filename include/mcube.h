/*
 * mcube.h -- C ABI of the B200-native Magicube hot path (libmcube.so).
 *
 * Drop-in boundary for the reference package `qsparse` (Python, numpy):
 * every entry point below replaces one reference function, cited as
 * reference-file:line under /root/reference/pkg/src/qsparse/. Arguments are
 * plain pointers and sizes (no torch types). All data pointers are CUDA
 * device pointers; `stream` is a cudaStream_t (NULL = legacy default stream).
 * Calls are stream-ordered and asynchronous; the caller owns every buffer.
 * The library holds no global state except the thread-local last-error text
 * and is safe for concurrent callers on distinct streams.
 *
 * Return codes map 1:1 onto the reference's exception taxonomy
 * (errors.py:4-33). Data-dependent failures found on the device (int32
 * overflow of a result, a column index outside the matrix) are reported
 * through a caller-provided device status word (`status`, may be NULL) that
 * mc_status_fetch() converts to a return code after synchronising.
 */
#ifndef MCUBE_H
#define MCUBE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes (errors.py:4-33) ---- */
#define MC_OK 0
#define MC_ERR_VALUE 1                 /* ValueError                      */
#define MC_ERR_UNSUPPORTED_PRECISION 2 /* UnsupportedPrecisionError       */
#define MC_ERR_SHUFFLE_STATE 3         /* ShuffleStateError               */
#define MC_ERR_FORMAT 4                /* FormatError                     */
#define MC_ERR_OVERFLOW 5              /* OverflowRiskError               */
#define MC_ERR_CUDA 6                  /* CUDA runtime / launch failure   */

/* ---- device status word bits (OR-ed by kernels) ---- */
#define MC_STATUS_OVERFLOW 1u  /* a result left int32: OverflowRiskError     */
#define MC_STATUS_BAD_INDEX 2u /* a column index >= K (not the sentinel)     */

#define MC_SENTINEL_INDEX 0xFFFFFFFFu /* sparse_format.py:25 */

/* Layout tags for mc_dense.layout (qint.py:17-18). */
#define MC_ROW_MAJOR 0
#define MC_COL_MAJOR 1

/* SR-BCRS matrix (sparse_format.py:129-230, SrBcrsMatrix).
 * Element (v, j) of stored stride s lives at s*V*stride + v*stride + j;
 * values are `bit_width`-bit two's complement packed LSB-first in uint32
 * words (qint.py:41-62). shuffled != 0 means col_indices were permuted by
 * SHUFFLE_PERMUTATION in blocks of 8 (sparse_format.py:373-385). */
typedef struct mc_srbcrs {
  int64_t scalar_rows;          /* M                                   */
  int64_t scalar_cols;          /* K                                   */
  int32_t vector_length;        /* V in {2,4,8}                        */
  int32_t stride;               /* S, stored vectors per stride        */
  int32_t bit_width;            /* 4, 8, 12 or 16                      */
  int32_t shuffled;             /* 0/1                                 */
  int64_t stored_vectors;       /* length of col_indices               */
  const int64_t* row_begin;     /* [M/V] first stored vector of row    */
  const int64_t* row_end;       /* [M/V] one past the last valid one   */
  const uint32_t* col_indices;  /* [stored_vectors], sentinel padded   */
  const uint32_t* words;        /* packed values                       */
} mc_srbcrs;

/* Dense packed matrix (qint.py:110-147, PackedMatrix). */
typedef struct mc_dense {
  int64_t rows;
  int64_t cols;
  int32_t bit_width;            /* 4, 8 or 16                          */
  int32_t layout;               /* MC_ROW_MAJOR / MC_COL_MAJOR          */
  const uint32_t* words;
} mc_dense;

/* BCRS sparsity pattern (sparse_format.py:67-126, BcrsMatrix minus values). */
typedef struct mc_bcrs {
  int64_t scalar_rows;
  int64_t scalar_cols;
  int32_t vector_length;
  int32_t reserved;
  int64_t n_blocks;
  const int64_t* row_offsets;   /* [M/V + 1]                           */
  const uint32_t* col_indices;  /* [n_blocks], strictly increasing/row */
} mc_bcrs;

/* Fused output epilogue (the reference's Epilogue hook, kernels.py:37,
 * specialised to the dequantisation epilogues of attention.py:149-173).
 * The int32 accumulators are always exact; when out_f16 != NULL the kernel
 * also writes fp16(round_to_nearest((double)acc * alpha[b])), alpha being
 * per batch item (device array) or alpha_host when alpha == NULL. */
typedef struct mc_epilogue {
  const double* alpha;          /* device [batch] or NULL              */
  double alpha_host;
  uint16_t* out_f16;            /* device, same shape as the int32 out */
  int64_t out_f16_batch_stride; /* elements                            */
} mc_epilogue;

/* ---------------------------------------------------------------------
 * SpMM: out[M x N] (int32, row-major) = lhs (SR-BCRS) x rhs (row-major).
 * Replaces kernels.spmm (kernels.py:293-298) / spmm_pipelined (:301-311);
 * validation mirrors SpmmProblem.__post_init__ (kernels.py:65-83) and
 * check_accumulation_bound (emulation.py:108-113). bs_n in {64,128} is the
 * reference tiling hint (kernels.py:52-53); results do not depend on it.
 * ------------------------------------------------------------------- */
int mc_spmm(const mc_srbcrs* lhs, const mc_dense* rhs, int32_t bs_n,
            int32_t* out, uint32_t* status, void* stream);

/* SpMM with a caller-provided device workspace (same contract as mc_spmm otherwise).
 * At moderate sparsity (stored*V >= 8% of M*K, M/N/K multiples of 128) the library
 * densifies the LHS into int8 chunk planes inside the workspace and runs an exact
 * tcgen05 GEMM; on the row-segment gather path with a 4-bit RHS the workspace holds a
 * copy of the RHS with the low-nibble sign bits flipped (one operation less per gathered
 * word). Results are bit-identical either way. mc_spmm_workspace returns the bytes the
 * chosen path can use (0: the problem runs on the gather kernels without one and the
 * workspace may be NULL; a smaller workspace than asked is simply not used).
 * Replaces kernels.spmm (kernels.py:293-298). */
int mc_spmm_workspace(const mc_srbcrs* lhs, const mc_dense* rhs, size_t* bytes);
/* Which kernel mc_spmm_ws (with the workspace mc_spmm_workspace asked for) runs for this
 * problem -- for reports and profiling; the result never depends on it. */
enum {
  MC_SPMM_PATH_GATHER = 0,  /* spmm.cu: mma.sync, 64-column tasks, cp.async ring        */
  MC_SPMM_PATH_SEGMENT = 1, /* spmm_seg.cu: mma.sync, 128-byte row-segment tasks        */
  MC_SPMM_PATH_DENSE = 2,   /* dense.cu + gemm_tc.cu: densify + tcgen05 GEMM            */
  MC_SPMM_PATH_TC = 3,      /* spmm_tc.cu: tcgen05 gather (MCUBE_SPMM_PATH=tc only)     */
  MC_SPMM_PATH_NIBBLE = 4   /* spmm.cu with the reference's per-nibble chunk products   */
};
int mc_spmm_path(const mc_srbcrs* lhs, const mc_dense* rhs, int32_t* path);
int mc_spmm_ws(const mc_srbcrs* lhs, const mc_dense* rhs, int32_t bs_n,
               int32_t* out, uint32_t* status, void* workspace,
               size_t workspace_bytes, void* stream);
/* Batched SpMM over `batch` problems sharing the SR-BCRS structure
 * (row offsets and column indices) -- e.g. the attention heads of
 * attention.py:190-197. Item b uses lhs->words + b*lhs_words_stride,
 * rhs->words + b*rhs_words_stride and writes out + b*out_stride
 * (out may be NULL when only epi->out_f16 is wanted). */
int mc_spmm_batched(const mc_srbcrs* lhs, int64_t lhs_words_stride,
                    const mc_dense* rhs, int64_t rhs_words_stride,
                    int32_t batch, const mc_epilogue* epi,
                    int32_t* out, int64_t out_stride,
                    uint32_t* status, void* stream);

/* ---------------------------------------------------------------------
 * SDDMM: out_values[n_blocks*V] (int32, block-major, BCRS order) =
 * (a[M x K] row-major) x (b[K x N] column-major) sampled at `pattern`.
 * Replaces kernels.sddmm (kernels.py:367-435) with out_format "bcrs";
 * "sr-bcrs" output is mc_bcrs_to_srbcrs applied to these values.
 * ------------------------------------------------------------------- */
int mc_sddmm(const mc_dense* a, const mc_dense* b, const mc_bcrs* pattern,
             int32_t* out_values, uint32_t* status, void* stream);

/* Which SDDMM kernel mc_sddmm / mc_sddmm_batched run for this problem (for reports and
 * profiling; no launch). */
enum {
  MC_SDDMM_PATH_DENSE = 1,   /* sddmm_tc.cu: dense 128-column tiles on tcgen05 kind::i8     */
  MC_SDDMM_PATH_GATHER8 = 2, /* sddmm.cu: pipelined 8-bit mma.sync gather (sparse patterns)  */
  MC_SDDMM_PATH_GATHER = 3   /* sddmm.cu: generic mma.sync gather (16/4-bit, fp16 epilogue) */
};
int mc_sddmm_path(const mc_dense* a, const mc_dense* b, const mc_bcrs* pattern, int32_t* path);

int mc_sddmm_batched(const mc_dense* a, int64_t a_words_stride,
                     const mc_dense* b, int64_t b_words_stride,
                     const mc_bcrs* pattern, int32_t batch,
                     const mc_epilogue* epi,
                     int32_t* out_values, int64_t out_stride,
                     uint32_t* status, void* stream);

/* ---------------------------------------------------------------------
 * SR-BCRS packer (sparse_format.py:284-315, bcrs_to_srbcrs) in two calls:
 *   mc_srbcrs_plan: row_begin/row_end from row_offsets and the stride,
 *                   total stored vectors into *stored_total (device int64);
 *   mc_srbcrs_fill: sentinel-padded col_indices and the strided values.
 * `values` are `bits`-bit packed words (4/8/12/16), raw 32-bit elements
 * (bits == 32: int32 accumulators / float32 epilogue outputs) or raw 64-bit
 * elements (bits == 64: int64 / float64 epilogue outputs). Raw 16-bit
 * elements (float16 / int16) are moved as bits == 16 words. The element type
 * is kept, as the reference's values.astype(b.values.dtype) does.
 * ------------------------------------------------------------------- */
int mc_srbcrs_plan(const mc_bcrs* pattern, int32_t stride, int64_t* row_begin,
                   int64_t* row_end, int64_t* stored_total, void* stream);
int mc_srbcrs_fill(const mc_bcrs* pattern, int32_t stride,
                   const int64_t* row_begin, const int64_t* row_end,
                   int64_t stored_total, const uint32_t* values, int32_t bits,
                   uint32_t* col_out, uint32_t* values_out, void* stream);

/* Block-of-8 index shuffle (sparse_format.py:373-385), out-of-place. */
int mc_shuffle_indices(const uint32_t* col_in, int64_t n, int32_t stride,
                       uint32_t* col_out, void* stream);

/* ---------------------------------------------------------------------
 * Quantised sparse attention (attention.py:130-197) for `batch` heads that
 * share one 8x1 block mask. q/k/v are [batch, L, d] contiguous in
 * in_dtype; out_f16 is [batch, L, d]. mode MC_ATTN_PARITY reproduces the
 * reference's float64 softmax / rounding chain; MC_ATTN_FAST computes the
 * softmax in float32 (stated tolerance: max-abs 1e-3 after dequant).
 * Optional stage outputs (NULL to skip) expose the integer stages that the
 * reference returns in AttentionResult (attention.py:95-105).
 * ------------------------------------------------------------------- */
#define MC_DTYPE_F16 0
#define MC_DTYPE_F32 1
#define MC_DTYPE_F64 2
#define MC_ATTN_PARITY 0
#define MC_ATTN_FAST 1

typedef struct mc_attention_args {
  int32_t batch, seq_len, head_dim;
  int32_t softmax_bits, qkv_bits;     /* (16,8), (8,8) or (8,4)          */
  int32_t in_dtype, mode;
  const void* q;
  const void* k;
  const void* v;
  const mc_bcrs* mask;                /* L x L, V = 8                    */
  uint16_t* out_f16;                  /* [batch, L, d]                   */
  int32_t* scores_int;                /* [batch, n_blocks*8] or NULL     */
  uint16_t* scores_f16;               /* [batch, n_blocks*8] or NULL     */
  uint16_t* probs_f16;                /* [batch, n_blocks*8] or NULL     */
  int32_t* probs_int;                 /* [batch, n_blocks*8] or NULL     */
  int32_t* mix_int;                   /* [batch, L, d] or NULL           */
  double* scales;                     /* [batch, 4] (q, k, v, softmax)   */
  void* workspace;
  size_t workspace_bytes;
} mc_attention_args;

int mc_attention_workspace(const mc_attention_args* args, size_t* bytes);
int mc_sparse_attention(const mc_attention_args* args, uint32_t* status, void* stream);

/* ---- utilities ---- */
/* Synchronise `stream`, read the device status word, reset it to 0 and map
 * it to a return code (MC_ERR_OVERFLOW / MC_ERR_FORMAT / MC_OK). */
int mc_status_fetch(uint32_t* status, void* stream);
/* Flush the L2 cache by writing `bytes` of scratch (benchmark hygiene). */
int mc_l2_flush(void* scratch, size_t bytes, void* stream);
const char* mc_last_error(void);
int mc_version(void);
/* Number of kernel launches issued by this thread since the last reset. */
int64_t mc_launch_count(int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* MCUBE_H */
