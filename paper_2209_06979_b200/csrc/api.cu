// api.cu -- extern "C" entry points of libmcube.so (see include/mcube.h).
//
// Each entry point validates its arguments exactly like the reference's
// problem constructors (kernels.py:58-118) and precision planner
// (emulation.py:67-113), maps failures to the reference's exception taxonomy
// (errors.py:4-33) via return codes + mc_last_error(), and launches the CUDA
// kernels stream-ordered. There is no host compute path.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"
#include "kernels.h"

namespace mcube {
cudaError_t launch_attention(const mc_attention_args* a, uint32_t* status, cudaStream_t stream, size_t* ws_needed);

static thread_local std::string g_last_error;
static thread_local int64_t g_launches = 0;
void count_launch() { ++g_launches; }

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

static int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return MC_OK;
  return fail(MC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// emulation.py:23-30 (Table IV)
static bool spmm_pair_ok(int l, int r) {
  return (l == 16 && r == 16) || (l == 16 && r == 8) || (l == 16 && r == 4) || (l == 12 && r == 4) ||
         (l == 8 && r == 4) || (l == 8 && r == 8) || (l == 4 && r == 4);
}
static bool sddmm_pair_ok(int l, int r) { return (l == 16 && r == 16) || (l == 8 && r == 8) || (l == 4 && r == 4); }
static int plan_width(int l, int r) { return (l % 8 == 0 && r % 8 == 0) ? 8 : 4; }  // emulation.py:80

// emulation.check_accumulation_bound (emulation.py:108-113)
static bool bound_ok(int64_t k, int w) {
  const long long worst = (1LL << w) - 1;
  return static_cast<long double>(k) * worst * worst <= 2147483647.0L;
}

static int check_spmm(const mc_srbcrs* a, const mc_dense* b, int bs_n) {
  if (!a || !b) return fail(MC_ERR_VALUE, "null argument");
  if (bs_n != 64 && bs_n != 128) return fail(MC_ERR_VALUE, "BS_n must be 64 or 128, got %d", bs_n);
  if (b->layout != MC_ROW_MAJOR) return fail(MC_ERR_VALUE, "SpMM RHS must be row-major");
  if (a->scalar_cols != b->rows)
    return fail(MC_ERR_VALUE, "K mismatch: lhs has %lld columns, rhs %lld rows", (long long)a->scalar_cols,
                (long long)b->rows);
  if (!spmm_pair_ok(a->bit_width, b->bit_width))
    return fail(MC_ERR_UNSUPPORTED_PRECISION, "L%d-R%d is not supported for spmm", a->bit_width, b->bit_width);
  if (b->bit_width == 4 && !a->shuffled)
    return fail(MC_ERR_SHUFFLE_STATE, "4-bit RHS requires shuffled LHS column indices");
  if (b->bit_width != 4 && a->shuffled)
    return fail(MC_ERR_SHUFFLE_STATE, "shuffled LHS indices are only valid with a 4-bit RHS");
  const int w = plan_width(a->bit_width, b->bit_width);
  const int tile_k = w == 8 ? 16 : 32;
  if (a->stride <= 0 || a->stride % tile_k)
    return fail(MC_ERR_VALUE, "format stride %d must be a multiple of the tile k %d", a->stride, tile_k);
  const int v = a->vector_length;
  if (v != 2 && v != 4 && v != 8) return fail(MC_ERR_FORMAT, "vector length must be 2, 4 or 8");
  if (a->scalar_rows % v) return fail(MC_ERR_FORMAT, "scalar_rows %lld not divisible by V=%d", (long long)a->scalar_rows, v);
  if (!bound_ok(a->scalar_cols, w))
    return fail(MC_ERR_OVERFLOW, "reduction size %lld risks int32 overflow for %d-bit chunk products",
                (long long)a->scalar_cols, w);
  return MC_OK;
}

static int check_sddmm(const mc_dense* a, const mc_dense* b, const mc_bcrs* p) {
  if (!a || !b || !p) return fail(MC_ERR_VALUE, "null argument");
  if (a->layout != MC_ROW_MAJOR) return fail(MC_ERR_VALUE, "SDDMM A must be row-major");
  if (b->layout != MC_COL_MAJOR) return fail(MC_ERR_VALUE, "SDDMM B must be column-major");
  if (a->cols != b->rows) return fail(MC_ERR_VALUE, "K mismatch: %lld vs %lld", (long long)a->cols, (long long)b->rows);
  if (p->scalar_rows != a->rows) return fail(MC_ERR_VALUE, "pattern rows must match A rows");
  if (p->scalar_cols != b->cols) return fail(MC_ERR_VALUE, "pattern columns must match B columns");
  if (!sddmm_pair_ok(a->bit_width, b->bit_width))
    return fail(MC_ERR_UNSUPPORTED_PRECISION, "L%d-R%d is not supported for sddmm", a->bit_width, b->bit_width);
  const int v = p->vector_length;
  if (v != 2 && v != 4 && v != 8) return fail(MC_ERR_FORMAT, "vector length must be 2, 4 or 8");
  if (p->scalar_rows % v) return fail(MC_ERR_FORMAT, "scalar_rows not divisible by V");
  if (!bound_ok(a->cols, plan_width(a->bit_width, b->bit_width)))
    return fail(MC_ERR_OVERFLOW, "reduction size %lld risks int32 overflow", (long long)a->cols);
  return MC_OK;
}

__global__ void l2_read_kernel(const uint4* __restrict__ p, int64_t n16) {
  uint32_t acc = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint4 v = __ldcg(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9E3779B9u) asm volatile("trap;");  // keeps the loads alive; never true for the 0x5A fill
}

}  // namespace mcube

using namespace mcube;

extern "C" {

int mc_version(void) { return 1; }

const char* mc_last_error(void) { return g_last_error.c_str(); }

int64_t mc_launch_count(int32_t reset) {
  const int64_t n = g_launches;
  if (reset) g_launches = 0;
  return n;
}

static SpmmParams spmm_params(const mc_srbcrs* lhs, int64_t lhs_words_stride, const mc_dense* rhs,
                               int64_t rhs_words_stride, int32_t batch, const mc_epilogue* epi, int32_t* out,
                               int64_t out_stride, uint32_t* status) {
  SpmmParams p{};
  p.M = lhs->scalar_rows;
  p.K = lhs->scalar_cols;
  p.N = rhs->cols;
  p.V = lhs->vector_length;
  p.vrows = p.M / p.V;
  p.S = lhs->stride;
  p.LB = lhs->bit_width;
  p.RB = rhs->bit_width;
  p.shuffled = lhs->shuffled;
  p.batch = batch;
  p.row_begin = lhs->row_begin;
  p.row_end = lhs->row_end;
  p.stored = lhs->stored_vectors;
  p.col_indices = lhs->col_indices;
  p.lhs_words = lhs->words;
  p.lhs_stride = lhs_words_stride;
  p.rhs_words = rhs->words;
  p.rhs_stride = rhs_words_stride;
  p.out = out;
  p.out_stride = out_stride;
  if (epi) {
    p.alpha = epi->alpha;
    p.alpha_host = epi->alpha_host;
    p.out_f16 = epi->out_f16;
    p.f16_stride = epi->out_f16_batch_stride;
  }
  p.status = status;
  return p;
}

int mc_spmm_batched(const mc_srbcrs* lhs, int64_t lhs_words_stride, const mc_dense* rhs, int64_t rhs_words_stride,
                    int32_t batch, const mc_epilogue* epi, int32_t* out, int64_t out_stride, uint32_t* status,
                    void* stream) {
  int rc = check_spmm(lhs, rhs, 64);
  if (rc) return rc;
  if (batch < 0) return fail(MC_ERR_VALUE, "batch must be >= 0");
  SpmmParams p = spmm_params(lhs, lhs_words_stride, rhs, rhs_words_stride, batch, epi, out, out_stride, status);
  if (p.M == 0 || p.N == 0 || batch == 0) return MC_OK;
  return cuda_status(launch_spmm(p, static_cast<cudaStream_t>(stream)), "mc_spmm");
}

int mc_spmm(const mc_srbcrs* lhs, const mc_dense* rhs, int32_t bs_n, int32_t* out, uint32_t* status, void* stream) {
  int rc = check_spmm(lhs, rhs, bs_n);
  if (rc) return rc;
  return mc_spmm_batched(lhs, 0, rhs, 0, 1, nullptr, out, 0, status, stream);
}

int mc_spmm_workspace(const mc_srbcrs* lhs, const mc_dense* rhs, size_t* bytes) {
  int rc = check_spmm(lhs, rhs, 64);
  if (rc) return rc;
  if (!bytes) return fail(MC_ERR_VALUE, "bytes must not be NULL");
  // a placeholder output pointer: eligibility only looks at its alignment
  SpmmParams p = spmm_params(lhs, 0, rhs, 0, 1, nullptr, reinterpret_cast<int32_t*>(256), 0, nullptr);
  const size_t dense = dense_spmm_workspace(p);
  *bytes = dense > 0 ? dense : spmm_seg_workspace(p);
  return MC_OK;
}

int mc_spmm_path(const mc_srbcrs* lhs, const mc_dense* rhs, int32_t* path) {
  int rc = check_spmm(lhs, rhs, 64);
  if (rc) return rc;
  if (!path) return fail(MC_ERR_VALUE, "path must not be NULL");
  SpmmParams p = spmm_params(lhs, 0, rhs, 0, 1, nullptr, reinterpret_cast<int32_t*>(256), 0, nullptr);
  if (dense_spmm_workspace(p) > 0) *path = MC_SPMM_PATH_DENSE;
  else if (spmm_tc_supported(p)) *path = MC_SPMM_PATH_TC;
  else if (spmm_needs_nibble_chunks(p)) *path = MC_SPMM_PATH_NIBBLE;
  else if (spmm_seg_supported(p)) *path = MC_SPMM_PATH_SEGMENT;
  else *path = MC_SPMM_PATH_GATHER;
  return MC_OK;
}

int mc_spmm_ws(const mc_srbcrs* lhs, const mc_dense* rhs, int32_t bs_n, int32_t* out, uint32_t* status,
               void* workspace, size_t workspace_bytes, void* stream) {
  int rc = check_spmm(lhs, rhs, bs_n);
  if (rc) return rc;
  SpmmParams p = spmm_params(lhs, 0, rhs, 0, 1, nullptr, out, 0, status);
  if (p.M == 0 || p.N == 0) return MC_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t need = dense_spmm_workspace(p);
  if (workspace && need > 0 && workspace_bytes >= need)
    return cuda_status(launch_dense_spmm(p, workspace, s), "mc_spmm_ws");
  const size_t seg = need > 0 ? 0 : spmm_seg_workspace(p);
  // the pre-XORed copy is gathered with 16-byte cp.async: a misaligned workspace is not used
  if (workspace && seg > 0 && workspace_bytes >= seg && (reinterpret_cast<uintptr_t>(workspace) & 15) == 0)
    return cuda_status(launch_spmm_seg_ws(p, workspace, s), "mc_spmm_ws");
  return cuda_status(launch_spmm(p, s), "mc_spmm_ws");
}

static SddmmParams sddmm_params(const mc_dense* a, int64_t a_words_stride, const mc_dense* b, int64_t b_words_stride,
                                const mc_bcrs* pattern, int32_t batch, const mc_epilogue* epi, int32_t* out_values,
                                int64_t out_stride, uint32_t* status) {
  SddmmParams p{};
  p.M = a->rows;
  p.K = a->cols;
  p.N = b->cols;
  p.V = pattern->vector_length;
  p.vrows = p.M / p.V;
  p.n_blocks = pattern->n_blocks;
  p.LB = a->bit_width;
  p.RB = b->bit_width;
  p.batch = batch;
  p.a_words = a->words;
  p.a_stride = a_words_stride;
  p.b_words = b->words;
  p.b_stride = b_words_stride;
  p.row_offsets = pattern->row_offsets;
  p.col_indices = pattern->col_indices;
  p.out = out_values;
  p.out_stride = out_stride;
  if (epi) {
    p.alpha = epi->alpha;
    p.alpha_host = epi->alpha_host;
    p.out_f16 = epi->out_f16;
    p.f16_stride = epi->out_f16_batch_stride;
  }
  p.status = status;
  return p;
}

int mc_sddmm_batched(const mc_dense* a, int64_t a_words_stride, const mc_dense* b, int64_t b_words_stride,
                     const mc_bcrs* pattern, int32_t batch, const mc_epilogue* epi, int32_t* out_values,
                     int64_t out_stride, uint32_t* status, void* stream) {
  int rc = check_sddmm(a, b, pattern);
  if (rc) return rc;
  const SddmmParams p =
      sddmm_params(a, a_words_stride, b, b_words_stride, pattern, batch, epi, out_values, out_stride, status);
  if (p.n_blocks == 0 || batch == 0) return MC_OK;
  return cuda_status(launch_sddmm(p, static_cast<cudaStream_t>(stream)), "mc_sddmm");
}

int mc_sddmm_path(const mc_dense* a, const mc_dense* b, const mc_bcrs* pattern, int32_t* path) {
  int rc = check_sddmm(a, b, pattern);
  if (rc) return rc;
  if (!path) return fail(MC_ERR_VALUE, "path must not be NULL");
  // a 256-byte aligned stand-in output: only the problem's shape and operands decide
  *path = sddmm_path(sddmm_params(a, 0, b, 0, pattern, 1, nullptr, reinterpret_cast<int32_t*>(256), 0, nullptr));
  return MC_OK;
}

int mc_sddmm(const mc_dense* a, const mc_dense* b, const mc_bcrs* pattern, int32_t* out_values, uint32_t* status,
             void* stream) {
  return mc_sddmm_batched(a, 0, b, 0, pattern, 1, nullptr, out_values, 0, status, stream);
}

int mc_srbcrs_plan(const mc_bcrs* pattern, int32_t stride, int64_t* row_begin, int64_t* row_end,
                   int64_t* stored_total, void* stream) {
  if (!pattern) return fail(MC_ERR_VALUE, "null pattern");
  if (stride <= 0) return fail(MC_ERR_FORMAT, "stride must be positive");
  const int64_t vrows = pattern->scalar_rows / pattern->vector_length;
  if (vrows == 0) {
    cudaMemsetAsync(stored_total, 0, 8, static_cast<cudaStream_t>(stream));
    return MC_OK;
  }
  return cuda_status(launch_srbcrs_plan(pattern->row_offsets, vrows, stride, row_begin, row_end, stored_total,
                                        static_cast<cudaStream_t>(stream)),
                     "mc_srbcrs_plan");
}

int mc_srbcrs_fill(const mc_bcrs* pattern, int32_t stride, const int64_t* row_begin, const int64_t* row_end,
                   int64_t stored_total, const uint32_t* values, int32_t bits, uint32_t* col_out,
                   uint32_t* values_out, void* stream) {
  if (!pattern) return fail(MC_ERR_VALUE, "null pattern");
  if (bits != 4 && bits != 8 && bits != 12 && bits != 16 && bits != 32 && bits != 64)
    return fail(MC_ERR_VALUE, "bits must be 4, 8, 12, 16, 32 or 64");
  const int64_t vrows = pattern->scalar_rows / pattern->vector_length;
  return cuda_status(launch_srbcrs_fill(pattern->row_offsets, pattern->col_indices, vrows, pattern->n_blocks,
                                        pattern->vector_length, stride, row_begin, row_end, stored_total, values, bits,
                                        col_out, values_out, static_cast<cudaStream_t>(stream)),
                     "mc_srbcrs_fill");
}

int mc_shuffle_indices(const uint32_t* col_in, int64_t n, int32_t stride, uint32_t* col_out, void* stream) {
  if (stride % 8) return fail(MC_ERR_VALUE, "stride %d not divisible by shuffle block 8", stride);
  if (n % 8) return fail(MC_ERR_FORMAT, "index count %lld not divisible by 8", (long long)n);
  return cuda_status(launch_shuffle(col_in, n, col_out, static_cast<cudaStream_t>(stream)), "mc_shuffle_indices");
}

int mc_attention_workspace(const mc_attention_args* a, size_t* bytes) {
  if (!a || !a->mask || !bytes) return fail(MC_ERR_VALUE, "null argument");
  mc_attention_args tmp = *a;
  tmp.workspace = nullptr;
  return cuda_status(launch_attention(&tmp, nullptr, nullptr, bytes), "mc_attention_workspace");
}

int mc_sparse_attention(const mc_attention_args* a, uint32_t* status, void* stream) {
  if (!a || !a->mask) return fail(MC_ERR_VALUE, "null argument");
  if (a->seq_len % 8) return fail(MC_ERR_VALUE, "sequence length must be a multiple of 8");
  const int sb = a->softmax_bits, qb = a->qkv_bits;
  if (!((sb == 16 && qb == 8) || (sb == 8 && qb == 8) || (sb == 8 && qb == 4)))
    return fail(MC_ERR_UNSUPPORTED_PRECISION, "%db-%db not in supported set [16b-8b, 8b-8b, 8b-4b]", sb, qb);
  if (a->mask->vector_length != 8) return fail(MC_ERR_VALUE, "attention mask must use 8x1 blocks");
  if (a->mask->scalar_rows != a->seq_len || a->mask->scalar_cols != a->seq_len)
    return fail(MC_ERR_VALUE, "mask must be seq_len x seq_len");
  if (a->in_dtype < 0 || a->in_dtype > 2) return fail(MC_ERR_VALUE, "unknown input dtype");
  size_t need = 0;
  mc_attention_args probe = *a;
  probe.workspace = nullptr;
  launch_attention(&probe, nullptr, nullptr, &need);
  if (a->workspace_bytes < need)
    return fail(MC_ERR_VALUE, "workspace too small: %zu < %zu bytes", a->workspace_bytes, need);
  if (a->batch == 0 || a->seq_len == 0) return MC_OK;
  return cuda_status(launch_attention(a, status, static_cast<cudaStream_t>(stream), nullptr), "mc_sparse_attention");
}

int mc_status_fetch(uint32_t* status, void* stream) {
  if (!status) return MC_OK;
  uint32_t h = 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(&h, status, 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_status(e, "mc_status_fetch");
  if (h) cudaMemsetAsync(status, 0, 4, s);
  if (h & MC_STATUS_BAD_INDEX) return fail(MC_ERR_FORMAT, "column index out of range");
  if (h & MC_STATUS_OVERFLOW) return fail(MC_ERR_OVERFLOW, "output exceeds int32");
  return MC_OK;
}

int mc_l2_flush(void* scratch, size_t bytes, void* stream) {
  // Write the scratch (evicts every line), then read it back: the L2 ends up full of
  // clean scratch lines, so the next kernel starts cold without inheriting a
  // write-back backlog of dirty lines.
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(scratch, 0x5A, bytes, s);
  if (e != cudaSuccess) return cuda_status(e, "mc_l2_flush");
  const int64_t n16 = static_cast<int64_t>(bytes / 16);
  l2_read_kernel<<<1184, 512, 0, s>>>(static_cast<const uint4*>(scratch), n16);
  return cuda_status(cudaGetLastError(), "mc_l2_flush");
}

}  // extern "C"
