// pack.cu -- device SR-BCRS packer and index shuffle.
//
// bcrs_to_srbcrs (sparse_format.py:284-315): per vector row, stored =
// ceil(true / S) * S vectors; begin = running sum (exclusive scan); indices are
// sentinel padded; each stride of S vectors is stored as V rows of S elements
// (element (v, j) of stride s at s*V*S + v*S + j), padding slots zero.
// shuffle_indices (sparse_format.py:373-385): new[p] = old[P[p]] within every
// block of 8, P = SHUFFLE_PERMUTATION (tile_engine.py:35).
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "kernels.h"

namespace mcube {
namespace {

constexpr int kScanThreads = 1024;

__global__ void __launch_bounds__(kScanThreads)
srbcrs_plan_kernel(const int64_t* __restrict__ offs, int64_t vrows, int stride,
                   int64_t* __restrict__ begin, int64_t* __restrict__ end, int64_t* __restrict__ total) {
  using Scan = cub::BlockScan<long long, kScanThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < vrows; base += kScanThreads) {
    const int64_t r = base + threadIdx.x;
    long long stored = 0, tru = 0;
    if (r < vrows) {
      tru = offs[r + 1] - offs[r];
      stored = ((tru + stride - 1) / stride) * stride;
    }
    long long excl, agg;
    Scan(tmp).ExclusiveSum(stored, excl, agg);
    if (r < vrows) {
      begin[r] = carry + excl;
      end[r] = carry + excl + tru;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// last index r with a[r] <= x (a non-decreasing, a[0] <= x)
__device__ __forceinline__ int64_t upper_row(const int64_t* __restrict__ a, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;  // answer in [lo, hi)
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid;
    else hi = mid;
  }
  return lo;
}

__global__ void srbcrs_fill_idx_kernel(const int64_t* __restrict__ offs, const uint32_t* __restrict__ cols,
                                       int64_t vrows, int64_t n_blocks, const int64_t* __restrict__ begin,
                                       int64_t stored_total, uint32_t* __restrict__ col_out) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= stored_total) return;
  const int64_t r = upper_row(begin, vrows, p);
  const int64_t j = p - begin[r];
  const int64_t tru = offs[r + 1] - offs[r];
  col_out[p] = (j < tru) ? cols[offs[r] + j] : kSentinel;
}

__device__ __forceinline__ uint32_t extract_raw(const uint32_t* __restrict__ w, int64_t e, int bits) {
  if (bits == 32) return w[e];
  const int64_t bit = e * bits;
  const int64_t wi = bit >> 5;
  const int sh = static_cast<int>(bit & 31);
  uint64_t v = static_cast<uint64_t>(w[wi]) >> sh;
  if (sh + bits > 32) v |= static_cast<uint64_t>(w[wi + 1]) << (32 - sh);
  return static_cast<uint32_t>(v) & ((1u << bits) - 1u);
}

// one thread per output word; each word gathers the (bit slices of) elements it covers
__global__ void srbcrs_fill_val_kernel(const int64_t* __restrict__ offs, int64_t vrows, int V, int S,
                                       const int64_t* __restrict__ begin, const int64_t* __restrict__ end,
                                       int64_t n_elems, const uint32_t* __restrict__ src, int bits,
                                       uint32_t* __restrict__ dst, int64_t n_words) {
  const int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (w >= n_words) return;
  const int64_t bit0 = w * 32;
  const int64_t e_first = bit0 / bits;
  const int64_t e_last = min_i64((bit0 + 31) / bits, n_elems - 1);
  uint64_t acc = 0;
  for (int64_t e = e_first; e <= e_last; ++e) {
    const int64_t vs = static_cast<int64_t>(V) * S;
    const int64_t s = e / vs;
    const int64_t within = e - s * vs;
    const int64_t v = within / S;
    const int64_t jj = within - v * S;
    const int64_t pst = s * S + jj;
    const int64_t r = upper_row(begin, vrows, pst);
    const int64_t j = pst - begin[r];
    uint32_t x = 0;
    if (j < end[r] - begin[r]) x = extract_raw(src, (offs[r] + j) * V + v, bits);
    const int64_t sh = e * bits - bit0;  // may be negative for the straddling first element
    const uint64_t xv = static_cast<uint64_t>(x);
    if (sh >= 0) acc |= xv << sh;
    else acc |= xv >> (-sh);
  }
  dst[w] = static_cast<uint32_t>(acc);
}

// raw 64-bit values (float64 / int64 block values, e.g. dequantised SDDMM outputs): one
// thread per output element, zero for padding slots (sparse_format.py:303-304 keeps dtype)
__global__ void srbcrs_fill_val64_kernel(const int64_t* __restrict__ offs, int64_t vrows, int V, int S,
                                         const int64_t* __restrict__ begin, const int64_t* __restrict__ end,
                                         int64_t n_elems, const uint2* __restrict__ src, uint2* __restrict__ dst) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n_elems) return;
  const int64_t vs = static_cast<int64_t>(V) * S;
  const int64_t s = e / vs;
  const int64_t within = e - s * vs;
  const int64_t v = within / S;
  const int64_t pst = s * S + (within - v * S);
  const int64_t r = upper_row(begin, vrows, pst);
  const int64_t j = pst - begin[r];
  dst[e] = (j < end[r] - begin[r]) ? src[(offs[r] + j) * V + v] : make_uint2(0u, 0u);
}

__global__ void shuffle_kernel(const uint32_t* __restrict__ in, int64_t n, uint32_t* __restrict__ out) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int w = static_cast<int>(p & 7);
  const int src = (w < 4) ? 2 * w : 2 * (w - 4) + 1;  // SHUFFLE_PERMUTATION = (0,2,4,6,1,3,5,7)
  out[p] = in[(p & ~7LL) | src];
}

}  // namespace

cudaError_t launch_srbcrs_plan(const int64_t* row_offsets, int64_t vrows, int stride, int64_t* row_begin,
                               int64_t* row_end, int64_t* total, cudaStream_t stream) {
  srbcrs_plan_kernel<<<1, kScanThreads, 0, stream>>>(row_offsets, vrows, stride, row_begin, row_end, total);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_srbcrs_fill(const int64_t* row_offsets, const uint32_t* col_indices, int64_t vrows,
                               int64_t n_blocks, int V, int stride, const int64_t* row_begin,
                               const int64_t* row_end, int64_t stored_total, const uint32_t* values,
                               int bits, uint32_t* col_out, uint32_t* values_out, cudaStream_t stream) {
  (void)n_blocks;
  if (stored_total <= 0) return cudaSuccess;
  if (col_out) {
    const unsigned grid = static_cast<unsigned>((stored_total + 255) / 256);
    srbcrs_fill_idx_kernel<<<grid, 256, 0, stream>>>(row_offsets, col_indices, vrows, n_blocks, row_begin,
                                                     stored_total, col_out);
    count_launch();
  }
  if (values_out && bits == 64) {
    const int64_t n_elems = stored_total * V;
    const unsigned grid = static_cast<unsigned>((n_elems + 255) / 256);
    srbcrs_fill_val64_kernel<<<grid, 256, 0, stream>>>(row_offsets, vrows, V, stride, row_begin, row_end, n_elems,
                                                       reinterpret_cast<const uint2*>(values),
                                                       reinterpret_cast<uint2*>(values_out));
    count_launch();
  } else if (values_out) {
    const int64_t n_elems = stored_total * V;
    const int64_t n_words = (n_elems * bits + 31) / 32;
    const unsigned grid = static_cast<unsigned>((n_words + 255) / 256);
    srbcrs_fill_val_kernel<<<grid, 256, 0, stream>>>(row_offsets, vrows, V, stride, row_begin, row_end,
                                                     n_elems, values, bits, values_out, n_words);
    count_launch();
  }
  return cudaGetLastError();
}

cudaError_t launch_shuffle(const uint32_t* in, int64_t n, uint32_t* out, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  shuffle_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(in, n, out);
  count_launch();
  return cudaGetLastError();
}

}  // namespace mcube
