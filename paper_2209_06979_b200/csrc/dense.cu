// dense.cu -- SpMM "dense tile" path for moderate sparsity: SR-BCRS -> int8 planes
// (densify), packed RHS -> int8 planes (widen), then the tcgen05 GEMM of gemm_tc.cu.
//
// At C3 densities (2-30 % of the vectors present) a B200 SpMM is bound by gathering
// one B row per stored vector through L2 (~5 TB/s); the same product
// as a dense int8 GEMM over the densified LHS costs M*K*N MACs at tensor-core rate
// plus one pass over M*K bytes. Values and products are identical: each plane holds
// exact int8 chunks (qint.py:185-225 split: low byte unsigned, high part signed) and
// the GEMM recombines chunk products in int64 with the reference's int32 checks.
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.h"

namespace mcube {
namespace {

constexpr int kKC = 4096;  // densified columns per block (shared-memory row chunk)
// staged value words per batch: ~2048 positions' worth (a C3 row at 70 % sparsity has 1229),
// at most 16 KB -- small stages let V = 2 / 4 blocks reach 8 per SM (one wave fewer)
__host__ __device__ constexpr int densify_vb(int v, int lb) { return v * lb * 64 < 4096 ? v * lb * 64 : 4096; }

// value position q of a row -> stored index position (SHUFFLE_PERMUTATION^-1, sparse_format.py:222-230)
__device__ __forceinline__ int64_t index_pos(int64_t q, bool shuffled) {
  if (!shuffled) return q;
  const int w = static_cast<int>(q & 7);
  return (q & ~7LL) | ((w >> 1) | ((w & 1) << 2));
}

// grid (vrows, ceil(K / kKC)): the V scalar rows of vector row r over columns
// [k0, k0 + kKC), built in shared memory, written as LC int8 planes [M x K].
template <int LB, int V>
__global__ void __launch_bounds__(256)
densify_kernel(const SpmmParams p, int8_t* __restrict__ plane0, int8_t* __restrict__ plane1, int after_widen) {
  constexpr int LC = LB >= 12 ? 2 : 1;
  constexpr int kVB = densify_vb(V, LB);
  extern __shared__ __align__(16) uint8_t sm[];  // [LC][V][kKC] planes + kVB staged value words
  if (threadIdx.x == 0) pdl_launch_dependents();
  // after_widen: the previous kernel is widen_kernel, which released this grid only after
  // every kernel before it completed (its own griddepcontrol.wait), so the SR-BCRS inputs
  // are ready and the two passes overlap; the wait moves to the end so that this grid
  // completes after widen does (the GEMM's griddepcontrol.wait then covers both)
  if (!after_widen) pdl_wait();
  const int64_t r = blockIdx.x;
  const int64_t k0 = static_cast<int64_t>(blockIdx.y) * kKC;
  const int kc = static_cast<int>((p.K - k0 < kKC) ? p.K - k0 : kKC);
  const int64_t pb = p.row_begin[r];
  const int64_t n_true = p.row_end[r] - pb;
  const bool shuffled = p.shuffled != 0;
  uint4* sm4 = reinterpret_cast<uint4*>(sm);
  for (int i = threadIdx.x; i < LC * V * kKC / 16; i += blockDim.x) sm4[i] = make_uint4(0, 0, 0, 0);
  const int S = p.S;
  // the row's values are one contiguous run of (stored * V) LB-bit elements starting at
  // element pb * V (rows start on stride boundaries); stage them in shared memory in
  // batches of kVB words so the scatter below reads shared memory, not 8 strided global
  // bytes per entry
  uint32_t* vals = reinterpret_cast<uint32_t*>(sm + LC * V * kKC);
  const int64_t bit0 = pb * V * LB;
  int64_t per_batch = (static_cast<int64_t>(kVB) * 32 - 32) / (V * LB) / S * S;  // positions per batch
  if (per_batch > 8 * static_cast<int64_t>(blockDim.x)) per_batch = (8 * blockDim.x) / S * S;  // kQ per thread
  for (int64_t qb = 0; qb < n_true; qb += per_batch) {
    const int64_t qe = (qb + per_batch < n_true) ? qb + per_batch : n_true;
    const int64_t w0 = (bit0 + qb * V * LB) >> 5;
    const int64_t qe_s = ((qe + S - 1) / S) * S;  // whole stride blocks: element (v, q) spans V*S per stride
    const int64_t w1 = ((bit0 + qe_s * V * LB) + 31) >> 5;
    // staged words start at word w0: the batch's first element sits stage_skew bytes in
    const int stage_skew = static_cast<int>(((bit0 + qb * V * LB) - (w0 << 5)) >> 3);
    __syncthreads();  // previous batch's scatter (and the zero fill) done
    // 16-byte cp.async, all in flight together (w0 is 4-word aligned: rows start on stride
    // boundaries, pb * V * LB is a multiple of 128 bits); the tail chunk is zero-filled
    {
      const uint32_t vs = smem_u32(vals);
      const int64_t nw = w1 - w0;
      for (int64_t c = threadIdx.x; c * 4 < nw; c += blockDim.x) {
        const int64_t left = nw - c * 4;
        const uint32_t bytes = left >= 4 ? 16u : static_cast<uint32_t>(left) * 4u;
        cp_async16(vs + static_cast<uint32_t>(c) * 16, p.lhs_words + w0 + c * 4, bytes);
      }
      cp_async_commit();
    }
    // this thread's column indices of the batch, loaded together with the staged values
    constexpr int kQ = 8;
    uint32_t cols[kQ];
#pragma unroll
    for (int u = 0; u < kQ; ++u) {
      const int q = static_cast<int>(qb) + static_cast<int>(threadIdx.x) + u * static_cast<int>(blockDim.x);
      cols[u] = q < qe ? __ldg(p.col_indices + pb + index_pos(q, shuffled)) : kSentinel;
    }
    cp_async_wait<0>();
    __syncthreads();
    // positions and element offsets of a row fit 32 bits (n_true <= K < 2^31); strides are
    // powers of two in every reference plan (tile k), so q / S and q % S are a shift and a mask
    const bool s_pow2 = (S & (S - 1)) == 0;
    const int s_sh = __ffs(S) - 1;
    const int qb32 = static_cast<int>(qb);
#pragma unroll
    for (int u = 0; u < kQ; ++u) {
      const int q = qb32 + static_cast<int>(threadIdx.x) + u * static_cast<int>(blockDim.x);
      if (q >= qe) continue;
      const uint32_t col = cols[u];
      if (col >= static_cast<uint32_t>(p.K)) {
        if (col != kSentinel) flag_status(p.status, MC_STATUS_BAD_INDEX);
        continue;
      }
      const int c = static_cast<int>(static_cast<int64_t>(col) - k0);
      if (c < 0 || c >= kc) continue;
      // element (v, q) of the row: stride q / S, offset v * S + q % S (sparse_format.py:131-139)
      const int sq = s_pow2 ? (q >> s_sh) : q / S;
      const int e0 = sq * V * S + (q - sq * S);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        // element offset inside the staged run (fits 32 bits: <= kVB words)
        const int eo = e0 - qb32 * V + v * S;
        int32_t x;
        if constexpr (LB == 8) {
          x = reinterpret_cast<const int8_t*>(vals)[eo + stage_skew];
        } else if constexpr (LB == 16) {
          x = reinterpret_cast<const int16_t*>(vals)[eo + stage_skew / 2];
        } else {  // 4 / 12-bit: generic bit extraction (32-bit arithmetic)
          const int bit = eo * LB + stage_skew * 8;
          const int wi = bit >> 5, sh = bit & 31;
          uint64_t u = static_cast<uint64_t>(vals[wi]) >> sh;
          if (sh + LB > 32) u |= static_cast<uint64_t>(vals[wi + 1]) << (32 - sh);
          x = static_cast<int32_t>(static_cast<uint32_t>(u) & ((1u << LB) - 1u));
          x = (x ^ (1 << (LB - 1))) - (1 << (LB - 1));
        }
        if constexpr (LC == 1) {
          sm[v * kKC + c] = static_cast<uint8_t>(x);
        } else {
          sm[v * kKC + c] = static_cast<uint8_t>(x & 0xFF);      // low byte, unsigned chunk
          sm[(V + v) * kKC + c] = static_cast<uint8_t>(x >> 8);  // high part, signed chunk
        }
      }
    }
  }
  // copy-out by the bulk-copy engine: one kc-byte row per plane row (kc % 16 == 0 and
  // 16-byte aligned rows: the dense path requires K % 128 == 0)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < LC * V) {
    const int pl = threadIdx.x / V, v = threadIdx.x - pl * V;
    int8_t* dst = (pl == 0 ? plane0 : plane1) + (r * V + v) * p.K + k0;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(sm + threadIdx.x * kKC)), "r"(static_cast<uint32_t>(kc)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  if (after_widen) pdl_wait();
}

// packed R-bit RHS [K x N] -> RC int8 planes (R4: sign-extended nibbles; R16: low byte
// unsigned + high byte signed). 16 elements per thread.
template <int RB>
__global__ void widen_kernel(const uint32_t* __restrict__ words, int64_t n16, int8_t* __restrict__ plane0,
                             int8_t* __restrict__ plane1) {
  pdl_wait();  // every earlier kernel complete before densify_kernel (dependent) is released
  if (threadIdx.x == 0) pdl_launch_dependents();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n16) return;
  if constexpr (RB == 4) {
    const uint2 w = reinterpret_cast<const uint2*>(words)[i];
    uint32_t e0, o0, e1, o1;
    unpack_s4x8(w.x, e0, o0);
    unpack_s4x8(w.y, e1, o1);
    // interleave even/odd bytes back into element order
    const uint32_t a0 = prmt(e0, o0, 0x5140), a1 = prmt(e0, o0, 0x7362);
    const uint32_t a2 = prmt(e1, o1, 0x5140), a3 = prmt(e1, o1, 0x7362);
    reinterpret_cast<uint4*>(plane0)[i] = make_uint4(a0, a1, a2, a3);
  } else {  // RB == 16
    const uint4 w0 = reinterpret_cast<const uint4*>(words)[2 * i];
    const uint4 w1 = reinterpret_cast<const uint4*>(words)[2 * i + 1];
    uint32_t lo[4], hi[4];
    split16(w0.x, w0.y, lo[0], hi[0]);
    split16(w0.z, w0.w, lo[1], hi[1]);
    split16(w1.x, w1.y, lo[2], hi[2]);
    split16(w1.z, w1.w, lo[3], hi[3]);
    reinterpret_cast<uint4*>(plane0)[i] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    reinterpret_cast<uint4*>(plane1)[i] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  }
}

template <int LB, int V>
cudaError_t launch_densify_v(const SpmmParams& p, int8_t* a0, int8_t* a1, cudaStream_t s, int after_widen) {
  constexpr int LC = LB >= 12 ? 2 : 1;
  const int smem = LC * V * kKC + densify_vb(V, LB) * 4;
  auto k = densify_kernel<LB, V>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  dim3 grid(static_cast<unsigned>(p.vrows), static_cast<unsigned>((p.K + kKC - 1) / kKC));
  const cudaError_t e = launch_pdl(k, grid, dim3(256), smem, s, p, a0, a1, after_widen);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int LB>
cudaError_t launch_densify_l(const SpmmParams& p, int8_t* a0, int8_t* a1, cudaStream_t s, int after_widen) {
  switch (p.V) {
    case 2: return launch_densify_v<LB, 2>(p, a0, a1, s, after_widen);
    case 4: return launch_densify_v<LB, 4>(p, a0, a1, s, after_widen);
    default: return launch_densify_v<LB, 8>(p, a0, a1, s, after_widen);
  }
}

}  // namespace

// densify_kernel stages a row's values in batches of whole strides; a stride wider than
// one batch cannot be staged (the batch loop would not advance), so such problems take
// the gather kernels.
bool densify_stride_ok(const SpmmParams& p) {
  if (p.S <= 0 || p.V <= 0 || p.LB <= 0) return false;
  int64_t per_batch = (static_cast<int64_t>(densify_vb(p.V, p.LB)) * 32 - 32) / (static_cast<int64_t>(p.V) * p.LB);
  if (per_batch > 8 * 256) per_batch = 8 * 256;  // kQ positions per thread x 256 threads
  return per_batch / p.S * p.S >= p.S;
}

int dense_lhs_planes(int lb) { return lb >= 12 ? 2 : 1; }
int dense_rhs_planes(int rb) { return rb == 16 ? 2 : 1; }

// Workspace of the dense path: LC planes of M x K int8 (+ RC planes of K x N int8 unless
// the RHS already is int8). 0 when the problem is not eligible.
size_t dense_spmm_workspace(const SpmmParams& p) {
  if (!dense_spmm_eligible(p)) return 0;
  const size_t a = static_cast<size_t>(dense_lhs_planes(p.LB)) * p.M * p.K;
  const size_t b = p.RB == 8 ? 0 : static_cast<size_t>(dense_rhs_planes(p.RB)) * p.K * p.N;
  return a + b + 1024;
}

cudaError_t launch_dense_spmm(SpmmParams p, void* workspace, cudaStream_t stream) {
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  ws += (1024 - (reinterpret_cast<uintptr_t>(ws) & 1023)) & 1023;
  const size_t plane_a = static_cast<size_t>(p.M) * p.K;
  int8_t* a0 = reinterpret_cast<int8_t*>(ws);
  int8_t* a1 = dense_lhs_planes(p.LB) == 2 ? a0 + plane_a : nullptr;
  uint8_t* bws = ws + dense_lhs_planes(p.LB) * plane_a;
  const int8_t* b0 = reinterpret_cast<const int8_t*>(p.rhs_words);
  const int8_t* b1 = nullptr;
  cudaError_t e;
  // widen (R4 / R16) first: densify then runs alongside it (densify_kernel's after_widen)
  if (p.RB != 8) {
    const size_t plane_b = static_cast<size_t>(p.K) * p.N;
    int8_t* w0 = reinterpret_cast<int8_t*>(bws);
    int8_t* w1 = p.RB == 16 ? w0 + plane_b : nullptr;
    const int64_t n16 = static_cast<int64_t>(plane_b / 16);
    const unsigned grid = static_cast<unsigned>((n16 + 255) / 256);
    if (p.RB == 4) e = launch_pdl(widen_kernel<4>, dim3(grid), dim3(256), 0, stream, p.rhs_words, n16, w0, w1);
    else e = launch_pdl(widen_kernel<16>, dim3(grid), dim3(256), 0, stream, p.rhs_words, n16, w0, w1);
    count_launch();
    if (e != cudaSuccess) return e;
    b0 = w0;
    b1 = w1;
  }
  const int after_widen = p.RB != 8 ? 1 : 0;
  switch (p.LB) {
    case 4: e = launch_densify_l<4>(p, a0, a1, stream, after_widen); break;
    case 8: e = launch_densify_l<8>(p, a0, a1, stream, after_widen); break;
    case 12: e = launch_densify_l<12>(p, a0, a1, stream, after_widen); break;
    default: e = launch_densify_l<16>(p, a0, a1, stream, after_widen); break;
  }
  if (e != cudaSuccess) return e;
  return launch_gemm_tc(p, a0, a1, b0, b1, stream);
}

}  // namespace mcube
