// sddmm.cu -- block-sampled dense x dense integer product (SDDMM) for B200.
//
// out[blk, v] = sum_k A[r*V + v, k] * B[k, c]   for each pattern block (r, c),
// bit-exact with the reference kernels.sddmm (kernels.py:367-435).
//
// B is column-major, i.e. B^T is row-major with k contiguous, so both MMA
// operands are already k-major: no transposes. Per warp task
// (vector row r, a contiguous share of its blocks) 16 pattern blocks form the
// MMA M dimension of mma.sync m16n8k32, the V rows of A the N dimension, and k
// the reduction. 16/4-bit operands are split / sign-extended into int8 chunks
// exactly as in spmm.cu; chunk products are recombined in int64 with the
// reference's int32 checks (kernels.py:418-427).
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.h"

namespace mcube {
namespace {

constexpr int kWarps = 4;

__device__ __forceinline__ void tc_prefetch_l2(const void* ptr) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
}

// 16 consecutive k values of one operand row -> 4 int8-chunk words per chunk.
template <int BITS, bool ALIGNED>
__device__ __forceinline__ void load_k16(const uint32_t* __restrict__ words, int64_t row, int64_t K,
                                         int64_t k0, bool row_ok, uint32_t (&w)[2][4]) {
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int x = 0; x < 4; ++x) w[c][x] = 0u;
  if (!row_ok) return;
  if constexpr (ALIGNED) {
    const uint8_t* base = reinterpret_cast<const uint8_t*>(words) + (row * K * BITS) / 8;
    if constexpr (BITS == 8) {
      if (k0 < K) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(base + k0));
        w[0][0] = u.x; w[0][1] = u.y; w[0][2] = u.z; w[0][3] = u.w;
      }
    } else if constexpr (BITS == 16) {
      uint4 u0 = make_uint4(0, 0, 0, 0), u1 = make_uint4(0, 0, 0, 0);
      if (k0 < K) u0 = __ldg(reinterpret_cast<const uint4*>(base + 2 * k0));
      if (k0 + 8 < K) u1 = __ldg(reinterpret_cast<const uint4*>(base + 2 * k0 + 16));
      split16(u0.x, u0.y, w[0][0], w[1][0]);
      split16(u0.z, u0.w, w[0][1], w[1][1]);
      split16(u1.x, u1.y, w[0][2], w[1][2]);
      split16(u1.z, u1.w, w[0][3], w[1][3]);
    } else {  // 4-bit
      if (k0 < K) {
        const uint2 u = __ldg(reinterpret_cast<const uint2*>(base + k0 / 2));
        unpack_s4x8(u.x, w[0][0], w[0][1]);
        unpack_s4x8(u.y, w[0][2], w[0][3]);
      }
    }
  } else {
    // generic path: element-wise, any K / alignment
    int32_t e[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) e[i] = (k0 + i < K) ? fetch_packed(words, row * K + k0 + i, BITS) : 0;
    auto pack4 = [](int32_t a, int32_t b, int32_t c, int32_t d) {
      return (static_cast<uint32_t>(a) & 0xFF) | ((static_cast<uint32_t>(b) & 0xFF) << 8) |
             ((static_cast<uint32_t>(c) & 0xFF) << 16) | ((static_cast<uint32_t>(d) & 0xFF) << 24);
    };
    if constexpr (BITS == 16) {
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        w[0][x] = pack4(e[4 * x], e[4 * x + 1], e[4 * x + 2], e[4 * x + 3]);
        w[1][x] = pack4(e[4 * x] >> 8, e[4 * x + 1] >> 8, e[4 * x + 2] >> 8, e[4 * x + 3] >> 8);
      }
    } else {
#pragma unroll
      for (int x = 0; x < 4; ++x) w[0][x] = pack4(e[4 * x], e[4 * x + 1], e[4 * x + 2], e[4 * x + 3]);
    }
  }
}

template <int LB, int RB, int V, bool ALIGNED>
__global__ void __launch_bounds__(kWarps * 32)
sddmm_kernel(const SddmmParams p) {
  constexpr int LC = (LB == 16) ? 2 : 1;
  constexpr int RC = (RB == 16) ? 2 : 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();  // inputs may come from the previous kernel on the stream
  const int64_t task = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
  if (task >= p.tasks) return;
  const int64_t per_batch = p.vrows * p.splits;
  const int64_t b = task / per_batch;
  const int64_t rem = task - b * per_batch;
  const int64_t r = rem / p.splits;
  const int split = static_cast<int>(rem - r * p.splits);
  // Speculative column-index load for this warp's first group, positioned as if all rows
  // had n_blocks / vrows blocks (exact for uniform patterns); it overlaps the row-offset
  // round trip and is discarded when the real offsets disagree.
  const int64_t lo_g = (r * p.n_blocks) / p.vrows, hi_g = ((r + 1) * p.n_blocks) / p.vrows;
  const int64_t ng_g = (hi_g - lo_g + 15) >> 4;
  const int64_t gb_g = (ng_g * split) / p.splits;
  const int64_t blk0_g = lo_g + gb_g * 16;
  const uint32_t spec_col =
      (gb_g < (ng_g * (split + 1)) / p.splits && blk0_g + lane < hi_g) ? __ldg(p.col_indices + blk0_g + lane) : 0u;
  const int64_t lo = p.row_offsets[r], hi = p.row_offsets[r + 1];
  const bool spec_ok = (lo == lo_g) && (hi == hi_g);
  const int64_t nb = hi - lo;
  const int64_t ngroups = (nb + 15) >> 4;
  const int64_t gbeg = (ngroups * split) / p.splits, gend = (ngroups * (split + 1)) / p.splits;
  const uint32_t* __restrict__ A = p.a_words + b * p.a_stride;
  const uint32_t* __restrict__ Bt = p.b_words + b * p.b_stride;
  const int64_t arow = r * V + g;
  const bool a_ok = g < V;
  double alpha = 0.0;
  if (p.out_f16) alpha = p.alpha ? p.alpha[b] : p.alpha_host;
  const float alpha_f = static_cast<float>(alpha);
  bool overflow = false;

  // one group of 16 pattern blocks starting at CSR position blk0: gathers + MMAs into acc
  auto compute = [&](int nvalid, uint32_t mycol, int (&acc)[LC][RC][4]) {
    if (lane >= nvalid) mycol = 0u;
    if (lane < nvalid && mycol >= static_cast<uint32_t>(p.N)) {
      flag_status(p.status, MC_STATUS_BAD_INDEX);
      mycol = 0u;
    }
    const uint32_t c_lo = __shfl_sync(0xffffffffu, mycol, g);
    const uint32_t c_hi = __shfl_sync(0xffffffffu, mycol, g + 8);
    const bool lo_ok = g < nvalid, hi_ok = g + 8 < nvalid;

#pragma unroll
    for (int c = 0; c < LC; ++c)
#pragma unroll
      for (int j = 0; j < RC; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[c][j][e] = 0;

    // K in chunks of 256: all loads of a chunk are issued before its MMAs (memory-level parallelism)
    for (int64_t kc = 0; kc < p.K; kc += 256) {
      uint32_t wa[4][2][4], wl[4][2][4], wh[4][2][4];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int64_t k0 = kc + 64 * s + 16 * t;
        load_k16<LB, ALIGNED>(A, arow, p.K, k0, a_ok, wa[s]);
        load_k16<RB, ALIGNED>(Bt, c_lo, p.K, k0, lo_ok, wl[s]);
        load_k16<RB, ALIGNED>(Bt, c_hi, p.K, k0, hi_ok, wh[s]);
      }
#pragma unroll
      for (int s = 0; s < 4; ++s) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
#pragma unroll
          for (int j = 0; j < RC; ++j) {
#pragma unroll
            for (int c = 0; c < LC; ++c) {
              const uint32_t a0 = wl[s][j][2 * half], a2 = wl[s][j][2 * half + 1];
              const uint32_t a1 = wh[s][j][2 * half], a3 = wh[s][j][2 * half + 1];
              const uint32_t b0 = wa[s][c][2 * half], b1 = wa[s][c][2 * half + 1];
              const bool au = (RB == 16) && (j == 0);
              const bool bu = (LB == 16) && (c == 0);
              if (au && bu) mma16832<true, true>(acc[c][j], a0, a1, a2, a3, b0, b1);
              else if (au) mma16832<true, false>(acc[c][j], a0, a1, a2, a3, b0, b1);
              else if (bu) mma16832<false, true>(acc[c][j], a0, a1, a2, a3, b0, b1);
              else mma16832<false, false>(acc[c][j], a0, a1, a2, a3, b0, b1);
            }
          }
        }
      }
    }

  };
  auto store = [&](int64_t blk0, int nvalid, const int (&acc)[LC][RC][4]) {
    // epilogue: D[m = block, n = v]; c0:(g,2t) c1:(g,2t+1) c2:(g+8,2t) c3:(g+8,2t+1)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int m = (e < 2) ? g : g + 8;
      const int v = 2 * t + (e & 1);
      long long total = 0;
#pragma unroll
      for (int j = 0; j < RC; ++j) {
        long long tj;
        if constexpr (LC == 2) {
          const long long lo_p = acc[0][j][e];
          const long long hi_p = 256LL * acc[1][j][e];
          if constexpr (V == 8) overflow |= !fits_i32(hi_p);
          else overflow |= !fits_i32(lo_p + hi_p);
          tj = lo_p + hi_p;
        } else {
          tj = acc[0][j][e];
        }
        total += tj << (8 * j);
      }
      if (m < nvalid && v < V) {
        overflow |= !fits_i32(total);
        const int64_t o = (blk0 + m) * V + v;
        if (p.out) p.out[b * p.out_stride + o] = static_cast<int32_t>(total);
        if (p.out_f16) p.out_f16[b * p.f16_stride + o] = f16_dequant(static_cast<int32_t>(total), alpha, alpha_f);
      }
    }
  };

  int64_t gi = gbeg;
  // Speculative first group: with the uniform-row guess its column indices (spec_col) were
  // loaded alongside the row offsets, so the B^T gathers start without waiting for them;
  // the result is stored only if the real offsets confirm the guess (else recomputed).
  const int64_t ge_g = (ng_g * (split + 1)) / p.splits;
  if (gb_g < ge_g) {
    const int nvalid_g = static_cast<int>(min_i64(16, hi_g - blk0_g));
    int acc[LC][RC][4];
    compute(nvalid_g, spec_col, acc);
    if (spec_ok && gbeg == gb_g && gbeg < gend) {
      store(blk0_g, nvalid_g, acc);
      ++gi;
    }
  }
  for (; gi < gend; ++gi) {
    const int64_t blk0 = lo + gi * 16;
    const int nvalid = static_cast<int>(min_i64(16, hi - blk0));
    const uint32_t mycol = (lane < nvalid) ? __ldg(p.col_indices + blk0 + lane) : 0u;
    int acc[LC][RC][4];
    compute(nvalid, mycol, acc);
    store(blk0, nvalid, acc);
  }
  if (overflow) flag_status(p.status, MC_STATUS_OVERFLOW);
}

// 8-bit x 8-bit gather SDDMM for sparse patterns (C2 at <= 10 % density), software-
// pipelined across groups of 16 blocks: while group j's MMAs run, the B^T rows of group j+1
// are already in flight (two register buffers), and the column indices of the next two
// groups are loaded one pair ahead. A warp task is a run of `p.splits`-th of a vector row's
// groups; its V rows of A (K bytes each, the MMA B operand) are loaded once per task. Each
// lane loads 16 contiguous bytes [64 s + 16 t, +16) of its two gathered rows per 64-byte
// K chunk s; the reduction order inside a chunk is permuted identically for both operands
// (MMA k-step (s, half) = bytes 64 s + 16 t + 8 half + 0..7), which leaves the int32 sums
// exact. Stores: two 8-byte stores per lane, 256 contiguous bytes per warp instruction.
// int8 products cannot overflow int32 for K <= 33025 (emulation.py:108-113, checked on the
// host), so no overflow test is needed.
template <int V, int KS>
__global__ void __launch_bounds__(kWarps * 32)
sddmm_g8_kernel(const SddmmParams p) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  constexpr int K = 64 * KS;
  const int64_t task = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
  const int64_t per_batch = p.vrows * p.splits;
  const int64_t b = task / per_batch;
  const int64_t rem = task - b * per_batch;
  const int64_t r = rem / p.splits;
  const int split = static_cast<int>(rem - r * p.splits);
  // Uniform-row guess of this task's first blocks (exact for the reference generator's
  // patterns): its column indices are loaded together with the row offsets instead of
  // after them, and discarded if the offsets disagree. Before pdl_wait only L2 prefetches
  // are issued (L2 is the coherence point: they cannot make a later read stale).
  const int64_t lo_g = (r * p.n_blocks) / p.vrows, hi_g = ((r + 1) * p.n_blocks) / p.vrows;
  const int64_t ng_g = (hi_g - lo_g + 15) >> 4;
  const int64_t gb_g = (ng_g * split) / p.splits;
  const uint8_t* __restrict__ Ar = reinterpret_cast<const uint8_t*>(p.a_words + b * p.a_stride) +
                                   (r * V + (g < V ? g : 0)) * static_cast<int64_t>(K) + 16 * t;
  if (task < p.tasks) {
    if (lane == 0) tc_prefetch_l2(p.row_offsets + r);
    if (lane < 2 && lo_g + gb_g * 16 < p.n_blocks) tc_prefetch_l2(p.col_indices + lo_g + gb_g * 16 + 16 * lane);
    if (t == 0 && g < V) tc_prefetch_l2(Ar);
  }
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();
  if (task >= p.tasks) return;
  const int64_t q_g = gb_g * 16 + lane;
  const uint32_t spec = q_g < hi_g - lo_g ? __ldg(p.col_indices + lo_g + q_g) : 0u;
  uint4 af[KS];
#pragma unroll
  for (int s = 0; s < KS; ++s)
    af[s] = g < V ? __ldg(reinterpret_cast<const uint4*>(Ar + 64 * s)) : make_uint4(0u, 0u, 0u, 0u);
  const int64_t lo = p.row_offsets[r], hi = p.row_offsets[r + 1];
  const int64_t nb = hi - lo;
  const int64_t ngroups = (nb + 15) >> 4;
  const int64_t gbeg = (ngroups * split) / p.splits, gend = (ngroups * (split + 1)) / p.splits;
  if (gbeg >= gend) return;
  const uint32_t* __restrict__ cols = p.col_indices + lo;
  const uint8_t* __restrict__ Bt = reinterpret_cast<const uint8_t*>(p.b_words + b * p.b_stride) + 16 * t;
  int32_t* __restrict__ out = p.out + b * p.out_stride + lo * V;
  const uint32_t ncols = static_cast<uint32_t>(p.N);

  // columns of blocks [q0, q0 + 32) of the row (0 past the end; out-of-range ones flagged)
  auto check = [&](int64_t q, uint32_t c) -> uint32_t {
    if (q >= nb) return 0u;
    if (c >= ncols) {
      flag_status(p.status, MC_STATUS_BAD_INDEX);
      return 0u;
    }
    return c;
  };
  auto colload = [&](int64_t q0) -> uint32_t {
    const int64_t q = q0 + lane;
    return check(q, q < nb ? __ldg(cols + q) : 0u);
  };

  // the two gathered rows (blocks g and g + 8 of the group in half `h` of colreg)
  auto load = [&](uint32_t colreg, int h, uint4 (&xa)[KS], uint4 (&xb)[KS]) {
    const uint32_t c_lo = __shfl_sync(0xffffffffu, colreg, 16 * h + g);
    const uint32_t c_hi = __shfl_sync(0xffffffffu, colreg, 16 * h + g + 8);
    const uint8_t* ra = Bt + static_cast<size_t>(c_lo) * K;
    const uint8_t* rb = Bt + static_cast<size_t>(c_hi) * K;
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      xa[s] = __ldg(reinterpret_cast<const uint4*>(ra + 64 * s));
      xb[s] = __ldg(reinterpret_cast<const uint4*>(rb + 64 * s));
    }
  };
  auto compute_store = [&](int64_t gi, const uint4 (&xa)[KS], const uint4 (&xb)[KS]) {
    int acc[4] = {0, 0, 0, 0};
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      mma16832<false, false>(acc, xa[s].x, xb[s].x, xa[s].y, xb[s].y, af[s].x, af[s].y);
      mma16832<false, false>(acc, xa[s].z, xb[s].z, xa[s].w, xb[s].w, af[s].z, af[s].w);
    }
    const int64_t blk0 = gi * 16;
    const int64_t nvalid = nb - blk0;
    if (2 * t < V) {
      if (g < nvalid) *reinterpret_cast<int2*>(out + (blk0 + g) * V + 2 * t) = make_int2(acc[0], acc[1]);
      if (g + 8 < nvalid) *reinterpret_cast<int2*>(out + (blk0 + g + 8) * V + 2 * t) = make_int2(acc[2], acc[3]);
    }
  };

  uint4 fa[KS], fb[KS], ga[KS], gb[KS];
  const bool spec_ok = lo == lo_g && hi == hi_g;  // then gbeg == gb_g and spec holds its columns
  uint32_t colreg = spec_ok ? check(gbeg * 16 + lane, spec) : colload(gbeg * 16);
  load(colreg, 0, fa, fb);
  for (int64_t gi = gbeg; gi < gend; gi += 2) {
    const bool has1 = gi + 1 < gend, has2 = gi + 2 < gend;
    if (has1) load(colreg, 1, ga, gb);
    const uint32_t colnext = has2 ? colload((gi + 2) * 16) : 0u;
    compute_store(gi, fa, fb);
    if (has2) load(colnext, 0, fa, fb);
    if (has1) compute_store(gi + 1, ga, gb);
    colreg = colnext;
  }
}

// the pipelined 8-bit kernel takes int32 output, 8-bit operands, V in {4, 8} and
// K a multiple of 64 up to 256 with 16-byte aligned rows
bool sddmm_g8_supported(const SddmmParams& p) {
  return p.LB == 8 && p.RB == 8 && (p.V == 4 || p.V == 8) && p.out != nullptr && p.out_f16 == nullptr &&
         p.K > 0 && p.K % 64 == 0 && p.K <= 256 && (reinterpret_cast<uintptr_t>(p.a_words) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(p.b_words) & 15) == 0 && (reinterpret_cast<uintptr_t>(p.out) & 7) == 0 &&
         (p.a_stride * 4) % 16 == 0 && (p.b_stride * 4) % 16 == 0 && (p.out_stride % 2) == 0 &&
         !getenv("MCUBE_SDDMM_G8_OFF");
}

template <int V>
cudaError_t launch_g8_v(const SddmmParams& p, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>((p.tasks + kWarps - 1) / kWarps);
  if (grid == 0) return cudaSuccess;
  cudaError_t e;
  switch (p.K / 64) {
    case 1: e = launch_pdl(sddmm_g8_kernel<V, 1>, dim3(grid), dim3(kWarps * 32), 0, s, p); break;
    case 2: e = launch_pdl(sddmm_g8_kernel<V, 2>, dim3(grid), dim3(kWarps * 32), 0, s, p); break;
    case 3: e = launch_pdl(sddmm_g8_kernel<V, 3>, dim3(grid), dim3(kWarps * 32), 0, s, p); break;
    default: e = launch_pdl(sddmm_g8_kernel<V, 4>, dim3(grid), dim3(kWarps * 32), 0, s, p); break;
  }
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int LB, int RB, int V>
cudaError_t launch_v(const SddmmParams& p, cudaStream_t s) {
  const bool aligned = ((p.K * LB) % 128 == 0) && ((p.K * RB) % 128 == 0) &&
                       ((reinterpret_cast<uintptr_t>(p.a_words) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>(p.b_words) & 15) == 0) &&
                       ((p.a_stride * 4) % 16 == 0) && ((p.b_stride * 4) % 16 == 0);
  const unsigned grid = static_cast<unsigned>((p.tasks + kWarps - 1) / kWarps);
  if (grid == 0) return cudaSuccess;
  // same shared-memory carveout as the dense tcgen05 kernel: alternating launches of the two
  // (the C2 sweep) then need no L1/shared reconfiguration between kernels
  static bool carve = false;
  if (!carve) {
    cudaFuncSetAttribute(sddmm_kernel<LB, RB, V, true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(sddmm_kernel<LB, RB, V, false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    carve = true;
  }
  const cudaError_t e = aligned ? launch_pdl(sddmm_kernel<LB, RB, V, true>, dim3(grid), dim3(kWarps * 32), 0, s, p)
                                : launch_pdl(sddmm_kernel<LB, RB, V, false>, dim3(grid), dim3(kWarps * 32), 0, s, p);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int LB, int RB>
cudaError_t launch_lr(const SddmmParams& p, cudaStream_t s) {
  switch (p.V) {
    case 2: return launch_v<LB, RB, 2>(p, s);
    case 4: return launch_v<LB, RB, 4>(p, s);
    default: return launch_v<LB, RB, 8>(p, s);
  }
}

}  // namespace

// Path selection: the dense tcgen05 tile kernel reads 3*M*N*K/512 operand bytes through
// shared memory regardless of the pattern, the gather kernel reads n_blocks*K*bits/8;
// the crossover on B200 sits near a block density of 8%.
static int sddmm_path_override() {
  const char* e = getenv("MCUBE_SDDMM_PATH");
  if (!e) return 0;
  if (e[0] == 'd') return 1;  // dense
  if (e[0] == 'g') return 2;  // gather
  return 0;
}

// which kernel launch_sddmm runs (MC_SDDMM_PATH_*)
int sddmm_path(const SddmmParams& p) {
  const int ov = sddmm_path_override();
  const double density = (p.M > 0 && p.N > 0) ? static_cast<double>(p.n_blocks) * p.V / (static_cast<double>(p.M) * p.N) : 0.0;
  // K = 64 (attention heads, d = 64) stays on a gather kernel by default: with only two
  // K-steps per tile the dense path is bound by draining the whole accumulator tile.
  // Dense tile above a block density of 0.08 (the 16-bit / 4-bit gather kernel) or 0.15
  // (the pipelined 8-bit gather kernel; C2 90 %: 8.1 us gather vs 12.0 us dense tile).
  const bool g8 = sddmm_g8_supported(p);
  double dense_min = g8 ? 0.15 : 0.08;
  if (const char* e = getenv("MCUBE_SDDMM_DENSE_MIN")) dense_min = atof(e);
  if (ov != 2 && sddmm_tc_supported(p) && (ov == 1 || (density >= dense_min && p.K >= 128))) return MC_SDDMM_PATH_DENSE;
  return g8 ? MC_SDDMM_PATH_GATHER8 : MC_SDDMM_PATH_GATHER;
}

cudaError_t launch_sddmm(SddmmParams p, cudaStream_t stream) {
  const int path = sddmm_path(p);
  if (path == MC_SDDMM_PATH_DENSE) return launch_sddmm_tc(p, stream);
  // warps per vector row: about one group of 16 blocks each
  const double avg_groups = p.vrows ? (static_cast<double>(p.n_blocks) / p.vrows) / 16.0 : 0.0;
  if (path == MC_SDDMM_PATH_GATHER8) {
    // pipelined 8-bit kernel: as many warps per vector row as fit one wave of resident
    // warps (measured on C2 90/95/98 %: a second partial wave costs more than the longer
    // per-warp group runs; 4 warps per row there: 8.1 / 5.8 / ~4.8 us)
    static int wave_warps = 0;
    if (!wave_warps) {
      int dev = 0, sms = 148, per_sm = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sddmm_g8_kernel<8, 4>, kWarps * 32, 0);
      wave_warps = sms * (per_sm > 0 ? per_sm : 1) * kWarps;
    }
    const int64_t rows = static_cast<int64_t>(p.batch) * p.vrows;
    int64_t splits = rows > 0 ? wave_warps / rows : 1;
    const int64_t max_groups = static_cast<int64_t>(avg_groups + 0.999);
    if (splits > max_groups) splits = max_groups;
    if (const char* e = getenv("MCUBE_SDDMM_SPLITS")) splits = atoi(e);
    p.splits = static_cast<int>(splits < 1 ? 1 : (splits > 256 ? 256 : splits));
    p.tasks = rows * p.splits;
    return p.V == 8 ? launch_g8_v<8>(p, stream) : launch_g8_v<4>(p, stream);
  }
  // groups of 16 blocks per warp: 1, or 2 when one group per warp would need more than
  // one wave of resident warps (C2 95 %: 1.6 waves -> 0.86; 10.2 -> 8.9 us, same-box A/B)
  double gpw = 1.0;
  {
    static int wave_warps = 0;
    if (!wave_warps) {
      int dev = 0, sms = 148, per_sm = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sddmm_kernel<8, 8, 8, true>, kWarps * 32, 0);
      wave_warps = sms * (per_sm > 0 ? per_sm : 1) * kWarps;
    }
    const double warps1 = static_cast<double>(p.batch) * p.vrows * static_cast<int>(avg_groups + 0.999);
    if (warps1 > wave_warps) gpw = 2.0;
  }
  if (const char* e = getenv("MCUBE_SDDMM_GPW")) gpw = atof(e) > 0 ? atof(e) : 1.0;
  int splits = static_cast<int>(avg_groups / gpw + 0.999);
  p.splits = splits < 1 ? 1 : (splits > 256 ? 256 : splits);
  p.tasks = static_cast<int64_t>(p.batch) * p.vrows * p.splits;
  switch (p.LB * 100 + p.RB) {
    case 1616: return launch_lr<16, 16>(p, stream);
    case 808: return launch_lr<8, 8>(p, stream);
    case 404: return launch_lr<4, 4>(p, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mcube
