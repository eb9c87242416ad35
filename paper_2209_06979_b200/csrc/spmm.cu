// spmm.cu -- SR-BCRS x dense integer SpMM for B200 (sm_100a).
//
// Computes out[M x N] = A (SR-BCRS, L-bit, vector length V) x B (K x N row-major,
// R-bit), bit-exact with the reference kernels.spmm (kernels.py:293-340).
//
// Formulation (transposed, B200 view of PAPER.md §4.2): per vector row r and a
// 64-column tile, D^T[n, v] = sum_k B[idx_k, n] * A_r[v, k], so dense columns are
// the MMA M dimension (16 per mma.sync m16n8k32), the V rows are MMA N (8) and the
// gathered k is MMA K (32). Every operand chunk is int8 (s8/u8): 16-bit operands
// split into (u8 low byte, s8 high byte) chunks, 4-bit operands are sign-extended
// to s8, 12-bit LHS values split like 16-bit ones (qint.py:209-225). Chunk products
// live in separate exact int32 accumulators and are recombined with shift-add in
// the epilogue, where the reference's int32 checks (kernels.py:286-288,
// tile_engine.py:246-247) are evaluated exactly in int64.
//
// Data movement (the Alg. 1 prefetch pipeline of PAPER.md:272-301, kernels.py:343-364):
// each warp owns a (row, 64-column tile) task and runs a STAGES-deep cp.async ring:
// stage s holds the 32 gathered B-row segments of k-step s (zero-filled for
// sentinel/padding slots, kernels.py:224-236) plus the matching 2 x V x 16 LHS
// values. The gathered rows are stored in a slot order and XOR swizzle that makes
// the consumer's shared-memory reads bank-conflict free for any column indices.
// Consumers transpose 4x4 byte blocks with PRMT into the k-major
// MMA fragments. Column indices for the next issue are prefetched one step ahead.
#include <cuda_fp16.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace mcube {

namespace {

constexpr int kWarps = 4;
#ifndef MCUBE_SPMM_KSTAGES
#define MCUBE_SPMM_KSTAGES 4  // 2/3/4 measured within 2 % at C5 and C3 (same-box A/B)
#endif
constexpr int kStages = MCUBE_SPMM_KSTAGES;  // cp.async ring depth per warp
constexpr int kSubN = 64;  // dense columns per MMA sub-tile (4 x m16 tiles)

// A warp task covers NS sub-tiles of 64 columns: NS > 1 widens each gathered row
// segment to 128 bytes (one L2 line) for 4- and 8-bit RHS at large N.
// NIB: the reference's 4-bit-width plan chunks (emulation.py:80-83) -- one LHS chunk per
// nibble (lower nibbles u8, the top one s8) instead of byte chunks. Used for RB = 4 with an
// 8/12/16-bit LHS when K is large enough for one of the reference's per-nibble group checks
// (tile_engine.py:246-247 via kernels.py:265-275) to fire, or for a byte-chunk int32
// accumulator to wrap (spmm_needs_nibble_chunks).
template <int LB, int RB, int V, int NS, bool NIB = false>
struct SpmmCfg {
  static constexpr int LC = NIB ? LB / 4 : ((LB >= 12) ? 2 : 1);  // LHS int8 chunks
  static constexpr int RC = (RB == 16) ? 2 : 1;        // RHS int8 chunks
  static constexpr int TN = kSubN * NS;                // dense columns per task
  static constexpr int SUB = kSubN * RB / 8;           // bytes of one 64-column sub-segment
  static constexpr int RBYTES = TN * RB / 8;           // bytes of one gathered row segment
  static constexpr int CPR = RBYTES / 16;              // 16-byte copies per row segment
  static constexpr int ABYTES = 2 * LB;                // bytes of 16 LHS values
  static constexpr int B_STAGE = 32 * RBYTES;
  static constexpr int A_STAGE = 2 * V * ABYTES;
  static constexpr int STAGE = B_STAGE + A_STAGE;
  static constexpr int A_COPIES = A_STAGE / 8;         // 8-byte copies
};

__device__ __forceinline__ int slot_of(int kk) {
  return ((kk >> 4) << 4) | ((kk & 3) << 2) | ((kk >> 2) & 3);
}

template <int RBYTES>
__device__ __forceinline__ int swz(int t) {
  if constexpr (RBYTES == 128) return 32 * t;
  if constexpr (RBYTES == 64) return 32 * (t >> 1);
  return 0;
}

// value position -> stored index position (SHUFFLE_PERMUTATION inverse, sparse_format.py:222-230)
__device__ __forceinline__ int64_t idx_pos(int64_t q, bool shuffled) {
  if (!shuffled) return q;
  const int w = static_cast<int>(q & 7);
  return (q & ~7LL) | ((w >> 1) | ((w & 1) << 2));
}

#ifndef MCUBE_SPMM_MINB
#define MCUBE_SPMM_MINB 1
#endif
// X16 (RB = 4): a gathered nibble x enters the MMA as the byte 16 x (the nibble moved to the
// high half of its byte: one mask for odd columns, shift + mask for even ones) instead of
// a sign-extended s8, so every chunk product is 16 times the true one; the epilogue shifts
// the int32 accumulators right by 4. Exact while |16 * sum| < 2^31 (spmm_x16_ok).
template <int LB, int RB, int V, int NS, bool ALIGNED, bool NIB, bool X16 = false>
__global__ void __launch_bounds__(kWarps * 32, MCUBE_SPMM_MINB)
spmm_kernel(const SpmmParams p) {
  static_assert(!X16 || RB == 4, "X16 is the 4-bit RHS operand form");
  using C = SpmmCfg<LB, RB, V, NS, NIB>;
  static_assert(!NIB || (RB == 4 && LB >= 8), "nibble chunks are the 4-bit-width plans of an 8/12/16-bit LHS");
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();  // inputs may come from the previous kernel on the stream (e.g. the attention softmax)
  const int64_t task = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
  if (task >= p.tasks) return;
  const int64_t per_batch = p.vrows * p.ntiles;
  const int64_t b = task / per_batch;
  const int64_t rem = task - b * per_batch;
  const int64_t r = rem / p.ntiles;
  const int64_t c0 = (rem - r * p.ntiles) * C::TN;

  const uint32_t* __restrict__ lhs = p.lhs_words + b * p.lhs_stride;
  const uint32_t* __restrict__ rhs = p.rhs_words + b * p.rhs_stride;
  const int64_t p_begin = p.row_begin[r];
  const int64_t n_true = p.row_end[r] - p_begin;
  const int64_t stored = ((n_true + p.S - 1) / p.S) * p.S;
  const int64_t p_end = p_begin + stored;
  const int nsteps = static_cast<int>((stored + 31) >> 5);
  const bool shuffled = p.shuffled != 0;

  uint8_t* wbuf = smem + warp * (kStages * C::STAGE);
  const uint32_t wbuf_s = smem_u32(wbuf);

  // ---- producer state: column indices for this lane's copies, one step ahead ----
  // Column indices are staged through a per-warp smem ring: chunk c (stored positions
  // [p_begin + 256c, +256), i.e. k-steps 8c..8c+7) is fetched by cp.async one chunk ahead.
  uint32_t* sidx = reinterpret_cast<uint32_t*>(smem + kWarps * kStages * C::STAGE) + warp * 512;
  const uint32_t sidx_s = smem_u32(sidx);
  auto fetch_idx_chunk = [&](int c) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int ch = lane + 32 * u;
      const int64_t e0 = p_begin + 256LL * c + 4 * ch;
      const int64_t avail = p_end - e0;
      const uint32_t bytes = avail >= 4 ? 16u : (avail > 0 ? static_cast<uint32_t>(avail) * 4u : 0u);
      cp_async16(sidx_s + ((c & 1) * 256 + 4 * ch) * 4, p.col_indices + (bytes ? e0 : 0), bytes);
    }
  };
  // per-lane invariants of the producer (hoisted out of the k-loop)
  const int stored32 = static_cast<int>(stored);
  const uint64_t row_bytes = static_cast<uint64_t>(p.N) * RB / 8;
  const uint64_t c0_bytes = static_cast<uint64_t>(c0) * RB / 8;
  const uint8_t* rhs_b = reinterpret_cast<const uint8_t*>(rhs);
  const uint32_t kdim = static_cast<uint32_t>(p.K);
  // copy u of this lane moves 16-byte chunk ch of gathered row kk (CPR chunks per row);
  // computed on demand (a hoisted array per copy costs 5 registers per chunk at CPR = 8)
  auto kk_of = [&](int u) { return (lane + 32 * u) / C::CPR; };
  auto kkp_of = [&](int kk) {  // P^-1 within 8-groups
    return shuffled ? ((kk & ~7) | (((kk & 7) >> 1) | ((kk & 1) << 2))) : kk;
  };
  // LHS value copies: lane -> (half h, row v, 8-byte part), constant per lane
  constexpr int kAPer = C::ABYTES / 8;
  constexpr int kACopies = (C::A_COPIES + 31) / 32;
  const int64_t a_task_base = (p_begin / p.S) * V * p.S;  // element index of the row's first stride
  const int S = p.S;
  int a_blk = 0, a_within = 0;  // stride-block offset (elements) and offset within stride for pos = 32*step

  // every copy of this lane moves the same 16-byte chunk of its rows (CPR chunks per row)
  const uint32_t chx = static_cast<uint32_t>((lane % C::CPR) * 16);
  const uint32_t colofs = static_cast<uint32_t>(c0_bytes) + chx;
  const bool chunk_ok = c0_bytes + chx < row_bytes;
  bool bad_idx = false;  // an index >= K that is not the sentinel (flagged once, at the end)

  uint32_t nidx[C::CPR];
  auto load_idx = [&](int step) {
    const int base = ((step >> 3) & 1) * 256 + 32 * (step & 7);
#pragma unroll
    for (int u = 0; u < C::CPR; ++u)
      nidx[u] = (32 * step + kk_of(u) < stored32) ? sidx[base + kkp_of(kk_of(u))] : kSentinel;
  };

  auto issue = [&](int step) {
    if ((step & 7) == 0 && 256LL * ((step >> 3) + 1) < stored) {
      __syncwarp();  // every lane is done reading the ring slot being refilled
      fetch_idx_chunk((step >> 3) + 1);
    }
    const uint32_t sbase = wbuf_s + (step % kStages) * C::STAGE;
#pragma unroll
    for (int u = 0; u < C::CPR; ++u) {
      const int slot = slot_of(kk_of(u));
      const uint32_t dst = sbase + slot * C::RBYTES + (chx ^ swz<C::RBYTES>(slot & 3));
      const uint32_t col = nidx[u];
      const bool ok = col < kdim;
      bad_idx |= !ok && col != kSentinel;
      if constexpr (ALIGNED) {
        // branch-free: sentinel / out-of-range rows and chunks past N are zero-filled
        const bool go = ok && chunk_ok;
        const uint64_t off = go ? static_cast<uint64_t>(col) * row_bytes + colofs : 0ull;
        cp_async16(dst, rhs_b + off, go ? 16u : 0u);
      } else {
        const int ch = (lane + 32 * u) % C::CPR;
        // generic path: element-wise fetch for rows that are not 16-byte aligned
        constexpr int EPC = 128 / RB;  // elements per 16-byte chunk
        uint32_t wv[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int e = 0; e < EPC; ++e) {
          const int64_t n = c0 + ch * EPC + e;
          uint32_t x = 0;
          if (ok && n < p.N)
            x = static_cast<uint32_t>(fetch_packed(rhs, static_cast<int64_t>(col) * p.N + n, RB)) &
                ((1u << RB) - 1u);
          const int bit = e * RB;
          wv[bit >> 5] |= x << (bit & 31);
        }
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(dst), "r"(wv[0]), "r"(wv[1]),
                     "r"(wv[2]), "r"(wv[3]));
      }
    }
    // LHS values of this step: 2 halves x V rows x 16 elements, 8-byte copies.
    // Element (v, pos) lives at stride-block base + v*S + (pos mod S) (sparse_format.py:131-139).
    const uint32_t abase = sbase + C::B_STAGE;
    const uint8_t* lhs_b = reinterpret_cast<const uint8_t*>(lhs);
#pragma unroll
    for (int u = 0; u < kACopies; ++u) {
      const int q = lane + 32 * u;
      if (q < C::A_COPIES) {
        const int row = q / kAPer;  // row = h*V + v
        const int part = q % kAPer;
        const int h = row / V, v = row % V;
        int blk = a_blk, within = a_within + 16 * h;
        if (within >= S) {
          within -= S;
          blk += V * S;
        }
        const bool ok = 32 * step + 16 * h < stored32;
        const int64_t e = a_task_base + blk + v * S + within;
        const uint8_t* src = ok ? lhs_b + (e * LB) / 8 + part * 8 : lhs_b;
        cp_async8(abase + row * C::ABYTES + part * 8, src, ok ? 8u : 0u);
      }
    }
    // advance the stride cursor to pos = 32*(step+1)
    a_within += 32;
    while (a_within >= S) {
      a_within -= S;
      a_blk += V * S;
    }
  };

  int acc[NS][C::LC][C::RC][4][4];
#pragma unroll
  for (int st = 0; st < NS; ++st)
#pragma unroll
    for (int c = 0; c < C::LC; ++c)
#pragma unroll
      for (int j = 0; j < C::RC; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[st][c][j][q][e] = 0;

  if (nsteps > 0) {
    fetch_idx_chunk(0);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    load_idx(0);
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
      if (s < nsteps) {
        issue(s);
        if (s + 1 < nsteps) load_idx(s + 1);
      }
      cp_async_commit();
    }
  }

  for (int s = 0; s < nsteps; ++s) {
    const int nxt = s + kStages - 1;
    if (nxt < nsteps) {
      issue(nxt);
      if (nxt + 1 < nsteps) load_idx(nxt + 1);
    }
    cp_async_commit();
    cp_async_wait<kStages - 1>();
    __syncwarp();

    const uint8_t* sb = wbuf + (s % kStages) * C::STAGE;
    const uint8_t* sa = sb + C::B_STAGE;

    // ---- MMA B operand: LHS chunk words for kk = 16h + 4t .. +3 of row v = g ----
    uint32_t bf[C::LC > 2 ? C::LC : 2][2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint8_t* ar = sa + (h * V + (g < V ? g : 0)) * C::ABYTES;
      if constexpr (LB == 8) {
        bf[0][h] = *reinterpret_cast<const uint32_t*>(ar + 4 * t);
      } else if constexpr (LB == 4) {
        bf[0][h] = unpack_s4x4_ordered(*reinterpret_cast<const uint16_t*>(ar + 2 * t));
      } else if constexpr (LB == 16) {
        const uint2 w = *reinterpret_cast<const uint2*>(ar + 8 * t);
        split16(w.x, w.y, bf[0][h], bf[1][h]);
      } else {  // LB == 12: 4 elements = 48 bits starting at bit 48t
        const uint32_t* aw = reinterpret_cast<const uint32_t*>(ar);
        const int w0 = (3 * t) >> 1;
        const uint64_t bits = (static_cast<uint64_t>(aw[w0]) | (static_cast<uint64_t>(aw[w0 + 1]) << 32)) >>
                              (16 * (t & 1));
        uint32_t e0 = static_cast<uint32_t>(bits) & 0xFFFu, e1 = static_cast<uint32_t>(bits >> 12) & 0xFFFu;
        uint32_t e2 = static_cast<uint32_t>(bits >> 24) & 0xFFFu, e3 = static_cast<uint32_t>(bits >> 36) & 0xFFFu;
        // low byte (unsigned chunk), high nibble sign-extended (signed chunk)
        bf[0][h] = (e0 & 0xFF) | ((e1 & 0xFF) << 8) | ((e2 & 0xFF) << 16) | ((e3 & 0xFF) << 24);
        bf[1][h] = sext_nibble_bytes((e0 >> 8) | ((e1 >> 8) << 8) | ((e2 >> 8) << 16) | ((e3 >> 8) << 24));
      }
      if constexpr (NIB) {
        // byte chunks -> nibble chunks (qint.py:209-225 at w = 4): lower nibbles unsigned,
        // the top nibble signed
        if constexpr (LB == 8) {
          const uint32_t w = bf[0][h];
          bf[0][h] = w & 0x0F0F0F0Fu;
          bf[1][h] = sext_nibble_bytes((w >> 4) & 0x0F0F0F0Fu);
        } else {
          const uint32_t lo = bf[0][h], hi = bf[1][h];  // u8 low byte, s8 high part
          bf[0][h] = lo & 0x0F0F0F0Fu;
          bf[1][h] = (lo >> 4) & 0x0F0F0F0Fu;
          if constexpr (LB == 16) {
            bf[2][h] = hi & 0x0F0F0F0Fu;
            bf[3][h] = sext_nibble_bytes((hi >> 4) & 0x0F0F0F0Fu);
          } else {
            bf[2][h] = hi;  // 12-bit: the high part already is the signed top nibble
          }
        }
      }
      if (g >= V) {
#pragma unroll
        for (int c = 0; c < C::LC; ++c) bf[c][h] = 0u;
      }
    }

    // NS column sub-tiles share the LHS fragments of the step
#pragma unroll
    for (int st = 0; st < NS; ++st) {
    // ---- MMA A operand: gathered rows, transposed to k-major words per column ----
    uint32_t T[C::RC][2][8];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t raw[4][RB / 4 > 0 ? RB / 4 : 1];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int slot = 16 * h + 4 * i + t;
        const uint8_t* rp = sb + slot * C::RBYTES + ((st * C::SUB + g * RB) ^ swz<C::RBYTES>(t));
        if constexpr (RB == 8) {
          const uint2 w = *reinterpret_cast<const uint2*>(rp);
          raw[i][0] = w.x;
          raw[i][1] = w.y;
        } else if constexpr (RB == 16) {
          const uint4 w = *reinterpret_cast<const uint4*>(rp);
          raw[i][0] = w.x;
          raw[i][1] = w.y;
          raw[i][2] = w.z;
          raw[i][3] = w.w;
        } else {
          raw[i][0] = *reinterpret_cast<const uint32_t*>(rp);
        }
      }
      if constexpr (RB == 8) {
        transpose4x4(raw[0][0], raw[1][0], raw[2][0], raw[3][0], T[0][h][0], T[0][h][1], T[0][h][2], T[0][h][3]);
        transpose4x4(raw[0][1], raw[1][1], raw[2][1], raw[3][1], T[0][h][4], T[0][h][5], T[0][h][6], T[0][h][7]);
      } else if constexpr (RB == 16) {
        uint32_t lo0[4], lo1[4], hi0[4], hi1[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          split16(raw[i][0], raw[i][1], lo0[i], hi0[i]);
          split16(raw[i][2], raw[i][3], lo1[i], hi1[i]);
        }
        transpose4x4(lo0[0], lo0[1], lo0[2], lo0[3], T[0][h][0], T[0][h][1], T[0][h][2], T[0][h][3]);
        transpose4x4(lo1[0], lo1[1], lo1[2], lo1[3], T[0][h][4], T[0][h][5], T[0][h][6], T[0][h][7]);
        transpose4x4(hi0[0], hi0[1], hi0[2], hi0[3], T[1][h][0], T[1][h][1], T[1][h][2], T[1][h][3]);
        transpose4x4(hi1[0], hi1[1], hi1[2], hi1[3], T[1][h][4], T[1][h][5], T[1][h][6], T[1][h][7]);
      } else {
        uint32_t ev[4], od[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if constexpr (X16) {
            ev[i] = (raw[i][0] << 4) & 0xF0F0F0F0u;  // 16 x of columns 0, 2, 4, 6
            od[i] = raw[i][0] & 0xF0F0F0F0u;         // 16 x of columns 1, 3, 5, 7
          } else {
            unpack_s4x8(raw[i][0], ev[i], od[i]);
          }
        }
        // even columns 0,2,4,6 -> T[0..3]; odd columns 1,3,5,7 -> T[4..7]
        transpose4x4(ev[0], ev[1], ev[2], ev[3], T[0][h][0], T[0][h][1], T[0][h][2], T[0][h][3]);
        transpose4x4(od[0], od[1], od[2], od[3], T[0][h][4], T[0][h][5], T[0][h][6], T[0][h][7]);
      }
    }

#pragma unroll
    for (int j = 0; j < C::RC; ++j) {
      constexpr bool kDummy = false;
      (void)kDummy;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        // m = g <-> column 8g + 2q, m = g + 8 <-> column 8g + 2q + 1
        const int x0 = (RB == 4) ? q : 2 * q;
        const int x1 = (RB == 4) ? 4 + q : 2 * q + 1;
        const uint32_t a0 = T[j][0][x0], a1 = T[j][0][x1];
        const uint32_t a2 = T[j][1][x0], a3 = T[j][1][x1];
#pragma unroll
        for (int c = 0; c < C::LC; ++c) {
          const bool au = (RB == 16) && (j == 0);
          const bool bu = NIB ? (c < C::LC - 1) : ((LB >= 12) && (c == 0));
          if (au && bu) mma16832<true, true>(acc[st][c][j][q], a0, a1, a2, a3, bf[c][0], bf[c][1]);
          else if (au) mma16832<true, false>(acc[st][c][j][q], a0, a1, a2, a3, bf[c][0], bf[c][1]);
          else if (bu) mma16832<false, true>(acc[st][c][j][q], a0, a1, a2, a3, bf[c][0], bf[c][1]);
          else mma16832<false, false>(acc[st][c][j][q], a0, a1, a2, a3, bf[c][0], bf[c][1]);
        }
      }
    }
    }
    __syncwarp();
  }
  cp_async_wait<0>();

  // ---- epilogue: exact shift-add recombination + the reference's int32 checks ----
  if constexpr (X16) {
#pragma unroll
    for (int st = 0; st < NS; ++st)
#pragma unroll
      for (int c = 0; c < C::LC; ++c)
#pragma unroll
        for (int j = 0; j < C::RC; ++j)
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[st][c][j][q][e] >>= 4;  // exact: every term is a multiple of 16
  }
  bool overflow = false;
  double alpha = 0.0;
  if (p.out_f16) alpha = p.alpha ? p.alpha[b] : p.alpha_host;
  const float alpha_f = static_cast<float>(alpha);
  const int64_t row0 = r * V;
#pragma unroll
  for (int st = 0; st < NS; ++st) {
  int32_t vals[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      long long total = 0;
#pragma unroll
      for (int j = 0; j < C::RC; ++j) {
        long long tj;
        if constexpr (NIB) {
          // the reference's stacking groups at w = 4 (kernels.py:121-128): V = 8 one chunk per
          // group, V = 4 pairs, V = 2 quads; each weighted group sum must fit int32
          // (tile_engine.py:246-247)
          constexpr int per = V < 8 ? 8 / V : 1;
          tj = 0;
#pragma unroll
          for (int g0 = 0; g0 < C::LC; g0 += per) {
            long long comb = 0;
#pragma unroll
            for (int c = g0; c < g0 + per && c < C::LC; ++c)
              comb += static_cast<long long>(acc[st][c][j][q][e]) << (4 * c);
            overflow |= !fits_i32(comb);
            tj += comb;
          }
        } else if constexpr (C::LC == 2) {
          const long long lo = acc[st][0][j][q][e];
          const long long hi = 256LL * acc[st][1][j][q][e];
          constexpr bool w8 = (RB != 4);
          if constexpr (w8) {
            if constexpr (V == 8) overflow |= !fits_i32(hi);
            else overflow |= !fits_i32(lo + hi);
          } else {
            if constexpr (V == 4) overflow |= !fits_i32(hi);
          }
          tj = lo + hi;
        } else {
          tj = acc[st][0][j][q][e];
        }
        total += tj << (8 * j);
      }
      overflow |= !fits_i32(total);
      vals[q][e] = static_cast<int32_t>(total);
    }
  }
#pragma unroll
  for (int vv = 0; vv < 2; ++vv) {
    const int v = 2 * t + vv;
    if (v >= V) continue;
    int32_t rowv[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      rowv[2 * q] = vals[q][vv];
      rowv[2 * q + 1] = vals[q][2 + vv];
    }
    const int64_t n0 = c0 + st * kSubN + 8 * g;
    const int64_t base = (row0 + v) * p.N + n0;
    if (p.out) {
      int32_t* o = p.out + b * p.out_stride + base;
      if (n0 + 8 <= p.N && (p.N & 3) == 0) {
        reinterpret_cast<int4*>(o)[0] = make_int4(rowv[0], rowv[1], rowv[2], rowv[3]);
        reinterpret_cast<int4*>(o)[1] = make_int4(rowv[4], rowv[5], rowv[6], rowv[7]);
      } else {
#pragma unroll
        for (int x = 0; x < 8; ++x)
          if (n0 + x < p.N) o[x] = rowv[x];
      }
    }
    if (p.out_f16) {
      uint16_t* o = p.out_f16 + b * p.f16_stride + base;
#pragma unroll
      for (int x = 0; x < 8; ++x)
        if (n0 + x < p.N) o[x] = f16_dequant(rowv[x], alpha, alpha_f);
    }
  }
  }  // st
  if (overflow) flag_status(p.status, MC_STATUS_OVERFLOW);
  if (bad_idx) flag_status(p.status, MC_STATUS_BAD_INDEX);
}

// |16 * sum| < 2^31 for every byte-chunk accumulator: K (>= every row's true vectors),
// rounded up to the stride, times the largest 16 * |chunk x nibble| term.
bool spmm_x16_ok(const SpmmParams& p) {
  const long double sb = static_cast<long double>(((p.K + p.S - 1) / p.S) * p.S);
  const long double term = p.LB >= 12 ? 255.0L * 8.0L : (p.LB == 4 ? 64.0L : 1024.0L);
  return sb * term * 16.0L <= 2147483647.0L;
}

template <int LB, int RB, int V, int NS, bool NIB = false>
cudaError_t launch_spmm_v(SpmmParams p, cudaStream_t stream) {
  constexpr bool kX16 = RB == 4 && !NIB;
  using C = SpmmCfg<LB, RB, V, NS, NIB>;
  p.ntiles = (p.N + C::TN - 1) / C::TN;
  p.tasks = static_cast<int64_t>(p.batch) * p.vrows * p.ntiles;
  const int smem = kWarps * kStages * C::STAGE + kWarps * 2048;  // + per-warp index ring
  const bool aligned = ((p.N * RB) % 128 == 0) && ((reinterpret_cast<uintptr_t>(p.rhs_words) & 15) == 0) &&
                       ((p.rhs_stride * 4) % 16 == 0);
  const unsigned grid = static_cast<unsigned>((p.tasks + kWarps - 1) / kWarps);
  if (grid == 0) return cudaSuccess;
  if (aligned && kX16 && spmm_x16_ok(p)) {
    auto k = spmm_kernel<LB, RB, V, NS, true, NIB, kX16>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (const cudaError_t e = launch_pdl(k, dim3(grid), dim3(kWarps * 32), smem, stream, p)) return e;
  } else if (aligned) {
    auto k = spmm_kernel<LB, RB, V, NS, true, NIB>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (const cudaError_t e = launch_pdl(k, dim3(grid), dim3(kWarps * 32), smem, stream, p)) return e;
  } else {
    auto k = spmm_kernel<LB, RB, V, NS, false, NIB>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (const cudaError_t e = launch_pdl(k, dim3(grid), dim3(kWarps * 32), smem, stream, p)) return e;
  }
  count_launch();
  return cudaGetLastError();
}

// Task width: 128-byte row segments (NS = 4 for R4, 2 for R8) when the problem still has
// enough warp tasks to fill the GPU (C5-sized), else 64 columns (C3-sized, more tasks).
template <int LB, int RB, int V>
cudaError_t launch_spmm_ns(const SpmmParams& p, cudaStream_t stream) {
  constexpr int kWide = RB == 4 ? (LB >= 12 ? 2 : 4) : (RB == 8 ? 2 : 1);  // two LHS chunks: register budget
  const char* e = getenv("MCUBE_SPMM_NS");
  const int64_t wide_tasks = static_cast<int64_t>(p.batch) * p.vrows * ((p.N + kSubN * kWide - 1) / (kSubN * kWide));
  bool wide = kWide > 1 && p.N >= kSubN * kWide && wide_tasks >= 148LL * 48;
  if (e) wide = atoi(e) > 1;
  if constexpr (kWide > 1 && V == 8) {
    if (wide) return launch_spmm_v<LB, RB, V, kWide>(p, stream);
  }
  return launch_spmm_v<LB, RB, V, 1>(p, stream);
}

template <int LB, int RB>
cudaError_t launch_spmm_lr(const SpmmParams& p, cudaStream_t stream) {
  if constexpr (RB == 4 && LB >= 8) {
    if (spmm_needs_nibble_chunks(p)) {
      switch (p.V) {
        case 2: return launch_spmm_v<LB, RB, 2, 1, true>(p, stream);
        case 4: return launch_spmm_v<LB, RB, 4, 1, true>(p, stream);
        default: return launch_spmm_v<LB, RB, 8, 1, true>(p, stream);
      }
    }
  }
  switch (p.V) {
    case 2: return launch_spmm_ns<LB, RB, 2>(p, stream);
    case 4: return launch_spmm_ns<LB, RB, 4>(p, stream);
    default: return launch_spmm_ns<LB, RB, 8>(p, stream);
  }
}

}  // namespace

// 4-bit-width plans with an 8/12/16-bit LHS (emulation.py:80-83) run as int8 byte-chunk
// products unless K (which bounds every row's stored vectors, rounded up to the stride) is
// large enough that (a) a byte-chunk int32 accumulator could wrap, or (b) at V = 8 one of
// the reference's per-nibble group checks |2^(4c) * sum_k chunk_c(a) * b| <= INT32_MAX
// (tile_engine.py:246-247) could fail while the final result still fits. Then the kernel
// keeps one accumulator per nibble chunk, as the reference does, and evaluates every check.
bool spmm_needs_nibble_chunks(const SpmmParams& p) {
  if (p.RB != 4 || p.LB < 8) return false;
  const long double sb = static_cast<long double>(((p.K + p.S - 1) / p.S) * p.S);
  const long double lim = 2147483647.0L;
  // byte chunks x s4: s8 * s4 <= 128 * 8; u8 * s4 <= 255 * 8
  const long double byte_term = p.LB == 8 ? 1024.0L : 2040.0L;
  if (sb * byte_term > lim) return true;
  if (p.V != 8) return false;  // V = 4 / 2 group sums are byte-chunk (or final) sums: exact
  const int nch = p.LB / 4;
  for (int c = 1; c < nch; ++c) {  // chunk 0: |sum| <= K * 120, bounded by the K check
    const long double term = (c == nch - 1 ? 64.0L : 120.0L) * static_cast<long double>(1LL << (4 * c));
    if (sb * term > lim) return true;
  }
  return false;
}

cudaError_t launch_spmm(SpmmParams p, cudaStream_t stream) {
  if (spmm_tc_supported(p)) return launch_spmm_tc(p, stream);
  if (!spmm_needs_nibble_chunks(p) && spmm_seg_supported(p)) return launch_spmm_seg(p, stream);
  const int key = p.LB * 100 + p.RB;
  switch (key) {
    case 1616: return launch_spmm_lr<16, 16>(p, stream);
    case 1608: return launch_spmm_lr<16, 8>(p, stream);
    case 1604: return launch_spmm_lr<16, 4>(p, stream);
    case 1204: return launch_spmm_lr<12, 4>(p, stream);
    case 804: return launch_spmm_lr<8, 4>(p, stream);
    case 808: return launch_spmm_lr<8, 8>(p, stream);
    case 404: return launch_spmm_lr<4, 4>(p, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mcube
