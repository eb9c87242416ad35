// spmm_seg.cu -- SR-BCRS x dense SpMM for the large gather-bound problems (sm_100a).
//
// Same product and formulation as spmm.cu (kernels.spmm, kernels.py:293-340; transposed:
// D^T[n, v] = sum_k B[idx_k, n] * A_r[v, k], mma.sync m16n8k32 with the dense columns as
// MMA M, the V rows as MMA N and 32 gathered indices as MMA K), specialised for C5 (L8-R4,
// 32768^2 x 2048) and other problems with enough row segments to fill the GPU, where the
// instructions spent per gathered byte set the speed (ncu: ALU pipe bound):
//
// * a warp task is one vector row x one 128-byte segment of the dense rows (256 columns at
//   4 bits, 128 at 8 bits);
// * column indices are turned into row numbers (-1 for sentinel / padding / out-of-range,
//   sparse_format.py:25) once per 8 k-steps by all lanes, already in copy order and with
//   the shuffle permutation (SHUFFLE_PERMUTATION, tile_engine.py:35) undone, so a k-step's
//   producer is 2 LDS.128 + 8 x (IMAD.WIDE, SEL, cp.async) per lane;
// * the gathered row of MMA k = 16h + 4t + i sits in slot 16h + 8(i >> 1) + 2t + (i & 1),
//   its 16-byte chunk c at c ^ (slot & 7): every consumer LDS.128 is bank-conflict free, and
//   one LDS.128 holds a lane's bytes for all NS 64-column sub-tiles of the k-step;
// * 4-bit rows are byte-transposed (8 PRMT per 4 x 4 bytes) and then split into the two
//   nibble columns of each byte as 16 x the value -- lo = y & 0x0F0F0F0F, 16 lo and y - lo
//   on the FMA pipe -- so the MMA sees exact 16x products (shifted back in the epilogue;
//   exact while |16 sum| < 2^31, spmm_seg_supported);
// * LHS values: strides 16 / 32 (the plans' tile k) make a k-step's values one contiguous
//   run of whole stride blocks (sparse_format.py:131-139), one 8-byte cp.async per lane.
//
// Dense column mapping: lane group g of sub-tile s owns the 8 columns 8 (NS g + s) + 0..7
// (its own 16-byte chunk of the segment), so a lane's NS sub-tiles are contiguous columns
// and the epilogue writes NS * 8 contiguous int32 per output row.
#include <cuda.h>
#include <cuda_fp16.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace mcube {
namespace {

constexpr int kW = 4;         // warps (independent tasks) per CTA
constexpr int kSeg = 128;     // bytes of a gathered row segment (one TMA box row, SW128)
constexpr int kBStage = 32 * kSeg;

template <int LB, int RB, int V, int STAGES>
struct SegCfg {
  static constexpr int LC = (LB >= 12) ? 2 : 1;
  static constexpr int TN = kSeg * 8 / RB;     // dense columns per task
  static constexpr int NS = TN / 64;           // 64-column MMA sub-tiles per task
  static constexpr int ABYTES = 2 * LB;        // bytes of 16 LHS values
  static constexpr int A_STAGE = 2 * V * ABYTES;
  static constexpr int OFF_A = STAGES * kBStage;
  static constexpr int OFF_IDX = OFF_A + STAGES * A_STAGE;
  // + 1 KB raw indices + 2 x 2 KB row addresses; 128-byte aligned (the consumer XORs chunk
  // offsets into its row address)
  static constexpr int WARP_BYTES = (OFF_IDX + 5120 + 127) / 128 * 128;
  static constexpr int SMEM = kW * WARP_BYTES + 1024;  // + alignment slack
};

// 128 zero bytes: the source of gathered rows for sentinel / padding / out-of-range slots
__device__ __align__(128) uint8_t g_seg_zero[128] = {};

// 16-byte cp.async; `zero` ignores the source and fills zeros (PTX ignore-src operand)
__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void* src, bool zero) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
      "cp.async.cg.shared.global [%0], [%1], 16, p;\n}" ::"r"(dst),
      "l"(src), "r"(static_cast<int>(zero)));
}

// smem slot of MMA k = 16h + 4t + i: the k itself for the ldmatrix consumer (lane k of an
// LDSM.x2 points at row k; rows 8j..8j+7 of a phase sit in 8 distinct 16-byte bank groups by
// the c ^ (slot & 7) chunk swizzle); the PRMT consumer (MCUBE_SEG_PRMT) interleaves the rows
// so that its per-lane LDS.128 are conflict-free
#ifdef MCUBE_SEG_PRMT
__device__ __forceinline__ constexpr int seg_slot(int h, int i, int t) { return 16 * h + 8 * (i >> 1) + 2 * t + (i & 1); }
#else
__device__ __forceinline__ constexpr int seg_slot(int h, int i, int t) { return 16 * h + 4 * t + i; }
#endif

// ldmatrix.m16n16.x2.trans.b8 (LDSM.8.MT1616.2): lanes 0-15 give the 16-byte rows k = 0..15
// of matrix 0, lanes 16-31 rows k = 16..31 of matrix 1; lane (g, t) receives bytes (row k,
// column g) / (k, g + 8) for k = 4t..4t+3 of matrix 0 in r0 / r1 and of matrix 1 in r2 / r3:
// exactly the m16n8k32 A fragment of the 16 x 32 transpose (tools/micro/ldsm_probe.cu)
__device__ __forceinline__ void ldsm_t16x2(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m16n16.x2.trans.shared.b8 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

template <int LB, int RB, int V, int STAGES>
__global__ void __launch_bounds__(kW * 32)
spmm_seg_kernel(const SpmmParams p) {
  using C = SegCfg<LB, RB, V, STAGES>;
  constexpr int NS = C::NS;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  uint8_t* wbuf = smem + warp * C::WARP_BYTES;
  const uint32_t wbuf_s = smem_u32(wbuf);
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();
  const int64_t task = static_cast<int64_t>(blockIdx.x) * kW + warp;
  if (task >= p.tasks) return;
  const int64_t per_batch = p.vrows * p.ntiles;
  const int64_t b = task / per_batch;
  const int64_t rem = task - b * per_batch;
  const int64_t r = rem / p.ntiles;
  const int64_t c0 = (rem - r * p.ntiles) * C::TN;

  const uint32_t* __restrict__ lhs = p.lhs_words + b * p.lhs_stride;
  const int64_t p_begin = p.row_begin[r];
  const int64_t n_true = p.row_end[r] - p_begin;
  const int64_t stored = ((n_true + p.S - 1) / p.S) * p.S;
  const int64_t p_end = p_begin + stored;
  const int nsteps = static_cast<int>((stored + 31) >> 5);
  const bool shuffled = p.shuffled != 0;
  const uint32_t kdim = static_cast<uint32_t>(p.K);
  const int64_t brow0 = p.rhs_stride ? b * p.K : 0;  // batch item's first RHS row
  const int col_byte = static_cast<int>(c0 * RB / 8);
  const int S = p.S;  // 16 or 32 (spmm_seg_supported)
  const uint64_t row_bytes = static_cast<uint64_t>(p.N) * RB / 8;
  // this lane copies 16-byte chunk (lane & 7) of its rows; a chunk past the row end (last
  // column segment) is zero-filled (cp.async ignore-src)
  const uint64_t chunk_off = 16 * (lane & 7);
  const bool seg_out = static_cast<uint64_t>(col_byte) + chunk_off >= row_bytes;

  // ---- column indices -> gather rows. The raw indices of 256 stored positions (8 k-steps,
  // "chunk") are staged by cp.async one chunk ahead; halfway through a chunk every lane turns
  // 8 of the next chunk's indices into TMA row coordinates (row -1 for sentinel / padding /
  // out-of-range: zero fill) and stores them in gather order -- slot seg_slot(k) of MMA k,
  // k = P(position) when the indices are shuffled (SHUFFLE_PERMUTATION, tile_engine.py:35;
  // sparse_format.py:222-230) -- into a 2 x 256 ring; per k-step lanes 0-7 then read the 4
  // row coordinates of their gather4 with one LDS.128.
  uint32_t* sraw = reinterpret_cast<uint32_t*>(wbuf + C::OFF_IDX);
  uint64_t* srow = reinterpret_cast<uint64_t*>(wbuf + C::OFF_IDX + 1024);
  const uint32_t sraw_s = smem_u32(sraw);
  auto fetch_raw = [&](int c) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int ch = lane + 32 * u;
      const int64_t e0 = p_begin + 256LL * c + 4 * ch;
      const int64_t avail = p_end - e0;
      const uint32_t bytes = avail >= 4 ? 16u : (avail > 0 ? static_cast<uint32_t>(avail) * 4u : 0u);
      cp_async16(sraw_s + 16 * ch, p.col_indices + (bytes ? e0 : 0), bytes);
    }
  };
  bool bad_idx = false;
  const uint64_t seg_base = reinterpret_cast<uint64_t>(p.rhs_words) + static_cast<uint64_t>(brow0) * row_bytes +
                            static_cast<uint64_t>(col_byte);
  const uint64_t zero_row = reinterpret_cast<uint64_t>(g_seg_zero);
  // raw chunk c -> rows ring half c & 1; `newer` = cp.async groups committed after the
  // chunk's fetch (they may stay in flight)
  auto convert = [&](int c, auto newer) {
    cp_async_wait<decltype(newer)::value>();
    __syncwarp();
    const uint4 w0 = *reinterpret_cast<const uint4*>(sraw + 8 * lane);
    const uint4 w1 = *reinterpret_cast<const uint4*>(sraw + 8 * lane + 4);
    const uint32_t cw[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    uint64_t* dst = srow + (c & 1) * 256 + 32 * (lane >> 2);  // k-step (lane >> 2) of the chunk
    const int64_t pos0 = 256LL * c + 8 * lane;            // stored position of cw[0] in the row
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int pp = 8 * (lane & 3) + e;                   // position within the k-step
      const int kk = shuffled ? ((pp & ~7) | ((e & 3) << 1) | (e >> 2)) : pp;  // P: 0,2,4,6,1,3,5,7
      const uint32_t col = pos0 + e < stored ? cw[e] : kSentinel;
      const bool ok = col < kdim;
      bad_idx |= !ok && col != kSentinel;
      const int h = kk >> 4, t4 = (kk >> 2) & 3, i = kk & 3;
      const int sl = seg_slot(h, i, t4);
      // the row segment's global address; invalid slots read a zero row instead
      dst[(sl & 3) * 8 + (sl >> 2)] = ok ? seg_base + static_cast<uint64_t>(col) * row_bytes : zero_row;
    }
  };

  // LHS values: strides of 16 or 32 (the tile k of every plan, bench.py:103) make a k-step's
  // 32 positions one contiguous run of whole stride blocks -- [2 blocks][V][16] (S = 16) or
  // [V][32] (S = 32) -- fetched by one bulk copy on the stage barrier
  const uint8_t* lhs_run = reinterpret_cast<const uint8_t*>(lhs) + (p_begin * V * LB) / 8;

  // cp.async producer: lane (j, c) = (lane / 8, lane % 8) copies 16-byte chunk c of slots
  // j + 4u (u = 0..7) -- the 8 gather rows of a lane are one 32-byte run of the rows ring --
  // into the slot's 128-byte row at chunk c ^ (slot & 7) (the consumer's conflict-free
  // swizzle); row -1 (sentinel / padding / out of range) is a 0-byte copy (zero fill).

  auto issue = [&](int step) {
    if ((step & 7) == 0 && 256LL * ((step >> 3) + 1) < stored) {
      __syncwarp();  // the staging buffer's previous chunk was converted 4 steps ago
      fetch_raw((step >> 3) + 1);
    }
    if ((step & 7) == 4 && 256LL * ((step >> 3) + 1) < stored)
      convert((step >> 3) + 1, std::integral_constant<int, 3>());  // fetched by issue(step - 4)
    const int st = step % STAGES;
    const uint64_t* rr = srow + ((step >> 3) & 1) * 256 + 32 * (step & 7) + 8 * (lane >> 3);
    const uint32_t bst = wbuf_s + st * kBStage;
#pragma unroll
    for (int u2 = 0; u2 < 4; ++u2) {
      const ulonglong2 a2 = *reinterpret_cast<const ulonglong2*>(rr + 2 * u2);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int u = 2 * u2 + e;
        const int sl = (lane >> 3) + 4 * u;
        const uint64_t a = (e ? a2.y : a2.x) + chunk_off;
        cp_async16_zfill(bst + sl * kSeg + (((lane & 7) ^ (sl & 7)) << 4), reinterpret_cast<const void*>(a), seg_out);
      }
    }
    // LHS values of the step: A_STAGE contiguous bytes (whole stride blocks), 8 per lane
    {
      const int64_t left = (stored - 32LL * step) * V * LB / 8;  // bytes of this row left
#pragma unroll
      for (int q = lane; q < C::A_STAGE / 8; q += 32) {
        const bool ok = 8 * q < left;
        cp_async8(wbuf_s + C::OFF_A + st * C::A_STAGE + 8 * q,
                  ok ? lhs_run + static_cast<int64_t>(step) * C::A_STAGE + 8 * q : lhs_run, ok ? 8u : 0u);
      }
    }
    cp_async_commit();
  };

#ifndef MCUBE_SEG_PRMT
  // ---- ldmatrix consumer. Chunk j (16 bytes) of the segment holds 16 byte-columns: 16 dense
  // columns at 8 bits, 32 at 4 bits. One LDSM.x2 over the 32 gathered rows gives the A
  // fragment of its 16 byte-columns x 32 k. 4-bit rows: a byte y = 16 hi + lo_u (hi signed, lo
  // unsigned) enters two MMAs, y' = y ^ 0x08 per byte (= 16 hi + lo + 8 with lo the signed low
  // nibble) and h = y & 0xF0 (= 16 hi):  odd column = acc(h) / 16 and even column =
  // acc(y') - acc(h) - 8 sum_k a_k (the LHS sums: one DP4A per fragment word), all exact in
  // int32 under spmm_seg_supported's |16 sum| bound -- 2 LOP per word, no transposes.
  constexpr int NCH = kSeg / 16;            // 16-byte chunks per segment
  constexpr int MM = RB == 4 ? 2 : 1;       // MMAs per chunk and LHS chunk
  int acc[NCH][C::LC][MM][4];
#pragma unroll
  for (int j = 0; j < NCH; ++j)
#pragma unroll
    for (int c = 0; c < C::LC; ++c)
#pragma unroll
      for (int m = 0; m < MM; ++m)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[j][c][m][e] = 0;
  int asum = 0;  // 4-bit RHS: this lane's share of sum_k a[v = g][k]
  // lane's LDSM row: slot `lane`, chunk j at j ^ (lane & 7)
  const uint32_t ldsm_off = static_cast<uint32_t>(lane * kSeg + ((lane & 7) << 4));

  if (nsteps > 0) {
    fetch_raw(0);
    cp_async_commit();
    convert(0, std::integral_constant<int, 0>());
    __syncwarp();
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < nsteps) issue(s);
      else cp_async_commit();
    }
  }
  for (int s = 0; s < nsteps; ++s) {
    const int nxt = s + STAGES - 1;
    if (nxt < nsteps) issue(nxt);
    else cp_async_commit();
    cp_async_wait<STAGES - 1>();
    const int st = s % STAGES;
    __syncwarp();

    const uint8_t* sa = wbuf + C::OFF_A + st * C::A_STAGE;
    // ---- MMA B operand: LHS chunk words for k = 16h + 4t .. +3 of row v = g ----
    uint32_t bf[C::LC][2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gv = g < V ? g : 0;
      const uint8_t* ar = sa + (S == 32 ? 2 * gv + h : h * V + gv) * C::ABYTES;
      if constexpr (LB == 8) {
        bf[0][h] = *reinterpret_cast<const uint32_t*>(ar + 4 * t);
      } else if constexpr (LB == 4) {
        bf[0][h] = unpack_s4x4_ordered(*reinterpret_cast<const uint16_t*>(ar + 2 * t));
      } else {  // LB == 16
        const uint2 w = *reinterpret_cast<const uint2*>(ar + 8 * t);
        split16(w.x, w.y, bf[0][h], bf[1][h]);
      }
      if (g >= V) {
#pragma unroll
        for (int c = 0; c < C::LC; ++c) bf[c][h] = 0u;
      }
    }
    if constexpr (RB == 4) {
      asum = __dp4a(static_cast<int>(bf[0][0]), 0x01010101, asum);
      asum = __dp4a(static_cast<int>(bf[0][1]), 0x01010101, asum);
    }
    const uint32_t row_addr = wbuf_s + st * kBStage + ldsm_off;
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      uint32_t a[4];
      ldsm_t16x2(row_addr ^ (j << 4), a[0], a[1], a[2], a[3]);
      if constexpr (RB == 4) {
        uint32_t y[4], hh[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          y[e] = a[e] ^ 0x08080808u;
          hh[e] = a[e] & 0xF0F0F0F0u;
        }
        mma16832<false, false>(acc[j][0][0], y[0], y[1], y[2], y[3], bf[0][0], bf[0][1]);
        mma16832<false, false>(acc[j][0][1], hh[0], hh[1], hh[2], hh[3], bf[0][0], bf[0][1]);
      } else {
#pragma unroll
        for (int c = 0; c < C::LC; ++c) {
          if (LB == 16 && c == 0)
            mma16832<false, true>(acc[j][c][0], a[0], a[1], a[2], a[3], bf[c][0], bf[c][1]);
          else
            mma16832<false, false>(acc[j][c][0], a[0], a[1], a[2], a[3], bf[c][0], bf[c][1]);
        }
      }
    }
    __syncwarp();
  }
  cp_async_wait<0>();  // a raw index chunk past the last step may still be in flight

  // ---- epilogue: exact recombination + the reference's int32 checks. Lane (g, t) holds
  // byte-columns g and g + 8 of every chunk for rows v = 2t, 2t + 1 ----
  bool overflow = false;
  const int64_t row0 = r * V;
  int32_t* outb = p.out + b * p.out_stride;
  long long vsum[2] = {0, 0};
  if constexpr (RB == 4) {
    asum += __shfl_xor_sync(0xffffffffu, asum, 1);
    asum += __shfl_xor_sync(0xffffffffu, asum, 2);  // sum_k a[g][k] in every lane of group g
    vsum[0] = __shfl_sync(0xffffffffu, asum, 8 * t);      // v = 2t
    vsum[1] = __shfl_sync(0xffffffffu, asum, 8 * t + 4);  // v = 2t + 1
  }
#pragma unroll
  for (int vv = 0; vv < 2; ++vv) {
    const int v = 2 * t + vv;
    if (v >= V) continue;
    int32_t* o = outb + (row0 + v) * p.N;
#pragma unroll
    for (int j = 0; j < NCH; ++j)
#pragma unroll
      for (int hi = 0; hi < 2; ++hi) {
        const int e = 2 * hi + vv;
        if constexpr (RB == 4) {
          const long long hsum = acc[j][0][1][e];
          const long long odd = hsum >> 4;
          const long long even = static_cast<long long>(acc[j][0][0][e]) - hsum - 8 * vsum[vv];
          overflow |= !fits_i32(even) || !fits_i32(odd);
          const int64_t n = c0 + 32 * j + 16 * hi + 2 * g;
          if (n < p.N) *reinterpret_cast<int2*>(o + n) = make_int2(static_cast<int32_t>(even), static_cast<int32_t>(odd));
        } else {
          long long total;
          if constexpr (C::LC == 2) {
            const long long lo = acc[j][0][0][e];
            const long long hh = 256LL * acc[j][1][0][e];
            if constexpr (V == 8) overflow |= !fits_i32(hh);
            else overflow |= !fits_i32(lo + hh);
            total = lo + hh;
          } else {
            total = acc[j][0][0][e];
          }
          overflow |= !fits_i32(total);
          const int64_t n = c0 + 16 * j + 8 * hi + g;
          if (n < p.N) o[n] = static_cast<int32_t>(total);
        }
      }
  }
#else
  int acc[NS][C::LC][4][4];
#pragma unroll
  for (int s = 0; s < NS; ++s)
#pragma unroll
    for (int c = 0; c < C::LC; ++c)
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[s][c][q][e] = 0;

  if (nsteps > 0) {
    fetch_raw(0);
    cp_async_commit();
    convert(0, std::integral_constant<int, 0>());
    __syncwarp();
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < nsteps) issue(s);
      else cp_async_commit();
    }
  }
  for (int s = 0; s < nsteps; ++s) {
    const int nxt = s + STAGES - 1;
    if (nxt < nsteps) issue(nxt);
    else cp_async_commit();
    cp_async_wait<STAGES - 1>();
    const int st = s % STAGES;
    __syncwarp();

    const uint8_t* sb = wbuf + st * kBStage;
    const uint8_t* sa = wbuf + C::OFF_A + st * C::A_STAGE;
    // ---- MMA B operand: LHS chunk words for k = 16h + 4t .. +3 of row v = g ----
    uint32_t bf[C::LC][2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gv = g < V ? g : 0;
      const uint8_t* ar = sa + (S == 32 ? 2 * gv + h : h * V + gv) * C::ABYTES;
      if constexpr (LB == 8) {
        bf[0][h] = *reinterpret_cast<const uint32_t*>(ar + 4 * t);
      } else if constexpr (LB == 4) {
        bf[0][h] = unpack_s4x4_ordered(*reinterpret_cast<const uint16_t*>(ar + 2 * t));
      } else {  // LB == 16
        const uint2 w = *reinterpret_cast<const uint2*>(ar + 8 * t);
        split16(w.x, w.y, bf[0][h], bf[1][h]);
      }
      if (g >= V) {
#pragma unroll
        for (int c = 0; c < C::LC; ++c) bf[c][h] = 0u;
      }
    }
    // ---- MMA A operand: one LDS.128 per (h, i) = the lane's chunk g of row k = 16h + 4t + i ----
    uint4 raw[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int sl = seg_slot(h, i, t);
        raw[h][i] = *reinterpret_cast<const uint4*>(sb + sl * kSeg + ((g ^ (sl & 7)) << 4));
      }
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      uint32_t T[2][8];  // per h: words for dense columns 0..7 of the lane's group (k 4t..4t+3)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        auto word = [&](int i, int w) -> uint32_t {
          const uint4 x = raw[h][i];
          return w == 0 ? x.x : (w == 1 ? x.y : (w == 2 ? x.z : x.w));
        };
        if constexpr (RB == 4) {
          // word s of the chunk = columns 8 s .. 8 s + 7 (2 per byte); byte-transpose the 4
          // rows, then split each byte's nibbles as 16 x value (even / odd column)
          uint32_t y[4];
          transpose4x4(word(0, s), word(1, s), word(2, s), word(3, s), y[0], y[1], y[2], y[3]);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            // lo = low nibbles (one LOP3); column 2j = 16 lo, column 2j + 1 = y - lo: both on
            // the FMA pipe (IMAD), leaving the ALU pipe to the PRMT transposes
            const uint32_t lo = y[j] & 0x0F0F0F0Fu;
            uint32_t ev, od;
            asm("mul.lo.u32 %0, %1, 16;" : "=r"(ev) : "r"(lo));
            asm("mad.lo.u32 %0, %1, 0xFFFFFFFF, %2;" : "=r"(od) : "r"(lo), "r"(y[j]));
            T[h][2 * j] = ev;      // column 2j
            T[h][2 * j + 1] = od;  // column 2j + 1
          }
        } else {  // RB == 8: words 2s, 2s + 1 = columns 8s .. 8s + 7
          transpose4x4(word(0, 2 * s), word(1, 2 * s), word(2, 2 * s), word(3, 2 * s), T[h][0], T[h][1], T[h][2],
                       T[h][3]);
          transpose4x4(word(0, 2 * s + 1), word(1, 2 * s + 1), word(2, 2 * s + 1), word(3, 2 * s + 1), T[h][4],
                       T[h][5], T[h][6], T[h][7]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // m = g <-> column 2q, m = g + 8 <-> column 2q + 1 (of the group)
#pragma unroll
        for (int c = 0; c < C::LC; ++c) {
          if (LB == 16 && c == 0)
            mma16832<false, true>(acc[s][c][q], T[0][2 * q], T[0][2 * q + 1], T[1][2 * q], T[1][2 * q + 1], bf[c][0],
                                  bf[c][1]);
          else
            mma16832<false, false>(acc[s][c][q], T[0][2 * q], T[0][2 * q + 1], T[1][2 * q], T[1][2 * q + 1], bf[c][0],
                                   bf[c][1]);
        }
      }
    }
    __syncwarp();
  }
  cp_async_wait<0>();  // a raw index chunk past the last step may still be in flight

  // ---- epilogue: (X16 shift,) exact shift-add recombination + the reference's int32 checks ----
  bool overflow = false;
  const int64_t row0 = r * V;
  int32_t* outb = p.out + b * p.out_stride;
#pragma unroll
  for (int vv = 0; vv < 2; ++vv) {
    const int v = 2 * t + vv;
    int32_t rowv[NS][8];
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int hi = 0; hi < 2; ++hi) {
          long long total;
          if constexpr (C::LC == 2) {
            const long long lo = acc[s][0][q][2 * hi + vv];
            const long long hh = 256LL * acc[s][1][q][2 * hi + vv];
            if constexpr (V == 8) overflow |= !fits_i32(hh);
            else overflow |= !fits_i32(lo + hh);
            total = lo + hh;
          } else {
            total = RB == 4 ? (acc[s][0][q][2 * hi + vv] >> 4) : acc[s][0][q][2 * hi + vv];
          }
          overflow |= !fits_i32(total);
          rowv[s][2 * q + hi] = static_cast<int32_t>(total);
        }
    if (v < V) {
      const int64_t n0 = c0 + 8 * NS * g;
      int32_t* o = outb + (row0 + v) * p.N + n0;
      if (n0 + 8 * NS <= p.N) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          reinterpret_cast<int4*>(o)[2 * s] = make_int4(rowv[s][0], rowv[s][1], rowv[s][2], rowv[s][3]);
          reinterpret_cast<int4*>(o)[2 * s + 1] = make_int4(rowv[s][4], rowv[s][5], rowv[s][6], rowv[s][7]);
        }
      } else {
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
          for (int x = 0; x < 8; ++x)
            if (n0 + 8 * s + x < p.N) o[8 * s + x] = rowv[s][x];
      }
    }
  }
#endif
  if (overflow) flag_status(p.status, MC_STATUS_OVERFLOW);
  if (bad_idx) flag_status(p.status, MC_STATUS_BAD_INDEX);
}

template <int LB, int RB, int V>
cudaError_t launch_seg_v(SpmmParams p, cudaStream_t stream) {
  constexpr int kStages = 3;
  using C = SegCfg<LB, RB, V, kStages>;
  p.ntiles = (p.N + C::TN - 1) / C::TN;
  p.tasks = static_cast<int64_t>(p.batch) * p.vrows * p.ntiles;
  const unsigned grid = static_cast<unsigned>((p.tasks + kW - 1) / kW);
  if (grid == 0) return cudaSuccess;
  auto k = spmm_seg_kernel<LB, RB, V, kStages>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  const cudaError_t e = launch_pdl(k, dim3(grid), dim3(kW * 32), C::SMEM, stream, p);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int LB, int RB>
cudaError_t launch_seg_lr(const SpmmParams& p, cudaStream_t stream) {
  switch (p.V) {
    case 2: return launch_seg_v<LB, RB, 2>(p, stream);
    case 4: return launch_seg_v<LB, RB, 4>(p, stream);
    default: return launch_seg_v<LB, RB, 8>(p, stream);
  }
}

}  // namespace

// The gather4 kernel takes the single-chunk-product int8 operand forms it was built for:
// L8-R4 / L4-R4 (4-bit RHS as 16 x nibble, exact while |16 sum| < 2^31), L8-R8 and L16-R8
// (two LHS byte chunks); row pitch a multiple of 16 bytes (tensor-map stride), enough
// tasks to fill the GPU, int32 output only. MCUBE_SPMM_PATH=mma forces spmm.cu.
bool spmm_seg_supported(const SpmmParams& p) {
  const int key = p.LB * 100 + p.RB;
  if (key != 804 && key != 404 && key != 808 && key != 1608) return false;
  const char* e = getenv("MCUBE_SPMM_PATH");
  if (e && e[0] != 's') return false;
  if (p.out == nullptr || p.out_f16 != nullptr || p.batch < 1) return false;
  if (p.S != 16 && p.S != 32) return false;  // k-step = whole stride blocks (one bulk copy)
  if (p.lhs_stride != 0 && (p.lhs_stride * 4) % 16 != 0) return false;
  if ((static_cast<int64_t>(p.N) * p.RB / 8) % 16 != 0 || (reinterpret_cast<uintptr_t>(p.rhs_words) & 15)) return false;
  if (p.rhs_stride != 0 && p.rhs_stride * 4 != p.K * p.N * p.RB / 8) return false;
  if (p.K >= (1ll << 31) - 1) return false;
  if (p.RB == 4) {  // X16 exactness: |16 * sum| < 2^31 with sum <= roundup(K, S) * max |a * b|
    const long double sb = static_cast<long double>(((p.K + p.S - 1) / p.S) * p.S);
    if (sb * (p.LB == 4 ? 64.0L : 1024.0L) * 16.0L > 2147483647.0L) return false;
  }
  if (e && e[0] == 's') return true;
  // Problems with enough 128-byte row segments to fill the GPU (C5), and the V = 8 cells
  // at ~90 % sparsity where, measured on C3 (tools/bench_spmm.py c3, forced paths), the
  // segment kernel beats both the dense-tile GEMM and the 64-column mma.sync tasks for a
  // 4-bit RHS or a 16-bit LHS (28.6 -> 20.4 us L8-R4 / L4-R4, 40.9 -> 28.6 us L16-R8);
  // smaller / sparser problems keep spmm.cu's 64-column tasks (more tasks per row).
  // V < 8: fewer uses per gathered byte than MMA N = 8 provides; the 64-column tasks and
  // the dense tile win there (C3 V = 2: 64 -> 168 us when forced)
  if (p.V != 8) return false;
  const int64_t tn = 128 * 8 / p.RB;
  const int64_t tasks = static_cast<int64_t>(p.batch) * p.vrows * ((p.N + tn - 1) / tn);
  if (tasks >= 148LL * 48) return true;
  const double density = p.stored > 0 ? static_cast<double>(p.stored) * p.V / (static_cast<double>(p.M) * p.K) : 1.0;
  return (p.RB == 4 || p.LB == 16) && density > 0.05 && density <= 0.11;
}

cudaError_t launch_spmm_seg(const SpmmParams& p, cudaStream_t stream) {
  switch (p.LB * 100 + p.RB) {
    case 804: return launch_seg_lr<8, 4>(p, stream);
    case 404: return launch_seg_lr<4, 4>(p, stream);
    case 808: return launch_seg_lr<8, 8>(p, stream);
    default: return launch_seg_lr<16, 8>(p, stream);
  }
}

}  // namespace mcube
