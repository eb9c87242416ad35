// spmm_seg.cu -- SR-BCRS x dense SpMM for the large gather-bound problems (sm_100a).
//
// Same product and formulation as spmm.cu (kernels.spmm, kernels.py:293-340; transposed:
// D^T[n, v] = sum_k B[idx_k, n] * A_r[v, k], mma.sync m16n8k32 with the dense columns as
// MMA M, the V rows as MMA N and 32 gathered indices as MMA K), specialised for C5 (L8-R4,
// 32768^2 x 2048) and other problems with enough row segments to fill the GPU, where the
// instructions spent per gathered byte set the speed:
//
// * a warp task is one vector row x one 128-byte segment of the dense rows (256 columns at
//   4 bits, 128 at 8 bits);
// * column indices are turned into 64-bit row-segment addresses (a zero row for sentinel /
//   padding / out-of-range, sparse_format.py:25) once per 8 k-steps by all lanes, with the
//   shuffle permutation (SHUFFLE_PERMUTATION, tile_engine.py:35) undone, so a k-step's
//   producer is 4 LDS.128 + 8 x (64-bit add, cp.async) per lane;
// * gathered row k sits in a 128-byte slot with 16-byte chunk c at c ^ (k & 7): the consumer's
//   8-row ldmatrix phases hit 8 distinct bank groups;
// * the consumer is ldmatrix.m16n16.x2.trans.b8 (LDSM.8.MT1616): one instruction turns 32
//   gathered rows x 16 bytes into the k-major MMA A fragment -- no register transposes;
// * 4-bit rows: byte y = 16 hi + lo_u (hi signed, lo unsigned) feeds two MMAs, y' = y ^ 0x08
//   per byte (= 16 hi + lo + 8, lo the signed low nibble) and h = y & 0xF0 (= 16 hi): odd
//   column = acc(h) / 16, even column = acc(y') - acc(h) - 8 sum_k a_k (DP4A over the LHS
//   fragment), exact in int32 under spmm_seg_supported's bound. With a workspace the XOR is
//   applied to B once per call (seg_prexor_kernel), leaving one LOP per fragment word;
// * LHS values: strides 16 / 32 (the plans' tile k) make a k-step's values one contiguous
//   run of whole stride blocks (sparse_format.py:131-139), one 8-byte cp.async per lane.
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace mcube {
namespace {

constexpr int kW = 4;          // warps (independent tasks) per CTA
constexpr int kSeg = 128;      // bytes of a gathered row segment
constexpr int kBStage = 32 * kSeg;
constexpr int kChunk = 8;      // k-steps per index-conversion chunk (256 stored positions)

template <int LB, int RB, int V, int STAGES>
struct SegCfg {
  static constexpr int LC = (LB >= 12) ? 2 : 1;
  static constexpr int TN = kSeg * 8 / RB;     // dense columns per task
  static constexpr int ABYTES = 2 * LB;        // bytes of 16 LHS values
  static constexpr int A_STAGE = 2 * V * ABYTES;
  static constexpr int OFF_A = STAGES * kBStage;
  static constexpr int OFF_RAW = OFF_A + STAGES * A_STAGE;       // 256 raw indices
  static constexpr int OFF_ROW = OFF_RAW + 4 * 32 * kChunk;      // 2 x 256 row addresses
  static constexpr int WARP_BYTES = (OFF_ROW + 2 * 8 * 32 * kChunk + 127) / 128 * 128;
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

// B ^ 0x08 in every byte (the low nibble's sign bit): 4-bit right-hand sides enter the
// segment kernel's y' MMA without a per-use XOR
__global__ void seg_prexor_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n16) {
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint4 w = src[i];
    w.x ^= 0x08080808u;
    w.y ^= 0x08080808u;
    w.z ^= 0x08080808u;
    w.w ^= 0x08080808u;
    dst[i] = w;
  }
}

template <int LB, int RB, int V, int STAGES, bool PREX>
__global__ void __launch_bounds__(kW * 32, 3)
spmm_seg_kernel(const SpmmParams p) {
  using C = SegCfg<LB, RB, V, STAGES>;
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

  // ---- producer lane map: lane (j, c) = (lane / 8, lane % 8) copies 16-byte chunk c of the
  // gathered rows j + 4u (u = 0..7): one cp.async instruction = 4 whole 128-byte rows (4 cache
  // lines; a 16-row instruction costs 4x the L1TEX tag lookups, measured 3.3x slower), into
  // the row's 128-byte slot at chunk c ^ (row & 7): the consumer's ldmatrix phases (8 rows,
  // one chunk) then hit 8 distinct bank groups. (A 144-byte pitch without the XOR moved 1.5x
  // the L2 -> SM bytes for the same copies and ran 1.6x slower.)
  const int pj = lane >> 3, pc = lane & 7;
  // a chunk past the row end (last column segment) is zero-filled
  const bool chunk_out = static_cast<uint64_t>(col_byte) + 16 * pc >= row_bytes;
  const bool full_seg = static_cast<uint64_t>(col_byte) + kSeg <= row_bytes;  // warp-uniform

  // ---- column indices -> row-segment addresses. The raw indices of 256 stored positions (8
  // k-steps, "chunk") are staged by cp.async one chunk ahead; halfway through a chunk every
  // lane turns 4 of the next chunk's indices into the global addresses of their row segments
  // (the zero row for sentinel / padding / out-of-range) and stores them at the slot of their
  // MMA k -- k = P(position) when the indices are shuffled (SHUFFLE_PERMUTATION,
  // tile_engine.py:35; sparse_format.py:222-230) -- in a 2 x 256 ring, slot k of a k-step at
  // entry 8 (k % 4) + k / 4 so that producer lane j reads its 8 rows with 4 LDS.128.
  const uint32_t sraw_s = wbuf_s + C::OFF_RAW;
  const uint32_t* sraw = reinterpret_cast<const uint32_t*>(wbuf + C::OFF_RAW);
  uint64_t* srow = reinterpret_cast<uint64_t*>(wbuf + C::OFF_ROW);
  auto fetch_raw = [&](int c) {
#pragma unroll
    for (int u = 0; u < kChunk / 4; ++u) {
      const int ch = lane + 32 * u;
      const int64_t e0 = p_begin + 32LL * kChunk * c + 4 * ch;
      const int64_t avail = p_end - e0;
      const uint32_t bytes = avail >= 4 ? 16u : (avail > 0 ? static_cast<uint32_t>(avail) * 4u : 0u);
      cp_async16(sraw_s + 16 * ch, p.col_indices + (bytes ? e0 : 0), bytes);
    }
  };
  bool bad_idx = false;
  const uint64_t seg_base = reinterpret_cast<uint64_t>(p.rhs_words) + static_cast<uint64_t>(brow0) * row_bytes +
                            static_cast<uint64_t>(col_byte);
  const uint64_t zero_row = reinterpret_cast<uint64_t>(g_seg_zero);
  // raw chunk c -> ring half c & 1; `newer` = cp.async groups committed after the chunk's
  // fetch (they may stay in flight)
  auto convert = [&](int c, auto newer) {
    cp_async_wait<decltype(newer)::value>();
    __syncwarp();
    const uint4 w0 = *reinterpret_cast<const uint4*>(sraw + 8 * lane);
    const uint4 w1 = *reinterpret_cast<const uint4*>(sraw + 8 * lane + 4);
    const uint32_t cw[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    uint64_t* dst = srow + (c & 1) * (32 * kChunk) + 32 * (lane >> 2);  // k-step lane / 4 of the chunk
    const int64_t pos0 = 32LL * kChunk * c + 8 * lane;                   // stored position of cw[0]
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int pp = 8 * (lane & 3) + e;  // position within the k-step
      const int q = pp & 7;
      const int kk = shuffled ? ((pp & ~7) | ((q & 3) << 1) | (q >> 2)) : pp;  // P: 0,2,4,6,1,3,5,7
      const uint32_t col = pos0 + e < stored ? cw[e] : kSentinel;
      const bool ok = col < kdim;
      bad_idx |= !ok && col != kSentinel;
      dst[(kk & 3) * 8 + (kk >> 2)] = ok ? seg_base + static_cast<uint64_t>(col) * row_bytes : zero_row;
    }
  };

  // LHS values: strides of 16 or 32 (the tile k of every plan, bench.py:103) make a k-step's
  // 32 positions one contiguous run of whole stride blocks -- [2 blocks][V][16] (S = 16) or
  // [V][32] (S = 32)
  const uint8_t* lhs_run = reinterpret_cast<const uint8_t*>(lhs) + (p_begin * V * LB) / 8;
  const int lhs_bytes = static_cast<int>(stored * V * LB / 8);
  const uint32_t srow_s = wbuf_s + C::OFF_ROW;

  auto issue = [&](int step, int st) {
    const int ck = step / kChunk, ks = step % kChunk;
    if (ks == 0 && 32LL * kChunk * (ck + 1) < stored) {
      __syncwarp();  // the staging buffer's previous chunk was converted 4 steps ago
      fetch_raw(ck + 1);
    }
    if (ks == kChunk / 2 && 32LL * kChunk * (ck + 1) < stored)
      convert(ck + 1, std::integral_constant<int, kChunk / 2 - 1>());  // fetched by issue(step - 4)
    const uint64_t* rr = srow + (ck & 1) * (32 * kChunk) + 32 * ks + 8 * pj;
    const uint32_t bst = wbuf_s + st * kBStage + pj * kSeg;
#pragma unroll
    for (int u2 = 0; u2 < 4; ++u2) {
      const ulonglong2 a2 = *reinterpret_cast<const ulonglong2*>(rr + 2 * u2);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int u = 2 * u2 + e;
        const char* src = reinterpret_cast<const char*>(e ? a2.y : a2.x) + 16 * pc;
        const uint32_t dst = bst + 4 * u * kSeg + ((pc ^ ((pj + 4 * u) & 7)) << 4);
        if (full_seg) cp_async16_full(dst, src);
        else cp_async16_zfill(dst, src, chunk_out);
      }
    }
    // LHS values of the step: A_STAGE contiguous bytes (whole stride blocks), 8 per lane
#pragma unroll
    for (int q = lane; q < C::A_STAGE / 8; q += 32) {
      const int off = step * C::A_STAGE + 8 * q;
      const bool ok = off < lhs_bytes;
      cp_async8(wbuf_s + C::OFF_A + st * C::A_STAGE + 8 * q, ok ? lhs_run + off : lhs_run, ok ? 8u : 0u);
    }
    cp_async_commit();
  };
  (void)srow_s;

  // ---- consumer. Chunk j (16 bytes) of the segment holds 16 byte-columns: 16 dense columns
  // at 8 bits, 32 at 4 bits; one LDSM.x2 over the 32 gathered rows is the A fragment of its 16
  // byte-columns x 32 k.
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

  int st_i = 0;  // stage of the next issued step
  if (nsteps > 0) {
    fetch_raw(0);
    cp_async_commit();
    convert(0, std::integral_constant<int, 0>());
    __syncwarp();
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < nsteps) issue(s, st_i);
      else cp_async_commit();
      st_i = st_i + 1 == STAGES ? 0 : st_i + 1;
    }
  }
  int st = 0;
  for (int s = 0; s < nsteps; ++s) {
    if (s + STAGES - 1 < nsteps) issue(s + STAGES - 1, st_i);
    else cp_async_commit();
    st_i = st_i + 1 == STAGES ? 0 : st_i + 1;
    cp_async_wait<STAGES - 1>();
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
    // this lane's ldmatrix row: slot `lane`, chunk j at j ^ (lane & 7)
    const uint32_t row_addr = wbuf_s + st * kBStage + lane * kSeg + ((lane & 7) << 4);
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      uint32_t a[4];
      ldsm_t16x2(row_addr ^ (j << 4), a[0], a[1], a[2], a[3]);
      if constexpr (RB == 4) {
        uint32_t y[4], hh[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          y[e] = PREX ? a[e] : a[e] ^ 0x08080808u;
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
    st = st + 1 == STAGES ? 0 : st + 1;
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
  if (overflow) flag_status(p.status, MC_STATUS_OVERFLOW);
  if (bad_idx) flag_status(p.status, MC_STATUS_BAD_INDEX);
}

template <int LB, int RB, int V, bool PREX>
cudaError_t launch_seg_v(SpmmParams p, cudaStream_t stream) {
  constexpr int kStages = 3;
  using C = SegCfg<LB, RB, V, kStages>;
  p.ntiles = (p.N + C::TN - 1) / C::TN;
  p.tasks = static_cast<int64_t>(p.batch) * p.vrows * p.ntiles;
  const unsigned grid = static_cast<unsigned>((p.tasks + kW - 1) / kW);
  if (grid == 0) return cudaSuccess;
  auto k = spmm_seg_kernel<LB, RB, V, kStages, PREX>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  const cudaError_t e = launch_pdl(k, dim3(grid), dim3(kW * 32), C::SMEM, stream, p);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int LB, int RB, bool PREX>
cudaError_t launch_seg_lr(const SpmmParams& p, cudaStream_t stream) {
  switch (p.V) {
    case 2: return launch_seg_v<LB, RB, 2, PREX>(p, stream);
    case 4: return launch_seg_v<LB, RB, 4, PREX>(p, stream);
    default: return launch_seg_v<LB, RB, 8, PREX>(p, stream);
  }
}

// bytes of the right-hand side(s) the kernel reads
size_t seg_rhs_bytes(const SpmmParams& p) {
  const int64_t one = p.K * p.N * p.RB / 8;
  return static_cast<size_t>(p.rhs_stride ? one * p.batch : one);
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
    case 804: return launch_seg_lr<8, 4, false>(p, stream);
    case 404: return launch_seg_lr<4, 4, false>(p, stream);
    case 808: return launch_seg_lr<8, 8, false>(p, stream);
    default: return launch_seg_lr<16, 8, false>(p, stream);
  }
}

// Workspace of the segment path: a copy of a 4-bit right-hand side with the low-nibble sign
// bits flipped (seg_prexor_kernel), one LOP per fragment word less in the main loop.
size_t spmm_seg_workspace(const SpmmParams& p) {
  if (p.RB != 4 || spmm_needs_nibble_chunks(p) || !spmm_seg_supported(p)) return 0;
  const char* e = getenv("MCUBE_SEG_PREXOR");
  if (e && e[0] == '0') return 0;
  return (seg_rhs_bytes(p) + 255) / 256 * 256;
}

cudaError_t launch_spmm_seg_ws(SpmmParams p, void* workspace, cudaStream_t stream) {
  const size_t bytes = seg_rhs_bytes(p);
  const int64_t n16 = static_cast<int64_t>(bytes / 16);
  if (n16 > 0) {
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n16 + 255) / 256, 148 * 8));
    const cudaError_t e = launch_pdl(seg_prexor_kernel, dim3(grid), dim3(256), 0, stream,
                                     reinterpret_cast<const uint4*>(p.rhs_words), static_cast<uint4*>(workspace), n16);
    count_launch();
    if (e != cudaSuccess) return e;
  }
  p.rhs_words = static_cast<const uint32_t*>(workspace);
  return p.LB == 8 ? launch_seg_lr<8, 4, true>(p, stream) : launch_seg_lr<4, 4, true>(p, stream);
}

}  // namespace mcube
