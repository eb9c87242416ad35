// gemm_sp.cu -- dense-tile SpMM without a densified copy of the LHS: builder warps write the
// SR-BCRS vectors of each 128 x 128 LHS tile straight into the shared-memory operand of an
// exact int8-plane tcgen05 GEMM (same product, planes and epilogue as gemm_tc.cu).
//
// The LHS tile is the UMMA A operand in the MN-major 128-byte-swizzled layout (128 m-bytes
// per k line, 8-line atoms 1024 B apart, 16-byte chunk c of line k at c ^ (k & 7)): a stored
// vector (V rows, one column) is V consecutive m-bytes of one line -- one 8/4/2-byte shared
// store per vector and plane, the SR-BCRS value split into the reference's chunks (qint.py:
// 185-225: low byte unsigned + high part signed for 12/16-bit, the value itself for 4/8-bit).
// This removes densify_kernel's HBM write + re-read of M*K*LC bytes (8-17 us of the 24-55 us
// C3 dense cells, measured warm).
//
// CTA (one per SM, persistent over 128 x 128 output tiles):
//   warp 0      TMA producer of the RC right-hand-side planes (128 k x 128 n boxes);
//   warp 1      TMEM allocator + single-thread MMA issuer (UMMA M=128 N=128 K=32, A and B MN-major);
//   warps 2-5   epilogue (TMEM lane quarter per warp, exact int64 recombination + int32 checks);
//   warps 6-13  LHS builders: warp b owns m-bytes [16 b, 16 b + 16) of every k line (one
//               16-byte chunk), i.e. the 16/V vector rows there. Each row streams its column
//               indices and stride blocks of values (contiguous per row, sparse_format.py:
//               131-139) through a 128/256-position shared-memory ring by cp.async, topped
//               up every k-block with kLook k-blocks of copies in flight. Per k-block the
//               warp zeroes its chunk of the LC planes and stores the block's vectors; a
//               row's cursor advances through its column list, which must be non-decreasing
//               per row (BcrsMatrix guarantees it; the caller asserts it with
//               MC_SRBCRS_SORTED, else the densify path runs). Shuffled indices
//               (sparse_format.py:222-230) advance in groups of 8 positions.
#include <cuda_fp16.h>

#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace mcube {
namespace {

constexpr int kTM = 128, kKB = 128;
constexpr int kBox = kTM * kKB;  // 16 KB per 128 x 128-byte plane tile
constexpr int kBuild = 8;        // builder warps (one 16-byte m chunk each)
constexpr int kLook = 4;         // cp.async groups (k-blocks of top-ups) kept in flight
constexpr int kFirstBuild = 6;
constexpr int kThreads = (kFirstBuild + kBuild) * 32;

template <int LB, int V, int LC, int RC>
struct SpCfg {
  static constexpr int TN = 128;
  static constexpr int STAGE = (LC + RC) * kBox;
  static constexpr int RPW = 16 / V;                 // vector rows per builder warp
  static constexpr int VB = V * LB / 8;              // value bytes per stored position
  static constexpr int BUILD_AT(int ring) { return kBuild * (RPW * ring * (4 + VB) + 16); }
  static constexpr int FIT_AT(int ring) { return (227 * 1024 - 2048 - BUILD_AT(ring)) / STAGE; }
  // positions per row ring: 256 (about kLook + 2 k-blocks at 30 % density) while three
  // operand stages still fit, else 128
  static constexpr int RING = FIT_AT(256) >= 3 ? 256 : 128;
  static constexpr int WARP_BUILD = RPW * RING * (4 + VB) + 16;  // + read slack of the 12-bit extractor
  static constexpr int BUILD = kBuild * WARP_BUILD;
  static constexpr int FIT = FIT_AT(RING);
  static constexpr int STAGES = FIT >= 5 ? 5 : (FIT < 2 ? 2 : FIT);
  static constexpr int NACC = LC * RC;
  static constexpr int SETS = NACC * TN <= 256 ? 2 : 1;
  static constexpr int CW = NACC == 4 ? 16 : 32;     // epilogue TMEM columns per load (registers)
  static constexpr int OFF_BUILD = STAGES * STAGE;
  static constexpr int OFF_BAR = OFF_BUILD + BUILD;
  static constexpr int N_BARS = 2 * STAGES + 2 * SETS;
  static constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
  static constexpr int TOTAL = OFF_TMEM + 16 + 1024;
};

__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t saddr, uint32_t lbo_bytes) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16) |
         (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// value position q of a row -> index position (SHUFFLE_PERMUTATION^-1, as dense.cu::index_pos)
__device__ __forceinline__ int idx_pos(int q, bool shuffled) {
  if (!shuffled) return q;
  const int w = q & 7;
  return (q & ~7) | ((w >> 1) | ((w & 1) << 2));
}
// index position -> value position
__device__ __forceinline__ int val_pos(int ip, bool shuffled) {
  if (!shuffled) return ip;
  const int w = ip & 7;
  return (ip & ~7) | (((w & 3) << 1) | (w >> 2));
}

// one LHS element (sign-extended), element index into the packed LB-bit value stream
template <int LB>
__device__ __forceinline__ int32_t lhs_elem(const uint32_t* __restrict__ words, int64_t e) {
  if constexpr (LB == 8) return __ldg(reinterpret_cast<const int8_t*>(words) + e);
  else if constexpr (LB == 16) return __ldg(reinterpret_cast<const int16_t*>(words) + e);
  else return fetch_packed(words, e, LB);
}

// element e of a stride block held in shared memory (LSB-first packing, qint.py:41-62),
// sign-extended
template <int LB>
__device__ __forceinline__ int32_t blk_elem(const uint8_t* blk, int e) {
  if constexpr (LB == 8) return static_cast<int8_t>(blk[e]);
  else if constexpr (LB == 16) return reinterpret_cast<const int16_t*>(blk)[e];
  else if constexpr (LB == 4) {
    const int32_t x = (blk[e >> 1] >> (4 * (e & 1))) & 0xF;
    return (x ^ 8) - 8;
  } else {  // 12
    const int bit = 12 * e;
    const int32_t x = ((blk[bit >> 3] | (blk[(bit >> 3) + 1] << 8)) >> (bit & 7)) & 0xFFF;
    return (x ^ 0x800) - 0x800;
  }
}

template <int N>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[N]);
template <>
__device__ __forceinline__ void tmem_ld_cols<32>(uint32_t taddr, uint32_t (&r)[32]) {
  tc::tmem_ld32_issue(taddr, r);
}
template <>
__device__ __forceinline__ void tmem_ld_cols<16>(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

struct SpMaps {
  CUtensorMap b[2];
};

template <int LB, int V, int LC, int RC>
__global__ void __launch_bounds__(kThreads, 1)
gemm_sp_kernel(const __grid_constant__ SpMaps maps, const SpmmParams p) {
  using C = SpCfg<LB, V, LC, RC>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar0 = sbase + C::OFF_BAR;
  auto full_bar = [&](int s) { return bar0 + 8 * s; };
  auto empty_bar = [&](int s) { return bar0 + 8 * (C::STAGES + s); };
  auto tfull_bar = [&](int a) { return bar0 + 8 * (2 * C::STAGES + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8 * (2 * C::STAGES + C::SETS + a); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);
  constexpr int kTN = C::TN;
  const int mt = static_cast<int>(p.M / kTM), nt = static_cast<int>(p.N / kTN);
  const int tiles = mt * nt;
  const int KB = static_cast<int>(p.K / kKB);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      tc::mbar_init(full_bar(s), 1 + kBuild);  // the TMA thread's expect_tx + one arrival per builder warp
      tc::mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < C::SETS; ++a) {
      tc::mbar_init(tfull_bar(a), 1);
      tc::mbar_init(tempty_bar(a), 4);
    }
    tc::fence_barrier_init();
    for (int j = 0; j < RC; ++j) tc::prefetch_tmap(&maps.b[j]);
  }
  if (warp == 1) tc::tmem_alloc<512>(smem_u32(tmem_holder));
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();  // the RHS planes may be written by the widen kernel just before
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ---------------- TMA producer (right-hand-side planes) ----------------
    if (lane == 0) {
      uint32_t g = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int n0 = (t % nt) * kTN;
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int s = g % C::STAGES;
          tc::mbar_wait(empty_bar(s), ((g / C::STAGES) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(full_bar(s), RC * kBox);
          const uint32_t st = sbase + s * C::STAGE;
#pragma unroll
          for (int j = 0; j < RC; ++j) tc::tma_load_2d(st + (LC + j) * kBox, &maps.b[j], full_bar(s), n0, kb * kKB);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      uint32_t g = 0;
      int it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
        const int set = it % C::SETS;
        tc::mbar_wait(tempty_bar(set), ((it / C::SETS) & 1) ^ 1);
        tc::tc_fence_after();
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int s = g % C::STAGES;
          tc::mbar_wait(full_bar(s), (g / C::STAGES) & 1);
          tc::tc_fence_after();
          const uint32_t st = sbase + s * C::STAGE;
#pragma unroll
          for (int i = 0; i < LC; ++i) {
#pragma unroll
            for (int j = 0; j < RC; ++j) {
              // A and B both MN-major (bits 15 / 16)
              const uint32_t idesc =
                  tc::idesc_i8(kTM, kTN, LC == 2 && i == 0, RC == 2 && j == 0) | (1u << 15) | (1u << 16);
              const uint32_t d = tmem + (set * C::NACC + i * RC + j) * kTN;
#pragma unroll
              for (int ks = 0; ks < kKB / 32; ++ks) {
                const uint64_t adesc = desc_mn_sw128(st + i * kBox + ks * 4096, kBox);
                const uint64_t bdesc = desc_mn_sw128(st + (LC + j) * kBox + ks * 4096, kBox);
                tc::mma_i8(d, adesc, bdesc, idesc, (kb > 0 || ks > 0) ? 1u : 0u);
              }
            }
          }
          tc::mma_commit(empty_bar(s));
        }
        tc::mma_commit(tfull_bar(set));
      }
    }
  } else if (warp < kFirstBuild) {
    // ---------------- epilogue: warp w reads TMEM lanes 32*(w%4).. (output rows) ----------------
    const int q = warp & 3;
    int it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int set = it % C::SETS;
      const int m0 = (t / nt) * kTM, n0 = (t % nt) * kTN;
      tc::mbar_wait(tfull_bar(set), (it / C::SETS) & 1);
      tc::tc_fence_after();
      const uint32_t tl = tmem + (static_cast<uint32_t>(32 * q) << 16) + set * C::NACC * kTN;
      int32_t* orow = p.out + static_cast<int64_t>(m0 + 32 * q + lane) * p.N + n0;
      bool overflow = false;
#pragma unroll 1
      for (int c = 0; c < kTN / C::CW; ++c) {
        uint32_t acc[C::NACC][C::CW];
#pragma unroll
        for (int a = 0; a < C::NACC; ++a) tmem_ld_cols<C::CW>(tl + a * kTN + C::CW * c, acc[a]);
        tc::tmem_wait_ld();
        int32_t res[C::CW];
#pragma unroll
        for (int x = 0; x < C::CW; ++x) {
          long long total = 0;
#pragma unroll
          for (int j = 0; j < RC; ++j) {
            long long tj;
            if constexpr (LC == 2) {
              const long long lo = static_cast<int32_t>(acc[0 * RC + j][x]);
              const long long hi = 256LL * static_cast<int32_t>(acc[1 * RC + j][x]);
              // the reference's stacked-group / nibble checks (as spmm.cu's epilogue)
              if (p.RB != 4) overflow |= (p.V == 8) ? !fits_i32(hi) : !fits_i32(lo + hi);
              else if (p.V == 4) overflow |= !fits_i32(hi);
              tj = lo + hi;
            } else {
              tj = static_cast<int32_t>(acc[j][x]);
            }
            total += tj << (8 * j);
          }
          overflow |= !fits_i32(total);
          res[x] = static_cast<int32_t>(total);
        }
#pragma unroll
        for (int x = 0; x < C::CW / 4; ++x)
          reinterpret_cast<int4*>(orow + C::CW * c)[x] =
              make_int4(res[4 * x], res[4 * x + 1], res[4 * x + 2], res[4 * x + 3]);
      }
      if (overflow) flag_status(p.status, MC_STATUS_OVERFLOW);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tempty_bar(set));
    }
  } else {
    // ---------------- LHS builders ----------------
    constexpr int RPW = C::RPW;
    constexpr int VB = C::VB;
    constexpr int kR = C::RING;
    const int bw = warp - kFirstBuild;
    const bool shuffled = p.shuffled != 0;
    const int S = p.S;  // power of two, 4 <= S <= kR (gemm_sp_ok)
    const uint32_t kdim = static_cast<uint32_t>(p.K);
    uint8_t* wb = smem + C::OFF_BUILD + bw * C::WARP_BUILD;
    const uint32_t wb_s = smem_u32(wb);
    const uint8_t* lhs_bytes = reinterpret_cast<const uint8_t*>(p.lhs_words);
    // row i's rings: indices at wb + i * 4 kR, values at wb + RPW * 4 kR + i * VB kR
    auto idx_ring = [&](int i) { return reinterpret_cast<const uint32_t*>(wb + i * 4 * kR); };
    auto val_ring = [&](int i) { return wb + RPW * 4 * kR + i * VB * kR; };
    // cp.async the positions [fill, to) (multiples of S, within the ring window) of row i
    auto fetch = [&](int i, int64_t pb, int fill, int to) {
      const int ni = (to - fill) / 4;          // 16-byte index chunks
      const int nv = (to - fill) * VB / 16;    // 16-byte value chunks
      for (int c = lane; c < ni + nv; c += 32) {
        if (c < ni) {
          const int pos = fill + 4 * c;
          cp_async16(wb_s + i * 4 * kR + (pos & (kR - 1)) * 4, p.col_indices + pb + pos, 16);
        } else {
          const int off = fill * VB + 16 * (c - ni);  // byte of the row's value stream
          cp_async16(wb_s + RPW * 4 * kR + i * VB * kR + (off % (VB * kR)),
                     lhs_bytes + pb * VB + off, 16);
        }
      }
    };
    bool bad = false;
    uint32_t g = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int m0 = (t / nt) * kTM;
      const int64_t vr0 = m0 / V + bw * RPW;
      // lane i < RPW holds row vr0 + i: begin, true / stored counts, cursor, fetched and landed fronts
      int64_t my_pb = 0;
      int my_nt = 0, my_st = 0, my_cur = 0, my_fill = 0, my_land = 0;
      int fh[kLook] = {};  // this lane's row: fetched front after the top-ups of the last kLook k-blocks
      if (lane < RPW && vr0 + lane < p.vrows) {
        my_pb = p.row_begin[vr0 + lane];
        my_nt = static_cast<int>(p.row_end[vr0 + lane] - my_pb);
        my_st = (my_nt + S - 1) / S * S;
      }
      cp_async_wait<0>();  // the previous tile's copies may not land in the rings afterwards
      __syncwarp();
      for (int kb = 0; kb < KB; ++kb, ++g) {
#ifdef MCUBE_SP_PROBE
        if (p.gather_tma == 7) {  // timing probe: stage handshake only (wrong results)
          const int s = g % C::STAGES;
          tc::mbar_wait(empty_bar(s), ((g / C::STAGES) & 1) ^ 1);
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(full_bar(s));
          continue;
        }
        if (p.gather_tma == 6) {  // timing probe: no ring top-ups (wrong results)
          const int s = g % C::STAGES;
          tc::mbar_wait(empty_bar(s), ((g / C::STAGES) & 1) ^ 1);
          const uint32_t st = sbase + s * C::STAGE;
#pragma unroll
          for (int pl = 0; pl < LC; ++pl)
#pragma unroll
            for (int x = 0; x < kKB / 32; ++x) {
              const int line = lane + 32 * x;
              const uint32_t a = st + pl * kBox + (line >> 3) * 1024 + (line & 7) * 128 + ((bw ^ (line & 7)) << 4);
              asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(a), "r"(0) : "memory");
            }
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(full_bar(s));
          continue;
        }
#endif
        // ---- top up every row's ring (positions from the cursor's stride block on) ----
        for (int i = 0; i < RPW; ++i) {
          const int64_t pb = __shfl_sync(0xffffffffu, my_pb, i);
          const int sto = __shfl_sync(0xffffffffu, my_st, i);
          const int cur = __shfl_sync(0xffffffffu, my_cur, i);
          const int fill = __shfl_sync(0xffffffffu, my_fill, i);
          const int lim = min(sto, (cur & ~(S - 1)) + kR);
          if (lim > fill) {
            fetch(i, pb, fill, lim);
            if (lane == i) my_fill = lim;
          }
        }
        cp_async_commit();
        // all but the last kLook groups have landed: the fronts of kLook k-blocks ago
        cp_async_wait<kLook>();
        __syncwarp();
        my_land = fh[kb % kLook];
        fh[kb % kLook] = my_fill;
        bool all_landed = false;

        const int s = g % C::STAGES;
        tc::mbar_wait(empty_bar(s), ((g / C::STAGES) & 1) ^ 1);
        const uint32_t st = sbase + s * C::STAGE;
        // zero this warp's 16-byte chunk bw of every k line of the LC planes
#pragma unroll
        for (int pl = 0; pl < LC; ++pl)
#pragma unroll
          for (int x = 0; x < kKB / 32; ++x) {
            const int line = lane + 32 * x;
            const uint32_t a = st + pl * kBox + (line >> 3) * 1024 + (line & 7) * 128 + ((bw ^ (line & 7)) << 4);
            asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(a), "r"(0) : "memory");
          }
        __syncwarp();
        const uint32_t kb0 = static_cast<uint32_t>(kb) * kKB, kb1 = kb0 + kKB;
        for (int i = 0; i < RPW; ++i) {
          const int64_t pb = __shfl_sync(0xffffffffu, my_pb, i);
          const int ntr = __shfl_sync(0xffffffffu, my_nt, i);
          const int sto = __shfl_sync(0xffffffffu, my_st, i);
          int pos = __shfl_sync(0xffffffffu, my_cur, i);
          int fill = __shfl_sync(0xffffffffu, my_fill, i);
          int land = __shfl_sync(0xffffffffu, my_land, i);
          const uint32_t* ir = idx_ring(i);
          const uint8_t* vr = val_ring(i);
          const uint32_t mo = static_cast<uint32_t>(V * i);  // m-byte of the row inside the chunk
          while (pos < sto) {
            const int need = min(pos + 32, sto);
            if (need > fill) {  // the row outran its ring (a dense stretch): refill from the cursor
              const int lim = min(sto, (pos & ~(S - 1)) + kR);
              fetch(i, pb, fill, lim);
              cp_async_commit();
              fill = lim;
              if (lane == i) my_fill = lim;
              all_landed = false;
            }
            if (need > land) {
              if (!all_landed) {
                cp_async_wait<0>();
                __syncwarp();
                all_landed = true;
              }
              land = fill;
            }
            const int ip = pos + lane;
            const bool inr = ip < sto;
            const uint32_t col = inr ? ir[ip & (kR - 1)] : kSentinel;
            const int qv = val_pos(ip, shuffled);
            const bool real = inr && qv < ntr;
            bad |= real && col >= kdim && col != kSentinel;
            const bool valid = real && col < kdim;
            if (valid && col >= kb0 && col < kb1) {
              // element (v, q) of the row: stride block q / S, offset v * S + q % S
              // (sparse_format.py:131-139); the block sits whole in the value ring
              const int qb = qv & ~(S - 1), j = qv & (S - 1);
              const uint8_t* blk = vr + (qb & (kR - 1)) * VB;
              uint32_t w0[2] = {0u, 0u}, w1[2] = {0u, 0u};
#pragma unroll
              for (int v = 0; v < V; ++v) {
                const int32_t x = blk_elem<LB>(blk, v * S + j);
                w0[v >> 2] |= (static_cast<uint32_t>(x) & 0xFFu) << (8 * (v & 3));
                if constexpr (LC == 2) w1[v >> 2] |= ((static_cast<uint32_t>(x) >> 8) & 0xFFu) << (8 * (v & 3));
              }
              const uint32_t kl = col - kb0;
              const uint32_t a = st + (kl >> 3) * 1024 + (kl & 7) * 128 + ((static_cast<uint32_t>(bw) ^ (kl & 7)) << 4) + mo;
#pragma unroll
              for (int pl = 0; pl < LC; ++pl) {
                const uint32_t* w = pl == 0 ? w0 : w1;
                const uint32_t ap = a + pl * kBox;
                if constexpr (V == 8) asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(ap), "r"(w[0]), "r"(w[1]) : "memory");
                else if constexpr (V == 4) asm volatile("st.shared.u32 [%0], %1;" ::"r"(ap), "r"(w[0]) : "memory");
                else asm volatile("st.shared.u16 [%0], %1;" ::"r"(ap), "h"(static_cast<uint16_t>(w[0])) : "memory");
              }
            }
            // advance past the leading positions (groups of 8 when shuffled) that are done
            const uint32_t beyond = __ballot_sync(0xffffffffu, valid && col >= kb1);
            int adv = 32;
            if (beyond) adv = shuffled ? ((__ffs(beyond) - 1) & ~7) : (__ffs(beyond) - 1);
            pos += adv;
            if (adv < 32) break;
          }
          if (lane == i) my_cur = pos;
          if (all_landed && lane < RPW) my_land = my_fill;
        }
        tc::fence_proxy_async();  // generic-proxy stores -> visible to the tensor-core (async) proxy
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(full_bar(s));
      }
    }
    cp_async_wait<0>();
    if (bad) flag_status(p.status, MC_STATUS_BAD_INDEX);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem);
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn sp_encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(f);
  }
  return fn;
}

// 2-D int8 map [rows x cols] row-major, box 128 x 128, 128-byte swizzle
bool sp_map128(CUtensorMap* m, const void* base, int64_t rows, int64_t cols) {
  EncodeFn fn = sp_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols)};
  cuuint32_t box[2] = {128, 128};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int LB, int V, int LC, int RC>
cudaError_t launch_sp(const SpMaps& maps, const SpmmParams& p, cudaStream_t stream) {
  using C = SpCfg<LB, V, LC, RC>;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles = static_cast<int>((p.M / kTM) * (p.N / C::TN));
  auto k = gemm_sp_kernel<LB, V, LC, RC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::TOTAL);
  const cudaError_t e = launch_pdl(k, dim3(tiles < sms ? tiles : sms), dim3(kThreads), C::TOTAL, stream, maps, p);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int LB, int LC, int RC>
cudaError_t launch_sp_v(const SpMaps& maps, const SpmmParams& p, cudaStream_t stream) {
  switch (p.V) {
    case 2: return launch_sp<LB, 2, LC, RC>(maps, p, stream);
    case 4: return launch_sp<LB, 4, LC, RC>(maps, p, stream);
    default: return launch_sp<LB, 8, LC, RC>(maps, p, stream);
  }
}

template <int RC>
cudaError_t launch_sp_l(const SpMaps& maps, const SpmmParams& p, cudaStream_t stream) {
  switch (p.LB) {
    case 4: return launch_sp_v<4, 1, RC>(maps, p, stream);
    case 8: return launch_sp_v<8, 1, RC>(maps, p, stream);
    case 12: return launch_sp_v<12, 2, RC>(maps, p, stream);
    default: return launch_sp_v<16, 2, RC>(maps, p, stream);
  }
}

}  // namespace

// The fused kernel's requirements beyond dense_spmm_eligible: rows asserted non-decreasing
// (MC_SRBCRS_SORTED), power-of-two strides that fit the ring, 16-byte stride blocks.
bool gemm_sp_ok(const SpmmParams& p) {
  if (!p.sorted || p.S < 4 || p.S > 128 || (p.S & (p.S - 1))) return false;
  if ((static_cast<int64_t>(p.S) * p.V * p.LB / 8) % 16 != 0) return false;
  return (reinterpret_cast<uintptr_t>(p.lhs_words) & 15) == 0 && (reinterpret_cast<uintptr_t>(p.col_indices) & 15) == 0;
}

// The fused dense-tile SpMM: b0 / b1 are the RHS int8 planes [K x N] (the packed words
// themselves for an 8-bit RHS, widen_kernel's planes otherwise).
cudaError_t launch_gemm_sp(const SpmmParams& p, const int8_t* b0, const int8_t* b1, cudaStream_t stream) {
  SpMaps maps;
  memset(&maps, 0, sizeof(maps));
  const int rc = p.RB == 16 ? 2 : 1;
  if (!sp_map128(&maps.b[0], b0, p.K, p.N) || (rc == 2 && !sp_map128(&maps.b[1], b1, p.K, p.N)))
    return cudaErrorInvalidValue;
  return rc == 2 ? launch_sp_l<2>(maps, p, stream) : launch_sp_l<1>(maps, p, stream);
}

}  // namespace mcube
