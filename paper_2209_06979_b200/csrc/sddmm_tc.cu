// sddmm_tc.cu -- dense-tile SDDMM on the 5th-gen tensor cores (tcgen05 kind::i8, TMEM, TMA).
//
// For pattern densities above ~8% (C2 at 50..90% sparsity) the cheapest way to
// produce the sampled dot products on B200 is to compute whole 128 x 256 tiles of
// D^T = B^T A^T on tcgen05 at int8 tensor-core rate and write out only the pattern
// blocks: the tile product reads each operand byte from shared memory once per
// 128/256 outputs, whereas a gather reads one K-byte B^T row per block.
// Bit-exact: int8 x int8 products accumulate exactly in int32 TMEM for K <= 33025
// (check_accumulation_bound, emulation.py:108-113), identical to kernels.sddmm.
//
// CTA (448 threads, 1 per SM, persistent over a contiguous panel-major tile range):
//   warp 0      TMA producer: A panel (256 rows x K, resident while the panel is
//               unchanged) and a 2-stage ring of B^T tiles (128 rows x K);
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (M = 128 pattern columns, N = 256 scalar rows, K step 32);
//   warps 2..9  consumers (two per TMEM lane quarter, each draining half of the
//               accumulator columns): tcgen05.ld the accumulator (TMEM lane = pattern column,
//               TMEM column = scalar row, double-buffered loads) and store each
//               present block's V int32 values as one sector-sized vector store;
//   warps 10..13 builders: walk the pattern with one forward cursor per vector row
//               (the first found by interpolation search) through a shared-memory
//               window of column indices, and publish a per-tile
//               column -> block-slot map, double buffered ahead of the consumers.
// TMEM holds two 256-column accumulators so MMA of tile i+1 overlaps the drain of i.
#include <cuda_fp16.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace mcube {

// Debug timeline (MCUBE_DEBUG_TIMELINE=1): globaltimer stamps per CTA, read by mc_debug_timeline.
__device__ unsigned long long g_timeline[148 * 64];
__device__ __forceinline__ void stamp(bool on, int slot) {
  if (on && slot < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_timeline[blockIdx.x * 64 + slot] = t;
  }
}

namespace {

constexpr int kPanel = 256;   // scalar rows of A per tile (UMMA N)
constexpr int kCols = 128;    // pattern columns per tile (UMMA M)
constexpr int kStages = 2;
constexpr int kThreads = 448;
constexpr uint32_t kIdesc = tc::idesc_i8(128, 256);

template <int V>
struct Smem {
  static constexpr int VR = kPanel / V;                    // vector rows per panel
  static constexpr int WIN = V == 8 ? 512 : 256;           // cached column indices per row (uint32)
  static constexpr int A_BYTES = 2 * kPanel * 128;         // 64 KB (K <= 256)
  static constexpr int B_STAGE = 2 * kCols * 128;          // 32 KB
  static constexpr int POSMAP = kCols * VR;                // [column][vector row] slot codes
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = OFF_A + A_BYTES;
  static constexpr int OFF_POS = OFF_B + kStages * B_STAGE;
  static constexpr int OFF_WIN = OFF_POS + 2 * POSMAP;     // uint32 [VR][WIN]
  static constexpr int OFF_CUR = OFF_WIN + VR * WIN * 4;   // int64 cursor[VR]
  static constexpr int OFF_WLO = OFF_CUR + 128 * 8;        // int64 window start[VR]
  static constexpr int OFF_WN = OFF_WLO + 128 * 8;         // int32 window count[VR]
  static constexpr int OFF_TBASE = OFF_WN + 128 * 4;       // int64 [2][VR]
  static constexpr int OFF_BAR = OFF_TBASE + 2 * 128 * 8;
  static constexpr int N_BARS = 2 * kStages + 2 + 4 + 4;
  static constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
  static constexpr int TOTAL = OFF_TMEM + 16 + 1024;       // + alignment slack
};

// first index j in [lo, hi) with cols[j] >= c0 (cols sorted): interpolation + 64-wide windows
__device__ int64_t lower_bound_interp(const uint32_t* __restrict__ cols, int64_t lo, int64_t hi, uint32_t c0,
                                      uint32_t ncols) {
  if (c0 == 0 || lo >= hi) return lo;
  uint32_t clo = 0, chi = ncols;  // cols[lo..hi) lie in [clo, chi)
  while (hi - lo > 0) {
    const int64_t n = hi - lo;
    const double frac = chi > clo ? static_cast<double>(c0 - clo) / static_cast<double>(chi - clo) : 0.5;
    const int64_t g = lo + static_cast<int64_t>(frac * static_cast<double>(n));
    int64_t w0 = g - 32;
    if (w0 < lo) w0 = lo;
    int64_t w1 = w0 + 64;
    if (w1 > hi) {
      w1 = hi;
      w0 = (hi - 64 > lo) ? hi - 64 : lo;
    }
    uint32_t win[64];
#pragma unroll
    for (int x = 0; x < 64; ++x) win[x] = (w0 + x < w1) ? __ldg(cols + w0 + x) : 0xFFFFFFFFu;
    int cnt = 0;
    uint32_t last = win[0];
#pragma unroll
    for (int x = 0; x < 64; ++x) {
      const bool in = w0 + x < w1;
      cnt += in && (win[x] < c0);
      if (in) last = win[x];
    }
    if (cnt == 0 && w0 > lo) {
      hi = w0;
      chi = win[0];
      continue;
    }
    if (cnt == static_cast<int>(w1 - w0) && w1 < hi) {
      lo = w1;
      clo = last + 1;
      continue;
    }
    return w0 + cnt;
  }
  return lo;
}

template <int V>
__global__ void __launch_bounds__(kThreads, 1)
sddmm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const SddmmTcParams p) {
  using L = Smem<V>;
  constexpr int VR = L::VR;
  constexpr int WIN = L::WIN;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // align to 1024 B with pointer arithmetic (keeps the shared address space for LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = static_cast<int>(p.K / 128);
  uint8_t* posmap0 = smem + L::OFF_POS;
  uint32_t* win = reinterpret_cast<uint32_t*>(smem + L::OFF_WIN);
  int64_t* cursor = reinterpret_cast<int64_t*>(smem + L::OFF_CUR);
  int64_t* win_lo = reinterpret_cast<int64_t*>(smem + L::OFF_WLO);
  int32_t* win_n = reinterpret_cast<int32_t*>(smem + L::OFF_WN);
  int64_t* tbase_arr = reinterpret_cast<int64_t*>(smem + L::OFF_TBASE);
  const uint32_t bar0 = sbase + L::OFF_BAR;
  auto full_bar = [&](int s) { return bar0 + 8 * s; };
  auto empty_bar = [&](int s) { return bar0 + 8 * (kStages + s); };
  const uint32_t a_full = bar0 + 8 * (2 * kStages), a_empty = a_full + 8;
  auto tfull_bar = [&](int a) { return bar0 + 8 * (2 * kStages + 2 + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8 * (2 * kStages + 4 + a); };
  auto pfull_bar = [&](int b) { return bar0 + 8 * (2 * kStages + 6 + b); };
  auto pempty_bar = [&](int b) { return bar0 + 8 * (2 * kStages + 8 + b); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

  const bool dbg = p.debug != 0;
  stamp(dbg && threadIdx.x == 0, 0);
  const int64_t t0 = (p.tiles * blockIdx.x) / gridDim.x;
  const int64_t t1 = (p.tiles * (blockIdx.x + 1)) / gridDim.x;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(full_bar(s), 1);
      tc::mbar_init(empty_bar(s), 1);
    }
    tc::mbar_init(a_full, 1);
    tc::mbar_init(a_empty, 1);
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(tfull_bar(a), 1);
      tc::mbar_init(tempty_bar(a), 8);
      tc::mbar_init(pfull_bar(a), 128);
      tc::mbar_init(pempty_bar(a), 8);
    }
    tc::fence_barrier_init();
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
  }
  if (warp == 1) tc::tmem_alloc<512>(smem_u32(tmem_holder));
  // Builders: start fetching the first panel's pattern window right away, positioned by
  // the average row length (validated against the real row offsets after the sync).
  int64_t pre_a0 = 0, pre_lo = 0, pre_end = 0;
  if (warp >= 10 && t0 < t1) {
    const int bt = threadIdx.x - 320;
    constexpr int TPR = 128 / VR;
    const int rl = bt / TPR, sub = bt % TPR;
    const int64_t panel = t0 / p.n_ctiles;
    const uint32_t c0 = static_cast<uint32_t>((t0 % p.n_ctiles) * kCols);
    const int64_t r = panel * VR + rl;
    if (r < p.vrows) {
      pre_lo = p.row_offsets[r];  // consumed after the barrier: the load latency overlaps setup
      pre_end = p.row_offsets[r + 1];
    }
    if (r < p.vrows && p.n_blocks > 0) {
      const double avg = static_cast<double>(p.n_blocks) / static_cast<double>(p.vrows);
      const int64_t g = static_cast<int64_t>(avg * (static_cast<double>(r) + static_cast<double>(c0) / p.N));
      pre_a0 = (g - 64 > 0 ? g - 64 : 0) & ~3LL;
      uint32_t* wrow = win + rl * WIN;
      for (int ch = sub; ch < WIN / 4; ch += TPR) {
        const int64_t e0 = pre_a0 + 4 * ch;
        const uint32_t bytes =
            e0 < p.n_blocks ? static_cast<uint32_t>((p.n_blocks - e0) >= 4 ? 16 : (p.n_blocks - e0) * 4) : 0u;
        cp_async16(smem_u32(wrow) + 16 * ch, p.col_indices + (bytes ? e0 : 0), bytes);
      }
    }
    cp_async_commit();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  stamp(dbg && threadIdx.x == 0, 1);

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int64_t cur_panel = -1;
      int n_a = 0;
      for (int64_t t = t0; t < t1; ++t) {
        const int64_t i = t - t0;
        const int64_t panel = t / p.n_ctiles, ct = t % p.n_ctiles;
        if (panel != cur_panel) {
          if (n_a > 0) tc::mbar_wait(a_empty, (n_a - 1) & 1);
          tc::mbar_arrive_expect_tx(a_full, KB * kPanel * 128);
          for (int kb = 0; kb < KB; ++kb)
            tc::tma_load_2d(sbase + L::OFF_A + kb * kPanel * 128, &tmA, a_full, kb * 128,
                            static_cast<int>(panel * kPanel));
          ++n_a;
          cur_panel = panel;
        }
        const int s = static_cast<int>(i % kStages);
        const uint32_t u = static_cast<uint32_t>(i / kStages);
        tc::mbar_wait(empty_bar(s), (u & 1) ^ 1);
        tc::mbar_arrive_expect_tx(full_bar(s), KB * kCols * 128);
        for (int kb = 0; kb < KB; ++kb)
          tc::tma_load_2d(sbase + L::OFF_B + s * L::B_STAGE + kb * kCols * 128, &tmB, full_bar(s), kb * 128,
                          static_cast<int>(ct * kCols));
        stamp(dbg && i < 6, 2 + static_cast<int>(i));
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      int64_t cur_panel = -1;
      int n_a = 0;
      for (int64_t t = t0; t < t1; ++t) {
        const int64_t i = t - t0;
        const int64_t panel = t / p.n_ctiles;
        if (panel != cur_panel) {
          tc::mbar_wait(a_full, n_a & 1);
          ++n_a;
          cur_panel = panel;
        }
        const int s = static_cast<int>(i % kStages);
        const uint32_t u = static_cast<uint32_t>(i / kStages);
        const int acc = static_cast<int>(i & 1);
        const uint32_t u2 = static_cast<uint32_t>(i >> 1);
        tc::mbar_wait(tempty_bar(acc), (u2 & 1) ^ 1);
        tc::mbar_wait(full_bar(s), u & 1);
        tc::tc_fence_after();
        stamp(dbg && i < 6, 10 + static_cast<int>(i));
        const uint32_t d = tmem + acc * 256;
        const uint32_t bs = sbase + L::OFF_B + s * L::B_STAGE;
        const uint32_t as = sbase + L::OFF_A;
        for (int ks = 0; ks < KB * 4; ++ks) {
          const int kb = ks >> 2, off = (ks & 3) * 32;
          const uint64_t adesc = tc::desc_k_sw128(bs + kb * kCols * 128 + off);   // B^T tile: M = 128
          const uint64_t bdesc = tc::desc_k_sw128(as + kb * kPanel * 128 + off);  // A panel:  N = 256
          tc::mma_i8(d, adesc, bdesc, kIdesc, ks > 0 ? 1u : 0u);
        }
        tc::mma_commit(empty_bar(s));
        tc::mma_commit(tfull_bar(acc));
        stamp(dbg && i < 6, 16 + static_cast<int>(i));
        if (t + 1 == t1 || (t + 1) / p.n_ctiles != panel) tc::mma_commit(a_empty);
      }
    }
  } else if (warp < 10) {
    // ---------------- consumers: TMEM -> registers -> 32-byte block stores ----------------
    // two warps per TMEM lane quarter; warp group `half` drains accumulator columns
    // [128*half, 128*half + 128) (chunks 4*half .. 4*half+3)
    const int ct_id = threadIdx.x - 64;
    const int half = (warp - 2) >> 2;
    const int q = warp & 3;  // TMEM lane quarter accessible to this warp
    const int c_local = 32 * q + lane;
    constexpr int rpc = 32 / V;  // vector rows per 32-row chunk
    double alpha = 0.0;
    if (p.out_f16) alpha = p.alpha ? p.alpha[0] : p.alpha_host;
    for (int64_t t = t0; t < t1; ++t) {
      const int64_t i = t - t0;
      const int b = static_cast<int>(i & 1);
      const uint32_t ub = static_cast<uint32_t>(i >> 1);
      tc::mbar_wait(pfull_bar(b), ub & 1);
      // this column's slot codes for all VR vector rows (posmap is [column][vector row])
      uint32_t codes[VR / 4];
      const uint32_t* pc = reinterpret_cast<const uint32_t*>(posmap0 + b * L::POSMAP + c_local * VR);
#pragma unroll
      for (int x = 0; x < VR / 4; ++x) codes[x] = pc[x];
      const int64_t* tb = tbase_arr + b * 128;
      tc::mbar_wait(tfull_bar(b), ub & 1);  // accumulator index == posmap index == i & 1
      tc::tc_fence_after();
      stamp(dbg && ct_id == 0 && i < 6, 23 + 3 * static_cast<int>(i));
      const uint32_t tl = tmem + (static_cast<uint32_t>(32 * q) << 16) + b * 256;
      uint32_t va[32], vb[32];
      constexpr int kChunks = kPanel / 64;  // chunks per consumer warp group
      tc::tmem_ld32_issue(tl + 128 * half, va);
      tc::tmem_wait_ld();
#pragma unroll
      for (int kk = 0; kk < kChunks; ++kk) {
        const int k = kChunks * half + kk;
        uint32_t(&cur)[32] = (kk & 1) ? vb : va;
        uint32_t(&nxt)[32] = (kk & 1) ? va : vb;
        if (kk + 1 < kChunks) tc::tmem_ld32_issue(tl + 32 * (k + 1), nxt);
#pragma unroll
        for (int w = 0; w < rpc; ++w) {
          const int rl = k * rpc + w;
          const int code = (codes[rl >> 2] >> (8 * (rl & 3))) & 0xFF;
          if (code) {
            const int64_t pos = tb[rl] + code - 1;
            int32_t* o = p.out + pos * V;
            if constexpr (V == 8) {
              tc::st_global_v8(o, cur[8 * w], cur[8 * w + 1], cur[8 * w + 2], cur[8 * w + 3], cur[8 * w + 4],
                               cur[8 * w + 5], cur[8 * w + 6], cur[8 * w + 7]);
            } else if constexpr (V == 4) {
              *reinterpret_cast<int4*>(o) = make_int4(cur[4 * w], cur[4 * w + 1], cur[4 * w + 2], cur[4 * w + 3]);
            } else {
              *reinterpret_cast<int2*>(o) = make_int2(cur[2 * w], cur[2 * w + 1]);
            }
            if (p.out_f16) {
#pragma unroll
              for (int v = 0; v < V; ++v)
                p.out_f16[pos * V + v] = f16_bits_rn(static_cast<double>(static_cast<int32_t>(cur[V * w + v])) * alpha);
            }
          }
        }
        if (kk + 1 < kChunks) tc::tmem_wait_ld();
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        tc::mbar_arrive(tempty_bar(b));
        tc::mbar_arrive(pempty_bar(b));
      }
      stamp(dbg && ct_id == 0 && i < 6, 24 + 3 * static_cast<int>(i));
    }
  } else {
    // ---------------- builders: pattern cursor -> per-tile column map ----------------
    const int bt = threadIdx.x - 320;
    constexpr int TPR = 128 / VR;  // builder threads per vector row (a group of lanes in one warp)
    const int rl = bt / TPR, sub = bt % TPR;
    uint32_t* wrow = win + rl * WIN;
    const unsigned gmask = ((1u << TPR) - 1u) << (lane & ~(TPR - 1));
    int64_t cur_panel = -1;
    for (int64_t t = t0; t < t1; ++t) {
      const int64_t i = t - t0;
      const int b = static_cast<int>(i & 1);
      const uint32_t ub = static_cast<uint32_t>(i >> 1);
      const int64_t panel = t / p.n_ctiles, ct = t % p.n_ctiles;
      const uint32_t c0 = static_cast<uint32_t>(ct * kCols);
      const int64_t r = panel * VR + rl;
      const bool row_ok = r < p.vrows;
      const int64_t end = row_ok ? (t == t0 ? pre_end : p.row_offsets[r + 1]) : 0;
      if (panel != cur_panel) {
        // First cursor of the panel: fetch a WIN-entry window around the interpolated
        // position of c0 (one round trip) and locate the cursor inside it; fall back to
        // the interpolation search only when the window misses.
        const int64_t lo = row_ok ? (t == t0 ? pre_lo : p.row_offsets[r]) : 0;
        int64_t a0 = lo;
        if (t == t0) {
          a0 = pre_a0;  // window prefetched before the setup barrier
        } else if (row_ok && end > lo) {
          const int64_t g = lo + static_cast<int64_t>((static_cast<double>(c0) / p.N) * static_cast<double>(end - lo));
          a0 = (g - 64 > lo ? g - 64 : lo) & ~3LL;
          for (int ch = sub; ch < WIN / 4; ch += TPR) {
            const int64_t e0 = a0 + 4 * ch;
            const uint32_t bytes = e0 < end ? static_cast<uint32_t>((end - e0) >= 4 ? 16 : (end - e0) * 4) : 0u;
            cp_async16(smem_u32(wrow) + 16 * ch, p.col_indices + (bytes ? e0 : 0), bytes);
          }
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        // cached entries of this row: [s0, e1)
        const int64_t s0 = a0 > lo ? a0 : lo;
        const int64_t e1 = (a0 + WIN < end) ? a0 + WIN : end;
        const int64_t n_eff = e1 > s0 ? e1 - s0 : 0;
        int cnt = 0;
        for (int64_t x = sub; x < n_eff; x += TPR) cnt += wrow[s0 - a0 + x] < c0;
#pragma unroll
        for (int o = 1; o < TPR; o <<= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        const int64_t n = e1 > a0 ? e1 - a0 : 0;
        if (sub == 0) {
          int64_t lb = s0 + cnt;
          // the window must bracket the lower bound; a short tail is refilled by the main loop
          const bool miss = row_ok && end > lo &&
                            (n_eff == 0 || (cnt == 0 && s0 > lo) || (cnt == n_eff && e1 < end));
          if (miss) {
            lb = lower_bound_interp(p.col_indices, lo, end, c0, static_cast<uint32_t>(p.N));
            win_lo[rl] = 0;
            win_n[rl] = 0;
          } else {
            win_lo[rl] = a0;
            win_n[rl] = static_cast<int32_t>(n);
          }
          cursor[rl] = row_ok ? lb : 0;
        }
        cur_panel = panel;
        stamp(dbg && bt == 0, 40);
      }
      cp_async_wait<0>();  // an asynchronous window refill issued after the previous tile
      __syncwarp();
      const int64_t base = cursor[rl];
      // refill the row's cached window (cp.async, 16-byte chunks) when the next 128
      // candidates are not all cached
      if (row_ok && base + kCols > win_lo[rl] + win_n[rl] && win_lo[rl] + win_n[rl] < end) {
        const int64_t a0 = base & ~3LL;
        const int64_t n = (end - a0 < WIN) ? (end - a0) : WIN;
        for (int ch = sub; ch < WIN / 4; ch += TPR) {
          const int64_t e0 = a0 + 4 * ch;
          const uint32_t bytes = e0 < end ? static_cast<uint32_t>((end - e0) >= 4 ? 16 : (end - e0) * 4) : 0u;
          cp_async16(smem_u32(wrow) + 16 * ch, p.col_indices + (bytes ? e0 : 0), bytes);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp(gmask);
        if (sub == 0) {
          win_lo[rl] = a0;
          win_n[rl] = static_cast<int32_t>(n);
        }
        __syncwarp(gmask);
      }
      tc::mbar_wait(pempty_bar(b), (ub & 1) ^ 1);
      uint8_t* posmap = posmap0 + b * L::POSMAP;
      {
        uint4* pm = reinterpret_cast<uint4*>(posmap);
        constexpr int n16 = L::POSMAP / 16;
        for (int x = bt; x < n16; x += 128) pm[x] = make_uint4(0, 0, 0, 0);
      }
      tc::named_bar(2, 128);
      int64_t stop = 0;
      if (row_ok) {
        const int64_t lim = (end < base + kCols) ? end : base + kCols;
        stop = lim;
        const int64_t wl = win_lo[rl];
        for (int64_t j = base + sub; j < lim; j += TPR) {
          const uint32_t c = wrow[j - wl];
          if (c >= c0 + kCols) {
            stop = j;
            break;
          }
          posmap[(c - c0) * VR + rl] = static_cast<uint8_t>(j - base + 1);
        }
      }
      __syncwarp();
#pragma unroll
      for (int o = 1; o < TPR; o <<= 1) {
        const int64_t other = __shfl_xor_sync(0xffffffffu, stop, o);
        stop = other < stop ? other : stop;
      }
      if (sub == 0) {
        tbase_arr[b * 128 + rl] = base;
        if (row_ok) cursor[rl] = stop;
      }
      tc::mbar_arrive(pfull_bar(b));
      stamp(dbg && bt == 0 && i < 6, 22 + 3 * static_cast<int>(i));
      // Prefetch the next tile's candidates now (asynchronously) if the cached window
      // will not cover them; the copy lands while the builder waits for a free map.
      if (t + 1 < t1 && (t + 1) / p.n_ctiles == panel && row_ok && stop + kCols > win_lo[rl] + win_n[rl] &&
          win_lo[rl] + win_n[rl] < end) {
        __syncwarp(gmask);
        const int64_t a0 = stop & ~3LL;
        const int64_t n = (end - a0 < WIN) ? (end - a0) : WIN;
        for (int ch = sub; ch < WIN / 4; ch += TPR) {
          const int64_t e0 = a0 + 4 * ch;
          const uint32_t bytes = e0 < end ? static_cast<uint32_t>((end - e0) >= 4 ? 16 : (end - e0) * 4) : 0u;
          cp_async16(smem_u32(wrow) + 16 * ch, p.col_indices + (bytes ? e0 : 0), bytes);
        }
        cp_async_commit();
        __syncwarp(gmask);
        if (sub == 0) {
          win_lo[rl] = a0;
          win_n[rl] = static_cast<int32_t>(n);
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  stamp(dbg && threadIdx.x == 0, 63);
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem);
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(f);
  }
  return fn;
}

bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t kbytes, int box_rows) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(kbytes), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(kbytes)};
  cuuint32_t box[2] = {128, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool sddmm_tc_supported(const SddmmParams& p) {
  return p.LB == 8 && p.RB == 8 && (p.V == 4 || p.V == 8) && (p.K == 128 || p.K == 256) && p.batch == 1 &&
         p.out != nullptr && (reinterpret_cast<uintptr_t>(p.col_indices) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(p.a_words) & 15) == 0 && (reinterpret_cast<uintptr_t>(p.b_words) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(p.out) & 15) == 0 && p.M > 0 && p.N > 0 && p.N < (1ll << 31) &&
         p.M < (1ll << 31) && encode_fn() != nullptr;
}

cudaError_t launch_sddmm_tc(const SddmmParams& p, cudaStream_t stream) {
  CUtensorMap ta, tb;
  if (!make_map(&ta, p.a_words, p.M, p.K, kPanel) || !make_map(&tb, p.b_words, p.N, p.K, kCols))
    return cudaErrorInvalidValue;
  SddmmTcParams q{};
  q.M = p.M;
  q.N = p.N;
  q.K = p.K;
  q.V = p.V;
  q.vrows = p.vrows;
  q.n_blocks = p.n_blocks;
  q.row_offsets = p.row_offsets;
  q.col_indices = p.col_indices;
  q.out = p.out;
  q.alpha = p.alpha;
  q.alpha_host = p.alpha_host;
  q.out_f16 = p.out_f16;
  q.n_panels = static_cast<int>((p.M + kPanel - 1) / kPanel);
  q.n_ctiles = static_cast<int>((p.N + kCols - 1) / kCols);
  q.tiles = static_cast<int64_t>(q.n_panels) * q.n_ctiles;
  q.debug = getenv("MCUBE_DEBUG_TIMELINE") != nullptr;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = static_cast<int>(q.tiles < sms ? q.tiles : sms);
  auto kern = p.V == 8 ? sddmm_tc_kernel<8> : sddmm_tc_kernel<4>;
  const int smem = p.V == 8 ? Smem<8>::TOTAL : Smem<4>::TOTAL;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<grid, kThreads, smem, stream>>>(ta, tb, q);
  count_launch();
  return cudaGetLastError();
}

}  // namespace mcube

extern "C" int mc_debug_timeline(unsigned long long* host, int n) {
  if (n > 148 * 64) n = 148 * 64;
  return cudaMemcpyFromSymbol(host, mcube::g_timeline, n * sizeof(unsigned long long)) == cudaSuccess ? 0 : 6;
}
