// sddmm_tc.cu -- dense-tile SDDMM on the 5th-gen tensor cores (tcgen05 kind::i8, TMEM, TMA).
//
// For pattern densities above a few percent (C2 at 50..90% sparsity) the cheapest way
// to produce the sampled dot products (kernels.sddmm, kernels.py:367-435) on B200 is
// to compute whole 128 x 256 tiles of D^T = B^T A^T at int8 tensor-core rate and write
// out only the pattern blocks. Bit-exact: int8 x int8 products accumulate exactly in
// int32 TMEM for K <= 33025 (check_accumulation_bound, emulation.py:108-113).
//
// Tile: 128 pattern columns (UMMA M, TMEM lanes) x 32 vector rows = 32*V scalar rows
// of A (UMMA N, TMEM columns; 256 for V=8, 128 for V=4). A thread that owns TMEM lane c holds, after one
// 32-column tcgen05.ld, the V contiguous values of block (r, c) for 32/V vector rows,
// so every present block leaves the SM as one V*4-byte vector store.
//
// CTA (576 threads, 1 per SM, persistent over a contiguous tile range, panel-major):
//   warp 0      TMA producer: A panel (32*V rows x K, resident while the panel is
//               unchanged) and a 2-stage (V=8) / 3-stage (V=4) ring of B^T tiles;
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer; two accumulators
//               so the MMA of tile i+1 overlaps the drain of tile i;
//   warps 2..9  pattern builders, 4 vector rows each, 8 lanes per row: one cursor per
//               row into its CSR column list (located once per panel segment by an
//               interpolation probe + binary search), the list streamed through a
//               per-row shared-memory ring prefetched by position; per tile a 128-bit
//               column bitmap per vector row plus the CSR position of each 32-column
//               quarter, into a 4-deep map ring;
//   warps 10..17 consumers, two per TMEM lane quarter (each drains half of the
//               accumulator columns): bit test + popcount give the output block position.
#include <cuda_fp16.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace mcube {

// Debug timeline: build with -DMCUBE_TIMELINE to record globaltimer stamps per CTA
// (read back by mc_debug_timeline). Compiled out otherwise: even an untaken stamp costs
// every warp a constant-bank load of the buffer address in the prologue.
#ifdef MCUBE_TIMELINE
__device__ unsigned long long g_timeline[148 * 128];
__device__ __forceinline__ void stamp(bool on, int slot) {
  if (on && slot < 128 && blockIdx.x < 148) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_timeline[blockIdx.x * 128 + slot] = t;
  }
}
#define MC_STAMP(cond, slot) stamp(dbg && (cond), (slot))
#else
#define MC_STAMP(cond, slot) ((void)0)
#endif

namespace {


constexpr int kCols = 128;   // pattern columns per tile (UMMA M)
constexpr int kRing = 4;     // pattern-map ring (power of two: slot = i & 3, phase = i >> 2)
constexpr int kBuildWarps = 8;
constexpr int kConsWarps = 8;
constexpr int kFirstBuild = 2;
constexpr int kFirstCons = kFirstBuild + kBuildWarps;
constexpr int kThreads = 32 * (kFirstCons + kConsWarps);
constexpr int kRingStride = 516;  // uint32 per row ring (512 + 4 pad)
constexpr uint32_t kNone = 0xFFFFFFFFu;

// One 32-column quarter of one vector row of one tile: presence bits and the CSR
// position (= output block index) of the quarter's first present block.
struct __align__(16) QuarterMap {
  uint32_t bits;
  uint32_t pad;
  long long pos;
};

template <int V, int VR_>
struct Lay {
  static constexpr int VR = VR_;  // vector rows per tile (32, or 16 for finer load balance)
  static constexpr int PANEL = VR_ * V;  // scalar rows of A per tile (UMMA N, TMEM columns)
  static constexpr int STAGES = (V == 8 && VR_ == 32) ? 2 : 3;  // B^T tile ring depth (smem budget)
  static constexpr int A_BYTES = PANEL * 256;  // K <= 256
  static constexpr int B_STAGE = kCols * 256;
  static constexpr int MAP = VR * 4 * 16;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = OFF_A + A_BYTES;
  static constexpr int OFF_MAP = OFF_B + STAGES * B_STAGE;
  static constexpr int OFF_RING = OFF_MAP + kRing * MAP;  // uint32 [VR][kRingStride] column-index rings
  static constexpr int OFF_BAR = OFF_RING + VR * kRingStride * 4;
  static constexpr int N_BARS = 2 * STAGES + 2 + 4 + 2 * kRing;
  static constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
  static constexpr int TOTAL = OFF_TMEM + 16 + 1024;  // + alignment slack
};

// Predicated V*4-byte block store (no branch: one @p STG per block).
template <int V>
__device__ __forceinline__ void store_block_if(bool pred, int32_t* o, const uint32_t* v) {
  const uint32_t pr = pred ? 1u : 0u;
  if constexpr (V == 8) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %9, 0;\n\t"
        "@p st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n}" ::"l"(o),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(pr)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
        "@p st.global.v4.b32 [%0], {%1,%2,%3,%4};\n}" ::"l"(o),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(pr)
        : "memory");
  }
}

// First position in [lo, hi) whose column is >= c0 (columns strictly increasing):
// warp-parallel 32-ary search, about log32(hi - lo) round trips. All lanes return it.
__device__ int64_t warp_lower_bound(const uint32_t* __restrict__ cols, int64_t lo, int64_t hi, uint32_t c0,
                                    int lane) {
  int64_t a = lo, b = hi;
  while (b > a) {
    const int64_t n = b - a;
    const int64_t step = (n + 31) / 32;
    const int64_t p = a + lane * step;
    const bool in = p < b;
    const bool less = in && __ldg(cols + p) < c0;
    const unsigned m = __ballot_sync(0xffffffffu, less);
    const int cnt = __popc(m);
    if (step == 1) return a + cnt;
    const int np = static_cast<int>((n + step - 1) / step);
    const int64_t na = cnt > 0 ? a + (cnt - 1) * step + 1 : a;
    const int64_t nb = cnt < np ? a + cnt * step : b;
    a = na;
    b = nb;
  }
  return a;
}

// Tile coordinates advanced incrementally (a 64-bit division per tile costs a software
// routine on every role's critical path). Tiles are ordered item-major, then panel, then
// 128-column tile.
struct TileCursor {
  long long item, panel, ct, gpanel;
  int n_panels, n_ctiles;
  __device__ TileCursor(long long t, int np, int nc) : n_panels(np), n_ctiles(nc) {
    gpanel = t / nc;
    ct = t - gpanel * nc;
    item = gpanel / np;
    panel = gpanel - item * np;
  }
  __device__ __forceinline__ void next() {
    if (++ct == n_ctiles) {
      ct = 0;
      ++gpanel;
      if (++panel == n_panels) {
        panel = 0;
        ++item;
      }
    }
  }
};

template <int V, int VR_>
__global__ void __launch_bounds__(kThreads, 1)
sddmm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const SddmmTcParams p) {
  using L = Lay<V, VR_>;
  constexpr int kStages = L::STAGES;
  constexpr int VR = L::VR;
  constexpr int PANEL = L::PANEL;
  constexpr int kRowsPerBuilder = 32 / kBuildWarps;  // vector rows per builder warp
  constexpr int kLanesPerRow = 32 / kRowsPerBuilder;  // builder lanes per vector row
  constexpr int kBW = VR / kRowsPerBuilder;  // active builder warps (the rest idle when VR = 16)
  constexpr uint32_t kIdesc = tc::idesc_i8(128, PANEL);
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // align to 1024 B (SW128 atoms) with pointer arithmetic (keeps the shared window)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // K is staged in blocks of KBLK bytes: 128 (SWIZZLE_128B, K = 128/256) or 64 (SWIZZLE_64B, K = 64)
  const int KBLK = p.K >= 128 ? 128 : 64;
  const int KB = static_cast<int>(p.K / KBLK);
  QuarterMap* maps = reinterpret_cast<QuarterMap*>(smem + L::OFF_MAP);
  const uint32_t bar0 = sbase + L::OFF_BAR;
  auto full_bar = [&](int s) { return bar0 + 8 * s; };
  auto empty_bar = [&](int s) { return bar0 + 8 * (kStages + s); };
  const uint32_t a_full = bar0 + 8 * (2 * kStages), a_empty = a_full + 8;
  auto tfull_bar = [&](int a) { return bar0 + 8 * (2 * kStages + 2 + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8 * (2 * kStages + 4 + a); };
  auto pfull_bar = [&](int s) { return bar0 + 8 * (2 * kStages + 6 + s); };
  auto pempty_bar = [&](int s) { return bar0 + 8 * (2 * kStages + 6 + kRing + s); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

  const bool dbg = p.debug != 0;
  (void)dbg;
  MC_STAMP(threadIdx.x == 0, 0);
  const int64_t t0 = (p.tiles * blockIdx.x) / gridDim.x;
  const int64_t t1 = (p.tiles * (blockIdx.x + 1)) / gridDim.x;
  const int64_t tiles_per_item = static_cast<int64_t>(p.n_panels) * p.n_ctiles;

  // ---- pattern-builder state; their first loads are issued before the setup barrier ----
  const int bw = warp - kFirstBuild;
  const int jr = lane / kLanesPerRow, sub = lane % kLanesPerRow;
  const int rl = kRowsPerBuilder * bw + jr;  // builder lane's vector row within the tile
  uint32_t* rrow = reinterpret_cast<uint32_t*>(smem + L::OFF_RING) + (rl & (VR - 1)) * kRingStride;
  const uint32_t rrow_s = smem_u32(rrow);
  // lane (j, s) issues its quarter of chunks [c_from, c_to) of row j; chunk c of a row
  // starting at `lo` covers absolute positions [((lo >> 6) + c) * 64, +64)
  auto fetch_chunks = [&](long long lo_, int c_from, int c_to) {
    for (int c = c_from; c < c_to; ++c) {
      const long long base = ((lo_ >> 6) + c) * 64;
#pragma unroll
      for (int u = 0; u < 16 / kLanesPerRow; ++u) {
        const long long pos0 = base + (sub * (16 / kLanesPerRow) + u) * 4;
        const long long avail = p.n_blocks - pos0;
        const uint32_t bytes = avail >= 4 ? 16u : (avail > 0 ? static_cast<uint32_t>(avail) * 4u : 0u);
        cp_async16(rrow_s + static_cast<uint32_t>(pos0 & 511) * 4, p.col_indices + (bytes ? pos0 : 0), bytes);
      }
    }
  };
  // chunks kept in flight past the cursor: two tiles' worth of entries at the row's density
  auto prefetch_depth = [&](int len_) {
    const int per_tile = static_cast<int>((static_cast<long long>(len_) * kCols + p.N - 1) / p.N);
    const int d = (2 * per_tile + 48 + 63) / 64 + 1;
    return d < 2 ? 2 : (d > 7 ? 7 : d);
  };
  // probe window [chunk x, chunk y) around the interpolated position of c0 (<= 8 chunks)
  auto probe_window = [&](int len_, uint32_t c0_, int lo63_) {
    int start = 0, end = 0;
    const int per_tile = static_cast<int>((static_cast<long long>(len_) * kCols + p.N - 1) / p.N);
    if (c0_ > 0) {
      // interpolated position of c0; for columns sampled uniformly its spread is binomial
      // (sigma = sqrt(len q (1 - q))), so +-(16 + 3 sigma) brackets it; rows that are not
      // bracketed fall back to a binary search in global memory (correct, only slower)
      const double q = static_cast<double>(c0_) / static_cast<double>(p.N);
      const int g = static_cast<int>(q * len_);
      const int margin = 16 + static_cast<int>(3.0 * sqrt(static_cast<double>(len_) * q * (1.0 - q)));
      start = g - margin > 0 ? g - margin : 0;
      end = g + margin;
    }
    end += 2 * per_tile + 48;
    if (end > len_) end = len_;
    const int cs = (lo63_ + start) >> 6;
    int ce = ((lo63_ + (end > 0 ? end - 1 : 0)) >> 6) + 1;
    if (ce > cs + 8) ce = cs + 8;
    if (ce < cs + 1) ce = cs + 1;
    return make_int2(cs, ce);
  };
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(full_bar(s), 1);
      tc::mbar_init(empty_bar(s), 1);
    }
    tc::mbar_init(a_full, 1);
    tc::mbar_init(a_empty, 1);
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(tfull_bar(a), 1);
      tc::mbar_init(tempty_bar(a), kConsWarps);
    }
    for (int s = 0; s < kRing; ++s) {
      tc::mbar_init(pfull_bar(s), kBW);  // one arrival per active builder warp
      tc::mbar_init(pempty_bar(s), kConsWarps);
    }
    tc::fence_barrier_init();
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
    MC_STAMP(true, 100);
  }
  if (warp == 1) {
    tc::tmem_alloc<512>(smem_u32(tmem_holder));
    MC_STAMP(lane == 0, 101);
  }
  // everything above touches only this CTA's resources and the kernel parameters; inputs
  // written by a previous kernel are read only after pdl_wait
  if (threadIdx.x == 0) pdl_launch_dependents();
  // Warm L2 with this CTA's first operand boxes and pattern rows while the previous kernel
  // drains: L2 is the coherence point, so a prefetch issued before pdl_wait cannot make a
  // later read observe stale data; it only hides the first HBM round trips.
  if (t0 < t1) {
    const TileCursor c(t0, p.n_panels, p.n_ctiles);
    if (warp == 0 && lane == 0) {
      for (int kb = 0; kb < KB; ++kb) {
        tc::tma_prefetch_2d(&tmA, kb * KBLK, static_cast<int>(c.item * p.M + c.panel * PANEL));
        tc::tma_prefetch_2d(&tmB, kb * KBLK, static_cast<int>(c.item * p.N + c.ct * kCols));
      }
    } else if (warp >= kFirstBuild && warp < kFirstBuild + kBW && (lane & (kLanesPerRow - 1)) == 0) {
      const long long r = c.panel * VR + rl;
      if (r < p.vrows) {
        tc::prefetch_l2(p.row_offsets + r);
        const long long g = (r * p.n_blocks) / p.vrows +
                            static_cast<long long>((static_cast<double>(c.ct * kCols) / p.N) *
                                                   (static_cast<double>(p.n_blocks) / p.vrows));
        tc::prefetch_l2(p.col_indices + (g < p.n_blocks ? g : 0));
      }
    }
  }
  pdl_wait();
  // the first tile's A panel and B^T tile go out before the setup barrier: the barriers were
  // initialised by this thread, and the loads overlap the TMEM allocation, the barrier and
  // the pattern builders' first window
  if (warp == 0 && lane == 0 && t0 < t1) {
    const TileCursor c(t0, p.n_panels, p.n_ctiles);
    tc::mbar_arrive_expect_tx(a_full, KB * PANEL * KBLK);
    for (int kb = 0; kb < KB; ++kb)
      tc::tma_load_2d(sbase + L::OFF_A + kb * PANEL * KBLK, &tmA, a_full, kb * KBLK,
                      static_cast<int>(c.item * p.M + c.panel * PANEL));
    tc::mbar_arrive_expect_tx(full_bar(0), KB * kCols * KBLK);
    for (int kb = 0; kb < KB; ++kb)
      tc::tma_load_2d(sbase + L::OFF_B + kb * kCols * KBLK, &tmB, full_bar(0), kb * KBLK,
                      static_cast<int>(c.item * p.N + c.ct * kCols));
  }
  MC_STAMP(threadIdx.x == 0, 102);
  long long lo = 0, b_lo = 0, b_hi = 0, spec_lo = -1, spec_hi = -1;
  int len = 0, cur = 0, mtop = 0, landed = 0, lo511 = 0, lo63 = 0, depth = 2, c_first = 0;
  int mtop_last = 0;  // chunk bound of all cp.async groups but the most recent one
  long long b_r = -1;
  uint32_t b_c00 = 0;
  if (warp >= kFirstBuild && warp < kFirstBuild + kBW && t0 < t1) {
    const int64_t rem0 = t0 % tiles_per_item;
    b_r = (rem0 / p.n_ctiles) * VR + rl;
    b_c00 = static_cast<uint32_t>((rem0 % p.n_ctiles) * kCols);
    if (b_r < p.vrows) {  // the first panel's row offsets: in flight across the setup barrier
      b_lo = p.row_offsets[b_r];
      b_hi = p.row_offsets[b_r + 1];
      // speculate rows of equal length (exact for the reference generator's patterns): the
      // first probe window goes out now, overlapping the offsets round trip and the setup
      // barrier, and is discarded if the offsets disagree
      spec_lo = (b_r * p.n_blocks) / p.vrows;
      spec_hi = ((b_r + 1) * p.n_blocks) / p.vrows;
      const int slen = static_cast<int>(spec_hi - spec_lo);
      const int2 w = probe_window(slen, b_c00, static_cast<int>(spec_lo & 63));
      c_first = w.x;
      if (slen > 0) fetch_chunks(spec_lo, w.x, w.y);
      mtop = w.y;
    }
    cp_async_commit();
  }
  MC_STAMP(threadIdx.x == 0, 103);
  MC_STAMP(threadIdx.x == 32 * kFirstBuild, 104);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  MC_STAMP(threadIdx.x == 0, 1);

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int64_t cur_panel = -1;
      int n_a = 0;
      TileCursor tc_(t0, p.n_panels, p.n_ctiles);
      for (int64_t t = t0; t < t1; ++t, tc_.next()) {
        const int i = static_cast<int>(t - t0);
        const long long item = tc_.item, panel = tc_.panel, ct = tc_.ct, gpanel = tc_.gpanel;
        if (gpanel != cur_panel) {
          if (i > 0) {  // tile 0's loads were issued before the setup barrier
            if (n_a > 0) tc::mbar_wait(a_empty, (n_a - 1) & 1);
            tc::mbar_arrive_expect_tx(a_full, KB * PANEL * KBLK);
            for (int kb = 0; kb < KB; ++kb)
              tc::tma_load_2d(sbase + L::OFF_A + kb * PANEL * KBLK, &tmA, a_full, kb * KBLK,
                              static_cast<int>(item * p.M + panel * PANEL));
          }
          ++n_a;
          cur_panel = gpanel;
        }
        if (i == 0) continue;
        const int s = static_cast<int>(i % kStages);
        const uint32_t u = static_cast<uint32_t>(i / kStages);
        tc::mbar_wait(empty_bar(s), (u & 1) ^ 1);
        tc::mbar_arrive_expect_tx(full_bar(s), KB * kCols * KBLK);
        for (int kb = 0; kb < KB; ++kb)
          tc::tma_load_2d(sbase + L::OFF_B + s * L::B_STAGE + kb * kCols * KBLK, &tmB, full_bar(s), kb * KBLK,
                          static_cast<int>(item * p.N + ct * kCols));
        MC_STAMP(i < 6, 2 + static_cast<int>(i));
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      int64_t cur_panel = -1;
      int n_a = 0;
      TileCursor tc_(t0, p.n_panels, p.n_ctiles);
      for (int64_t t = t0; t < t1; ++t, tc_.next()) {
        const int i = static_cast<int>(t - t0);
        const long long gpanel = tc_.gpanel;
        if (gpanel != cur_panel) {
          tc::mbar_wait(a_full, n_a & 1);
          ++n_a;
          cur_panel = gpanel;
        }
        const int s = static_cast<int>(i % kStages);
        const uint32_t u = static_cast<uint32_t>(i / kStages);
        const int acc = static_cast<int>(i & 1);
        const uint32_t u2 = static_cast<uint32_t>(i >> 1);
        tc::mbar_wait(tempty_bar(acc), (u2 & 1) ^ 1);
        tc::mbar_wait(full_bar(s), u & 1);
        tc::tc_fence_after();
        MC_STAMP(i < 6, 10 + static_cast<int>(i));
        const uint32_t d = tmem + acc * PANEL;
        const uint32_t bs = sbase + L::OFF_B + s * L::B_STAGE;
        const uint32_t as = sbase + L::OFF_A;
        const int kpb = KBLK / 32;  // K=32 MMA steps per staged block
        for (int ks = 0; ks < KB * kpb; ++ks) {
          const int kb = ks / kpb, off = (ks % kpb) * 32;
          const uint32_t aaddr = bs + kb * kCols * KBLK + off;  // B^T tile: M = 128
          const uint32_t baddr = as + kb * PANEL * KBLK + off;  // A panel:  N = PANEL
          const uint64_t adesc = KBLK == 128 ? tc::desc_k_sw128(aaddr) : tc::desc_k_sw64(aaddr);
          const uint64_t bdesc = KBLK == 128 ? tc::desc_k_sw128(baddr) : tc::desc_k_sw64(baddr);
          tc::mma_i8(d, adesc, bdesc, kIdesc, ks > 0 ? 1u : 0u);
        }
        tc::mma_commit(empty_bar(s));
        tc::mma_commit(tfull_bar(acc));
        MC_STAMP(i < 6, 16 + static_cast<int>(i));
        if (t + 1 == t1 || tc_.ct + 1 == p.n_ctiles) tc::mma_commit(a_empty);  // panel's last tile
      }
    }
  } else {
  if (warp < kFirstBuild + kBW) {
    // ---------------- pattern builders (independent warps) ----------------
    // Builder warp bw owns vector rows 4*bw .. 4*bw+3 of the tile; lane = (row j, sub s),
    // eight lanes per row. Each row streams its CSR column list through a 512-entry ring
    // in shared memory (64-entry chunks, absolute position x in slot x & 511), fetched by
    // POSITION with cp.async `depth` chunks ahead of the cursor (depth follows the row's
    // density). Reads are bounded by the chunks known to have landed; a tile that runs
    // past them waits (cp.async.wait_all). Positions are relative to the row start.
    // Per tile, lane (j, s) tests candidates s, s+8, s+16, ... of row j until the row
    // leaves the tile (columns strictly increasing), the eight lanes OR their bitmaps with
    // three shuffles, and lane (j, s < 4) writes the QuarterMap of quarter s. No cross-warp
    // synchronisation: each warp arrives on the tile's pfull barrier.
    // (the speculative first window was issued before the setup barrier)
    int64_t cur_panel = -1;
    TileCursor tc_(t0, p.n_panels, p.n_ctiles);
    for (int64_t t = t0; t < t1; ++t, tc_.next()) {
      const int i = static_cast<int>(t - t0);
      const int slot = i & (kRing - 1);
      const long long panel = tc_.panel, ct = tc_.ct, gpanel = tc_.gpanel;
      const uint32_t c0 = static_cast<uint32_t>(ct * kCols);
      if (gpanel != cur_panel) {
        // ---- segment start: locate the row's cursor at column c0 ----
        long long hi;
        bool spec_ok;
        if (t == t0) {  // offsets + speculative window were issued before the setup barrier
          lo = b_lo;
          hi = b_hi;
          spec_ok = (lo == spec_lo) && (hi == spec_hi);
        } else {
          const long long r = panel * VR + rl;
          lo = hi = 0;
          if (r < p.vrows) {
            lo = p.row_offsets[r];
            hi = p.row_offsets[r + 1];
          }
          spec_ok = false;
        }
        len = static_cast<int>(hi - lo);
        lo63 = static_cast<int>(lo & 63);
        lo511 = static_cast<int>(lo & 511);
        depth = prefetch_depth(len);
        cp_async_wait<0>();  // nothing of an older window may land after the new copies
        if (!spec_ok) {
          const int2 w = probe_window(len, c0, lo63);
          c_first = w.x;
          if (len > 0) fetch_chunks(lo, w.x, w.y);
          mtop = w.y;
          cp_async_commit();
          cp_async_wait<0>();
        }
        __syncwarp();
        landed = mtop_last = mtop;
        cur = 0;
        if (c0 > 0 && len > 0) {
          // lower bound of c0 inside the landed window [ws, we) (binary search in smem)
          const int ws = (c_first * 64 - lo63 > 0) ? c_first * 64 - lo63 : 0;
          const int we = (landed * 64 - lo63 < len) ? landed * 64 - lo63 : len;
          int a = ws, b = we;
          while (a < b) {
            const int mid = (a + b) >> 1;
            if (rrow[(lo511 + mid) & 511] < c0) a = mid + 1;
            else b = mid;
          }
          cur = a;
          if ((cur == ws && ws > 0) || (cur == we && we < len)) {
            // the probe did not bracket c0 (irregular row): binary search in global memory;
            // the ring holds nothing useful for the new cursor
            long long ga = lo, gb = hi;
            while (ga < gb) {
              const long long mid = (ga + gb) >> 1;
              if (__ldg(p.col_indices + mid) < c0) ga = mid + 1;
              else gb = mid;
            }
            cur = static_cast<int>(ga - lo);
            mtop = landed = mtop_last = (lo63 + cur) >> 6;
          }
        }
        cur_panel = gpanel;
        MC_STAMP(lane == 0 && bw == 0, 40);
      }
      else {
        // every cp.async group but the one committed after the previous tile is complete
        cp_async_wait<1>();
        __syncwarp();
        landed = mtop_last;
      }
      MC_STAMP(lane == 0 && bw == 0 && i < 5, 64 + 5 * static_cast<int>(i));
      // ---- this tile's bitmap of row j (lanes of the row split the candidates) ----
      const int lim = (len - cur < kCols) ? len - cur : kCols;  // candidates in the tile window
      uint32_t w0 = 0u, w1 = 0u, w2 = 0u, w3 = 0u;
      bool bad = false;
      {
        // the whole candidate window [cur, cur + lim) must have landed: one check per tile
        // (the prefetch depth keeps two tiles of entries in flight, so this rarely waits)
        const int landed_rel = landed * 64 - lo63;
        const bool need = lim > 0 && cur + lim > landed_rel && landed_rel < len;
        if (__any_sync(0xffffffffu, need)) {
          if (need) {
            const int c_need = ((lo63 + cur + lim - 1) >> 6) + 1;
            if (c_need > mtop) {
              const int c_cap = ((lo63 + cur) >> 6) + 8;  // never overwrite the cursor's chunk
              const int c_to = (c_need + depth - 1 < c_cap) ? c_need + depth - 1 : c_cap;
              fetch_chunks(lo, mtop, c_to);
              mtop = c_to;
            }
          }
          cp_async_commit();
          cp_async_wait<0>();
          __syncwarp();
          landed = mtop_last = mtop;
        }
      }
      MC_STAMP(lane == 0 && bw == 0 && i < 5, 90 + static_cast<int>(i));
      // candidates s, s + L, s + 2L, s + 3L of the step (L = lanes per row) per lane; a
      // candidate outside the tile (off = c - c0 >= 128, kNone past the window) selects no
      // bitmap word, so the routing is four predicated ORs (the loop is ALU-pipe bound). A
      // step continues while some lane's last candidate was inside the tile (columns
      // strictly increasing: then all its earlier ones were too) -- one vote per step.
      // Out-of-range columns (>= N) can only fall inside the last column tile.
      const bool last_ct = c0 + static_cast<uint32_t>(kCols) > static_cast<uint32_t>(p.N);
      for (int k0 = 0; k0 < kCols; k0 += 4 * kLanesPerRow) {
        uint32_t c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + sub + kLanesPerRow * u;
          c[u] = k < lim ? rrow[(lo511 + cur + k) & 511] : kNone;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t off = c[u] - c0;
          asm("{\n\t.reg .pred q;\n\t.reg .b32 t, ws;\n\t"
              "shf.l.wrap.b32 t, 0, 1, %4;\n\t"  // 1 << (off & 31)
              "shr.u32 ws, %4, 5;\n\t"
              "setp.eq.u32 q, ws, 0;\n\t@q or.b32 %0, %0, t;\n\t"
              "setp.eq.u32 q, ws, 1;\n\t@q or.b32 %1, %1, t;\n\t"
              "setp.eq.u32 q, ws, 2;\n\t@q or.b32 %2, %2, t;\n\t"
              "setp.eq.u32 q, ws, 3;\n\t@q or.b32 %3, %3, t;\n\t}"
              : "+r"(w0), "+r"(w1), "+r"(w2), "+r"(w3)
              : "r"(off));
        }
        if (last_ct) {
#pragma unroll
          for (int u = 0; u < 4; ++u) bad |= (c[u] - c0 < static_cast<uint32_t>(kCols)) && c[u] >= static_cast<uint32_t>(p.N);
        }
        if (!__any_sync(0xffffffffu, c[3] - c0 < static_cast<uint32_t>(kCols))) break;
      }
      MC_STAMP(lane == 0 && bw == 0 && i < 5, 65 + 5 * static_cast<int>(i));
      if (bad) flag_status(p.status, MC_STATUS_BAD_INDEX);
#pragma unroll
      for (int o = 1; o < kLanesPerRow; o <<= 1) {
        w0 |= __shfl_xor_sync(0xffffffffu, w0, o);
        w1 |= __shfl_xor_sync(0xffffffffu, w1, o);
        w2 |= __shfl_xor_sync(0xffffffffu, w2, o);
        w3 |= __shfl_xor_sync(0xffffffffu, w3, o);
      }
      const int p0 = __popc(w0), p1 = __popc(w1), p2 = __popc(w2), p3 = __popc(w3);
      const int pre = (sub > 0 ? p0 : 0) + (sub > 1 ? p1 : 0) + (sub > 2 ? p2 : 0);
      MC_STAMP(lane == 0 && bw == 0 && i < 5, 66 + 5 * static_cast<int>(i));
      tc::mbar_wait(pempty_bar(slot), ((i >> 2) & 1) ^ 1);
      MC_STAMP(lane == 0 && bw == 0 && i < 5, 67 + 5 * static_cast<int>(i));
      if (sub < 4) {
        QuarterMap qm;
        qm.bits = sub == 0 ? w0 : sub == 1 ? w1 : sub == 2 ? w2 : w3;
        qm.pad = 0;
        qm.pos = lo + cur + pre;
        maps[slot * (VR * 4) + rl * 4 + sub] = qm;
      }
      cur += p0 + p1 + p2 + p3;
      // keep `depth` chunks in flight past the cursor
      const int want = ((lo63 + cur) >> 6) + depth;
      mtop_last = mtop;  // bound of the groups committed so far
      if (want > mtop && len > 0) {
        fetch_chunks(lo, mtop, want);
        mtop = want;
      }
      cp_async_commit();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(pfull_bar(slot));
      MC_STAMP(lane == 0 && bw == 0 && i < 6, 22 + 3 * static_cast<int>(i));
    }
    cp_async_wait<0>();
  }
  if (warp >= kFirstCons) {
    // ---------------- consumers: TMEM -> registers -> V*4-byte block stores ----------------
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int half = (warp - kFirstCons) >> 2;
    const uint32_t ltmask = (1u << lane) - 1u;
    constexpr int rpc = 32 / V;  // vector rows per 32-column chunk
    constexpr int kChunks = PANEL / 64;  // 32-column TMEM chunks per consumer warp
    TileCursor tc_(t0, p.n_panels, p.n_ctiles);
    for (int64_t t = t0; t < t1; ++t, tc_.next()) {
      const int i = static_cast<int>(t - t0);
      const int slot = i & (kRing - 1);
      const int acc = i & 1;
      const long long item = tc_.item;
      const QuarterMap* m = maps + slot * (VR * 4);
      tc::mbar_wait(pfull_bar(slot), (i >> 2) & 1);
      tc::mbar_wait(tfull_bar(acc), (i >> 1) & 1);
      tc::tc_fence_after();
      MC_STAMP(warp == kFirstCons && lane == 0 && i < 6, 23 + 3 * static_cast<int>(i));
      const uint32_t tl = tmem + (static_cast<uint32_t>(32 * q) << 16) + acc * PANEL + (PANEL / 2) * half;
      uint32_t va[32], vb[32];
      tc::tmem_ld32_issue(tl, va);
      tc::tmem_wait_ld();
      MC_STAMP(warp == kFirstCons && lane == 0 && i < 3, 110 + static_cast<int>(i));
      if (p.out_f16 == nullptr) {
        int32_t* out = p.out + item * p.out_stride;
#pragma unroll
        for (int kk = 0; kk < kChunks; ++kk) {
          uint32_t(&cur)[32] = (kk & 1) ? vb : va;
          uint32_t(&nxt)[32] = (kk & 1) ? va : vb;
          if (kk + 1 < kChunks) tc::tmem_ld32_issue(tl + 32 * (kk + 1), nxt);
          QuarterMap qm[rpc];
#pragma unroll
          for (int w = 0; w < rpc; ++w) qm[w] = m[((kChunks * half + kk) * rpc + w) * 4 + q];
#pragma unroll
          for (int w = 0; w < rpc; ++w) {
            const bool present = (qm[w].bits >> lane) & 1u;
            const long long pos = qm[w].pos + __popc(qm[w].bits & ltmask);
#ifdef MCUBE_NOSTORE
            if (present && cur[V * w] == 0x7fffffffu) store_block_if<V>(present, out + pos * V, &cur[V * w]);
#else
            store_block_if<V>(present, out + pos * V, &cur[V * w]);
#endif
          }
          if (kk + 1 < kChunks) tc::tmem_wait_ld();
        }
        MC_STAMP(warp == kFirstCons && lane == 0 && i < 3, 113 + static_cast<int>(i));
      } else {
        // fused dequant epilogue (attention.py:147-154): fp16(acc * alpha) per block as one
        // V*2-byte store (+ the int32 accumulators when requested), rounded exactly as the
        // reference's float64 product (f16_dequant).
        int32_t* out = p.out ? p.out + item * p.out_stride : nullptr;
        uint16_t* out16 = p.out_f16 + item * p.f16_stride;
        const double alpha = p.alpha ? p.alpha[item] : p.alpha_host;
        const float alpha_f = static_cast<float>(alpha);
#pragma unroll 1
        for (int kk = 0; kk < kChunks; ++kk) {
          if (kk > 0) tc::tmem_ld32(tl + 32 * kk, va);
#pragma unroll
          for (int w = 0; w < rpc; ++w) {
            const QuarterMap qm = m[((kChunks * half + kk) * rpc + w) * 4 + q];
            const bool present = (qm.bits >> lane) & 1u;
            const long long pos = qm.pos + __popc(qm.bits & ltmask);
            if (out) store_block_if<V>(present, out + pos * V, &va[V * w]);
            uint32_t h2[V / 2];
#pragma unroll
            for (int x = 0; x < V / 2; ++x) {
              const int32_t a0 = static_cast<int32_t>(va[V * w + 2 * x]), a1 = static_cast<int32_t>(va[V * w + 2 * x + 1]);
              const uint16_t l = f16_dequant(a0, alpha, alpha_f), h = f16_dequant(a1, alpha, alpha_f);
              h2[x] = static_cast<uint32_t>(l) | (static_cast<uint32_t>(h) << 16);
            }
            if (present) {
              if constexpr (V == 8) *reinterpret_cast<uint4*>(out16 + pos * V) = make_uint4(h2[0], h2[1], h2[2], h2[3]);
              else *reinterpret_cast<uint2*>(out16 + pos * V) = make_uint2(h2[0], h2[1]);
            }
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        tc::mbar_arrive(tempty_bar(acc));
        tc::mbar_arrive(pempty_bar(slot));
      }
      MC_STAMP(warp == kFirstCons && lane == 0 && i < 6, 24 + 3 * static_cast<int>(i));
      MC_STAMP(warp == kFirstCons + 7 && lane == 0 && i < 3, 116 + static_cast<int>(i));
    }
  }
  }
  tc::tc_fence_before();
  __syncthreads();
  MC_STAMP(threadIdx.x == 0, 63);
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
  const int kblk = kbytes >= 128 ? 128 : 64;  // 128-byte (SW128) or 64-byte (SW64) K blocks
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(kbytes), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(kbytes)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kblk), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, kblk == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool sddmm_tc_supported(const SddmmParams& p) {
  const bool dense_items = p.batch == 1 || (p.a_stride * 4 == p.M * p.K && p.b_stride * 4 == p.N * p.K);
  const uintptr_t out_align = static_cast<uintptr_t>(4 * p.V);
  return p.LB == 8 && p.RB == 8 && (p.V == 4 || p.V == 8) && (p.K == 64 || p.K == 128 || p.K == 256) &&
         (p.out_f16 == nullptr || (reinterpret_cast<uintptr_t>(p.out_f16) % (2 * p.V)) == 0) &&
         p.batch >= 1 && dense_items && (p.out != nullptr || p.out_f16 != nullptr) &&
         (p.out == nullptr || ((reinterpret_cast<uintptr_t>(p.out) % out_align) == 0 && (p.out_stride % p.V) == 0)) &&
         (reinterpret_cast<uintptr_t>(p.a_words) & 15) == 0 && (reinterpret_cast<uintptr_t>(p.b_words) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(p.col_indices) & 15) == 0 && p.M > 0 && p.N > 0 && static_cast<int64_t>(p.batch) * p.N < (1ll << 31) &&
         static_cast<int64_t>(p.batch) * p.M < (1ll << 31) && p.N < (1ll << 32) - 256 && encode_fn() != nullptr;
}

cudaError_t launch_sddmm_tc(const SddmmParams& p, cudaStream_t stream) {
  // tile height: 32 vector rows; 16 (MCUBE_SDDMM_VR=16) halves the per-tile epilogue for a
  // finer last wave but measured slower at every C2 density (per-tile costs dominate)
  int vr = 32;
  if (const char* e = getenv("MCUBE_SDDMM_VR")) vr = atoi(e) == 16 ? 16 : 32;
  CUtensorMap ta, tb;
  if (!make_map(&ta, p.a_words, p.batch * p.M, p.K, vr * p.V) || !make_map(&tb, p.b_words, p.batch * p.N, p.K, kCols))
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
  q.out_stride = p.out_stride;
  q.alpha = p.alpha;
  q.alpha_host = p.alpha_host;
  q.out_f16 = p.out_f16;
  q.f16_stride = p.f16_stride;
  q.status = p.status;
  q.n_panels = static_cast<int>((p.M + vr * p.V - 1) / (vr * p.V));
  q.n_ctiles = static_cast<int>((p.N + kCols - 1) / kCols);
  q.tiles = static_cast<int64_t>(p.batch) * q.n_panels * q.n_ctiles;
  q.debug = getenv("MCUBE_DEBUG_TIMELINE") != nullptr;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = static_cast<int>(q.tiles < sms ? q.tiles : sms);
  if (grid == 0) return cudaSuccess;
  decltype(&sddmm_tc_kernel<8, 32>) kern;
  int smem;
  if (p.V == 8) {
    kern = vr == 16 ? sddmm_tc_kernel<8, 16> : sddmm_tc_kernel<8, 32>;
    smem = vr == 16 ? Lay<8, 16>::TOTAL : Lay<8, 32>::TOTAL;
  } else {
    kern = vr == 16 ? sddmm_tc_kernel<4, 16> : sddmm_tc_kernel<4, 32>;
    smem = vr == 16 ? Lay<4, 16>::TOTAL : Lay<4, 32>::TOTAL;
  }
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const cudaError_t e = launch_pdl(kern, dim3(grid), dim3(kThreads), smem, stream, ta, tb, q);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace mcube

extern "C" int mc_debug_timeline(unsigned long long* host, int n) {
#ifdef MCUBE_TIMELINE
  if (n > 148 * 128) n = 148 * 128;
  return cudaMemcpyFromSymbol(host, mcube::g_timeline, n * sizeof(unsigned long long)) == cudaSuccess ? 0 : 6;
#else
  (void)host;
  (void)n;
  return 1;  // built without -DMCUBE_TIMELINE
#endif
}
