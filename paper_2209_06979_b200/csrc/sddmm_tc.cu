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
// CTA (448 threads, 1 per SM, persistent over a contiguous tile range, panel-major):
//   warp 0      TMA producer: A panel (32*V rows x K, resident while the panel is
//               unchanged) and a 2-stage (V=8) / 3-stage (V=4) ring of B^T tiles;
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer; two accumulators
//               so the MMA of tile i+1 overlaps the drain of tile i;
//   warps 2..5  pattern builders, 8 vector rows each, 4 lanes per row: one cursor per
//               row into its CSR column list (located once per panel segment by an
//               interpolation probe + binary search), the list streamed through a
//               per-row shared-memory ring prefetched by position; per tile a 128-bit
//               column bitmap per vector row plus the CSR position of each 32-column
//               quarter, into a 4-deep map ring;
//   warps 6..13 consumers, two per TMEM lane quarter (each drains half of the
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

constexpr int kVRows = 32;    // vector rows per tile: 32*V scalar rows of A (UMMA N)
constexpr int kCols = 128;   // pattern columns per tile (UMMA M)
constexpr int kRing = 4;     // pattern-map ring
constexpr int kBuildWarps = 4;
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

template <int V>
struct Lay {
  static constexpr int VR = kVRows;
  static constexpr int PANEL = kVRows * V;  // scalar rows of A per tile (UMMA N, TMEM columns)
  static constexpr int STAGES = V == 8 ? 2 : 3;  // B^T tile ring depth (smem budget)
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

template <int V>
__global__ void __launch_bounds__(kThreads, 1)
sddmm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const SddmmTcParams p) {
  using L = Lay<V>;
  constexpr int kStages = L::STAGES;
  constexpr int VR = L::VR;
  constexpr int PANEL = L::PANEL;
  constexpr uint32_t kIdesc = tc::idesc_i8(128, PANEL);
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // align to 1024 B (SW128 atoms) with pointer arithmetic (keeps the shared window)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = static_cast<int>(p.K / 128);
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
      tc::mbar_init(pfull_bar(s), kBuildWarps);  // one arrival per builder warp
      tc::mbar_init(pempty_bar(s), kConsWarps);
    }
    tc::fence_barrier_init();
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
  }
  if (warp == 1) tc::tmem_alloc<512>(smem_u32(tmem_holder));
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
      for (int64_t t = t0; t < t1; ++t) {
        const int64_t i = t - t0;
        const int64_t item = t / tiles_per_item, rem = t % tiles_per_item;
        const int64_t panel = rem / p.n_ctiles, ct = rem % p.n_ctiles;
        const int64_t gpanel = t / p.n_ctiles;
        if (gpanel != cur_panel) {
          if (n_a > 0) tc::mbar_wait(a_empty, (n_a - 1) & 1);
          tc::mbar_arrive_expect_tx(a_full, KB * PANEL * 128);
          for (int kb = 0; kb < KB; ++kb)
            tc::tma_load_2d(sbase + L::OFF_A + kb * PANEL * 128, &tmA, a_full, kb * 128,
                            static_cast<int>(item * p.M + panel * PANEL));
          ++n_a;
          cur_panel = gpanel;
        }
        const int s = static_cast<int>(i % kStages);
        const uint32_t u = static_cast<uint32_t>(i / kStages);
        tc::mbar_wait(empty_bar(s), (u & 1) ^ 1);
        tc::mbar_arrive_expect_tx(full_bar(s), KB * kCols * 128);
        for (int kb = 0; kb < KB; ++kb)
          tc::tma_load_2d(sbase + L::OFF_B + s * L::B_STAGE + kb * kCols * 128, &tmB, full_bar(s), kb * 128,
                          static_cast<int>(item * p.N + ct * kCols));
        MC_STAMP(i < 6, 2 + static_cast<int>(i));
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      int64_t cur_panel = -1;
      int n_a = 0;
      for (int64_t t = t0; t < t1; ++t) {
        const int64_t i = t - t0;
        const int64_t gpanel = t / p.n_ctiles;
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
        for (int ks = 0; ks < KB * 4; ++ks) {
          const int kb = ks >> 2, off = (ks & 3) * 32;
          const uint64_t adesc = tc::desc_k_sw128(bs + kb * kCols * 128 + off);   // B^T tile: M = 128
          const uint64_t bdesc = tc::desc_k_sw128(as + kb * PANEL * 128 + off);  // A panel:  N = PANEL
          tc::mma_i8(d, adesc, bdesc, kIdesc, ks > 0 ? 1u : 0u);
        }
        tc::mma_commit(empty_bar(s));
        tc::mma_commit(tfull_bar(acc));
        MC_STAMP(i < 6, 16 + static_cast<int>(i));
        if (t + 1 == t1 || (t + 1) / p.n_ctiles != gpanel) tc::mma_commit(a_empty);
      }
    }
  } else if (warp < kFirstCons) {
    // ---------------- pattern builders (4 independent warps) ----------------
    // Builder warp bw owns vector rows 8*bw .. 8*bw+7 of the tile; lane = (row j, sub s),
    // four lanes per row. Each row streams its CSR column list through a 512-entry ring
    // in shared memory (eight 64-entry chunks, absolute position x in slot x & 511),
    // fetched by POSITION with cp.async up to 8 chunks from the cursor's chunk, so the
    // chunks a tile reads were issued at least one tile earlier. Positions are relative
    // to the row start (32-bit). A tile takes at most 128 entries of a row (columns are
    // strictly increasing). Per tile, lane (j, s) tests candidates s, s+4, s+8, ... of
    // row j, the four lanes OR their bitmaps with two shuffles, and lane (j, s) writes
    // the QuarterMap of quarter s. No cross-warp synchronisation: each warp arrives on
    // the tile's pfull barrier when its rows are published.
    const int bw = warp - kFirstBuild;
    const int jr = lane >> 2, sub = lane & 3;
    const int rl = 8 * bw + jr;  // this lane's vector row within the tile
    uint32_t* rrow = reinterpret_cast<uint32_t*>(smem + L::OFF_RING) + rl * kRingStride;
    const uint32_t rrow_s = smem_u32(rrow);
    // lane (j, s) issues its quarter of chunks [c_from, c_to) of row j; chunk c of a row
    // starting at `lo` covers absolute positions [((lo >> 6) + c) * 64, +64)
    auto fetch_chunks = [&](long long lo, int c_from, int c_to) {
      for (int c = c_from; c < c_to; ++c) {
        const long long base = ((lo >> 6) + c) * 64;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const long long pos0 = base + (sub * 4 + u) * 4;
          const long long avail = p.n_blocks - pos0;
          const uint32_t bytes = avail >= 4 ? 16u : (avail > 0 ? static_cast<uint32_t>(avail) * 4u : 0u);
          cp_async16(rrow_s + static_cast<uint32_t>(pos0 & 511) * 4, p.col_indices + (bytes ? pos0 : 0), bytes);
        }
      }
    };
    long long lo = 0;
    int len = 0, cur = 0, mtop = 0, lo511 = 0, lo63 = 0;
    // first panel's row offsets: issued before anything waits on them
    long long pre_lo = 0, pre_hi = 0;
    if (t0 < t1) {
      const long long r = ((t0 % tiles_per_item) / p.n_ctiles) * VR + rl;
      if (r < p.vrows) {
        pre_lo = p.row_offsets[r];
        pre_hi = p.row_offsets[r + 1];
      }
    }
    int64_t cur_panel = -1;
    for (int64_t t = t0; t < t1; ++t) {
      const int64_t i = t - t0;
      const int slot = static_cast<int>(i % kRing);
      const int64_t rem = t % tiles_per_item;
      const int64_t panel = rem / p.n_ctiles, ct = rem % p.n_ctiles;
      const int64_t gpanel = t / p.n_ctiles;
      const uint32_t c0 = static_cast<uint32_t>(ct * kCols);
      if (gpanel != cur_panel) {
        // ---- segment start: locate the row's cursor at column c0 ----
        cp_async_wait<0>();
        __syncwarp();
        long long hi = pre_hi;
        lo = pre_lo;
        if (t != t0) {
          const long long r = panel * VR + rl;
          lo = hi = 0;
          if (r < p.vrows) {
            lo = p.row_offsets[r];
            hi = p.row_offsets[r + 1];
          }
        }
        len = static_cast<int>(hi - lo);
        lo63 = static_cast<int>(lo & 63);
        lo511 = static_cast<int>(lo & 511);
        int start = 0;  // probe window start (relative)
        if (c0 > 0 && len > 512) {  // interpolated position of c0, minus a margin
          const int g = static_cast<int>((static_cast<double>(c0) / static_cast<double>(p.N)) * len);
          start = g - 192;
          if (start > len - 512) start = len - 512;
          if (start < 0) start = 0;
        }
        const int c_start = (lo63 + start) >> 6;
        if (len > 0) fetch_chunks(lo, c_start, c_start + 8);
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        cur = 0;
        mtop = c_start + 8;
        if (c0 > 0) {
          // lower bound of c0 inside the fetched window [ws, we) (binary search in smem)
          const int ws = (c_start * 64 - lo63 > 0) ? c_start * 64 - lo63 : 0;
          const int we = ((c_start + 8) * 64 - lo63 < len) ? (c_start + 8) * 64 - lo63 : len;
          int a = ws, b = we;
          while (a < b) {
            const int mid = (a + b) >> 1;
            if (rrow[(lo511 + mid) & 511] < c0) a = mid + 1;
            else b = mid;
          }
          cur = a;
          const bool miss = len > 0 && ((cur == ws && ws > 0) || (cur == we && we < len));
          if (miss) {  // rare: the probe did not bracket c0 -> binary search in global memory
            long long ga = lo, gb = lo + len;
            while (ga < gb) {
              const long long mid = (ga + gb) >> 1;
              if (__ldg(p.col_indices + mid) < c0) ga = mid + 1;
              else gb = mid;
            }
            cur = static_cast<int>(ga - lo);
          }
          const int c_lb = (lo63 + cur) >> 6;
          if (len > 0) {
            const int from = miss ? c_lb : (mtop > c_lb ? mtop : c_lb);
            fetch_chunks(lo, from, c_lb + 8);
          }
          cp_async_commit();
          if (__any_sync(0xffffffffu, miss || c_lb + 3 > mtop)) {
            cp_async_wait<0>();
            __syncwarp();
          }
          mtop = c_lb + 8;
        }
        cur_panel = gpanel;
        MC_STAMP(lane == 0 && bw == 0, 40);
      }
      // ---- this tile's bitmap of row j (lanes of the row split the candidates) ----
      const int left = len - cur;
      const int nvalid = (left < kCols) ? left : kCols;
      uint32_t w0 = 0u, w1 = 0u, w2 = 0u, w3 = 0u;
      bool bad = false;
      for (int k = sub; __any_sync(0xffffffffu, k < nvalid); k += 16) {
        uint32_t c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) c[u] = (k + 4 * u < nvalid) ? rrow[(lo511 + cur + k + 4 * u) & 511] : kNone;
        bool more = true;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t off = c[u] - c0;
          const bool in = off < static_cast<uint32_t>(kCols);
          more &= in;
          bad |= in && c[u] >= static_cast<uint32_t>(p.N);
          const uint32_t bit = in ? (1u << (off & 31)) : 0u;
          const uint32_t wsel = off >> 5;
          w0 |= wsel == 0 ? bit : 0u;
          w1 |= wsel == 1 ? bit : 0u;
          w2 |= wsel == 2 ? bit : 0u;
          w3 |= wsel == 3 ? bit : 0u;
        }
        // columns are strictly increasing: once a candidate is past the tile, so are
        // all later ones of this row -> retire the lane
        if (!more) k = kCols;
      }
      if (bad) flag_status(p.status, MC_STATUS_BAD_INDEX);
#pragma unroll
      for (int o = 1; o < 4; o <<= 1) {
        w0 |= __shfl_xor_sync(0xffffffffu, w0, o);
        w1 |= __shfl_xor_sync(0xffffffffu, w1, o);
        w2 |= __shfl_xor_sync(0xffffffffu, w2, o);
        w3 |= __shfl_xor_sync(0xffffffffu, w3, o);
      }
      const int p0 = __popc(w0), p1 = __popc(w1), p2 = __popc(w2), p3 = __popc(w3);
      const int pre = (sub > 0 ? p0 : 0) + (sub > 1 ? p1 : 0) + (sub > 2 ? p2 : 0);
      cp_async_wait<0>();  // chunks issued one tile ago (read from the next tile on)
      tc::mbar_wait(pempty_bar(slot), ((i / kRing) & 1) ^ 1);
      QuarterMap qm;
      qm.bits = sub == 0 ? w0 : sub == 1 ? w1 : sub == 2 ? w2 : w3;
      qm.pad = 0;
      qm.pos = lo + cur + pre;
      maps[slot * (VR * 4) + rl * 4 + sub] = qm;
      cur += p0 + p1 + p2 + p3;
      const int want = ((lo63 + cur) >> 6) + 8;
      if (want > mtop) {
        if (len > 0) fetch_chunks(lo, mtop, want);
        mtop = want;
      }
      cp_async_commit();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(pfull_bar(slot));
      MC_STAMP(lane == 0 && bw == 0 && i < 6, 22 + 3 * static_cast<int>(i));
    }
    cp_async_wait<0>();
  } else {
    // ---------------- consumers: TMEM -> registers -> V*4-byte block stores ----------------
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int half = (warp - kFirstCons) >> 2;
    const uint32_t ltmask = (1u << lane) - 1u;
    constexpr int rpc = 32 / V;  // vector rows per 32-column chunk
    constexpr int kChunks = PANEL / 64;  // 32-column TMEM chunks per consumer warp
    for (int64_t t = t0; t < t1; ++t) {
      const int64_t i = t - t0;
      const int slot = static_cast<int>(i % kRing);
      const int acc = static_cast<int>(i & 1);
      const int64_t item = t / tiles_per_item;
      const QuarterMap* m = maps + slot * (VR * 4);
      tc::mbar_wait(pfull_bar(slot), (i / kRing) & 1);
      tc::mbar_wait(tfull_bar(acc), (i >> 1) & 1);
      tc::tc_fence_after();
      MC_STAMP(warp == kFirstCons && lane == 0 && i < 6, 23 + 3 * static_cast<int>(i));
      const uint32_t tl = tmem + (static_cast<uint32_t>(32 * q) << 16) + acc * PANEL + (PANEL / 2) * half;
      uint32_t va[32], vb[32];
      tc::tmem_ld32_issue(tl, va);
      tc::tmem_wait_ld();
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
            store_block_if<V>(present, out + pos * V, &cur[V * w]);
          }
          if (kk + 1 < kChunks) tc::tmem_wait_ld();
        }
      } else {
        // fused dequant epilogue (attention.py:149-153): int32 (optional) + fp16(acc * alpha)
        int32_t* out = p.out ? p.out + item * p.out_stride : nullptr;
        uint16_t* out16 = p.out_f16 + item * p.f16_stride;
        const double alpha = p.alpha ? p.alpha[item] : p.alpha_host;
        for (int kk = 0; kk < kChunks; ++kk) {
          if (kk > 0) tc::tmem_ld32(tl + 32 * kk, va);
          for (int w = 0; w < rpc; ++w) {
            const QuarterMap qm = m[((kChunks * half + kk) * rpc + w) * 4 + q];
            if ((qm.bits >> lane) & 1u) {
              const long long pos = qm.pos + __popc(qm.bits & ltmask);
              uint32_t v[V];
#pragma unroll
              for (int x = 0; x < V; ++x) v[x] = va[V * w + x];
              if (out) store_block_if<V>(true, out + pos * V, v);
#pragma unroll
              for (int x = 0; x < V; ++x) out16[pos * V + x] = f16_bits_rn(static_cast<double>(static_cast<int32_t>(v[x])) * alpha);
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
  const bool dense_items = p.batch == 1 || (p.a_stride * 4 == p.M * p.K && p.b_stride * 4 == p.N * p.K);
  const uintptr_t out_align = static_cast<uintptr_t>(4 * p.V);
  return p.LB == 8 && p.RB == 8 && (p.V == 4 || p.V == 8) && (p.K == 128 || p.K == 256) &&
         p.batch >= 1 && dense_items && (p.out != nullptr || p.out_f16 != nullptr) &&
         (p.out == nullptr || ((reinterpret_cast<uintptr_t>(p.out) % out_align) == 0 && (p.out_stride % p.V) == 0)) &&
         (reinterpret_cast<uintptr_t>(p.a_words) & 15) == 0 && (reinterpret_cast<uintptr_t>(p.b_words) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(p.col_indices) & 15) == 0 && p.M > 0 && p.N > 0 && static_cast<int64_t>(p.batch) * p.N < (1ll << 31) &&
         static_cast<int64_t>(p.batch) * p.M < (1ll << 31) && p.N < (1ll << 32) - 256 && encode_fn() != nullptr;
}

cudaError_t launch_sddmm_tc(const SddmmParams& p, cudaStream_t stream) {
  CUtensorMap ta, tb;
  if (!make_map(&ta, p.a_words, p.batch * p.M, p.K, kVRows * p.V) || !make_map(&tb, p.b_words, p.batch * p.N, p.K, kCols))
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
  q.n_panels = static_cast<int>((p.M + kVRows * p.V - 1) / (kVRows * p.V));
  q.n_ctiles = static_cast<int>((p.N + kCols - 1) / kCols);
  q.tiles = static_cast<int64_t>(p.batch) * q.n_panels * q.n_ctiles;
  q.debug = getenv("MCUBE_DEBUG_TIMELINE") != nullptr;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = static_cast<int>(q.tiles < sms ? q.tiles : sms);
  if (grid == 0) return cudaSuccess;
  decltype(&sddmm_tc_kernel<8>) kern;
  int smem;
  switch (p.V) {
    case 8: kern = sddmm_tc_kernel<8>; smem = Lay<8>::TOTAL; break;
    default: kern = sddmm_tc_kernel<4>; smem = Lay<4>::TOTAL; break;
  }
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<grid, kThreads, smem, stream>>>(ta, tb, q);
  count_launch();
  return cudaGetLastError();
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
