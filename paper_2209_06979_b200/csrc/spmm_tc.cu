// spmm_tc.cu -- SR-BCRS x dense SpMM on the 5th-gen tensor cores (tcgen05 kind::i8).
//
// out[M x N] = A (SR-BCRS, V = 8, 8-bit) x B (K x N row-major, 8-bit), bit-exact with
// kernels.spmm (kernels.py:293-340). Transposed formulation, one task = (vector row r,
// 128-column tile): D^T[n, v] = sum_k B[idx_k, n] * A_r[v, k] with
//   UMMA M = 128 dense columns n   (A operand: the 32 gathered B rows of a k-step, MN-major,
//                                   fetched by TMA tile::gather4 straight into the
//                                   128-byte-swizzled canonical layout),
//   UMMA N = 8 vector-row lanes v  (B operand: the SR-BCRS stride blocks of the k-step,
//                                   fetched by a 2-D TMA box; K-major, no swizzle for
//                                   S = 16 (two 8 x 16 B core matrices), 32-byte swizzle
//                                   for S % 32 == 0),
//   UMMA K = 32 gathered indices.
// int8 x int8 products accumulate exactly in the TMEM int32 accumulator (the host-side
// check_accumulation_bound, emulation.py:108-113, guarantees K*(2^8-1)^2 < 2^31).
// Sentinel / padding slots (sparse_format.py:25) gather row -1: TMA zero-fills it.
//
// CTA (288 threads; several CTAs per SM):
//   warps 0-3 producers (k-steps dealt round-robin): per task the row's column indices are
//             bulk-copied (1024-entry chunks, double buffered); per k-step the warp copies
//             the 32 gathered rows (8 lanes per 128-byte row, coalesced cp.async) into the
//             swizzled operand layout plus the stride blocks, arriving on the step's
//             mbarrier through cp.async.mbarrier.arrive;
//   warp 4    TMEM allocator + single-thread MMA issuer (one tcgen05.mma per k-step,
//             kAcc accumulators in flight so a task's MMAs overlap the previous drain);
//   warps 5-8 epilogue: tcgen05.ld of the 8 accumulator columns of lane quarter q, then
//             coalesced 128-byte stores of each output row (optional fused fp16 dequant).
#include <cuda_fp16.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace mcube {
namespace {

constexpr int kNT = 128;       // dense columns per task (UMMA M)
constexpr int kAcc = 4;        // TMEM accumulators (8 columns each)
constexpr int kIdxChunk = 1024;
constexpr int kProd = 4;        // producer warps (k-steps dealt round-robin)
constexpr int kMmaWarp = kProd;  // then the MMA warp, then 4 epilogue warps
constexpr int kThreads = 32 * (kProd + 1 + 4);
constexpr int kATile = 32 * kNT;  // 4 KB: 32 gathered rows x 128 bytes
constexpr int kLTile = 256;       // 8 rows x 32 bytes of LHS values

template <int kStages>
struct SmemL {
  static constexpr int OFF_A = 0;                                  // kStages x 4 KB (1024-aligned)
  static constexpr int OFF_L = OFF_A + kStages * kATile;           // kStages x 256 B
  static constexpr int OFF_IDX = OFF_L + kStages * kLTile;         // 2 x kIdxChunk uint32
  static constexpr int OFF_BAR = OFF_IDX + 2 * kIdxChunk * 4;
  static constexpr int N_BARS = 2 * kStages + 2 * kAcc + 2;        // full/empty, tfull/tempty, idx[2]
  static constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
  static constexpr int TOTAL = OFF_TMEM + 16 + 1024;
};

__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, uint32_t bar, int col, int r0,
                                            int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// arrive on `bar` once all prior cp.async of this thread have completed (no pending-count increment)
__device__ __forceinline__ void cp_async_mbar_arrive(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}

// tcgen05.ld 32 lanes x 8 consecutive 32-bit columns
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA descriptor, MN-major, 128-byte swizzle: 128-byte rows along M, 8-row K groups 1024 B apart.
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
// UMMA descriptor, K-major, no swizzle: 8 rows x 16 B core matrices, the two 16-byte K halves 128 B apart.
__device__ __forceinline__ uint64_t desc_k_interleave(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (8ull << 16) | (16ull << 32) | (1ull << 46) | (0ull << 61);
}
// UMMA descriptor, K-major, 32-byte swizzle: 8 rows x 32 B.
__device__ __forceinline__ uint64_t desc_k_sw32(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (1ull << 16) | (16ull << 32) | (1ull << 46) | (6ull << 61);
}

struct TaskCursor {  // task t -> (batch item, vector row, column tile), advanced incrementally
  long long item, r, nt;
  long long vrows, ntiles;
  __device__ TaskCursor(long long t, long long vr, long long nti) : vrows(vr), ntiles(nti) {
    const long long rt = t / nti;
    nt = t - rt * nti;
    item = rt / vr;
    r = rt - item * vr;
  }
  __device__ __forceinline__ void advance(long long by) {  // by may exceed ntiles (grid stride)
    nt += by;
    if (nt >= ntiles) {
      const long long carry = nt / ntiles;
      nt -= carry * ntiles;
      r += carry;
      if (r >= vrows) {
        const long long c2 = r / vrows;
        r -= c2 * vrows;
        item += c2;
      }
    }
  }
};

template <int kStages>
__global__ void __launch_bounds__(kThreads)
spmm_tc_kernel(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmL, const SpmmParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar0 = sbase + SmemL<kStages>::OFF_BAR;
  auto full_bar = [&](int s) { return bar0 + 8 * s; };
  auto empty_bar = [&](int s) { return bar0 + 8 * (kStages + s); };
  auto tfull_bar = [&](int a) { return bar0 + 8 * (2 * kStages + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8 * (2 * kStages + kAcc + a); };
  auto idx_bar = [&](int b) { return bar0 + 8 * (2 * kStages + 2 * kAcc + b); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + SmemL<kStages>::OFF_TMEM);
  const uint32_t* idx_s = reinterpret_cast<const uint32_t*>(smem + SmemL<kStages>::OFF_IDX);
  const long long tasks = p.tasks;
  const long long stride = gridDim.x;
  const int S = p.S;

  if (warp == kMmaWarp && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(full_bar(s), p.gather_tma ? 1 : 32);  // TMA: tx bytes; cp.async: one arrival per lane
      tc::mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < kAcc; ++a) {
      tc::mbar_init(tfull_bar(a), 1);
      tc::mbar_init(tempty_bar(a), 4);
    }
    tc::mbar_init(idx_bar(0), 1);
    tc::mbar_init(idx_bar(1), 1);
    tc::fence_barrier_init();
    tc::prefetch_tmap(&tmB);
    tc::prefetch_tmap(&tmL);
  }
  if (warp == kMmaWarp) tc::tmem_alloc<32>(smem_u32(tmem_holder));
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp < kProd) {
    // ---------------- producers ----------------
    const int pw = warp;
    const bool shuffled = p.shuffled != 0;
    // value position -> stored index position within an 8-group (sparse_format.py:222-230)
    const int kperm = shuffled ? ((lane & ~7) | (((lane & 7) >> 1) | ((lane & 1) << 2))) : lane;
    const uint32_t kdim = static_cast<uint32_t>(p.K);
    const uint8_t* rhs_b = reinterpret_cast<const uint8_t*>(p.rhs_words);
    const uint8_t* lhs_b = reinterpret_cast<const uint8_t*>(p.lhs_words);
    const uint8_t* lhs_end = lhs_b + p.batch * p.stored * 8;  // 8-bit values, V = 8
    uint32_t g = 0;       // global k-step counter (ring position)
    uint32_t nchunk = 0;  // index chunks consumed so far (buffer = nchunk & 1)
    // index chunk (pb + c0, cn) -> buffer b; lane 0 issues
    auto load_chunk = [&](uint32_t b, long long src, int cn) {
      if (pw == 0 && lane == 0) {
        tc::mbar_arrive_expect_tx(idx_bar(b), cn * 4);
        bulk_load(sbase + SmemL<kStages>::OFF_IDX + b * kIdxChunk * 4, p.col_indices + src, cn * 4, idx_bar(b));
      }
    };
    TaskCursor tcur(blockIdx.x, p.vrows, p.ntiles);
    long long pb = 0, n_true = 0;
    if (blockIdx.x < tasks) {
      pb = p.row_begin[tcur.r];
      n_true = p.row_end[tcur.r] - pb;
      const int st0 = static_cast<int>(((n_true + S - 1) / S) * S);
      if (st0 > 0) load_chunk(0, pb, st0 < kIdxChunk ? st0 : kIdxChunk);
    }
    for (long long t = blockIdx.x; t < tasks; t += stride) {
      const int stored = static_cast<int>(((n_true + S - 1) / S) * S);
      const int col_byte = static_cast<int>(tcur.nt * kNT);  // 8-bit B: column offset in bytes
      const long long brow0 = tcur.item * p.K;               // batch item's first B row
      const long long lrow0 = tcur.item * (p.stored / S) * 8 + (pb / S) * 8;  // first LHS box row
      // next task (its offsets load now; consumed when its first chunk is prefetched)
      TaskCursor ncur = tcur;
      ncur.advance(stride);
      const bool has_next = t + stride < tasks;
      long long npb = 0, nend = 0;
      if (has_next) {
        npb = p.row_begin[ncur.r];
        nend = p.row_end[ncur.r];
      }
      for (int c0 = 0; c0 < stored; c0 += kIdxChunk) {
        const int cn = (stored - c0 < kIdxChunk) ? stored - c0 : kIdxChunk;
        const uint32_t buf = nchunk & 1;
        // every producer is done with the previous chunk: its buffer may be refilled
        tc::named_bar(1, 32 * kProd);
        // prefetch the following chunk (this task's next one, or the next task's first)
        if (c0 + kIdxChunk < stored) {
          const int cn2 = (stored - c0 - kIdxChunk < kIdxChunk) ? stored - c0 - kIdxChunk : kIdxChunk;
          load_chunk(buf ^ 1, pb + c0 + kIdxChunk, cn2);
        } else if (has_next) {
          const long long nst = ((nend - npb + S - 1) / S) * S;
          if (nst > 0) load_chunk(buf ^ 1, npb, static_cast<int>(nst < kIdxChunk ? nst : kIdxChunk));
        }
        tc::mbar_wait(idx_bar(buf), (nchunk >> 1) & 1);
        ++nchunk;
        const uint32_t* ix = idx_s + buf * kIdxChunk;
        const int s_end = (c0 + cn + 31) >> 5;
        for (int s = c0 >> 5; s < s_end; ++s, ++g) {
          if (static_cast<int>(g % kProd) != pw) continue;  // this warp's k-steps
          const int q = 32 * s + lane;  // value position of this lane's k slot (= A-operand row k)
          const int slot = g % kStages;
          if (p.gather_tma) {
            // TMA: 8 x gather4 (4 rows of 128 B each, 128-byte swizzle applied by the TMA unit)
            // + one 2-D box of stride blocks; completion counted in bytes on the step barrier
            int row = -1;
            if (q < stored) {
              const uint32_t col = ix[(32 * s + kperm) - c0];
              if (col < kdim) row = static_cast<int>(brow0 + col);
              else if (col != kSentinel) flag_status(p.status, MC_STATUS_BAD_INDEX);
            }
            tc::mbar_wait(empty_bar(slot), ((g / kStages) & 1) ^ 1);
            if (lane == 0) tc::mbar_arrive_expect_tx(full_bar(slot), kATile + kLTile);
            __syncwarp();
            const int r0 = __shfl_sync(0xffffffffu, row, (4 * lane) & 31);
            const int r1 = __shfl_sync(0xffffffffu, row, (4 * lane + 1) & 31);
            const int r2 = __shfl_sync(0xffffffffu, row, (4 * lane + 2) & 31);
            const int r3 = __shfl_sync(0xffffffffu, row, (4 * lane + 3) & 31);
            const uint32_t adst = sbase + SmemL<kStages>::OFF_A + slot * kATile;
            if (lane < 8) tma_gather4(adst + lane * 512, &tmB, full_bar(slot), col_byte, r0, r1, r2, r3);
            if (lane == 8) {
              const uint32_t ldst = sbase + SmemL<kStages>::OFF_L + slot * kLTile;
              if (S == 16) tc::tma_load_2d(ldst, &tmL, full_bar(slot), 0, static_cast<int>(lrow0 + 16 * s));
              else
                tc::tma_load_2d(ldst, &tmL, full_bar(slot), (32 * s) % S,
                                static_cast<int>(lrow0 + ((32 * s) / S) * 8));
            }
            continue;
          }
          const uint8_t* src = nullptr;
          if (q < stored) {
            const uint32_t col = ix[(32 * s + kperm) - c0];
            if (col < kdim) src = rhs_b + (brow0 + col) * p.N + col_byte;
            else if (col != kSentinel) flag_status(p.status, MC_STATUS_BAD_INDEX);
          }
          tc::mbar_wait(empty_bar(slot), ((g / kStages) & 1) ^ 1);
          // row k of the MN-major SW128 operand: 8-row group k/8 (1024 B), row k%8 (128 B),
          // 16-byte chunk c stored at chunk c ^ (k % 8); a sentinel row is zero-filled.
          // Copy j moves rows 4j..4j+3 with 8 lanes per row: one coalesced 128-byte row each.
          const int c = lane & 7;
          const bool col_ok = col_byte + 16 * c < p.N;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int k = 4 * j + (lane >> 3);
            const uint8_t* rs = reinterpret_cast<const uint8_t*>(
                __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(src), k));
            const bool ok = rs != nullptr && col_ok;
            const uint32_t dst = sbase + SmemL<kStages>::OFF_A + slot * kATile + (k >> 3) * 1024 + (k & 7) * 128 +
                                 ((c ^ (k & 7)) << 4);
            cp_async16(dst, ok ? rs + 16 * c : rhs_b, ok ? 16u : 0u);
          }
          // the k-step's stride blocks: S = 16 -> two 8 x 16 B core matrices (plain copy);
          // S % 32 == 0 -> 8 rows x 32 B with the 32-byte swizzle (chunk ^= (row >> 2) & 1)
          if (lane < 16) {
            const uint32_t ldst = sbase + SmemL<kStages>::OFF_L + slot * kLTile;
            const uint8_t* lsrc;
            uint32_t loff;
            if (S == 16) {
              lsrc = lhs_b + (lrow0 + 16 * s) * 16 + 16 * lane;
              loff = 16 * lane;
            } else {
              const int v = lane >> 1, cc = lane & 1;
              lsrc = lhs_b + (lrow0 + ((32 * s) / S) * 8 + v) * S + (32 * s) % S + 16 * cc;
              loff = v * 32 + ((cc ^ ((v >> 2) & 1)) << 4);
            }
            // (the second stride of a row's last S = 16 step may lie past the array end)
            const bool in = lsrc < lhs_end;
            cp_async16(ldst + loff, in ? lsrc : lhs_b, in ? 16u : 0u);
          }
          cp_async_mbar_arrive(full_bar(slot));
        }
        __syncwarp();
      }
      tcur = ncur;
      pb = npb;
      n_true = nend - npb;
    }
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_i8(128, 8) | (1u << 15);  // A (gathered rows) MN-major
      uint32_t g = 0;
      int i = 0;
      TaskCursor tcur(blockIdx.x, p.vrows, p.ntiles);
      long long n_true = blockIdx.x < tasks ? p.row_end[tcur.r] - p.row_begin[tcur.r] : 0;
      for (long long t = blockIdx.x; t < tasks; t += stride, ++i) {
        tcur.advance(stride);
        long long n_next = 0;  // next task's row length, loaded one task ahead
        if (t + stride < tasks) n_next = p.row_end[tcur.r] - p.row_begin[tcur.r];
        const int nsteps = static_cast<int>((((n_true + S - 1) / S) * S + 31) >> 5);
        const int acc = i % kAcc;
        tc::mbar_wait(tempty_bar(acc), ((i / kAcc) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem + acc * 8;
        for (int s = 0; s < nsteps; ++s, ++g) {
          const int slot = g % kStages;
          tc::mbar_wait(full_bar(slot), (g / kStages) & 1);
          tc::fence_proxy_async();  // cp.async (generic proxy) writes -> tcgen05.mma (async proxy) reads
          tc::tc_fence_after();
          const uint32_t a_addr = sbase + SmemL<kStages>::OFF_A + slot * kATile;
          const uint32_t l_addr = sbase + SmemL<kStages>::OFF_L + slot * kLTile;
          const uint64_t adesc = desc_mn_sw128(a_addr);
          const uint64_t bdesc = S == 16 ? desc_k_interleave(l_addr) : desc_k_sw32(l_addr);
          tc::mma_i8(d, adesc, bdesc, idesc, s > 0 ? 1u : 0u);
          tc::mma_commit(empty_bar(slot));
        }
        tc::mma_commit(tfull_bar(acc));
        n_true = n_next;
      }
    }
  } else {
    // ---------------- epilogue (warps 5..8 -> TMEM lane quarters 1,2,3,0) ----------------
    const int q = warp & 3;
    int i = 0;
    TaskCursor tcur(blockIdx.x, p.vrows, p.ntiles);
    long long n_true = blockIdx.x < tasks ? p.row_end[tcur.r] - p.row_begin[tcur.r] : 0;
    for (long long t = blockIdx.x; t < tasks; t += stride, ++i) {
      const long long r = tcur.r, item = tcur.item, nt = tcur.nt;
      tcur.advance(stride);
      long long n_next = 0;
      if (t + stride < tasks) n_next = p.row_end[tcur.r] - p.row_begin[tcur.r];
      const int acc = i % kAcc;
      tc::mbar_wait(tfull_bar(acc), (i / kAcc) & 1);
      tc::tc_fence_after();
      uint32_t v[8];
      tmem_ld8(tmem + (static_cast<uint32_t>(32 * q) << 16) + acc * 8, v);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tempty_bar(acc));
      if (n_true <= 0) {  // no k-steps: the accumulator was never written
#pragma unroll
        for (int x = 0; x < 8; ++x) v[x] = 0u;
      }
      const long long n = nt * kNT + 32 * q + lane;
      if (n < p.N) {
        const long long base = (r * 8) * p.N + n;
        if (p.out) {
          int32_t* o = p.out + item * p.out_stride + base;
#pragma unroll
          for (int x = 0; x < 8; ++x) o[x * p.N] = static_cast<int32_t>(v[x]);
        }
        if (p.out_f16) {
          const double alpha = p.alpha ? p.alpha[item] : p.alpha_host;
          const float alpha_f = static_cast<float>(alpha);
          uint16_t* o = p.out_f16 + item * p.f16_stride + base;
#pragma unroll
          for (int x = 0; x < 8; ++x) o[x * p.N] = f16_dequant(static_cast<int32_t>(v[x]), alpha, alpha_f);
        }
      }
      n_true = n_next;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc::tc_fence_after();
    tc::tmem_dealloc<32>(tmem);
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
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

bool encode2d(CUtensorMap* m, const void* base, uint64_t inner_bytes, uint64_t rows, uint32_t box_inner,
              uint32_t box_rows, CUtensorMapSwizzle sw) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner_bytes, rows};
  cuuint64_t strides[1] = {inner_bytes};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool spmm_tc_supported(const SpmmParams& p) {
  // Opt-in (MCUBE_SPMM_PATH=tc): on C3 this path matches the mma.sync kernel at 70% sparsity
  // and trails it at 90-98% -- both are bound near 5 TB/s of gathered L2 rows
  const char* e = getenv("MCUBE_SPMM_PATH");
  if (!e || e[0] != 't') return false;
  const bool dense_items = p.batch == 1 || (p.rhs_stride * 4 == p.K * p.N && p.lhs_stride * 4 == p.stored * 8);
  return p.LB == 8 && p.RB == 8 && p.V == 8 && (p.S == 16 || p.S % 32 == 0) && p.N % 16 == 0 && dense_items &&
         p.stored > 0 && (reinterpret_cast<uintptr_t>(p.rhs_words) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(p.lhs_words) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(p.col_indices) & 15) == 0 && p.K * p.batch < (1ll << 31) &&
         encode_fn() != nullptr;
}

cudaError_t launch_spmm_tc(SpmmParams p, cudaStream_t stream) {
  CUtensorMap tb, tl;
  // B: [batch*K rows, N bytes]; box = 128 bytes x 1 row, gathered 4 rows per instruction
  if (!encode2d(&tb, p.rhs_words, static_cast<uint64_t>(p.N), static_cast<uint64_t>(p.batch * p.K), kNT, 1,
                CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  // LHS values: [batch*stored/S*8 rows, S bytes]; box = 16 rows x 16 B (S = 16) or 8 rows x 32 B
  const uint64_t lrows = static_cast<uint64_t>(p.batch) * (p.stored / p.S) * 8;
  const bool ok = p.S == 16 ? encode2d(&tl, p.lhs_words, 16, lrows, 16, 16, CU_TENSOR_MAP_SWIZZLE_NONE)
                            : encode2d(&tl, p.lhs_words, static_cast<uint64_t>(p.S), lrows, 32, 8,
                                       CU_TENSOR_MAP_SWIZZLE_32B);
  if (!ok) return cudaErrorInvalidValue;
  p.ntiles = (p.N + kNT - 1) / kNT;
  p.tasks = static_cast<int64_t>(p.batch) * p.vrows * p.ntiles;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // ring depth x CTAs per SM = k-steps in flight per SM (tunable for experiments)
  const char* es = getenv("MCUBE_SPMM_STAGES");
  const char* ec = getenv("MCUBE_SPMM_CTAS");
  const int stages = es ? atoi(es) : 16;
  const char* eg = getenv("MCUBE_SPMM_GATHER");
  p.gather_tma = (eg && eg[0] == 't') ? 1 : 0;
  const int per_sm = ec ? atoi(ec) : 2;
  const long long want = static_cast<long long>(sms) * per_sm;
  const int grid = static_cast<int>(p.tasks < want ? p.tasks : want);
  if (grid == 0) return cudaSuccess;
  if (stages >= 16) {
    cudaFuncSetAttribute(spmm_tc_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, SmemL<16>::TOTAL);
    spmm_tc_kernel<16><<<grid, kThreads, SmemL<16>::TOTAL, stream>>>(tb, tl, p);
  } else if (stages >= 12) {
    cudaFuncSetAttribute(spmm_tc_kernel<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, SmemL<12>::TOTAL);
    spmm_tc_kernel<12><<<grid, kThreads, SmemL<12>::TOTAL, stream>>>(tb, tl, p);
  } else {
    cudaFuncSetAttribute(spmm_tc_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, SmemL<8>::TOTAL);
    spmm_tc_kernel<8><<<grid, kThreads, SmemL<8>::TOTAL, stream>>>(tb, tl, p);
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace mcube
