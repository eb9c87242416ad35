// gemm_tc.cu -- exact int8-plane GEMM on tcgen05 for the dense-tile SpMM path (dense.cu).
//
// out[M x N] (int32) = sum_{i<LC, j<RC} 2^(8(i+j)) * A_i[M x K] * B_j[K x N], with A_i / B_j
// the int8 chunk planes of the LHS / RHS (plane 0 unsigned when the operand has two planes,
// qint.py:185-206). Each plane product accumulates exactly in its own TMEM int32
// accumulator; the epilogue recombines in int64 and applies the same int32 checks as the
// gather kernel (spmm.cu epilogue; kernels.py:286-288, tile_engine.py:246-247).
//
// Tile 128 (M) x 256/128 (N), K in 128-byte blocks; UMMA M=128 N=256/128 K=32, A K-major
// (A plane [M x K] row-major, 128-byte swizzle), B MN-major (B plane [K x N] row-major:
// 128 n-bytes per k row, 8-row groups 1024 B apart). One persistent CTA per SM:
//   warp 0     TMA producer (LC + RC boxes of 128 x 128 bytes per k-block stage);
//   warp 1     TMEM allocator + single-thread MMA issuer;
//   warps 2-5  epilogue (TMEM lane quarter per warp; a thread owns one output row).
#include <cuda_fp16.h>

#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace mcube {
namespace {

constexpr int kTM = 128, kKB = 128;
constexpr int kBox = kTM * kKB;  // 16 KB per 128 x 128-byte box

template <int LC, int RC, int TN_ = 0>
struct GemmCfg {
  // 128 x 128 tiles by default (twice the CTAs of 128 x 256, which measured slower at
  // C3 sizes: both are bound by L2 delivery of the re-read operand boxes); TN_ = 256 is
  // available for single-plane products (MCUBE_GEMM_TN=256)
  static constexpr int TN = TN_ ? TN_ : 128;
  static constexpr int NB = TN / 128;                  // 128-column B boxes per plane
  static constexpr int STAGE = (LC + RC * NB) * kBox;
  static constexpr int STAGES = STAGE <= 32768 ? 5 : (STAGE <= 49152 ? 4 : 3);
  static constexpr int NACC = LC * RC;                 // accumulators per tile (TN cols each)
  static constexpr int SETS = NACC * TN <= 256 ? 2 : 1;  // tiles in flight in TMEM
  static constexpr int OFF_BAR = STAGES * STAGE;
  static constexpr int N_BARS = 2 * STAGES + 2 * SETS;
  static constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
  static constexpr int TOTAL = OFF_TMEM + 16 + 1024;
};

__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t saddr, uint32_t lbo_bytes) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16) |
         (64ull << 32) | (1ull << 46) | (2ull << 61);
}

struct GemmMaps {
  CUtensorMap a[2];
  CUtensorMap b[2];
};

// CL > 1: clusters of CL CTAs along M, one tile per CTA; each B box is fetched in CL
// row slices, one per CTA, multicast to the whole cluster (B traffic / CL), and every
// CTA's MMA completion is multicast to the empty barriers of all CTAs of the cluster.
template <int LC, int RC, int TN_, int CL>
__global__ void __launch_bounds__(192, 1)
gemm_tc_kernel(const __grid_constant__ GemmMaps maps, const SpmmParams p) {
  using C = GemmCfg<LC, RC, TN_>;
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
      tc::mbar_init(full_bar(s), 1);
      tc::mbar_init(empty_bar(s), CL);  // one MMA-commit arrival per CTA of the cluster
    }
    for (int a = 0; a < C::SETS; ++a) {
      tc::mbar_init(tfull_bar(a), 1);
      tc::mbar_init(tempty_bar(a), 4);
    }
    tc::fence_barrier_init();
    for (int i = 0; i < LC; ++i) tc::prefetch_tmap(&maps.a[i]);
    for (int j = 0; j < RC; ++j) tc::prefetch_tmap(&maps.b[j]);
  }
  if (warp == 1) tc::tmem_alloc<512>(smem_u32(tmem_holder));
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();  // the A planes are written by the densify kernel just before
  tc::tc_fence_before();
  __syncthreads();
  if constexpr (CL > 1) tc::cluster_sync();  // peers' barriers initialised before any multicast
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const uint32_t crank = CL > 1 ? tc::cluster_ctarank() : 0u;
  constexpr uint16_t kMask = static_cast<uint16_t>((1u << CL) - 1u);
  // tile schedule: persistent over all tiles (CL = 1) or one tile per CTA, the CL CTAs
  // of a cluster on consecutive M tiles of one N tile (CL > 1)
  const int t_first = CL > 1 ? ((blockIdx.x / CL) % nt) + (((blockIdx.x / CL) / nt) * CL + crank) * nt
                             : static_cast<int>(blockIdx.x);
  const int t_step = CL > 1 ? tiles : static_cast<int>(gridDim.x);

  if (warp == 0) {
    if (lane == 0) {
      uint32_t g = 0;
      for (int t = t_first; t < tiles; t += t_step) {
        const int m0 = (t / nt) * kTM, n0 = (t % nt) * kTN;
        // rotated k start (CL = 1): tiles sharing an operand box read it at different times;
        // a cluster walks k in lockstep (its CTAs share every B box)
        const int kr = CL > 1 ? 0 : t % KB;
        for (int kk = 0; kk < KB; ++kk, ++g) {
          const int kb = (kk + kr) % KB;
          const int s = g % C::STAGES;
          tc::mbar_wait(empty_bar(s), ((g / C::STAGES) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(full_bar(s), C::STAGE);
          const uint32_t st = sbase + s * C::STAGE;
#pragma unroll
          for (int i = 0; i < LC; ++i) tc::tma_load_2d(st + i * kBox, &maps.a[i], full_bar(s), kb * kKB, m0);
#pragma unroll
          for (int j = 0; j < RC; ++j)
#pragma unroll
            for (int nb = 0; nb < C::NB; ++nb) {
              if constexpr (CL > 1)  // this CTA's 128/CL k-row slice of the box, to every CTA
                tc::tma_load_2d_mc(st + (LC + j * C::NB + nb) * kBox + crank * (kBox / CL), &maps.b[j], full_bar(s),
                                   n0 + 128 * nb, kb * kKB + static_cast<int>(crank) * (kKB / CL), kMask);
              else
                tc::tma_load_2d(st + (LC + j * C::NB + nb) * kBox, &maps.b[j], full_bar(s), n0 + 128 * nb, kb * kKB);
            }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t g = 0;
      int it = 0;
      for (int t = t_first; t < tiles; t += t_step, ++it) {
        const int set = it % C::SETS;
        tc::mbar_wait(tempty_bar(set), ((it / C::SETS) & 1) ^ 1);
        tc::tc_fence_after();
        for (int kb = 0; kb < KB; ++kb, ++g) {  // kb = position in the (rotated) k order
          const int s = g % C::STAGES;
          tc::mbar_wait(full_bar(s), (g / C::STAGES) & 1);
          tc::tc_fence_after();
          const uint32_t st = sbase + s * C::STAGE;
#pragma unroll
          for (int i = 0; i < LC; ++i) {
#pragma unroll
            for (int j = 0; j < RC; ++j) {
              const uint32_t idesc = tc::idesc_i8(kTM, kTN, LC == 2 && i == 0, RC == 2 && j == 0) | (1u << 16);
              const uint32_t d = tmem + (set * C::NACC + i * RC + j) * kTN;
#pragma unroll
              for (int ks = 0; ks < kKB / 32; ++ks) {
                const uint64_t adesc = tc::desc_k_sw128(st + i * kBox + ks * 32);
                // B: NB 128-column atoms 16 KB apart (LBO), 8-row k groups 1024 B apart (SBO)
                const uint64_t bdesc = desc_mn_sw128(st + (LC + j * C::NB) * kBox + ks * 4096, kBox);
                tc::mma_i8(d, adesc, bdesc, idesc, (kb > 0 || ks > 0) ? 1u : 0u);
              }
            }
          }
          if constexpr (CL > 1) tc::mma_commit_mc(empty_bar(s), kMask);
          else tc::mma_commit(empty_bar(s));
        }
        tc::mma_commit(tfull_bar(set));
      }
    }
  } else {
    // epilogue: warp w reads TMEM lanes 32*(w%4).., i.e. output rows m0 + 32*(w%4) + lane
    const int q = warp & 3;
    int it = 0;
    for (int t = t_first; t < tiles; t += t_step, ++it) {
      const int set = it % C::SETS;
      const int m0 = (t / nt) * kTM, n0 = (t % nt) * kTN;
      tc::mbar_wait(tfull_bar(set), (it / C::SETS) & 1);
      tc::tc_fence_after();
      const uint32_t tl = tmem + (static_cast<uint32_t>(32 * q) << 16) + set * C::NACC * kTN;
      int32_t* orow = p.out + static_cast<int64_t>(m0 + 32 * q + lane) * p.N + n0;
      bool overflow = false;
#pragma unroll 1
      for (int c = 0; c < kTN / 32; ++c) {
        uint32_t acc[C::NACC][32];
#pragma unroll
        for (int a = 0; a < C::NACC; ++a) tc::tmem_ld32_issue(tl + a * kTN + 32 * c, acc[a]);
        tc::tmem_wait_ld();
        int32_t res[32];
#pragma unroll
        for (int x = 0; x < 32; ++x) {
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
        for (int x = 0; x < 8; ++x)
          reinterpret_cast<int4*>(orow + 32 * c)[x] = make_int4(res[4 * x], res[4 * x + 1], res[4 * x + 2], res[4 * x + 3]);
      }
      if (overflow) flag_status(p.status, MC_STATUS_OVERFLOW);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tempty_bar(set));
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if constexpr (CL > 1) tc::cluster_sync();  // no CTA leaves while peers may still signal it
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
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(f);
  }
  return fn;
}

// 2-D int8 map [rows x cols] row-major, box 128 x 128, 128-byte swizzle
bool map128(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows = 128) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols)};
  cuuint32_t box[2] = {128, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int LC, int RC, int TN_>
cudaError_t launch_lr(const GemmMaps& maps, const SpmmParams& p, cudaStream_t stream, bool cluster) {
  using C = GemmCfg<LC, RC, TN_>;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles = static_cast<int>((p.M / kTM) * (p.N / C::TN));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = C::TOTAL;
  cfg.stream = stream;
  cfg.attrs = attr;
  cudaError_t e;
  if (cluster) {
    constexpr int kCL = 4;
    auto k = gemm_tc_kernel<LC, RC, TN_, kCL>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::TOTAL);
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = kCL;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.gridDim = dim3(tiles);
    cfg.numAttrs = 2;
    e = cudaLaunchKernelEx(&cfg, k, maps, p);
  } else {
    auto k = gemm_tc_kernel<LC, RC, TN_, 1>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::TOTAL);
    cfg.gridDim = dim3(tiles < sms ? tiles : sms);
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k, maps, p);
  }
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

// Eligible: one problem (no batch), int32 output only, tile-aligned shapes, density high
// enough that a dense tensor-core pass beats the L2 gather (crossover measured on C3).
static bool e_forced_dense() {
  const char* e = getenv("MCUBE_SPMM_PATH");
  return e && e[0] == 'd';
}

bool dense_spmm_eligible(const SpmmParams& p) {
  if (p.batch != 1 || p.out == nullptr || p.out_f16 != nullptr) return false;
  if (p.M % kTM || p.N % 128 || p.K % kKB || p.M <= 0 || p.N <= 0 || p.K <= 0) return false;
  if (p.stored <= 0 || encode_fn() == nullptr) return false;
  // byte-chunk planes only: nibble-chunk plans and strides wider than a staging batch take
  // the gather kernels
  if (spmm_needs_nibble_chunks(p) || !densify_stride_ok(p)) return false;
  if (!(e_forced_dense()) && spmm_seg_supported(p)) return false;  // the segment gather kernel is faster there
  if ((reinterpret_cast<uintptr_t>(p.rhs_words) & 15) || (reinterpret_cast<uintptr_t>(p.out) & 15)) return false;
  const double density = static_cast<double>(p.stored) * p.V / (static_cast<double>(p.M) * p.K);
  const char* e = getenv("MCUBE_SPMM_PATH");
  if (e && e[0] == 'd') return true;   // forced dense
  if (e && e[0] != 'd') return false;  // forced gather (mma / tc)
  // The gather moves one RHS row per stored vector (bytes ~ density / V), the dense pass a
  // fixed M*K + GEMM: measured C3 crossovers (tools/c3_path_probe.py, 5 pairs x V in
  // {2, 4, 8} x 95/98 %) sit at density / V ~ 0.008 (L16-R16), 0.012 (other 2-plane LHS)
  // and 0.010 (8/4-bit LHS). With fewer than 64 output tiles the GEMM cannot fill the GPU
  // (C1, 8 tiles: 14.3 us dense vs 8.2 us gather).
  const long long tiles = (p.M / kTM) * (p.N / 128);
  const double thr = p.LB >= 12 ? (p.RB == 16 ? 0.008 : 0.012) : 0.010;
  return density / p.V >= thr && tiles >= 64;
}

cudaError_t launch_gemm_tc(const SpmmParams& p, const int8_t* a0, const int8_t* a1, const int8_t* b0,
                           const int8_t* b1, cudaStream_t stream) {
  GemmMaps maps;
  memset(&maps, 0, sizeof(maps));
  const int lc = p.LB >= 12 ? 2 : 1, rc = p.RB == 16 ? 2 : 1;
  // opt-in (MCUBE_GEMM_CLUSTER=1): clusters of 4 along M sharing each B box by TMA multicast.
  // Measured: no L2-traffic or time saving at C3 (L2 already merges near-simultaneous
  // unicast reads of a box by <= 4 CTAs), so the default is the persistent unicast kernel.
  const char* ec = getenv("MCUBE_GEMM_CLUSTER");
  const bool cluster = (p.M / kTM) % 4 == 0 && ec && ec[0] == '1';
  const int brows = cluster ? kKB / 4 : kKB;
  if (!map128(&maps.a[0], a0, p.M, p.K) || (lc == 2 && !map128(&maps.a[1], a1, p.M, p.K)) ||
      !map128(&maps.b[0], b0, p.K, p.N, brows) || (rc == 2 && !map128(&maps.b[1], b1, p.K, p.N, brows)))
    return cudaErrorInvalidValue;
  if (lc == 1 && rc == 1) {
    const char* e = getenv("MCUBE_GEMM_TN");
    if (e && atoi(e) == 256 && p.N % 256 == 0) return launch_lr<1, 1, 256>(maps, p, stream, cluster);
    return launch_lr<1, 1, 0>(maps, p, stream, cluster);
  }
  if (lc == 2 && rc == 1) return launch_lr<2, 1, 0>(maps, p, stream, cluster);
  if (lc == 1 && rc == 2) return launch_lr<1, 2, 0>(maps, p, stream, cluster);
  return launch_lr<2, 2, 0>(maps, p, stream, cluster);
}

}  // namespace mcube
