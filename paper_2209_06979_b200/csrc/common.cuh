// common.cuh -- shared device helpers for the Magicube B200 kernels (sm_100a).
//
// Integer MMA: mma.sync m16n8k32 with s8/u8 operands (SASS IMMA.16832.*),
// the narrow-N engine for V <= 8 vector rows. Byte transposes are PRMT
// (the register transpose of PAPER.md:247); 4-bit operands are sign-extended
// to s8 with LOP3/IMAD because sm_100a has no native int4 IMMA (the s4
// mma.sync form is emulated on ALUs).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/mcube.h"

namespace mcube {

constexpr uint32_t kSentinel = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// 4x4 byte transpose: in r[i] holds bytes (i, 0..3); out o[c] holds (0..3, c).
__device__ __forceinline__ void transpose4x4(uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3,
                                             uint32_t& o0, uint32_t& o1, uint32_t& o2,
                                             uint32_t& o3) {
  const uint32_t t0 = prmt(r0, r1, 0x5140);  // r0b0 r1b0 r0b1 r1b1
  const uint32_t t1 = prmt(r0, r1, 0x7362);  // r0b2 r1b2 r0b3 r1b3
  const uint32_t t2 = prmt(r2, r3, 0x5140);
  const uint32_t t3 = prmt(r2, r3, 0x7362);
  o0 = prmt(t0, t2, 0x5410);
  o1 = prmt(t0, t2, 0x7632);
  o2 = prmt(t1, t3, 0x5410);
  o3 = prmt(t1, t3, 0x7632);
}

// Sign-extend four nibbles held in the low nibble of each byte to s8.
__device__ __forceinline__ uint32_t sext_nibble_bytes(uint32_t x) {
  return x | ((x & 0x08080808u) * 0x1Eu);
}

// 8 packed s4 values (LSB-first) -> even-index and odd-index s8 words.
__device__ __forceinline__ void unpack_s4x8(uint32_t w, uint32_t& even, uint32_t& odd) {
  even = sext_nibble_bytes(w & 0x0F0F0F0Fu);
  odd = sext_nibble_bytes((w >> 4) & 0x0F0F0F0Fu);
}

// 4 packed s4 values in the low 16 bits -> one s8 word in element order.
__device__ __forceinline__ uint32_t unpack_s4x4_ordered(uint32_t h) {
  const uint32_t spread = (h & 0xFu) | ((h & 0xF0u) << 4) | ((h & 0xF00u) << 8) |
                          ((h & 0xF000u) << 12);
  return sext_nibble_bytes(spread);
}

// Two 16-bit words (4 int16 elements) -> low-byte chunk (u8) and high-byte chunk (s8).
__device__ __forceinline__ void split16(uint32_t w0, uint32_t w1, uint32_t& lo, uint32_t& hi) {
  lo = prmt(w0, w1, 0x6420);
  hi = prmt(w0, w1, 0x7531);
}

// D += A(16x32, row) * B(32x8, col), int32 accumulate, wrapping (no .satfinite).
template <bool AU, bool BU>
__device__ __forceinline__ void mma16832(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  if constexpr (!AU && !BU) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  } else if constexpr (AU && !BU) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  } else if constexpr (!AU && BU) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
}

// ldmatrix.m16n16.x2.trans.b8 (LDSM.8.MT1616.2): lanes 0-15 give the 16-byte rows k = 0..15
// of matrix 0, lanes 16-31 rows k = 16..31 of matrix 1; lane (g, t) receives bytes (row k,
// column g) / (k, g + 8) for k = 4t..4t+3 of matrix 0 in r0 / r1 and of matrix 1 in r2 / r3:
// exactly the m16n8k32 A fragment of the 16 x 32 transpose (tools/micro/ldsm_probe.cu,
// profiles/r02s3_ldsm_layout.json).
// Used by the row-segment SpMM consumer and the attention P x V step.
__device__ __forceinline__ void ldsm_t16x2(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m16n16.x2.trans.shared.b8 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async with zero fill: copies `src_bytes` (0..16) and zero-fills the rest.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async16_full(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

// Generic element fetch from a packed LSB-first stream (qint.py:65-82).
// Works for any width in {4, 8, 12, 16} and any element offset.
__device__ __forceinline__ int32_t fetch_packed(const uint32_t* __restrict__ words, int64_t elem,
                                                int bits) {
  const int64_t bit = elem * bits;
  const int64_t w = bit >> 5;
  const int sh = static_cast<int>(bit & 31);
  uint64_t v = static_cast<uint64_t>(__ldg(words + w)) >> sh;
  if (sh + bits > 32) v |= static_cast<uint64_t>(__ldg(words + w + 1)) << (32 - sh);
  const uint32_t mask = (1u << bits) - 1u;
  int32_t x = static_cast<int32_t>(static_cast<uint32_t>(v) & mask);
  return (x ^ (1 << (bits - 1))) - (1 << (bits - 1));  // sign extend
}

__device__ __forceinline__ void flag_status(uint32_t* status, uint32_t bits) {
  if (status) atomicOr(status, bits);
}

__device__ __forceinline__ int64_t min_i64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ bool fits_i32(long long x) {
  return x >= -2147483648LL && x <= 2147483647LL;
}

// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may start while
// the previous kernel on the stream drains; pdl_wait() blocks until that kernel has
// completed and its memory is visible, so it must precede the first read of any input a
// previous kernel could have produced. pdl_launch_dependents() lets the next kernel be
// scheduled early. Both are no-ops for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }

__device__ __forceinline__ uint16_t f16_bits_rn(double x) {
  __half h = __double2half(x);
  return *reinterpret_cast<uint16_t*>(&h);
}

// fp16(round_to_nearest((double)acc * alpha)) -- the reference's dequant rounding chain
// (attention.py:62-65, :149-153, :170-173) -- evaluated in fp32 whenever fp32 decides it:
// the fp32 product is within 4 * 2^-24 relative of the float64 one, so if scaling it by
// 1 -/+ 2^-21 rounds to the same fp16 value the float64 product does too; otherwise (a
// product next to an fp16 rounding boundary, ~1e-3 of the cases) take float64.
__device__ __forceinline__ uint16_t f16_dequant(int32_t acc, double alpha, float alpha_f) {
  const float y = static_cast<float>(acc) * alpha_f;
  // both roundings in one packed F2FP
  const __half2 h = __floats2half2_rn(y * 0.99999952316284180f, y * 1.00000047683715820f);
  const uint32_t hb = *reinterpret_cast<const uint32_t*>(&h);
  if ((hb & 0xffffu) == (hb >> 16)) return static_cast<uint16_t>(hb);
  return f16_bits_rn(static_cast<double>(acc) * alpha);
}

// Launch `kern` with the programmatic-stream-serialization attribute (see pdl_wait).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace mcube
