// attention.cu -- quantised sparse self-attention (attention.py:130-197) on B200.
//
// Pipeline per head (all heads share one 8x1 block mask, attention.py:190-197):
//   quantize Q, K, V (symmetric absmax, attention.py:40-56)         -> quant kernels
//   SDDMM Q_q K_q^T at the mask, fused dequant to fp16 (:147-154)   -> sddmm.cu
//   row softmax over stored blocks + fused requant (:108-127, :157-162) -> softmax kernel
//   SpMM probs (SR-BCRS) x V_q, fused dequant to fp16 (:164-176)    -> spmm.cu
// Parity mode evaluates every rounding step exactly as the reference does
// (float64 math, round-to-nearest-even into fp16, rint requant); fast mode runs
// the softmax in float32.
#include <cuda_fp16.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace mcube {

cudaError_t launch_attention(const mc_attention_args* a, uint32_t* status, cudaStream_t stream, size_t* ws_needed);

namespace {

__device__ __forceinline__ double load_in(const void* p, int dtype, int64_t i) {
  if (dtype == MC_DTYPE_F16) return static_cast<double>(__half2float(reinterpret_cast<const __half*>(p)[i]));
  if (dtype == MC_DTYPE_F32) return static_cast<double>(reinterpret_cast<const float*>(p)[i]);
  return reinterpret_cast<const double*>(p)[i];
}

// grid (batch, 3): absmax of one [L x d] tensor -> scale (attention.py:52-54)
__global__ void __launch_bounds__(512)
absmax_kernel(const void* q, const void* k, const void* v, int dtype, int64_t n, int bits, double* scales,
              int smax) {
  const int64_t b = blockIdx.x;
  const int which = blockIdx.y;
  const void* src = which == 0 ? q : (which == 1 ? k : v);
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, fabs(load_in(src, dtype, b * n + i)));
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = (threadIdx.x < blockDim.x / 32) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) {
      const double qmax = static_cast<double>((1 << (bits - 1)) - 1);
      scales[b * 4 + which] = m > 0.0 ? m / qmax : 1.0;
      if (which == 0) scales[b * 4 + 3] = 1.0 / static_cast<double>(smax);
    }
  }
}

// one thread per output word of the packed [L x d] tensor
__global__ void quant_kernel(const void* q, const void* k, const void* v, int dtype, int64_t n, int bits,
                             const double* scales, uint32_t* out, int64_t words_per, int64_t batch) {
  const int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int which = blockIdx.y;
  if (w >= words_per * batch) return;
  const int64_t b = w / words_per;
  const int64_t wi = w - b * words_per;
  const void* src = which == 0 ? q : (which == 1 ? k : v);
  const double scale = scales[b * 4 + which];
  const double qmax = static_cast<double>((1 << (bits - 1)) - 1);
  const int per = 32 / bits;
  uint32_t word = 0;
  for (int e = 0; e < per; ++e) {
    const int64_t i = wi * per + e;
    if (i >= n) break;
    double x = rint(load_in(src, dtype, b * n + i) / scale);
    x = fmin(fmax(x, -qmax), qmax);
    const uint32_t qv = static_cast<uint32_t>(static_cast<int32_t>(x)) & ((1u << bits) - 1u);
    word |= qv << (e * bits);
  }
  out[(static_cast<int64_t>(which) * batch + b) * words_per + wi] = word;
}

__global__ void alpha_kernel(const double* scales, int64_t batch, int head_dim, double* alpha_s, double* alpha_m) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const double sq = scales[b * 4], sk = scales[b * 4 + 1], sv = scales[b * 4 + 2], ss = scales[b * 4 + 3];
  alpha_s[b] = sq * sk / sqrt(static_cast<double>(head_dim));  // attention.py:147
  alpha_m[b] = ss * sv;                                          // attention.py:169
}

__device__ __forceinline__ double h2d(uint16_t h) {
  __half x;
  *reinterpret_cast<uint16_t*>(&x) = h;
  return static_cast<double>(__half2float(x));
}

// fp16(e / sum) and its requantised value clip(rint(p16 / (1/smax))) (attention.py:127,
// :157-162), both exactly as the reference's float64 chain: the product e * (1/sum) is within
// 2 ulp of the quotient, so it decides the fp16 rounding unless a 2^-45 perturbation crosses
// an fp16 boundary (then the division is taken); p16 * smax is exact in fp32 and never lies
// within rounding distance of a .5 tie, so rintf of it equals rint(p16 / (1/smax)).
__device__ __forceinline__ void prob_requant(double e, double sum, double inv_sum, int smax, uint16_t& pf,
                                             int32_t& qi) {
  const double pr = e * inv_sum;
  pf = f16_bits_rn(pr);
  if (f16_bits_rn(pr * 0.9999999999999716) != f16_bits_rn(pr * 1.0000000000000284)) pf = f16_bits_rn(e / sum);
  __half h;
  *reinterpret_cast<uint16_t*>(&h) = pf;
  int q = static_cast<int>(rintf(__half2float(h) * static_cast<float>(smax)));
  qi = q > smax ? smax : (q < -smax ? -smax : q);
}

// FAST-mode exp(x - max) shared by every kernel of the fast pipeline: ex2 of the fma
// x * log2(e) - max * log2(e) (flush-to-zero), with mneg = -(max * log2 e) per row.
constexpr float kLog2e = 1.4426950408889634f;
__device__ __forceinline__ float att_exp_fast(float x, float mneg) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(fmaf(x, kLog2e, mneg)));
  return y;
}

// Requant level from float32 arithmetic (FAST pipeline): p32 = e * fp32(1/sum) is within
// 2^-23 (relative) of the float64 quotient e / sum, so fp16 of p32 * (1 -+ 2^-21) brackets
// fp16(e / sum); when both ends give the same level that level is exact (it is what
// prob_requant returns). Otherwise -1: the caller takes prob_requant (rare: p within 2^-21 of
// an fp16 tie whose two neighbours straddle a requant level).
__device__ __forceinline__ int prob_q_fast(float e, float inv_f, float smax_f) {
  const float p = e * inv_f;
  const float2 f = __half22float2(__floats2half2_rn(p * 0.99999952316284180f, p * 1.00000047683715820f));
  const float ql = rintf(f.x * smax_f), qh = rintf(f.y * smax_f);
  return ql == qh ? static_cast<int>(ql) : -1;
}

// packed fp32 pairs (FADD2 / FFMA2 on sm_100a)
__device__ __forceinline__ unsigned long long f2_pack(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2_unpack(unsigned long long r) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
__device__ __forceinline__ unsigned long long f2_add(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2_sub(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// one warp per (head, vector row); lane owns blocks j = lane, lane+32, ...
template <bool FAST>
__global__ void softmax_requant_kernel(const uint16_t* __restrict__ scores, int64_t nblk8, const int64_t* offs,
                                       int64_t vrows, const int64_t* sr_begin, int S, int smax, int sbits,
                                       uint32_t* sr_vals, int64_t sr_stride_words, uint16_t* probs_f16,
                                       int32_t* probs_int, int64_t batch) {
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= batch * vrows) return;
  const int64_t b = gw / vrows, r = gw - b * vrows;
  const int64_t lo = offs[r], hi = offs[r + 1], nb = hi - lo;
  const int64_t sbeg = sr_begin[r];
  const int64_t stored = ((nb + S - 1) / S) * S;
  const uint16_t* sc = scores + b * nblk8 + lo * 8;
  uint8_t* sv8 = reinterpret_cast<uint8_t*>(sr_vals + b * sr_stride_words);
  uint16_t* sv16 = reinterpret_cast<uint16_t*>(sr_vals + b * sr_stride_words);

  double mx[8], sum[8];
#pragma unroll
  for (int v = 0; v < 8; ++v) { mx[v] = -INFINITY; sum[v] = 0.0; }
  for (int64_t j = lane; j < nb; j += 32) {
    const uint4 u = *reinterpret_cast<const uint4*>(sc + j * 8);
    const uint16_t* hs = reinterpret_cast<const uint16_t*>(&u);
#pragma unroll
    for (int v = 0; v < 8; ++v) mx[v] = fmax(mx[v], h2d(hs[v]));
  }
#pragma unroll
  for (int v = 0; v < 8; ++v)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx[v] = fmax(mx[v], __shfl_xor_sync(0xffffffffu, mx[v], o));
  float mneg[8];
#pragma unroll
  for (int v = 0; v < 8; ++v) mneg[v] = -static_cast<float>(mx[v]) * kLog2e;
  for (int64_t j = lane; j < nb; j += 32) {
    const uint4 u = *reinterpret_cast<const uint4*>(sc + j * 8);
    const uint16_t* hs = reinterpret_cast<const uint16_t*>(&u);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      if constexpr (FAST) sum[v] += static_cast<double>(att_exp_fast(static_cast<float>(h2d(hs[v])), mneg[v]));
      else sum[v] += exp(h2d(hs[v]) - mx[v]);
    }
  }
#pragma unroll
  for (int v = 0; v < 8; ++v)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum[v] += __shfl_xor_sync(0xffffffffu, sum[v], o);
  double inv_sum[8];
#pragma unroll
  for (int v = 0; v < 8; ++v) inv_sum[v] = 1.0 / sum[v];

  for (int64_t j = lane; j < stored; j += 32) {
    const int64_t pos = sbeg + j;
    const int64_t s = pos / S, jj = pos - s * S;
    if (j < nb) {
      const uint4 u = *reinterpret_cast<const uint4*>(sc + j * 8);
      const uint16_t* hs = reinterpret_cast<const uint16_t*>(&u);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        double e;
        if constexpr (FAST) e = static_cast<double>(att_exp_fast(static_cast<float>(h2d(hs[v])), mneg[v]));
        else e = exp(h2d(hs[v]) - mx[v]);
        uint16_t pf;
        int32_t qi;
        prob_requant(e, sum[v], inv_sum[v], smax, pf, qi);  // attention.py:127, :158
        const int64_t el = s * 8 * S + static_cast<int64_t>(v) * S + jj;
        if (sbits == 8) sv8[el] = static_cast<uint8_t>(qi);
        else sv16[el] = static_cast<uint16_t>(qi);
        if (probs_f16) probs_f16[b * nblk8 + (lo + j) * 8 + v] = pf;
        if (probs_int) probs_int[b * nblk8 + (lo + j) * 8 + v] = qi;
      }
    } else {
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int64_t el = s * 8 * S + static_cast<int64_t>(v) * S + jj;
        if (sbits == 8) sv8[el] = 0;
        else sv16[el] = 0;
      }
    }
  }
}

// ---- fp16-input fast paths (the C4 configuration) ----

// 8-bit quantisation of 16 fp16 values into one 16-byte output (attention.py:55):
// q = clip(rint(x / scale)) with the quotient in float64.
__device__ __forceinline__ uint4 quant16_f16_exact(uint4 u0, uint4 u1, double scale) {
  const __half* h = reinterpret_cast<const __half*>(&u0);
  const __half* h1 = reinterpret_cast<const __half*>(&u1);
  uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const double d = rint(static_cast<double>(__half2float(e < 8 ? h[e] : h1[e - 8])) / scale);
    const int qi = static_cast<int>(fmin(fmax(d, -127.0), 127.0));
    w[e >> 2] |= (static_cast<uint32_t>(qi) & 0xFFu) << (8 * (e & 3));
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}
// FAST: the quotient as x * fp32(1 / scale) (packed FMUL2) is within 2^-23 relative
// (<= 1.6e-5 absolute for |q| <= 127.5) of the float64 one, so rounding it (magic-number
// FADD2, whose low byte is the two's-complement level) gives the float64 result unless it
// lies within 5e-5 of a tie; a group with such an element takes quant16_f16_exact. The
// level never exceeds 127 in magnitude (|x| <= absmax = 127 * scale), so no clip is needed.
template <bool FAST>
__device__ __forceinline__ uint4 quant16_f16(uint4 u0, uint4 u1, double scale, float inv_f) {
  if constexpr (!FAST) {
    return quant16_f16_exact(u0, u1, scale);
  } else {
    const uint4 uu[2] = {u0, u1};
    const unsigned long long inv2 = f2_pack(inv_f, inv_f), mag2 = f2_pack(12582912.0f, 12582912.0f);
    uint32_t w[4];
    float dmax = 0.f;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const __half2* h = reinterpret_cast<const __half2*>(&uu[i]);
      uint32_t tb[8];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const float2 f = __half22float2(h[x]);
        const unsigned long long qf = f2_mul(f2_pack(f.x, f.y), inv2);
        const unsigned long long tq = f2_add(qf, mag2);
        const float2 dd = f2_unpack(f2_sub(qf, f2_sub(tq, mag2)));
        dmax = fmaxf(dmax, fmaxf(fabsf(dd.x), fabsf(dd.y)));
        const float2 tt = f2_unpack(tq);
        tb[2 * x] = __float_as_uint(tt.x);
        tb[2 * x + 1] = __float_as_uint(tt.y);
      }
      w[2 * i] = __byte_perm(__byte_perm(tb[0], tb[1], 0x0040), __byte_perm(tb[2], tb[3], 0x0040), 0x5410);
      w[2 * i + 1] = __byte_perm(__byte_perm(tb[4], tb[5], 0x0040), __byte_perm(tb[6], tb[7], 0x0040), 0x5410);
    }
    if (dmax > 0.49995f) return quant16_f16_exact(u0, u1, scale);
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// One 8-CTA cluster per [L x d] fp16 tensor (grid (8 * batch, 3) = Q, K, V of each head):
// each CTA stages its 1/8 slice (up to kQuantSmem bytes; a larger remainder is streamed from
// global twice) in shared memory with one bulk copy (the copy engine keeps 64 KB per CTA,
// three CTAs per SM, in flight -- the register-tile version held two), the slice maxima meet
// through distributed shared memory (|x| max, attention.py:52-54; exact in fp32 for fp16
// magnitudes), and the slice is quantised from shared memory -- one HBM read and one int8
// write per element. The last of a head's three rank-0 CTAs (per-head arrival counter, reset
// for the next launch) derives alpha_s (:147) and alpha_m (:169).
constexpr int kQuantThreads = 256, kQuantCluster = 8;
constexpr int kQuantSmem = 64 * 1024;  // staged slice bytes per CTA
__device__ __forceinline__ void st_cluster_f32(const float* local_addr, uint32_t rank, float v) {
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(local_addr)), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ra), "f"(v) : "memory");
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <bool FAST>
__global__ void __cluster_dims__(kQuantCluster, 1, 1) __launch_bounds__(kQuantThreads, 3)
absquant_f16_kernel(const __half* q, const __half* k, const __half* v, int64_t n, int smax, int head_dim,
                    double* scales, double* alpha_s, double* alpha_m, uint32_t* out, int64_t words_per,
                    int64_t batch, uint32_t* arrivals) {
  extern __shared__ __align__(128) uint8_t qsm[];  // the staged slice: groups of 2 x uint4
  __shared__ float red[kQuantThreads / 32];
  __shared__ float slice_max[kQuantCluster];
  __shared__ __align__(8) uint64_t qbar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int64_t b = blockIdx.x / kQuantCluster;
  const int which = blockIdx.y;
  const uint4* src = reinterpret_cast<const uint4*>((which == 0 ? q : (which == 1 ? k : v)) + b * n);
  uint4* dst = reinterpret_cast<uint4*>(out + (static_cast<int64_t>(which) * batch + b) * words_per);
  // slice: 16-element groups [g0, g1) of this CTA; group g = 2 uint4 of input, 1 of output
  const int64_t n16 = n / 16;
  const int64_t g0 = n16 * rank / kQuantCluster, g1 = n16 * (rank + 1) / kQuantCluster;
  const int64_t held = (g1 - g0) < kQuantSmem / 32 ? (g1 - g0) : kQuantSmem / 32;
  const uint32_t bar = smem_u32(&qbar), sq = smem_u32(qsm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t bytes = static_cast<uint32_t>(held * 32);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    if (bytes)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sq), "l"(src + 2 * g0), "r"(bytes), "r"(bar) : "memory");
  }
  float m = 0.f;
  // slices larger than the stage: the remainder's maximum while the bulk copy lands
  for (int64_t g = g0 + held + threadIdx.x; g < g1; g += kQuantThreads) {
    const uint4 w[2] = {__ldg(src + 2 * g), __ldg(src + 2 * g + 1)};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const __half2* h = reinterpret_cast<const __half2*>(&w[i]);
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const float2 f = __half22float2(h[x]);
        m = fmaxf(m, fmaxf(fabsf(f.x), fabsf(f.y)));
      }
    }
  }
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "QW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
      "@!P1 bra QW_%=;\n}" ::"r"(bar)
      : "memory");
  const uint4* s4 = reinterpret_cast<const uint4*>(qsm);
  __half2 m2 = __float2half2_rn(0.f);
  for (int i = threadIdx.x; i < 2 * held; i += kQuantThreads) {
    const uint4 u = s4[i];
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int x = 0; x < 4; ++x) m2 = __hmax2(m2, __habs2(h[x]));  // exact on fp16
  }
  {
    const float2 f = __half22float2(m2);
    m = fmaxf(m, fmaxf(f.x, f.y));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < kQuantThreads / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x < kQuantCluster) st_cluster_f32(&slice_max[rank], threadIdx.x, m);  // to every CTA
  }
  cluster_barrier();  // no remote shared-memory access after this point
  m = 0.f;
#pragma unroll
  for (int i = 0; i < kQuantCluster; ++i) m = fmaxf(m, slice_max[i]);
  const double md = static_cast<double>(m);
  const double scale = md > 0.0 ? md / 127.0 : 1.0;
  const float inv_f = static_cast<float>(1.0 / scale);
  for (int64_t i = threadIdx.x; i < held; i += kQuantThreads)
    dst[g0 + i] = quant16_f16<FAST>(s4[2 * i], s4[2 * i + 1], scale, inv_f);
  for (int64_t g = g0 + held + threadIdx.x; g < g1; g += kQuantThreads)
    dst[g] = quant16_f16<FAST>(__ldg(src + 2 * g), __ldg(src + 2 * g + 1), scale, inv_f);
  if (rank == 0 && threadIdx.x == 0) {
    scales[b * 4 + which] = scale;
    uint32_t prev;  // release publishes the scale, acquire (for the last) sees the others'
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(arrivals + b) : "memory");
    if (prev == 2u) {
      const double s0 = __ldcg(scales + b * 4), s1 = __ldcg(scales + b * 4 + 1), s2 = __ldcg(scales + b * 4 + 2);
      const double ss = 1.0 / static_cast<double>(smax);
      scales[b * 4 + 3] = ss;
      alpha_s[b] = s0 * s1 / sqrt(static_cast<double>(head_dim));
      alpha_m[b] = ss * s2;
      arrivals[b] = 0u;
    }
  }
}

// Fused score SDDMM + softmax + requant for 8-bit Q/K and d = 64 (attention.py:147-162):
// one warp per (head, vector row). The row's scores are computed with mma.sync (16 mask
// blocks x 8 query rows per MMA, K rows gathered from L2, d split 16 bytes per thread)
// and dequantised exactly like the SDDMM epilogue (f16_dequant); they stay in shared
// memory (kCap blocks per warp; longer rows recompute their chunks in each pass) and go
// through the same float64 max / exp-sum / prob / requant sequence as
// softmax_requant_kernel, which writes the SR-BCRS probability values the SpMM consumes.
// Saves the fp16 score round trip through HBM and the score kernel's K = 64 padding.
// cached mask blocks per warp (fp16 scores [kCap][8]); MIX trims it so that four 4-warp
// CTAs fit an SM (16 warps)
template <bool MIX>
constexpr int att_cap() { return MIX ? 480 : 512; }
// per-warp shared memory of the fused kernel: scores [kCap][8] fp16, column indices
// [kCap], the row sums (float64, for the rare exact-division fallback), and with MIX the
// int8 probabilities of one k-step [8][32] + a 2-slot ring of 32 V rows
template <bool MIX>
constexpr int att_warp_smem() {
  return att_cap<MIX>() * 20 + 64 + (MIX ? 8 * 32 + 2 * 32 * 64 : 0);
}

// MIX: also the P x V product (attention.py:164-176) -- the requantised probabilities stay
// in shared memory as the MMA B operand, the V rows of each 32-block k-step are gathered
// by cp.async in the slot order / XOR swizzle of spmm.cu and byte-transposed with PRMT,
// and the output is dequantised to fp16 in the epilogue (one kernel per layer after
// quantisation); otherwise pass 3 writes the SR-BCRS probabilities for the SpMM kernel.
template <bool FAST, bool MIX>
__global__ void __launch_bounds__(128, (MIX && FAST) ? 4 : 1)
score_softmax_kernel(const uint32_t* __restrict__ qw, const uint32_t* __restrict__ kw, int64_t head_words,
                     const int64_t* __restrict__ offs, const uint32_t* __restrict__ cols, int64_t vrows,
                     int64_t L, const double* __restrict__ alpha_s, const int64_t* __restrict__ sr_begin, int S,
                     int smax, int sbits, uint32_t* sr_vals, int64_t sr_stride_words, int64_t batch,
                     uint32_t* status, const uint32_t* __restrict__ vw, const double* __restrict__ alpha_m,
                     uint16_t* __restrict__ out_f16) {
  constexpr int kCap = att_cap<MIX>();
  extern __shared__ __align__(16) uint8_t att_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wsm = att_smem + warp * att_warp_smem<MIX>();
  uint16_t* sc = reinterpret_cast<uint16_t*>(wsm);
  uint32_t* ix = reinterpret_cast<uint32_t*>(wsm + kCap * 16);
  double* wsum = reinterpret_cast<double*>(wsm + kCap * 20);      // row sums [8]
  int8_t* pm = reinterpret_cast<int8_t*>(wsm + kCap * 20 + 64);   // MIX: P[v][32] of one k-step
  uint8_t* vring = wsm + kCap * 20 + 64 + 256;                    // MIX: 2 x 32 V rows x 64 B
  const int g = lane >> 2, t = lane & 3;
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * 4 + warp;
  if (gw >= batch * vrows) return;
  const int64_t b = gw / vrows, r = gw - b * vrows;
  const int64_t lo = offs[r], nb = offs[r + 1] - lo;
  const double alpha = alpha_s[b];
  const float alpha_f = static_cast<float>(alpha);
  // query rows r*8 .. r*8+7 (MMA N = 8): this thread's 16 bytes d = 16t .. 16t+15 of row g
  const uint4 qv = __ldg(reinterpret_cast<const uint4*>(qw + b * head_words + (r * 8 + g) * 16) + t);
  const uint32_t* kh = kw + b * head_words;
  const uint8_t* khb = reinterpret_cast<const uint8_t*>(kh) + t * 16;  // this lane's 16 bytes of a K row

  // dequantisation brackets: fp16 of acc * alpha_{lo,hi} (alpha * (1 -+ 2^-22) in fp32) brackets
  // fp16(acc * alpha) (fp32 error <= 2^-23); equal ends are the exact f16_dequant result
  const float alpha_lo = static_cast<float>(alpha * 0.99999976158142090), alpha_hi = static_cast<float>(alpha * 1.00000023841857910);
  // two scores per packed fp16 word, exact (falls back to f16_dequant when a bracket is open)
  auto dequant2 = [&](int a0, int a1) -> uint32_t {
    const float y0 = static_cast<float>(a0), y1 = static_cast<float>(a1);
    const __half2 l = __floats2half2_rn(y0 * alpha_lo, y1 * alpha_lo);
    const __half2 h = __floats2half2_rn(y0 * alpha_hi, y1 * alpha_hi);
    const uint32_t lb = *reinterpret_cast<const uint32_t*>(&l), hb = *reinterpret_cast<const uint32_t*>(&h);
    if (lb == hb) return lb;
    return static_cast<uint32_t>(f16_dequant(a0, alpha, alpha_f)) | (static_cast<uint32_t>(f16_dequant(a1, alpha, alpha_f)) << 16);
  };

  // scores of blocks [j0, j0 + jn) into sc[(j - j0) * 8 + v]: the chunk's column indices
  // are staged in shared memory by one coalesced pass (padded with column 0 to a multiple
  // of 32 for the MIX gathers), then the K rows of 4 groups of 16 blocks are loaded before
  // their MMAs (8 independent 16-byte loads in flight per lane)
  auto compute = [&](int64_t j0, int jn) {
    const int jpad = (jn + 31) & ~31;
    for (int i = lane; i < jpad; i += 32) {
      uint32_t c = 0;
      if (i < jn) {
        c = __ldg(cols + lo + j0 + i);
        if (c >= static_cast<uint32_t>(L)) {
          flag_status(status, MC_STATUS_BAD_INDEX);
          c = 0;
        }
      }
      ix[i] = c;
    }
    __syncwarp();
    for (int grp0 = 0; grp0 < jn; grp0 += 64) {
      uint4 ka[4], kb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int m0 = grp0 + 16 * u + g, m1 = m0 + 8;
        const uint32_t c_lo = m0 < jn ? ix[m0] : 0u;
        const uint32_t c_hi = m1 < jn ? ix[m1] : 0u;
        ka[u] = __ldg(reinterpret_cast<const uint4*>(khb + static_cast<size_t>(c_lo) * 64));
        kb[u] = __ldg(reinterpret_cast<const uint4*>(khb + static_cast<size_t>(c_hi) * 64));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int m0 = grp0 + 16 * u + g, m1 = m0 + 8;
        int acc[4] = {0, 0, 0, 0};
        mma16832<false, false>(acc, ka[u].x, kb[u].x, ka[u].y, kb[u].y, qv.x, qv.y);  // d 16t + 0..7
        mma16832<false, false>(acc, ka[u].z, kb[u].z, ka[u].w, kb[u].w, qv.z, qv.w);  // d 16t + 8..15
        // c0 = S[block g][query 2t], c1 = [g][2t+1], c2 = [g+8][2t], c3 = [g+8][2t+1]
        const uint32_t h01 = dequant2(acc[0], acc[1]);
        const uint32_t h23 = dequant2(acc[2], acc[3]);
        if (m0 < jn) reinterpret_cast<uint32_t*>(sc)[(m0 * 8 + 2 * t) >> 1] = h01;
        if (m1 < jn) reinterpret_cast<uint32_t*>(sc)[(m1 * 8 + 2 * t) >> 1] = h23;
      }
    }
    __syncwarp();
  };
  const bool cached = nb <= kCap;
  if (cached) compute(0, static_cast<int>(nb));

  // pass 1: row maxima (fp16 scores compare exactly; packed half2 max)
  __half2 mx2[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) mx2[p] = __float2half2_rn(-INFINITY);
  for (int64_t j0 = 0; j0 < nb; j0 += kCap) {
    const int jn = static_cast<int>(nb - j0 < kCap ? nb - j0 : kCap);
    if (!cached) { __syncwarp(); compute(j0, jn); }
    for (int j = lane; j < jn; j += 32) {
      const uint4 u = *reinterpret_cast<const uint4*>(sc + j * 8);
      const __half2* hs = reinterpret_cast<const __half2*>(&u);
#pragma unroll
      for (int p = 0; p < 4; ++p) mx2[p] = __hmax2(mx2[p], hs[p]);
    }
  }
  float mxf[8], mneg[8];
  double mx[8], sum[8];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const float2 f = __half22float2(mx2[p]);
    mxf[2 * p] = f.x;
    mxf[2 * p + 1] = f.y;
  }
#pragma unroll
  for (int v = 0; v < 8; ++v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mxf[v] = fmaxf(mxf[v], __shfl_xor_sync(0xffffffffu, mxf[v], o));
    mx[v] = static_cast<double>(mxf[v]);
    mneg[v] = -mxf[v] * kLog2e;
    sum[v] = 0.0;
  }
  // pass 2: sum of exp(x - max) (attention.py:120-124). Parity: float64 exp; fast:
  // att_exp_fast accumulated as fp32 (hi, lo) TwoSum pairs, two rows per FADD2.
  unsigned long long shi[4], slo[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) shi[p] = slo[p] = 0ull;
  for (int64_t j0 = 0; j0 < nb; j0 += kCap) {
    const int jn = static_cast<int>(nb - j0 < kCap ? nb - j0 : kCap);
    if (!cached) { __syncwarp(); compute(j0, jn); }
    for (int j = lane; j < jn; j += 32) {
      const uint4 u = *reinterpret_cast<const uint4*>(sc + j * 8);
      const __half2* hs = reinterpret_cast<const __half2*>(&u);
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const float2 x = __half22float2(hs[p]);
        if constexpr (FAST) {
          const unsigned long long e = f2_pack(att_exp_fast(x.x, mneg[2 * p]), att_exp_fast(x.y, mneg[2 * p + 1]));
          const unsigned long long t1 = f2_add(shi[p], e);
          const unsigned long long bp = f2_sub(t1, shi[p]);
          const unsigned long long err = f2_add(f2_sub(shi[p], f2_sub(t1, bp)), f2_sub(e, bp));
          slo[p] = f2_add(slo[p], err);
          shi[p] = t1;
        } else {
          sum[2 * p] += exp(static_cast<double>(x.x) - mx[2 * p]);
          sum[2 * p + 1] += exp(static_cast<double>(x.y) - mx[2 * p + 1]);
        }
      }
    }
  }
  double inv_sum[8];
  float thr[8], inv_f[8];
  const float smax_f = static_cast<float>(smax);
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    if constexpr (FAST) {
      const float2 h = f2_unpack(shi[v >> 1]), l = f2_unpack(slo[v >> 1]);
      sum[v] = (v & 1) ? static_cast<double>(h.y) + static_cast<double>(l.y)
                       : static_cast<double>(h.x) + static_cast<double>(l.x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum[v] += __shfl_xor_sync(0xffffffffu, sum[v], o);
    inv_sum[v] = 1.0 / sum[v];
    inv_f[v] = static_cast<float>(inv_sum[v]);
    if (lane == 0) wsum[v] = sum[v];
    // requant level q >= 1 needs p16 * smax >= 0.5, i.e. p > 0.4998 / smax, i.e.
    // x - max > ln(0.4998 * sum / smax); below the (10 % lower) threshold q is exactly 0
    thr[v] = mxf[v] + static_cast<float>(log(0.45 * sum[v] / static_cast<double>(smax)));
  }
  // requant level of score x in row v (attention.py:127, :157-162)
  auto level = [&](float xf, int v) -> int32_t {
    if constexpr (FAST) {
      const float e = att_exp_fast(xf, mneg[v]);
      int q = prob_q_fast(e, inv_f[v], smax_f);
      if (q < 0) {  // rare: the float64 chain with the row sum kept in shared memory
        uint16_t pf;
        const double sv = wsum[v];
        prob_requant(static_cast<double>(e), sv, 1.0 / sv, smax, pf, q);
      }
      return q;
    } else {
      int32_t q = 0;
      if (xf >= thr[v]) {
        uint16_t pf;
        prob_requant(exp(static_cast<double>(xf) - mx[v]), sum[v], inv_sum[v], smax, pf, q);
      }
      return q;
    }
  };
  // levels of rows 2p, 2p+1 of one block as bytes (FAST, smax <= 2047): packed fp32 pairs;
  // the level is the low byte of fl(p16 * smax + 1.5 * 2^23) (exact: p16 * smax has <= 22 bits)
  auto level_pair = [&](__half2 x2, int p, uint32_t& qa, uint32_t& qb) {
    const float2 x = __half22float2(x2);
    const float pa = att_exp_fast(x.x, mneg[2 * p]) * inv_f[2 * p];
    const float pb = att_exp_fast(x.y, mneg[2 * p + 1]) * inv_f[2 * p + 1];
    const __half2 l = __floats2half2_rn(pa * 0.99999952316284180f, pb * 0.99999952316284180f);
    const __half2 h = __floats2half2_rn(pa * 1.00000047683715820f, pb * 1.00000047683715820f);
    const float2 fl = __half22float2(l);
    qa = __float_as_uint(fmaf(fl.x, smax_f, 12582912.0f));
    qb = __float_as_uint(fmaf(fl.y, smax_f, 12582912.0f));
    if (*reinterpret_cast<const uint32_t*>(&l) != *reinterpret_cast<const uint32_t*>(&h)) {
      qa = static_cast<uint32_t>(level(x.x, 2 * p));
      qb = static_cast<uint32_t>(level(x.y, 2 * p + 1));
    }
  };
  if constexpr (MIX) {
    // pass 3 + P x V: per chunk, the int8 probabilities go to pm[v][j]; then k-steps of
    // 32 blocks: V rows col_j (64 B each) gathered into slot order, D^T[n, v] += V^T P^T
    // (mma.sync m16n8k32: M = 16 head dims per MMA, 4 per k-step; N = 8 query rows)
    const uint8_t* vbl = reinterpret_cast<const uint8_t*>(vw + b * head_words) + (lane & 3) * 16;
    const uint32_t vring_s = smem_u32(vring);
    // gathered V row kk of a k-step sits in slot kk (64 bytes), its 16-byte chunk c (head
    // dims 16c..16c+15) at c ^ ((kk >> 1) & 3): the copies (8 lanes = 2 rows x 4 chunks) and
    // the ldmatrix phases (8 rows, one chunk) both hit 8 distinct bank groups. This lane
    // copies chunk lane & 3 of rows lane / 4 + 8u, i.e. at goff + 512 u.
    const uint32_t goff = 64 * (lane >> 2) + (((lane & 3) ^ ((lane >> 3) & 3)) << 4);
    // this lane's ldmatrix row (k = lane) of a slot; chunk c at c ^ ((lane >> 1) & 3)
    const uint32_t loff = 64 * lane;
    const int lsw = (lane >> 1) & 3;
    int acc[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[q][e] = 0;
    for (int64_t j0 = 0; j0 < nb; j0 += kCap) {
      const int jn = static_cast<int>(nb - j0 < kCap ? nb - j0 : kCap);
      if (!cached) { __syncwarp(); compute(j0, jn); }
      const int jpad = (jn + 31) & ~31;
      // gather of k-step s into ring slot s & 1: copy u of this lane moves 16-byte chunk
      // ch = lane & 3 of gathered row kk = lane / 4 + 8u. The column padding of ix (column 0)
      // pairs with P = 0, so the copies are unconditional.
      auto gather = [&](int s) {
        const uint32_t base = vring_s + (s & 1) * 2048;
        const uint32_t* ixs = ix + 32 * s + (lane >> 2);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          cp_async16_full(base + goff + 512 * u, vbl + static_cast<size_t>(ixs[8 * u]) * 64);
        cp_async_commit();
      };
      const int nsteps = jpad >> 5;
      gather(0);
      for (int s_ = 0; s_ < nsteps; ++s_) {
        if (s_ + 1 < nsteps) gather(s_ + 1);
        // pass 3 for the k-step's blocks (overlaps the gathers): levels of block 32 s + lane
        {
          const int j = 32 * s_ + lane;
          uint32_t qb[8];
#pragma unroll
          for (int v = 0; v < 8; ++v) qb[v] = 0;
          if (j < jn) {
            const uint4 u = *reinterpret_cast<const uint4*>(sc + j * 8);
            const __half2* hs = reinterpret_cast<const __half2*>(&u);
#pragma unroll
            for (int p = 0; p < 4; ++p) level_pair(hs[p], p, qb[2 * p], qb[2 * p + 1]);
          }
#pragma unroll
          for (int v = 0; v < 8; ++v) pm[v * 32 + lane] = static_cast<int8_t>(qb[v]);
        }
        if (s_ + 1 < nsteps) cp_async_wait<1>();
        else cp_async_wait<0>();
        __syncwarp();
        const uint32_t sbs = vring_s + (s_ & 1) * 2048 + loff;
        // B operand: P[g][32 s + 16 h + 4 t .. +3]
        uint32_t bf[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) bf[h] = *reinterpret_cast<const uint32_t*>(pm + g * 32 + 16 * h + 4 * t);
        // A operand: one ldmatrix.m16n16.x2.trans per 16 head dims -- the k-major fragment of
        // V^T (m = g <-> dim 16c + g, m = g + 8 <-> dim 16c + g + 8), no register transposes
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t a[4];
          ldsm_t16x2(sbs + ((c ^ lsw) << 4), a[0], a[1], a[2], a[3]);
          mma16832<false, false>(acc[c], a[0], a[1], a[2], a[3], bf[0], bf[1]);
        }
        __syncwarp();
      }
    }
    // epilogue: fp16(mix * alpha_m) (attention.py:169-176); acc[c]: (dim 16c+g, v 2t),
    // (16c+g, 2t+1), (16c+g+8, 2t), (16c+g+8, 2t+1)
    const double am = alpha_m[b];
    const float am_f = static_cast<float>(am);
#pragma unroll
    for (int vv = 0; vv < 2; ++vv) {
      const int v = 2 * t + vv;
      uint16_t* o = out_f16 + (b * L + r * 8 + v) * 64 + g;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        o[16 * c] = f16_dequant(acc[c][vv], am, am_f);
        o[16 * c + 8] = f16_dequant(acc[c][2 + vv], am, am_f);
      }
    }
    return;
  }
  // pass 3: requantised probabilities into the SR-BCRS values (:157-162); only the few
  // elements above the threshold evaluate exp and the fp16 rounding chain
  const int64_t sbeg = sr_begin[r];
  const int64_t stored = ((nb + S - 1) / S) * S;
  uint8_t* sv8 = reinterpret_cast<uint8_t*>(sr_vals + b * sr_stride_words);
  uint16_t* sv16 = reinterpret_cast<uint16_t*>(sr_vals + b * sr_stride_words);
  for (int64_t j0 = 0; j0 < stored; j0 += kCap) {
    const int jn = static_cast<int>(nb - j0 < kCap ? (nb - j0 > 0 ? nb - j0 : 0) : kCap);
    const int jst = static_cast<int>(stored - j0 < kCap ? stored - j0 : kCap);
    if (!cached && jn > 0) { __syncwarp(); compute(j0, jn); }
    for (int j = lane; j < jst; j += 32) {
      const int64_t pos = sbeg + j0 + j;
      const int64_t s_ = pos / S, jj = pos - s_ * S;
      int32_t qv[8];
      if (j < jn) {
        const uint4 u = *reinterpret_cast<const uint4*>(sc + j * 8);
        const __half* hs = reinterpret_cast<const __half*>(&u);
#pragma unroll
        for (int v = 0; v < 8; ++v) qv[v] = level(__half2float(hs[v]), v);
      } else {
#pragma unroll
        for (int v = 0; v < 8; ++v) qv[v] = 0;
      }
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int64_t el = s_ * 8 * S + static_cast<int64_t>(v) * S + jj;
        if (sbits == 8) sv8[el] = static_cast<uint8_t>(qv[v]);
        else sv16[el] = static_cast<uint16_t>(qv[v]);
      }
    }
  }
}

size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

}  // namespace

cudaError_t launch_attention(const mc_attention_args* a, uint32_t* status, cudaStream_t stream, size_t* ws_needed) {
  const int64_t B = a->batch, L = a->seq_len, d = a->head_dim;
  const int sb = a->softmax_bits, qb = a->qkv_bits;
  const int S = (sb % 8 == 0 && qb % 8 == 0) ? 16 : 32;  // plan(sb, qb).tile.k (attention.py:164-165)
  const int64_t vrows = L / 8;
  const int64_t nblk = a->mask->n_blocks;
  const int64_t n = L * d;
  const int64_t qwords = (n * qb + 31) / 32;
  const int64_t max_stored = nblk + vrows * (S - 1);
  const int64_t sr_words = (max_stored * 8 * sb + 31) / 32;

  size_t off = 0;
  const size_t o_qkv = off; off = align256(off + 3 * B * qwords * 4);
  const size_t o_scales = off; off = align256(off + B * 4 * 8);
  const size_t o_alpha = off; off = align256(off + B * 2 * 8);
  const size_t o_scores = off; off = align256(off + B * nblk * 8 * 2);
  const size_t o_begin = off; off = align256(off + vrows * 8);
  const size_t o_end = off; off = align256(off + vrows * 8);
  const size_t o_total = off; off = align256(off + 8);
  const size_t o_idx = off; off = align256(off + max_stored * 4);
  const size_t o_idx2 = off; off = align256(off + max_stored * 4);
  const size_t o_sr = off; off = align256(off + B * sr_words * 4);
  const size_t o_amax = off; off = align256(off + B * 3 * 4);
  if (ws_needed) *ws_needed = off;
  if (!a->workspace) return cudaSuccess;

  uint8_t* ws = static_cast<uint8_t*>(a->workspace);
  uint32_t* qkv = reinterpret_cast<uint32_t*>(ws + o_qkv);
  double* scales = a->scales ? a->scales : reinterpret_cast<double*>(ws + o_scales);
  double* alpha_s = reinterpret_cast<double*>(ws + o_alpha);
  double* alpha_m = alpha_s + B;
  uint16_t* scores = a->scores_f16 ? a->scores_f16 : reinterpret_cast<uint16_t*>(ws + o_scores);
  int64_t* sr_begin = reinterpret_cast<int64_t*>(ws + o_begin);
  int64_t* sr_end = reinterpret_cast<int64_t*>(ws + o_end);
  int64_t* sr_total = reinterpret_cast<int64_t*>(ws + o_total);
  uint32_t* sr_idx = reinterpret_cast<uint32_t*>(ws + o_idx);
  uint32_t* sr_idx2 = reinterpret_cast<uint32_t*>(ws + o_idx2);
  uint32_t* sr_vals = reinterpret_cast<uint32_t*>(ws + o_sr);
  cudaError_t err;

  const int smax = (1 << (sb - 1)) - 1;
  const bool fast = a->mode == MC_ATTN_FAST;
  if (a->in_dtype == MC_DTYPE_F16 && qb == 8 && n % 16 == 0 && (reinterpret_cast<uintptr_t>(a->q) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(a->k) & 15) == 0 && (reinterpret_cast<uintptr_t>(a->v) & 15) == 0) {
    // vectorised fp16 path: one kernel (absmax, scale, 16-wide quant, alphas) per tensor
    uint32_t* arrivals = reinterpret_cast<uint32_t*>(ws + o_amax);
    cudaMemsetAsync(arrivals, 0, B * 4, stream);
    auto kq = fast ? absquant_f16_kernel<true> : absquant_f16_kernel<false>;
    cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, kQuantSmem);
    kq<<<dim3(static_cast<unsigned>(B * kQuantCluster), 3), kQuantThreads, kQuantSmem, stream>>>(
        static_cast<const __half*>(a->q), static_cast<const __half*>(a->k), static_cast<const __half*>(a->v), n, smax,
        a->head_dim, scales, alpha_s, alpha_m, qkv, qwords, B, arrivals);
    count_launch();
  } else {
    absmax_kernel<<<dim3(static_cast<unsigned>(B), 3), 512, 0, stream>>>(a->q, a->k, a->v, a->in_dtype, n, qb,
                                                                         scales, smax);
    count_launch();
    quant_kernel<<<dim3(static_cast<unsigned>((B * qwords + 255) / 256), 3), 256, 0, stream>>>(
        a->q, a->k, a->v, a->in_dtype, n, qb, scales, qkv, qwords, B);
    count_launch();
    alpha_kernel<<<static_cast<unsigned>((B + 127) / 128), 128, 0, stream>>>(scales, B, a->head_dim, alpha_s, alpha_m);
    count_launch();
  }

  const bool fused = qb == 8 && d == 64 && !a->scores_int && !a->scores_f16 && !a->probs_f16 && !a->probs_int &&
                     !getenv("MCUBE_ATTN_UNFUSED");
  // whole layer in the fused kernel (P x V included) unless the int32 mix is requested
  const bool mix = fused && sb == 8 && !a->mix_int && a->out_f16 && !getenv("MCUBE_ATTN_NOMIX");
  if (mix) {
    const unsigned fgrid = static_cast<unsigned>((B * vrows + 3) / 4);
    const uint32_t* kq = qkv + B * qwords;
    const uint32_t* vq = qkv + 2 * B * qwords;
    const int smem = 4 * att_warp_smem<true>();
    auto kf = a->mode == MC_ATTN_FAST ? score_softmax_kernel<true, true> : score_softmax_kernel<false, true>;
    cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const cudaError_t e2 = launch_pdl(kf, dim3(fgrid), dim3(128), static_cast<size_t>(smem), stream, qkv, kq, qwords,
                                      a->mask->row_offsets, a->mask->col_indices, vrows, L, alpha_s,
                                      static_cast<const int64_t*>(nullptr), S, smax, sb, static_cast<uint32_t*>(nullptr),
                                      sr_words, B, status, vq, static_cast<const double*>(alpha_m), a->out_f16);
    count_launch();
    return e2;
  }

  // mask -> SR-BCRS structure of the probability matrix (stride = plan tile k)
  if ((err = launch_srbcrs_plan(a->mask->row_offsets, vrows, S, sr_begin, sr_end, sr_total, stream)) != cudaSuccess)
    return err;
  // column indices for the worst-case stored count; padding tail stays sentinel
  cudaMemsetAsync(sr_idx, 0xFF, max_stored * 4, stream);
  if ((err = launch_srbcrs_fill(a->mask->row_offsets, a->mask->col_indices, vrows, nblk, 8, S, sr_begin, sr_end,
                                max_stored, nullptr, 32, sr_idx, nullptr, stream)) != cudaSuccess)
    return err;
  const uint32_t* spmm_idx = sr_idx;
  if (qb == 4) {  // attention.py:166-167
    if ((err = launch_shuffle(sr_idx, max_stored, sr_idx2, stream)) != cudaSuccess) return err;
    spmm_idx = sr_idx2;
  }

  if (fused) {
    // score SDDMM + softmax + requant in one kernel (scores never leave the SM)
    const unsigned fgrid = static_cast<unsigned>((B * vrows + 3) / 4);
    const uint32_t* kq = qkv + B * qwords;
    const int smem = 4 * att_warp_smem<false>();
    auto kf = a->mode == MC_ATTN_FAST ? score_softmax_kernel<true, false> : score_softmax_kernel<false, false>;
    cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaError_t e2 = launch_pdl(kf, dim3(fgrid), dim3(128), static_cast<size_t>(smem), stream, qkv, kq, qwords,
                                a->mask->row_offsets, a->mask->col_indices, vrows, L, alpha_s,
                                static_cast<const int64_t*>(sr_begin), S, smax, sb, sr_vals, sr_words, B, status,
                                static_cast<const uint32_t*>(nullptr), static_cast<const double*>(nullptr),
                                static_cast<uint16_t*>(nullptr));
    count_launch();
    if (e2 != cudaSuccess) return e2;
  } else {
  SddmmParams sp{};
  sp.M = L; sp.K = d; sp.N = L; sp.vrows = vrows; sp.n_blocks = nblk;
  sp.V = 8; sp.LB = qb; sp.RB = qb; sp.batch = static_cast<int>(B);
  sp.a_words = qkv; sp.a_stride = qwords;
  sp.b_words = qkv + B * qwords; sp.b_stride = qwords;
  sp.row_offsets = a->mask->row_offsets; sp.col_indices = a->mask->col_indices;
  sp.out = a->scores_int; sp.out_stride = nblk * 8;
  sp.alpha = alpha_s; sp.out_f16 = scores; sp.f16_stride = nblk * 8;
  sp.status = status;
  if ((err = launch_sddmm(sp, stream)) != cudaSuccess) return err;

  const int64_t warps = B * vrows;
  const unsigned grid = static_cast<unsigned>((warps * 32 + 255) / 256);
  if (fast)
    softmax_requant_kernel<true><<<grid, 256, 0, stream>>>(scores, nblk * 8, a->mask->row_offsets, vrows, sr_begin, S,
                                                           smax, sb, sr_vals, sr_words, a->probs_f16, a->probs_int, B);
  else
    softmax_requant_kernel<false><<<grid, 256, 0, stream>>>(scores, nblk * 8, a->mask->row_offsets, vrows, sr_begin, S,
                                                            smax, sb, sr_vals, sr_words, a->probs_f16, a->probs_int, B);
  count_launch();
  }

  SpmmParams mp{};
  mp.M = L; mp.K = L; mp.N = d; mp.vrows = vrows;
  mp.V = 8; mp.S = S; mp.LB = sb; mp.RB = qb; mp.shuffled = qb == 4 ? 1 : 0; mp.batch = static_cast<int>(B);
  mp.row_begin = sr_begin; mp.row_end = sr_end; mp.col_indices = spmm_idx;
  mp.lhs_words = sr_vals; mp.lhs_stride = sr_words;
  mp.rhs_words = qkv + 2 * B * qwords; mp.rhs_stride = qwords;
  mp.out = a->mix_int; mp.out_stride = L * d;
  mp.alpha = alpha_m; mp.out_f16 = a->out_f16; mp.f16_stride = L * d;
  mp.status = status;
  return launch_spmm(mp, stream);
}

}  // namespace mcube
