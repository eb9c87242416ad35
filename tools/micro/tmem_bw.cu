// tmem_bw.cu -- TMEM -> register read throughput per SM (tcgen05.ld), the drain bound of the
// dense-tile SDDMM epilogue (sddmm_tc.cu). One CTA per SM, W warps (warp w reads lane quarter
// w & 3), each warp issues `depth` tcgen05.ld.32x32b.x32 (4 KB each) per tcgen05.wait::ld.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/tmem_bw tools/micro/tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

#define LD32(taddr, r)                                                                                       \
  asm volatile(                                                                                              \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"       \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                             \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),     \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),           \
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),           \
        "=r"(r[30]), "=r"(r[31])                                                                             \
      : "r"(taddr))

template <int DEPTH>
__global__ void tmem_read(int iters, unsigned long long* cycles, uint32_t* sink) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = holder + (static_cast<uint32_t>(32 * (warp & 3)) << 16);
  uint32_t x = 0;
  uint32_t r[DEPTH][32];
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) LD32(tmem + 32 * ((i * DEPTH + d + warp) & 15), r[d]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int d = 0; d < DEPTH; ++d)
#pragma unroll
      for (int j = 0; j < 32; ++j) x ^= r[d][j];
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (x == 0x12345678u) sink[threadIdx.x] = x;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(holder));
}

template <int DEPTH>
void run(int warps, int iters, unsigned long long* dcyc, uint32_t* sink) {
  tmem_read<DEPTH><<<148, 32 * warps>>>(iters, dcyc, sink);
  tmem_read<DEPTH><<<148, 32 * warps>>>(iters, dcyc, sink);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, dcyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double bytes = static_cast<double>(warps) * iters * DEPTH * 4096.0;
  printf("{\"warps\": %d, \"depth\": %d, \"bytes_per_sm\": %.0f, \"cycles\": %.0f, \"B_per_clk_per_sm\": %.1f}\n", warps,
         DEPTH, bytes, avg, bytes / avg);
}

int main() {
  unsigned long long* dcyc;
  uint32_t* sink;
  cudaMalloc(&dcyc, 148 * sizeof(unsigned long long));
  cudaMalloc(&sink, 1024 * sizeof(uint32_t));
  const int iters = 4096;
  for (int w : {4, 8, 16}) {
    run<1>(w, iters, dcyc, sink);
    run<2>(w, iters / 2, dcyc, sink);
    run<4>(w, iters / 4, dcyc, sink);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
