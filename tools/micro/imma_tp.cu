// imma_tp.cu -- mma.sync m16n8k32 s8 x s8 -> s32 throughput per SM on sm_100a (the legacy
// integer tensor-core path the gather kernels use), W warps per CTA, 8 independent
// accumulators per warp. build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/imma_tp tools/micro/imma_tp.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void imma(int iters, unsigned long long* cycles, int* sink) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  int acc[8][4] = {};
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+r"(acc[j][0]), "+r"(acc[j][1]), "+r"(acc[j][2]), "+r"(acc[j][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  int x = 0;
  for (int j = 0; j < 8; ++j) x += acc[j][0] + acc[j][1] + acc[j][2] + acc[j][3];
  if (x == 0x12345) sink[threadIdx.x] = x;
}

int main() {
  unsigned long long* dcyc;
  int* sink;
  cudaMalloc(&dcyc, 148 * sizeof(unsigned long long));
  cudaMalloc(&sink, 1024 * sizeof(int));
  const int iters = 2048;
  for (int w : {4, 8, 16, 32}) {
    imma<<<148, 32 * w>>>(iters, dcyc, sink);
    imma<<<148, 32 * w>>>(iters, dcyc, sink);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, dcyc, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const double macs = static_cast<double>(w) * iters * 8 * 16 * 8 * 32;
    printf("{\"warps\": %d, \"mac_per_clk_per_sm\": %.0f, \"tops_at_1965mhz\": %.0f}\n", w, macs / avg,
           2.0 * macs / avg * 148 * 1.965e9 / 1e12);
  }
  return 0;
}
