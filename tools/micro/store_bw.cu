// Microbenchmark: per-SM global write bandwidth with STG.256 (8 consumer warps, contiguous
// 1 KB warp stores) vs cp.async.bulk shared->global, one CTA per SM, 1 MB per CTA (148 MB:
// larger than L2, so the rate includes the HBM write-back).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 1) stg_kernel(uint32_t* out, int per_cta_bytes) {
  uint32_t* o = out + (size_t)blockIdx.x * (per_cta_bytes / 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t v[8];
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 8 + i;
  for (int off = warp * 1024; off < per_cta_bytes; off += 8 * 1024) {
    uint32_t* p = o + off / 4 + lane * 8;
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
  }
}

__global__ void __launch_bounds__(256, 1) bulk_kernel(uint32_t* out, int per_cta_bytes, int chunk) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint32_t* o = out + (size_t)blockIdx.x * (per_cta_bytes / 4);
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    for (int off = 0; off < per_cta_bytes; off += chunk) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"((uint8_t*)o + off),
                   "r"(s + (off % 16384)), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int per = 1024 * 1024;
  uint32_t* out;
  cudaMalloc(&out, (size_t)sms * per);
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    cudaEventRecord(a);
    stg_kernel<<<sms, 256>>>(out, per);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("STG.256 : %.2f us, %.1f GB/s per SM, %.2f TB/s total\n", ms * 1e3, per / (ms * 1e-3) / 1e9,
           (double)sms * per / (ms * 1e-3) / 1e12);
    for (int chunk : {4096}) {
      cudaEventRecord(a);
      bulk_kernel<<<sms, 256, 16384>>>(out, per, chunk);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("bulk %4d: %.2f us, %.1f GB/s per SM, %.2f TB/s total\n", chunk, ms * 1e3, per / (ms * 1e-3) / 1e9,
             (double)sms * per / (ms * 1e-3) / 1e12);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
