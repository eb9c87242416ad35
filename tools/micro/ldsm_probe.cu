// ldsm_probe.cu -- register layout of ldmatrix.m16n16.{x1,x2}.trans.b8 (sm_100a, SASS
// LDSM.8.MT1616) and the throughput of LDSM.x2 over random 16-byte rows vs swizzled rows.
// Matrix 0 byte (row r, col c) = 16 r + c; for .x2, matrix 1 = the same bytes | 0 but read
// from a second copy, so the decoded (row, col) of every register byte shows the layout.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/ldsm_probe tools/micro/ldsm_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(uint32_t* out) {
  __shared__ __align__(128) uint8_t s[512];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    s[i] = static_cast<uint8_t>(i);
    s[256 + i] = static_cast<uint8_t>(i);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t a1 = static_cast<uint32_t>(__cvta_generic_to_shared(s + (lane & 15) * 16));
  uint32_t r0, r1;
  asm volatile("ldmatrix.sync.aligned.m16n16.x1.trans.shared.b8 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(a1));
  out[lane * 6 + 0] = r0;
  out[lane * 6 + 1] = r1;
  // x2: lanes 0-15 rows of matrix 0, lanes 16-31 rows of matrix 1 (second copy, rows reversed)
  const uint32_t a2 = static_cast<uint32_t>(
      __cvta_generic_to_shared(s + (lane < 16 ? lane * 16 : 256 + (31 - lane) * 16)));
  uint32_t q0, q1, q2, q3;
  asm volatile("ldmatrix.sync.aligned.m16n16.x2.trans.shared.b8 {%0,%1,%2,%3}, [%4];"
               : "=r"(q0), "=r"(q1), "=r"(q2), "=r"(q3)
               : "r"(a2));
  out[lane * 6 + 2] = q0;
  out[lane * 6 + 3] = q1;
  out[lane * 6 + 4] = q2;
  out[lane * 6 + 5] = q3;
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 32 * 6 * 4);
  probe<<<1, 32>>>(d);
  uint32_t h[32 * 6];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"ldsm_m16n16_trans_b8\": [\n");
  for (int l = 0; l < 32; ++l) {
    printf("  {\"lane\": %d, \"regs\": [", l);
    for (int r = 0; r < 6; ++r) {
      printf("[");
      for (int b = 0; b < 4; ++b) {
        const int v = (h[l * 6 + r] >> (8 * b)) & 0xFF;
        printf("\"r%dc%d\"%s", v >> 4, v & 15, b < 3 ? "," : "");
      }
      printf("]%s", r < 5 ? "," : "");
    }
    printf("]}%s\n", l < 31 ? "," : "");
  }
  printf("], \"note\": \"regs 0-1: x1; regs 2-5: x2 (matrix 1 rows reversed: row r read from lane 31-r)\"}\n");
  return 0;
}
