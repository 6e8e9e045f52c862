// Microbenchmark: mma.sync b1 (m16n8k256 and.popc) vs int8 (m16n8k32) throughput on sm_100a. Measured on
// B200: b1 has no BMMA in the SASS (emulated): 0.02 mma/clk/SM; IMMA.16832 0.49 mma/clk/SM. So a
// bit-plane formulation of the binary scan is not viable.
#include <cstdio>
#include <cstdint>
__global__ void probe_b1(uint32_t* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x55, b1 = a0 ^ 0x33;
  int c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[k][0]), "+r"(c[k][1]), "+r"(c[k][2]), "+r"(c[k][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0 + k), "r"(b1));
  }
  int s = 0;
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void probe_i8(uint32_t* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x55, b1 = a0 ^ 0x33;
  int c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[k][0]), "+r"(c[k][1]), "+r"(c[k][2]), "+r"(c[k][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0 + k), "r"(b1));
  }
  int s = 0;
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  uint32_t* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    for (int w = 4; w <= 16; w *= 2) {
      probe_b1<<<148 * 2, 32 * w>>>(out, 16); cudaEventRecord(e0);
      probe_b1<<<148 * 2, 32 * w>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double mmas = 148.0 * 2 * w * iters * 8;
      printf("b1  warps/CTA %2d: %.3f ms, %.2f mma/clk/SM (at 1.9 GHz), %.1f Tbitop/s\n", w, ms, mmas / (ms * 1e-3) / 148 / 1.9e9,
             mmas * 16 * 8 * 256 * 2 / (ms * 1e-3) / 1e12);
      probe_i8<<<148 * 2, 32 * w>>>(out, 16); cudaEventRecord(e0);
      probe_i8<<<148 * 2, 32 * w>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("i8  warps/CTA %2d: %.3f ms, %.2f mma/clk/SM (at 1.9 GHz), %.1f TOPS\n", w, ms, mmas / (ms * 1e-3) / 148 / 1.9e9,
             mmas * 16 * 8 * 32 * 2 / (ms * 1e-3) / 1e12);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
