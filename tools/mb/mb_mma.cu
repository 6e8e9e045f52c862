// Microbenchmark: legacy mma.sync throughput on sm_100a (IMMA u8s8 m16n8k32, HMMA f16 m16n8k16).
#include <cstdio>
#include <cstdint>
template <int KIND>
__global__ void k(int* out, int iters, uint32_t seed) {
  int acc[8][4] = {};
  float facc[8][4] = {};
  uint32_t a = seed ^ threadIdx.x, b = seed * 3u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (KIND == 0)
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(acc[c][0]), "+r"(acc[c][1]), "+r"(acc[c][2]), "+r"(acc[c][3])
                     : "r"(a), "r"(a + 1), "r"(a + 2), "r"(a + 3), "r"(b), "r"(b + 1));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(facc[c][0]), "+f"(facc[c][1]), "+f"(facc[c][2]), "+f"(facc[c][3])
                     : "r"(a), "r"(a + 1), "r"(a + 2), "r"(a + 3), "r"(b), "r"(b + 1));
    }
  }
  int s = 0;
  for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3] + (int)facc[c][0];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int kind = 0; kind < 2; ++kind)
    for (int warps = 4; warps <= 32; warps *= 2) {
      const int iters = 4096;
      auto fn = kind == 0 ? k<0> : k<1>;
      fn<<<sms, warps * 32>>>(out, 16, 1);
      cudaEventRecord(e0);
      fn<<<sms, warps * 32>>>(out, iters, 1);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double mmas = (double)sms * warps * iters * 8;
      printf("%s warps/SM=%d: %.3f ms, %.2f mma/clk/SM @1.965GHz, %.1f Tops\n", kind ? "HMMA16816" : "IMMA16832", warps, ms,
             mmas / sms / (ms * 1e-3 * 1.965e9), mmas * (kind ? 4096.0 : 8192.0) / (ms * 1e-3) / 1e12);
    }
  return 0;
}
