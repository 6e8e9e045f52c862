// otf_binary.cu — K4 binary-code scoring (score_binary, ranker.py:78-94), unpack_bits
// (binary.py:110-120), binarize (binary.py:86-107) and Hamming distance (binary.py:123-128).
//
// Scoring: s_i = float32( sum_{j < n_bits, bit j set} float32(w_j) ), bit j = byte j/8,
// bit j%8 (LSB first); padding bits are ignored (the reference unpacks with
// count=output_bits). Instead of unpacking 2048 bits to floats (the reference's 32x
// expansion) each 4-bit nibble indexes a 16-entry float64 table T_p[v] = sum of the
// float32 weights of the set bits of v (added in bit order, exact in float64 for any
// realistic weight range). The tables live in shared memory laid out so that every lane of
// a half-warp reads its own bank pair (conflict-free); the per-row sum uses a fixed lane
// tree (as in otf_dense.cu), so a row's score does not depend on its position.
//
// HBM roofline: n_bits/8 bytes per row (256 B for 2048-bit codes). The nibble lookups
// (512 per 2048-bit row) make this kernel shared-memory bound at ~35% of HBM.
#include "otf_common.cuh"
#include "otf_internal.h"

namespace otf {

// Table layout for the fast path: codes are read as 16-byte chunks; lane l of a 16-lane
// group owns chunks {l + 16*t}. Nibble i (0..31) of chunk c has value v; its table entry
// T[c][i][v] is stored at double index ((t*32 + i)*16 + v)*16 + (c % 16), with t = c/16,
// so the 16 lanes of a half-warp always hit 16 distinct bank pairs.
__device__ __forceinline__ double nibble_entry(const double* __restrict__ w, int n_bits, int e,
                                               int* slot) {
  const int v = e & 15;
  const int i = (e >> 4) & 31;
  const int c = e >> 9;
  const int bit0 = c * 128 + i * 4;
  double s = 0.0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int j = bit0 + b;
    if ((v >> b) & 1) s = __dadd_rn(s, j < n_bits ? (double)__double2float_rn(w[j]) : 0.0);
  }
  const int t = c >> 4, lane = c & 15;
  *slot = ((t * 32 + i) * 16 + v) * 16 + lane;
  return s;
}

// Fast path: row bytes == 16 * CH (CH chunks of 16 bytes, CH % 16 == 0), R rows per group
// per iteration; 2 groups (half-warps) per warp. The nibble tables are built per CTA from w.
template <int CH, int R>
__global__ void __launch_bounds__(256) bin_score_fast(const uint8_t* __restrict__ codes, int64_t n,
                                                      const double* __restrict__ w, int n_bits,
                                                      float* __restrict__ out,
                                                      uint32_t* __restrict__ ghist) {
  constexpr int TPL = CH / 16;  // chunks per lane
  extern __shared__ double lut[];  // CH*32*16 doubles
  __shared__ uint32_t sh[kHistBins];
  for (int e = threadIdx.x; e < CH * 32 * 16; e += blockDim.x) {
    int slot;
    const double v = nibble_entry(w, n_bits, e, &slot);
    lut[slot] = v;
  }
  if (ghist) hist_zero(sh);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int cl = lane & 15;    // chunk lane
  const int grp = lane >> 4;   // row group within the warp
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint4* C4 = reinterpret_cast<const uint4*>(codes);
  for (int64_t r0 = warp * (2 * R); r0 < n; r0 += nwarp * (2 * R)) {
    uint4 v[R][TPL];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int64_t row = r0 + grp * R + i;
#pragma unroll
      for (int t = 0; t < TPL; ++t) {
        if (row < n) v[i][t] = ld_stream_u4(C4 + row * CH + cl + 16 * t);
        else v[i][t] = make_uint4(0, 0, 0, 0);
      }
    }
    double p[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t < TPL; ++t) {
        const uint32_t words[4] = {v[i][t].x, v[i][t].y, v[i][t].z, v[i][t].w};
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const uint32_t nib = (words[q >> 3] >> (4 * (q & 7))) & 15u;
          acc = __dadd_rn(acc, lut[((t * 32 + q) * 16 + nib) * 16 + cl]);
        }
      }
      p[i] = acc;
    }
    transposed_reduce<R, 16>(p, lane);
    bool writer;
    const int slot = row_of_lane<R, 16>(lane, &writer);
    const int64_t row = r0 + grp * R + slot;
    const bool active = writer && row < n;
    const float s = __double2float_rn(p[0]);
    if (active) out[row] = s;
    if (ghist) hist_add(sh, active, hist_bin(s));
  }
  if (ghist) {
    __syncthreads();
    hist_flush(sh, ghist);
  }
}

// Generic path: any n_bits. One warp per row; lane l owns bytes {l + 32*t}, bits in order;
// float32(w_j) converted on the fly.
__global__ void __launch_bounds__(256) bin_score_generic(const uint8_t* __restrict__ codes, int64_t n,
                                                         int n_bits, int row_bytes,
                                                         const double* __restrict__ w,
                                                         float* __restrict__ out,
                                                         uint32_t* __restrict__ ghist) {
  __shared__ uint32_t sh[kHistBins];
  if (ghist) hist_zero(sh);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = warp; row < n; row += nwarp) {
    const uint8_t* c = codes + row * row_bytes;
    double acc = 0.0;
    for (int b = lane; b < row_bytes; b += 32) {
      const uint32_t byte = c[b];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = 8 * b + q;
        if (((byte >> q) & 1u) && j < n_bits) acc = __dadd_rn(acc, (double)__double2float_rn(w[j]));
      }
    }
    double p[1] = {acc};
    transposed_reduce<1, 32>(p, lane);
    const float s = __double2float_rn(p[0]);
    if (lane == 0) out[row] = s;
    if (ghist) hist_add(sh, lane == 0, hist_bin(s));
  }
  if (ghist) {
    __syncthreads();
    hist_flush(sh, ghist);
  }
}

// unpack_bits: out[r, j] = bit j of row r as float32 {0, 1}.
__global__ void bin_unpack(const uint8_t* __restrict__ codes, int64_t n, int n_bits, int row_bytes,
                           float* __restrict__ out) {
  const int64_t total = n * (int64_t)n_bits;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t r = e / n_bits;
    const int j = (int)(e - r * n_bits);
    out[e] = (float)((codes[r * row_bytes + (j >> 3)] >> (j & 7)) & 1u);
  }
}

// binarize: bit j of row r = ((x_r - mu) . U_j) > 0 in float64, packed LSB-first.
// One warp per (row, byte): lane q<8 computes bit 8*byte+q with a serial float64 dot in
// column order (numpy's dgemm order differs; exact-zero / sub-ulp ties can flip — tolerance).
__global__ void bin_binarize(const double* __restrict__ U, const float* __restrict__ mu, int m,
                             int n_bits, const double* __restrict__ X, int64_t n,
                             uint8_t* __restrict__ out) {
  const int row_bytes = (n_bits + 7) >> 3;
  const int64_t total = n * (int64_t)row_bytes * 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;  // multiple of 32
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e - (threadIdx.x & 31) < total;
       e += stride) {
    const bool valid = e < total;
    const int64_t r = valid ? e / ((int64_t)row_bytes * 8) : 0;
    const int j = valid ? (int)(e - r * (int64_t)row_bytes * 8) : 0;
    int bit = 0;
    if (valid && j < n_bits) {
      const double* x = X + r * m;
      const double* u = U + (int64_t)j * m;
      double acc = 0.0;
      for (int q = 0; q < m; ++q) acc = __fma_rn(__dsub_rn(x[q], (double)mu[q]), u[q], acc);
      bit = acc > 0.0;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, bit);
    // lanes 0,8,16,24 of each warp own one output byte each (e is warp-aligned below)
    if ((threadIdx.x & 7) == 0 && valid) {
      const int sh = threadIdx.x & 31;
      out[r * row_bytes + (j >> 3)] = (uint8_t)((mask >> sh) & 0xffu);
    }
  }
}

__global__ void bin_hamming(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, int64_t n,
                            int width, int64_t* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    int64_t d = 0;
    for (int q = 0; q < width; ++q) d += __popc((uint32_t)(a[r * width + q] ^ b[r * width + q]));
    out[r] = d;
  }
}

size_t bin_lut_bytes(int n_bits) {
  const int row_bytes = (n_bits + 7) / 8;
  if (row_bytes % 256 != 0 || row_bytes > 512) return 0;  // fast path: CH in {16, 32}
  return (size_t)(row_bytes / 16) * 32 * 16 * sizeof(double);
}

template <int CH, int R>
static int launch_fast(const uint8_t* codes, int64_t n, const double* w, int n_bits, float* out,
                       uint32_t* hist, int device, cudaStream_t st) {
  auto fn = bin_score_fast<CH, R>;
  const size_t smem = (size_t)CH * 32 * 16 * sizeof(double);
  static bool configured[64] = {false};
  if (!configured[device & 63]) {
    cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured[device & 63] = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)per_sm * sm_count(device);
  const int64_t need = (n + 16 * R - 1) / (16 * R);
  if (need < grid) grid = need;
  fn<<<(int)grid, 256, smem, st>>>(codes, n, w, n_bits, out, hist);
  OTF_LAUNCH_CHECK("bin_score_fast");
  return OTF_OK;
}

// w: float64 model (device); cast to float32 in-kernel (ranker.py:89). hist: see dense.
int launch_bin_score(const uint8_t* codes, int64_t n, int n_bits, const double* w, float* out,
                     uint32_t* hist, int device, cudaStream_t st) {
  if (n <= 0) return OTF_OK;
  const int row_bytes = (n_bits + 7) / 8;
  const bool aligned = (((uintptr_t)codes) & 15) == 0;
  if (aligned && bin_lut_bytes(n_bits) > 0) {
    if (row_bytes == 256) return launch_fast<16, 8>(codes, n, w, n_bits, out, hist, device, st);
    if (row_bytes == 512) return launch_fast<32, 4>(codes, n, w, n_bits, out, hist, device, st);
  }
  int64_t grid = (n + 7) / 8;
  const int64_t cap = 8LL * sm_count(device);
  if (grid > cap) grid = cap;
  bin_score_generic<<<(int)grid, 256, 0, st>>>(codes, n, n_bits, row_bytes, w, out, hist);
  OTF_LAUNCH_CHECK("bin_score_generic");
  return OTF_OK;
}

int launch_bin_unpack(const uint8_t* codes, int64_t n, int n_bits, float* out, int device,
                      cudaStream_t st) {
  const int64_t total = n * (int64_t)n_bits;
  if (total <= 0) return OTF_OK;
  int64_t grid = (total + 255) / 256;
  const int64_t cap = 16LL * sm_count(device);
  if (grid > cap) grid = cap;
  bin_unpack<<<(int)grid, 256, 0, st>>>(codes, n, n_bits, (n_bits + 7) / 8, out);
  OTF_LAUNCH_CHECK("bin_unpack");
  return OTF_OK;
}

int launch_binarize(const double* U, const float* mu, int m, int n_bits, const double* X,
                    int64_t n, uint8_t* out, int device, cudaStream_t st) {
  const int row_bytes = (n_bits + 7) >> 3;
  const int64_t total = n * (int64_t)row_bytes * 8;
  if (total <= 0) return OTF_OK;
  // total is a multiple of 8; use a block size multiple of 32 and keep grid-stride
  // iterations warp-aligned so the ballot covers whole bytes.
  int64_t grid = (total + 255) / 256;
  const int64_t cap = 16LL * sm_count(device);
  if (grid > cap) grid = cap;
  bin_binarize<<<(int)grid, 256, 0, st>>>(U, mu, m, n_bits, X, n, out);
  OTF_LAUNCH_CHECK("bin_binarize");
  return OTF_OK;
}

int launch_hamming(const uint8_t* a, const uint8_t* b, int64_t n, int width, int64_t* out,
                   int device, cudaStream_t st) {
  if (n <= 0) return OTF_OK;
  int64_t grid = (n + 255) / 256;
  const int64_t cap = 8LL * sm_count(device);
  if (grid > cap) grid = cap;
  bin_hamming<<<(int)grid, 256, 0, st>>>(a, b, n, width, out);
  OTF_LAUNCH_CHECK("bin_hamming");
  return OTF_OK;
}

}  // namespace otf
