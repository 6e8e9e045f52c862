// otf_pq.cu — K2/K3: product-quantized scoring (score_pq, ranker.py:72-75;
// build_score_lut pq.py:248-259; score_codes pq.py:262-276).
//
// Bit-exact with the reference's numpy arithmetic:
//  * LUT[m][j] = einsum("mkq,mq->mk") in float64 with the FULL float64 w (no float32 cast,
//    pq.py:255). numpy's einsum inner kernel (SSE2, two lanes, no FMA) multiplies each
//    c*w term separately and adds them into two accumulators in a fixed pattern:
//    each 8-block contributes p6,p4,p2,p0 to acc0 and p7,p5,p3,p1 to acc1; the tail adds
//    pairs (even->acc0, odd->acc1) and a final odd element to acc0; result 0.0+(acc0+acc1).
//    Restated (and pinned against numpy) in oracle/otf_oracle.py::lut_entry_numpy_order.
//  * s_i = lut[cols, codes[i]].sum(axis=1): numpy pairwise summation over the M entries
//    (n<8: sequential from -0.0; 8<=n<=128: 8 strided accumulators, tree, sequential tail;
//    n>128: split at n/2 rounded down to a multiple of 8). Restated in
//    oracle/otf_oracle.py::pairwise_sum_numpy_order.
// __dmul_rn/__dadd_rn keep nvcc from contracting into FMAs.
//
// HBM roofline: M bytes per row (16 B for C3). The LUT (M*256*8 B) lives in shared memory;
// the scan is shared-memory-lookup bound for M=16.
#include <algorithm>
#include <cstdlib>

#include "otf_common.cuh"
#include "otf_internal.h"
#include "otf_topk_dev.cuh"
#include "otf_pairwise.cuh"

namespace otf {

__device__ __forceinline__ double lut_entry_einsum(const float* __restrict__ c,
                                                   const double* __restrict__ w, int Q) {
  double acc0 = 0.0, acc1 = 0.0;
  int i = 0;
  for (; Q - i >= 8; i += 8) {
    acc0 = __dadd_rn(acc0, __dmul_rn((double)c[i + 6], w[i + 6]));
    acc1 = __dadd_rn(acc1, __dmul_rn((double)c[i + 7], w[i + 7]));
    acc0 = __dadd_rn(acc0, __dmul_rn((double)c[i + 4], w[i + 4]));
    acc1 = __dadd_rn(acc1, __dmul_rn((double)c[i + 5], w[i + 5]));
    acc0 = __dadd_rn(acc0, __dmul_rn((double)c[i + 2], w[i + 2]));
    acc1 = __dadd_rn(acc1, __dmul_rn((double)c[i + 3], w[i + 3]));
    acc0 = __dadd_rn(acc0, __dmul_rn((double)c[i + 0], w[i + 0]));
    acc1 = __dadd_rn(acc1, __dmul_rn((double)c[i + 1], w[i + 1]));
  }
  for (; Q - i >= 2; i += 2) {
    acc0 = __dadd_rn(acc0, __dmul_rn((double)c[i], w[i]));
    acc1 = __dadd_rn(acc1, __dmul_rn((double)c[i + 1], w[i + 1]));
  }
  if (i < Q) acc0 = __dadd_rn(acc0, __dmul_rn((double)c[i], w[i]));
  return __dadd_rn(0.0, __dadd_rn(acc0, acc1));
}

// lut is (M, K) row-major float64 (the reference's layout).
// replicas > 1: copies r = 1.. at lut + r * M * K (the cut path's CTAs each read one copy, so
// 148 SMs do not all hit the same 32 KB of L2 at once)
__global__ void pq_build_lut_kernel(const float* __restrict__ cents, int M, int K, int Q,
                                    const double* __restrict__ w, double* __restrict__ lut, int replicas) {
  // the dependent scan (programmatic launch) may start its own setup now
  asm volatile("griddepcontrol.launch_dependents;");
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= M * K) return;
  const int m = t / K;
  const double v = lut_entry_einsum(cents + (int64_t)t * Q, w + (int64_t)m * Q, Q);
  for (int r = 0; r < replicas; ++r) lut[(int64_t)r * M * K + t] = v;
}

struct GlobalLut {
  const double* lut; int K; const uint8_t* code;
  __device__ __forceinline__ double operator()(int m) const { return lut[m * K + code[m]]; }
};

// Fast path, compile-time M (M in {4, 8, 16, 32}): one thread per row, codes loaded as
// vectors, the LUT (M x 256 float64, zero padded beyond K) built per CTA in shared memory
// straight from the centroids and the float64 w (no separate LUT launch), and the coarse
// score histogram for the top-k kernel accumulated on the fly.
template <int M>
__global__ void __launch_bounds__(256) pq_scan_fast(const uint8_t* __restrict__ codes, int64_t n,
                                                    const float* __restrict__ cents,
                                                    const double* __restrict__ w,
                                                    const double* __restrict__ lut_g, int K, int Q,
                                                    double* __restrict__ out,
                                                    uint32_t* __restrict__ ghist) {
  extern __shared__ double lut[];  // M * 256
  __shared__ uint32_t sh[kHistBins];
  for (int t = threadIdx.x; t < M * 256; t += blockDim.x) {
    const int m = t >> 8, j = t & 255;
    double v = 0.0;
    if (j < K) v = lut_g ? lut_g[m * K + j]
                         : lut_entry_einsum(cents + ((int64_t)m * K + j) * Q, w + (int64_t)m * Q, Q);
    lut[t] = v;
  }
  if (ghist) hist_zero(sh);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n; base += stride) {
    const int64_t row = base + lane;
    const bool active = row < n;
    double res = 0.0;
    if (active) {
      uint8_t c[M];
      if constexpr (M >= 16) {
#pragma unroll
        for (int v = 0; v < M / 16; ++v) {
          uint4 u = ld_stream_u4(reinterpret_cast<const uint4*>(codes + row * M) + v);
          const uint32_t words[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int q = 0; q < 16; ++q) c[16 * v + q] = (words[q >> 2] >> (8 * (q & 3))) & 0xff;
        }
      } else if constexpr (M == 8) {
        uint2 u = __ldg(reinterpret_cast<const uint2*>(codes + row * M));
#pragma unroll
        for (int q = 0; q < 8; ++q) c[q] = ((q < 4 ? u.x : u.y) >> (8 * (q & 3))) & 0xff;
      } else {
        uint32_t u = __ldg(reinterpret_cast<const uint32_t*>(codes + row * M));
#pragma unroll
        for (int q = 0; q < M; ++q) c[q] = (u >> (8 * q)) & 0xff;
      }
      double a[M];
#pragma unroll
      for (int m = 0; m < M; ++m) a[m] = lut[m * 256 + c[m]];
      if constexpr (M < 8) {
        res = -0.0;
#pragma unroll
        for (int m = 0; m < M; ++m) res = __dadd_rn(res, a[m]);
      } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = a[j];
#pragma unroll
        for (int i = 8; i < M; i += 8) {
#pragma unroll
          for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
        }
        res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                        __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
      }
      out[row] = res;
    }
    if (ghist) hist_add(sh, active, hist_bin(res));
  }
  if (ghist) {
    __syncthreads();
    hist_flush(sh, ghist);
  }
}

// Generic path: any M, K; LUT (built by pq_build_lut_kernel) read through L1.
__global__ void __launch_bounds__(256) pq_scan_generic(const uint8_t* __restrict__ codes, int64_t n,
                                                       int M, const double* __restrict__ lut,
                                                       int K, double* __restrict__ out,
                                                       uint32_t* __restrict__ ghist) {
  __shared__ uint32_t sh[kHistBins];
  if (ghist) hist_zero(sh);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n; base += stride) {
    const int64_t row = base + lane;
    const bool active = row < n;
    double res = 0.0;
    if (active) {
      GlobalLut g{lut, K, codes + row * M};
      res = pairwise_sum(g, 0, M);
      out[row] = res;
    }
    if (ghist) hist_add(sh, active, hist_bin(res));
  }
  if (ghist) {
    __syncthreads();
    hist_flush(sh, ghist);
  }
}

// flag if any code >= K (validation, pq.py:240-241 semantics).
__global__ void pq_check_codes(const uint8_t* __restrict__ codes, int64_t total, int K,
                               unsigned int* __restrict__ bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int found = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride)
    found |= codes[i] >= K;
  if (__syncthreads_or(found) && threadIdx.x == 0) atomicOr(bad, 1u);
}

int launch_pq_lut(const float* cents, int M, int K, int Q, const double* w, double* lut,
                  cudaStream_t st, int replicas) {
  const int total = M * K;
  pq_build_lut_kernel<<<(total + 255) / 256, 256, 0, st>>>(cents, M, K, Q, w, lut, replicas);
  OTF_LAUNCH_CHECK("pq_build_lut");
  return OTF_OK;
}

int launch_pq_check(const uint8_t* codes, int64_t total, int K, unsigned int* bad,
                    int device, cudaStream_t st) {
  if (total <= 0 || K >= 256) return OTF_OK;
  int64_t blocks = (total + 255) / 256;
  const int64_t cap = 4LL * sm_count(device);
  if (blocks > cap) blocks = cap;
  pq_check_codes<<<(int)blocks, 256, 0, st>>>(codes, total, K, bad);
  OTF_LAUNCH_CHECK("pq_check_codes");
  return OTF_OK;
}

template <int M>
static int launch_fast(const uint8_t* codes, int64_t n, const float* cents, const double* w,
                       const double* lut, int K, int Q, double* out, uint32_t* hist, int device,
                       cudaStream_t st) {
  auto fn = pq_scan_fast<M>;
  const size_t smem = (size_t)M * 256 * sizeof(double);
  static bool configured[64] = {false};
  if (!configured[device & 63]) {
    cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured[device & 63] = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)per_sm * sm_count(device);
  const int64_t need = (n + 255) / 256;
  if (need < grid) grid = need;
  fn<<<(int)grid, 256, smem, st>>>(codes, n, cents, w, lut, K, Q, out, hist);
  OTF_LAUNCH_CHECK("pq_scan_fast");
  return OTF_OK;
}

// ---- M == 16: conflict-free XOR-swizzled scan -------------------------------------------------
// numpy's pairwise tree for 16 terms pairs (j, j^8), then (j, j^1), (j, j^2), (j, j^4): it is
// invariant (up to operand order of commutative IEEE adds) under any XOR relabelling
// t -> t ^ s of the terms. Lane l therefore reads its row's sub-codes in the order t ^ s with
// s = l & 15, so at every step the 16 lanes of a half-warp touch 16 different sub-quantizer
// tables; with entry (m, j) stored at double index j*16 + m (bank pair m) every 64-bit LUT read
// is conflict-free (2 wavefronts per warp, the minimum), ~4x fewer than random bank pairs.
// The sum is still bit-identical to pq.py:275.
__device__ __forceinline__ uint32_t sel_u32(bool c, uint32_t a, uint32_t b) { return c ? a : b; }
// packed float32 pairs (sm_100 FADD2): x in the low half, y in the high half
__device__ __forceinline__ uint64_t pack_f2(float x, float y) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

template <int ROWS>
__global__ void __launch_bounds__(256) pq_scan16_xor(const uint8_t* __restrict__ codes, int64_t n,
                                                     const float* __restrict__ cents,
                                                     const double* __restrict__ w,
                                                     const double* __restrict__ lut_g, int K, int Q,
                                                     double* __restrict__ out,
                                                     uint16_t* __restrict__ bins_out,
                                                     uint32_t* __restrict__ ghist) {
  // bins_out != nullptr: write the 16-bit score bin per row instead of the float64 score (the
  // top-k kernel recomputes the exact score of the few candidates; otf_topk.cu PqBinSrc).
  // static (not dynamic) shared memory so the LUT base is an immediate in every LDS
  __shared__ __align__(128) double lut[256 * 16];  // entry (m, j) at byte (j << 7) | (m << 3)
  __shared__ uint32_t sh[kHistBins];
  for (int t = threadIdx.x; t < 16 * 256; t += blockDim.x) {
    const int m = t >> 8, j = t & 255;
    double v = 0.0;
    if (j < K) v = lut_g ? lut_g[m * K + j]
                         : lut_entry_einsum(cents + ((int64_t)m * K + j) * Q, w + (int64_t)m * Q, Q);
    lut[j * 16 + m] = v;
  }
  if (ghist) hist_zero(sh);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t s = lane & 15;
  uint32_t cm[16];  // byte offset of sub-quantizer table t ^ s inside a 128-byte LUT line
#pragma unroll
  for (int t = 0; t < 16; ++t) cm[t] = ((uint32_t)t ^ s) << 3;
  const char* lutb = reinterpret_cast<const char*>(lut);
  const uint4* C4 = reinterpret_cast<const uint4*>(codes);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * ROWS;
  // software pipeline: the next batch of ROWS code rows is in flight while this one is scored
  uint4 nu[ROWS];
  int64_t base = ((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) * ROWS;
#pragma unroll
  for (int i = 0; i < ROWS; ++i) {
    const int64_t row = base + 32 * i + lane;
    nu[i] = row < n ? ld_stream_u4(C4 + row) : make_uint4(0, 0, 0, 0);
  }
  for (; base < n; base += stride) {
    uint4 u[ROWS];
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
      u[i] = nu[i];
      const int64_t row = base + stride + 32 * i + lane;
      nu[i] = row < n ? ld_stream_u4(C4 + row) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
      const int64_t row = base + 32 * i + lane;
      const bool active = row < n;
      // b[t] = code[t ^ s]: XOR by 8 swaps 8-byte halves, by 4 swaps words, by 2 swaps
      // 16-bit halves, by 1 swaps bytes inside halves.
      uint32_t w0 = u[i].x, w1 = u[i].y, w2 = u[i].z, w3 = u[i].w;
      uint32_t t0 = sel_u32(s & 8, w2, w0), t1 = sel_u32(s & 8, w3, w1);
      uint32_t t2 = sel_u32(s & 8, w0, w2), t3 = sel_u32(s & 8, w1, w3);
      w0 = sel_u32(s & 4, t1, t0); w1 = sel_u32(s & 4, t0, t1);
      w2 = sel_u32(s & 4, t3, t2); w3 = sel_u32(s & 4, t2, t3);
      const uint32_t sel = (s & 2 ? 0x1032u : 0x3210u) ^ (s & 1 ? 0x1111u : 0u);
      w0 = __byte_perm(w0, 0, sel); w1 = __byte_perm(w1, 0, sel);
      w2 = __byte_perm(w2, 0, sel); w3 = __byte_perm(w3, 0, sel);
      const uint32_t wd[4] = {w0, w1, w2, w3};
      double b[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int q = t & 3;  // byte q of the word, moved to bits [7, 15) = code << 7
        const uint32_t hi = q == 0 ? (wd[t >> 2] << 7) : (wd[t >> 2] >> (8 * q - 7));
        b[t] = *reinterpret_cast<const double*>(lutb + ((hi & 0x7F80u) | cm[t]));
      }
      double r[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) r[t] = __dadd_rn(b[t], b[t + 8]);
      const double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                                   __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
      const uint32_t bin = hist_bin(res);
      if (active) {
        if (bins_out) bins_out[row] = (uint16_t)bin;
        else out[row] = res;
      }
      if (ghist) hist_add(sh, active, bin);
    }
  }
  if (ghist) {
    __syncthreads();
    hist_flush(sh, ghist);
  }
}

// ---- M == 16 score() path: float64 scores, one byte_perm per lookup (round 2) -------------------
// pq_scan16_xor computes every lookup address with a shift and a mask (ncu: ALU pipe 64%, 142
// warp instructions per 32 rows — issue-bound). Here the float64 entry (m, j) sits at byte
// (j << 8) | (m << 3) of a 256-byte line per code value j (the rank path's line layout, float32
// half unused), so the address of sub-code t ^ s is ONE byte_perm of the code word with a
// per-lane constant, as in the float32 screening; lanes of a half-warp read 16 different m:
// conflict-free. The XOR order of the terms keeps numpy's pairwise sum bit-identical
// (pq_scan16_xor's argument).
constexpr int kScore16Threads = 512;  // 2 CTAs x 16 warps per SM (64 KB of lines each)
constexpr size_t kScore16Smem = 256 * 256;

template <int ROWS>
__global__ void __launch_bounds__(kScore16Threads, 2) pq_score16_lines(const uint8_t* __restrict__ codes, int64_t n,
                                                                  const double* __restrict__ lut_g, int K,
                                                                  double* __restrict__ out) {
  extern __shared__ __align__(1024) unsigned char sm[];  // 256 lines x 256 B (float64 half used)
  asm volatile("griddepcontrol.wait;" ::: "memory");      // (after the LUT kernel)
  {
    // all loads in flight before the first store (a load-store loop pays one L2 round trip per entry batch)
    constexpr int kPer = 16 * 256 / kScore16Threads;
    const int m = threadIdx.x & 15;  // 16 lanes fill one 128-byte run of a line
    double v[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int j = (threadIdx.x + i * kScore16Threads) >> 4;
      v[i] = j < K ? __ldg(lut_g + m * K + j) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i)
      *reinterpret_cast<double*>(sm + (((threadIdx.x + i * kScore16Threads) >> 4) << 8) + (m << 3)) = v[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t s = lane & 15;
  uint32_t kw[8];  // byte 0 / 1: (2u ^ s) << 3, (2u + 1 ^ s) << 3 — the entry offset inside a line
#pragma unroll
  for (int u = 0; u < 8; ++u) kw[u] = (((uint32_t)(2 * u) ^ s) << 3) | ((((uint32_t)(2 * u + 1) ^ s) << 3) << 8);
  uint32_t sel[4];  // result byte 0 <- kw byte (t & 1), byte 1 <- code byte ((t ^ s) & 3), bytes 2, 3 <- 0
#pragma unroll
  for (int q = 0; q < 4; ++q) sel[q] = 0x7604u | (uint32_t)(q & 1) | ((((uint32_t)q ^ s) & 3u) << 4);
  const uint4* C4 = reinterpret_cast<const uint4*>(codes);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * ROWS;
  uint4 nu[ROWS];
  int64_t base = ((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) * ROWS;
#pragma unroll
  for (int i = 0; i < ROWS; ++i) {
    const int64_t row = base + 32 * i + lane;
    nu[i] = row < n ? ld_stream_u4(C4 + row) : make_uint4(0, 0, 0, 0);
  }
  for (; base < n; base += stride) {
    uint4 u[ROWS];
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
      u[i] = nu[i];
      const int64_t row = base + stride + 32 * i + lane;
      nu[i] = row < n ? ld_stream_u4(C4 + row) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
      const int64_t row = base + 32 * i + lane;
      // words permuted by s & 8 (halves) and s & 4 (words): word t >> 2 holds sub-codes 4 (t >> 2) ^ s..
      const uint32_t x0 = u[i].x, x1 = u[i].y, x2 = u[i].z, x3 = u[i].w;
      const uint32_t t0 = sel_u32(s & 8, x2, x0), t1 = sel_u32(s & 8, x3, x1);
      const uint32_t t2 = sel_u32(s & 8, x0, x2), t3 = sel_u32(s & 8, x1, x3);
      const uint32_t wd[4] = {sel_u32(s & 4, t1, t0), sel_u32(s & 4, t0, t1), sel_u32(s & 4, t3, t2),
                              sel_u32(s & 4, t2, t3)};
      double b[16];
#pragma unroll
      for (int t = 0; t < 16; ++t)
        b[t] = *reinterpret_cast<const double*>(sm + __byte_perm(wd[t >> 2], kw[t >> 1], sel[t & 3]));
      double r[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) r[t] = __dadd_rn(b[t], b[t + 8]);
      const double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                                   __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
      if (row < n) out[row] = res;
    }
  }
}

static int launch_scan16(const uint8_t* codes, int64_t n, const float* cents, const double* w,
                         const double* lut, int K, int Q, double* out, uint16_t* bins,
                         uint32_t* hist, int device, cudaStream_t st) {
  constexpr int ROWS = 4;
  static const bool xor_kernel = getenv("OTF_PQ_SCORE_XOR") != nullptr;  // A/B switch (tools/)
  if (lut && out && !bins && !hist && !xor_kernel) {
    // the float64 score() path (round 2): one byte_perm per lookup
    auto fs = pq_score16_lines<ROWS>;
    static int per_sm_s[64] = {0};
    if (!per_sm_s[device & 63]) {
      OTF_CUDA(cudaFuncSetAttribute((const void*)fs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScore16Smem));
      int b = 0;
      OTF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fs, kScore16Threads, kScore16Smem));
      per_sm_s[device & 63] = b > 0 ? b : 1;
    }
    int64_t grid = (int64_t)per_sm_s[device & 63] * sm_count(device);
    const int64_t need = (n + kScore16Threads * ROWS - 1) / (kScore16Threads * ROWS);
    if (need < grid) grid = need;
    fs<<<(int)grid, kScore16Threads, kScore16Smem, st>>>(codes, n, lut, K, out);
    OTF_LAUNCH_CHECK("pq_score16_lines");
    return OTF_OK;
  }
  auto fn = pq_scan16_xor<ROWS>;  // 48 KB static shared memory (LUT + histogram)
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)per_sm * sm_count(device);
  const int64_t need = (n + 256 * ROWS - 1) / (256 * ROWS);
  if (need < grid) grid = need;
  fn<<<(int)grid, 256, 0, st>>>(codes, n, cents, w, lut, K, Q, out, bins, hist);
  OTF_LAUNCH_CHECK("pq_scan16_xor");
  return OTF_OK;
}

// ---- M == 16 rank path: float32 screening, exact bins -----------------------------------------
// The rank path needs only each row's 16-bit score bin (the top-k recomputes the candidates'
// exact float64 scores, otf_topk.cu PqBinSrc), and a bin is a monotone function of the score.
// So each row is first summed from a float32 copy of the LUT: |s32 - s64| <= eps with
// eps = 2^-20 * sum_m max_j |LUT[m][j]| (entries rounded to float32: 2^-24 each, a depth-4
// float32 tree: 4 * 2^-24 of the sum, numpy's float64 tree: negligible — a >3x margin). If
// [s32 - eps, s32 + eps] (outward-rounded) lies inside one bin, that IS the bin of the exact
// score; otherwise (near a bin edge, or non-finite LUT) the row's exact float64 score is
// computed with numpy's pairwise order from the float64 LUT, as in pq_scan16_xor.
// Shared-memory line j (256 B) holds the float64 entries (m, j) at bytes m*8 and two float32
// copies at 128 + 64*c + 4*m. Lane l reads sub-code t ^ (l & 15) at step t from copy
// (l >> 4): 32 lanes hit 32 different banks (one wavefront per LDS.32), and the whole
// address is ONE byte_perm (code byte -> bits 8..15, a per-lane constant in bits 0..7).
constexpr int kScanF32Threads = 512;
constexpr size_t kScanF32Smem = 256 * 256 + kPqHistBins * sizeof(uint32_t) + 32 * sizeof(uint32_t);

template <int ROWS>
__global__ void __launch_bounds__(kScanF32Threads, 1) pq_scan16_f32bins(const uint8_t* __restrict__ codes, int64_t n,
                                                                     const double* __restrict__ lut_g, int K,
                                                                     uint16_t* __restrict__ bins_out,
                                                                     uint32_t* __restrict__ ghist,
                                                                     uint16_t* __restrict__ cmax) {
  extern __shared__ __align__(1024) unsigned char sm[];  // [256 lines x 256 B][hist][m maxima]
  uint32_t* sh = reinterpret_cast<uint32_t*>(sm + 65536);
  uint32_t* smax = sh + kPqHistBins;
  if (threadIdx.x < 16) smax[threadIdx.x] = 0u;
  hist_zero(sh, kPqHistBins);
  __syncthreads();
  // launched programmatically after the LUT kernel: wait for its writes before reading lut_g
  // (a no-op for a normal launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  {
    // thread t always handles sub-quantizer m = t & 15 (blockDim = 512): 16 lanes fill one
    // 128-byte run of a line, and the per-m maxima need one atomic per thread
    const int m = threadIdx.x & 15;
    uint32_t mx = 0u;
    constexpr int kPer = 16 * 256 / kScanF32Threads;
    double vs[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {  // all loads in flight before the first store
      const int j = (threadIdx.x + i * kScanF32Threads) >> 4;
      vs[i] = j < K ? lut_g[m * K + j] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int j = (threadIdx.x + i * kScanF32Threads) >> 4;
      const double v = vs[i];
      unsigned char* line = sm + (j << 8);
      *reinterpret_cast<double*>(line + 8 * m) = v;
      const float f = __double2float_rn(v);
      *reinterpret_cast<float*>(line + 128 + 4 * m) = f;
      *reinterpret_cast<float*>(line + 192 + 4 * m) = f;
      // |v| as float rounded up: non-negative floats (and NaN above inf) order like their bits
      mx = max(mx, __float_as_uint(fabsf(__double2float_ru(fabs(v)))));
    }
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
    if ((threadIdx.x & 31) < 16) atomicMax(&smax[m], mx);
  }
  __syncthreads();
  float eps;
  bool screen;
  {
    double e = 0.0;  // S = sum_m max_j |LUT[m][j]| bounds every partial sum of the float32 tree
#pragma unroll
    for (int m = 0; m < 16; ++m) e += (double)__uint_as_float(smax[m]);
    eps = __double2float_ru(e * 0x1p-20);
    eps = fmaxf(eps, 0x1p-140f);  // absolute floor: float32 underflow of tiny entries
    // no float32 partial sum can overflow when S <= 1e38 (and NaN/inf LUTs fail the test):
    // otherwise every row takes the exact path
    screen = e <= 1.0e38;
  }
  const int lane = threadIdx.x & 31;
  const uint32_t s = lane & 15;
  // per step pair u: K word [offset of table 2u^s, offset of table (2u+1)^s, 0, 0] (copy lane>>4)
  // and per t&3 the selector [K byte t&1, byte (t^s)&3 of the permuted word -> bits 8..15, 0, 0]
  uint32_t kw[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const uint32_t c = 128u | ((uint32_t)(lane >> 4) << 6);
    kw[u] = (c | (((uint32_t)(2 * u) ^ s) << 2)) | ((c | (((uint32_t)(2 * u + 1) ^ s) << 2)) << 8);
  }
  uint32_t sel[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) sel[q] = 0x7604u | (uint32_t)(q & 1) | ((((uint32_t)q ^ s) & 3u) << 4);
  const uint4* C4 = reinterpret_cast<const uint4*>(codes);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * ROWS;
  // software pipeline: the next batch of ROWS code rows is in flight while this one is scored
  uint4 nu[ROWS];
  int64_t base = ((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) * ROWS;
#pragma unroll
  for (int i = 0; i < ROWS; ++i) {
    const int64_t row = base + 32 * i + lane;
    nu[i] = row < n ? ld_stream_u4(C4 + row) : make_uint4(0, 0, 0, 0);
  }
  for (; base < n; base += stride) {
    uint4 u[ROWS];
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
      u[i] = nu[i];
      const int64_t row = base + stride + 32 * i + lane;
      nu[i] = row < n ? ld_stream_u4(C4 + row) : make_uint4(0, 0, 0, 0);
    }
    // 1) screening scores of all ROWS rows (branch-free, so the rows' lookup chains interleave)
    float s32[ROWS];
    uint32_t need_exact = 0;
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
      // word t>>2 of the permuted row = word (t>>2) ^ (s>>2) of the code row
      const uint32_t x0 = u[i].x, x1 = u[i].y, x2 = u[i].z, x3 = u[i].w;
      const uint32_t t0 = sel_u32(s & 8, x2, x0), t1 = sel_u32(s & 8, x3, x1);
      const uint32_t t2 = sel_u32(s & 8, x0, x2), t3 = sel_u32(s & 8, x1, x3);
      const uint32_t wd[4] = {sel_u32(s & 4, t1, t0), sel_u32(s & 4, t0, t1), sel_u32(s & 4, t3, t2),
                              sel_u32(s & 4, t2, t3)};
      float b[16];
#pragma unroll
      for (int t = 0; t < 16; ++t)
        b[t] = *reinterpret_cast<const float*>(sm + __byte_perm(wd[t >> 2], kw[t >> 1], sel[t & 3]));
      // depth-4 float32 tree on packed pairs (FADD2): P_k = (b_2k, b_2k+1); Q_k = P_k + P_k+4;
      // R_k = Q_k + Q_k+2; S = R_0 + R_1; s32 = S.x + S.y (any fixed depth-4 tree fits eps)
      uint64_t P[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) P[k] = pack_f2(b[2 * k], b[2 * k + 1]);
#pragma unroll
      for (int k = 0; k < 4; ++k) P[k] = fadd2(P[k], P[k + 4]);
      P[0] = fadd2(P[0], P[2]);
      P[1] = fadd2(P[1], P[3]);
      P[0] = fadd2(P[0], P[1]);
      // + 0.0f turns -0.0 into +0.0 (they share a bin, score_key)
      s32[i] = __fadd_rn(__fadd_rn(__uint_as_float((uint32_t)P[0]), __uint_as_float((uint32_t)(P[0] >> 32))), 0.0f);
      // [lo, hi] inside one bin <=> their order keys agree in the top 12 bits <=> their bit
      // patterns do (same sign; -0.0 vs +0.0 counts as different: conservative)
      const float lo = __fsub_rd(s32[i], eps), hi = __fadd_ru(s32[i], eps);
      if (!screen || (__float_as_uint(lo) ^ __float_as_uint(hi)) >= (1u << (32 - kPqHistBits))) need_exact |= 1u << i;
    }
    uint32_t bin[ROWS];
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {  // order key of a float without the -0.0 test (done above)
      const uint32_t v = __float_as_uint(s32[i]);
      bin[i] = (v ^ ((uint32_t)((int32_t)v >> 31) | 0x80000000u)) >> (32 - kPqHistBits);
    }
    // 2) rare: rows whose interval straddles a bin edge take the exact float64 score (numpy's
    //    pairwise order) and its bin
    if (need_exact) {
#pragma unroll
      for (int i = 0; i < ROWS; ++i) {
        if ((need_exact >> i) & 1u) {
          const uint32_t xw[4] = {u[i].x, u[i].y, u[i].z, u[i].w};
          double a[16];
#pragma unroll
          for (int m = 0; m < 16; ++m)
            a[m] = *reinterpret_cast<const double*>(sm + (((xw[m >> 2] >> (8 * (m & 3))) & 0xffu) << 8) + 8 * m);
          double rr[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) rr[j] = __dadd_rn(a[j], a[j + 8]);
          bin[i] = pq_hist_bin(__dadd_rn(__dadd_rn(__dadd_rn(rr[0], rr[1]), __dadd_rn(rr[2], rr[3])),
                                      __dadd_rn(__dadd_rn(rr[4], rr[5]), __dadd_rn(rr[6], rr[7]))));
        }
      }
    }
    // 3) bins, histogram, chunk maximum
    uint32_t mb = 0;  // max bin of the active rows of this lane
    if (base + 32 * ROWS <= n) {  // full batch (all but the last): no per-row bounds checks
#pragma unroll
      for (int i = 0; i < ROWS; ++i) {
        bins_out[base + 32 * i + lane] = (uint16_t)bin[i];
        if (ghist) hist_add(sh, true, bin[i]);
        mb = max(mb, bin[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < ROWS; ++i) {
        const int64_t row = base + 32 * i + lane;
        const bool active = row < n;
        if (active) bins_out[row] = (uint16_t)bin[i];
        if (ghist) hist_add(sh, active, bin[i]);
        if (active) mb = max(mb, bin[i]);
      }
    }
    // the warp's 32 * ROWS consecutive rows are one top-k chunk
    if (cmax) {
      const uint32_t wm = __reduce_max_sync(0xffffffffu, mb);
      if (lane == 0) cmax[base / (32 * ROWS)] = (uint16_t)wm;
    }
  }
  if (ghist) {
    __syncthreads();
    hist_flush(sh, ghist, kPqHistBins);
  }
}

// ---- M == 16 cut path: one cooperative kernel (sampled threshold, candidate emission, select) ---
// The rank path needs the k best rows, not every row's score. pq_rank_cut_kernel (one CTA per SM,
// cooperative, launched programmatically after the LUT kernel) streams the codes through shared
// memory (1-D bulk copies, see below) and
//   1. scores the first half of its first chunk (a sample spread over the whole repository: 2048
//      rows per CTA) in float32 and publishes the sample's two largest screening keys; a SPLIT
//      grid barrier: while the other CTAs finish their sample, each CTA scores the next three
//      batches of its ring (held: their screening scores stay in registers, their codes in the
//      stages); then every CTA takes T = the r-th largest of the 2 G published keys at 16-bit key
//      resolution (r ~ want x sample / n, want ~ 1.56 k_eff + 128, so ~want rows are expected at or
//      above T), rounded down to that prefix's lower edge;
//   2. emits every row whose float32 screening score s32 can reach T (s32 >= T - eps, |s32 -
//      s64| <= eps as in pq_scan16_f32bins) AND whose exact float64 score (numpy's order, from
//      the float64 LUT in shared memory) is >= T: (exact key, ~id), the row and the key's top 32
//      bits go to a candidate list (warp-aggregated atomics; ~0.02% of the rows); nothing is
//      written for the other rows (no per-row bins, histogram or score writes);
//   3. one more grid barrier; every row with exact score >= T is a candidate, so when at least
//      k_eff and at most kRcCand rows reached T the global top-k is among them: every CTA copies
//      the candidates' 32-bit key prefixes into shared memory and ranks its share by counting
//      (candidate i on CTA i mod G; full keys, ids and rows read only for prefix ties), writing
//      each straight to its output slot. Otherwise (T too high: fewer than k rows reached it; or
//      too many candidates: heavy ties, w = 0; or a non-finite LUT) the kernel computes every
//      row's exact score and runs the exact radix select (otf_topk_dev.cuh) — slower, same result.
// Bit-exact with the reference either way (pq.py:248-276 scores, ranker.py:97-143 order).
#ifdef OTF_CUT_TRACE  // diagnostic build (tools/gpu_cut_trace.sh): per-CTA globaltimer stamps
#define CUT_STAMP(i) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts[i]))
#else
#define CUT_STAMP(i)
#endif

__device__ __forceinline__ float key_to_f32(uint32_t k) {
  return __uint_as_float((k >> 31) ? (k ^ 0x80000000u) : ~k);
}

// Rare: the lanes with screening bits compute their rows' exact float64 score (numpy's pairwise
// order from the float64 entries of the LUT lines); rows whose exact key reaches T append
// (exact key, ~id), the row and the key's top 32 bits (warp-aggregated slot reservation).
template <int ROWS>
__device__ __noinline__ void cut_emit(const unsigned char* sm, uint4 u0, uint4 u1, uint4 u2, uint4 u3, uint32_t emit,
                                      int64_t row0, const int64_t* ids, int64_t id_base,
                                      unsigned long long* cut_count, uint64_t tkey64, ulonglong2* cut_rec,
                                      int64_t* cut_row, uint32_t* key32, int64_t cut_cap, int64_t key32_cap) {
  static_assert(ROWS == 4, "four rows per lane");
  const int lane = threadIdx.x & 31;
  const uint4 uu[4] = {u0, u1, u2, u3};
#pragma unroll
  for (int i = 0; i < ROWS; ++i) {
    uint64_t key = 0;
    if ((emit >> i) & 1u) {
      const uint32_t xw[4] = {uu[i].x, uu[i].y, uu[i].z, uu[i].w};
      double a[16];
#pragma unroll
      for (int m = 0; m < 16; ++m)
        a[m] = *reinterpret_cast<const double*>(sm + (((xw[m >> 2] >> (8 * (m & 3))) & 0xffu) << 8) + 8 * m);
      double rr[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) rr[j] = __dadd_rn(a[j], a[j + 8]);
      const double ex = __dadd_rn(__dadd_rn(__dadd_rn(rr[0], rr[1]), __dadd_rn(rr[2], rr[3])),
                                  __dadd_rn(__dadd_rn(rr[4], rr[5]), __dadd_rn(rr[6], rr[7])));
      key = score_key(ex);
    }
    const bool take = ((emit >> i) & 1u) && key >= tkey64;
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    if (bal == 0u) continue;
    unsigned long long slot0 = 0;
    if (lane == 0) slot0 = atomicAdd(cut_count, (unsigned long long)__popc(bal));
    const int64_t slot = (int64_t)__shfl_sync(0xffffffffu, slot0, 0) + __popc(bal & ((1u << lane) - 1u));
    // past the capacity only the count matters (the selection falls back)
    if (take && slot < cut_cap) {
      const int64_t row = row0 + 32 * i;
      cut_rec[slot] = make_ulonglong2(key, inv_id(id_of(ids, id_base, row)));
      cut_row[slot] = row;
      if (slot < key32_cap) key32[slot] = (uint32_t)(key >> 32);
    }
  }
}

// The codes stream through shared memory: 4096-row chunks (64 KB) land by 1-D bulk copies
// (cp.async.bulk, the TMA engine) in a ring of kCutStages stages, each armed on an mbarrier with
// its byte count (L2 evict-first: the repository is read once per query). CTA b owns a
// contiguous range of chunks; its first stages are requested before griddepcontrol.wait (the
// codes do not depend on the LUT kernel). Warp w scores rows [256 w, 256 w + 256) of a chunk in
// two batches of 4 rows per lane (one conflict-free 16-byte shared load per row); the last warp
// done with a stage refills it with the CTA's chunk kCutStages ahead.
#ifndef OTF_CUT_THREADS
#define OTF_CUT_THREADS 512
#endif
#ifndef OTF_CUT_STAGES
#define OTF_CUT_STAGES 2
#endif
#ifndef OTF_CUT_BATCHES
#define OTF_CUT_BATCHES 2
#endif
// Ring plans: 2 stages x 2 batches (64 KB chunks: one in flight while one is scored; the
// default), or S >= 4 stages x 1 batch (32 KB chunks: up to S - 1 in flight). Measured (round 2,
// -DOTF_CUT_NOCOMPUTE: the codes stream through the ring unscored): the 2 x 64 KB ring alone moves
// C3x's 1.6 GB at 7.6 TB/s, so the scan is bound by the scoring (~55 warp instructions per row,
// 16 warps per SM, latency-bound at ~40% issue), not the ring; 4 x 32 KB was 0.393 vs 0.317 ms
// on C3x with scoring (code generation), 12 warps x 3 x 48 KB 0.404.
constexpr int kCutScanThreads = OTF_CUT_THREADS;  // x 4 rows per lane (1024 x 2 and 1024 x 1 measured slower)
constexpr int kCutRows = 4;           // rows per lane per batch
constexpr int kCutBatches = OTF_CUT_BATCHES;  // batches per warp per chunk
constexpr int kCutStages = OTF_CUT_STAGES;
static_assert((kCutBatches == 2 && kCutStages == 2) || (kCutBatches == 1 && kCutStages >= 4), "ring plan");
// the sample and the held batches: chunk c0's batches then the prologue's chunks (stage, batch)
constexpr int kCutHeld = kCutBatches == 2 ? 3 : kCutStages - 2;  // batches scored while T is found
constexpr int kCutHeldStages = kCutBatches == 2 ? 2 : kCutStages - 1;  // stages consumed before the main loop
__host__ __device__ constexpr int cut_held_stage(int hb) { return kCutBatches == 2 ? (hb == 0 ? 0 : 1) : hb + 1; }
__host__ __device__ constexpr int cut_held_batch(int hb) { return kCutBatches == 2 ? (hb == 0 ? 1 : hb - 1) : 0; }
constexpr int kCutBatchRows = kCutScanThreads * kCutRows;      // 2048 (the sample: batch 0 of chunk 0)
constexpr int kCutChunkRows = kCutBatchRows * kCutBatches;      // 4096
constexpr int kCutChunkBytes = kCutChunkRows * 16;

__device__ __forceinline__ uint32_t cut_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// rows [r0, min(r0 + kCutChunkRows, end)) -> dst
__device__ __forceinline__ void cut_issue(const uint8_t* codes, int64_t end, int64_t r0, unsigned char* dst,
                                          uint64_t* bar, int64_t max_rows = kCutChunkRows) {
  const int64_t rows = min(max_rows, end - r0);
  const uint32_t bytes = (uint32_t)(rows * 16);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(cut_smem_u32(bar)), "r"(bytes)
               : "memory");
#ifndef OTF_NO_EVICT_FIRST
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                   cut_smem_u32(dst)),
               "l"(codes + r0 * 16), "r"(bytes), "r"(cut_smem_u32(bar)), "l"(l2_evict_first())
               : "memory");
#else
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   cut_smem_u32(dst)),
               "l"(codes + r0 * 16), "r"(bytes), "r"(cut_smem_u32(bar))
               : "memory");
#endif
}

__device__ __forceinline__ void cut_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(cut_smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

// Screening scores only (the sample chunk, before T is known).
template <int ROWS>
__device__ __forceinline__ void cut_scores(const unsigned char* sm, const uint4 (&u)[ROWS], const uint32_t (&kw)[8],
                                           const uint32_t (&sel)[4], uint32_t s, float (&out)[ROWS]) {
#pragma unroll
  for (int i = 0; i < ROWS; ++i) {
    const uint32_t x0 = u[i].x, x1 = u[i].y, x2 = u[i].z, x3 = u[i].w;
    const uint32_t t0 = sel_u32(s & 8, x2, x0), t1 = sel_u32(s & 8, x3, x1);
    const uint32_t t2 = sel_u32(s & 8, x0, x2), t3 = sel_u32(s & 8, x1, x3);
    const uint32_t wd[4] = {sel_u32(s & 4, t1, t0), sel_u32(s & 4, t0, t1), sel_u32(s & 4, t3, t2),
                            sel_u32(s & 4, t2, t3)};
    float b[16];
#pragma unroll
    for (int t = 0; t < 16; ++t)
      b[t] = *reinterpret_cast<const float*>(sm + __byte_perm(wd[t >> 2], kw[t >> 1], sel[t & 3]));
    uint64_t P[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) P[k] = pack_f2(b[2 * k], b[2 * k + 1]);
#pragma unroll
    for (int k = 0; k < 4; ++k) P[k] = fadd2(P[k], P[k + 4]);
    P[0] = fadd2(P[0], P[2]);
    P[1] = fadd2(P[1], P[3]);
    P[0] = fadd2(P[0], P[1]);
    out[i] = __fadd_rn(__uint_as_float((uint32_t)P[0]), __uint_as_float((uint32_t)(P[0] >> 32)));
  }
}

constexpr size_t kRcSmem = 256 * 256 + (size_t)kCutStages * kCutChunkBytes;  // 208 KB
// the raw (M, K) LUT replica lands in the last stage (filled only after the rearrangement) when
// there are three or more stages, else in the second half of stage 0
constexpr bool kCutLutInLast = kCutStages > kCutHeldStages;
constexpr size_t kCutLutOff = kCutLutInLast ? (size_t)(kCutStages - 1) * kCutChunkBytes : (size_t)kCutBatchRows * 16;
static_assert(kCutLutOff + 16 * 256 * 8 <= (size_t)kCutStages * kCutChunkBytes, "LUT replica fits its stage");
static_assert(kCutLutInLast || kCutBatches == 2, "stage plan");
constexpr int kRcCand = 8192;  // candidates the selection ranks in shared memory (32-bit key prefixes)
static_assert((size_t)kRcCand * 4 <= kRcSmem, "selection reuses the scan's shared memory");

// max of four floats (emission test of a batch: one compare instead of four)
__device__ __forceinline__ float max4(const float (&v)[4]) { return fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3])); }

__global__ void __launch_bounds__(kCutScanThreads, 1)
pq_rank_cut_kernel(const uint8_t* __restrict__ codes, int64_t n, const double* __restrict__ lut_g, int K,
                   const int64_t* __restrict__ ids, int64_t id_base, int64_t k_eff, int r, TopkWs ws,
                   double* __restrict__ scratch, int64_t* __restrict__ out_ids, double* __restrict__ out_scores,
                   int64_t* __restrict__ out_rows) {
  constexpr int ROWS = kCutRows;
  // [256 LUT lines x 256 B][kCutStages x 64 KB code chunks]; the selection reuses all of it
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* stage = sm + 65536;
  __shared__ __align__(8) uint64_t full[kCutStages];
  __shared__ __align__(8) uint64_t sbar;  // the sample: the first half of chunk c0, requested first
  __shared__ __align__(8) uint64_t lbar;  // the LUT replica (into the second half of stage 0)
  __shared__ unsigned done[kCutStages];
  __shared__ int64_t stage_chunk[kCutStages];  // chunk held by each stage (-1: none left)
  __shared__ uint32_t smx[16];
  __shared__ uint32_t s_top[2 * (kCutScanThreads / 32)];
  __shared__ uint32_t s_tkey;
  __shared__ uint32_t h[256];
  __shared__ int s_b;
  __shared__ int64_t s_above;
  __shared__ unsigned s_last, s_gen;
  __shared__ unsigned long long s_pre;  // static round-robin rounds this CTA has taken
#ifdef OTF_CUT_TRACE
  unsigned long long ts[7] = {0, 0, 0, 0, 0, 0, 0};
  CUT_STAMP(0);
#endif
  const unsigned G = gridDim.x, vb = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = kCutScanThreads / 32;
  // chunks of kCutChunkRows rows: CTA b's first chunk is c0 = floor(b nchunks / G) (the sample:
  // spread over the whole repository, never the last, partial chunk); every other chunk is taken
  // dynamically in row order from a global counter (skipping the G first chunks), so CTAs that
  // stream faster take more chunks and all finish together
  const int64_t nchunks = (n + kCutChunkRows - 1) / kCutChunkRows;  // >= 4 G (pq_cut_plan)
  const int64_t c0 = (int64_t)vb * nchunks / G;
  const int64_t rb = c0 * kCutChunkRows, re = n;
  unsigned long long* chunk_ctr = reinterpret_cast<unsigned long long*>(ws.cut_word + 8);
  const bool small32 = (uint64_t)nchunks * G < (1ull << 32);  // 32-bit divisions suffice (every real size)
  auto is_first = [&](int64_t c) {  // chunk c is some CTA's first chunk c0
    if (small32) {
      const uint32_t nc = (uint32_t)nchunks, cc = (uint32_t)c;
      const uint32_t b = (cc * G + nc - 1u) / nc;  // the only CTA whose c0 could be c
      return b < G && b * nc / G == cc;
    }
    const int64_t b = (c * G + nchunks - 1) / nchunks;
    return b < (int64_t)G && b * nchunks / G == c;
  };
  // chunks after each CTA's first: the first 7/8 (whole rounds of G) in static round robin —
  // CTA b takes b, b + G, b + 2G, ... with no atomic — then the tail from a global counter, so
  // CTAs that stream faster take more of it and all finish together. (A claim's atomic stalls
  // the warp that refills a stage, and that warp is the stage's laggard: claiming every chunk
  // cost C3x 0.333 vs 0.317 ms with 7/8 static (3/4: 0.320, 1/2: 0.324); all-static was 2 us
  // slower on C3 from the imbalance.)
#ifndef OTF_CUT_STAT16  // sixteenths of the chunks in static rounds
#define OTF_CUT_STAT16 14
#endif
  const int64_t stat_rounds = nchunks * OTF_CUT_STAT16 / 16 / G;
  auto next_chunk = [&]() -> int64_t {
    for (;;) {
      int64_t c;
      if ((int64_t)s_pre < stat_rounds) {
        c = (int64_t)s_pre * G + vb;
        s_pre = s_pre + 1ull;
        __threadfence_block();  // (the next refill may be another warp's)
      } else {
        c = stat_rounds * G + (int64_t)atomicAdd(chunk_ctr, 1ull);
      }
      if (c >= nchunks) return -1;
      if (!is_first(c)) return c;
    }
  };
  const uint32_t lut_bytes = (uint32_t)(16 * K * 8);
  if (threadIdx.x == 0) {
    s_pre = 0ull;  // static rounds taken
    for (int st = 0; st < kCutStages; ++st) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cut_smem_u32(&full[st])));
      done[st] = 0u;
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cut_smem_u32(&sbar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cut_smem_u32(&lbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the codes do not depend on the LUT kernel: the sample (batch 0 of chunk c0) and chunk 1
    // stream in while it finishes
    cut_issue(codes, re, rb, stage, kCutBatches == 2 ? &sbar : &full[0], kCutBatchRows);
    stage_chunk[0] = c0;
    for (int st = 1; st < kCutStages; ++st) {
      const int64_t c = next_chunk();
      stage_chunk[st] = c;
      if (kCutLutInLast && st == kCutStages - 1) continue;  // the LUT lands there first
      if (c >= 0) cut_issue(codes, re, c * kCutChunkRows, stage + st * kCutChunkBytes, &full[st]);
      else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(cut_smem_u32(&full[st])) : "memory");
    }
    s_tkey = 0u;
  }
  if (threadIdx.x < 16) smx[threadIdx.x] = 0u;
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the LUT: one bulk copy of this CTA's replica into the second half of stage 0, then
  // rearranged into the lookup lines (entry (m, j) of the (M, K) table -> line j)
  if (threadIdx.x == 0) {
    const double* rep = lut_g + (int64_t)(vb % kCutLutReplicas) * 16 * K;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(cut_smem_u32(&lbar)), "r"(lut_bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     cut_smem_u32(stage + kCutLutOff)),
                 "l"(rep), "r"(lut_bytes), "r"(cut_smem_u32(&lbar))
                 : "memory");
  }
  cut_wait(&lbar, 0u);
  {
    // 16 x 16 diagonal blocks per half-warp: lane l moves entry (m = l & 15, j = j0 + m) — the
    // raw reads (bank 2 j) and the line writes (bank 2 m) are both conflict-free
    const double* raw = reinterpret_cast<const double*>(stage + kCutLutOff);
    const int m = lane & 15;
    uint32_t mx = 0u;
    for (int j0 = 2 * wid + (lane >> 4); j0 < 256; j0 += 2 * nw) {
      const int jj = (j0 & ~15) | ((j0 + m) & 15);  // a permutation of the 16 j of the block
      const double v = jj < K ? raw[m * K + jj] : 0.0;
      unsigned char* line = sm + (jj << 8);
      *reinterpret_cast<double*>(line + 8 * m) = v;
      const float f = __double2float_rn(v);
      *reinterpret_cast<float*>(line + 128 + 4 * m) = f;
      *reinterpret_cast<float*>(line + 192 + 4 * m) = f;
      mx = max(mx, __float_as_uint(fabsf(__double2float_ru(fabs(v)))));
    }
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
    if (lane < 16) atomicMax(&smx[m], mx);
  }
  __syncthreads();  // every read of the raw LUT is done: chunk c0's second half (or the last stage's chunk) may land there
  if (threadIdx.x == 0) {
    if (kCutBatches == 2)
      cut_issue(codes, re, rb + kCutBatchRows, stage + kCutBatchRows * 16, &full[0], kCutChunkRows - kCutBatchRows);
    if (kCutLutInLast) {
      constexpr int st = kCutStages - 1;
      const int64_t c = stage_chunk[st];
      if (c >= 0) cut_issue(codes, re, c * kCutChunkRows, stage + st * kCutChunkBytes, &full[st]);
      else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(cut_smem_u32(&full[st])) : "memory");
    }
  }
  // (pq_cut_plan keeps c0 + 1 <= nchunks - 1, so chunk c0 is full)
  float eps;
  bool screen;
  {
    double e = 0.0;
#pragma unroll
    for (int m = 0; m < 16; ++m) e += (double)__uint_as_float(smx[m]);
    eps = __double2float_ru(e * 0x1p-20);
    eps = fmaxf(eps, 0x1p-140f);
    screen = e <= 1.0e38;
  }
  const uint32_t s = lane & 15;
  uint32_t kw[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const uint32_t c = 128u | ((uint32_t)(lane >> 4) << 6);
    kw[u] = (c | (((uint32_t)(2 * u) ^ s) << 2)) | ((c | (((uint32_t)(2 * u + 1) ^ s) << 2)) << 8);
  }
  uint32_t sel[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) sel[q] = 0x7604u | (uint32_t)(q & 1) | ((((uint32_t)q ^ s) & 3u) << 4);
  unsigned long long* cut_count = reinterpret_cast<unsigned long long*>(ws.cut_word);
  ulonglong2* cut_rec = reinterpret_cast<ulonglong2*>(ws.cut_key);
  uint32_t* key32 = reinterpret_cast<uint32_t*>(ws.key);  // prefixes of the first kRcCand candidates
  const int boff = wid * (32 * ROWS) + lane;  // this lane's first row inside a batch

  // ---- 1. the sample: batch 0 of chunk c0 ----------------------------------------------------------
  uint4 u0[ROWS];
  float s0[ROWS];
  const int64_t row00 = rb + boff;
  {
    uint32_t ka = 0u, kb = 0u;  // this lane's two largest sample keys (0: below every key)
    cut_wait(kCutBatches == 2 ? &sbar : &full[0], 0u);
    const uint4* rows4 = reinterpret_cast<const uint4*>(stage) + boff;
#pragma unroll
    for (int i = 0; i < ROWS; ++i) u0[i] = row00 + 32 * i < re ? rows4[32 * i] : make_uint4(0, 0, 0, 0);
    cut_scores<ROWS>(sm, u0, kw, sel, s, s0);
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
      const uint32_t k = row00 + 32 * i < re ? (uint32_t)score_key(s0[i]) : 0u;
      if (k > ka) { kb = ka; ka = k; } else if (k > kb) { kb = k; }
    }
    uint32_t m1, m2;
    warp_top2(ka, kb, m1, m2);
    if (lane == 0) { s_top[2 * wid] = m1; s_top[2 * wid + 1] = m2; }
    __syncthreads();
    if (wid == 0) {
      const uint32_t v = lane < 2 * nw ? s_top[lane] : 0u;
      uint32_t c1, c2;
      warp_top2(v, 0u, c1, c2);
      if (lane == 0) { ws.cut_smax[2 * vb] = c1; ws.cut_smax[2 * vb + 1] = c2; }
    }
  }
  CUT_STAMP(1);
  // split grid barrier: while the other CTAs finish their sample, score the batches already in
  // the ring (kCutHeld: chunk c0's second batch and stage 1's chunk, or stages 1 .. S - 2) and
  // hold their scores
  const unsigned gen = grid_arrive(ws.bar, G, &s_gen);
  float hs[kCutHeld][ROWS];
#pragma unroll
  for (int hb = 0; hb < kCutHeld; ++hb) {
    const int st = cut_held_stage(hb), bt = cut_held_batch(hb);
    if (hb == 0 || st != cut_held_stage(hb - 1)) cut_wait(&full[st], 0u);
    const int64_t c = stage_chunk[st];
    if (c >= 0) {
      const int64_t r0 = c * kCutChunkRows + bt * kCutBatchRows + boff;
      const uint4* q4 = reinterpret_cast<const uint4*>(stage + st * kCutChunkBytes) + bt * kCutBatchRows + boff;
      uint4 u[ROWS];
#pragma unroll
      for (int i = 0; i < ROWS; ++i) u[i] = r0 + 32 * i < re ? q4[32 * i] : make_uint4(0, 0, 0, 0);
      cut_scores<ROWS>(sm, u, kw, sel, s, hs[hb]);
    } else {
#pragma unroll
      for (int i = 0; i < ROWS; ++i) hs[hb][i] = -INFINITY;
    }
  }
  grid_wait(ws.bar, G, gen);
  CUT_STAMP(2);
  // T = the r-th largest of the 2 G sample maxima at 16-bit key resolution (two 8-bit radix
  // passes in shared memory), rounded down to that key's lower edge
  {
    const int nv = 2 * (int)G;  // <= blockDim (pq_cut_plan)
    const uint32_t v = (int)threadIdx.x < nv ? __ldcg(ws.cut_smax + threadIdx.x) : 0u;
    const bool real = v != 0u;
    uint32_t prefix = 0;
    int64_t need = r;
    for (int pass = 0; pass < 2; ++pass) {
      const int shift = 24 - 8 * pass;
      if (threadIdx.x < 256) h[threadIdx.x] = 0u;
      __syncthreads();
      if (real && (pass == 0 || (v >> 24) == prefix)) atomicAdd(&h[(v >> shift) & 255u], 1u);
      const int have = __syncthreads_count(real && (pass == 0 || (v >> 24) == prefix));
      if (have < need) break;  // fewer than r sampled values (uniform)
      pick_bin256(h, need, &s_b, &s_above);
      __syncthreads();
      need -= s_above;
      prefix = pass == 0 ? (uint32_t)s_b : (prefix << 8) | (uint32_t)s_b;
      if (pass == 1 && threadIdx.x == 0) s_tkey = prefix << 16;
      __syncthreads();
    }
    __syncthreads();
  }
  const uint32_t tkey = s_tkey;
  const float T = key_to_f32(tkey);
  // every row whose exact score x >= T has s32 >= x - eps >= T - eps: it is screened in
  const float t_emit = __fsub_rd(T, eps);
  const bool usable = screen && tkey != 0u && !isnan(t_emit) && !isinf(T);
  const uint64_t tkey64 = score_key((double)T);
  CUT_STAMP(3);

  // ---- 2. emission: the sample rows, the held batches, then the rest of the codes ------------------
  auto emit_batch = [&](const uint4 (&u)[ROWS], const float (&sc)[ROWS], int64_t row0) {
    uint32_t emit = 0;
#pragma unroll
    for (int i = 0; i < ROWS; ++i)
      if (sc[i] >= t_emit && row0 + 32 * i < re) emit |= 1u << i;
    cut_emit<ROWS>(sm, u[0], u[1], u[2], u[3], emit, row0, ids, id_base, cut_count, tkey64, cut_rec, ws.cut_row,
                   key32, ws.cut_cap, kRcCand);
  };
  if (usable) {
    if (__any_sync(0xffffffffu, max4(s0) >= t_emit)) emit_batch(u0, s0, row00);
#pragma unroll 1
    for (int hb = 0; hb < kCutHeld; ++hb) {  // (the held batches' codes are still in their stages)
      if (!__any_sync(0xffffffffu, max4(hs[hb]) >= t_emit)) continue;
      const int st = cut_held_stage(hb), bt = cut_held_batch(hb);
      const int64_t r0 = stage_chunk[st] * kCutChunkRows + bt * kCutBatchRows + boff;
      const uint4* q4 = reinterpret_cast<const uint4*>(stage + st * kCutChunkBytes) + bt * kCutBatchRows + boff;
      uint4 u[ROWS];
#pragma unroll
      for (int i = 0; i < ROWS; ++i) u[i] = r0 + 32 * i < re ? q4[32 * i] : make_uint4(0, 0, 0, 0);
      emit_batch(u, hs[hb], r0);
    }
  }
#ifdef OTF_CUT_NOCOMPUTE
  uint32_t nc_acc = 0u;
#endif
  // stages below kCutHeldStages are consumed: the last warp done with each refills it; a later
  // stage s is first scored at j = s (its phase j / kCutStages, as for every later pass of every stage)
  for (int j = 0;; ++j) {
    const int st = j % kCutStages;
    if (j >= kCutHeldStages) {
      cut_wait(&full[st], (uint32_t)((j / kCutStages) & 1));
      const int64_t c = stage_chunk[st];
      if (c < 0) break;
      const int64_t cr0 = c * kCutChunkRows;
      const bool full_chunk = cr0 + kCutChunkRows <= re;
#pragma unroll 1
      for (int bt = 0; bt < kCutBatches; ++bt) {
        const int off = bt * kCutBatchRows + boff;
        const uint4* rows4 = reinterpret_cast<const uint4*>(stage + st * kCutChunkBytes) + off;
        const int64_t row0 = cr0 + off;
        uint4 u[ROWS];
        float sc[ROWS];
        if (full_chunk) {
#pragma unroll
          for (int i = 0; i < ROWS; ++i) u[i] = rows4[32 * i];
        } else {
#pragma unroll
          for (int i = 0; i < ROWS; ++i) u[i] = row0 + 32 * i < re ? rows4[32 * i] : make_uint4(0, 0, 0, 0);
        }
        if (!usable) continue;
#ifdef OTF_CUT_NOCOMPUTE  // (diagnostic) the ring alone: codes read from the stage, no scoring
#pragma unroll
        for (int i = 0; i < ROWS; ++i) nc_acc ^= u[i].x ^ u[i].y ^ u[i].z ^ u[i].w;
        continue;
#endif
        cut_scores<ROWS>(sm, u, kw, sel, s, sc);
        if (__any_sync(0xffffffffu, max4(sc) >= t_emit)) emit_batch(u, sc, row0);
      }
    } else if (stage_chunk[st] < 0) {
      break;
    }
    __syncwarp();  // this warp's reads of the stage are complete (consumed above)
    if (lane == 0 && atomicAdd(&done[st], 1u) == (unsigned)(nw - 1)) {
      done[st] = 0u;
      const int64_t nc = next_chunk();
      stage_chunk[st] = nc;  // published to the consumers by the barrier phase below
      if (nc >= 0) cut_issue(codes, re, nc * kCutChunkRows, stage + st * kCutChunkBytes, &full[st]);
      else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(cut_smem_u32(&full[st])) : "memory");
    }
  }
  CUT_STAMP(4);
  grid_barrier(ws.bar, G);  // every candidate record is in place
  CUT_STAMP(5);
#ifdef OTF_CUT_NOCOMPUTE
  if (nc_acc == 0x9e3779b9u) ws.cut_word[3] += 1u;  // (keeps the reads)
#ifdef OTF_CUT_TRACE
  if (threadIdx.x == 0)
    printf("cutT cta %d C 0 sample %.2f held %.2f threshold %.2f scan %.2f barrier %.2f select 0 total %.2f\n", (int)vb,
           (ts[1] - ts[0]) * 1e-3, (ts[2] - ts[1]) * 1e-3, (ts[3] - ts[2]) * 1e-3, (ts[4] - ts[3]) * 1e-3,
           (ts[5] - ts[4]) * 1e-3, (ts[5] - ts[0]) * 1e-3);
#endif
#endif

  // ---- 3. selection ----------------------------------------------------------------------------
  // the first kSelPre candidate keys are requested together with the count (one L2 round trip
  // instead of two; keys past the count are stale and ignored)
  constexpr int kSelPre = 4;
  uint32_t kpre[kSelPre];
#pragma unroll
  for (int u = 0; u < kSelPre; ++u) kpre[u] = __ldcg(key32 + threadIdx.x + u * kCutScanThreads);
  const unsigned long long c_all = __ldcg(cut_count);
  const bool ok = usable && c_all >= (unsigned long long)k_eff && c_all <= (unsigned long long)kRcCand;
  // the last CTA done with the shared counters clears them for the next query (on the fast path
  // by the last warp after the keys are in place, off the ranking's critical path)
  auto release_counters = [&]() {
    __threadfence();
    s_last = atomicAdd(ws.cut_word + 6, 1u) == G - 1;
    if (s_last) { ws.cut_word[0] = 0u; ws.cut_word[1] = 0u; ws.cut_word[8] = 0u; ws.cut_word[9] = 0u; ws.cut_word[6] = 0u; }
  };
  if (ok) {
    uint32_t* sk = reinterpret_cast<uint32_t*>(sm);
    const int C = (int)c_all;
#pragma unroll
    for (int u = 0; u < kSelPre; ++u) {
      const int t = threadIdx.x + u * kCutScanThreads;
      if (t < C) sk[t] = kpre[u];
    }
#pragma unroll 4
    for (int t = threadIdx.x + kSelPre * kCutScanThreads; t < C; t += blockDim.x) sk[t] = __ldcg(key32 + t);
    __syncthreads();  // (every thread of the CTA has read the count)
    if (threadIdx.x == kCutScanThreads - 32) release_counters();
    // rank candidates i == vb (mod G): one warp per candidate counts who beats it
    for (int q = (int)vb + wid * (int)G; q < C; q += nw * (int)G) {
      const uint32_t ki = sk[q];
      // the candidate's record and row are in flight during the count (L2 round trips)
      const ulonglong2 ci = __ldcg(cut_rec + q);
      const int64_t ri = __ldcg(ws.cut_row + q);
      int cnt = 0;
      unsigned tie = 0;
#pragma unroll 8
      for (int jj = lane; jj < C; jj += 32) {
        const uint32_t kj = sk[jj];
        cnt += kj > ki;
        tie |= kj == ki && jj != q;
      }
      if (__any_sync(0xffffffffu, tie)) {  // equal prefixes: the full key, then ~id, then the row
        for (int jj = lane; jj < C; jj += 32) {
          if (sk[jj] != ki || jj == q) continue;
          const ulonglong2 cj = __ldcg(cut_rec + jj);
          cnt += cand_greater(cj.x, cj.y, ci.x, ci.y) ||
                 (cj.x == ci.x && cj.y == ci.y && __ldcg(ws.cut_row + jj) < ri);
        }
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      if (lane == 0 && cnt < k_eff) {
        out_ids[cnt] = id_of_inv(ci.y);
        out_scores[cnt] = key_to_f64(ci.x);
        if (out_rows) out_rows[cnt] = ri;
      }
    }
#ifdef OTF_CUT_TRACE
    CUT_STAMP(6);
    if (threadIdx.x == 0)
      printf("cutT cta %d C %d sample %.2f held %.2f threshold %.2f scan %.2f barrier %.2f select %.2f total %.2f\n",
             (int)vb, C, (ts[1] - ts[0]) * 1e-3, (ts[2] - ts[1]) * 1e-3, (ts[3] - ts[2]) * 1e-3, (ts[4] - ts[3]) * 1e-3,
             (ts[5] - ts[4]) * 1e-3, (ts[6] - ts[5]) * 1e-3, (ts[6] - ts[0]) * 1e-3);
#endif
    return;
  }
  // ---- fallback: exact scores of every row, then the exact radix select -------------------------
  // (the LUT replica 0 in global memory is the float64 table the exact scores read)
  __syncthreads();
  if (threadIdx.x == 0) release_counters();
  __syncthreads();
  PqCutSrc src{PqBinSrc{nullptr, codes, lut_g, 16, K}};
  const int64_t nthreads = (int64_t)G * blockDim.x;
  for (int64_t i = (int64_t)vb * blockDim.x + threadIdx.x; i < n; i += nthreads) scratch[i] = src.exact(i, 0u);
  grid_barrier(ws.bar, G);
  if (vb == 0 && threadIdx.x == 0) ws.cut_word[3] += 1u;  // fallbacks taken (diagnostics: otf_repo_cut_fallbacks)
  radix_select_emit(static_cast<const double*>(scratch), src, n, ids, id_base, k_eff, ws, k_eff >= n, sm, out_ids,
                    out_scores, out_rows, h, &s_b, &s_above, vb, G);
}

bool pq_cut_plan(int M, const uint8_t* codes, int64_t n, int64_t k_eff, int device, int* r) {
  static const bool off = getenv("OTF_PQ_NO_CUT") != nullptr;  // A/B switch (tools/)
  if (off || M != 16 || !pq_fast_path(M, codes) || k_eff <= 0) return false;
  const int g = std::min(rank_sms(device), kCutSampleCtasMax);
  if (n < (int64_t)g * kCutChunkRows * 4) return false;  // >= 4 chunks per CTA
  if (2 * g > kCutScanThreads) return false;              // one sample maximum per selecting thread
  const int64_t S = (int64_t)g * kCutBatchRows;            // batch 0 of every CTA's first chunk
  // ~want rows are expected at or above the r-th largest of the S sampled scores (the
  // r-th order statistic of the sample: relative spread ~1/sqrt(r), so fewer than k_eff rows or
  // more than the kRcCand candidate slots of the selection are both many sigmas away); the CTAs
  // publish their top two, so r <= g / 2 keeps the estimate close to the true r-th sample
#ifndef OTF_CUT_WANT16  // expected candidates = k (OTF_CUT_WANT16 / 16) + 128
#define OTF_CUT_WANT16 25
#endif
  // ~k (1 + 4.5 / sqrt(64)) + 128 candidates expected: at r ~ 64 the count's relative spread is
  // ~1/8, so fewer than k (the exact fallback) is ~3.5 sigma away; the rounding of T down to its
  // 16-bit prefix adds margin. Measured: C3 62.5 (2 k + 128) -> 61.8 us, C1 / C2 unchanged;
  // 1.25 k + 128 was faster on C3 (59.9 us) but only ~2 sigma from a fallback.
  const int64_t want = k_eff * OTF_CUT_WANT16 / 16 + 128;
  if (2 * want > kRcCand) return false;
  const int64_t rr = (want * S + n - 1) / n;
  if (rr > g / 2) return false;
  *r = (int)std::max<int64_t>(rr, 1);
  return true;
}

int launch_pq_rank_cut(const float* cents, int K, int Q, const double* w, double* lut, const uint8_t* codes,
                       int64_t n, const int64_t* ids, int64_t id_base, int64_t k_eff, int r, TopkWs* ws,
                       double* scratch, int64_t* out_ids, double* out_scores, int64_t* out_rows, int device,
                       cudaStream_t st) {
  int rc = launch_pq_lut(cents, 16, K, Q, w, lut, st, kCutLutReplicas);
  if (rc) return rc;
  auto fn = pq_rank_cut_kernel;
  static bool configured[64] = {false};
  if (!configured[device & 63]) {
    OTF_CUDA(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRcSmem));
    configured[device & 63] = true;
  }
  const int g = std::min(rank_sms(device), kCutSampleCtasMax);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)g);
  cfg.blockDim = dim3(kCutScanThreads);
  cfg.dynamicSmemBytes = kRcSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap the LUT kernel
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const bool no_pdl = getenv("OTF_PQ_NO_PDL") != nullptr;
  cfg.numAttrs = no_pdl ? 1 : 2;
  OTF_CUDA(cudaLaunchKernelEx(&cfg, fn, codes, n, static_cast<const double*>(lut), K, ids, id_base, k_eff, r, *ws,
                              scratch, out_ids, out_scores, out_rows));
  OTF_LAUNCH_CHECK("pq_rank_cut_kernel");
  return OTF_OK;
}

bool pq_fast_path(int M, const uint8_t* codes) {
  return (((uintptr_t)codes) & 15) == 0 && (M == 4 || M == 8 || M == 16 || M == 32);
}

bool pq_bins_path(int M, const uint8_t* codes) { return M == 16 && pq_fast_path(M, codes); }

int launch_pq_scan_bins(const uint8_t* codes, int64_t n, const double* lut, int K, uint16_t* bins,
                        uint32_t* hist, int device, cudaStream_t st, uint16_t* cmax, int* clog) {
  if (n <= 0) return OTF_OK;
  // 4 rows per thread (software-pipelined, ~112 registers, one 512-thread CTA per SM); 2 rows at
  // 64 registers (two CTAs per SM) rematerialises the per-lane constants and ran 33% slower
  constexpr int ROWS = 4;
  auto fn = pq_scan16_f32bins<ROWS>;
  static int per_sm[64] = {0};
  if (!per_sm[device & 63]) {
    OTF_CUDA(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScanF32Smem));
    int b = 0;
    OTF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kScanF32Threads, kScanF32Smem));
    per_sm[device & 63] = b > 0 ? b : 1;
  }
  int64_t grid = (int64_t)per_sm[device & 63] * sm_count(device);
  const int64_t need = (n + kScanF32Threads * ROWS - 1) / (kScanF32Threads * ROWS);
  if (need < grid) grid = need;
  static const bool no_pdl = getenv("OTF_PQ_NO_PDL") != nullptr;  // A/B switch (tools/)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kScanF32Threads);
  cfg.dynamicSmemBytes = kScanF32Smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap the LUT kernel
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = no_pdl ? 0 : 1;
  OTF_CUDA(cudaLaunchKernelEx(&cfg, fn, codes, n, lut, K, bins, hist, cmax));
  if (cmax && clog) *clog = 7;  // 32 * ROWS rows per chunk
  OTF_LAUNCH_CHECK("pq_scan16_f32bins");
  return OTF_OK;
}

// Scores n code rows. Fast path: the LUT is built in-kernel from (cents, w) when cents is
// non-null, else copied from `lut`. Generic path: `lut` must hold the (M, K) table from
// launch_pq_lut. hist: see launch_dense_score.
int launch_pq_scan(const uint8_t* codes, int64_t n, int M, const float* cents, const double* w,
                   const double* lut, int K, int Q, double* out, uint32_t* hist, int device,
                   cudaStream_t st) {
  if (n <= 0) return OTF_OK;
  if (pq_fast_path(M, codes)) {
    switch (M) {
      case 4: return launch_fast<4>(codes, n, cents, w, cents ? nullptr : lut, K, Q, out, hist, device, st);
      case 8: return launch_fast<8>(codes, n, cents, w, cents ? nullptr : lut, K, Q, out, hist, device, st);
      case 16: return launch_scan16(codes, n, cents, w, cents ? nullptr : lut, K, Q, out, nullptr, hist, device, st);
      case 32: return launch_fast<32>(codes, n, cents, w, cents ? nullptr : lut, K, Q, out, hist, device, st);
      default: break;
    }
  }
  int64_t grid = (n + 255) / 256;
  const int64_t cap = 8LL * sm_count(device);
  if (grid > cap) grid = cap;
  pq_scan_generic<<<(int)grid, 256, 0, st>>>(codes, n, M, lut, K, out, hist);
  OTF_LAUNCH_CHECK("pq_scan_generic");
  return OTF_OK;
}

// ---- pq_encode (pq.py:206-230): the ingest path of PQ repositories ----------------------------
// code[i, m] = argmin_j (|c_mj|^2 - 2 x_im . c_mj) in float64 (|x|^2 is dropped, as the reference
// does), ties and NaNs resolved like numpy's argmin (first minimum / first NaN). |c|^2 follows
// numpy's pairwise order (np.sum, pq.py:222) and 2.0*dot is exact, so the only arithmetic that
// can differ from the reference is the Q-term dot (OpenBLAS dgemm order, not pinnable): codes
// agree except at genuine rounding-level near-ties (tests accept a differing code only where
// the two float64 distances differ by < 1e-12 relative).
//
// Float32 screening, float64 decision: every distance is first computed in float32 (FFMA, twice
// the float64 rate and no float32->float64 conversions), tracking the best and second-best. The
// float32 error of a distance is below eps = 2^-20 (max_j |c_j|^2 + 2 |x| max_j |c_j|) (a 4x
// margin over the FFMA-chain bound), so when the runner-up is more than 2 eps behind, the
// float32 winner is the float64 argmin. Otherwise (near-ties, duplicate centroids, NaN/Inf
// anywhere) the (row, block) is decided by the exact float64 loop with numpy's semantics.
// One thread per row; a CTA keeps the float32 centroids, both norms and per-block bounds of a
// group of G sub-quantizers in shared memory (all lanes read the same centroid: broadcast).
__global__ void pq_cent_norms_kernel(const float* __restrict__ cents, int MK, int Q, double* __restrict__ norms) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < MK; t += gridDim.x * blockDim.x) {
    const float* c = cents + (int64_t)t * Q;
    auto sq = [c](int i) { const double v = (double)c[i]; return __dmul_rn(v, v); };
    norms[t] = pairwise_sum(sq, 0, Q);
  }
}

// per block m: [max_j |c_j|^2, max_j |c_j|, 1 if any centroid or norm is not finite]
__global__ void pq_block_bounds_kernel(const float* __restrict__ cents, const double* __restrict__ norms, int M,
                                       int K, int Q, float* __restrict__ bounds) {
  const int m = blockIdx.x;
  __shared__ float s_n[32], s_c[32];
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  float nmax = 0.f, cmax = 0.f;
  int bad = 0;
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    const double nj = norms[(int64_t)m * K + j];
    if (!isfinite(nj)) bad = 1;
    nmax = fmaxf(nmax, (float)nj);
    cmax = fmaxf(cmax, (float)sqrt(nj));
  }
  for (int o = 16; o; o >>= 1) {
    nmax = fmaxf(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
    cmax = fmaxf(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
  }
  if (bad) atomicOr(&s_bad, 1);
  if ((threadIdx.x & 31) == 0) { s_n[threadIdx.x >> 5] = nmax; s_c[threadIdx.x >> 5] = cmax; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { nmax = fmaxf(nmax, s_n[w]); cmax = fmaxf(cmax, s_c[w]); }
    bounds[3 * m] = nmax;
    bounds[3 * m + 1] = cmax;
    bounds[3 * m + 2] = s_bad ? 1.f : 0.f;
  }
}

__device__ int encode_exact(const float* __restrict__ xs, const float* __restrict__ cg, const double* __restrict__ ng,
                            int K, int Q) {
  double best = 0.0;
  int arg = 0;
  bool nan_seen = false;
  for (int j = 0; j < K; ++j) {
    const float* c = cg + (size_t)j * Q;
    double dot = 0.0;
    for (int q = 0; q < Q; ++q) dot = __fma_rn((double)__ldg(xs + q), (double)c[q], dot);
    const double sq = __dsub_rn(ng[j], 2.0 * dot);
    if (j == 0) {
      best = sq;
      nan_seen = isnan(sq);
    } else if (!nan_seen) {
      if (isnan(sq)) { arg = j; nan_seen = true; }
      else if (sq < best) { best = sq; arg = j; }
    }
  }
  return arg;
}

template <int QR>  // QR > 0: Q == QR, float32 screening in registers; QR == 0: any Q, exact path only
__global__ void __launch_bounds__(256) pq_encode_kernel(const float* __restrict__ X, int64_t n, int dim,
                                                        const float* __restrict__ cents,
                                                        const double* __restrict__ norms,
                                                        const float* __restrict__ bounds, int M, int K, int Q,
                                                        int G, uint8_t* __restrict__ codes) {
  // Two rows per thread and centroids read as float4 (broadcast) so a warp issues ~1 shared
  // load per 7 FFMAs (scalar loads made the first version LSU-bound at 9 loads per 8 FFMAs).
  constexpr int RPT = 2;
  extern __shared__ __align__(16) unsigned char enc_smem[];
  const int m0 = blockIdx.y * G;
  const int g_n = min(G, M - m0);
  const int Kp = (K + 3) & ~3;                                   // padded to whole float4s
  double* sn = reinterpret_cast<double*>(enc_smem);            // [g][Kp] float64 norms
  float* sn32 = reinterpret_cast<float*>(sn + (size_t)G * Kp);  // [g][Kp] float32 norms (+inf pad)
  float* sb = sn32 + (size_t)G * Kp;                            // [g][4] bounds
  float* sc = sb + 4 * G;                                       // [g][Kp][Q] centroids (16-B aligned)
  for (int t = threadIdx.x; t < g_n * Kp; t += blockDim.x) {
    const int g = t / Kp, j = t % Kp;
    const double v = j < K ? norms[(int64_t)(m0 + g) * K + j] : 0.0;
    sn[t] = v;
    sn32[t] = j < K ? (float)v : __int_as_float(0x7f800000);
  }
  for (int t = threadIdx.x; t < 3 * g_n; t += blockDim.x) sb[(t / 3) * 4 + t % 3] = bounds[3 * m0 + t];
  for (int t = threadIdx.x; t < g_n * Kp * Q; t += blockDim.x) {
    const int g = t / (Kp * Q), r = t % (Kp * Q);
    sc[t] = r < K * Q ? cents[((int64_t)(m0 + g) * K) * Q + r] : 0.f;
  }
  __syncthreads();
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * RPT; r0 < n; r0 += nthreads * RPT) {
    for (int g = 0; g < g_n; ++g) {
      const int m = m0 + g;
      const float* cg = sc + (size_t)g * Kp * Q;
      int code[RPT];
#pragma unroll
      for (int u = 0; u < RPT; ++u) code[u] = -1;
      if constexpr (QR > 0) {
        static_assert(QR % 4 == 0, "float4 centroid loads");
        float x[RPT][QR], xx[RPT], d1[RPT], d2[RPT];
        int a1[RPT];
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int64_t row = r0 + u < n ? r0 + u : n - 1;
          const float* xs = X + row * dim + (int64_t)m * QR;
          xx[u] = 0.f;
#pragma unroll
          for (int q = 0; q < QR; ++q) { x[u][q] = __ldg(xs + q); xx[u] = fmaf(x[u][q], x[u][q], xx[u]); }
          d1[u] = d2[u] = __int_as_float(0x7f800000);
          a1[u] = 0;
        }
        const float4* n4 = reinterpret_cast<const float4*>(sn32 + (size_t)g * Kp);
        for (int j0 = 0; j0 < Kp; j0 += 4) {
          const float4 nn = n4[j0 >> 2];
          const float nj[4] = {nn.x, nn.y, nn.z, nn.w};
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const float4* c4 = reinterpret_cast<const float4*>(cg + (size_t)(j0 + jj) * QR);
            float c[QR];
#pragma unroll
            for (int v = 0; v < QR / 4; ++v) {
              const float4 t4 = c4[v];
              c[4 * v] = t4.x; c[4 * v + 1] = t4.y; c[4 * v + 2] = t4.z; c[4 * v + 3] = t4.w;
            }
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
              float dot = 0.f;
#pragma unroll
              for (int q = 0; q < QR; ++q) dot = fmaf(x[u][q], c[q], dot);
              const float d = fmaf(-2.f, dot, nj[jj]);
              const bool lt = d < d1[u];
              d2[u] = lt ? d1[u] : fminf(d2[u], d);
              a1[u] = lt ? j0 + jj : a1[u];
              d1[u] = lt ? d : d1[u];
            }
          }
        }
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const float eps = 0x1p-20f * (sb[4 * g] + 2.f * sqrtf(xx[u]) * sb[4 * g + 1]);
          if (sb[4 * g + 2] == 0.f && d2[u] - d1[u] > 2.f * eps) code[u] = a1[u];  // NaN fails this test
        }
      }
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int64_t row = r0 + u;
        if (row >= n) continue;
        if (code[u] < 0) code[u] = encode_exact(X + row * dim + (int64_t)m * Q, cg, sn + (size_t)g * Kp, K, Q);
        codes[row * M + m] = (uint8_t)code[u];
      }
    }
  }
}

// ---- pq_encode with the dot products on the tensor cores (Q == 8, K <= 256) --------------------
// The FFMA kernel above is energy-bound: 9 FFMA of dot product + 5 compare/select per (row,
// centroid), and back-to-back launches run into power excursions (tools/enc_probe.py). Here the
// x·c dots of a 16-row tile against 8 centroids are ONE legacy tensor-core tile (mma.sync
// m16n8k8 TF32) with three split products (x_hi c_hi + x_hi c_lo + x_lo c_hi, v_hi = v with 13
// low mantissa bits cleared: |dot error| <= 2^-18 sum|x_q c_q|), so only the distance and the
// running (best, second-best) stay on the SIMT pipes. The centroid index rides in the low 8
// mantissa bits of each distance (relative perturbation <= 2^-15), so the running minimum and
// second minimum are 3 FMNMX per candidate with the argmin included. The float32 winner is
// taken when the runner-up is more than 2 eps + the perturbation behind, eps = 2^-16 (max_j
// |c_j|^2 + 2 |x| max_j |c_j|) (>2x the bound above); otherwise (near-ties, non-finite data) the
// (row, block) is decided by encode_exact in float64 with numpy's semantics, as before.
// One warp = 16 rows of one sub-quantizer; blockIdx.y = the sub-quantizer.
constexpr int kEncMmaThreads = 256;

// encode_exact for Q == 8 with the whole warp: lane l scores centroids l, l + 32, ... in float64
// (the same arithmetic as encode_exact), then a warp argmin with numpy's semantics (the first
// NaN if any, else the first minimum).
__device__ int encode_exact_warp(const float* __restrict__ xs, const float* __restrict__ cg,
                                 const double* __restrict__ ng, int K, int lane) {
  double x[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) x[q] = (double)__ldg(xs + q);
  int arg = -1;
  double best = 0.0;
  bool nan_seen = false;
  for (int j = lane; j < K; j += 32) {
    const float* c = cg + j * 8;
    double dot = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) dot = __fma_rn(x[q], (double)c[q], dot);
    const double sq = __dsub_rn(ng[j], 2.0 * dot);
    if (arg < 0) {
      best = sq; arg = j; nan_seen = isnan(sq);
    } else if (!nan_seen) {
      if (isnan(sq)) { best = sq; arg = j; nan_seen = true; }
      else if (sq < best) { best = sq; arg = j; }
    }
  }
  // (nan first, then smaller value, then smaller index); lanes without a centroid lose
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
    const bool on = __shfl_xor_sync(0xffffffffu, (int)nan_seen, o) != 0;
    bool take;
    if (oa < 0) take = false;
    else if (arg < 0) take = true;
    else if (nan_seen != on) take = on;
    else if (nan_seen) take = oa < arg;
    else take = ob < best || (ob == best && oa < arg);
    if (take) { best = ob; arg = oa; nan_seen = on; }
  }
  return arg;
}

__device__ __forceinline__ void mma_tf32_m16n8k8(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t tf32_hi(float v) { return __float_as_uint(v) & 0xFFFFE000u; }
__device__ __forceinline__ uint32_t tf32_lo(float v) { return __float_as_uint(__fsub_rn(v, __uint_as_float(tf32_hi(v)))); }
// distance with the centroid index in its low 8 mantissa bits (padding: +inf -> a NaN pattern,
// which fminf/fmaxf ignore)
__device__ __forceinline__ float enc_key(float d, int j) {
  return __uint_as_float((__float_as_uint(d) & ~0xFFu) | (uint32_t)j);
}
__device__ __forceinline__ void enc_upd(float& b, float& s, float k) {
  s = fminf(s, fmaxf(b, k));
  b = fminf(b, k);
}

__global__ void __launch_bounds__(kEncMmaThreads) pq_encode_mma(const float* __restrict__ X, int64_t n, int dim,
                                                                const float* __restrict__ cents,
                                                                const double* __restrict__ norms,
                                                                const float* __restrict__ bounds, int M, int K,
                                                                uint8_t* __restrict__ codes) {
  constexpr int Q = 8;
  const int m = blockIdx.y;
  __shared__ __align__(16) uint4 sB[32 * 32];  // [n-tile][lane]: {hi(c[j][t4]), hi(c[j][t4+4]), lo(..), lo(..)}, j = 8nt+g
  __shared__ __align__(16) float sC[256 * Q];  // natural layout (exact path)
  __shared__ __align__(8) float sN[256];       // float32 norms, +inf past K
  __shared__ double sN64[256];                 // float64 norms (exact path)
  const float* cm = cents + (int64_t)m * K * Q;
  for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
    const int l = e & 31, j = (e >> 5) * 8 + (l >> 2), t4 = l & 3;
    const float c0 = j < K ? cm[j * Q + t4] : 0.f, c1 = j < K ? cm[j * Q + t4 + 4] : 0.f;
    sB[e] = make_uint4(tf32_hi(c0), tf32_hi(c1), tf32_lo(c0), tf32_lo(c1));
  }
  for (int e = threadIdx.x; e < 256 * Q; e += blockDim.x) sC[e] = e < K * Q ? cm[e] : 0.f;
  for (int j = threadIdx.x; j < 256; j += blockDim.x) {
    const double v = j < K ? norms[(int64_t)m * K + j] : 0.0;
    sN64[j] = v;
    sN[j] = j < K ? (float)v : __int_as_float(0x7f800000);
  }
  __syncthreads();
  const float cmax2 = bounds[3 * m], cmax = bounds[3 * m + 1];
  const bool bad = bounds[3 * m + 2] != 0.f;
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const int ntiles = (K + 7) >> 3;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 16; r0 < n; r0 += warps * 16) {
    const int64_t ra = r0 + g, rb = ra + 8;
    const float* xa = X + (ra < n ? ra : n - 1) * dim + m * Q;
    const float* xb = X + (rb < n ? rb : n - 1) * dim + m * Q;
    const float xa0 = __ldg(xa + t4), xa1 = __ldg(xa + t4 + 4), xb0 = __ldg(xb + t4), xb1 = __ldg(xb + t4 + 4);
    // A fragments (m16n8k8 row-major): a0 (row g, k t4), a1 (row g+8, k t4), a2 (row g, k t4+4), a3 (row g+8, k t4+4)
    const uint32_t ah[4] = {tf32_hi(xa0), tf32_hi(xb0), tf32_hi(xa1), tf32_hi(xb1)};
    const uint32_t al[4] = {tf32_lo(xa0), tf32_lo(xb0), tf32_lo(xa1), tf32_lo(xb1)};
    float qa = fmaf(xa0, xa0, xa1 * xa1), qb = fmaf(xb0, xb0, xb1 * xb1);  // |x|^2 over the quad
    qa += __shfl_xor_sync(0xffffffffu, qa, 1);
    qb += __shfl_xor_sync(0xffffffffu, qb, 1);
    qa += __shfl_xor_sync(0xffffffffu, qa, 2);
    qb += __shfl_xor_sync(0xffffffffu, qb, 2);
    const float inf = __int_as_float(0x7f800000);
    float ba = inf, sa = inf, bb = inf, sb2 = inf;  // (best, second) keys of rows g and g+8
    for (int nt = 0; nt < ntiles; ++nt) {
      const uint4 f = sB[nt * 32 + lane];
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      mma_tf32_m16n8k8(acc, ah, f.x, f.y);
      mma_tf32_m16n8k8(acc, ah, f.z, f.w);
      mma_tf32_m16n8k8(acc, al, f.x, f.y);
      const int j0 = nt * 8 + 2 * t4;  // C fragment: c0,c1 (row g, cols 2t4, 2t4+1), c2,c3 (row g+8)
      const float2 nn = *reinterpret_cast<const float2*>(sN + j0);
      enc_upd(ba, sa, enc_key(fmaf(-2.f, acc[0], nn.x), j0));
      enc_upd(ba, sa, enc_key(fmaf(-2.f, acc[1], nn.y), j0 + 1));
      enc_upd(bb, sb2, enc_key(fmaf(-2.f, acc[2], nn.x), j0));
      enc_upd(bb, sb2, enc_key(fmaf(-2.f, acc[3], nn.y), j0 + 1));
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {  // merge the quad's (best, second) pairs
      const float oba = __shfl_xor_sync(0xffffffffu, ba, o), osa = __shfl_xor_sync(0xffffffffu, sa, o);
      const float obb = __shfl_xor_sync(0xffffffffu, bb, o), osb = __shfl_xor_sync(0xffffffffu, sb2, o);
      sa = fminf(fminf(sa, osa), fmaxf(ba, oba));
      ba = fminf(ba, oba);
      sb2 = fminf(fminf(sb2, osb), fmaxf(bb, obb));
      bb = fminf(bb, obb);
    }
    // decide: lanes t4 == 0 hold rows g (h = 0) and g + 8 (h = 1)
    bool amb[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t row = h ? rb : ra;
      const float b = h ? bb : ba, s2 = h ? sb2 : sa;
      const float eps = 0x1p-16f * (cmax2 + 2.f * sqrtf(h ? qb : qa) * cmax);
      const float pert = 0x1p-14f * (fabsf(b) + fabsf(s2)) + 0x1p-140f;
      const bool ok = !bad && s2 - b > 2.f * eps + pert;  // NaN fails this test
      amb[h] = t4 == 0 && row < n && !ok;
      if (t4 == 0 && row < n && ok) codes[row * M + m] = (uint8_t)(__float_as_uint(b) & 0xFFu);
    }
    // rare: near-ties / non-finite data — the whole warp computes that (row, block)'s float64
    // distances (8 centroids per lane) and takes numpy's argmin
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      unsigned todo = __ballot_sync(0xffffffffu, amb[h]);
      while (todo) {
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
        const int64_t row = r0 + (src >> 2) + 8 * h;
        const int code = encode_exact_warp(X + row * dim + (int64_t)m * Q, sC, sN64, K, lane);
        if (lane == 0) codes[row * M + m] = (uint8_t)code;
      }
    }
  }
}

// vectors (n, M*Q) float32, centroids (M, K, Q) float32 on the device -> codes (n, M) uint8.
// scratch: M*K float64 norms + 3*M float32 bounds (pq_encode_scratch_bytes).
size_t pq_encode_scratch_bytes(int M, int K) { return (size_t)M * K * 8 + (size_t)M * 3 * 4 + 16; }

int launch_pq_encode(const float* X, int64_t n, int M, int K, int Q, const float* cents, void* scratch,
                     uint8_t* codes, int device, cudaStream_t st) {
  if (n <= 0) return OTF_OK;
  if (K < 1 || K > 256) return fail(OTF_ERR_CONFIG, "num_centroids must be in 1..256");
  double* norms = static_cast<double*>(scratch);
  float* bounds = reinterpret_cast<float*>(norms + (size_t)M * K);
  const int MK = M * K;
  pq_cent_norms_kernel<<<(MK + 255) / 256, 256, 0, st>>>(cents, MK, Q, norms);
  OTF_LAUNCH_CHECK("pq_cent_norms_kernel");
  pq_block_bounds_kernel<<<M, 256, 0, st>>>(cents, norms, M, K, Q, bounds);
  OTF_LAUNCH_CHECK("pq_block_bounds_kernel");
  static const bool ffma = getenv("OTF_PQ_ENCODE_FFMA") != nullptr;  // A/B switch (tools/)
  if (Q == 8 && !ffma) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pq_encode_mma, kEncMmaThreads, 0);
    if (per_sm < 1) per_sm = 1;
    int64_t bx = ((int64_t)per_sm * sm_count(device) + M - 1) / M;  // CTAs per sub-quantizer
    const int64_t need = (n + (kEncMmaThreads / 32) * 16 - 1) / ((kEncMmaThreads / 32) * 16);
    if (need < bx) bx = need;
    if (bx < 1) bx = 1;
    pq_encode_mma<<<dim3((unsigned)bx, (unsigned)M), kEncMmaThreads, 0, st>>>(X, n, M * Q, cents, norms, bounds, M,
                                                                             K, codes);
    OTF_LAUNCH_CHECK("pq_encode_mma");
    return OTF_OK;
  }
  const size_t Kp = (size_t)((K + 3) & ~3);
  const size_t per_m = Kp * Q * 4 + Kp * 12 + 16;
  const size_t budget = 200 * 1024;
  if (per_m > budget) return fail(OTF_ERR_CONFIG, "sub-quantizer too large for pq_encode (K*Q*4 > 200 KB)");
  const int G = (int)std::min<size_t>((size_t)M, budget / per_m);
  const size_t smem = per_m * G;
  const int groups = (M + G - 1) / G;
  const int dim = M * Q;
  auto launch = [&](auto fn) -> int {
    OTF_CUDA(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem);
    if (per_sm < 1) per_sm = 1;
    int64_t bx = (int64_t)per_sm * sm_count(device);
    const int64_t need = (n + 511) / 512;  // two rows per thread
    if (need < bx) bx = need;
    fn<<<dim3((unsigned)bx, (unsigned)groups), 256, smem, st>>>(X, n, dim, cents, norms, bounds, M, K, Q, G, codes);
    OTF_LAUNCH_CHECK("pq_encode_kernel");
    return OTF_OK;
  };
  switch (Q) {
    case 4: return launch(pq_encode_kernel<4>);
    case 8: return launch(pq_encode_kernel<8>);
    case 16: return launch(pq_encode_kernel<16>);
    default: return launch(pq_encode_kernel<0>);
  }
}

}  // namespace otf
