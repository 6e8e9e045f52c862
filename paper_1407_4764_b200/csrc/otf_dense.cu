// otf_dense.cu — K1: dense float32 linear-SVM scoring (score_dense, ranker.py:63-69).
//
// s_i = float32( sum_j x_ij * float32(w_j) ). The reference computes this dot product with an
// OpenBLAS sgemv (float32 FMA accumulation, host-CPU dependent order), so parity is a stated
// tolerance. Here each 4-column chunk is a float32 FMA chain and the chunk
// sums are accumulated in float64, so the error is that of a 4-term float32 dot, well inside
// the reference's own rounding. Every row is reduced with the same fixed tree whatever its
// position, GPU or shard, so a row's score is bit-identical across repositories, subsets
// (without_ids) and GPU counts.
//
// Canonical per-row order (shared by all variants below): lane l of a 32-lane group owns the
// 4-column chunks {128*c + 4*l : c = 0..}; chunk sums (chunk_dot) are added in c order into a
// float64 partial; the 32 partials are then combined by the xor-butterfly tree
// (l, l^16), (l, l^8), ..., (l, l^1).
//
// The float64 -> float32 cast of w (ranker.py:69) happens while w is staged into shared
// memory, and the kernel also builds the coarse score histogram the top-k kernel starts from
// (otf_common.cuh, hist_*), so one query = this kernel + the top-k kernel.
//
// HBM roofline: 4*d bytes per row; 0.5 flop/byte. Loads are 128-bit, coalesced, streamed
// past L1 (ld.global.nc.L1::no_allocate); the grid is persistent (a multiple of the 148 SMs).
#include "otf_common.cuh"
#include "otf_internal.h"

namespace otf {

// One 4-column chunk: float32 FMA chain x0*w0 (+x1*w1)(+x2*w2)(+x3*w3), the same in every
// variant. Chunk sums are then accumulated in float64; this keeps the float64->float32 XU
// conversions at one per 4 columns (two per column saturated the XU pipe at 77%, ncu r1).
__device__ __forceinline__ float chunk_dot(const float4 x, const float4 w) {
  float s = __fmul_rn(x.x, w.x);
  s = __fmaf_rn(x.y, w.y, s);
  s = __fmaf_rn(x.z, w.z, s);
  return __fmaf_rn(x.w, w.w, s);
}

// Fast path: d == 128 * CPL. Each warp handles R rows per iteration, then a transposed
// butterfly gives ~2 shuffles per row.
template <int CPL, int R>
__global__ void __launch_bounds__(256, 2) dense_score_fast(const float* __restrict__ X, int64_t n,
                                                           const double* __restrict__ w,
                                                           float* __restrict__ out,
                                                           uint32_t* __restrict__ ghist,
                                                           uint16_t* __restrict__ cmax) {
  const int lane = threadIdx.x & 31;
  __shared__ float4 wr[32 * CPL];
  __shared__ uint32_t sh[kHistBins];
  for (int t = threadIdx.x; t < 32 * CPL; t += blockDim.x)
    wr[t] = make_float4(__double2float_rn(w[4 * t]), __double2float_rn(w[4 * t + 1]),
                        __double2float_rn(w[4 * t + 2]), __double2float_rn(w[4 * t + 3]));
  if (ghist) hist_zero(sh);
  __syncthreads();
  const int64_t row_f4 = 32 * CPL;  // float4 per row
  const float4* X4 = reinterpret_cast<const float4*>(X);
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int LB = CPL < 8 ? CPL : 8;  // float4 loads per row per batch
  for (int64_t r0 = warp * R; r0 < n; r0 += nwarp * R) {
    double p[R];
#pragma unroll
    for (int i = 0; i < R; ++i) p[i] = 0.0;
#pragma unroll
    for (int c0 = 0; c0 < CPL; c0 += LB) {
      float4 v[R][LB];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int64_t row = r0 + i;
#pragma unroll
        for (int c = 0; c < LB; ++c) {
          if (row < n) v[i][c] = ld_stream_f4(X4 + row * row_f4 + lane + 32 * (c0 + c));
          else v[i][c] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int i = 0; i < R; ++i) {
        double acc = p[i];
#pragma unroll
        for (int c = 0; c < LB; ++c) {
          acc = __dadd_rn(acc, (double)chunk_dot(v[i][c], wr[lane + 32 * (c0 + c)]));
        }
        p[i] = acc;
      }
    }
    transposed_reduce<R, 32>(p, lane);
    bool writer;
    const int slot = row_of_lane<R, 32>(lane, &writer);
    const int64_t row = r0 + slot;
    const bool active = writer && row < n;
    const float s = __double2float_rn(p[0]);
    if (active) out[row] = s;
    if (ghist) hist_add(sh, active, hist_bin(s));
    if (R > 1 && cmax) {  // the warp's R consecutive rows are one top-k chunk
      const uint32_t wm = __reduce_max_sync(0xffffffffu, active ? hist_bin(s) : 0u);
      if (lane == 0) cmax[r0 / R] = (uint16_t)wm;
    }
  }
  if (ghist) {
    __syncthreads();
    hist_flush(sh, ghist);
  }
}

// Generic path: any d (and any alignment). One warp per row, same canonical order.
__global__ void __launch_bounds__(256) dense_score_generic(const float* __restrict__ X, int64_t n,
                                                           int32_t d, const double* __restrict__ w,
                                                           float* __restrict__ out,
                                                           uint32_t* __restrict__ ghist) {
  __shared__ uint32_t sh[kHistBins];
  if (ghist) hist_zero(sh);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = warp; row < n; row += nwarp) {
    const float* x = X + row * (int64_t)d;
    double acc = 0.0;
    for (int base = 4 * lane; base < d; base += 128) {
      const int m = d - base < 4 ? d - base : 4;
      float cs = __fmul_rn(__ldg(x + base), __double2float_rn(w[base]));
      for (int e = 1; e < m; ++e) cs = __fmaf_rn(__ldg(x + base + e), __double2float_rn(w[base + e]), cs);
      acc = __dadd_rn(acc, (double)cs);
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

static int grid_for(const void* fn, int threads, int device) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0);
  if (per_sm < 1) per_sm = 1;
  return per_sm * sm_count(device);
}

template <int CPL, int R>
static int launch_fast(const float* X, int64_t n, const double* w, float* out, uint32_t* hist,
                       int device, cudaStream_t st, uint16_t* cmax, int* clog) {
  auto fn = dense_score_fast<CPL, R>;
  int grid = grid_for((const void*)fn, 256, device);
  const int64_t need = (n + (8 * R) - 1) / (8 * R);  // 8 warps per block
  if (need < grid) grid = (int)(need > 0 ? need : 1);
  if (R < 8) cmax = nullptr;  // chunks of >= 8 rows only (topk_cmax_ensure)
  fn<<<grid, 256, 0, st>>>(X, n, w, out, hist, cmax);
  OTF_LAUNCH_CHECK("dense_score_fast");
  if (cmax && clog) *clog = R == 8 ? 3 : R == 16 ? 4 : 5;  // log2(R)
  return OTF_OK;
}

// Scores n rows against the float64 model w (cast to float32 in-kernel). Pointers must be
// 16-byte aligned for the fast path (all device buffers this library allocates are).
// hist (nullable): kHistBins counters (zero on entry) receiving the coarse score histogram.
int launch_dense_score(const float* X, int64_t n, int32_t d, const double* w, float* out,
                       uint32_t* hist, int device, cudaStream_t st, uint16_t* cmax, int* clog) {
  if (n <= 0) return OTF_OK;
  const bool aligned = (((uintptr_t)X) & 15) == 0;
  if (aligned && d % 128 == 0) {
    switch (d / 128) {
      case 1: return launch_fast<1, 32>(X, n, w, out, hist, device, st, cmax, clog);  // R 8/16: 5% slower (C1)
      case 2: return launch_fast<2, 4>(X, n, w, out, hist, device, st, cmax, clog);
      case 4: return launch_fast<4, 2>(X, n, w, out, hist, device, st, cmax, clog);
      case 8: return launch_fast<8, 1>(X, n, w, out, hist, device, st, cmax, clog);
      case 16: return launch_fast<16, 2>(X, n, w, out, hist, device, st, cmax, clog);  // R 1 / 4: +0.6% / +2.8%
      case 32: return launch_fast<32, 1>(X, n, w, out, hist, device, st, cmax, clog);
      default: break;
    }
  }
  int grid = grid_for((const void*)dense_score_generic, 256, device);
  const int64_t need = (n + 7) / 8;
  if (need < grid) grid = (int)need;
  dense_score_generic<<<grid, 256, 0, st>>>(X, n, d, w, out, hist);
  OTF_LAUNCH_CHECK("dense_score_generic");
  return OTF_OK;
}

}  // namespace otf
