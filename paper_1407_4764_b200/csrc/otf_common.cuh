// otf_common.cuh — shared device/host helpers for the sm_100a retrieval kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "otf_b200.h"

namespace otf {

// ---- error plumbing ------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
void count_launch(int n = 1);

#define OTF_CUDA(expr)                                   \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return ::otf::cuda_fail(_e, #expr); \
  } while (0)

#define OTF_LAUNCH_CHECK(name)                                  \
  do {                                                          \
    ::otf::count_launch();                                      \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e != cudaSuccess) return ::otf::cuda_fail(_e, name);   \
  } while (0)

// ---- device properties (cached per device) ----------------------------------------------
int sm_count(int device);

// ---- order-preserving keys ------------------------------------------------------------------
// Larger key <=> larger score. -0.0 is canonicalised to +0.0 so that they tie
// (the reference's np.partition / lexsort treat them as equal, ranker.py:126-134).
__device__ __forceinline__ uint64_t score_key(float s) {
  uint32_t u = __float_as_uint(s);
  if (u == 0x80000000u) u = 0u;
  uint32_t k = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return (uint64_t)k;
}
__device__ __forceinline__ uint64_t score_key(double s) {
  uint64_t u = (uint64_t)__double_as_longlong(s);
  if (u == 0x8000000000000000ull) u = 0ull;
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
template <typename T> struct KeyBits;
template <> struct KeyBits<float> { static constexpr int value = 32; };
template <> struct KeyBits<double> { static constexpr int value = 64; };

// ---- coarse score histogram fused into the scoring kernels ---------------------------------
// 4096 bins = the top 12 bits of the float32 order key (sign, 8 exponent bits, 3 mantissa
// bits). float64 scores are bucketed through their float32 rounding, which is monotone, so a
// bin ordering is always consistent with the exact score ordering. The top-k kernel uses the
// histogram to find the bin that holds the k-th best entry without another pass over N.
constexpr int kHistBins = 4096;
__device__ __forceinline__ uint32_t hist_bin(float s) { return (uint32_t)(score_key(s) >> 20); }
__device__ __forceinline__ uint32_t hist_bin(double s) { return hist_bin(__double2float_rn(s)); }

// The PQ rank path (exact bins, otf_pq.cu pq_scan16_f32bins) uses 13 key bits / 8192 bins: its
// threshold bin holds about half the rows, so the top-k ranks about half the candidates; the
// dense and binary scans keep 4096 bins (their scans pay for a larger histogram more than their
// top-k gains). kHistBinsMax sizes the shared workspace.
constexpr int kPqHistBits = 13;
constexpr int kPqHistBins = 1 << kPqHistBits;
constexpr int kHistBinsMax = kPqHistBins;
__device__ __forceinline__ uint32_t pq_hist_bin(float s) { return (uint32_t)(score_key(s) >> (32 - kPqHistBits)); }
__device__ __forceinline__ uint32_t pq_hist_bin(double s) { return pq_hist_bin(__double2float_rn(s)); }

__device__ __forceinline__ void hist_zero(uint32_t* sh, int nb = kHistBins) {
  for (int b = threadIdx.x; b < nb; b += blockDim.x) sh[b] = 0u;
}
// Shared-memory histogram update. Plain per-lane ATOMS: the scores of neighbouring rows
// rarely share a bin, and __match_any_sync (ADU pipe) cost more than the replays it saves
// (57% ADU utilisation in the r1 PQ profile).
__device__ __forceinline__ void hist_add(uint32_t* sh, bool active, uint32_t bin) {
  if (active) atomicAdd(&sh[bin], 1u);
}
__device__ __forceinline__ void hist_flush(const uint32_t* sh, uint32_t* g, int nb = kHistBins) {
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (sh[b]) atomicAdd(&g[b], sh[b]);
}

// Streaming 128-bit loads of the repository (read once per query): no L1 allocation, and an
// L2 evict-first policy, so a 0.16-51 GB scan does not push the hot lines out of L2 every query
// (the top-k kernel's code and workspaces, the LUT, the histogram, the candidate buffers).
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
#ifndef OTF_NO_EVICT_FIRST
__device__ __forceinline__ float4 ld_stream_f4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(l2_evict_first()));
  return r;
}
__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(l2_evict_first()));
  return r;
}
#else
__device__ __forceinline__ float4 ld_stream_f4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
#endif

__device__ __forceinline__ double shfl_xor_d(double v, int o) {
  return __shfl_xor_sync(0xffffffffu, v, o);
}

// Transposed butterfly reduction of R per-lane partial vectors across the LPR lanes of a
// lane group (LPR power of two <= 32, R power of two <= LPR). On return p[0] of lane
// (g*LPR + j) holds the full sum for row index ((j / (LPR/R)) ... ) — see row_of_lane().
// Every row is summed with the SAME tree: pairs (l, l^(LPR/2)), then (l, l^(LPR/4)), ...
// so the result for a row does not depend on which lane or slot it occupied.
template <int R, int LPR>
__device__ __forceinline__ void transposed_reduce(double (&p)[R], int lane) {
  int count = R;
#pragma unroll
  for (int o = LPR / 2; o >= 1; o >>= 1) {
    if (count > 1) {
      const int half = count >> 1;
      const bool upper = (lane & o) != 0;
#pragma unroll
      for (int j = 0; j < R / 2; ++j) {
        if (j < half) {
          double send = upper ? p[j] : p[j + half];
          double keep = upper ? p[j + half] : p[j];
          double recv = shfl_xor_d(send, o);
          p[j] = __dadd_rn(keep, recv);
        }
      }
      count = half;
    } else {
      p[0] = __dadd_rn(p[0], shfl_xor_d(p[0], o));
    }
  }
}
// float32 variant (same tree).
template <int R, int LPR>
__device__ __forceinline__ void transposed_reduce_f(float (&p)[R], int lane) {
  int count = R;
#pragma unroll
  for (int o = LPR / 2; o >= 1; o >>= 1) {
    if (count > 1) {
      const int half = count >> 1;
      const bool upper = (lane & o) != 0;
#pragma unroll
      for (int j = 0; j < R / 2; ++j) {
        if (j < half) {
          const float send = upper ? p[j] : p[j + half];
          const float keep = upper ? p[j + half] : p[j];
          p[j] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, o));
        }
      }
      count = half;
    } else {
      p[0] = __fadd_rn(p[0], __shfl_xor_sync(0xffffffffu, p[0], o));
    }
  }
}
// Row slot (0..R-1) that lane `lane` holds after transposed_reduce<R, LPR>, and whether it
// is the designated writer for that row.
template <int R, int LPR>
__device__ __forceinline__ int row_of_lane(int lane, bool* writer) {
  int row = 0, half = R;
  int o = LPR / 2;
  int levels_transposed = 0;
  for (int c = R; c > 1; c >>= 1) ++levels_transposed;
  for (int l = 0; l < levels_transposed; ++l) {
    half >>= 1;
    if (lane & o) row += half;
    o >>= 1;
  }
  // remaining low lane bits (below o*2) were plain-reduced: lanes agree; lowest writes
  const int low_mask = (LPR / R) - 1;
  *writer = ((lane & (LPR - 1)) & low_mask) == 0;
  return row;
}

}  // namespace otf
