// otf_train.cu — K6: the Pegasos hinge-loss update (trainer.py:51-71) on a sampled balanced
// mini-batch (trainer.py:95-106), plus row/id gathers used by Repository.without_ids.
//
// One CTA does the whole step (B = 2*half rows of d floats is tiny); it runs on the
// trainer's own high-priority stream so it overlaps the ranker's HBM-bound scan.
//   margins_b = y_b * <x_b, w>             (float64; BLAS dgemv order differs -> tolerance)
//   V = margins < 1
//   g_j = 0.0 + sum_{b in V, in order} y_b x_bj   (numpy add.reduce over axis 0: sequential
//                                                  from the identity, exact sign flips)
//   w'_j = RN(RN(shrink*w_j) + RN(eta_over_b*g_j))  with shrink = 1-eta*lam, eta_over_b = eta/B
//   if project and ||w'|| > radius: w' *= RN(radius/||w'||)
// __dmul_rn/__dadd_rn stop FMA contraction so the elementwise update matches numpy exactly.
#include "otf_common.cuh"
#include "otf_internal.h"

namespace otf {

__device__ __forceinline__ double load_as_f64(const void* base, int dtype, int64_t idx) {
  return dtype == OTF_F32 ? (double)static_cast<const float*>(base)[idx]
                          : static_cast<const double*>(base)[idx];
}

__global__ void __launch_bounds__(1024, 1)
pegasos_kernel(double* __restrict__ w, int d, const void* __restrict__ pos, int pos_dtype,
               const void* __restrict__ neg, int neg_dtype, const int64_t* __restrict__ pos_idx,
               const int64_t* __restrict__ neg_idx, int half, double shrink, double eta_over_b,
               int project, double radius) {
  extern __shared__ double sm[];  // [B] labels*margins flags, then reduction scratch
  int* viol = reinterpret_cast<int*>(sm);
  double* red = sm + 2 * half;    // 32 doubles
  const int B = 2 * half;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int b = wid; b < B; b += nw) {
    const bool is_pos = b < half;
    const int64_t r = is_pos ? pos_idx[b] : neg_idx[b - half];
    const void* base = is_pos ? pos : neg;
    const int dt = is_pos ? pos_dtype : neg_dtype;
    double acc = 0.0;
    for (int j = lane; j < d; j += 32) acc = __fma_rn(load_as_f64(base, dt, r * d + j), w[j], acc);
    for (int o = 16; o >= 1; o >>= 1) acc = __dadd_rn(acc, shfl_xor_d(acc, o));
    if (lane == 0) {
      const double margin = is_pos ? acc : -acc;
      viol[b] = margin < 1.0;
    }
  }
  __syncthreads();
  double sq = 0.0;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double g = 0.0;
    for (int b = 0; b < B; ++b) {
      if (!viol[b]) continue;
      const bool is_pos = b < half;
      const int64_t r = is_pos ? pos_idx[b] : neg_idx[b - half];
      const double x = load_as_f64(is_pos ? pos : neg, is_pos ? pos_dtype : neg_dtype, r * d + j);
      g = __dadd_rn(g, is_pos ? x : -x);
    }
    const double nw_j = __dadd_rn(__dmul_rn(shrink, w[j]), __dmul_rn(eta_over_b, g));
    w[j] = nw_j;
    sq = __fma_rn(nw_j, nw_j, sq);
  }
  if (!project) return;
  for (int o = 16; o >= 1; o >>= 1) sq = __dadd_rn(sq, shfl_xor_d(sq, o));
  if (lane == 0) red[wid] = sq;
  __syncthreads();
  if (wid == 0) {
    double v = lane < nw ? red[lane] : 0.0;
    for (int o = 16; o >= 1; o >>= 1) v = __dadd_rn(v, shfl_xor_d(v, o));
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  const double norm = sqrt(red[0]);
  if (norm > radius) {
    const double scale = __ddiv_rn(radius, norm);
    for (int j = threadIdx.x; j < d; j += blockDim.x) w[j] = __dmul_rn(w[j], scale);
  }
}

int launch_pegasos(double* w, int d, const void* pos, int pos_dtype, int64_t n_pos,
                   const void* neg, int neg_dtype, int64_t n_neg, const int64_t* pos_idx,
                   const int64_t* neg_idx, int half, double shrink, double eta_over_b,
                   int project, double radius, cudaStream_t st) {
  (void)n_pos; (void)n_neg;
  int threads = 1024;
  if (d < 1024) threads = ((d + 31) / 32) * 32 < 256 ? 256 : ((d + 31) / 32) * 32;
  const size_t smem = (size_t)(2 * half) * sizeof(double) + 32 * sizeof(double);
  pegasos_kernel<<<1, threads, smem, st>>>(w, d, pos, pos_dtype, neg, neg_dtype, pos_idx, neg_idx,
                                           half, shrink, eta_over_b, project, radius);
  OTF_LAUNCH_CHECK("pegasos_kernel");
  return OTF_OK;
}

// ---- gathers for Repository.without_ids (ranker.py:254-270) -------------------------------
__global__ void gather_rows_kernel(const uint8_t* __restrict__ src, int64_t row_bytes,
                                   const int64_t* __restrict__ rows, int64_t n,
                                   uint8_t* __restrict__ dst) {
  // one warp per row, 16-byte chunks when both ends are aligned, bytes otherwise
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec = (row_bytes % 16) == 0 && (((uintptr_t)src | (uintptr_t)dst) & 15) == 0;
  for (int64_t i = warp; i < n; i += nwarp) {
    const uint8_t* s = src + rows[i] * row_bytes;
    uint8_t* t = dst + i * row_bytes;
    if (vec) {
      const uint4* s4 = reinterpret_cast<const uint4*>(s);
      uint4* t4 = reinterpret_cast<uint4*>(t);
      for (int64_t q = lane; q < row_bytes / 16; q += 32) t4[q] = s4[q];
    } else {
      for (int64_t q = lane; q < row_bytes; q += 32) t[q] = s[q];
    }
  }
}

__global__ void gather_i64_kernel(const int64_t* __restrict__ src, const int64_t* __restrict__ rows,
                                  int64_t n, int64_t base, int64_t* __restrict__ dst) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = src ? src[rows[i]] : base + rows[i];
}

int launch_gather_rows(const uint8_t* src, int64_t row_bytes, const int64_t* rows, int64_t n,
                       uint8_t* dst, int device, cudaStream_t st) {
  if (n <= 0) return OTF_OK;
  int64_t grid = (n + 7) / 8;
  const int64_t cap = 8LL * sm_count(device);
  if (grid > cap) grid = cap;
  gather_rows_kernel<<<(int)grid, 256, 0, st>>>(src, row_bytes, rows, n, dst);
  OTF_LAUNCH_CHECK("gather_rows_kernel");
  return OTF_OK;
}

int launch_gather_i64(const int64_t* src, const int64_t* rows, int64_t n, int64_t base,
                      int64_t* dst, cudaStream_t st) {
  if (n <= 0) return OTF_OK;
  int64_t grid = (n + 255) / 256;
  if (grid > 4096) grid = 4096;
  gather_i64_kernel<<<(int)grid, 256, 0, st>>>(src, rows, n, base, dst);
  OTF_LAUNCH_CHECK("gather_i64_kernel");
  return OTF_OK;
}

}  // namespace otf
