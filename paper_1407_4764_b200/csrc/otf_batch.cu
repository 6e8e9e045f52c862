// otf_batch.cu — T5: fixed-set SVM training (train_batch, trainer.py:204-257) and the hinge
// objective (hinge_objective, trainer.py:197-201) on the GPU.
//
// The reference runs epochs * ceil(n / B) sequential Pegasos steps over the pooled labeled set
// (lam = 1 / (c n)), keeps the tail average of the last quarter of iterates and the best iterate
// seen at epoch boundaries (objective evaluated over all n rows), and returns whichever scores
// the lower objective. Every step depends on the previous w, so the whole run is ONE persistent
// CTA: the feature matrix stays in HBM/L2, w, the tail sum and the best iterate live in shared
// memory, and the B sampled indices per step come from the host (numpy PCG64, drawn exactly as
// the reference draws them). Per step: margins (one warp per sampled row, float64), violators,
// the sequential violator gradient, the elementwise update with __dmul_rn/__dadd_rn (numpy
// order), the projection; per epoch: the objective (one warp per row, fixed-order sums).
// Float64 dot orders differ from BLAS, so parity is a tolerance.
#include "otf_common.cuh"
#include "otf_internal.h"

namespace otf {

constexpr int kBatchThreads = 1024;

__device__ __forceinline__ double feat(const void* X, int dt, int64_t idx) {
  return dt == OTF_F32 ? (double)static_cast<const float*>(X)[idx] : static_cast<const double*>(X)[idx];
}

// Block-wide float64 sum with a fixed order (warp xor tree, then warp 0 over warp partials).
__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int o = 16; o >= 1; o >>= 1) v = __dadd_rn(v, shfl_xor_d(v, o));
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double s = lane < nw ? red[lane] : 0.0;
    for (int o = 16; o >= 1; o >>= 1) s = __dadd_rn(s, shfl_xor_d(s, o));
    if (lane == 0) red[32] = s;
  }
  __syncthreads();
  return red[32];
}

// lam/2 |w|^2 + mean(max(0, 1 - y <w, x>)) over all n rows (rows < n_pos have y = +1).
__device__ double objective(const void* X, int dt, int64_t n_pos, int64_t n, int d, const double* w,
                            double lam, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double loss = 0.0;  // per-warp running sum over its rows (row order fixed per warp)
  for (int64_t r = wid; r < n; r += nw) {
    double acc = 0.0;
    for (int j = lane; j < d; j += 32) acc = __fma_rn(feat(X, dt, r * d + j), w[j], acc);
    for (int o = 16; o >= 1; o >>= 1) acc = __dadd_rn(acc, shfl_xor_d(acc, o));
    const double margin = r < n_pos ? acc : -acc;
    const double h = 1.0 - margin;
    loss = __dadd_rn(loss, h > 0.0 ? h : 0.0);
  }
  double sq = 0.0;
  for (int j = threadIdx.x; j < d; j += blockDim.x) sq = __fma_rn(w[j], w[j], sq);
  sq = block_sum(sq, red);
  // lane 0 of each warp holds its loss; sum warps in order
  const double tot = block_sum(lane == 0 ? loss : 0.0, red);
  return __dadd_rn(__dmul_rn(__dmul_rn(0.5, lam), sq), __ddiv_rn(tot, (double)n));
}

__global__ void __launch_bounds__(kBatchThreads, 1)
batch_train_kernel(const void* __restrict__ X, int dt, int64_t n_pos, int64_t n, int d,
                   const int64_t* __restrict__ idx, int64_t total, int bs, int64_t spe,
                   int64_t tail_start, int64_t tail_len, double lam, int project,
                   double* __restrict__ w_out, double* __restrict__ obj_hist) {
  extern __shared__ double sm[];
  double* w = sm;             // d
  double* tail = w + d;       // d
  double* best = tail + d;    // d
  double* red = best + d;     // 33
  int* viol = reinterpret_cast<int*>(red + 40);  // bs
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = threadIdx.x; j < d; j += blockDim.x) { w[j] = 0.0; tail[j] = 0.0; best[j] = 0.0; }
  __syncthreads();
  double best_obj = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  const double radius = project ? 1.0 / sqrt(lam) : 0.0;
  int64_t epoch = 0;
  for (int64_t t = 1; t <= total; ++t) {
    const int64_t* bi = idx + (t - 1) * bs;
    const double eta = 1.0 / (lam * (double)t);
    const double shrink = 1.0 - eta * lam;
    const double eob = eta / (double)bs;
    // margins
    for (int b = wid; b < bs; b += nw) {
      const int64_t r = bi[b];
      double acc = 0.0;
      for (int j = lane; j < d; j += 32) acc = __fma_rn(feat(X, dt, r * d + j), w[j], acc);
      for (int o = 16; o >= 1; o >>= 1) acc = __dadd_rn(acc, shfl_xor_d(acc, o));
      if (lane == 0) viol[b] = (r < n_pos ? acc : -acc) < 1.0;
    }
    __syncthreads();
    // gradient + update (thread per column; sequential over violators, numpy axis-0 order)
    double sq = 0.0;
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      double g = 0.0;
      for (int b = 0; b < bs; ++b) {
        if (!viol[b]) continue;
        const int64_t r = bi[b];
        const double x = feat(X, dt, r * d + j);
        g = __dadd_rn(g, r < n_pos ? x : -x);
      }
      const double nwj = __dadd_rn(__dmul_rn(shrink, w[j]), __dmul_rn(eob, g));
      w[j] = nwj;
      sq = __fma_rn(nwj, nwj, sq);
    }
    if (project) {
      sq = block_sum(sq, red);  // includes __syncthreads
      const double norm = sqrt(sq);
      if (norm > radius) {
        const double scale = __ddiv_rn(radius, norm);
        for (int j = threadIdx.x; j < d; j += blockDim.x) w[j] = __dmul_rn(w[j], scale);
      }
    }
    if (t > tail_start)
      for (int j = threadIdx.x; j < d; j += blockDim.x) tail[j] = __dadd_rn(tail[j], w[j]);
    __syncthreads();
    if (t % spe == 0) {
      const double obj = objective(X, dt, n_pos, n, d, w, lam, red);
      if (threadIdx.x == 0 && obj_hist) obj_hist[epoch] = obj;
      ++epoch;
      if (obj < best_obj) {
        best_obj = obj;
        for (int j = threadIdx.x; j < d; j += blockDim.x) best[j] = w[j];
      }
      __syncthreads();
    }
  }
  // tail average vs best epoch iterate (trainer.py:253-256)
  for (int j = threadIdx.x; j < d; j += blockDim.x) tail[j] = __ddiv_rn(tail[j], (double)tail_len);
  __syncthreads();
  const double avg_obj = objective(X, dt, n_pos, n, d, tail, lam, red);
  const bool use_avg = avg_obj <= best_obj;
  for (int j = threadIdx.x; j < d; j += blockDim.x) w_out[j] = use_avg ? tail[j] : best[j];
  if (threadIdx.x == 0 && obj_hist) obj_hist[epoch] = avg_obj;  // slot after the epochs
}

size_t batch_smem_bytes(int d, int bs) {
  return (size_t)3 * d * sizeof(double) + 40 * sizeof(double) + (size_t)bs * sizeof(int);
}

int launch_batch_train(const void* X, int dt, int64_t n_pos, int64_t n, int d, const int64_t* idx,
                       int64_t total, int bs, int64_t spe, int64_t tail_start, int64_t tail_len,
                       double lam, int project, double* w_out, double* obj_hist, cudaStream_t st) {
  const size_t smem = batch_smem_bytes(d, bs);
  if (smem > 220 * 1024) return fail(OTF_ERR_CONFIG, "train_batch: dim too large for the on-chip iterate");
  OTF_CUDA(cudaFuncSetAttribute((const void*)batch_train_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  batch_train_kernel<<<1, kBatchThreads, smem, st>>>(X, dt, n_pos, n, d, idx, total, bs, spe, tail_start,
                                                      tail_len, lam, project, w_out, obj_hist);
  OTF_LAUNCH_CHECK("batch_train_kernel");
  return OTF_OK;
}

__global__ void __launch_bounds__(kBatchThreads, 1)
hinge_objective_kernel(const void* __restrict__ X, int dt, int64_t n_pos, int64_t n, int d,
                       const double* __restrict__ w_g, double lam, double* __restrict__ out) {
  extern __shared__ double sm[];
  double* w = sm;
  double* red = w + d;
  for (int j = threadIdx.x; j < d; j += blockDim.x) w[j] = w_g[j];
  __syncthreads();
  const double obj = objective(X, dt, n_pos, n, d, w, lam, red);
  if (threadIdx.x == 0) *out = obj;
}

int launch_hinge_objective(const void* X, int dt, int64_t n_pos, int64_t n, int d, const double* w,
                           double lam, double* out, cudaStream_t st) {
  const size_t smem = (size_t)d * sizeof(double) + 40 * sizeof(double);
  if (smem > 220 * 1024) return fail(OTF_ERR_CONFIG, "hinge_objective: dim too large");
  OTF_CUDA(cudaFuncSetAttribute((const void*)hinge_objective_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  hinge_objective_kernel<<<1, kBatchThreads, smem, st>>>(X, dt, n_pos, n, d, w, lam, out);
  OTF_LAUNCH_CHECK("hinge_objective_kernel");
  return OTF_OK;
}

}  // namespace otf
