// otf_kmeans.cu — Lloyd iterations of PQ codebook learning (learn_pq_codebook, pq.py:116-203),
// the offline step before pq_encode, on the GPU.
//
// One step = _assign (pq.py:100-113) + the plain mean update (pq.py:155-162):
//   sq[i, j] = (|x_i|^2 - 2 x_i.c_j) + |c_j|^2  -> assign[i] = argmin_j (first minimum / first NaN),
//   best[i] = max(sq[i, assign[i]], 0), objective = sum_i best[i],
//   counts[j] = #members, c_j <- mean of its members (clusters with members only).
// Orders follow numpy where they are pinnable: |x|^2 and |c|^2 are np.sum over the contiguous
// axis (pairwise order), the objective is np.sum of a 1-D array (pairwise order), a mean is the
// sequential sum of the members in row order (np.mean over axis 0 reduces the outer axis
// row by row) divided by the count. Only the Q-term dot (BLAS dgemm in the reference) rounds
// differently, so assignments agree except at rounding-level near-ties and the objective agrees
// to ~1e-15 relative. The empty-cluster re-seeding (pq.py:163-171) is sequential and rare; the
// Python driver runs it with numpy on the host copy of (assign, counts, centroids).
#include "otf_common.cuh"
#include "otf_internal.h"

namespace otf {

template <typename Get>
__device__ double km_pairwise(const Get& a, int64_t s, int64_t n);

// numpy pairwise_sum over a contiguous run (8 accumulators up to 128, split otherwise)
template <typename Get>
__device__ double km_block(const Get& a, int64_t s, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a(s + i));
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a(s + j);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a(s + i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a(s + i));
  return res;
}
template <typename Get>
__device__ double km_pairwise(const Get& a, int64_t s, int64_t n) {
  if (n <= 128) return km_block(a, s, n);
  struct Frame { int64_t s, n; int stage; double left; };
  Frame st[48];
  int top = 0;
  st[0] = {s, n, 0, 0.0};
  double ret = 0.0;
  while (top >= 0) {
    Frame& f = st[top];
    if (f.n <= 128) { ret = km_block(a, f.s, f.n); --top; continue; }
    int64_t n2 = f.n / 2; n2 -= n2 % 8;
    if (f.stage == 0) { f.stage = 1; st[top + 1] = {f.s, n2, 0, 0.0}; ++top; continue; }
    if (f.stage == 1) { f.left = ret; f.stage = 2; st[top + 1] = {f.s + n2, f.n - n2, 0, 0.0}; ++top; continue; }
    ret = __dadd_rn(f.left, ret);
    --top;
  }
  return ret;
}

// |row|^2 of every row (n rows of Q doubles), numpy pairwise order
__global__ void km_sqnorms(const double* __restrict__ a, int64_t n, int Q, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double* r = a + i * Q;
    auto sq = [r](int64_t q) { return __dmul_rn(r[q], r[q]); };
    out[i] = km_pairwise(sq, 0, Q);
  }
}

// assignment: one thread per row, centroids + their norms in shared memory (broadcast reads)
__global__ void km_assign(const double* __restrict__ X, const double* __restrict__ xx, int64_t n, int Q,
                          const double* __restrict__ C, const double* __restrict__ cc, int K,
                          int32_t* __restrict__ assign, double* __restrict__ best, unsigned long long* __restrict__ counts) {
  extern __shared__ double km_smem[];
  double* sC = km_smem;               // K*Q
  double* scc = km_smem + (size_t)K * Q;  // K
  for (int t = threadIdx.x; t < K * Q; t += blockDim.x) sC[t] = C[t];
  for (int t = threadIdx.x; t < K; t += blockDim.x) scc[t] = cc[t];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double* x = X + i * Q;
    const double xi = xx[i];
    double bv = 0.0;
    int arg = 0;
    bool nan_seen = false;
    for (int j = 0; j < K; ++j) {
      const double* c = sC + (size_t)j * Q;
      double dot = 0.0;
      for (int q = 0; q < Q; ++q) dot = __fma_rn(x[q], c[q], dot);
      const double sq = __dadd_rn(__dsub_rn(xi, 2.0 * dot), scc[j]);
      if (j == 0) { bv = sq; nan_seen = isnan(sq); }
      else if (!nan_seen) {
        if (isnan(sq)) { arg = j; bv = sq; nan_seen = true; }
        else if (sq < bv) { bv = sq; arg = j; }
      }
    }
    assign[i] = arg;
    best[i] = (isnan(bv) || bv >= 0.0) ? bv : 0.0;  // np.maximum(sq, 0.0): NaN and -0.0 kept
    atomicAdd(&counts[arg], 1ull);
  }
}

// objective = numpy pairwise sum of best[0..n), one CTA: thread 0 enumerates numpy's leaves
// (blocks of <= 128 after the recursive splits at n2 = n/2 rounded down to a multiple of 8),
// the CTA sums the leaves in parallel (8 accumulators each, independent loads), and thread 0
// combines them along the same recursion tree. Bit-identical to a single-thread pairwise sum.
constexpr int kObjMaxLeaves = 1536;
__global__ void km_objective(const double* __restrict__ best, int64_t n, double* __restrict__ out) {
  __shared__ int64_t ls[kObjMaxLeaves];
  __shared__ int32_t ln[kObjMaxLeaves];
  __shared__ double lv[kObjMaxLeaves];
  __shared__ int n_leaves;
  auto get = [best](int64_t i) { return best[i]; };
  // leaves: nodes of <= leaf_max elements (128 = numpy's block; larger leaves for very long
  // arrays are summed by km_pairwise, which continues the same recursion inside the leaf)
  int64_t leaf_max = 128;
  while (2 * n / leaf_max + 2 > kObjMaxLeaves) leaf_max *= 2;
  if (threadIdx.x == 0) {
    struct F { int64_t s, n; };
    F st[64];
    int top = 0, c = 0;
    st[0] = {0, n};
    while (top >= 0) {  // in-order enumeration of the recursion's leaves
      const F f = st[top--];
      if (f.n <= leaf_max) { ls[c] = f.s; ln[c] = (int32_t)f.n; ++c; continue; }
      int64_t n2 = f.n / 2; n2 -= n2 % 8;
      st[++top] = {f.s + n2, f.n - n2};  // popped after the left half
      st[++top] = {f.s, n2};
    }
    n_leaves = c;
  }
  __syncthreads();
  const int L = n_leaves;
  for (int t = threadIdx.x; t < L; t += blockDim.x) lv[t] = km_pairwise(get, ls[t], ln[t]);
  __syncthreads();
  if (threadIdx.x == 0) {  // replay the recursion over the leaf values, same tree
    struct G { int64_t n; int stage; double left; };
    G st[64];
    int top = 0, next = 0;
    st[0] = {n, 0, 0.0};
    double ret = 0.0;
    while (top >= 0) {
      G& f = st[top];
      if (f.n <= leaf_max) { ret = lv[next++]; --top; continue; }
      int64_t n2 = f.n / 2; n2 -= n2 % 8;
      if (f.stage == 0) { f.stage = 1; st[top + 1] = {n2, 0, 0.0}; ++top; continue; }
      if (f.stage == 1) { f.left = ret; f.stage = 2; st[top + 1] = {f.n - n2, 0, 0.0}; ++top; continue; }
      ret = __dadd_rn(f.left, ret);
      --top;
    }
    *out = ret;
  }
}

// plain mean update: one warp per cluster j scans the assignment in row order (ballot per 32
// rows); lane q < Q accumulates coordinate q over the members in that order (sequential sum,
// first member as the initial value), then divides by the count.
__global__ void km_means(const double* __restrict__ X, int64_t n, int Q, const int32_t* __restrict__ assign,
                         const unsigned long long* __restrict__ counts, int K, double* __restrict__ C) {
  const int lane = threadIdx.x & 31;
  const int j = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (j >= K) return;
  const unsigned long long cnt = counts[j];
  if (cnt == 0) return;
  for (int q0 = 0; q0 < Q; q0 += 32) {
    const int q = q0 + lane;
    double s = 0.0;
    bool first = true;
    for (int64_t i0 = 0; i0 < n; i0 += 32) {
      const int64_t i = i0 + lane;
      unsigned m = __ballot_sync(0xffffffffu, i < n && __ldg(assign + i) == j);
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        if (q < Q) {
          const double v = __ldg(X + (i0 + b) * Q + q);
          s = first ? v : __dadd_rn(s, v);
          first = false;
        }
      }
    }
    if (q < Q) C[(int64_t)j * Q + q] = __ddiv_rn(s, (double)cnt);
  }
}

int kmeans_step(const double* X, const double* xx, int64_t n, int Q, int K, double* C, double* cc, int32_t* assign,
                double* best, unsigned long long* counts, double* objective, int device, cudaStream_t st) {
  km_sqnorms<<<(K + 127) / 128, 128, 0, st>>>(C, K, Q, cc);
  OTF_LAUNCH_CHECK("km_sqnorms");
  OTF_CUDA(cudaMemsetAsync(counts, 0, (size_t)K * sizeof(unsigned long long), st));
  const size_t smem = ((size_t)K * Q + K) * sizeof(double);
  if (smem > 200 * 1024) return fail(OTF_ERR_CONFIG, "num_centroids * subdim too large for the assignment kernel");
  static bool configured[64] = {false};
  if (!configured[device & 63]) {
    OTF_CUDA(cudaFuncSetAttribute((const void*)km_assign, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    configured[device & 63] = true;
  }
  int64_t grid = (n + 255) / 256;
  const int64_t cap = 2LL * sm_count(device);
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  km_assign<<<(int)grid, 256, smem, st>>>(X, xx, n, Q, C, cc, K, assign, best, counts);
  OTF_LAUNCH_CHECK("km_assign");
  km_objective<<<1, 256, 0, st>>>(best, n, objective);
  OTF_LAUNCH_CHECK("km_objective");
  km_means<<<(K * 32 + 127) / 128, 128, 0, st>>>(X, n, Q, assign, counts, K, C);
  OTF_LAUNCH_CHECK("km_means");
  return OTF_OK;
}

int kmeans_row_norms(const double* X, int64_t n, int Q, double* xx, cudaStream_t st) {
  int64_t grid = (n + 255) / 256;
  if (grid > 4096) grid = 4096;
  if (grid < 1) grid = 1;
  km_sqnorms<<<(int)grid, 256, 0, st>>>(X, n, Q, xx);
  OTF_LAUNCH_CHECK("km_sqnorms");
  return OTF_OK;
}

}  // namespace otf
