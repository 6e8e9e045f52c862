// otf_topk.cu — K5: exact top-k selection (top_k, ranker.py:97-143).
//
// Semantics: the first k entries of a full sort by (-score, id) — descending score, ties
// toward the smallest id, -0.0 tied with +0.0, k_eff = min(max(k, 0), n), k_eff == n is a
// full sort. Output scores are float64 (ranker.py:141), ids int64.
//
// One cooperative launch (persistent grid, one 1024-thread CTA per SM):
//   A. coarse 4096-bin histogram of the scores (top 12 bits of the float32 order key) — this
//      phase is skipped when the scoring kernel already produced it (the fused path);
//   B. every CTA scans the histogram from the top and finds the bin b0 holding the k-th
//      entry, the count above it and its size: C = above + |b0| candidates;
//   C. (common case, C <= 8192) one gather pass appends every entry with bin >= b0
//      (warp-aggregated atomics), a grid barrier, and every CTA ranks a slice of the C
//      candidates by counting how many beat each one under (key desc, ~id desc); ranks < k_eff
//      go straight to their output slot (rank_emit);
//   D. (rare: a bin with > 8192 - above entries, e.g. massive ties) an exact MSD radix select
//      on the full order key, 8 bits per pass with a grid barrier each, then on ~id inside a
//      tied key; gather exactly k_eff entries and rank them (or a global bitonic sort when
//      k_eff > 8192).
// Scores are read from L2 (the scoring kernel just wrote them); the common case reads them
// once (phase C) after the fused histogram.
#include "otf_common.cuh"
#include "otf_internal.h"

namespace otf {

static constexpr int kTopkThreads = 1024;
static constexpr int kCandCap = 8192;                       // candidates ranked in smem
static constexpr size_t kTopkSmem = (size_t)kCandCap * 16;  // key + inv per candidate

__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vgen = bar + 1;
    const unsigned int gen = *vgen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ int64_t id_of(const int64_t* ids, int64_t id_base, int64_t row) {
  return ids ? ids[row] : id_base + row;
}

template <typename ST>
__device__ __forceinline__ uint64_t load_key(const ST* s, int64_t i) {
  return score_key(__ldcg(s + i));
}

__device__ __forceinline__ bool cand_greater(uint64_t ka, uint64_t ia, uint64_t kb, uint64_t ib) {
  return ka > kb || (ka == kb && ia > ib);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Appends (key, ~id, row) for every lane with `take`, one atomic per warp.
__device__ __forceinline__ void append_candidate(const TopkWs& ws, bool take, uint64_t key,
                                                 uint64_t inv, int64_t row, int64_t cap) {
  const unsigned m = __ballot_sync(0xffffffffu, take);
  if (m == 0u) return;
  unsigned base = 0;
  if ((threadIdx.x & 31) == 0) base = atomicAdd(ws.count, (unsigned)__popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (take) {
    const int64_t slot = (int64_t)base + __popc(m & lanemask_lt());
    if (slot < cap) {
      ws.key[slot] = key;
      ws.inv[slot] = inv;
      ws.row[slot] = row;
    }
  }
}

// Block-wide: bins scanned from 4095 down; finds the bin where the running count reaches
// `need`. Thread t owns bins 4095-4t .. 4092-4t.
__device__ void find_bin4096(const uint32_t* h, int64_t need, int* out_b, int64_t* out_above,
                             int64_t* out_cnt, int64_t* wsum) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  int64_t local = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) local += h[4095 - 4 * t - q];
  int64_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int64_t v = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
    int64_t s = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += u;
    }
    wsum[lane] = s - v;  // exclusive prefix of warp sums
  }
  __syncthreads();
  incl += wsum[wid];
  const int64_t excl = incl - local;
  if (excl < need && incl >= need) {
    int64_t cum = excl;
    for (int q = 0; q < 4; ++q) {
      const int bin = 4095 - 4 * t - q;
      if (cum + h[bin] >= need) {
        *out_b = bin;
        *out_above = cum;
        *out_cnt = h[bin];
        break;
      }
      cum += h[bin];
    }
  }
}

// Radix-digit picker for phase D (warp 0, 256 bins scanned from the top).
__device__ __forceinline__ void pick_bin256(const uint32_t* h, int64_t need, int* out_b,
                                            int64_t* out_above) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    int64_t local = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) local += h[255 - 8 * lane - q];
    int64_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int64_t excl = incl - local;
    const unsigned hit = __ballot_sync(0xffffffffu, incl >= need);
    const int first = hit ? __ffs(hit) - 1 : 31;
    if (lane == first) {
      int64_t cum = excl;
      int b = 255 - 8 * lane - 7;
      for (int q = 0; q < 8; ++q) {
        const int bin = 255 - 8 * lane - q;
        if (cum + h[bin] >= need) { b = bin; break; }
        cum += h[bin];
      }
      *out_b = b;
      *out_above = cum;
    }
  }
}

// Orders ws candidates [0, m) by counting: the rank of candidate i is the number of candidates
// j with (key_j, inv_j) > (key_i, inv_i) — a permutation of 0..m-1 because ids are unique.
// Every CTA copies the m (key, inv) pairs into shared memory and ranks the candidates
// i == blockIdx.x (mod gridDim.x), one warp per candidate; candidates with rank < k_eff are
// written straight to their output slot. O(m^2 / #SMs) comparisons, no sorting network, no
// barrier — the whole grid shares the work (m <= kCandCap).
template <typename ST>
__device__ void rank_emit(const ST* scores, const TopkWs& ws, int64_t m, int64_t k_eff,
                          unsigned char* dyn, int64_t* out_ids, double* out_scores,
                          int64_t* out_rows) {
  const int64_t mine = m > blockIdx.x ? (m - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (mine == 0) return;
  uint64_t* sk = reinterpret_cast<uint64_t*>(dyn);
  uint64_t* si = sk + m;
  for (int64_t t = threadIdx.x; t < m; t += blockDim.x) {
    sk[t] = __ldcg(ws.key + t);
    si[t] = __ldcg(ws.inv + t);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t q = wid; q < mine; q += nw) {
    const int64_t i = blockIdx.x + q * gridDim.x;
    const uint64_t ki = sk[i], ii = si[i];
    int64_t cnt = 0;
    for (int64_t j = lane; j < m; j += 32) cnt += cand_greater(sk[j], si[j], ki, ii);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0 && cnt < k_eff) {
      const int64_t r = __ldcg(ws.row + i);
      out_ids[cnt] = (int64_t)~ii;
      out_scores[cnt] = (double)__ldcg(scores + r);
      if (out_rows) out_rows[cnt] = r;
    }
  }
}

template <typename ST>
__global__ void __launch_bounds__(kTopkThreads, 1)
topk_coop_kernel(const ST* __restrict__ scores, int64_t n, const int64_t* __restrict__ ids,
                 int64_t id_base, int64_t k_eff, TopkWs ws, int hist_ready,
                 int64_t* __restrict__ out_ids, double* __restrict__ out_scores,
                 int64_t* __restrict__ out_rows) {
  constexpr int KB = KeyBits<ST>::value;
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ uint32_t h[256];
  __shared__ int s_b;
  __shared__ int64_t s_above, s_cnt;
  __shared__ int64_t wsum[32];
  const unsigned int nb = gridDim.x;
  const int lane = threadIdx.x & 31;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t wbase0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
  const bool all = k_eff >= n;

  // ---- A: coarse histogram (skipped when fused into the scoring kernel) --------------------
  if (!all && !hist_ready) {
    uint32_t* sh = reinterpret_cast<uint32_t*>(dyn);
    hist_zero(sh);
    __syncthreads();
    for (int64_t base = wbase0; base < n; base += nthreads) {
      const int64_t i = base + lane;
      const bool active = i < n;
      hist_add(sh, active, active ? hist_bin(__ldcg(scores + i)) : 0u);
    }
    __syncthreads();
    hist_flush(sh, ws.hist);
    grid_barrier(ws.bar, nb);
  }

  // ---- B: the bin holding the k-th entry ------------------------------------------------------
  int64_t C = n;
  uint32_t b0 = 0;
  if (!all) {
    uint32_t* sh = reinterpret_cast<uint32_t*>(dyn);
    for (int b = threadIdx.x; b < kHistBins; b += blockDim.x) sh[b] = __ldcg(ws.hist + b);
    __syncthreads();
    find_bin4096(sh, k_eff, &s_b, &s_above, &s_cnt, wsum);
    __syncthreads();
    b0 = (uint32_t)s_b;
    C = s_above + s_cnt;
    __syncthreads();
  }

  if (C <= kCandCap) {
    // ---- C: gather the candidates (8 loads in flight per thread), rank them -----------------
    constexpr int U = 8;
    for (int64_t base = wbase0 * U; base < n; base += nthreads * U) {
      ST v[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int64_t i = base + 32 * q + lane;
        v[q] = i < n ? __ldcg(scores + i) : ST(0);
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int64_t i = base + 32 * q + lane;
        const bool take = i < n && (all || hist_bin(v[q]) >= b0);
        uint64_t key = 0, inv = 0;
        if (take) { key = score_key(v[q]); inv = ~(uint64_t)id_of(ids, id_base, i); }
        append_candidate(ws, take, key, inv, i, C);
      }
    }
    grid_barrier(ws.bar, nb);
    if (blockIdx.x == 0) {  // every CTA has read hist and count is no longer needed
      for (int b = threadIdx.x; b < kHistBins; b += blockDim.x) ws.hist[b] = 0u;
      if (threadIdx.x == 0) *ws.count = 0u;
    }
    rank_emit(scores, ws, C, k_eff, dyn, out_ids, out_scores, out_rows);
    return;
  }

  // ---- D: exact MSD radix select on the full key, then on ~id within a tied key ------------
  uint64_t pre = 0, msk = 0, pre2 = 0, msk2 = 0;
  int64_t need = k_eff;
  int phase = all ? 2 : 0;  // k_eff == n: everything is gathered (mask 0)
  bool tie = false;
  int shift = KB - 8;
  int it = 0;
  while (phase < 2) {
    uint32_t* H = ws.rhist + (it % 3) * 256;
    if (blockIdx.x == 0 && threadIdx.x < 256) ws.rhist[((it + 1) % 3) * 256 + threadIdx.x] = 0u;
    if (threadIdx.x < 256) h[threadIdx.x] = 0u;
    __syncthreads();
    if (phase == 0) {
      for (int64_t i = tid; i < n; i += nthreads) {
        const uint64_t key = load_key(scores, i);
        if ((key & msk) == pre) atomicAdd(&h[(key >> shift) & 255u], 1u);
      }
    } else {
      for (int64_t i = tid; i < n; i += nthreads) {
        const uint64_t key = load_key(scores, i);
        if (key == pre) {
          const uint64_t inv = ~(uint64_t)id_of(ids, id_base, i);
          if ((inv & msk2) == pre2) atomicAdd(&h[(inv >> shift) & 255u], 1u);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x < 256 && h[threadIdx.x]) atomicAdd(&H[threadIdx.x], h[threadIdx.x]);
    grid_barrier(ws.bar, nb);
    if (threadIdx.x < 256) h[threadIdx.x] = __ldcg(H + threadIdx.x);
    __syncthreads();
    pick_bin256(h, need, &s_b, &s_above);
    __syncthreads();
    const int b = s_b;
    need -= s_above;
    const uint32_t cnt = h[b];
    if (phase == 0) {
      pre |= (uint64_t)b << shift;
      msk |= (uint64_t)0xff << shift;
    } else {
      pre2 |= (uint64_t)b << shift;
      msk2 |= (uint64_t)0xff << shift;
    }
    if ((int64_t)cnt == need) {
      phase = 2;
    } else if (shift == 0) {
      if (phase == 0) { phase = 1; tie = true; shift = 56; }
      else phase = 2;  // duplicate ids: the gather caps the count
    } else {
      shift -= 8;
    }
    ++it;
    __syncthreads();
  }
  for (int64_t base = wbase0; base < n; base += nthreads) {
    const int64_t i = base + lane;
    bool in = false;
    uint64_t key = 0, inv = 0;
    if (i < n) {
      key = load_key(scores, i);
      const uint64_t mk = key & msk;
      inv = ~(uint64_t)id_of(ids, id_base, i);
      in = mk > pre || (mk == pre && (!tie || (inv & msk2) >= pre2));
    }
    append_candidate(ws, in, key, inv, i, k_eff);
  }
  grid_barrier(ws.bar, nb);
  if (blockIdx.x == 0) {
    for (int t = threadIdx.x; t < 3 * 256; t += blockDim.x) ws.rhist[t] = 0u;
    for (int b = threadIdx.x; b < kHistBins; b += blockDim.x) ws.hist[b] = 0u;
  }
  if (k_eff <= kCandCap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *ws.count = 0u;
    rank_emit(scores, ws, k_eff, k_eff, dyn, out_ids, out_scores, out_rows);
    return;
  }
  // global bitonic sort over ws (capacity P)
  int64_t P = 1;
  while (P < k_eff) P <<= 1;
  for (int64_t t = tid + k_eff; t < P; t += nthreads) { ws.key[t] = 0; ws.inv[t] = 0; ws.row[t] = -1; }
  grid_barrier(ws.bar, nb);
  for (int64_t size = 2; size <= P; size <<= 1) {
    for (int64_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (int64_t t = tid; t < P; t += nthreads) {
        const int64_t j = t ^ stride;
        if (j > t) {
          const uint64_t kt = __ldcg(ws.key + t), kj = __ldcg(ws.key + j);
          const uint64_t it_ = __ldcg(ws.inv + t), ij = __ldcg(ws.inv + j);
          const bool desc = (t & size) == 0;
          const bool swap = desc ? cand_greater(kj, ij, kt, it_) : cand_greater(kt, it_, kj, ij);
          if (swap) {
            const int64_t rt = __ldcg(ws.row + t), rj = __ldcg(ws.row + j);
            ws.key[t] = kj; ws.key[j] = kt;
            ws.inv[t] = ij; ws.inv[j] = it_;
            ws.row[t] = rj; ws.row[j] = rt;
          }
        }
      }
      grid_barrier(ws.bar, nb);
    }
  }
  for (int64_t t = tid; t < k_eff; t += nthreads) {
    const int64_t r = __ldcg(ws.row + t);
    out_ids[t] = (int64_t)~__ldcg(ws.inv + t);
    out_scores[t] = (double)__ldcg(scores + r);
    if (out_rows) out_rows[t] = r;
  }
  if (tid == 0) *ws.count = 0u;
}

int topk_ws_alloc(TopkWs* ws, int64_t k_eff) {
  int64_t P = kCandCap;
  while (P < k_eff) P <<= 1;
  if (ws->hist == nullptr) {
    const size_t bytes = (kHistBins + 3 * 256 + 4) * sizeof(uint32_t);
    OTF_CUDA(cudaMalloc(&ws->hist, bytes));
    OTF_CUDA(cudaMemset(ws->hist, 0, bytes));
    ws->rhist = ws->hist + kHistBins;
    ws->bar = reinterpret_cast<unsigned int*>(ws->rhist + 3 * 256);
    ws->count = ws->bar + 2;
  }
  if (P > ws->cap) {
    cudaFree(ws->key); cudaFree(ws->inv); cudaFree(ws->row);
    ws->key = nullptr; ws->inv = nullptr; ws->row = nullptr; ws->cap = 0;
    OTF_CUDA(cudaMalloc(&ws->key, P * sizeof(uint64_t)));
    OTF_CUDA(cudaMalloc(&ws->inv, P * sizeof(uint64_t)));
    OTF_CUDA(cudaMalloc(&ws->row, P * sizeof(int64_t)));
    ws->cap = P;
  }
  return OTF_OK;
}

void topk_ws_free(TopkWs* ws) {
  cudaFree(ws->hist); cudaFree(ws->key); cudaFree(ws->inv); cudaFree(ws->row);
  *ws = TopkWs{};
}

template <typename ST>
static int launch_typed(const ST* scores, int64_t n, const int64_t* ids, int64_t id_base,
                        int64_t k_eff, TopkWs* ws, bool hist_ready, int64_t* out_ids,
                        double* out_scores, int64_t* out_rows, int device, cudaStream_t st) {
  auto fn = topk_coop_kernel<ST>;
  static bool configured[64] = {false};
  if (!configured[device & 63]) {
    OTF_CUDA(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kTopkSmem));
    configured[device & 63] = true;
  }
  int grid = sm_count(device);
  const int64_t useful = (n + kTopkThreads - 1) / kTopkThreads;
  if (useful < grid) grid = (int)(useful > 0 ? useful : 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTopkThreads);
  cfg.dynamicSmemBytes = kTopkSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OTF_CUDA(cudaLaunchKernelEx(&cfg, fn, scores, n, ids, id_base, k_eff, *ws, (int)hist_ready,
                              out_ids, out_scores, out_rows));
  count_launch();
  return OTF_OK;
}

int launch_topk(const void* scores, int dtype, int64_t n, const int64_t* ids, int64_t id_base,
                int64_t k_eff, TopkWs* ws, bool hist_ready, int64_t* out_ids, double* out_scores,
                int64_t* out_rows, int device, cudaStream_t st) {
  if (k_eff <= 0 || n <= 0) return OTF_OK;
  int rc = topk_ws_alloc(ws, k_eff);
  if (rc) return rc;
  if (dtype == OTF_F32)
    return launch_typed(static_cast<const float*>(scores), n, ids, id_base, k_eff, ws, hist_ready,
                        out_ids, out_scores, out_rows, device, st);
  return launch_typed(static_cast<const double*>(scores), n, ids, id_base, k_eff, ws, hist_ready,
                      out_ids, out_scores, out_rows, device, st);
}

}  // namespace otf
