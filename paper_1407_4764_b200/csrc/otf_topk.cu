// otf_topk.cu — K5: exact top-k selection (top_k, ranker.py:97-143).
//
// Semantics: the first k entries of a full sort by (-score, id) — descending score, ties
// toward the smallest id, -0.0 tied with +0.0, k_eff = min(max(k, 0), n), k_eff == n is a
// full sort. Output scores are float64 (ranker.py:141), ids int64.
//
// Design (one cooperative launch, persistent grid = one 1024-thread CTA per SM):
//   1. MSD radix select on the order-preserving score key, 8 bits per pass. Each pass
//      histograms the next digit of the keys that still match the resolved prefix (CTA
//      shared-memory histogram, then one global atomic per non-empty bin), a software grid
//      barrier, and every CTA redundantly scans the 256 bins to pick the digit holding the
//      k-th entry (so no second barrier is needed to broadcast the decision). A pass stops
//      the select as soon as the chosen bin holds exactly the entries still needed.
//   2. If every key bit is resolved and the boundary key still has more entries than needed
//      (a tie group), the same passes run on ~id restricted to that key: the smallest ids win.
//   3. Gather: every entry above the resolved threshold (exactly k_eff of them) is appended
//      to a candidate buffer; then CTA 0 bitonic-sorts them in shared memory by
//      (key desc, ~id desc) — or all CTAs run a global bitonic sort when k_eff > 4096.
// Scores are read from L2 (they were just written by the scoring kernel); the passes cost
// ~N*4 (float32) or N*8 (float64) bytes each.
#include <cooperative_groups.h>

#include "otf_common.cuh"
#include "otf_internal.h"

namespace otf {

static constexpr int kTopkThreads = 1024;
static constexpr int kSmemSortCap = 4096;

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

// Warp 0 finds, scanning bins from 255 down, the bin b where the running count reaches
// need; returns b and the count strictly above it (through shared memory).
__device__ __forceinline__ void pick_bin(const uint32_t* h, int64_t need, int* out_b,
                                         int64_t* out_above) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    // lane l covers bins 255-8l .. 248-8l (descending)
    int64_t local = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) local += h[255 - 8 * lane - q];
    int64_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
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

template <typename ST>
__global__ void __launch_bounds__(kTopkThreads, 1)
topk_coop_kernel(const ST* __restrict__ scores, int64_t n, const int64_t* __restrict__ ids,
                 int64_t id_base, int64_t k_eff, TopkWs ws, int64_t* __restrict__ out_ids,
                 double* __restrict__ out_scores, int64_t* __restrict__ out_rows) {
  constexpr int KB = KeyBits<ST>::value;
  __shared__ uint32_t h[256];
  __shared__ int s_b;
  __shared__ int64_t s_above;
  extern __shared__ unsigned char dyn[];
  const unsigned int nb = gridDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;

  uint64_t pre = 0, msk = 0, pre2 = 0, msk2 = 0;
  int64_t need = k_eff;
  int phase = (k_eff >= n) ? 2 : 0;
  bool tie = false;
  int shift = KB - 8;
  int it = 0;
  while (phase < 2) {
    uint32_t* H = ws.hist + (it % 3) * 256;
    if (blockIdx.x == 0 && threadIdx.x < 256) ws.hist[((it + 1) % 3) * 256 + threadIdx.x] = 0u;
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
    pick_bin(h, need, &s_b, &s_above);
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
      else phase = 2;  // duplicate ids: gather caps the count
    } else {
      shift -= 8;
    }
    ++it;
    __syncthreads();
  }

  // ---- gather exactly k_eff candidates ---------------------------------------------------
  for (int64_t i = tid; i < n; i += nthreads) {
    const uint64_t key = load_key(scores, i);
    const uint64_t mk = key & msk;
    bool in = mk > pre;
    uint64_t inv = 0;
    if (!in && mk == pre) {
      inv = ~(uint64_t)id_of(ids, id_base, i);
      in = !tie || ((inv & msk2) >= pre2);
    }
    if (in) {
      if (inv == 0) inv = ~(uint64_t)id_of(ids, id_base, i);
      const unsigned int slot = atomicAdd(ws.count, 1u);
      if ((int64_t)slot < k_eff) {
        ws.key[slot] = key;
        ws.inv[slot] = inv;
        ws.row[slot] = i;
      }
    }
  }
  grid_barrier(ws.bar, nb);
  if (blockIdx.x == 0) {
    for (int t = threadIdx.x; t < 3 * 256; t += blockDim.x) ws.hist[t] = 0u;
  }

  // ---- order the k_eff candidates --------------------------------------------------------
  int64_t P = 1;
  while (P < k_eff) P <<= 1;
  if (P <= kSmemSortCap) {
    if (blockIdx.x != 0) return;
    uint64_t* sk = reinterpret_cast<uint64_t*>(dyn);
    uint64_t* si = sk + P;
    int64_t* sr = reinterpret_cast<int64_t*>(si + P);
    for (int64_t t = threadIdx.x; t < P; t += blockDim.x) {
      if (t < k_eff) { sk[t] = __ldcg(ws.key + t); si[t] = __ldcg(ws.inv + t); sr[t] = __ldcg(ws.row + t); }
      else { sk[t] = 0; si[t] = 0; sr[t] = -1; }
    }
    __syncthreads();
    for (int64_t size = 2; size <= P; size <<= 1) {
      for (int64_t stride = size >> 1; stride > 0; stride >>= 1) {
        for (int64_t t = threadIdx.x; t < P; t += blockDim.x) {
          const int64_t j = t ^ stride;
          if (j > t) {
            const bool desc = (t & size) == 0;
            const bool gt = cand_greater(sk[j], si[j], sk[t], si[t]);
            if (desc ? gt : cand_greater(sk[t], si[t], sk[j], si[j])) {
              uint64_t a = sk[t]; sk[t] = sk[j]; sk[j] = a;
              a = si[t]; si[t] = si[j]; si[j] = a;
              int64_t r = sr[t]; sr[t] = sr[j]; sr[j] = r;
            }
          }
        }
        __syncthreads();
      }
    }
    for (int64_t t = threadIdx.x; t < k_eff; t += blockDim.x) {
      const int64_t r = sr[t];
      out_ids[t] = (int64_t)~si[t];
      out_scores[t] = (double)__ldcg(scores + r);
      if (out_rows) out_rows[t] = r;
    }
    if (threadIdx.x == 0) *ws.count = 0u;
    return;
  }
  // global bitonic sort over ws (capacity P)
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
  int64_t P = 1;
  while (P < k_eff) P <<= 1;
  if (ws->hist == nullptr) {
    OTF_CUDA(cudaMalloc(&ws->hist, 3 * 256 * sizeof(uint32_t) + 4 * sizeof(unsigned int)));
    OTF_CUDA(cudaMemset(ws->hist, 0, 3 * 256 * sizeof(uint32_t) + 4 * sizeof(unsigned int)));
    ws->bar = reinterpret_cast<unsigned int*>(ws->hist + 3 * 256);
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
                        int64_t k_eff, TopkWs* ws, int64_t* out_ids, double* out_scores,
                        int64_t* out_rows, int device, cudaStream_t st) {
  int64_t P = 1;
  while (P < k_eff) P <<= 1;
  const size_t smem = P <= kSmemSortCap ? (size_t)P * 24 : 0;
  auto fn = topk_coop_kernel<ST>;
  static bool configured[64] = {false};
  if (!configured[device & 63]) {
    OTF_CUDA(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemSortCap * 24));
    configured[device & 63] = true;
  }
  int grid = sm_count(device);
  const int64_t useful = (n + kTopkThreads - 1) / kTopkThreads;
  if (useful < grid) grid = (int)(useful > 0 ? useful : 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTopkThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OTF_CUDA(cudaLaunchKernelEx(&cfg, fn, scores, n, ids, id_base, k_eff, *ws, out_ids, out_scores,
                              out_rows));
  count_launch();
  return OTF_OK;
}

int launch_topk(const void* scores, int dtype, int64_t n, const int64_t* ids, int64_t id_base,
                int64_t k_eff, TopkWs* ws, int64_t* out_ids, double* out_scores,
                int64_t* out_rows, int device, cudaStream_t st) {
  if (k_eff <= 0 || n <= 0) return OTF_OK;
  int rc = topk_ws_alloc(ws, k_eff);
  if (rc) return rc;
  if (dtype == OTF_F32)
    return launch_typed(static_cast<const float*>(scores), n, ids, id_base, k_eff, ws, out_ids,
                        out_scores, out_rows, device, st);
  return launch_typed(static_cast<const double*>(scores), n, ids, id_base, k_eff, ws, out_ids,
                      out_scores, out_rows, device, st);
}

}  // namespace otf
