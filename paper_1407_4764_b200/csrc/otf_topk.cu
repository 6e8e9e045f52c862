// otf_topk.cu — K5: exact top-k selection (top_k, ranker.py:97-143).
//
// Semantics: the first k entries of a full sort by (-score, id) — descending score, ties
// toward the smallest id, -0.0 tied with +0.0, k_eff = min(max(k, 0), n), k_eff == n is a
// full sort. Output scores are float64 (ranker.py:141), ids int64.
//
// One cooperative launch (persistent grid, one 1024-thread CTA per SM):
//   A. coarse 4096-bin histogram of the scores (top 12 bits of the float32 order key; PQ bins:
//      8192 / 13 bits, written by the scan) — this
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
//
// Score sources: DirectSrc reads a score array the scoring kernel wrote (dense / binary float32,
// generic float64). PqBinSrc is the PQ fast path: the scan kernel writes only a 16-bit bin per
// row (2 B instead of 8 B) plus the histogram, and the exact float64 score of a candidate is
// recomputed here from its codes and the LUT (numpy order, bit-identical to the scan) — so the
// gather reads 2 B/row. Phase D first materialises all exact scores for such a source.
#include "otf_common.cuh"
#include "otf_internal.h"
#include "otf_topk_dev.cuh"

#include <algorithm>
#include <cstdlib>

namespace otf {

#ifdef OTF_TOPK_TRACE  // diagnostic build (tools/): per-phase globaltimer stamps of CTAs 0 and last
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TOPK_STAMP(i) \
  if (threadIdx.x == 0) tstamp[i] = gtimer()
#define TOPK_REPORT()                                                                                  \
  if (threadIdx.x == 0)                                                                                \
  printf("topk cta %d C=%lld: start %llu gend %llu hits %u maxwarp %u B %.2f gather %.2f barrier %.2f rank %.2f us\n", \
         (int)blockIdx.x, (long long)C, (unsigned long long)(tstamp[0] % 1000000000ull),                      \
         (unsigned long long)(tstamp[2] % 1000000000ull), s_trace[0], s_trace[1], (tstamp[1] - tstamp[0]) * 1e-3, \
         (tstamp[2] - tstamp[1]) * 1e-3, (tstamp[3] - tstamp[2]) * 1e-3, (tstamp[4] - tstamp[3]) * 1e-3)
#else
#define TOPK_STAMP(i)
#define TOPK_REPORT()
#endif

template <typename Src>
__global__ void __launch_bounds__(kTopkThreads, kTopkCtasPerSm)
topk_coop_kernel(Src src, int64_t n, const int64_t* __restrict__ ids, int64_t id_base,
                 int64_t k_eff, TopkWs ws, int hist_ready, typename Src::T* scratch,
                 int64_t* __restrict__ out_ids, double* __restrict__ out_scores,
                 int64_t* __restrict__ out_rows, int n_seg) {
  using ST = typename Src::T;
  // Segments (n_seg > 1, DirectSrc only): n_seg independent selections of k_eff out of n over
  // consecutive score arrays (the multi-classifier path), each on its own gridDim.x / n_seg CTAs
  // with its own workspace; vb / vnb are the CTA's index and count inside its segment.
  const unsigned per = gridDim.x / (unsigned)n_seg;
  const unsigned seg = blockIdx.x / per, vb = blockIdx.x % per, vnb = per;
  if (n_seg > 1) {
    src.shift((int64_t)seg * n);
    scratch += (int64_t)seg * n;
    out_ids += (int64_t)seg * k_eff;
    out_scores += (int64_t)seg * k_eff;
    ws = seg_ws(ws, seg);
  }
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ uint32_t h[256];
  __shared__ int s_b;
  __shared__ int64_t s_above, s_cnt;
  __shared__ int64_t wsum[32];
  const unsigned int nb = vnb;
  const int lane = threadIdx.x & 31;
  // launched programmatically after the scoring kernel (hist_ready): the CTAs come up while its
  // last CTAs drain, and wait here for its scores / histogram / chunk maxima (a no-op otherwise)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t nthreads = (int64_t)vnb * blockDim.x;
  const int64_t wbase0 = (int64_t)vb * blockDim.x + (threadIdx.x & ~31);
  const bool all = k_eff >= n;

  // ---- A: coarse histogram (skipped when fused into the scoring kernel) --------------------
  if (!all && !hist_ready) {
    uint32_t* sh = reinterpret_cast<uint32_t*>(dyn);
    hist_zero(sh);
    __syncthreads();
    // each lane reads 2 x 8 consecutive entries per pass (vector loads; 16 in flight)
    constexpr int UA = 8, RA = 2;
    using VA = decltype(src.load(0));
    for (int64_t wb = wbase0 * UA * RA; wb < n; wb += nthreads * UA * RA) {  // warp-uniform loop
      VA v[RA][UA];
#pragma unroll
      for (int g = 0; g < RA; ++g) {
        const int64_t base = wb + (int64_t)(g * 32 + lane) * UA;
        if (base + UA <= n) {
          src.load8(base, v[g]);
        } else {
#pragma unroll
          for (int q = 0; q < UA; ++q) v[g][q] = base + q < n ? src.load(base + q) : VA(0);
        }
      }
#pragma unroll
      for (int g = 0; g < RA; ++g) {
        const int64_t base = wb + (int64_t)(g * 32 + lane) * UA;
#pragma unroll
        for (int q = 0; q < UA; ++q) hist_add(sh, base + q < n, src.bin_of(v[g][q]));
      }
    }
    __syncthreads();
    hist_flush(sh, ws.hist);
    grid_barrier(ws.bar, nb);
  }

#ifdef OTF_TOPK_TRACE
  uint64_t tstamp[5] = {0, 0, 0, 0, 0};
  __shared__ unsigned s_trace[2];
  if (threadIdx.x < 2) s_trace[threadIdx.x] = 0;
  __syncthreads();
#endif
  TOPK_STAMP(0);
  // ---- B: the bin holding the k-th entry ------------------------------------------------------
  int64_t C = n;
  uint32_t b0 = 0;
  if (!all) {
    find_bin<Src::kBins>(ws.hist, k_eff, &s_b, &s_above, &s_cnt, wsum);
    __syncthreads();
    b0 = (uint32_t)s_b;
    C = s_above + s_cnt;
    __syncthreads();
  }
  TOPK_STAMP(1);

  // (the plain gather below reads 8 scores per thread per pass; with fewer than ~4 passes its
  // single round trip beats the chunk path's three)
  if (C <= kCandCap && ws.clog >= 0 && !all && n > 32 * nthreads) {
    // ---- C': gather through the chunk maxima ---------------------------------------------------
    // The scoring kernel recorded the max bin of every 2^clog-row chunk; only chunks whose max
    // reaches b0 can hold a candidate (typically ~C of n/2^clog chunks), so the gather reads the
    // chunk maxima (2 B per chunk) plus those few chunks instead of every score.
    const int CH = 1 << ws.clog;
    const int64_t nch = (n + CH - 1) >> ws.clog;
    // every warp takes a contiguous block of G chunks (hits then spread over all warps); lanes
    // read 8 chunk maxima each (one 16-byte load) when G > 32, else one each
    const int64_t nwarps = nthreads >> 5, wg = wbase0 >> 5;
    int64_t G = (nch + nwarps - 1) / nwarps;
    const bool vec = G > 32;
    if (vec) G = (G + 7) & ~(int64_t)7;  // block starts stay 8-chunk aligned
    const int64_t cend = min(nch, (wg + 1) * G);
    for (int64_t cb = wg * G; cb < cend; cb += vec ? 256 : 32) {  // warp-uniform loop
      uint32_t hits = 0;
      if (vec) {
        const int64_t c0 = cb + 8 * lane;  // ws.cmax has a zeroed tail past nch
        if (c0 < cend) {
          const uint4 q = __ldcg(reinterpret_cast<const uint4*>(ws.cmax + c0));
          const uint32_t wv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (c0 + e < cend && ((wv[e >> 1] >> (16 * (e & 1))) & 0xffffu) >= b0) hits |= 1u << e;
        }
      } else if (cb + lane < cend && __ldcg(ws.cmax + cb + lane) >= b0) {
        hits = 1u;
      }
      // the warp's hit chunks (offsets from cb) go to a per-warp list in the dynamic shared
      // memory (free until rank_emit), then are scanned KB at a time
      const unsigned nh = __popc(hits);
      unsigned pos = nh;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned u = __shfl_up_sync(0xffffffffu, pos, o);
        if (lane >= o) pos += u;
      }
      const unsigned H = __shfl_sync(0xffffffffu, pos, 31);
#ifdef OTF_TOPK_TRACE
      if (lane == 0) { atomicAdd(&s_trace[0], H); atomicMax(&s_trace[1], H); }
#endif
      if (H == 0u) continue;
      uint16_t* list = reinterpret_cast<uint16_t*>(dyn) + (threadIdx.x >> 5) * 256;
      pos -= nh;
      for (uint32_t b = hits; b; b &= b - 1) list[pos++] = (uint16_t)(vec ? 8 * lane + __ffs(b) - 1 : lane);
      __syncwarp();
      constexpr int KB = 2, RPL = 4;  // chunks per batch, rows per lane per chunk (<= 128 rows)
      using V = decltype(src.load(0));
      for (unsigned h = 0; h < H; h += KB) {
        V v[KB][RPL];
        int64_t r0[KB];
#pragma unroll
        for (int j = 0; j < KB; ++j) {
          r0[j] = h + j < H ? (cb + list[h + j]) << ws.clog : n;  // n: empty slot
          src.prefetch_chunk(r0[j], CH, n, lane);
#pragma unroll
          for (int q = 0; q < RPL; ++q) {
            const int64_t i = r0[j] + 32 * q + lane;
            v[j][q] = 32 * q + lane < CH && i < n ? src.load(i) : V(0);
          }
        }
        uint32_t take = 0;
#pragma unroll
        for (int j = 0; j < KB; ++j)
#pragma unroll
          for (int q = 0; q < RPL; ++q)
            if (32 * q + lane < CH && r0[j] + 32 * q + lane < n && src.bin_of(v[j][q]) >= b0)
              take |= 1u << (j * RPL + q);
        // one atomic for the batch, then each lane scores and stores its own candidates
        const unsigned cnt = __popc(take);
        unsigned incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += u;
        }
        const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
        if (total == 0u) continue;
        unsigned slot0 = 0;
        if (lane == 0) slot0 = atomicAdd(ws.count, total);
        int64_t slot = (int64_t)__shfl_sync(0xffffffffu, slot0, 0) + incl - cnt;
#pragma unroll
        for (int j = 0; j < KB; ++j)
#pragma unroll
          for (int q = 0; q < RPL; ++q)
            if ((take >> (j * RPL + q)) & 1u) {
              const int64_t i = r0[j] + 32 * q + lane;
              if (slot < C) {
                ws.key[slot] = score_key(src.exact(i, v[j][q]));
                ws.inv[slot] = inv_id(id_of(ids, id_base, i));
                ws.row[slot] = i;
              }
              ++slot;
            }
      }
      __syncwarp();
    }
    TOPK_STAMP(2);
    grid_barrier(ws.bar, nb);
    TOPK_STAMP(3);
    if (vb == 0) {  // every CTA has read hist and count is no longer needed
      for (int b = threadIdx.x; b < kHistBinsMax; b += blockDim.x) ws.hist[b] = 0u;
      if (threadIdx.x == 0) *ws.count = 0u;
    }
    rank_emit_any(src, ws, C, k_eff, dyn, out_ids, out_scores, out_rows, vb, vnb);
    TOPK_STAMP(4);
    TOPK_REPORT();
    return;
  }

  if (C <= kCandCap) {
    // ---- C: gather the candidates, rank them ----------------------------------------------------
    // Each lane reads 8 consecutive entries with vector loads (a warp covers 256 contiguous
    // entries); candidates are rare (C out of n), so one warp vote skips the append path.
    // Each lane reads R groups of 8 consecutive entries per iteration (R*8 entries in flight).
    constexpr int U = 8;
    constexpr int R = 1;  // more groups spill at 64 registers (1024 threads) and ran slower
    using V = decltype(src.load(0));
    for (int64_t wb = wbase0 * U * R; wb < n; wb += nthreads * U * R) {  // warp-uniform loop
      V v[R][U];
#pragma unroll
      for (int g = 0; g < R; ++g) {
        const int64_t base = wb + (int64_t)(g * 32 + lane) * U;
        if (base + U <= n) {
          src.load8(base, v[g]);
        } else {
#pragma unroll
          for (int q = 0; q < U; ++q) v[g][q] = base + q < n ? src.load(base + q) : V(0);
        }
      }
#pragma unroll
      for (int g = 0; g < R; ++g) {
        const int64_t base = wb + (int64_t)(g * 32 + lane) * U;
        unsigned takes = 0;
#pragma unroll
        for (int q = 0; q < U; ++q)
          if (base + q < n && (all || src.bin_of(v[g][q]) >= b0)) takes |= 1u << q;
        if (__any_sync(0xffffffffu, takes != 0u)) {
#pragma unroll
          for (int q = 0; q < U; ++q) {
            const bool take = (takes >> q) & 1u;
            uint64_t key = 0, inv = 0;
            if (take) {
              key = score_key(src.exact(base + q, v[g][q]));
              inv = inv_id(id_of(ids, id_base, base + q));
            }
            append_candidate(ws, take, key, inv, base + q, C);
          }
        }
      }
    }
    TOPK_STAMP(2);
    grid_barrier(ws.bar, nb);
    TOPK_STAMP(3);
    if (vb == 0) {  // every CTA has read hist and count is no longer needed
      for (int b = threadIdx.x; b < kHistBinsMax; b += blockDim.x) ws.hist[b] = 0u;
      if (threadIdx.x == 0) *ws.count = 0u;
    }
    rank_emit_any(src, ws, C, k_eff, dyn, out_ids, out_scores, out_rows, vb, vnb);
    TOPK_STAMP(4);
    TOPK_REPORT();
    return;
  }

  // ---- D: exact radix select over a materialised score array --------------------------------
  const ST* scores = scratch;
  if (Src::kLoadBytes == 2) {  // bins-only source: compute every exact score once
    for (int64_t i = (int64_t)vb * blockDim.x + threadIdx.x; i < n; i += nthreads)
      scratch[i] = src.exact(i, src.load(i));
    grid_barrier(ws.bar, nb);
  }
  radix_select_emit(scores, src, n, ids, id_base, k_eff, ws, all, dyn, out_ids, out_scores, out_rows,
                    h, &s_b, &s_above, vb, vnb);
}

int topk_cut_alloc(TopkWs* ws) {
  if (ws->cut_cap >= kCutCap) return OTF_OK;
  OTF_CUDA(cudaMalloc(&ws->cut_key, 2 * kCutCap * sizeof(uint64_t)));  // (key, ~id) records
  OTF_CUDA(cudaMalloc(&ws->cut_row, kCutCap * sizeof(int64_t)));
  OTF_CUDA(cudaMalloc(&ws->cut_word, kCutWords * sizeof(unsigned int)));
  OTF_CUDA(cudaMemset(ws->cut_word, 0, kCutWords * sizeof(unsigned int)));
  OTF_CUDA(cudaMalloc(&ws->cut_smax, kCutSmaxCap * sizeof(uint32_t)));
  ws->cut_cap = kCutCap;
  return OTF_OK;
}

int topk_ws_alloc(TopkWs* ws, int64_t k_eff, int n_seg) {
  int64_t P = kCandCap;
  while (P < k_eff) P <<= 1;
  if (n_seg > ws->n_seg) {
    cudaFree(ws->hist);
    ws->hist = nullptr;
    ws->n_seg = 0;
    const size_t bytes = (size_t)n_seg * kWsWords * sizeof(uint32_t);
    OTF_CUDA(cudaMalloc(&ws->hist, bytes));
    OTF_CUDA(cudaMemset(ws->hist, 0, bytes));
    ws->rhist = ws->hist + kHistBinsMax;
    ws->bar = reinterpret_cast<unsigned int*>(ws->rhist + 3 * 256);
    ws->count = ws->bar + 2;
    ws->n_seg = n_seg;
    ws->cap = 0;  // re-layout the candidate arrays for the new segment count
  }
  if (P > ws->cap || (size_t)ws->n_seg * P > ws->slots) {
    cudaFree(ws->key); cudaFree(ws->inv); cudaFree(ws->row);
    ws->key = nullptr; ws->inv = nullptr; ws->row = nullptr; ws->cap = 0; ws->slots = 0;
    const size_t slots = (size_t)ws->n_seg * P;
    OTF_CUDA(cudaMalloc(&ws->key, slots * sizeof(uint64_t)));
    OTF_CUDA(cudaMalloc(&ws->inv, slots * sizeof(uint64_t)));
    OTF_CUDA(cudaMalloc(&ws->row, slots * sizeof(int64_t)));
    ws->cap = P;
    ws->slots = slots;
  }
  return OTF_OK;
}

int topk_cmax_ensure(TopkWs* ws, int64_t n) {
  // chunks of >= 8 rows, plus a zeroed tail so the 8-chunk vector loads stay in bounds
  const size_t need = (size_t)((n + 7) / 8) + 256;
  if (need > ws->cmax_cap) {
    cudaFree(ws->cmax);
    ws->cmax = nullptr;
    ws->cmax_cap = 0;
    OTF_CUDA(cudaMalloc(&ws->cmax, need * sizeof(uint16_t)));
    OTF_CUDA(cudaMemset(ws->cmax, 0, need * sizeof(uint16_t)));
    ws->cmax_cap = need;
  }
  return OTF_OK;
}

void topk_ws_free(TopkWs* ws) {
  cudaFree(ws->hist); cudaFree(ws->key); cudaFree(ws->inv); cudaFree(ws->row); cudaFree(ws->cmax);
  cudaFree(ws->cut_key); cudaFree(ws->cut_row); cudaFree(ws->cut_word); cudaFree(ws->cut_smax);
  *ws = TopkWs{};
}

template <typename Src>
static int launch_src(const Src& src, int64_t n, const int64_t* ids, int64_t id_base, int64_t k_eff,
                      TopkWs* ws, bool hist_ready, typename Src::T* scratch, int64_t* out_ids,
                      double* out_scores, int64_t* out_rows, int device, cudaStream_t st, int n_seg = 1) {
  auto fn = topk_coop_kernel<Src>;
  static bool configured[64] = {false};
  if (!configured[device & 63]) {
    OTF_CUDA(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kTopkSmem));
    configured[device & 63] = true;
  }
  int per = sm_count(device) * kTopkCtasPerSm / n_seg;  // CTAs per segment
  if (per < 1) return fail(OTF_ERR_CONFIG, "more top-k segments than SMs");
  const int64_t useful = (n + kTopkThreads - 1) / kTopkThreads;
  if (useful < per) per = (int)(useful > 0 ? useful : 1);
  const int grid = per * n_seg;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTopkThreads);
  cfg.dynamicSmemBytes = kTopkSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // follows the fused scoring kernel
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const bool no_pdl = getenv("OTF_TOPK_NO_PDL") != nullptr;  // A/B switch (tools/)
  cfg.numAttrs = hist_ready && !no_pdl ? 2 : 1;
  OTF_CUDA(cudaLaunchKernelEx(&cfg, fn, src, n, ids, id_base, k_eff, *ws, (int)hist_ready, scratch,
                              out_ids, out_scores, out_rows, n_seg));
  count_launch();
  return OTF_OK;
}

int launch_topk(const void* scores, int dtype, int64_t n, const int64_t* ids, int64_t id_base,
                int64_t k_eff, TopkWs* ws, bool hist_ready, int64_t* out_ids, double* out_scores,
                int64_t* out_rows, int device, cudaStream_t st) {
  if (k_eff <= 0 || n <= 0) return OTF_OK;
  int rc = topk_ws_alloc(ws, k_eff);
  if (rc) return rc;
  if (dtype == OTF_F32) {
    DirectSrc<float> src{static_cast<const float*>(scores)};
    return launch_src(src, n, ids, id_base, k_eff, ws, hist_ready, const_cast<float*>(src.s), out_ids,
                      out_scores, out_rows, device, st);
  }
  DirectSrc<double> src{static_cast<const double*>(scores)};
  return launch_src(src, n, ids, id_base, k_eff, ws, hist_ready, const_cast<double*>(src.s), out_ids,
                    out_scores, out_rows, device, st);
}

// n_seg independent top-k selections over consecutive float32 score arrays (scores + s*n), one
// cooperative launch; outputs at out_ids/out_scores + s*k_eff. ws must be a segment workspace.
int launch_topk_segments(const float* scores, int n_seg, int64_t n, const int64_t* ids, int64_t id_base,
                         int64_t k_eff, TopkWs* ws, int64_t* out_ids, double* out_scores, int device,
                         cudaStream_t st) {
  if (k_eff <= 0 || n <= 0 || n_seg <= 0) return OTF_OK;
  int rc = topk_ws_alloc(ws, k_eff, n_seg);
  if (rc) return rc;
  DirectSrc<float> src{scores};
  return launch_src(src, n, ids, id_base, k_eff, ws, false, const_cast<float*>(scores), out_ids, out_scores,
                    nullptr, device, st, n_seg);
}

// ---- many selections at once, by a sampled threshold per segment (C5b's rank_many) -------------
// n_seg independent top-k selections over consecutive float32 score arrays (scores + s * n), one
// cooperative launch over the whole GPU:
//   1. sample: warp w takes (segment, chunk) pairs — 64 chunks of 4096 consecutive scores spread
//      over each segment — and publishes the chunk's four largest order keys;
//   2. grid barrier; every CTA derives each segment's T_s = the r-th largest of its 256 published
//      keys (r ~ (2 k + 128) x sample / n: ~2 k + 128 rows are expected at or above T_s);
//   3. one pass over every score appends (key, ~id, row) of the scores with key >= T_s to the
//      segment's candidate list (no histogram pass: scores concentrate in a few dozen 12-bit bins,
//      and the segmented histogram's shared atomics serialised on them);
//   4. grid barrier; the CTAs split into n_seg groups; a group ranks its segment's candidates by
//      counting (rank_emit) when k <= C_s <= kCandCap, else runs the exact radix select over the
//      segment (otf_topk_dev.cuh) — slower, same result.
// Same order as top_k (ranker.py:97-143): the selection is exact whatever T_s is.
constexpr int kSegSampleChunks = 64, kSegChunk = 4096, kSegPub = 4;

__global__ void __launch_bounds__(kTopkThreads, kTopkCtasPerSm)
topk_seg_cut_kernel(const float* __restrict__ scores, int n_seg, int64_t n, const int64_t* __restrict__ ids,
                    int64_t id_base, int64_t k_eff, int r, TopkWs ws, int64_t* __restrict__ out_ids,
                    double* __restrict__ out_scores) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ uint32_t s_T[64];
  __shared__ uint32_t h[256];
  __shared__ int s_b;
  __shared__ int64_t s_above;
  const unsigned G = gridDim.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = kTopkThreads / 32;
  const int64_t gw = (int64_t)blockIdx.x * nw + wid, ngw = (int64_t)G * nw;
  unsigned int* gbar = ws.cut_word + 12;  // the whole grid's barrier word (8-byte aligned)
#ifdef OTF_SEG_TRACE
  unsigned long long ts[6];
#define SEG_STAMP(i) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts[i]))
#else
#define SEG_STAMP(i)
#endif
  SEG_STAMP(0);
  // 1. the sample (and the segment counters are cleared before anyone appends)
  if (blockIdx.x == 0)
    for (int sg = threadIdx.x; sg < n_seg; sg += blockDim.x) *seg_ws(ws, (unsigned)sg).count = 0u;
  const int64_t stride = n / kSegSampleChunks;
  for (int64_t t = gw; t < (int64_t)n_seg * kSegSampleChunks; t += ngw) {
    const int sg = (int)(t / kSegSampleChunks), c = (int)(t % kSegSampleChunks);
    const float* sp = scores + (int64_t)sg * n + (int64_t)c * stride;
    uint32_t top[kSegPub] = {0u, 0u, 0u, 0u};  // this lane's largest keys, descending
#pragma unroll 4
    for (int i = lane; i < kSegChunk; i += 32) {
      const uint32_t k = (uint32_t)score_key(__ldcg(sp + i));
      if (k > top[3]) {
        top[3] = k;
#pragma unroll
        for (int q = 3; q > 0; --q)
          if (top[q] > top[q - 1]) { const uint32_t x = top[q]; top[q] = top[q - 1]; top[q - 1] = x; }
      }
    }
#pragma unroll
    for (int q = 0; q < kSegPub; ++q) {  // the warp's four largest: pop the maximum four times
      const uint32_t m = __reduce_max_sync(0xffffffffu, top[0]);
      const unsigned hit = __ballot_sync(0xffffffffu, top[0] == m);
      if (lane == __ffs(hit) - 1) { top[0] = top[1]; top[1] = top[2]; top[2] = top[3]; top[3] = 0u; }
      if (lane == 0) ws.cut_smax[((int64_t)sg * kSegSampleChunks + c) * kSegPub + q] = m;
    }
  }
  SEG_STAMP(1);
  grid_barrier(gbar, G);
  SEG_STAMP(2);
  // 2. T_s for every segment (each warp: segments wid, wid + nw; 256 keys, 8 per lane): the r-th
  // largest at 16-bit key resolution (two 8-bit radix passes over a per-warp shared histogram),
  // rounded down to that prefix's lower edge
  {
    uint32_t* wh = reinterpret_cast<uint32_t*>(dyn) + wid * 256;
    for (int sg = wid; sg < n_seg; sg += nw) {
      uint32_t v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = __ldcg(ws.cut_smax + (int64_t)sg * 256 + lane + 32 * q);
      uint32_t prefix = 0, T = 0;
      int need = r;
      for (int pass = 0; pass < 2; ++pass) {
        const int shift = 24 - 8 * pass;
#pragma unroll
        for (int q = 0; q < 8; ++q) wh[lane + 32 * q] = 0u;
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (v[q] != 0u && (pass == 0 || (v[q] >> 24) == prefix)) atomicAdd(&wh[(v[q] >> shift) & 255u], 1u);
        __syncwarp();
        // lane l owns bins 255 - 8 l - 7 .. 255 - 8 l (descending); the bin holding the need-th key
        uint32_t c[8];
        int local = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) { c[q] = wh[255 - 8 * lane - q]; local += (int)c[q]; }
        int incl = local;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        if (tot < need) { T = 0u; break; }  // fewer than r sampled keys: the segment falls back
        const unsigned hit = __ballot_sync(0xffffffffu, incl >= need);
        const int first = __ffs(hit) - 1;
        int bin = 0, above = 0;
        if (lane == first) {
          int cum = incl - local;
          for (int q = 0; q < 8; ++q) {
            if (cum + (int)c[q] >= need) { bin = 255 - 8 * lane - q; above = cum; break; }
            cum += (int)c[q];
          }
        }
        bin = __shfl_sync(0xffffffffu, bin, first);
        above = __shfl_sync(0xffffffffu, above, first);
        need -= above;
        prefix = pass == 0 ? (uint32_t)bin : (prefix << 8) | (uint32_t)bin;
        if (pass == 1) T = prefix << 16;
        __syncwarp();
      }
      if (lane == 0) s_T[sg] = T;
    }
  }
  __syncthreads();
  SEG_STAMP(3);
  // 3. emission: lane l of a warp takes two float4 (flat positions 4 l and 128 + 4 l of a 256-score
  // run); a take is rare (~0.02% of the scores), so one comparison per float4 decides
  const int64_t total = (int64_t)n_seg * n;
  auto emit = [&](int64_t f, float sc) {  // f: flat position of a score at or above its T
    const int sg = (int)(f / n);
    const int64_t row = f - (int64_t)sg * n;
    const TopkWs w = seg_ws(ws, (unsigned)sg);
    const unsigned slot = atomicAdd(w.count, 1u);
    if ((int64_t)slot < w.cap) {
      w.key[slot] = score_key(sc);
      w.inv[slot] = inv_id(id_of(ids, id_base, row));
      w.row[slot] = row;
    }
  };
  auto test4 = [&](int64_t f, float4 x, int cnt) {  // cnt valid scores from f
    const int sg = (int)(f / n);
    const int64_t bnd = (int64_t)(sg + 1) * n;  // the next segment starts here
    const uint32_t T0 = s_T[sg], T1 = bnd < f + cnt && sg + 1 < n_seg ? s_T[sg + 1] : T0;
    const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (q >= cnt) break;
      const uint32_t T = f + q < bnd ? T0 : T1;
      if (T != 0u && (uint32_t)score_key(xs[q]) >= T) emit(f + q, xs[q]);
    }
  };
  const bool aligned = (reinterpret_cast<uintptr_t>(scores) & 15) == 0;
  constexpr int kRuns = 8;  // float4 per lane in flight (1024 scores per warp iteration)
  for (int64_t f0 = gw * (128 * kRuns); f0 < total; f0 += ngw * (128 * kRuns)) {
    // the warp's run two iterations ahead streams into L2 meanwhile (one bulk prefetch): the
    // loads below then wait on L2, not HBM (32 warps x 4 KB in flight per SM is not enough)
    if (lane == 0 && aligned) {
      const int64_t fp = f0 + 2 * ngw * (128 * kRuns);
      if (fp + 128 * kRuns <= total)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(scores + fp), "r"(512u * kRuns) : "memory");
    }
    float4 x[kRuns];
    // one division per 1024 scores: a run spans at most two segments (n >= 1M, topk_seg_cut_plan)
    const int sg0 = (int)(f0 / n);
    const int64_t bnd0 = (int64_t)(sg0 + 1) * n;
    if (aligned && f0 + 128 * kRuns <= bnd0) {
      // (warp-uniform) the whole run is in range and in ONE segment: no per-score index checks —
      // round 2: the general path below spent ~106 instructions per float4 on 64-bit index tests
      // (C5b: 1.06 ms for 2.56 GB)
#pragma unroll
      for (int h = 0; h < kRuns; ++h)
        x[h] = ld_stream_f4(reinterpret_cast<const float4*>(scores + f0 + 128 * h + 4 * lane));
      const uint32_t t = s_T[sg0] ? s_T[sg0] : 0xffffffffu;
      if (t > 0x80000000u) {
        // T above +0.0 (the usual case): a key >= T needs a positive float whose bits, as a signed
        // integer, are >= T ^ 0x80000000; negative floats (and -0.0) are negative integers, and a
        // positive NaN passes to the exact test. One integer max per four scores.
        const int tb = (int)(t ^ 0x80000000u);
#pragma unroll
        for (int h = 0; h < kRuns; ++h) {
          const int m = max(max(__float_as_int(x[h].x), __float_as_int(x[h].y)),
                            max(__float_as_int(x[h].z), __float_as_int(x[h].w)));
          if (m >= tb) test4(f0 + 128 * h + 4 * lane, x[h], 4);
        }
      } else {
#pragma unroll
        for (int h = 0; h < kRuns; ++h) {
          const uint32_t kmax = max(max((uint32_t)score_key(x[h].x), (uint32_t)score_key(x[h].y)),
                                    max((uint32_t)score_key(x[h].z), (uint32_t)score_key(x[h].w)));
          if (kmax >= t) test4(f0 + 128 * h + 4 * lane, x[h], 4);
        }
      }
      continue;
    }
#pragma unroll
    for (int h = 0; h < kRuns; ++h) {
      const int64_t f = f0 + 128 * h + 4 * lane;
      if (f + 4 <= total && aligned) {
        x[h] = ld_stream_f4(reinterpret_cast<const float4*>(scores + f));  // (256 B L2 fetches, evict-first)
      } else {
        x[h].x = f < total ? __ldcs(scores + f) : 0.f;
        x[h].y = f + 1 < total ? __ldcs(scores + f + 1) : 0.f;
        x[h].z = f + 2 < total ? __ldcs(scores + f + 2) : 0.f;
        x[h].w = f + 3 < total ? __ldcs(scores + f + 3) : 0.f;
      }
    }
#pragma unroll
    for (int h = 0; h < kRuns; ++h) {
      const int64_t f = f0 + 128 * h + 4 * lane;
      if (f >= total) continue;
      const int cnt = (int)min((int64_t)4, total - f);
      // quick reject: the largest key of the four against the smaller of the (at most two) T's
      const int sg = f < bnd0 ? sg0 : sg0 + 1;
      const uint32_t t0 = s_T[sg] ? s_T[sg] : 0xffffffffu;
      const uint32_t t1 = sg + 1 < n_seg && (int64_t)(sg + 1) * n < f + cnt ? (s_T[sg + 1] ? s_T[sg + 1] : 0xffffffffu)
                                                                           : 0xffffffffu;
      const uint32_t kmax = max(max((uint32_t)score_key(x[h].x), cnt > 1 ? (uint32_t)score_key(x[h].y) : 0u),
                                max(cnt > 2 ? (uint32_t)score_key(x[h].z) : 0u, cnt > 3 ? (uint32_t)score_key(x[h].w) : 0u));
      if (kmax >= min(t0, t1)) test4(f, x[h], cnt);
    }
  }
  SEG_STAMP(4);
  grid_barrier(gbar, G);
  SEG_STAMP(5);
#ifdef OTF_SEG_TRACE
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == G - 1))
    printf("segT cta %d sample %.1f barrier %.1f T %.1f emit %.1f barrier %.1f us\n", (int)blockIdx.x,
           (ts[1] - ts[0]) * 1e-3, (ts[2] - ts[1]) * 1e-3, (ts[3] - ts[2]) * 1e-3, (ts[4] - ts[3]) * 1e-3,
           (ts[5] - ts[4]) * 1e-3);
#endif
  // 4. per-segment groups of G / n_seg CTAs: rank the candidates, or the exact select
  const unsigned per = G / (unsigned)n_seg;
  const unsigned sg = blockIdx.x / per, vb = blockIdx.x % per;
  if (sg >= (unsigned)n_seg) return;
  const TopkWs w = seg_ws(ws, sg);
  const unsigned C = __ldcg(w.count);
  DirectSrc<float> src{scores + (int64_t)sg * n};
  if (s_T[sg] != 0u && (int64_t)C >= k_eff && C <= (unsigned)kCandCap) {
    rank_emit_k32(src, w, (int64_t)C, k_eff, dyn, out_ids + (int64_t)sg * k_eff, out_scores + (int64_t)sg * k_eff,
                  nullptr, vb, per);
    grid_barrier(w.bar, per);  // (the other path's kernels expect a zero count)
    if (vb == 0 && threadIdx.x == 0) *w.count = 0u;
    return;
  }
  if (vb == 0 && threadIdx.x == 0) atomicAdd(ws.cut_word + 3, 1u);  // fallbacks taken (diagnostics)
  grid_barrier(w.bar, per);  // the group's CTAs have read the count
  if (vb == 0 && threadIdx.x == 0) *w.count = 0u;
  grid_barrier(w.bar, per);
  radix_select_emit(src.s, src, n, ids, id_base, k_eff, w, k_eff >= n, dyn, out_ids + (int64_t)sg * k_eff,
                    out_scores + (int64_t)sg * k_eff, nullptr, h, &s_b, &s_above, vb, per);
}

bool topk_seg_cut_plan(int n_seg, int64_t n, int64_t k_eff, int device, int* r) {
  static const bool off = getenv("OTF_SEG_NO_CUT") != nullptr;  // A/B switch (tools/)
  if (off || n_seg < 1 || n_seg > 64 || k_eff <= 0) return false;
  if (sm_count(device) / n_seg < 1) return false;
  const int64_t S = (int64_t)kSegSampleChunks * kSegChunk;
  if (n < 4 * S) return false;  // the sample is at most a quarter of a segment
  const int64_t want = 2 * k_eff + 128;
  if (2 * want > kCandCap) return false;
  const int64_t rr = (want * S + n - 1) / n;
  if (rr > kSegSampleChunks * kSegPub / 4) return false;  // the published keys must cover the top r
  *r = (int)std::max<int64_t>(rr, 1);
  return true;
}

int launch_topk_seg_cut(const float* scores, int n_seg, int64_t n, const int64_t* ids, int64_t id_base, int64_t k_eff,
                        int r, TopkWs* ws, int64_t* out_ids, double* out_scores, int device, cudaStream_t st) {
  int rc = topk_ws_alloc(ws, k_eff, n_seg);
  if (!rc) rc = topk_cut_alloc(ws);
  if (rc) return rc;
  auto fn = topk_seg_cut_kernel;
  static bool configured[64] = {false};
  if (!configured[device & 63]) {
    OTF_CUDA(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTopkSmem));
    configured[device & 63] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(sm_count(device) * kTopkCtasPerSm));
  cfg.blockDim = dim3(kTopkThreads);
  cfg.dynamicSmemBytes = kTopkSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OTF_CUDA(cudaLaunchKernelEx(&cfg, fn, scores, n_seg, n, ids, id_base, k_eff, r, *ws, out_ids, out_scores));
  count_launch();
  return OTF_OK;
}

int launch_topk_pq_bins(const uint16_t* bins, const uint8_t* codes, int M, const double* lut, int K,
                        int64_t n, const int64_t* ids, int64_t id_base, int64_t k_eff, TopkWs* ws,
                        double* scratch, int64_t* out_ids, double* out_scores, int64_t* out_rows,
                        int device, cudaStream_t st) {
  if (k_eff <= 0 || n <= 0) return OTF_OK;
  int rc = topk_ws_alloc(ws, k_eff);
  if (rc) return rc;
  PqBinSrc src{bins, codes, lut, M, K};
  return launch_src(src, n, ids, id_base, k_eff, ws, true, scratch, out_ids, out_scores, out_rows,
                    device, st);
}

}  // namespace otf
