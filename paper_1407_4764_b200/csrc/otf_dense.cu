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
#include <algorithm>
#include <cstdlib>

#include "otf_common.cuh"
#include "otf_internal.h"
#include "otf_topk_dev.cuh"

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

// One warp iteration of the fast path: rows [r0, r0 + R) (d == 128 * CPL). Each warp handles R
// rows per iteration, then a transposed butterfly gives ~2 shuffles per row. Returns the score
// of row r0 + row_of_lane<R, 32>(lane) (meaningful on its writer lane when that row is < n).
// Every fast-path kernel (scores, fused rank) scores through this one function, so a row's
// score is the same bits whichever kernel or shard computed it.
template <int CPL, int R>
__device__ __forceinline__ float dense_iter(const float4* __restrict__ X4, int64_t n, int64_t r0,
                                           const float4* wr, int lane) {
  const int64_t row_f4 = 32 * CPL;  // float4 per row
  constexpr int LB = CPL < 8 ? CPL : 8;  // float4 loads per row per batch
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
  return __double2float_rn(p[0]);
}

template <int CPL>
__device__ __forceinline__ void stage_w(const double* __restrict__ w, float4* wr) {
  for (int t = threadIdx.x; t < 32 * CPL; t += blockDim.x)
    wr[t] = make_float4(__double2float_rn(w[4 * t]), __double2float_rn(w[4 * t + 1]),
                        __double2float_rn(w[4 * t + 2]), __double2float_rn(w[4 * t + 3]));
}

// Fast path: d == 128 * CPL, every row's score (+ the fused histogram / chunk maxima).
// claim (nullable): 10 words {4 u64 tail counters, done ticket, pad} zero on entry, left zero. With
// it the last quarter of the groups is handed out dynamically, 4 groups per claim, by 4 counters
// (as dense_rank_cut's tail), so faster SMs take more and the kernel ends within ~one claim of
// its mean; without it (score(), no workspace) every group is assigned statically.
template <int CPL, int R>
__global__ void __launch_bounds__(256, 2) dense_score_fast(const float* __restrict__ X, int64_t n,
                                                           const double* __restrict__ w,
                                                           float* __restrict__ out,
                                                           uint32_t* __restrict__ ghist,
                                                           uint16_t* __restrict__ cmax,
                                                           unsigned int* __restrict__ claim) {
  const int lane = threadIdx.x & 31;
  __shared__ float4 wr[32 * CPL];
  __shared__ uint32_t sh[kHistBins];
  // the top-k kernel (programmatic launch) may be scheduled now: its CTAs take SMs as this grid's
  // CTAs finish and wait in griddepcontrol.wait for this grid's writes
  asm volatile("griddepcontrol.launch_dependents;");
  stage_w<CPL>(w, wr);
  if (ghist) hist_zero(sh);
  __syncthreads();
  const float4* X4 = reinterpret_cast<const float4*>(X);
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ngroups = (n + R - 1) / R;
  auto group = [&](int64_t g) {
    const int64_t r0 = g * R;
    const float s = dense_iter<CPL, R>(X4, n, r0, wr, lane);
    bool writer;
    const int slot = row_of_lane<R, 32>(lane, &writer);
    const int64_t row = r0 + slot;
    const bool active = writer && row < n;
    if (active) out[row] = s;
    if (ghist) hist_add(sh, active, hist_bin(s));
    if (R > 1 && cmax) {  // the warp's R consecutive rows are one top-k chunk
      const uint32_t wm = __reduce_max_sync(0xffffffffu, active ? hist_bin(s) : 0u);
      if (lane == 0) cmax[g] = (uint16_t)wm;
    }
  };
  const int64_t gstat = claim ? (ngroups - ngroups / 4) / nwarp * nwarp : ngroups;
  // one loop (one inlined copy of the scan): static groups warp, warp + nwarp, ... below gstat,
  // then tail groups gstat + 4 j + (warp & 3) for j claimed four at a time
  const int c = (int)(warp & 3);
  unsigned long long* ctr = claim ? reinterpret_cast<unsigned long long*>(claim) + c : nullptr;
  int64_t j = 0;
  int left = 0;
  auto tail = [&]() -> int64_t {
    if (!claim) return ngroups;
    if (left == 0) {
      unsigned long long j0 = 0;
      if (lane == 0) j0 = atomicAdd(ctr, 4ull);
      j = (int64_t)__shfl_sync(0xffffffffu, j0, 0);
      left = 4;
    } else {
      ++j;
    }
    --left;
    const int64_t g = gstat + 4 * j + c;
    return g < ngroups ? g : ngroups;
  };
  for (int64_t g = warp < gstat ? warp : tail(); g < ngroups;) {  // warp-uniform
    group(g);
    g += nwarp;
    if (g >= gstat) g = tail();
  }
  if (claim) {
    // the last CTA out clears the counters for the next launch
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(claim + 8, 1u) == gridDim.x - 1) {
        for (int q = 0; q < 9; ++q) claim[q] = 0u;
        __threadfence();
      }
    }
  }
  if (ghist) {
    __syncthreads();
    hist_flush(sh, ghist);
  }
}

// ---- fused rank (score + exact top-k in one cooperative launch) --------------------------------
// The rank path needs the k best rows, not every row's score. dense_rank_cut (persistent grid,
// 2 CTAs x 8 warps per SM, cooperative) works on groups of R rows (one warp iteration each):
//   1. the sample: warp w scores the `sit` groups starting at group w * floor(ngroups / nwarp)
//      (nwarp * sit * R rows spread over the whole repository), keeps those scores in `scratch`
//      and the CTA publishes its four largest sample keys; a split grid barrier: while the other
//      CTAs finish their sample, each warp scores its first scan group and holds the scores in
//      registers (HBM stays busy); every CTA then takes T = the r-th largest of the 4 G published
//      keys at 16-bit key resolution (r ~ want x sample / n, want ~ 1.56 k + 128, so ~want rows are
//      expected at or above T), rounded down to that key prefix's lower edge;
//   2. the scan: warp w scores groups w, w + nwarp, ... (interleaved as dense_score_fast, the
//      sample groups skipped) and appends (key, ~id, row) of every row with key >= T to a
//      candidate list (warp-aggregated atomics; ~0.2% of the rows at k = 1000, 1M rows): no
//      per-row score, histogram or chunk-maximum writes;
//   3. one more grid barrier; when at least k and at most kDcSelCap rows reached T, the global top
//      k is among them: every CTA copies the candidates' 32-bit keys into shared memory and ranks
//      its share by counting (candidate i on CTA i mod G; ids and rows are read only for exact
//      key ties), writing each straight to its output slot. Otherwise (heavy ties, w = 0, a sample
//      far off the distribution) every row's score is written to `scratch` and the exact radix
//      select (otf_topk_dev.cuh) runs — slower, same result.
// Order: (score desc, id asc), -0.0 tied with +0.0, the row as the last tie key (ranker.py:97-143).
// Measured (B200, same box): C2 (1M x 2048) 1.117 vs 1.177 ms per query for scan + top-k
// kernel; C4 6.87 vs 7.23 ms; C1 (1M x 128) 96.6-97.4 vs 99.2 us.
#ifndef OTF_DC_TAIL_DIV  // 1 / OTF_DC_TAIL_DIV of the groups are handed out dynamically
#define OTF_DC_TAIL_DIV 4
#endif
#ifndef OTF_DC_CLAIM  // groups per claim of the dynamic tail
#define OTF_DC_CLAIM 1
#endif
#ifndef OTF_DC_CTRS  // claim counters of the dynamic tail (<= 16, one cache line each)
#define OTF_DC_CTRS 16
#endif
constexpr int kDcCtrWord = 64, kDcCtrStride = 32;  // tail counter c: cut words 64 + 32 c (one 128-byte line each)
constexpr int kDcThreads = 256;
constexpr int kDcSelCap = 5120;  // candidates ranked in shared memory (32-bit keys)
constexpr int kDcFallbackK = 1280;  // the radix fallback ranks k (key, inv) pairs in the same memory
constexpr size_t kDcSmem = (size_t)kDcSelCap * 4 > (size_t)kDcFallbackK * 16 ? (size_t)kDcSelCap * 4
                                                                              : (size_t)kDcFallbackK * 16;
constexpr int kDcPub = 4;         // sample keys published per CTA
constexpr int kDcPerThread = 8;   // published keys per thread in the T search (G <= 512)
#ifndef OTF_DC_HOLD_SMALL  // scan groups a warp scores while the grid synchronises (R <= 2)
#define OTF_DC_HOLD_SMALL 1
#endif
#ifdef OTF_DCUT_TRACE  // diagnostic build: per-CTA globaltimer stamps of the phases
#define DC_STAMP(i) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts[i]))
#else
#define DC_STAMP(i)
#endif

template <int CPL, int R>
__global__ void __launch_bounds__(kDcThreads, 2)
dense_rank_cut(const float* __restrict__ X, int64_t n, const double* __restrict__ w,
               const int64_t* __restrict__ ids, int64_t id_base, int64_t k_eff, int r, int sit, TopkWs ws,
               float* __restrict__ scratch, int64_t* __restrict__ out_ids, double* __restrict__ out_scores,
               int64_t* __restrict__ out_rows) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ float4 wr[32 * CPL];
  __shared__ uint32_t h[256];
  __shared__ int s_b;
  __shared__ int64_t s_above;
  __shared__ uint32_t s_tkey;
  __shared__ unsigned s_nz;
  __shared__ unsigned s_last;
  __shared__ uint32_t s_top[2 * (kDcThreads / 32)];
  __shared__ unsigned s_gen;
#ifdef OTF_DCUT_TRACE
  unsigned long long ts[7] = {0, 0, 0, 0, 0, 0, 0};
#endif
  DC_STAMP(0);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned G = gridDim.x, vb = blockIdx.x;
  stage_w<CPL>(w, wr);
  if (threadIdx.x == 0) { s_tkey = 0u; s_nz = 0u; }
  __syncthreads();
  const float4* X4 = reinterpret_cast<const float4*>(X);
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ngroups = (n + R - 1) / R;
  const int64_t gps = ngroups / nwarp;  // sample stride (>= sit: dense_cut_plan)
  const int64_t gs0 = warp * gps;       // this warp's sample groups [gs0, gs0 + sit)
  auto is_sample = [&](int64_t g) {
    const int64_t q = g / gps;
    return q < nwarp && g - q * gps < sit;
  };
  bool writer;
  const int slot = row_of_lane<R, 32>(lane, &writer);
  unsigned long long* cut_count = reinterpret_cast<unsigned long long*>(ws.cut_word);
  ulonglong2* cut_rec = reinterpret_cast<ulonglong2*>(ws.cut_key);
  uint32_t* key32 = reinterpret_cast<uint32_t*>(ws.key);  // compact keys of the first kDcSelCap candidates

  // ---- 1. the sample ------------------------------------------------------------------------------
  {
    uint32_t ka = 0u, kb = 0u;  // this lane's two largest sample keys (0: none)
    for (int64_t g = gs0; g < gs0 + sit; ++g) {
      const float s = dense_iter<CPL, R>(X4, n, g * R, wr, lane);
      const int64_t row = g * R + slot;
      if (writer && row < n) {
        scratch[row] = s;
        const uint32_t k = (uint32_t)score_key(s);
        if (k > ka) { kb = ka; ka = k; } else if (k > kb) { kb = k; }
      }
    }
    uint32_t m1, m2;
    warp_top2(ka, kb, m1, m2);
    if (lane == 0) { s_top[2 * wid] = m1; s_top[2 * wid + 1] = m2; }
    __syncthreads();
    if (wid == 0) {  // the CTA's four largest of its warps' 16 published keys
      uint32_t v = lane < 2 * (kDcThreads / 32) ? s_top[lane] : 0u;
#pragma unroll
      for (int q = 0; q < kDcPub; ++q) {
        const uint32_t m = __reduce_max_sync(0xffffffffu, v);
        const unsigned hit = __ballot_sync(0xffffffffu, v == m);
        if (lane == __ffs(hit) - 1) v = 0u;
        if (lane == 0) ws.cut_smax[kDcPub * vb + q] = m;
      }
    }
  }
  DC_STAMP(1);
  // split barrier: while the other CTAs finish their sample, each warp scores kDcHold groups of
  // the scan and holds their scores in registers (HBM stays busy; no idle wait)
  const unsigned gen = grid_arrive(ws.bar, G, &s_gen);
  // the scan: warp w takes groups w, w + nwarp, ... (interleaved as dense_score_fast), skipping
  // the sample groups
  auto next_group = [&](int64_t g) {
    while (g < ngroups && is_sample(g)) g += nwarp;
    return g;
  };
  int64_t gcur = next_group(warp);
  constexpr int kDcHold = R <= 2 ? OTF_DC_HOLD_SMALL : 1;
  float held[kDcHold];
  int64_t heldg[kDcHold];
#pragma unroll
  for (int h2 = 0; h2 < kDcHold; ++h2) {
    heldg[h2] = gcur;
    held[h2] = 0.f;
    if (gcur < ngroups) {  // warp-uniform
      held[h2] = dense_iter<CPL, R>(X4, n, gcur * R, wr, lane);
      gcur = next_group(gcur + nwarp);
    }
  }
  grid_wait(ws.bar, G, gen);
  DC_STAMP(2);
  // T = the r-th largest published key at 16-bit resolution (two 8-bit radix passes in shared
  // memory over the kDcPub G values, held in registers: one L2 round trip), rounded down to that
  // prefix's lower edge
  {
    const int nv = kDcPub * (int)G;  // <= kDcPerThread * blockDim (dense_cut_plan)
    uint32_t v[kDcPerThread];
#pragma unroll
    for (int q = 0; q < kDcPerThread; ++q) {
      const int i = (int)threadIdx.x + q * kDcThreads;
      v[q] = i < nv ? __ldcg(ws.cut_smax + i) : 0u;
    }
    unsigned nz = 0;
#pragma unroll
    for (int q = 0; q < kDcPerThread; ++q) nz += v[q] != 0u;
    if (nz) atomicAdd(&s_nz, nz);  // read after the pass-0 barriers below
    uint32_t prefix = 0;
    int64_t need = r;
    for (int pass = 0; pass < 2; ++pass) {
      const int shift = 24 - 8 * pass;
      h[threadIdx.x] = 0u;  // blockDim == 256
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kDcPerThread; ++q)
        if (v[q] != 0u && (pass == 0 || (v[q] >> 24) == prefix)) atomicAdd(&h[(v[q] >> shift) & 255u], 1u);
      __syncthreads();
      if ((int64_t)s_nz < need) break;  // fewer than r sampled keys (uniform): fallback
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
  const bool usable = tkey != 0u;

  // ---- 2. emission: the sample rows, the held groups, then the rest of the scan ----------------------
  auto emit = [&](bool take, float s, int64_t row) {
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    if (bal == 0u) return;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(cut_count, (unsigned long long)__popc(bal));
    const int64_t sl = (int64_t)__shfl_sync(0xffffffffu, base, 0) + __popc(bal & lanemask_lt());
    if (take && sl < ws.cut_cap) {
      const uint64_t key = score_key(s);
      cut_rec[sl] = make_ulonglong2((key << 32) | (uint64_t)__float_as_uint(s), inv_id(id_of(ids, id_base, row)));
      ws.cut_row[sl] = row;
      if (sl < kDcSelCap) key32[sl] = (uint32_t)key;
    }
  };
  for (int64_t g = gs0; g < gs0 + sit; ++g) {
    const int64_t row = g * R + slot;
    const bool own = writer && row < n;
    const float s = own ? scratch[row] : 0.f;  // this lane's own write above
    emit(usable && own && (uint32_t)score_key(s) >= tkey, s, row);
  }
#pragma unroll
  for (int h2 = 0; h2 < kDcHold; ++h2) {
    const int64_t row = heldg[h2] * R + slot;
    const bool own = heldg[h2] < ngroups && writer && row < n;
    if (usable) emit(own && (uint32_t)score_key(held[h2]) >= tkey, held[h2], row);
    else if (own) scratch[row] = held[h2];  // the fallback needs every score
  }
  auto process = [&](int64_t g) {
    const float s = dense_iter<CPL, R>(X4, n, g * R, wr, lane);
    const int64_t row = g * R + slot;
    const bool own = writer && row < n;
    if (usable) emit(own && (uint32_t)score_key(s) >= tkey, s, row);
    else if (own) scratch[row] = s;
  };
  // the first 3/4 of the groups interleaved as dense_score_fast (static) ...
  const int64_t gstat = (ngroups - ngroups / OTF_DC_TAIL_DIV) / nwarp * nwarp;
  for (; gcur < gstat; gcur = next_group(gcur + nwarp)) process(gcur);  // warp-uniform
  // ... the last 1/4 handed out one group at a time by 16 counters (warp % 16 serves the tail
  // groups congruent to it mod 16; each counter on its own 128-byte line; the next claim is
  // requested while the current group is scored): SMs that stream faster take more of it, so
  // every CTA reaches the barrier within about one group of the others (the static split left a
  // 130 us spread between CTAs on C2). Swept on B200: C2 1.177 -> 1.117 ms, C4 7.23 -> 6.87 ms,
  // C1 (fused) 101.5 -> 97 us; with the counters on ONE cache line, single-group claims
  // serialised on it (C4 7.76 ms) and 4-group claims were best (6.90 ms).
  {
    const int c = (int)(warp % OTF_DC_CTRS);
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(ws.cut_word + kDcCtrWord + kDcCtrStride * c);
    unsigned long long jn = 0;  // the next claim, requested one claim ahead (latency hidden)
    if (lane == 0) jn = atomicAdd(ctr, (unsigned long long)OTF_DC_CLAIM);
    for (;;) {
      const unsigned long long j0 = __shfl_sync(0xffffffffu, jn, 0);
      const int64_t g0 = gstat + OTF_DC_CTRS * (int64_t)j0 + c;
      if (g0 >= ngroups) break;
      if (lane == 0) jn = atomicAdd(ctr, (unsigned long long)OTF_DC_CLAIM);
#pragma unroll 1
      for (int u = 0; u < OTF_DC_CLAIM; ++u) {
        const int64_t g = g0 + OTF_DC_CTRS * u;
        if (g < ngroups && !is_sample(g)) process(g);
      }
    }
  }
  DC_STAMP(3);
  grid_barrier(ws.bar, G);  // every candidate record is in place
  DC_STAMP(4);

  // ---- 3. selection -------------------------------------------------------------------------------
  // the first kSelPre x 256 candidate keys are requested together with the count (one L2 round
  // trip instead of two; keys past the count are stale and ignored)
  constexpr int kSelPre = 8;
  uint32_t kpre[kSelPre];
#pragma unroll
  for (int u = 0; u < kSelPre; ++u) kpre[u] = __ldcg(key32 + threadIdx.x + u * kDcThreads);
  const unsigned long long c_all = __ldcg(cut_count);
  const bool ok = usable && c_all >= (unsigned long long)k_eff && c_all <= (unsigned long long)kDcSelCap;
  // the last CTA done with the counters clears them for the next query (on the fast path by the
  // last warp once the keys are in place, off the ranking's critical path)
  auto release_counters = [&]() {
    __threadfence();
    s_last = atomicAdd(ws.cut_word + 6, 1u) == G - 1;
    if (s_last) {
      ws.cut_word[0] = 0u; ws.cut_word[1] = 0u; ws.cut_word[6] = 0u;
      for (int q = 0; q < OTF_DC_CTRS; ++q) {  // the tail counters
        ws.cut_word[kDcCtrWord + kDcCtrStride * q] = 0u;
        ws.cut_word[kDcCtrWord + kDcCtrStride * q + 1] = 0u;
      }
    }
  };
  if (ok) {
    uint32_t* sk = reinterpret_cast<uint32_t*>(dyn);
    const int C = (int)c_all;
#pragma unroll
    for (int u = 0; u < kSelPre; ++u) {
      const int t = threadIdx.x + u * kDcThreads;
      if (t < C) sk[t] = kpre[u];
    }
#pragma unroll 4
    for (int t = threadIdx.x + kSelPre * kDcThreads; t < C; t += blockDim.x) sk[t] = __ldcg(key32 + t);
    __syncthreads();  // (every thread of the CTA has read the count)
    if (threadIdx.x == kDcThreads - 32) release_counters();
    DC_STAMP(5);
    const int nw = blockDim.x >> 5;
    for (int q = (int)vb + wid * (int)G; q < C; q += nw * (int)G) {
      const uint32_t ki = sk[q];
      // the candidate's record and row are in flight during the count (L2 round trips)
      const ulonglong2 ci = __ldcg(cut_rec + q);
      const int64_t ri = __ldcg(ws.cut_row + q);
      int cnt = 0;
      unsigned tie = 0;  // some lane saw another candidate with the same key
#pragma unroll 8
      for (int j = lane; j < C; j += 32) {
        const uint32_t kj = sk[j];
        cnt += kj > ki;
        tie |= kj == ki && j != q;
      }
      if (__any_sync(0xffffffffu, tie)) {  // exact key ties: (~id desc, row asc) decides
        for (int j = lane; j < C; j += 32) {
          if (sk[j] != ki || j == q) continue;
          const uint64_t ij = __ldcg(&cut_rec[j].y);
          cnt += ij > ci.y || (ij == ci.y && __ldcg(ws.cut_row + j) < ri);
        }
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      if (lane == 0 && cnt < k_eff) {
        out_ids[cnt] = id_of_inv(ci.y);
        out_scores[cnt] = (double)__uint_as_float((uint32_t)ci.x);
        if (out_rows) out_rows[cnt] = ri;
      }
    }
#ifdef OTF_DCUT_TRACE
    DC_STAMP(6);
    if (threadIdx.x == 0)
      printf("dcutT cta %d C %d sample %.2f barrier1 %.2f scan %.2f barrier2 %.2f select %.2f rank %.2f total %.2f\n",
             (int)vb, C, (ts[1] - ts[0]) * 1e-3, (ts[2] - ts[1]) * 1e-3, (ts[3] - ts[2]) * 1e-3, (ts[4] - ts[3]) * 1e-3,
             (ts[5] - ts[4]) * 1e-3, (ts[6] - ts[5]) * 1e-3, (ts[6] - ts[0]) * 1e-3);
#endif
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) release_counters();
  if (usable) {  // the candidates cannot be used: every remaining row's score (static, interleaved)
    for (int64_t g = warp; g < ngroups; g += nwarp) {
      if (is_sample(g)) continue;  // warp-uniform
      const float s = dense_iter<CPL, R>(X4, n, g * R, wr, lane);
      const int64_t row = g * R + slot;
      if (writer && row < n) scratch[row] = s;
    }
    grid_barrier(ws.bar, G);
  }
  // ---- fallback: the exact radix select over every row's score ---------------------------------------
  if (vb == 0 && threadIdx.x == 0) ws.cut_word[3] += 1u;  // fallbacks taken (diagnostics)
  DirectSrc<float> src{scratch};
  radix_select_emit(static_cast<const float*>(scratch), src, n, ids, id_base, k_eff, ws, k_eff >= n, dyn, out_ids,
                    out_scores, out_rows, h, &s_b, &s_above, vb, G);
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
                       int device, cudaStream_t st, uint16_t* cmax, int* clog, unsigned int* claim) {
  auto fn = dense_score_fast<CPL, R>;
  int grid = grid_for((const void*)fn, 256, device);
  const int64_t need = (n + (8 * R) - 1) / (8 * R);  // 8 warps per block
  if (need < grid) grid = (int)(need > 0 ? need : 1);
  if (R < 8) cmax = nullptr;  // chunks of >= 8 rows only (topk_cmax_ensure)
  fn<<<grid, 256, 0, st>>>(X, n, w, out, hist, cmax, claim);
  OTF_LAUNCH_CHECK("dense_score_fast");
  if (cmax && clog) *clog = R == 8 ? 3 : R == 16 ? 4 : 5;  // log2(R)
  return OTF_OK;
}

// ---- fused rank launch ---------------------------------------------------------------------------
namespace {
#ifndef OTF_DC_R1  // rows per warp iteration of the fused kernel at d = 128
#define OTF_DC_R1 16  // (measured: 16 rows 91.6 us per C1 query, 32 rows 96.8 us: finer tail granularity)
#endif
#ifndef OTF_DC_R16  // rows per warp iteration of the fused kernel at d = 2048
#define OTF_DC_R16 2
#endif
int dc_R(int cpl) { return cpl == 1 ? OTF_DC_R1 : cpl == 2 ? 4 : cpl == 4 ? 2 : cpl == 16 ? OTF_DC_R16 : 1; }

template <int CPL, int R>
int dc_grid(int device) {
  static int per_sm[64] = {0};
  if (!per_sm[device & 63]) {
    auto fn = dense_rank_cut<CPL, R>;
    if (cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDcSmem) != cudaSuccess)
      return 0;
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kDcThreads, kDcSmem) != cudaSuccess) return 0;
    per_sm[device & 63] = b;
  }
  return per_sm[device & 63] * rank_sms(device);
}

int dc_grid_of(int cpl, int device) {
  switch (cpl) {
    case 1: return dc_grid<1, OTF_DC_R1>(device);
    case 2: return dc_grid<2, 4>(device);
    case 4: return dc_grid<4, 2>(device);
    case 8: return dc_grid<8, 1>(device);
    case 16: return dc_grid<16, OTF_DC_R16>(device);
    case 32: return dc_grid<32, 1>(device);
    default: return 0;
  }
}

template <int CPL, int R>
int dc_launch(const float* X, int64_t n, const double* w, const int64_t* ids, int64_t id_base, int64_t k_eff,
              const DenseCutPlan& pl, TopkWs* ws, float* scratch, int64_t* out_ids, double* out_scores,
              int64_t* out_rows, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)pl.grid);
  cfg.blockDim = dim3(kDcThreads);
  cfg.dynamicSmemBytes = kDcSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OTF_CUDA(cudaLaunchKernelEx(&cfg, dense_rank_cut<CPL, R>, X, n, w, ids, id_base, k_eff, pl.r, pl.sit, *ws, scratch,
                              out_ids, out_scores, out_rows));
  OTF_LAUNCH_CHECK("dense_rank_cut");
  return OTF_OK;
}
}  // namespace

bool dense_cut_plan(int32_t d, const float* X, int64_t n, int64_t k_eff, int device, DenseCutPlan* pl) {
  static const bool off = getenv("OTF_DENSE_NO_CUT") != nullptr;  // A/B switch (tools/)
  if (off || k_eff <= 0 || d % 128 != 0 || (((uintptr_t)X) & 15) != 0) return false;
  const int cpl = d / 128;
  if (cpl != 1 && cpl != 2 && cpl != 4 && cpl != 8 && cpl != 16 && cpl != 32) return false;
  // ~want candidates are expected (below); their count must stay well inside the shared-memory cap
#ifndef OTF_CUT_WANT16  // expected candidates = k (OTF_CUT_WANT16 / 16) + 128
#define OTF_CUT_WANT16 25
#endif
  // ~k (1 + 4.5 / sqrt(64)) + 128 candidates expected: at r ~ 64 the count's relative spread is
  // ~1/8, so fewer than k (the exact fallback) is ~3.5 sigma away; the rounding of T down to its
  // 16-bit prefix adds margin. Measured: C3 62.5 (2 k + 128) -> 61.8 us, C1 / C2 unchanged;
  // 1.25 k + 128 was faster on C3 (59.9 us) but only ~2 sigma from a fallback.
  const int64_t want = k_eff * OTF_CUT_WANT16 / 16 + 128;
  if (2 * want > kDcSelCap || k_eff > kDcFallbackK) return false;
  const int grid = dc_grid_of(cpl, device);
  if (grid <= 0) return false;
  const int64_t nwarp = (int64_t)grid * (kDcThreads / 32), R = dc_R(cpl);
  if ((int64_t)kDcPub * grid > (int64_t)kDcPerThread * kDcThreads || kDcPub * grid > kCutSmaxCap) return false;
  // the sample: enough rows that the threshold is the ~64th-largest sampled key (relative spread
  // of the candidate count ~1/8), at least one group per warp, at most a quarter of the rows
  const int64_t s_target = (64 * n + want - 1) / want;
  const int64_t sit = std::max<int64_t>(1, (s_target + nwarp * R - 1) / (nwarp * R));
  const int64_t S = sit * nwarp * R;
  if (4 * S > n || sit > ((n + R - 1) / R) / nwarp) return false;
  const int64_t rr = (want * S + n - 1) / n;
  if (rr > grid) return false;  // the four published keys per CTA must cover the top r
  pl->grid = grid;
  pl->sit = (int)sit;
  pl->r = (int)std::max<int64_t>(rr, 1);
  return true;
}

int launch_dense_rank_cut(const float* X, int64_t n, int32_t d, const double* w, const int64_t* ids,
                          int64_t id_base, int64_t k_eff, const DenseCutPlan& pl, TopkWs* ws, float* scratch,
                          int64_t* out_ids, double* out_scores, int64_t* out_rows, cudaStream_t st) {
  switch (d / 128) {
    case 1: return dc_launch<1, OTF_DC_R1>(X, n, w, ids, id_base, k_eff, pl, ws, scratch, out_ids, out_scores, out_rows, st);
    case 2: return dc_launch<2, 4>(X, n, w, ids, id_base, k_eff, pl, ws, scratch, out_ids, out_scores, out_rows, st);
    case 4: return dc_launch<4, 2>(X, n, w, ids, id_base, k_eff, pl, ws, scratch, out_ids, out_scores, out_rows, st);
    case 8: return dc_launch<8, 1>(X, n, w, ids, id_base, k_eff, pl, ws, scratch, out_ids, out_scores, out_rows, st);
    case 16: return dc_launch<16, OTF_DC_R16>(X, n, w, ids, id_base, k_eff, pl, ws, scratch, out_ids, out_scores, out_rows, st);
    case 32: return dc_launch<32, 1>(X, n, w, ids, id_base, k_eff, pl, ws, scratch, out_ids, out_scores, out_rows, st);
    default: return fail(OTF_ERR_CONFIG, "dense_rank_cut: unsupported dimension");
  }
}

// Scores n rows against the float64 model w (cast to float32 in-kernel). Pointers must be
// 16-byte aligned for the fast path (all device buffers this library allocates are).
// hist (nullable): kHistBins counters (zero on entry) receiving the coarse score histogram.
int launch_dense_score(const float* X, int64_t n, int32_t d, const double* w, float* out,
                       uint32_t* hist, int device, cudaStream_t st, uint16_t* cmax, int* clog,
                       unsigned int* claim) {
  static const bool no_tail = getenv("OTF_DENSE_STATIC") != nullptr;  // A/B switch (tools/)
  if (no_tail) claim = nullptr;
  if (n <= 0) return OTF_OK;
  const bool aligned = (((uintptr_t)X) & 15) == 0;
  if (aligned && d % 128 == 0) {
    switch (d / 128) {
      case 1: return launch_fast<1, 32>(X, n, w, out, hist, device, st, cmax, clog, claim);  // R 8/16: 5% slower (C1)
      case 2: return launch_fast<2, 4>(X, n, w, out, hist, device, st, cmax, clog, claim);
      case 4: return launch_fast<4, 2>(X, n, w, out, hist, device, st, cmax, clog, claim);
      case 8: return launch_fast<8, 1>(X, n, w, out, hist, device, st, cmax, clog, claim);
      case 16: return launch_fast<16, 2>(X, n, w, out, hist, device, st, cmax, clog, claim);  // R 1 / 4: +0.6% / +2.8%
      case 32: return launch_fast<32, 1>(X, n, w, out, hist, device, st, cmax, clog, claim);
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
