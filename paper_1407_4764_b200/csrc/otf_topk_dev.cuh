// otf_topk_dev.cuh — device-side building blocks of the exact top-k selection (otf_topk.cu),
// shared with the fused PQ rank kernel (otf_pq.cu): grid barrier, order keys of ids, score
// sources, the histogram threshold search, rank-by-counting and the exact radix select.
// Semantics: top_k, ranker.py:97-143 (see otf_topk.cu).
#pragma once

#include "otf_common.cuh"
#include "otf_internal.h"

namespace otf {

static constexpr int kTopkThreads = 1024;
static constexpr int kTopkCtasPerSm = 1;
static constexpr int kCandCap = 8192;                       // candidates ranked in smem
static constexpr size_t kTopkSmem = (size_t)kCandCap * 16;  // key + inv per candidate

// Grid barrier on one 64-bit word {count (low half), generation (high half)}. An arrival is one
// atomic add of 1; the last arrival of a generation also adds (1 << 32) - nblocks (a reduction
// nobody waits for) to keep the count small. The barrier a word state has completed is its
// effective generation gen + count / nblocks, so waiters are released by the last ARRIVAL itself
// (round 2: one L2 round trip sooner than waiting for the generation bump), and arrivals that
// overtake a pending bump (count >= nblocks) count toward the next generation correctly.
#ifndef OTF_BAR_GEN_ONLY
__device__ __forceinline__ unsigned int bar_eff_gen(unsigned long long v, unsigned int nblocks) {
  return (unsigned int)(v >> 32) + (unsigned int)v / nblocks;
}
// arrive: returns the effective generation this arrival belongs to (released once the word's
// effective generation exceeds it)
__device__ __forceinline__ unsigned int bar_arrive_t0(unsigned int* bar, unsigned int nblocks, bool* last = nullptr) {
  unsigned long long* word = reinterpret_cast<unsigned long long*>(bar);
  __threadfence();
  const unsigned long long old = atomicAdd(word, 1ull);
  const bool l = (unsigned int)old % nblocks == nblocks - 1;
  if (l) atomicAdd(word, (1ull << 32) - nblocks);
  if (last) *last = l;
  return bar_eff_gen(old, nblocks);
}
__device__ __forceinline__ void bar_wait_t0(unsigned int* bar, unsigned int nblocks, unsigned int mine) {
  volatile unsigned long long* vw = reinterpret_cast<volatile unsigned long long*>(bar);
  while ((int)(bar_eff_gen(*vw, nblocks) - mine) <= 0) __nanosleep(20);  // (wrap-safe)
  __threadfence();
}
#else  // (A/B) waiters poll the generation bump
__device__ __forceinline__ unsigned int bar_arrive_t0(unsigned int* bar, unsigned int nblocks, bool* last = nullptr) {
  unsigned long long* word = reinterpret_cast<unsigned long long*>(bar);
  __threadfence();
  const unsigned long long old = atomicAdd(word, 1ull);
  const bool l = (unsigned int)old == nblocks - 1;
  if (l) atomicAdd(word, (1ull << 32) - nblocks);
  if (last) *last = l;
  return (unsigned int)(old >> 32);
}
__device__ __forceinline__ void bar_wait_t0(unsigned int* bar, unsigned int, unsigned int gen) {
  volatile unsigned int* vgen = bar + 1;
  while (*vgen == gen) __nanosleep(20);
  __threadfence();
}
#endif

__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    bool last;
    const unsigned int mine = bar_arrive_t0(bar, nblocks, &last);
    if (!last) bar_wait_t0(bar, nblocks, mine);  // (the last arrival has nothing to wait for)
    else __threadfence();
  }
  __syncthreads();
}

// Split grid barrier (same word as grid_barrier): arrive, do independent work, then wait.
// grid_arrive returns the token to wait on (every thread of the CTA gets it).
__device__ __forceinline__ unsigned int grid_arrive(unsigned int* bar, unsigned int nblocks, unsigned int* s_gen) {
  __syncthreads();
  if (threadIdx.x == 0) *s_gen = bar_arrive_t0(bar, nblocks);
  __syncthreads();
  return *s_gen;
}
__device__ __forceinline__ void grid_wait(unsigned int* bar, unsigned int nblocks, unsigned int token) {
  __syncthreads();
  if (threadIdx.x == 0) bar_wait_t0(bar, nblocks, token);
  __syncthreads();
}

__device__ __forceinline__ int64_t id_of(const int64_t* ids, int64_t id_base, int64_t row) {
  return ids ? ids[row] : id_base + row;
}

// Tie key of an id: larger inv <=> smaller (signed) id. Flipping the sign bit maps the signed
// order onto the unsigned one, so negative ids (accepted by the reference) rank before positive
// ones exactly as np.lexsort orders them.
__device__ __forceinline__ uint64_t inv_id(int64_t id) { return ~((uint64_t)id ^ 0x8000000000000000ull); }
__device__ __forceinline__ int64_t id_of_inv(uint64_t inv) { return (int64_t)(~inv ^ 0x8000000000000000ull); }

__device__ __forceinline__ bool cand_greater(uint64_t ka, uint64_t ia, uint64_t kb, uint64_t ib) {
  return ka > kb || (ka == kb && ia > ib);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Inverse of score_key(double) (exact: the key is a bijection except -0.0 -> +0.0).
__device__ __forceinline__ double key_to_f64(uint64_t k) {
  const uint64_t u = (k >> 63) ? (k ^ 0x8000000000000000ull) : ~k;
  return __longlong_as_double((long long)u);
}

// top two of a warp's (a >= b) pairs: returns (m1, m2) on every lane
__device__ __forceinline__ void warp_top2(uint32_t a, uint32_t b, uint32_t& m1, uint32_t& m2) {
  m1 = __reduce_max_sync(0xffffffffu, a);
  const unsigned hit = __ballot_sync(0xffffffffu, a == m1);
  const int first = __ffs(hit) - 1;
  const uint32_t rest = ((int)(threadIdx.x & 31) == first) ? b : a;
  m2 = __reduce_max_sync(0xffffffffu, rest);
}

// ---- score sources ---------------------------------------------------------------------------
template <typename ST>
struct DirectSrc {
  using T = ST;
  static constexpr int kLoadBytes = sizeof(ST);
  static constexpr int kBins = kHistBins;
  const ST* s;
  __device__ __forceinline__ void shift(int64_t o) { s += o; }
  __device__ __forceinline__ ST load(int64_t i) const { return __ldcg(s + i); }
  // 8 consecutive entries from i (i % 8 == 0): two float4 / four double2 loads, or scalar loads
  // when the array does not start on 16 bytes (segments at c * n entries with n % 4 != 0, or a
  // caller's unaligned score array)
  __device__ __forceinline__ void load8(int64_t i, ST (&v)[8]) const {
    if ((reinterpret_cast<uintptr_t>(s) & 15) != 0) {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = __ldcg(s + i + q);
      return;
    }
    if constexpr (sizeof(ST) == 4) {
      const float4 a = __ldcg(reinterpret_cast<const float4*>(s + i));
      const float4 b = __ldcg(reinterpret_cast<const float4*>(s + i) + 1);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 a = __ldcg(reinterpret_cast<const double2*>(s + i) + q);
        v[2 * q] = a.x; v[2 * q + 1] = a.y;
      }
    }
  }
  __device__ __forceinline__ uint32_t bin_of(ST v) const { return hist_bin(v); }
  __device__ __forceinline__ ST exact(int64_t, ST v) const { return v; }
  __device__ __forceinline__ double out_score(int64_t row, uint64_t) const {
    return (double)__ldcg(s + row);  // keeps a caller's -0.0 bit pattern
  }
  __device__ __forceinline__ void prefetch_chunk(int64_t, int, int64_t, int) const {}
};

struct PqBinSrc {
  using T = double;
  static constexpr int kLoadBytes = 2;
  static constexpr int kBins = kPqHistBins;  // bins written by pq_scan16_f32bins
  const uint16_t* bins; const uint8_t* codes; const double* lut; int M, K;
  __device__ __forceinline__ void shift(int64_t) {}  // one segment only
  __device__ __forceinline__ uint32_t load(int64_t i) const { return __ldcg(bins + i); }
  __device__ __forceinline__ void load8(int64_t i, uint32_t (&v)[8]) const {
    const uint4 a = __ldcg(reinterpret_cast<const uint4*>(bins + i));
    const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) { v[2 * q] = w[q] & 0xffffu; v[2 * q + 1] = w[q] >> 16; }
  }
  __device__ __forceinline__ uint32_t bin_of(uint32_t v) const { return v; }
  // M == 16 (the only bins-path shape): one 16-byte code load, 16 independent LUT loads, then
  // numpy's pairwise tree (r_j = a_j + a_{j+8}, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))).
  __device__ __forceinline__ double exact(int64_t i, uint32_t) const {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(codes + i * 16));
    const uint32_t wd[4] = {u.x, u.y, u.z, u.w};
    double a[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) a[m] = __ldg(lut + m * K + ((wd[m >> 2] >> (8 * (m & 3))) & 0xffu));
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(a[j], a[j + 8]);
    return __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                     __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  }
  __device__ __forceinline__ double out_score(int64_t, uint64_t key) const { return key_to_f64(key); }
  // the codes of a hit chunk (16 B per row) are pulled into L2 while its bins are read, so
  // exact() of its candidates does not wait on a second HBM round trip
  __device__ __forceinline__ void prefetch_chunk(int64_t r0, int CH, int64_t n, int lane) const {
    if (8 * lane < CH && r0 + 8 * lane < n)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(codes + (r0 + 8 * lane) * 16));
  }
};

// PQ cut path source (pq_scan16_cut): the candidates arrive as (exact key, row) pairs; the
// exact score of an arbitrary row (fallback) is recomputed from codes + LUT as in PqBinSrc.
struct PqCutSrc {
  using T = double;
  static constexpr int kLoadBytes = 2;  // no score array: phase D materialises exact scores
  static constexpr int kBins = kPqHistBins;
  PqBinSrc pq;
  __device__ __forceinline__ void shift(int64_t) {}
  __device__ __forceinline__ uint32_t load(int64_t) const { return 0u; }
  __device__ __forceinline__ double exact(int64_t i, uint32_t v) const { return pq.exact(i, v); }
  __device__ __forceinline__ double out_score(int64_t, uint64_t key) const { return key_to_f64(key); }
};

// Workspace of segment `seg`: per segment one block of kWsWords counters (histogram, radix
// histograms, barrier, count) and `cap` candidate slots.
constexpr int64_t kWsWords = kHistBinsMax + 3 * 256 + 4;
__device__ __forceinline__ TopkWs seg_ws(TopkWs ws, unsigned seg) {
  ws.hist += (int64_t)seg * kWsWords;
  ws.rhist = ws.hist + kHistBinsMax;
  ws.bar = reinterpret_cast<unsigned int*>(ws.rhist + 3 * 256);
  ws.count = ws.bar + 2;
  ws.key += (int64_t)seg * ws.cap;
  ws.inv += (int64_t)seg * ws.cap;
  ws.row += (int64_t)seg * ws.cap;
  return ws;
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

// Block-wide: bins scanned from NB-1 down; finds the bin where the running count reaches
// `need`. Thread t owns the kBPT contiguous bins NB-kBPT*(t+1) .. NB-1-kBPT*t, read straight from
// the global histogram into registers (16-byte loads; one L2 round trip, no shared staging).
template <int NB, int NT = kTopkThreads, bool SMEM = false>  // SMEM: gh is a shared-memory histogram
__device__ void find_bin(const uint32_t* gh, int64_t need, int* out_b, int64_t* out_above,
                         int64_t* out_cnt, int64_t* wsum) {
  constexpr int kBPT = NB / NT;  // blockDim.x must be NT
  static_assert(kBPT % 4 == 0, "16-byte histogram loads");
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int base = NB - kBPT * (t + 1);
  uint32_t v[kBPT];
#pragma unroll
  for (int u = 0; u < kBPT / 4; ++u) {
    const uint4 q = SMEM ? reinterpret_cast<const uint4*>(gh + base)[u] : __ldcg(reinterpret_cast<const uint4*>(gh + base) + u);
    v[4 * u] = q.x; v[4 * u + 1] = q.y; v[4 * u + 2] = q.z; v[4 * u + 3] = q.w;
  }
  int64_t local = 0;
#pragma unroll
  for (int q = 0; q < kBPT; ++q) local += v[q];
  int64_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int64_t u = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
    int64_t s = u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t w = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += w;
    }
    wsum[lane] = s - u;  // exclusive prefix of warp sums
  }
  __syncthreads();
  incl += wsum[wid];
  const int64_t excl = incl - local;
  if (excl < need && incl >= need) {
    int64_t cum = excl;
#pragma unroll
    for (int q = kBPT - 1; q >= 0; --q) {
      if (cum >= 0 && cum + v[q] >= need) {
        *out_b = base + q;
        *out_above = cum;
        *out_cnt = v[q];
        cum = -1;  // found (keeps the loop unrolled: v stays in registers)
      } else if (cum >= 0) {
        cum += v[q];
      }
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
template <typename Src>
__device__ void rank_emit(const Src& src, const TopkWs& ws, int64_t m, int64_t k_eff,
                          unsigned char* dyn, int64_t* out_ids, double* out_scores,
                          int64_t* out_rows, unsigned vb, unsigned vnb) {
  const int64_t mine = m > vb ? (m - 1 - vb) / vnb + 1 : 0;
  if (mine == 0) return;
  ulonglong2* sc = reinterpret_cast<ulonglong2*>(dyn);  // (key, inv) pairs: one 16-byte load each
  for (int64_t t = threadIdx.x; t < m; t += blockDim.x)
    sc[t] = make_ulonglong2(__ldcg(ws.key + t), __ldcg(ws.inv + t));
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t q = wid; q < mine; q += nw) {
    const int64_t i = vb + q * vnb;
    const ulonglong2 ci = sc[i];
    const uint64_t ki = ci.x, ii = ci.y;
    const int64_t r = lane == 0 ? __ldcg(ws.row + i) : 0;  // in flight during the count
    int cnt = 0;
    const int mm = (int)m;  // m <= kCandCap
#pragma unroll 4
    for (int j = lane; j < mm; j += 32) {
      const ulonglong2 cj = sc[j];
      cnt += cand_greater(cj.x, cj.y, ki, ii);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0 && cnt < k_eff) {
      out_ids[cnt] = id_of_inv(ii);
      out_scores[cnt] = src.out_score(r, ki);
      if (out_rows) out_rows[cnt] = r;
    }
  }
}

// rank_emit for candidates whose keys fit in 32 bits (float32 scores): the count runs over 4-byte
// keys in shared memory (one wavefront per 32 comparisons instead of four for the 16-byte
// (key, inv) pairs); exact key ties — rare — are resolved by (~id desc, row asc) from global
// memory, so equal (key, id) pairs still get distinct ranks. Round 2 (topk_seg_cut_kernel: the
// 64 x ~2.1k-candidate rankings took ~285 us of its 0.74 ms with rank_emit).
template <typename Src>
__device__ void rank_emit_k32(const Src& src, const TopkWs& ws, int64_t m, int64_t k_eff, unsigned char* dyn,
                              int64_t* out_ids, double* out_scores, int64_t* out_rows, unsigned vb, unsigned vnb) {
  const int64_t mine = m > vb ? (m - 1 - vb) / vnb + 1 : 0;
  if (mine == 0) return;
  uint32_t* sk = reinterpret_cast<uint32_t*>(dyn);
  for (int64_t t = threadIdx.x; t < m; t += blockDim.x) sk[t] = (uint32_t)__ldcg(ws.key + t);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int mm = (int)m;  // m <= kCandCap
  for (int64_t q = wid; q < mine; q += nw) {
    const int i = (int)(vb + q * vnb);
    const uint32_t ki = sk[i];
    const uint64_t ii = __ldcg(ws.inv + i);  // (in flight during the count)
    const int64_t r = __ldcg(ws.row + i);
    int cnt = 0;
    unsigned tie = 0;
#pragma unroll 8
    for (int j = lane; j < mm; j += 32) {
      const uint32_t kj = sk[j];
      cnt += kj > ki;
      tie |= kj == ki && j != i;
    }
    if (__any_sync(0xffffffffu, tie)) {
      for (int j = lane; j < mm; j += 32) {
        if (sk[j] != ki || j == i) continue;
        const uint64_t ij = __ldcg(ws.inv + j);
        cnt += ij > ii || (ij == ii && __ldcg(ws.row + j) < r);
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0 && cnt < k_eff) {
      out_ids[cnt] = id_of_inv(ii);
      out_scores[cnt] = src.out_score(r, (uint64_t)ki);
      if (out_rows) out_rows[cnt] = r;
    }
  }
}

// Sources whose order keys fit in 32 bits (float32 scores): ranked with rank_emit_k32.
template <typename Src> struct Key32 { static constexpr bool value = false; };
template <> struct Key32<DirectSrc<float>> { static constexpr bool value = true; };
template <typename Src>
__device__ __forceinline__ void rank_emit_any(const Src& src, const TopkWs& ws, int64_t m, int64_t k_eff,
                                              unsigned char* dyn, int64_t* out_ids, double* out_scores,
                                              int64_t* out_rows, unsigned vb, unsigned vnb) {
  if constexpr (Key32<Src>::value) rank_emit_k32(src, ws, m, k_eff, dyn, out_ids, out_scores, out_rows, vb, vnb);
  else rank_emit(src, ws, m, k_eff, dyn, out_ids, out_scores, out_rows, vb, vnb);
}

// Phase D over a materialised score array (see header). Returns after writing the output.
template <typename ST, typename Src>
__device__ void radix_select_emit(const ST* scores, const Src& src, int64_t n, const int64_t* ids,
                                  int64_t id_base, int64_t k_eff, const TopkWs& ws, bool all,
                                  unsigned char* dyn, int64_t* out_ids, double* out_scores,
                                  int64_t* out_rows, uint32_t* h, int* s_b, int64_t* s_above, unsigned vb,
                                  unsigned vnb) {
  constexpr int KB = KeyBits<ST>::value;
  const unsigned int nb = vnb;
  const int lane = threadIdx.x & 31;
  const int64_t tid = (int64_t)vb * blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)vnb * blockDim.x;
  const int64_t wbase0 = (int64_t)vb * blockDim.x + (threadIdx.x & ~31);
  uint64_t pre = 0, msk = 0, pre2 = 0, msk2 = 0;
  int64_t need = k_eff;
  int phase = all ? 2 : 0;  // k_eff == n: everything is gathered (mask 0)
  bool tie = false;
  int shift = KB - 8;
  int it = 0;
  while (phase < 2) {
    uint32_t* H = ws.rhist + (it % 3) * 256;
    if (vb == 0 && threadIdx.x < 256) ws.rhist[((it + 1) % 3) * 256 + threadIdx.x] = 0u;
    if (threadIdx.x < 256) h[threadIdx.x] = 0u;
    __syncthreads();
    if (phase == 0) {
      for (int64_t i = tid; i < n; i += nthreads) {
        const uint64_t key = score_key(__ldcg(scores + i));
        if ((key & msk) == pre) atomicAdd(&h[(key >> shift) & 255u], 1u);
      }
    } else {
      for (int64_t i = tid; i < n; i += nthreads) {
        const uint64_t key = score_key(__ldcg(scores + i));
        if (key == pre) {
          const uint64_t inv = inv_id(id_of(ids, id_base, i));
          if ((inv & msk2) == pre2) atomicAdd(&h[(inv >> shift) & 255u], 1u);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x < 256 && h[threadIdx.x]) atomicAdd(&H[threadIdx.x], h[threadIdx.x]);
    grid_barrier(ws.bar, nb);
    if (threadIdx.x < 256) h[threadIdx.x] = __ldcg(H + threadIdx.x);
    __syncthreads();
    pick_bin256(h, need, s_b, s_above);
    __syncthreads();
    const int b = *s_b;
    need -= *s_above;
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
      key = score_key(__ldcg(scores + i));
      const uint64_t mk = key & msk;
      inv = inv_id(id_of(ids, id_base, i));
      in = mk > pre || (mk == pre && (!tie || (inv & msk2) >= pre2));
    }
    append_candidate(ws, in, key, inv, i, k_eff);
  }
  grid_barrier(ws.bar, nb);
  if (vb == 0) {
    for (int t = threadIdx.x; t < 3 * 256; t += blockDim.x) ws.rhist[t] = 0u;
    for (int b = threadIdx.x; b < kHistBinsMax; b += blockDim.x) ws.hist[b] = 0u;
  }
  if (k_eff <= kCandCap) {
    if (vb == 0 && threadIdx.x == 0) *ws.count = 0u;
    rank_emit_any(src, ws, k_eff, k_eff, dyn, out_ids, out_scores, out_rows, vb, vnb);
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
    out_ids[t] = id_of_inv(__ldcg(ws.inv + t));
    out_scores[t] = src.out_score(r, __ldcg(ws.key + t));
    if (out_rows) out_rows[t] = r;
  }
  if (tid == 0) *ws.count = 0u;
}


}  // namespace otf
