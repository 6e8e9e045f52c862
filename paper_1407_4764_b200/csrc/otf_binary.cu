// otf_binary.cu — K4 binary-code scoring (score_binary, ranker.py:78-94), unpack_bits
// (binary.py:110-120), binarize (binary.py:86-107) and Hamming distance (binary.py:123-128).
//
// Scoring: s_i = float32( sum_{j < n_bits, bit j set} float32(w_j) ), bit j = byte j/8,
// bit j%8 (LSB first); padding bits are ignored (the reference unpacks with
// count=output_bits). Instead of unpacking 2048 bits to floats (the reference's 32x
// expansion) each code byte indexes a 256-entry table of the summed weights of its set bits
// (bin_score_bytes below: one conflict-free 4-byte shared-memory lookup per code byte). The
// per-row sum uses a fixed lane tree (as in otf_dense.cu), so a row's score does not depend
// on its position. Parity with the reference's float32 sgemv is a tolerance.
//
// HBM roofline: n_bits/8 bytes per row (256 B for 2048-bit codes).
#include <cstdlib>
#include <cstring>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "otf_common.cuh"
#include "otf_internal.h"

namespace otf {

// Byte-table fast path (rows of RB bytes, RB % 128 == 0, e.g. 2048-bit codes = 256 B).
// A pass covers one 128-byte slice of every row: lane l reads the 4-byte word at slice offset
// 4l (one coalesced 128 B load per row per warp) and looks up each byte b_k (k = 0..3) in a
// float32 table T_{l,k}[v] = float32(sum of the float32 weights of the set bits of v)
// (summed in float64, bit order). Table entry (k, v, l) sits at byte address
//   (k >> 1) << 16 | v << 8 | (k & 1) << 7 | l << 2
// so every lane reads its own bank (conflict-free) and the whole address is ONE byte_perm of
// the code word with a per-lane constant (no shift/mask arithmetic per lookup). The 4 lane
// values are summed in float32 and the 32 lane partials of a row are reduced with the
// transposed float32 butterfly (32 rows per warp iteration, ~4 instructions per row). Slices
// are chained through a float64 partial per row (8 B/row per extra slice, +3% traffic for
// 2048-bit codes). Every row is summed in the same fixed order (position independent).
//
// WIDE (round 2, the default): the same lookups and the same sums, loaded 16 bytes at a time.
// Lane l = 8 b + a reads bytes [16 a, 16 a + 16) of a slice of row 4 g + b (g = 0..7: one
// LDG.128 per 4 rows instead of one LDG.32 per row), i.e. the words of "virtual lanes"
// v = 4 a + q, q = 0..3. At step j it looks up word q = (j + b) & 3 (the 32 lanes then read 32
// distinct virtual lanes = 32 banks: conflict-free). The transposed float32 reduction runs over
// the 8 lanes of a row (xor 4, 2, 1 = virtual-lane bits 4, 3, 2) and ends with
// (S0 + S2) + (S1 + S3) in-lane (bits 1, 0): the xor tree of the 32 virtual lanes, so every row's
// score is the same bits as the narrow kernel's. LSU instructions per 32 rows and lane:
// 8 + 128 + 28 (+2) instead of 32 + 128 + 31 (+2).
constexpr int kBinThreads = 512;
__device__ __forceinline__ uint32_t bin_sel(int c, uint32_t a, uint32_t b) { return c ? a : b; }

template <int RB, bool WIDE = true>  // row bytes (compile-time so per-row offsets are immediates)
__global__ void __launch_bounds__(kBinThreads, 1)
bin_score_bytes(const uint8_t* __restrict__ codes, int64_t n, int slice,
                const double* __restrict__ w, int n_bits, const double* __restrict__ partial_in,
                double* __restrict__ partial_out, float* __restrict__ out,
                uint32_t* __restrict__ ghist, const __grid_constant__ CUtensorMap map, int use_pf,
                uint16_t* __restrict__ cmax) {
  extern __shared__ __align__(16) unsigned char tabb[];  // 128 KB
  __shared__ uint32_t sh[kHistBins];
  for (int e = threadIdx.x; e < 4 * 256 * 32; e += blockDim.x) {
    const int l = e & 31, k = (e >> 5) & 3, v = e >> 7;  // consecutive threads -> consecutive banks
    const int bit0 = 8 * (slice * 128 + 4 * l + k);
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < 8; ++b)
      if ((v >> b) & 1) s = __dadd_rn(s, bit0 + b < n_bits ? (double)__double2float_rn(w[bit0 + b]) : 0.0);
    const uint32_t addr = ((uint32_t)(k >> 1) << 16) | ((uint32_t)v << 8) | ((uint32_t)(k & 1) << 7) | ((uint32_t)l << 2);
    *reinterpret_cast<float*>(tabb + addr) = __double2float_rn(s);
  }
  if (ghist && out) hist_zero(sh);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // per-lane constant bytes: [l<<2, l<<2 | 0x80, 0, 1]
  const uint32_t L = ((uint32_t)lane << 2) | (((uint32_t)lane << 2 | 0x80u) << 8) | (1u << 24);
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int R = 32;  // rows per warp iteration
  if (WIDE) {
    const int a = lane & 7, b = lane >> 3;
    uint32_t Lj[4];  // per-step constants: virtual lane 4 a + ((j + b) & 3)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t lv = 4u * a + ((j + b) & 3);
      Lj[j] = (lv << 2) | ((lv << 2 | 0x80u) << 8) | (1u << 24);
    }
    const uint8_t* base16 = codes + (int64_t)slice * 128 + 16 * a;
    const int slot = 4 * a + b;  // the row this lane finishes (transposed over g: g = a)
    for (int64_t r0 = warp * R; r0 < n; r0 += nwarp * R) {
      if (use_pf && lane == 0) {
        const int64_t nr = r0 + use_pf * nwarp * R;
        if (nr < n)
          asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(&map), "r"(slice * 128),
                       "r"((int)nr)
                       : "memory");
      }
      uint4 u[8];
      const uint8_t* rp = base16 + (r0 + b) * RB;
      if (r0 + R <= n) {
#pragma unroll
        for (int g = 0; g < 8; ++g) u[g] = __ldcs(reinterpret_cast<const uint4*>(rp + 4 * g * RB));
      } else {
#pragma unroll
        for (int g = 0; g < 8; ++g)
          u[g] = r0 + 4 * g + b < n ? __ldcs(reinterpret_cast<const uint4*>(rp + 4 * g * RB)) : make_uint4(0, 0, 0, 0);
      }
      const int64_t row = r0 + slot;
      const bool active = row < n;
      const double pin = active && partial_in ? __ldcs(partial_in + row) : 0.0;
      float p[R];  // p[4 g + j]
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        // word (j + b) & 3 at step j: rotate the four words by b
        const uint32_t t0 = bin_sel(b & 1, u[g].y, u[g].x), t1 = bin_sel(b & 1, u[g].z, u[g].y);
        const uint32_t t2 = bin_sel(b & 1, u[g].w, u[g].z), t3 = bin_sel(b & 1, u[g].x, u[g].w);
        const uint32_t r[4] = {bin_sel(b & 2, t2, t0), bin_sel(b & 2, t3, t1), bin_sel(b & 2, t0, t2),
                               bin_sel(b & 2, t1, t3)};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t x = r[j], L = Lj[j];
          float s = *reinterpret_cast<const float*>(tabb + __byte_perm(x, L, 0x6604));
          s = __fadd_rn(s, *reinterpret_cast<const float*>(tabb + __byte_perm(x, L, 0x6615)));
          s = __fadd_rn(s, *reinterpret_cast<const float*>(tabb + __byte_perm(x, L, 0x6724)));
          s = __fadd_rn(s, *reinterpret_cast<const float*>(tabb + __byte_perm(x, L, 0x6735)));
          p[4 * g + j] = s;
        }
      }
      transposed_reduce_f<R, 8>(p, lane);  // -> p[0..3]: row group g = a, steps j = 0..3
      double total = (double)__fadd_rn(__fadd_rn(p[0], p[2]), __fadd_rn(p[1], p[3]));
      if (active && partial_in) total = __dadd_rn(pin, total);
      if (out) {
        const float sc = __double2float_rn(total);
        if (active) out[row] = sc;
        if (ghist) hist_add(sh, active, hist_bin(sc));
        if (cmax) {
          const uint32_t wm = __reduce_max_sync(0xffffffffu, active ? hist_bin(sc) : 0u);
          if (lane == 0) cmax[r0 / R] = (uint16_t)wm;
        }
      } else if (active) {
        partial_out[row] = total;
      }
    }
    if (ghist && out) {
      __syncthreads();
      hist_flush(sh, ghist);
    }
    return;
  }
  const uint8_t* base = codes + (int64_t)slice * 128 + 4 * lane;
  bool writer;
  const int slot = row_of_lane<R, 32>(lane, &writer);  // the row this lane finishes
  for (int64_t r0 = warp * R; r0 < n; r0 += nwarp * R) {
    // the warp's next R rows of THIS slice go to L2 now (one 2-D bulk prefetch: 128 B x R rows,
    // row stride RB), so the next iteration's loads wait on L2 rather than HBM latency
    if (use_pf && lane == 0) {
      const int64_t nr = r0 + use_pf * nwarp * R;  // use_pf = prefetch distance in iterations
      if (nr < n)
        asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(&map), "r"(slice * 128),
                     "r"((int)nr)
                     : "memory");
    }
    uint32_t wd[R];
    const uint8_t* rp = base + r0 * RB;
    if (r0 + R <= n) {
#pragma unroll
      for (int i = 0; i < R; ++i) wd[i] = __ldcs(reinterpret_cast<const uint32_t*>(rp + i * RB));
    } else {
#pragma unroll
      for (int i = 0; i < R; ++i)
        wd[i] = r0 + i < n ? __ldcs(reinterpret_cast<const uint32_t*>(rp + i * RB)) : 0u;
    }
    const int64_t row = r0 + slot;
    const bool active = writer && row < n;
    // the previous slice's partial is loaded with the codes (its latency was exposed at the end)
    const double pin = active && partial_in ? __ldcs(partial_in + row) : 0.0;
    float p[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const uint32_t x = wd[i];
      float s = *reinterpret_cast<const float*>(tabb + __byte_perm(x, L, 0x6604));
      s = __fadd_rn(s, *reinterpret_cast<const float*>(tabb + __byte_perm(x, L, 0x6615)));
      s = __fadd_rn(s, *reinterpret_cast<const float*>(tabb + __byte_perm(x, L, 0x6724)));
      s = __fadd_rn(s, *reinterpret_cast<const float*>(tabb + __byte_perm(x, L, 0x6735)));
      p[i] = s;
    }
    transposed_reduce_f<R, 32>(p, lane);
    double total = (double)p[0];
    if (active && partial_in) total = __dadd_rn(pin, total);
    if (out) {
      const float sc = __double2float_rn(total);
      if (active) out[row] = sc;
      if (ghist) hist_add(sh, active, hist_bin(sc));
      if (cmax) {  // the warp's R consecutive rows are one top-k chunk
        const uint32_t wm = __reduce_max_sync(0xffffffffu, active ? hist_bin(sc) : 0u);
        if (lane == 0) cmax[r0 / R] = (uint16_t)wm;
      }
    } else if (active) {
      partial_out[row] = total;
    }
  }
  if (ghist && out) {
    __syncthreads();
    hist_flush(sh, ghist);
  }
}

// Multi-slice rows (2048-8192 bits) in ONE launch: a cluster of S = RB / 128 CTAs, one slice per
// CTA (each holds its slice's 128 KB byte table), all S CTAs on the same rows. Warp w of CTA s
// scores its slice of 32 rows exactly as bin_score_bytes does; the float32 slice sums then meet
// over distributed shared memory instead of a float64 partial round trip through HBM (-8 B
// written and read per row and slice): iteration i's rows are finished by CTA i mod S (the
// finishing work — score store, histogram, chunk maxima — rotates over the cluster so no SM does
// more than its share); the other CTAs send their sums with one st.async per lane into its
// receive ring, completing on that warp's transaction-count mbarrier. The finishing CTA adds them
// in slice order in float64 — the chain of the per-slice launches, (((double)p0 + (double)p1) +
// (double)p2) ..., so scores are bit-identical — and a ring slot is reused only after it released
// it (a remote arrive on the sender's `empty` barrier).
constexpr int kBinRing = 4;
constexpr int kBinWarps = kBinThreads / 32;
constexpr int kBinMaxS = 8;

__device__ __forceinline__ uint32_t bin_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t bin_mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// (default .acquire.cta: the slice sums land by st.async with complete_tx, like TMA writes)
__device__ __forceinline__ void bin_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.b32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"(bar), "r"(parity)
                 : "memory");
}

template <int RB>
__global__ void __launch_bounds__(kBinThreads, 1)
bin_score_cluster(const uint8_t* __restrict__ codes, int64_t n, const double* __restrict__ w, int n_bits,
                  float* __restrict__ out, uint32_t* __restrict__ ghist, const __grid_constant__ CUtensorMap map,
                  int use_pf, uint16_t* __restrict__ cmax) {
  constexpr int S = RB / 128;
  static_assert(S >= 2 && S <= kBinMaxS, "2..8 slices");
  extern __shared__ __align__(16) unsigned char tabb[];  // 128 KB table, then the receive ring
  float* recv = reinterpret_cast<float*>(tabb + 131072);  // [kBinRing][S - 1][kBinWarps][32]
  __shared__ uint32_t sh[kHistBins];
  __shared__ __align__(8) uint64_t full[kBinRing][kBinWarps];       // my ring slot (b, warp) landed
  __shared__ __align__(8) uint64_t empty[S][kBinRing][kBinWarps];   // CTA o read my sums in its slot (b, warp)
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int slice = (int)rank;
  for (int e = threadIdx.x; e < 4 * 256 * 32; e += blockDim.x) {
    const int l = e & 31, k = (e >> 5) & 3, v = e >> 7;
    const int bit0 = 8 * (slice * 128 + 4 * l + k);
    double sum = 0.0;
#pragma unroll
    for (int b = 0; b < 8; ++b)
      if ((v >> b) & 1) sum = __dadd_rn(sum, bit0 + b < n_bits ? (double)__double2float_rn(w[bit0 + b]) : 0.0);
    const uint32_t addr = ((uint32_t)(k >> 1) << 16) | ((uint32_t)v << 8) | ((uint32_t)(k & 1) << 7) | ((uint32_t)l << 2);
    *reinterpret_cast<float*>(tabb + addr) = __double2float_rn(sum);
  }
  for (int t = threadIdx.x; t < kBinRing * kBinWarps * (S + 1); t += blockDim.x) {
    uint64_t* bar = t < kBinRing * kBinWarps ? &full[0][0] + t : &empty[0][0][0] + (t - kBinRing * kBinWarps);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bin_smem_u32(bar)));
  }
  if (ghist) hist_zero(sh);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  // every CTA's tables and barriers exist before any remote access
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const uint32_t L = ((uint32_t)lane << 2) | (((uint32_t)lane << 2 | 0x80u) << 8) | (1u << 24);
  const int64_t cid = blockIdx.x / S, ncl = gridDim.x / S;
  const uint8_t* base = codes + (int64_t)slice * 128 + 4 * lane;
  constexpr int R = 32;
  bool writer;
  const int slot = row_of_lane<R, 32>(lane, &writer);
  const int64_t step = ncl * kBinWarps * R;
  int it = 0;
  for (int64_t r0 = (cid * kBinWarps + wi) * R; r0 < n; r0 += step, ++it) {
    if (use_pf && lane == 0) {
      const int64_t nr = r0 + use_pf * step;
      if (nr < n)
        asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(&map), "r"(slice * 128),
                     "r"((int)nr)
                     : "memory");
    }
    uint32_t wd[R];
    const uint8_t* rp = base + r0 * RB;
    if (r0 + R <= n) {
#pragma unroll
      for (int i = 0; i < R; ++i) wd[i] = __ldcs(reinterpret_cast<const uint32_t*>(rp + i * RB));
    } else {
#pragma unroll
      for (int i = 0; i < R; ++i) wd[i] = r0 + i < n ? __ldcs(reinterpret_cast<const uint32_t*>(rp + i * RB)) : 0u;
    }
    float p[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const uint32_t x = wd[i];
      float v = *reinterpret_cast<const float*>(tabb + __byte_perm(x, L, 0x6604));
      v = __fadd_rn(v, *reinterpret_cast<const float*>(tabb + __byte_perm(x, L, 0x6615)));
      v = __fadd_rn(v, *reinterpret_cast<const float*>(tabb + __byte_perm(x, L, 0x6724)));
      v = __fadd_rn(v, *reinterpret_cast<const float*>(tabb + __byte_perm(x, L, 0x6735)));
      p[i] = v;
    }
    transposed_reduce_f<R, 32>(p, lane);
    const int o = it % S;  // the CTA that finishes these rows
    const int j = it / S;  // its j-th finishing iteration
    const int b = j % kBinRing;
    const uint32_t ph = (uint32_t)(j / kBinRing) & 1u;
    if (o != slice) {
      // the slot's previous contents (o's finishing iteration j - kBinRing) must have been read
      if (j >= kBinRing) bin_wait(bin_smem_u32(&empty[o][b][wi]), ph ^ 1u);
      const int q = slice < o ? slice : slice - 1;  // my place among o's senders
      const uint32_t dst = bin_mapa(bin_smem_u32(recv + (((b * (S - 1) + q) * kBinWarps + wi) << 5) + lane), (uint32_t)o);
      const uint32_t bar = bin_mapa(bin_smem_u32(&full[b][wi]), (uint32_t)o);
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(dst),
                   "r"(__float_as_uint(p[0])), "r"(bar)
                   : "memory");
      continue;
    }
    const uint32_t fb = bin_smem_u32(&full[b][wi]);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"((S - 1) * 32 * 4) : "memory");
    bin_wait(fb, ph);
    double total = 0.0;
    uint32_t dep = 0;
#pragma unroll
    for (int sl = 0; sl < S; ++sl) {  // slice order, my own sum in place
      float v;
      if (sl == slice) {
        v = p[0];
      } else {
        v = recv[(((b * (S - 1) + (sl < slice ? sl : sl - 1)) * kBinWarps + wi) << 5) + lane];
        dep |= __float_as_uint(v);
      }
      total = sl == 0 ? (double)v : __dadd_rn(total, (double)v);
    }
    // release the slot to sender q (lane q): once every lane's read has returned (the arrive's
    // address depends on the values read, so it cannot be issued earlier; a relaxed arrive: a
    // .release.cluster one would also wait for this warp's outstanding global stores)
    dep = __reduce_or_sync(0xffffffffu, dep);
    asm volatile("and.b32 %0, %0, 0;" : "+r"(dep));  // an opaque zero that waits for the reads
    if (lane < S - 1) {
      const uint32_t snd = (uint32_t)(lane < slice ? lane : lane + 1);
      const uint32_t eb = bin_mapa(bin_smem_u32(&empty[slice][b][wi]) + dep, snd);
      asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(eb) : "memory");
    }
    const int64_t row = r0 + slot;
    const bool active = writer && row < n;
    const float sc = __double2float_rn(total);
    if (active) out[row] = sc;
    if (ghist) hist_add(sh, active, hist_bin(sc));
    if (cmax) {  // the warp's R consecutive rows are one top-k chunk
      const uint32_t wm = __reduce_max_sync(0xffffffffu, active ? hist_bin(sc) : 0u);
      if (lane == 0) cmax[r0 / R] = (uint16_t)wm;
    }
  }
  // no CTA leaves while a peer may still write into its shared memory or arrive on its barriers
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (ghist) hist_flush(sh, ghist);
}

// Generic path: any n_bits. One warp per row; lane l owns bytes {l + 32*t}, bits in order;
// float32(w_j) converted on the fly.
__global__ void __launch_bounds__(256) bin_score_generic(const uint8_t* __restrict__ codes, int64_t n,
                                                         int n_bits, int row_bytes,
                                                         const double* __restrict__ w,
                                                         float* __restrict__ out,
                                                         uint32_t* __restrict__ ghist) {
  __shared__ uint32_t sh[kHistBins];
  if (ghist) hist_zero(sh);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = warp; row < n; row += nwarp) {
    const uint8_t* c = codes + row * row_bytes;
    double acc = 0.0;
    for (int b = lane; b < row_bytes; b += 32) {
      const uint32_t byte = c[b];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = 8 * b + q;
        if (((byte >> q) & 1u) && j < n_bits) acc = __dadd_rn(acc, (double)__double2float_rn(w[j]));
      }
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

// unpack_bits: out[r, j] = bit j of row r as float32 {0, 1}.
__global__ void bin_unpack(const uint8_t* __restrict__ codes, int64_t n, int n_bits, int row_bytes,
                           float* __restrict__ out) {
  const int64_t total = n * (int64_t)n_bits;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t r = e / n_bits;
    const int j = (int)(e - r * n_bits);
    out[e] = (float)((codes[r * row_bytes + (j >> 3)] >> (j & 7)) & 1u);
  }
}

// binarize: bit j of row r = ((x_r - mu) . U_j) > 0 in float64, packed LSB-first.
// One warp per (row, byte): lane q<8 computes bit 8*byte+q with a serial float64 dot in
// column order (numpy's dgemm order differs; exact-zero / sub-ulp ties can flip — tolerance).
__global__ void bin_binarize(const double* __restrict__ U, const float* __restrict__ mu, int m,
                             int n_bits, const double* __restrict__ X, int64_t n,
                             uint8_t* __restrict__ out) {
  const int row_bytes = (n_bits + 7) >> 3;
  const int64_t total = n * (int64_t)row_bytes * 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;  // multiple of 32
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e - (threadIdx.x & 31) < total;
       e += stride) {
    const bool valid = e < total;
    const int64_t r = valid ? e / ((int64_t)row_bytes * 8) : 0;
    const int j = valid ? (int)(e - r * (int64_t)row_bytes * 8) : 0;
    int bit = 0;
    if (valid && j < n_bits) {
      const double* x = X + r * m;
      const double* u = U + (int64_t)j * m;
      double acc = 0.0;
      for (int q = 0; q < m; ++q) acc = __fma_rn(__dsub_rn(x[q], (double)mu[q]), u[q], acc);
      bit = acc > 0.0;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, bit);
    // lanes 0,8,16,24 of each warp own one output byte each (e is warp-aligned below)
    if ((threadIdx.x & 7) == 0 && valid) {
      const int sh = threadIdx.x & 31;
      out[r * row_bytes + (j >> 3)] = (uint8_t)((mask >> sh) & 0xffu);
    }
  }
}

__global__ void bin_hamming(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, int64_t n,
                            int width, int64_t* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    int64_t d = 0;
    for (int q = 0; q < width; ++q) d += __popc((uint32_t)(a[r * width + q] ^ b[r * width + q]));
    out[r] = d;
  }
}

// fast path when rows are whole 128-byte slices; scratch: n doubles when slices > 1
bool bin_bytes_path(int n_bits, const uint8_t* codes) {
  const int row_bytes = (n_bits + 7) / 8;
  return n_bits % 8 == 0 && (row_bytes == 128 || row_bytes == 256 || row_bytes == 512 || row_bytes == 1024) &&
         (((uintptr_t)codes) & 3) == 0;
}

// w: float64 model (device); cast to float32 in-kernel (ranker.py:89). hist: see dense.
int launch_bin_score(const uint8_t* codes, int64_t n, int n_bits, const double* w, float* out,
                     uint32_t* hist, double* scratch, int device, cudaStream_t st, uint16_t* cmax,
                     int* clog) {
  if (n <= 0) return OTF_OK;
  const int row_bytes = (n_bits + 7) / 8;
  if (bin_bytes_path(n_bits, codes) && (row_bytes == 128 || scratch != nullptr)) {
    const int slices = row_bytes / 128;
    const size_t smem = (size_t)4 * 256 * 32 * sizeof(float);
    static bool configured[64] = {false};
    if (!configured[device & 63]) {
      cudaFuncSetAttribute((const void*)bin_score_bytes<128, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute((const void*)bin_score_bytes<256, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute((const void*)bin_score_bytes<512, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute((const void*)bin_score_bytes<1024, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      configured[device & 63] = true;
    }
    // tensor map over the codes (u8, RB x n) for the in-kernel L2 prefetch of the next tile
    CUtensorMap map;
    memset(&map, 0, sizeof(map));
    int use_pf = 0;
    {
      static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
      if (!enc) {
        cudaDriverEntryPointQueryResult q;
        void* fp = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
          enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
      }
      const cuuint64_t dims[2] = {(cuuint64_t)row_bytes, (cuuint64_t)n};
      const cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
      const cuuint32_t box[2] = {128, 32};
      const cuuint32_t estr[2] = {1, 1};
      if (enc && !getenv("OTF_BIN_NO_PREFETCH") && n < (int64_t)0x7fffffff &&
          enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(codes), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
        use_pf = 1;  // distance 1..3 iterations measured the same
    }
    // The clustered single launch is opt-in (OTF_BIN_CLUSTER=1, read per call): bit-identical,
    // but measured slower than the per-slice launches on the same boxes (C5a 6.1-6.4 vs 5.7-5.8
    // ms under sw_power_cap)
    const char* cl = getenv("OTF_BIN_CLUSTER");
    if (slices > 1 && cl && cl[0] == '1') {
      // one launch: clusters of `slices` CTAs, the slice sums meet in the leader's shared memory
      const int S = slices;
      const size_t csmem = smem + (size_t)kBinRing * (S - 1) * kBinWarps * 32 * sizeof(float);
      const void* fn = row_bytes == 256 ? (const void*)bin_score_cluster<256>
                     : row_bytes == 512 ? (const void*)bin_score_cluster<512> : (const void*)bin_score_cluster<1024>;
      static bool cconf[64] = {false};
      if (!cconf[device & 63]) {
        cudaFuncSetAttribute((const void*)bin_score_cluster<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(smem + (size_t)kBinRing * 1 * kBinWarps * 128));
        cudaFuncSetAttribute((const void*)bin_score_cluster<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(smem + (size_t)kBinRing * 3 * kBinWarps * 128));
        cudaFuncSetAttribute((const void*)bin_score_cluster<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(smem + (size_t)kBinRing * 7 * kBinWarps * 128));
        cudaFuncSetAttribute((const void*)bin_score_cluster<1024>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cconf[device & 63] = true;
      }
      int64_t ncl = sm_count(device) / S;
      const int64_t cneed = (n + kBinWarps * 32 - 1) / (kBinWarps * 32);
      if (cneed < ncl) ncl = cneed;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(ncl * S));
      cfg.blockDim = dim3(kBinThreads);
      cfg.dynamicSmemBytes = csmem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = (unsigned)S;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      void* args[] = {(void*)&codes, (void*)&n, (void*)&w, (void*)&n_bits, (void*)&out, (void*)&hist, (void*)&map,
                      (void*)&use_pf, (void*)&cmax};
      OTF_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
      OTF_LAUNCH_CHECK("bin_score_cluster");
      if (cmax && clog) *clog = 5;
      return OTF_OK;
    }
    static const bool narrow_env = getenv("OTF_BIN_NARROW") != nullptr;  // A/B switch (tools/)
    // the wide kernel's 16-byte loads need 16-byte aligned rows (an adopted device pointer may only
    // be 4-byte aligned: bin_bytes_path's requirement)
    const bool narrow = narrow_env || (((uintptr_t)codes) & 15) != 0;
    if (!narrow) {
      static bool wconf[64] = {false};
      if (!wconf[device & 63]) {
        cudaFuncSetAttribute((const void*)bin_score_bytes<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute((const void*)bin_score_bytes<256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute((const void*)bin_score_bytes<512, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute((const void*)bin_score_bytes<1024, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        wconf[device & 63] = true;
      }
    }
    int64_t grid = sm_count(device);  // one 512-thread CTA per SM (128 KB table)
    const int64_t need = (n + (kBinThreads / 32) * 32 - 1) / ((kBinThreads / 32) * 32);
    if (need < grid) grid = need;
    for (int s = 0; s < slices; ++s) {
      const bool last = s == slices - 1;
      const double* pin = s ? scratch : nullptr;
      double* pout = last ? nullptr : scratch;
      float* o = last ? out : nullptr;
      switch (row_bytes) {
        case 128:
          if (narrow) bin_score_bytes<128, false><<<(int)grid, kBinThreads, smem, st>>>(codes, n, s, w, n_bits, pin, pout, o, hist, map, use_pf, last ? cmax : nullptr);
          else bin_score_bytes<128, true><<<(int)grid, kBinThreads, smem, st>>>(codes, n, s, w, n_bits, pin, pout, o, hist, map, use_pf, last ? cmax : nullptr);
          break;
        case 256:
          if (narrow) bin_score_bytes<256, false><<<(int)grid, kBinThreads, smem, st>>>(codes, n, s, w, n_bits, pin, pout, o, hist, map, use_pf, last ? cmax : nullptr);
          else bin_score_bytes<256, true><<<(int)grid, kBinThreads, smem, st>>>(codes, n, s, w, n_bits, pin, pout, o, hist, map, use_pf, last ? cmax : nullptr);
          break;
        case 512:
          if (narrow) bin_score_bytes<512, false><<<(int)grid, kBinThreads, smem, st>>>(codes, n, s, w, n_bits, pin, pout, o, hist, map, use_pf, last ? cmax : nullptr);
          else bin_score_bytes<512, true><<<(int)grid, kBinThreads, smem, st>>>(codes, n, s, w, n_bits, pin, pout, o, hist, map, use_pf, last ? cmax : nullptr);
          break;
        default:
          if (narrow) bin_score_bytes<1024, false><<<(int)grid, kBinThreads, smem, st>>>(codes, n, s, w, n_bits, pin, pout, o, hist, map, use_pf, last ? cmax : nullptr);
          else bin_score_bytes<1024, true><<<(int)grid, kBinThreads, smem, st>>>(codes, n, s, w, n_bits, pin, pout, o, hist, map, use_pf, last ? cmax : nullptr);
          break;
      }
      OTF_LAUNCH_CHECK("bin_score_bytes");
    }
    if (cmax && clog) *clog = 5;  // 32 rows per chunk
    return OTF_OK;
  }
  int64_t grid = (n + 7) / 8;
  const int64_t cap = 8LL * sm_count(device);
  if (grid > cap) grid = cap;
  bin_score_generic<<<(int)grid, 256, 0, st>>>(codes, n, n_bits, row_bytes, w, out, hist);
  OTF_LAUNCH_CHECK("bin_score_generic");
  return OTF_OK;
}

int launch_bin_unpack(const uint8_t* codes, int64_t n, int n_bits, float* out, int device,
                      cudaStream_t st) {
  const int64_t total = n * (int64_t)n_bits;
  if (total <= 0) return OTF_OK;
  int64_t grid = (total + 255) / 256;
  const int64_t cap = 16LL * sm_count(device);
  if (grid > cap) grid = cap;
  bin_unpack<<<(int)grid, 256, 0, st>>>(codes, n, n_bits, (n_bits + 7) / 8, out);
  OTF_LAUNCH_CHECK("bin_unpack");
  return OTF_OK;
}

int launch_binarize(const double* U, const float* mu, int m, int n_bits, const double* X,
                    int64_t n, uint8_t* out, int device, cudaStream_t st) {
  const int row_bytes = (n_bits + 7) >> 3;
  const int64_t total = n * (int64_t)row_bytes * 8;
  if (total <= 0) return OTF_OK;
  // total is a multiple of 8; use a block size multiple of 32 and keep grid-stride
  // iterations warp-aligned so the ballot covers whole bytes.
  int64_t grid = (total + 255) / 256;
  const int64_t cap = 16LL * sm_count(device);
  if (grid > cap) grid = cap;
  bin_binarize<<<(int)grid, 256, 0, st>>>(U, mu, m, n_bits, X, n, out);
  OTF_LAUNCH_CHECK("bin_binarize");
  return OTF_OK;
}

int launch_hamming(const uint8_t* a, const uint8_t* b, int64_t n, int width, int64_t* out,
                   int device, cudaStream_t st) {
  if (n <= 0) return OTF_OK;
  int64_t grid = (n + 255) / 256;
  const int64_t cap = 8LL * sm_count(device);
  if (grid > cap) grid = cap;
  bin_hamming<<<(int)grid, 256, 0, st>>>(a, b, n, width, out);
  OTF_LAUNCH_CHECK("bin_hamming");
  return OTF_OK;
}

}  // namespace otf
