// otf_multi.cu — K7: many classifiers at once (C5b): S = X · Wᵀ on the 5th-gen tensor cores.
//
// The reference scores one model per call (score_dense, ranker.py:63-69: float32 sgemv); C5b
// ranks the same repository under up to 64 classifiers, i.e. a skinny GEMM (N = 64) with 32
// flop/B — float32 SIMT would be ~3x slower than HBM, so it runs on tcgen05 with split operands
// for float32-level accuracy (three products; the fourth, lo·lo, is below float32 rounding).
//
// FP16 form (default, kind::f16): X is scaled by 2^ex (max |x| 2^ex in [2^14, 2^15): one pass
// per repository, multi_x_exponent) and classifier c by 2^ew_c, then
//     x1 = f16(x), x2 = f16(x − x1), w1 = f16(w), w2 = f16(w − w1),
//     x·w ≈ x1·w1 + x1·w2 + x2·w1     (each dropped / rounded term <= 2^-22 relative),
// undone exactly by 2^-(ex + ew_c) at the store. W is split once per call on the device into
// [w1; w2] (float16 tiles, SWIZZLE_64B); one N=128 MMA computes x1·w1 (accumulator columns
// 0..63) and x1·w2 (64..127), an N=64 MMA adds x2·w1 into 64..127, both with A = [x1 | x2] from
// a TMEM slot the split warps fill (packed float32-pair arithmetic: 3 instructions per element).
// kind::f16 runs at twice the TF32 rate and half its energy: the kernel is power-capped
// (sw_power_cap) at this size, so the FP16 form is ~15% faster.
//
// TF32 form (kind::tf32; X holding inf/NaN or extreme magnitudes, or OTF_MULTI_TF32=1):
//     x·w ≈ x_hi·w_hi + x_hi·w_lo + x_lo·w_hi,   v_hi = v with the low 13 mantissa bits cleared
//                                                 (exact TF32), v_lo = v − v_hi (exact float32).
// W is split into [w_hi; w_lo]; the N=128 MMA reads the raw float32 X tile straight from the TMA
// ring as x_hi (kind::tf32 reads a float32 operand as its TF32 truncation — the GPU parity test
// pins this: rounding would break its 2^-20 bound) and only x_lo is computed into the TMEM slot.
//
// The kernel runs on CTA pairs (cta_group::2, M = 256 rows per MMA; the default) or on single
// CTAs (M = 128; only for inputs of one 128-row tile). Per CTA, one per SM, persistent over
// (pair) tiles, warp-specialised:
//   warp 0      TMA producer: X tile (128 rows × 32 floats = 16 KB, SWIZZLE_128B), 8-stage ring
//   warp 3      TMA producer: W tile (L2-resident, paced by the MMAs)
//   warp 1      MMA issuer (leader CTA): per chunk of 32 K, TF32: 4 K-steps × (N=128 SS + N=64
//               TS), FP16: 2 K-steps × (N=128 TS + N=64 TS) tcgen05.mma; one elected lane of the
//               converged warp issues the whole chunk from uniform registers
//   warp 2      TMEM allocator: 512 columns = 2 × 128 accumulators + 8 × 32-column A slots
//   warps 4–7   epilogue: tcgen05.ld the accumulators, add halves, store scores classifier-major
//   warps 8–15  split: thread r reads row r of the swizzled X tile, writes x_lo (TF32) or x1|x2
//               (FP16) of that row into a TMEM slot (tcgen05.st); two warpgroups alternate chunks
// On a pair, each CTA holds its own 128 X rows and HALF of the classifier operand (2-CTA MMAs
// split B across the pair): per chunk a 96-row W tile = its 64-row half of [w_hi; w_lo] and its
// 32-row half of w_hi. Against single CTAs that halves the tensor core's shared-memory reads of W
// (24 -> 12 KB per chunk) and the W TMA writes (16 -> 12 KB) — shared-memory bandwidth was the
// bound — and halves the MMA instructions per SM. The leader's barriers count the peer's TMA bytes
// (wfull), split arrivals (a_full) and epilogue arrivals (tmem_empty); MMA commits are multicast
// to the same barrier in both CTAs. Remote arrivals use the default (.release.cta) semantics: a
// .release.cluster arrive per chunk doubled the kernel time.
// Every output row is computed by the same MMA sequence whatever its tile, so a row's scores do
// not depend on its position. Parity is a tolerance against the reference's float32 sgemv
// (DESIGN.md §Parity); ranking of each classifier is the exact top-k of these scores.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cuda_fp16.h>

#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "otf_common.cuh"
#include "otf_internal.h"

namespace otf {

constexpr int kMT = 128;          // rows per CTA tile
constexpr int kKC = 32;           // K floats per chunk (128 bytes = one swizzle row)
constexpr int kXStages = 8;       // X ring (freed by the split warps + the MMA commit)
constexpr int kASlots = 8;        // TMEM ring of 32-column x_lo slots
// The tensor core accumulates in float32 without round-to-nearest on every add: accumulated over
// all of K (d = 4096) the error reached 0.9 of the reference tolerance. Restarting the
// accumulation every 4 chunks (128 K values) and adding the group partials in float32 (RN) in the
// epilogue brings it to numpy's own float32 sgemm level (0.055 vs 0.041 of the tolerance at
// d = 4096; 0.155 vs 0.128 at d = 512) at ~1-3% of kernel time (tools/multi_err.py).
// FP16 form, measured against the exact dot (tools/multi_err.py, max over 20k rows x 64
// classifiers, fraction of the tolerance): 4 chunks 0.029 / 0.064 (d = 4096 / 512), 8 chunks
// 0.032 / 0.111, 16 chunks 0.055 / 0.186; numpy's own float32 sgemm: 0.041 / 0.128. 8 keeps
// the error below numpy's and halves the epilogue's group adds (C5b -2.5% under the power cap).
// The TF32 form keeps 4.
template <bool H>
constexpr int group_chunks() { return H ? 8 : 4; }
constexpr int kTileX = kMT * kKC * 4;  // 16 KB
constexpr int kMultiThreads = 512;
constexpr int kTmemCols = 512;
constexpr int kAccCols = 256;     // 2 accumulators x 128 columns

template <int P>
struct PairCfg;
template <>
struct PairCfg<1> {  // single CTA: W tile = [w_hi; w_lo] (128 rows); the N=64 MMA uses rows 0..63
  static constexpr int kWRows = 128, kWStages = 4, kW2Row = 0;
};
template <>
struct PairCfg<2> {  // pair: W tile = this CTA's 64-row half of [w_hi; w_lo] + 32-row half of w_hi
  static constexpr int kWRows = 96, kWStages = 6, kW2Row = 64;
};
// H: the FP16 form (kind::f16, below); W rows are 32 halves = 64 bytes (SWIZZLE_64B), else 32
// floats = 128 bytes (SWIZZLE_128B)
template <bool H>
constexpr int w_row_bytes() { return H ? kKC * 2 : kKC * 4; }
template <int P, bool H>
constexpr int ring_bytes() {
  return kXStages * kTileX + PairCfg<P>::kWStages * PairCfg<P>::kWRows * w_row_bytes<H>();
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  while (!mbar_try(b, parity)) {
  }
}
// shared::cluster address of the same variable in the pair's leader (rank 0)
__device__ __forceinline__ uint32_t mapa_rank0(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t caddr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// K-major, SWIZZLE_128B shared-memory matrix descriptor (rows of 128 B, 8-row atoms of 1 KB).
// A K-step of 8 tf32 (32 B) inside the swizzled row advances the start address field by 2.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);        // start address
  d |= (uint64_t)1u << 16;                        // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024u >> 4) << 32;              // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1u << 46;                        // descriptor version (sm100)
  d |= (uint64_t)2u << 61;                        // layout: SWIZZLE_128B
  return d;
}
// K-major, SWIZZLE_64B (rows of 64 B, 8-row atoms of 512 B): the FP16 W tiles. A K-step of 16
// halves (32 B) advances the start address field by 2, as for SW128.
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(512u >> 4) << 32;               // stride byte offset: 8 rows x 64 B
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)4u << 61;                        // layout: SWIZZLE_64B
  return d;
}
// Instruction descriptor: kind::f16 with F16 A/B, F32 accumulate, K-major.
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
// Instruction descriptor: kind::tf32, F32 accumulate, A/B K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4)                     // D format F32
         | (2u << 7)                   // A format TF32
         | (2u << 10)                  // B format TF32
         | ((uint32_t)(n >> 3) << 17)  // N >> 3
         | ((uint32_t)(m >> 4) << 24);  // M >> 4
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

// (a, b) -> x1 = f16x2(xs a, xs b) and x2 = f16x2 of the residuals (low half = a)
__device__ __forceinline__ void split_f16_pair(float a, float b, float xs, uint32_t& x1, uint32_t& x2) {
  asm("{\n\t.reg .b64 v, s, f, r;\n\t.reg .f32 e0, e1, g0, g1;\n\t.reg .f16 h0, h1;\n\t"
      "mov.b64 v, {%2, %3};\n\t"
      "mov.b64 s, {%4, %4};\n\t"
      "mul.rn.f32x2 r, v, s;\n\t"
      "mov.b64 {e0, e1}, r;\n\t"
      "cvt.rn.f16x2.f32 %0, e1, e0;\n\t"
      "mov.b32 {h0, h1}, %0;\n\t"
      "cvt.f32.f16 g0, h0;\n\t"
      "cvt.f32.f16 g1, h1;\n\t"
      "mov.b64 f, {g0, g1};\n\t"
      "sub.rn.f32x2 r, r, f;\n\t"
      "mov.b64 {e0, e1}, r;\n\t"
      "cvt.rn.f16x2.f32 %1, e1, e0;\n\t}"
      : "=r"(x1), "=r"(x2)
      : "f"(a), "f"(b), "f"(xs));
}

// The tcgen05 / TMA / barrier instructions that differ between a single CTA and a pair.
#define OTF_ELECT "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\t"

template <int P>
struct Ops;
template <>
struct Ops<1> {
  static __device__ __forceinline__ uint32_t leader_bar(const void* p) { return smem_u32(p); }
  static __device__ __forceinline__ void arrive_leader(uint32_t a) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
  }
  static __device__ __forceinline__ void load_w(uint32_t dst, const CUtensorMap* map, uint32_t bar, uint32_t bytes,
                                                int c1) {
    asm volatile(OTF_ELECT
                 "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%2], %3;\n\t"
                 "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%4, %5}], [%2];\n\t}" ::
                     "r"(dst),
                 "l"(map), "r"(bar), "r"(bytes), "r"(0), "r"(c1)
                 : "memory");
  }
  static __device__ __forceinline__ void commit(uint64_t* b) {
    asm volatile(OTF_ELECT "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
                     smem_u32(b))
                 : "memory");
  }
  static __device__ __forceinline__ void mma_chunk(uint32_t acc, uint64_t xd, uint32_t alo, uint64_t wd, uint64_t wd2,
                                                   int kc, uint32_t x_empty, uint32_t w_empty, uint32_t a_empty) {
    constexpr uint32_t id128 = idesc_tf32(128, 128), id64 = idesc_tf32(128, 64);
    asm volatile(OTF_ELECT
                 "setp.ne.b32 p, %5, 0;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %2, %4, %6, p;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %8, %9, %6, 1;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %10, %11, %6, 1;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %12, %13, %6, 1;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%20];\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [%3], %14, %7, 1;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [%15], %16, %7, 1;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [%17], %18, %7, 1;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [%19], %23, %7, 1;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%21];\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%22];\n\t}" ::"r"(acc),
                 "r"(acc + 64), "l"(xd), "r"(alo), "l"(wd), "r"(kc), "r"(id128), "r"(id64), "l"(xd + 2), "l"(wd + 2),
                 "l"(xd + 4), "l"(wd + 4), "l"(xd + 6), "l"(wd + 6), "l"(wd2), "r"(alo + 8), "l"(wd2 + 2),
                 "r"(alo + 16), "l"(wd2 + 4), "r"(alo + 24), "r"(x_empty), "r"(w_empty), "r"(a_empty), "l"(wd2 + 6)
                 : "memory");
  }
  // FP16 chunk: acc[0..127] += x1 · [w1; w2] and acc[64..127] += x2 · w1, both A operands from the
  // TMEM slot (x1 in columns 0..15, x2 in 16..31: two halves per column), 2 K-steps of 16
  static __device__ __forceinline__ void mma_chunk_h(uint32_t acc, uint32_t alo, uint64_t wd, uint64_t wd2, int kc,
                                                     uint32_t w_empty, uint32_t a_empty) {
    constexpr uint32_t id128 = idesc_f16(128, 128), id64 = idesc_f16(128, 64);
    asm volatile(OTF_ELECT
                 "setp.ne.b32 p, %5, 0;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %3, %6, p;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], %9, %6, 1;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%1], [%10], %4, %7, 1;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%1], [%11], %12, %7, 1;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%13];\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%14];\n\t}" ::"r"(acc),
                 "r"(acc + 64), "r"(alo), "l"(wd), "l"(wd2), "r"(kc), "r"(id128), "r"(id64), "r"(alo + 8), "l"(wd + 2),
                 "r"(alo + 16), "r"(alo + 24), "l"(wd2 + 2), "r"(w_empty), "r"(a_empty)
                 : "memory");
  }
};
template <>
struct Ops<2> {
  static __device__ __forceinline__ uint32_t leader_bar(const void* p) { return mapa_rank0(p); }
  static __device__ __forceinline__ void arrive_leader(uint32_t a) { mbar_arrive_cluster(a); }
  // this CTA's W half into its own shared memory, bytes counted on the leader's barrier
  static __device__ __forceinline__ void load_w(uint32_t dst, const CUtensorMap* map, uint32_t bar, uint32_t bytes,
                                                int c1) {
    asm volatile(OTF_ELECT
                 "@e mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%2], %3;\n\t"
                 "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%4, %5}], [%2];\n\t}" ::"r"(dst),
                 "l"(map), "r"(bar), "r"(bytes), "r"(0), "r"(c1)
                 : "memory");
  }
  static __device__ __forceinline__ void commit(uint64_t* b) {
    asm volatile(OTF_ELECT
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
                     smem_u32(b)),
                 "h"((unsigned short)3)
                 : "memory");
  }
  static __device__ __forceinline__ void mma_chunk(uint32_t acc, uint64_t xd, uint32_t alo, uint64_t wd, uint64_t wd2,
                                                   int kc, uint32_t x_empty, uint32_t w_empty, uint32_t a_empty) {
    constexpr uint32_t id128 = idesc_tf32(256, 128), id64 = idesc_tf32(256, 64);
    asm volatile(OTF_ELECT
                 "setp.ne.b32 p, %5, 0;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %2, %4, %6, p;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %8, %9, %6, 1;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %10, %11, %6, 1;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %12, %13, %6, 1;\n\t"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%20], %24;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::tf32 [%1], [%3], %14, %7, 1;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::tf32 [%1], [%15], %16, %7, 1;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::tf32 [%1], [%17], %18, %7, 1;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::tf32 [%1], [%19], %23, %7, 1;\n\t"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%21], %24;\n\t"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%22], %24;\n\t}" ::"r"(acc),
                 "r"(acc + 64), "l"(xd), "r"(alo), "l"(wd), "r"(kc), "r"(id128), "r"(id64), "l"(xd + 2), "l"(wd + 2),
                 "l"(xd + 4), "l"(wd + 4), "l"(xd + 6), "l"(wd + 6), "l"(wd2), "r"(alo + 8), "l"(wd2 + 2),
                 "r"(alo + 16), "l"(wd2 + 4), "r"(alo + 24), "r"(x_empty), "r"(w_empty), "r"(a_empty), "l"(wd2 + 6),
                 "h"((unsigned short)3)
                 : "memory");
  }
  static __device__ __forceinline__ void mma_chunk_h(uint32_t acc, uint32_t alo, uint64_t wd, uint64_t wd2, int kc,
                                                     uint32_t w_empty, uint32_t a_empty) {
    constexpr uint32_t id128 = idesc_f16(256, 128), id64 = idesc_f16(256, 64);
    asm volatile(OTF_ELECT
                 "setp.ne.b32 p, %5, 0;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%2], %3, %6, p;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%8], %9, %6, 1;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%1], [%10], %4, %7, 1;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%1], [%11], %12, %7, 1;\n\t"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%13], %15;\n\t"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%14], %15;\n\t}" ::"r"(acc),
                 "r"(acc + 64), "r"(alo), "l"(wd), "l"(wd2), "r"(kc), "r"(id128), "r"(id64), "r"(alo + 8), "l"(wd + 2),
                 "r"(alo + 16), "r"(alo + 24), "l"(wd2 + 2), "r"(w_empty), "r"(a_empty), "h"((unsigned short)3)
                 : "memory");
  }
};

template <int P, bool H>
__global__ void __launch_bounds__(kMultiThreads, 1)
multi_score_tc(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w, int64_t n,
               int d, int n_cls, float* __restrict__ out, float xs, const float* __restrict__ inv_scale) {
  // H (FP16 form): xs = 2^ex scales X into the float16 range; inv_scale[c] = 2^-(ex + ew_c) undoes
  // it and classifier c's own scale at the store (both exact powers of two)
  using C = PairCfg<P>;
  using O = Ops<P>;
  constexpr int kTileW = C::kWRows * w_row_bytes<H>();
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);  // swizzle atoms: 1 KB
  __shared__ uint64_t full[kXStages], empty[kXStages];           // X ring
  __shared__ uint64_t wfull[C::kWStages], wempty[C::kWStages];   // W ring
  __shared__ uint64_t a_full[kASlots], a_empty[kASlots];         // TMEM x_lo ring
  __shared__ uint64_t tmem_full[2], tmem_empty[2];               // accumulators
  __shared__ uint32_t tmem_base_slot;
  __shared__ float s_inv[64];
  if (H && threadIdx.x < 64) s_inv[threadIdx.x] = inv_scale[threadIdx.x];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = P == 2 ? cluster_ctarank() : 0u;
  const int64_t unit = blockIdx.x / P, n_units = gridDim.x / P;  // pair (or CTA) index
  const int64_t n_tiles = (n + P * kMT - 1) / (P * kMT);         // P*128-row tiles
  const int kchunks = d / kKC;
  unsigned char* const xring = smem;
  unsigned char* const wring = smem + kXStages * kTileX;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kXStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], H ? 4 : 5);  // 4 split warps (+ the TF32 MMA commit: x_hi is read from the tile)
    }
    for (int s = 0; s < C::kWStages; ++s) {
      mbar_init(&wfull[s], P);  // one expect_tx arrival per CTA
      mbar_init(&wempty[s], 1);
    }
    for (int a = 0; a < kASlots; ++a) {
      mbar_init(&a_full[a], 4 * P);
      mbar_init(&a_empty[a], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 4 * P);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
  }
  if (warp == 2) {
    if constexpr (P == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&tmem_base_slot)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&tmem_base_slot)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if constexpr (P == 2) cluster_sync_all();  // both CTAs' barriers exist before any remote arrival
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = tmem_base_slot;

  // Producers and the MMA issuer run their loops on the whole warp (warp-uniform operands in
  // uniform registers) and issue from one elected lane inside the asm block: issued from a
  // divergent single lane, every tcgen05.mma became a waterfall loop and the issue loop, not the
  // tensor pipe, set the pace.
  if (warp == 0) {
    // ---------------- TMA producer: this CTA's 128 X rows ----------------
    uint32_t it = 0;
    for (int64_t t = unit; t < n_tiles; t += n_units) {
      const int row0 = (int)(t * P * kMT + rank * kMT);
      for (int kc = 0; kc < kchunks; ++kc, ++it) {
        const int s = it % kXStages;
        mbar_wait(&empty[s], ((it / kXStages) & 1u) ^ 1u);
        asm volatile(OTF_ELECT
                     "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%2], %3;\n\t"
                     "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%4, %5}], [%2];\n\t}" ::
                         "r"(smem_u32(xring + s * kTileX)),
                     "l"(&map_x), "r"(smem_u32(&full[s])), "r"((uint32_t)kTileX), "r"(kc * kKC), "r"(row0)
                     : "memory");
      }
    }
  } else if (warp == 3) {
    // ---------------- TMA producer: W (L2-resident, paced by the MMAs) ----------------
    uint32_t it = 0;
    for (int64_t t = unit; t < n_tiles; t += n_units) {
      for (int kc = 0; kc < kchunks; ++kc, ++it) {
        const int s = it % C::kWStages;
        mbar_wait(&wempty[s], ((it / C::kWStages) & 1u) ^ 1u);
        O::load_w(smem_u32(wring + s * kTileW), &map_w, O::leader_bar(&wfull[s]), (uint32_t)kTileW,
                  (int)((kc * P + (int)rank) * C::kWRows));
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA) ----------------
    if (rank == 0) {
      const uint64_t wdesc0 = H ? umma_desc_sw64(smem_u32(wring)) : umma_desc_sw128(smem_u32(wring));
      const uint64_t xdesc0 = umma_desc_sw128(smem_u32(xring));
      // accumulation restarts every group_chunks<H>() chunks in the other accumulator; the epilogue
      // adds the group partials in float32 (round to nearest)
      uint32_t it = 0, j = 0;
      for (int64_t t = unit; t < n_tiles; t += n_units) {
        for (int g0 = 0; g0 < kchunks; g0 += group_chunks<H>(), ++j) {
          const int b = j & 1;
          mbar_wait(&tmem_empty[b], ((j >> 1) & 1u) ^ 1u);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t acc = tmem_base + b * 128;
          const int g1 = g0 + group_chunks<H>() < kchunks ? g0 + group_chunks<H>() : kchunks;
          for (int kc = g0; kc < g1; ++kc, ++it) {
            const int s = it % C::kWStages, sx = it % kXStages, a = it % kASlots;
            mbar_wait(&wfull[s], (it / C::kWStages) & 1u);  // W (both halves) landed
            mbar_wait(&a_full[a], (it / kASlots) & 1u);     // X landed and x_lo in TMEM (both CTAs)
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint64_t wd = wdesc0 + (uint64_t)((s * kTileW) >> 4);
            const uint64_t wd2 = wd + (uint64_t)((C::kW2Row * w_row_bytes<H>()) >> 4);
            if constexpr (H)
              O::mma_chunk_h(acc, tmem_base + kAccCols + a * 32, wd, wd2, kc - g0, smem_u32(&wempty[s]),
                             smem_u32(&a_empty[a]));
            else
              O::mma_chunk(acc, xdesc0 + (uint64_t)((sx * kTileX) >> 4), tmem_base + kAccCols + a * 32, wd, wd2,
                           kc - g0, smem_u32(&empty[sx]), smem_u32(&wempty[s]), smem_u32(&a_empty[a]));
          }
          O::commit(&tmem_full[b]);
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- epilogue: this CTA's 128 rows ----------------
    const int q = warp & 3;  // TMEM lanes 32q .. 32q+31
    const uint32_t te = O::leader_bar(&tmem_empty[0]);
    uint32_t j = 0;
    for (int64_t t = unit; t < n_tiles; t += n_units) {
      const int64_t row = t * P * kMT + rank * kMT + 32 * q + lane;
      float sum[64];
#pragma unroll
      for (int c = 0; c < 64; ++c) sum[c] = 0.f;
      for (int g0 = 0; g0 < kchunks; g0 += group_chunks<H>(), ++j) {
        const int b = j & 1;
        mbar_wait(&tmem_full[b], (j >> 1) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + b * 128;
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) {
          uint32_t h[16], l[16];
          tmem_ld16(taddr + c0, h);
          tmem_ld16(taddr + 64 + c0, l);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int u = 0; u < 16; ++u)
            sum[c0 + u] = __fadd_rn(sum[c0 + u], __fadd_rn(__uint_as_float(h[u]), __uint_as_float(l[u])));
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) O::arrive_leader(te + b * 8);
      }
      if (row < n) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (c < n_cls) out[(int64_t)c * n + row] = H ? __fmul_rn(sum[c], s_inv[c]) : sum[c];
      }
    }
  } else if (warp >= 8) {
    // ---------------- split: x_lo of row r into this CTA's TMEM slot ----------------
    const int q = warp & 3;
    const uint32_t par = (uint32_t)((warp - 8) >> 2);
    const int r = 32 * q + lane;
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    const uint32_t af = O::leader_bar(&a_full[0]);
    uint32_t it = 0;
    for (int64_t t = unit; t < n_tiles; t += n_units) {
      for (int kc = 0; kc < kchunks; ++kc, ++it) {
        if ((it & 1u) != par) continue;
        const int s = it % kXStages, a = it % kASlots;
        mbar_wait(&full[s], (it / kXStages) & 1u);
        // row r of the SWIZZLE_128B tile: 16-byte chunk c sits at chunk position c ^ (r & 7)
        const unsigned char* rowp = xring + s * kTileX + r * 128;
        uint32_t lo[32];
        if constexpr (H) {
          // x1 = f16(xs x), x2 = f16(xs x - x1): columns 0..15 hold x1 pairs, 16..31 x2 pairs.
          // Packed float32 pairs: FMUL2, F2FP, 2 HADD2.F32, FADD2, F2FP per two elements.
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 v = *reinterpret_cast<const float4*>(rowp + ((c ^ (r & 7)) << 4));
            split_f16_pair(v.x, v.y, xs, lo[2 * c], lo[16 + 2 * c]);
            split_f16_pair(v.z, v.w, xs, lo[2 * c + 1], lo[16 + 2 * c + 1]);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 v = *reinterpret_cast<const float4*>(rowp + ((c ^ (r & 7)) << 4));
            const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              lo[4 * c + u] = __float_as_uint(__fsub_rn(e[u], __uint_as_float(__float_as_uint(e[u]) & 0xFFFFE000u)));
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // read (TF32: the MMA commit also frees the tile, x_hi)
        mbar_wait(&a_empty[a], ((it / kASlots) & 1u) ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;");
        tmem_st32(tmem_base + lane_off + kAccCols + a * 32, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) O::arrive_leader(af + a * 8);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if constexpr (P == 2) cluster_sync_all();  // no remote arrival or pair MMA may target a CTA that left
  else __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    if constexpr (P == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

// W (n_cls x d float64) -> the split, pre-tiled classifier operand. Each chunk kc (K columns
// 32kc .. 32kc+31) becomes P contiguous tiles of kWRows x 32 floats, [kc][rank][row][32]:
//   P = 1: rows 0..63 = w_hi, rows 64..127 = w_lo
//   P = 2: rank 0: rows 0..63 = w_hi[0..63], rows 64..95 = w_hi[0..31]
//          rank 1: rows 0..63 = w_lo[0..63], rows 64..95 = w_hi[32..63]
// (w32 = float32(w); w_hi = TF32 truncation; w_lo = w32 - w_hi; rows >= n_cls are zero.)
template <int P>
__global__ void split_w_kernel(const double* __restrict__ W, int n_cls, int d, float* __restrict__ ws) {
  constexpr int R = PairCfg<P>::kWRows;
  const int64_t total = (int64_t)64 * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / d), k = (int)(e % d);
    const float w = c < n_cls ? __double2float_rn(W[e]) : 0.0f;
    const float hi = __uint_as_float(__float_as_uint(w) & 0xFFFFE000u);
    const float lo = __fsub_rn(w, hi);
    const int64_t t0 = (int64_t)(k / kKC) * P * R * kKC + (k % kKC);  // rank-0 tile of this chunk
    if (P == 1) {
      ws[t0 + (int64_t)c * kKC] = hi;
      ws[t0 + (int64_t)(64 + c) * kKC] = lo;
    } else {
      const int64_t t1 = t0 + (int64_t)R * kKC;
      ws[t0 + (int64_t)c * kKC] = hi;
      ws[t1 + (int64_t)c * kKC] = lo;
      if (c < 32) ws[t0 + (int64_t)(64 + c) * kKC] = hi;
      else ws[t1 + (int64_t)(32 + c) * kKC] = hi;
    }
  }
}

// FP16 form of the classifier operand: the same tile layout with w1 / w2 (float16) in place of
// w_hi / w_lo, per classifier scaled by 2^ew_c (max |w_c| in [2^14, 2^15)):
//   w1 = f16(2^ew_c w32), w2 = f16(2^ew_c w32 - w1)    (w32 = float32(w), ranker.py:69)
// and inv[c] = 2^-(ex + ew_c) after the 3 * 64 * d halves (0 for rows >= n_cls). One block per
// classifier row.
template <int P>
__global__ void split_w_half_kernel(const double* __restrict__ W, int n_cls, int d, int ex,
                                    __half* __restrict__ ws, float* __restrict__ inv) {
  constexpr int R = PairCfg<P>::kWRows;
  const int c = blockIdx.x;
  __shared__ float red[32];
  float m = 0.f;
  if (c < n_cls)
    for (int k = threadIdx.x; k < d; k += blockDim.x) m = fmaxf(m, fabsf(__double2float_rn(W[(int64_t)c * d + k])));
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  m = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) m = fmaxf(m, red[i]);
  int e = 0;
  if (m > 0.f && m <= 3.4e38f) frexpf(m, &e);  // m < 2^e
  const int ew = m > 0.f && m <= 3.4e38f ? max(-60, min(60, 15 - e)) : 0;
  const float sw = ldexpf(1.f, ew);
  if (threadIdx.x == 0) inv[c] = c < n_cls ? ldexpf(1.f, -(ex + ew)) : 0.f;
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    const float w = c < n_cls ? __fmul_rn(__double2float_rn(W[(int64_t)c * d + k]), sw) : 0.f;
    const __half w1 = __float2half_rn(w);
    const __half w2 = __float2half_rn(__fsub_rn(w, __half2float(w1)));
    const int64_t t0 = (int64_t)(k / kKC) * P * R * kKC + (k % kKC);  // rank-0 tile of this chunk
    if (P == 1) {
      ws[t0 + (int64_t)c * kKC] = w1;
      ws[t0 + (int64_t)(64 + c) * kKC] = w2;
    } else {
      const int64_t t1 = t0 + (int64_t)R * kKC;
      ws[t0 + (int64_t)c * kKC] = w1;
      ws[t1 + (int64_t)c * kKC] = w2;
      if (c < 32) ws[t0 + (int64_t)(64 + c) * kKC] = w1;
      else ws[t1 + (int64_t)(32 + c) * kKC] = w1;
    }
  }
}

// max |x| over the repository -> the FP16 data scale exponent ex (max |x| 2^ex in [2^14, 2^15)),
// plus the smallest non-zero per-row max |x| (the FP16 form's error has an absolute floor of about
// max|X| 2^-39.5 per element, so a row far below the largest element falls back to TF32). One
// warp per row: out[0] = max bits (0xffffffff: inf / NaN present), out[1] = min non-zero row max.
__global__ void absmax_kernel(const float4* __restrict__ X, int64_t n, int d4, unsigned int* __restrict__ out) {
  float m = 0.f, mrow = __int_as_float(0x7f800000);
  bool bad = false;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n; r += nwarps) {  // warp-uniform
    float rm = 0.f;
    for (int j = lane; j < d4; j += 32) {
      const float4 v = ld_stream_f4(X + r * d4 + j);
      rm = fmaxf(rm, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      bad |= !(fabsf(v.x) <= 3.4e38f && fabsf(v.y) <= 3.4e38f && fabsf(v.z) <= 3.4e38f && fabsf(v.w) <= 3.4e38f);
    }
    for (int o = 16; o; o >>= 1) rm = fmaxf(rm, __shfl_xor_sync(0xffffffffu, rm, o));
    m = fmaxf(m, rm);
    if (rm > 0.f) mrow = fminf(mrow, rm);
  }
  for (int o = 16; o; o >>= 1) bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  if (lane == 0) {
    atomicMax(out, bad ? 0xffffffffu : __float_as_uint(m));
    atomicMin(out + 1, __float_as_uint(mrow));
  }
}

// ---- host side --------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D tensor map, boxes of kKC x box_outer elements: float32 rows of 128 B (SWIZZLE_128B) or, with
// half = true, float16 rows of 64 B (SWIZZLE_64B)
static int make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_outer,
                    bool half = false) {
  auto enc = get_encode();
  if (!enc) return fail(OTF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {inner * (half ? 2 : 4)};
  const cuuint32_t box[2] = {kKC, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, half ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   half ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(OTF_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return OTF_OK;
}

bool multi_tc_supported(int d, const float* X) {
  return d % kKC == 0 && d >= kKC && (((uintptr_t)X) & 15) == 0;
}

template <int P, bool H>
static int launch_p(const CUtensorMap& mx, const float* X, int64_t n, int d, const double* W, int n_cls, float* ws,
                    float* out, int x_exp, int device, cudaStream_t st) {
  constexpr int R = PairCfg<P>::kWRows;
  CUtensorMap mw;
  const float* inv = nullptr;
  if constexpr (H) {
    __half* wh = reinterpret_cast<__half*>(ws);
    float* invw = reinterpret_cast<float*>(wh + (size_t)3 * 64 * d);
    split_w_half_kernel<P><<<64, 256, 0, st>>>(W, n_cls, d, x_exp, wh, invw);
    OTF_LAUNCH_CHECK("split_w_half_kernel");
    if (int rc = make_map(&mw, wh, (uint64_t)kKC, (uint64_t)(d / kKC) * P * R, R, true)) return rc;
    inv = invw;
  } else {
    split_w_kernel<P><<<64, 256, 0, st>>>(W, n_cls, d, ws);
    OTF_LAUNCH_CHECK("split_w_kernel");
    if (int rc = make_map(&mw, ws, (uint64_t)kKC, (uint64_t)(d / kKC) * P * R, R)) return rc;
  }
  const size_t smem = (size_t)ring_bytes<P, H>() + 1024;
  static bool configured[64] = {false};
  if (!configured[device & 63]) {
    OTF_CUDA(cudaFuncSetAttribute((const void*)multi_score_tc<P, H>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    configured[device & 63] = true;
  }
  const int64_t tiles = (n + P * kMT - 1) / (P * kMT);
  int units = sm_count(device) / P;
  if (tiles < units) units = (int)tiles;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)(units * P));
  cfg.blockDim = dim3(kMultiThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = P == 2 ? 1 : 0;
  const float xs = H ? ldexpf(1.f, x_exp) : 1.f;
  OTF_CUDA(cudaLaunchKernelEx(&cfg, multi_score_tc<P, H>, mx, mw, n, d, n_cls, out, xs, inv));
  OTF_LAUNCH_CHECK("multi_score_tc");
  return OTF_OK;
}

int multi_x_exponent(const float* X, int64_t n, int d, int device, cudaStream_t st, int* ex) {
  *ex = INT_MIN;
  unsigned int* dm = nullptr;
  OTF_CUDA(cudaMallocAsync(&dm, 2 * sizeof(unsigned int), st));
  OTF_CUDA(cudaMemsetAsync(dm, 0, sizeof(unsigned int), st));
  OTF_CUDA(cudaMemsetAsync(dm + 1, 0xff, sizeof(unsigned int), st));
  if (n > 0) {
    absmax_kernel<<<4 * sm_count(device), 512, 0, st>>>(reinterpret_cast<const float4*>(X), n, d / 4, dm);
    OTF_LAUNCH_CHECK("absmax_kernel");
  }
  unsigned int bits[2] = {0, 0};
  OTF_CUDA(cudaMemcpyAsync(bits, dm, sizeof(bits), cudaMemcpyDeviceToHost, st));
  OTF_CUDA(cudaFreeAsync(dm, st));
  OTF_CUDA(cudaStreamSynchronize(st));
  if (bits[0] == 0xffffffffu) return OTF_OK;  // inf / NaN in X: the TF32 form handles them
  float m, mrow;
  std::memcpy(&m, &bits[0], sizeof(m));
  std::memcpy(&mrow, &bits[1], sizeof(mrow));
  // FP16 error floor per element ~ m 2^-39.5, summed over |w|_1 <= sqrt(d) |w|_2; keep it below
  // ~5% of the reference tolerance 1e-6 |w| |x_row| (|x_row| >= its max element): TF32 when a
  // non-zero row's max element is more than 2^15 / sqrt(d) below the largest element
  if (m > 0.f && mrow > 0.f && mrow < 3.4e38f && (double)m / (double)mrow > 32768.0 / std::sqrt((double)d))
    return OTF_OK;
  int e = 0;
  if (m > 0.f) frexpf(m, &e);
  const int x = m > 0.f ? 15 - e : 0;
  if (x >= -60 && x <= 60) *ex = x;  // else (extreme magnitudes): TF32
  return OTF_OK;
}

// Scores n rows of X (n x d float32) under n_cls <= 64 classifiers W (n_cls x d float64) into
// out (n_cls x n float32, classifier-major). ws: multi_ws_floats(d) float32 scratch (split W).
int launch_multi_score(const float* X, int64_t n, int d, const double* W, int n_cls, float* ws, float* out,
                       int device, cudaStream_t st, int x_exp) {
  if (n <= 0) return OTF_OK;
  if (n_cls < 1 || n_cls > 64) return fail(OTF_ERR_CONFIG, "multi-classifier scoring takes 1..64 classifiers");
  if (!multi_tc_supported(d, X)) return fail(OTF_ERR_CONFIG, "multi-classifier scoring needs dim % 32 == 0");
  CUtensorMap mx;
  if (int rc = make_map(&mx, X, (uint64_t)d, (uint64_t)n, kMT)) return rc;
  // CTA pairs whenever there are two 128-row tiles (OTF_MULTI_SINGLE=1 forces single CTAs: tests)
  const char* fs = getenv("OTF_MULTI_SINGLE");
  const bool force_single = fs && atoi(fs) != 0;
  // FP16 form unless the data scale is unknown / X is not finite (x_exp == INT_MIN) or
  // OTF_MULTI_TF32=1 (A/B and tests)
  const char* ft = getenv("OTF_MULTI_TF32");
  const bool h = x_exp != INT_MIN && !(ft && atoi(ft) != 0);
  if (n > kMT && sm_count(device) >= 2 && !force_single)
    return h ? launch_p<2, true>(mx, X, n, d, W, n_cls, ws, out, x_exp, device, st)
             : launch_p<2, false>(mx, X, n, d, W, n_cls, ws, out, x_exp, device, st);
  return h ? launch_p<1, true>(mx, X, n, d, W, n_cls, ws, out, x_exp, device, st)
           : launch_p<1, false>(mx, X, n, d, W, n_cls, ws, out, x_exp, device, st);
}

}  // namespace otf
