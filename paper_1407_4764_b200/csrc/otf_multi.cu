// otf_multi.cu — K7: many classifiers at once (C5b): S = X · Wᵀ on the 5th-gen tensor cores.
//
// The reference scores one model per call (score_dense, ranker.py:63-69: float32 sgemv); C5b
// ranks the same repository under 64 classifiers, i.e. a skinny GEMM (N = 64) with 32 flop/B —
// float32 SIMT (~70 TFLOP/s) would be 3x slower than HBM, so it runs on tcgen05 in TF32 with a
// 3-product split for float32-level accuracy:
//     x·w ≈ x_hi·w_hi + x_hi·w_lo + x_lo·w_hi,   v_hi = v with the low 13 mantissa bits cleared
//                                                 (exact TF32), v_lo = v − v_hi (exact float32).
// W (≤ 64 classifiers) is split once on the device into a stacked [w_hi; w_lo] (128 × d) matrix,
// so one N=128 MMA computes x_hi·w_hi (accumulator columns 0..63) and x_hi·w_lo (64..127), and a
// second N=64 MMA adds x_lo·w_hi into columns 64..127; the epilogue adds the two halves.
//
// Per CTA (one per SM, persistent over 128-row tiles), warp-specialised:
//   warp 0      TMA producer: X tile (128 rows × 32 floats, SWIZZLE_128B) + W tile per stage
//               (6-stage shared-memory ring, 32 KB per stage)
//   warp 1      MMA issuer (one thread): per stage 4 K-steps × (N=128 + N=64) tcgen05.mma with the
//               A operands read from TMEM (kind::tf32, A in TMEM, B = W from shared memory)
//   warp 2      TMEM allocator (512 columns: 2 × 128 accumulators + 4 × 64 A slots)
//   warps 4–7   epilogue: tcgen05.ld the accumulators, sum halves, store scores (classifier-major)
//   warps 8–11  split: thread r reads row r of the swizzled X tile, writes x_hi and x_lo of that row
//               into a TMEM A slot (tcgen05.st) and frees the shared-memory X tile right away
// Keeping the split operands in TMEM halves the shared-memory traffic per stage (no x_lo tile, no
// A reads from shared memory) and lets the ring hold 6 stages of X in flight.
// Every output row is computed by the same MMA sequence whatever its tile, so a row's scores do
// not depend on its position. Parity is a tolerance against the reference's float32 sgemv
// (DESIGN.md §Parity); ranking of each classifier is the exact top-k of these scores.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "otf_common.cuh"
#include "otf_internal.h"

namespace otf {

constexpr int kMT = 128;          // rows per tile (UMMA M)
constexpr int kKC = 32;           // K floats per stage (128 bytes = one swizzle row)
#ifndef OTF_MULTI_XSTAGES
#define OTF_MULTI_XSTAGES 8
#endif
#ifndef OTF_MULTI_WSTAGES
#define OTF_MULTI_WSTAGES 4
#endif
constexpr int kXStages = OTF_MULTI_XSTAGES;  // shared-memory ring of X tiles (freed by the split warps)
constexpr int kWStages = OTF_MULTI_WSTAGES;  // shared-memory ring of W tiles (freed by the MMAs)
#ifndef OTF_MULTI_ACC_BUFS
#define OTF_MULTI_ACC_BUFS 2
#endif
constexpr int kAccBufs = OTF_MULTI_ACC_BUFS;  // accumulators (128 TMEM columns each)
#ifndef OTF_MULTI_TSHI
#define OTF_MULTI_SSHI 1
#endif
#ifdef OTF_MULTI_SSHI
// x_hi is not materialised: the N=128 MMA reads the raw X tile from shared memory (the tensor
// core reads float32 operands of kind::tf32 as their TF32 truncation) and only x_lo goes to TMEM
constexpr int kASlotCols = 32;
#else
constexpr int kASlotCols = 64;
#endif
constexpr int kASlots = (512 - 128 * kAccBufs) / kASlotCols;  // TMEM ring for the split A operands
constexpr int kTileX = kMT * kKC * 4;   // 16 KB
constexpr int kTileW = 128 * kKC * 4;   // 16 KB (stacked w_hi; w_lo)
constexpr int kRingBytes = kXStages * kTileX + kWStages * kTileW;
constexpr int kMultiThreads = 512;  // 16 warps: producer, MMA, alloc, -, 4 epilogue, 8 split
constexpr int kTmemCols = 512;    // 2 x 128 accumulator columns + 4 x 64 A columns
constexpr int kAccCols = 128 * kAccBufs;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
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
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// expect_tx(bytes) + 2D TMA load of one box, issued by one elected lane of a converged warp
__device__ __forceinline__ void tma_load_elect(void* dst, const CUtensorMap* map, uint64_t* bar, uint32_t bytes,
                                               int c0, int c1) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%2], %3;\n\t"
      "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%4, %5}], [%2];\n\t}" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(bytes), "r"(c0), "r"(c1)
      : "memory");
}
// K-major, SWIZZLE_128B shared-memory matrix descriptor (rows of 128 B, 8-row atoms of 1 KB).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);        // start address
  d |= (uint64_t)1u << 16;                        // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024u >> 4) << 32;              // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1u << 46;                        // descriptor version (sm100)
  d |= (uint64_t)2u << 61;                        // layout: SWIZZLE_128B
  return d;
}
// Instruction descriptor: kind::tf32, F32 accumulate, A/B K-major, M = 128.
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
  return (1u << 4)                     // D format F32
         | (2u << 7)                   // A format TF32
         | (2u << 10)                  // B format TF32
         | ((uint32_t)(n >> 3) << 17)  // N >> 3
         | ((uint32_t)(kMT >> 4) << 24);  // M >> 4
}
// D[tmem] (+)= A[tmem] · B[smem]ᵀ
__device__ __forceinline__ void umma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
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

__global__ void __launch_bounds__(kMultiThreads, 1)
multi_score_tc(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
               int64_t n, int d, int n_cls, float* __restrict__ out, int mode) {
  // mode: 0 in production; diagnostic bits (OTF_MULTI_MODE) switch parts off to find the
  // bottleneck: 1 = no MMA, 2 = no TMEM stores in the split, 4 = no score stores.
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for the swizzled tiles
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[kXStages], empty[kXStages];     // X ring (empty: the 4 split warps)
  __shared__ uint64_t wfull[kWStages], wempty[kWStages];   // W ring (empty: MMA commit)
  __shared__ uint64_t a_full[kASlots], a_empty[kASlots];  // TMEM A ring
  __shared__ uint64_t tmem_full[kAccBufs], tmem_empty[kAccBufs];
  __shared__ uint32_t tmem_base_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_tiles = (n + kMT - 1) / kMT;
  const int kchunks = d / kKC;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kXStages; ++s) {
      mbar_init(&full[s], 1);
#ifdef OTF_MULTI_SSHI
      mbar_init(&empty[s], 5);  // 4 split warps + the MMA commit
#else
      mbar_init(&empty[s], 4);
#endif
    }
    for (int s = 0; s < kWStages; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], 1);
    }
    for (int a = 0; a < kASlots; ++a) {
      mbar_init(&a_full[a], 4);
      mbar_init(&a_empty[a], 1);
    }
    for (int b = 0; b < kAccBufs; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = tmem_base_slot;

  unsigned char* const xring = smem;
  unsigned char* const wring = smem + kXStages * kTileX;
  // Producers, like the MMA issuer, run their loops on the whole warp (warp-uniform operands in
  // uniform registers) and issue from one elected lane inside the asm block.
  if (warp == 0) {
    // ---------------- TMA producer: X ----------------
    // X tiles never wait on the tensor cores: the split warps free a stage as soon as they have
    // read it, so the ring keeps kXStages x 16 KB of HBM reads in flight; the L2 prefetch runs
    // kPrefetch chunks further ahead
    constexpr int kPrefetch = 8;
    int64_t pf_tile = blockIdx.x;
    int pf_kc = 0;
    auto prefetch_next = [&]() {
      if (pf_tile >= n_tiles) return;
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];\n\t}" ::"l"(&map_x),
          "r"(pf_kc * kKC), "r"((int)(pf_tile * kMT))
          : "memory");
      if (++pf_kc == kchunks) { pf_kc = 0; pf_tile += gridDim.x; }
    };
    if (!(mode & 32))
      for (int p = 0; p < kPrefetch; ++p) prefetch_next();
    uint32_t it = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      for (int kc = 0; kc < kchunks; ++kc, ++it) {
        const int s = it % kXStages;
        const uint32_t ph = (it / kXStages) & 1u;
        if (!(mode & 32)) prefetch_next();
        mbar_wait(&empty[s], ph ^ 1u);
#ifdef OTF_MULTI_LANE0
        if (lane == 0) {
          mbar_expect_tx(&full[s], kTileX);
          tma_load_2d(xring + s * kTileX, &map_x, &full[s], kc * kKC, (int)(tile * kMT));
        }
#else
        tma_load_elect(xring + s * kTileX, &map_x, &full[s], kTileX, kc * kKC, (int)(tile * kMT));
#endif
      }
    }
  } else if (warp == 3) {
    // ---------------- TMA producer: W (L2-resident, paced by the MMAs) ----------------
    uint32_t it = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      for (int kc = 0; kc < kchunks; ++kc, ++it) {
        const int s = it % kWStages;
        const uint32_t ph = (it / kWStages) & 1u;
        mbar_wait(&wempty[s], ph ^ 1u);
#ifdef OTF_MULTI_LANE0
        if (lane == 0) {
          mbar_expect_tx(&wfull[s], kTileW);
          tma_load_2d(wring + s * kTileW, &map_w, &wfull[s], 0, kc * 128);
        }
#else
        if ((mode & 64) && it >= (uint32_t)kWStages) {  // diagnostic: no W traffic after the first ring
          if (lane == 0) mbar_arrive(&wfull[s]);
          continue;
        }
        tma_load_elect(wring + s * kTileW, &map_w, &wfull[s], kTileW, 0, kc * 128);
#endif
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // The whole warp runs the loop (so every operand is warp-uniform and lives in uniform
    // registers) and one elected lane issues a chunk's 8 MMAs + 2 commits in a single asm block:
    // issued from a divergent single lane, each MMA became an ELECT/waterfall loop and the issue
    // loop, not the tensor pipe, set the pace.
    constexpr uint32_t id128 = idesc_tf32(128), id64 = idesc_tf32(64);
    const uint64_t wdesc0 = umma_desc_sw128(smem_u32(wring));
    const uint64_t xdesc0 = umma_desc_sw128(smem_u32(xring));
    uint32_t it = 0, j = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++j) {
      const int b = j % kAccBufs;
      mbar_wait(&tmem_empty[b], ((j / kAccBufs) & 1u) ^ 1u);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t acc = tmem_base + b * 128;
      for (int kc = 0; kc < kchunks; ++kc, ++it) {
        const int s = it % kWStages;
        const uint32_t ph = (it / kWStages) & 1u;
        const int a = it % kASlots;
        const uint32_t aph = (it / kASlots) & 1u;
        mbar_wait(&wfull[s], ph);    // W tile landed
        mbar_wait(&a_full[a], aph);  // x_hi / x_lo written to TMEM
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint64_t wd = wdesc0 + (uint64_t)((s * kTileW) >> 4);  // +32 B per K-step = +2
#ifdef OTF_MULTI_SSHI
        const int sx = it % kXStages;
        mbar_wait(&full[sx], (it / kXStages) & 1u);
        const uint64_t xd = xdesc0 + (uint64_t)((sx * kTileX) >> 4);
        const uint32_t alo = tmem_base + kAccCols + a * kASlotCols;
        if (mode & 1) {
          asm volatile(
              "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t"
              "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%1];\n\t"
              "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%2];\n\t}" ::"r"(
                  smem_u32(&wempty[s])),
              "r"(smem_u32(&a_empty[a])), "r"(smem_u32(&empty[sx]))
              : "memory");
          continue;
        }
        asm volatile(
            "{\n\t.reg .pred e, p;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %6, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %2, %4, %7, p;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %9, %5, %7, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %11, %12, %7, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %14, %15, %7, 1;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%19];\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [%3], %4, %8, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [%10], %5, %8, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [%13], %12, %8, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [%16], %15, %8, 1;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%17];\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%18];\n\t}" ::"r"(acc),
            "r"(acc + 64), "l"(xd), "r"(alo), "l"(wd), "l"(wd + 2), "r"(kc), "r"(id128), "r"(id64),
            "l"(xd + 2), "r"(alo + 8), "l"(xd + 4), "l"(wd + 4), "r"(alo + 16), "l"(xd + 6), "l"(wd + 6),
            "r"(alo + 24), "r"(smem_u32(&wempty[s])), "r"(smem_u32(&a_empty[a])), "r"(smem_u32(&empty[sx]))
            : "memory");
        continue;
#endif
        const uint32_t ahi = tmem_base + kAccCols + a * 64;
        if (mode & 1) {
          asm volatile(
              "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t"
              "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%1];\n\t}" ::"r"(
                  smem_u32(&wempty[s])),
              "r"(smem_u32(&a_empty[a]))
              : "memory");
          continue;
        }
        if (mode & 24) {  // diagnostics: 4 MMAs per chunk, N = 128 (8) or N = 64 (16)
          const uint32_t idx = (mode & 8) ? id128 : id64;
          asm volatile(
              "{\n\t.reg .pred e, p;\n\t"
              "elect.sync _|e, 0xffffffff;\n\t"
              "setp.ne.b32 p, %3, 0;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%5], %6, %4, 1;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%7], %8, %4, 1;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%9], %10, %4, 1;\n\t"
              "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%11];\n\t"
              "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%12];\n\t}" ::"r"(acc),
              "r"(ahi), "l"(wd), "r"(kc), "r"(idx), "r"(ahi + 8), "l"(wd + 2), "r"(ahi + 16), "l"(wd + 4),
              "r"(ahi + 24), "l"(wd + 6), "r"(smem_u32(&wempty[s])), "r"(smem_u32(&a_empty[a]))
              : "memory");
          continue;
        }
        // K = 8 tf32 per MMA: 8 TMEM columns of A, 32 B (descriptor +2) of W per K-step
        asm volatile(
            "{\n\t.reg .pred e, p;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %6, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %4, %7, p;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [%3], %4, %8, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%9], %5, %7, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [%10], %5, %8, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%11], %12, %7, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [%13], %12, %8, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%14], %15, %7, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], [%16], %15, %8, 1;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%17];\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%18];\n\t}" ::"r"(acc),
            "r"(acc + 64), "r"(ahi), "r"(ahi + 32), "l"(wd), "l"(wd + 2), "r"(kc), "r"(id128), "r"(id64),
            "r"(ahi + 8), "r"(ahi + 40), "r"(ahi + 16), "l"(wd + 4), "r"(ahi + 48), "r"(ahi + 24), "l"(wd + 6),
            "r"(ahi + 56), "r"(smem_u32(&wempty[s])), "r"(smem_u32(&a_empty[a]))
            : "memory");
      }
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
              smem_u32(&tmem_full[b]))
          : "memory");
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- epilogue ----------------
    const int q = warp & 3;  // TMEM lanes 32q .. 32q+31
    uint32_t j = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++j) {
      const int b = j % kAccBufs;
      mbar_wait(&tmem_full[b], (j / kAccBufs) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int64_t row = tile * kMT + 32 * q + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + b * 128;
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 16) {
        uint32_t h[16], l[16];
        tmem_ld16(taddr + c0, h);
        tmem_ld16(taddr + 64 + c0, l);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < n) {
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int c = c0 + t;
            if (c < n_cls && !(mode & 4))
              out[(int64_t)c * n + row] = __fadd_rn(__uint_as_float(h[t]), __uint_as_float(l[t]));
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[b]);
    }
  } else if (warp >= 8) {
    // ---------------- split: row r -> x_hi, x_lo in TMEM ----------------
    // two warpgroups alternate chunks (even / odd) so one chunk's TMEM store latency overlaps
    // the next chunk's shared-memory reads
    const int q = warp & 3;             // TMEM lane quadrant of this warp
    const uint32_t par = (uint32_t)((warp - 8) >> 2);
    const int r = 32 * q + lane;        // tile row handled by this thread
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    uint32_t it = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      for (int kc = 0; kc < kchunks; ++kc, ++it) {
        if ((it & 1u) != par) continue;
        const int s = it % kXStages;
        const uint32_t ph = (it / kXStages) & 1u;
        const int a = it % kASlots;
        const uint32_t aph = (it / kASlots) & 1u;
        mbar_wait(&full[s], ph);
        // row r of the SWIZZLE_128B tile: 16-byte chunk c sits at chunk position c ^ (r & 7)
        const unsigned char* rowp = xring + s * kTileX + r * 128;
#ifdef OTF_MULTI_SSHI
        uint32_t lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 v = (mode & 128) ? make_float4(r * 1.5f, c * 1.25f, kc * 0.5f, 1.0f)
                                        : *reinterpret_cast<const float4*>(rowp + ((c ^ (r & 7)) << 4));
          const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int t = 0; t < 4; ++t)
            lo[4 * c + t] = __float_as_uint(__fsub_rn(e[t], __uint_as_float(__float_as_uint(e[t]) & 0xFFFFE000u)));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // X tile read (the MMA still reads it as x_hi)
        mbar_wait(&a_empty[a], aph ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (!(mode & 2)) tmem_st32(tmem_base + lane_off + kAccCols + a * kASlotCols, lo);
#else
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 v = *reinterpret_cast<const float4*>(rowp + ((c ^ (r & 7)) << 4));
          const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const uint32_t h = __float_as_uint(e[t]) & 0xFFFFE000u;
            hi[4 * c + t] = h;
            lo[4 * c + t] = __float_as_uint(__fsub_rn(e[t], __uint_as_float(h)));
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // X tile read: the producer may refill it
        mbar_wait(&a_empty[a], aph ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t aaddr = tmem_base + lane_off + kAccCols + a * 64;
        if (!(mode & 2)) {
          tmem_st32(aaddr, hi);
          tmem_st32(aaddr + 32, lo);
        }
#endif
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[a]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

// ================================================================================================
// CTA-pair version (cta_group::2, the default for >= 256 rows): two SMs of a TPC score a 256-row
// pair tile with one M=256 MMA stream issued by the leader CTA. Each CTA keeps its own 128 X rows
// (A operand: x_hi read by the tensor core straight from the TMA tile, x_lo from its TMEM) and
// HALF of the classifier operand: per chunk a 96-row W tile = its 64-row half of [w_hi; w_lo]
// (N=128 MMA) + its 32-row half of w_hi (N=64 MMA). Against the single-CTA kernel this halves the
// tensor core's shared-memory reads of W (24 -> 12 KB per chunk) and the W tile writes
// (16 -> 12 KB), which is what bounded it, and halves the MMA instructions per SM.
//   leader (rank 0): MMA issue; its barriers collect the peer's TMA bytes (W), the peer's split
//   arrivals (a_full) and the peer's epilogue arrivals (tmem_empty)
//   MMA commits are multicast to the same barrier in both CTAs
// ================================================================================================
constexpr int kW2Rows = 96;
constexpr int kTileW2 = kW2Rows * kKC * 4;  // 12 KB
#ifndef OTF_MULTI2_X
#define OTF_MULTI2_X 8
#endif
#ifndef OTF_MULTI2_W
#define OTF_MULTI2_W 6
#endif
constexpr int kX2Stages = OTF_MULTI2_X;
constexpr int kW2Stages = OTF_MULTI2_W;
constexpr int kRing2Bytes = kX2Stages * kTileX + kW2Stages * kTileW2;  // 200 KB
constexpr int kA2Slots = 8;                 // 32-column x_lo slots after 2 x 128 accumulator columns

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_rank0(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ bool mbar_try_cl(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cl(uint64_t* b, uint32_t parity) {
  while (!mbar_try_cl(b, parity)) {
  }
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t caddr) {
#ifdef OTF_MULTI_REL_CLUSTER
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
#else
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
#endif
}

// barriers that only see local arrivals or the leader's multicast commits
#ifdef OTF_MULTI_CL_ALL
#define OTF_WAIT_LOCAL mbar_wait_cl
#else
#define OTF_WAIT_LOCAL mbar_wait
#endif
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kMultiThreads, 1)
multi_score_tc2(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                int64_t n, int d, int n_cls, float* __restrict__ out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[kX2Stages], empty[kX2Stages];    // local X ring (empty: 4 split warps + commit)
  __shared__ uint64_t wfull[kW2Stages], wempty[kW2Stages];  // wfull: leader's, both CTAs' bytes
  __shared__ uint64_t a_full[kA2Slots], a_empty[kA2Slots];  // a_full: leader's, 8 split warps
  __shared__ uint64_t tmem_full[2], tmem_empty[2];          // tmem_empty: leader's, 8 epilogue warps
  __shared__ uint32_t tmem_base_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int64_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int64_t n_pt = (n + 2 * kMT - 1) / (2 * kMT);
  const int kchunks = d / kKC;
  unsigned char* const xring = smem;
  unsigned char* const wring = smem + kX2Stages * kTileX;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kX2Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 5);
    }
    for (int s = 0; s < kW2Stages; ++s) {
      mbar_init(&wfull[s], 2);   // one expect_tx arrival per CTA
      mbar_init(&wempty[s], 1);
    }
    for (int a = 0; a < kA2Slots; ++a) {
      mbar_init(&a_full[a], 8);
      mbar_init(&a_empty[a], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();  // barriers of both CTAs initialised before any remote arrival
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = tmem_base_slot;

  if (warp == 0) {
    // ---------------- TMA producer: this CTA's 128 X rows of each pair tile ----------------
    uint32_t it = 0;
    for (int64_t pt = pair; pt < n_pt; pt += npairs) {
      const int row0 = (int)(pt * 2 * kMT + rank * kMT);
      for (int kc = 0; kc < kchunks; ++kc, ++it) {
        const int s = it % kX2Stages;
        OTF_WAIT_LOCAL(&empty[s], ((it / kX2Stages) & 1u) ^ 1u);
        tma_load_elect(xring + s * kTileX, &map_x, &full[s], kTileX, kc * kKC, row0);
      }
    }
  } else if (warp == 3) {
    // ---------------- TMA producer: this CTA's W half, bytes counted on the leader's barrier ------
    uint32_t it = 0;
    for (int64_t pt = pair; pt < n_pt; pt += npairs) {
      for (int kc = 0; kc < kchunks; ++kc, ++it) {
        const int s = it % kW2Stages;
        OTF_WAIT_LOCAL(&wempty[s], ((it / kW2Stages) & 1u) ^ 1u);
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%2], %3;\n\t"
            "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%4, %5}], [%2];\n\t}" ::"r"(smem_u32(wring + s * kTileW2)),
            "l"(&map_w), "r"(mapa_rank0(&wfull[s])), "r"((uint32_t)kTileW2), "r"(0),
            "r"((int)((kc * 2 + (int)rank) * kW2Rows))
            : "memory");
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA only) ----------------
    if (rank == 0) {
      constexpr uint32_t id128 = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((256u >> 4) << 24);
      constexpr uint32_t id64 = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((256u >> 4) << 24);
      const uint64_t wdesc0 = umma_desc_sw128(smem_u32(wring));
      const uint64_t xdesc0 = umma_desc_sw128(smem_u32(xring));
      uint32_t it = 0, j = 0;
      for (int64_t pt = pair; pt < n_pt; pt += npairs, ++j) {
        const int b = j & 1;
        mbar_wait_cl(&tmem_empty[b], ((j >> 1) & 1u) ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t acc = tmem_base + b * 128;
        for (int kc = 0; kc < kchunks; ++kc, ++it) {
          const int s = it % kW2Stages, sx = it % kX2Stages, a = it % kA2Slots;
          mbar_wait_cl(&wfull[s], (it / kW2Stages) & 1u);   // both W halves landed
          mbar_wait_cl(&a_full[a], (it / kA2Slots) & 1u);   // both CTAs: X landed, x_lo in TMEM
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint64_t wd = wdesc0 + (uint64_t)((s * kTileW2) >> 4);
          const uint64_t wd2 = wd + (uint64_t)((64 * 128) >> 4);  // rows 64..95: the w_hi half
          const uint64_t xd = xdesc0 + (uint64_t)((sx * kTileX) >> 4);
          const uint32_t alo = tmem_base + 256 + a * 32;
          asm volatile(
              "{\n\t.reg .pred e, p;\n\t"
              "elect.sync _|e, 0xffffffff;\n\t"
              "setp.ne.b32 p, %5, 0;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %2, %4, %6, p;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %8, %9, %6, 1;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %10, %11, %6, 1;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %12, %13, %6, 1;\n\t"
              "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%20], %23;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::tf32 [%1], [%3], %14, %7, 1;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::tf32 [%1], [%15], %16, %7, 1;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::tf32 [%1], [%17], %18, %7, 1;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::tf32 [%1], [%19], %24, %7, 1;\n\t"
              "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%21], %23;\n\t"
              "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%22], %23;\n\t}" ::"r"(acc),
              "r"(acc + 64), "l"(xd), "r"(alo), "l"(wd), "r"(kc), "r"(id128), "r"(id64),
              "l"(xd + 2), "l"(wd + 2), "l"(xd + 4), "l"(wd + 4), "l"(xd + 6), "l"(wd + 6),
              "l"(wd2), "r"(alo + 8), "l"(wd2 + 2), "r"(alo + 16), "l"(wd2 + 4), "r"(alo + 24),
              "r"(smem_u32(&empty[sx])), "r"(smem_u32(&wempty[s])), "r"(smem_u32(&a_empty[a])),
              "h"((unsigned short)3), "l"(wd2 + 6)
              : "memory");
        }
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
                smem_u32(&tmem_full[b])),
            "h"((unsigned short)3)
            : "memory");
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- epilogue: this CTA's 128 rows ----------------
    const int q = warp & 3;
    const uint32_t te = mapa_rank0(&tmem_empty[0]);
    uint32_t j = 0;
    for (int64_t pt = pair; pt < n_pt; pt += npairs, ++j) {
      const int b = j & 1;
      OTF_WAIT_LOCAL(&tmem_full[b], (j >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int64_t row = pt * 2 * kMT + rank * kMT + 32 * q + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + b * 128;
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 16) {
        uint32_t h[16], l[16];
        tmem_ld16(taddr + c0, h);
        tmem_ld16(taddr + 64 + c0, l);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < n) {
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int c = c0 + t;
            if (c < n_cls) out[(int64_t)c * n + row] = __fadd_rn(__uint_as_float(h[t]), __uint_as_float(l[t]));
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(te + b * 8);
    }
  } else if (warp >= 8) {
    // ---------------- split: x_lo of row r into this CTA's TMEM slot ----------------
    const int q = warp & 3;
    const uint32_t par = (uint32_t)((warp - 8) >> 2);
    const int r = 32 * q + lane;
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    const uint32_t af = mapa_rank0(&a_full[0]);
    uint32_t it = 0;
    for (int64_t pt = pair; pt < n_pt; pt += npairs) {
      for (int kc = 0; kc < kchunks; ++kc, ++it) {
        if ((it & 1u) != par) continue;
        const int s = it % kX2Stages, a = it % kA2Slots;
        OTF_WAIT_LOCAL(&full[s], (it / kX2Stages) & 1u);
        const unsigned char* rowp = xring + s * kTileX + r * 128;
        uint32_t lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 v = *reinterpret_cast<const float4*>(rowp + ((c ^ (r & 7)) << 4));
          const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int t = 0; t < 4; ++t)
            lo[4 * c + t] = __float_as_uint(__fsub_rn(e[t], __uint_as_float(__float_as_uint(e[t]) & 0xFFFFE000u)));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        OTF_WAIT_LOCAL(&a_empty[a], ((it / kA2Slots) & 1u) ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;");
        tmem_st32(tmem_base + lane_off + 256 + a * 32, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(af + a * 8);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();  // no remote arrival or pair MMA may target a CTA that has left
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

// W (n_cls x d float64) -> the CTA-pair layout: per chunk kc and CTA rank r a 96-row tile
//   r = 0: rows 0..63 = w_hi[0..63],  rows 64..95 = w_hi[0..31]
//   r = 1: rows 0..63 = w_lo[0..63],  rows 64..95 = w_hi[32..63]
// stored [kc][r][96][32] (each tile one contiguous 12 KB block).
__global__ void split_w2_kernel(const double* __restrict__ W, int n_cls, int d, float* __restrict__ ws) {
  const int64_t total = (int64_t)64 * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / d), k = (int)(e % d);
    const float w = c < n_cls ? __double2float_rn(W[e]) : 0.0f;
    const float hi = __uint_as_float(__float_as_uint(w) & 0xFFFFE000u);
    const int64_t t0 = (int64_t)(k / kKC) * 2 * kW2Rows * kKC + (k % kKC);  // rank-0 tile of chunk
    const int64_t t1 = t0 + (int64_t)kW2Rows * kKC;                          // rank-1 tile
    ws[t0 + (int64_t)c * kKC] = hi;
    ws[t1 + (int64_t)c * kKC] = __fsub_rn(w, hi);
    if (c < 32) ws[t0 + (int64_t)(64 + c) * kKC] = hi;
    else ws[t1 + (int64_t)(32 + c) * kKC] = hi;
  }
}

// W (n_cls x d float64) -> stacked [tf32(w32); w32 - tf32(w32)] (128 x d float32, zero padded),
// stored pre-tiled: tile kc (K columns 32kc .. 32kc+31 of all 128 rows) is one contiguous 16 KB
// block, [kc][row][32], so every CTA's TMA of the shared W chunk reads 128 consecutive lines
// (a row-major W would put the chunk's lines 4·d bytes apart, all hot in the same L2 slices).
__global__ void split_w_kernel(const double* __restrict__ W, int n_cls, int d, float* __restrict__ ws) {
  const int64_t total = (int64_t)64 * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / d), k = (int)(e % d);
    const float w = c < n_cls ? __double2float_rn(W[e]) : 0.0f;
    const float hi = __uint_as_float(__float_as_uint(w) & 0xFFFFE000u);
    const int64_t base = ((int64_t)(k / kKC) * 128) * kKC + (k % kKC);
    ws[base + (int64_t)c * kKC] = hi;
    ws[base + (int64_t)(64 + c) * kKC] = __fsub_rn(w, hi);
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

static int make_map(CUtensorMap* m, const float* base, uint64_t inner, uint64_t outer, uint32_t box_outer) {
  auto enc = get_encode();
  if (!enc) return fail(OTF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {inner * sizeof(float)};
  const cuuint32_t box[2] = {kKC, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(OTF_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return OTF_OK;
}

bool multi_tc_supported(int d, const float* X) {
  return d % kKC == 0 && d >= kKC && (((uintptr_t)X) & 15) == 0;
}

// Scores n rows of X (n x d float32) under n_cls <= 64 classifiers W (n_cls x d float64) into
// out (n_cls x n float32, classifier-major). ws: 2*64*d float32 scratch for the split W.
int launch_multi_score(const float* X, int64_t n, int d, const double* W, int n_cls, float* ws, float* out,
                       int device, cudaStream_t st) {
  if (n <= 0) return OTF_OK;
  if (n_cls < 1 || n_cls > 64) return fail(OTF_ERR_CONFIG, "multi-classifier scoring takes 1..64 classifiers");
  if (!multi_tc_supported(d, X)) return fail(OTF_ERR_CONFIG, "multi-classifier scoring needs dim % 32 == 0");
  static const int mode = getenv("OTF_MULTI_MODE") ? atoi(getenv("OTF_MULTI_MODE")) : 0;
  const int64_t tiles = (n + kMT - 1) / kMT;
  const bool pair = tiles >= 2 && sm_count(device) >= 2 && !(mode & 256);
  CUtensorMap mx, mw;
  int rc = make_map(&mx, X, (uint64_t)d, (uint64_t)n, kMT);
  if (rc) return rc;
  if (pair) {
    split_w2_kernel<<<64, 256, 0, st>>>(W, n_cls, d, ws);
    OTF_LAUNCH_CHECK("split_w2_kernel");
    if ((rc = make_map(&mw, ws, (uint64_t)kKC, (uint64_t)(d / kKC) * 2 * kW2Rows, kW2Rows))) return rc;
    const size_t smem = (size_t)kRing2Bytes + 1024;
    static bool configured2[64] = {false};
    if (!configured2[device & 63]) {
      OTF_CUDA(cudaFuncSetAttribute((const void*)multi_score_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
      configured2[device & 63] = true;
    }
    const int64_t pts = (tiles + 1) / 2;
    int grid = sm_count(device) & ~1;
    if (2 * pts < grid) grid = (int)(2 * pts);
    multi_score_tc2<<<grid, kMultiThreads, smem, st>>>(mx, mw, n, d, n_cls, out);
    OTF_LAUNCH_CHECK("multi_score_tc2");
    return OTF_OK;
  }
  split_w_kernel<<<64, 256, 0, st>>>(W, n_cls, d, ws);
  OTF_LAUNCH_CHECK("split_w_kernel");
  if ((rc = make_map(&mw, ws, (uint64_t)kKC, (uint64_t)(d / kKC) * 128, 128))) return rc;
  const size_t smem = (size_t)kRingBytes + 1024;
  static bool configured[64] = {false};
  if (!configured[device & 63]) {
    OTF_CUDA(cudaFuncSetAttribute((const void*)multi_score_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured[device & 63] = true;
  }
  int grid = sm_count(device);
  if (tiles < grid) grid = (int)tiles;
  multi_score_tc<<<grid, kMultiThreads, smem, st>>>(mx, mw, n, d, n_cls, out, mode);
  OTF_LAUNCH_CHECK("multi_score_tc");
  return OTF_OK;
}

}  // namespace otf
