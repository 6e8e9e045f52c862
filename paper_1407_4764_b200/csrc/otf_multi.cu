// otf_multi.cu — K7: many classifiers at once (C5b): S = X · Wᵀ on the 5th-gen tensor cores.
//
// The reference scores one model per call (score_dense, ranker.py:63-69: float32 sgemv); C5b
// ranks the same repository under 64 classifiers, i.e. a skinny GEMM (N = 64) with 32 flop/B —
// float32 SIMT (~70 TFLOP/s) would be 3x slower than HBM, so it runs on tcgen05 in TF32 with a
// 3-product split for float32-level accuracy:
//     x·w ≈ x_hi·w_hi + x_hi·w_lo + x_lo·w_hi,   v_hi = tf32(v) (the MMA reads the top 19 bits),
//                                                 v_lo = v − v_hi (exact in float32).
// W (≤ 64 classifiers) is split once on the device into a stacked [w_hi; w_lo] (128 × d) matrix,
// so one N=128 MMA computes x_hi·w_hi (accumulator columns 0..63) and x_hi·w_lo (64..127), and a
// second N=64 MMA adds x_lo·w_hi into columns 64..127; the epilogue adds the two halves.
//
// Per CTA (one per SM, persistent over 128-row tiles), warp-specialised:
//   warp 0      TMA producer: X tile (128 rows × 32 floats, SWIZZLE_128B) + W tile per stage
//   warp 1      MMA issuer (one elected thread): 4 K-steps × (N=128 + N=64) tcgen05.mma per stage
//   warp 2      TMEM allocator (2 × 128 accumulator columns, double-buffered across tiles)
//   warps 4–7   epilogue: tcgen05.ld the accumulators, sum halves, store scores (classifier-major)
//   warps 8–11  split: x_lo = x − tf32(x) for each stage into a second shared-memory tile
// Every output row is computed by the same MMA sequence whatever its tile, so a row's scores do
// not depend on its position. Parity is a tolerance against the reference's float32 sgemv
// (DESIGN.md §Parity); ranking of each classifier is the exact top-k of these scores.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "otf_common.cuh"
#include "otf_internal.h"

namespace otf {

constexpr int kMT = 128;          // rows per tile (UMMA M)
constexpr int kKC = 32;           // K floats per stage (128 bytes = one swizzle row)
constexpr int kStages = 4;
constexpr int kTileX = kMT * kKC * 4;   // 16 KB
constexpr int kTileW = 128 * kKC * 4;   // 16 KB (stacked w_hi; w_lo)
constexpr int kStageBytes = 2 * kTileX + kTileW;
constexpr int kMultiThreads = 384;
constexpr int kTmemCols = 256;

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
__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(kMultiThreads, 1)
multi_score_tc(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
               int64_t n, int d, int n_cls, float* __restrict__ out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for the swizzled tiles
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full_tma[kStages], full_split[kStages], empty[kStages];
  __shared__ uint64_t tmem_full[2], tmem_empty[2];
  __shared__ uint32_t tmem_base_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_tiles = (n + kMT - 1) / kMT;
  const int kchunks = d / kKC;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_tma[s], 1);
      mbar_init(&full_split[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
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

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        for (int kc = 0; kc < kchunks; ++kc, ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1u;
          mbar_wait(&empty[s], ph ^ 1u);
          unsigned char* st = smem + s * kStageBytes;
          mbar_expect_tx(&full_tma[s], kTileX + kTileW);
          tma_load_2d(st, &map_x, &full_tma[s], kc * kKC, (int)(tile * kMT));
          tma_load_2d(st + 2 * kTileX, &map_w, &full_tma[s], kc * kKC, 0);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t id128 = idesc_tf32(128), id64 = idesc_tf32(64);
      uint32_t it = 0, j = 0;
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++j) {
        const int b = j & 1;
        mbar_wait(&tmem_empty[b], ((j >> 1) & 1u) ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t acc = tmem_base + b * 128;
        for (int kc = 0; kc < kchunks; ++kc, ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1u;
          mbar_wait(&full_tma[s], ph);
          mbar_wait(&full_split[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t xa = smem_u32(smem + s * kStageBytes);
          const uint32_t xl = xa + kTileX;
          const uint32_t wa = xa + 2 * kTileX;
#pragma unroll
          for (int k = 0; k < kKC / 8; ++k) {  // K = 8 tf32 = 32 bytes per MMA
            const uint32_t off = k * 32;
            umma_tf32(acc, umma_desc_sw128(xa + off), umma_desc_sw128(wa + off), id128,
                      (kc | k) != 0);
            umma_tf32(acc + 64, umma_desc_sw128(xl + off), umma_desc_sw128(wa + off), id64, 1u);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&tmem_full[b]);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- epilogue ----------------
    const int q = warp & 3;  // TMEM lanes 32q .. 32q+31
    uint32_t j = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++j) {
      const int b = j & 1;
      mbar_wait(&tmem_full[b], (j >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int64_t row = tile * kMT + 32 * q + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + b * 128;
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 16) {
        uint32_t h[16], l[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(h[0]), "=r"(h[1]), "=r"(h[2]), "=r"(h[3]), "=r"(h[4]), "=r"(h[5]), "=r"(h[6]),
              "=r"(h[7]), "=r"(h[8]), "=r"(h[9]), "=r"(h[10]), "=r"(h[11]), "=r"(h[12]), "=r"(h[13]),
              "=r"(h[14]), "=r"(h[15])
            : "r"(taddr + c0));
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(l[0]), "=r"(l[1]), "=r"(l[2]), "=r"(l[3]), "=r"(l[4]), "=r"(l[5]), "=r"(l[6]),
              "=r"(l[7]), "=r"(l[8]), "=r"(l[9]), "=r"(l[10]), "=r"(l[11]), "=r"(l[12]), "=r"(l[13]),
              "=r"(l[14]), "=r"(l[15])
            : "r"(taddr + 64 + c0));
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
      if (lane == 0) mbar_arrive(&tmem_empty[b]);
    }
  } else if (warp >= 8) {
    // ---------------- split: x_lo = x - tf32(x) ----------------
    const int t = threadIdx.x - 256;  // 0..127
    uint32_t it = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      for (int kc = 0; kc < kchunks; ++kc, ++it) {
        const int s = it % kStages;
        const uint32_t ph = (it / kStages) & 1u;
        mbar_wait(&full_tma[s], ph);
        // x_hi = x with the low 13 mantissa bits cleared (written back in place, so the tensor
        // core sees an exact TF32 value whether it truncates or rounds), x_lo = x - x_hi (exact).
        float4* hi = reinterpret_cast<float4*>(smem + s * kStageBytes);
        float4* dst = reinterpret_cast<float4*>(smem + s * kStageBytes + kTileX);
#pragma unroll
        for (int i = 0; i < kTileX / 16 / 128; ++i) {  // 8 float4 per thread
          const float4 v = hi[t + 128 * i];
          float4 h, lo;
          h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
          h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
          h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
          h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
          lo.x = __fsub_rn(v.x, h.x);
          lo.y = __fsub_rn(v.y, h.y);
          lo.z = __fsub_rn(v.z, h.z);
          lo.w = __fsub_rn(v.w, h.w);
          hi[t + 128 * i] = h;
          dst[t + 128 * i] = lo;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_split[s]);
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

// W (n_cls x d float64) -> stacked [tf32(w32); w32 - tf32(w32)] (128 x d float32), zero padded.
__global__ void split_w_kernel(const double* __restrict__ W, int n_cls, int d, float* __restrict__ ws) {
  const int64_t total = (int64_t)64 * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / d);
    const float w = c < n_cls ? __double2float_rn(W[e]) : 0.0f;
    const float hi = __uint_as_float(__float_as_uint(w) & 0xFFFFE000u);
    ws[e] = hi;
    ws[total + e] = __fsub_rn(w, hi);
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
  split_w_kernel<<<64, 256, 0, st>>>(W, n_cls, d, ws);
  OTF_LAUNCH_CHECK("split_w_kernel");
  CUtensorMap mx, mw;
  int rc = make_map(&mx, X, (uint64_t)d, (uint64_t)n, kMT);
  if (!rc) rc = make_map(&mw, ws, (uint64_t)d, 128, 128);
  if (rc) return rc;
  const size_t smem = (size_t)kStages * kStageBytes + 1024;
  static bool configured[64] = {false};
  if (!configured[device & 63]) {
    OTF_CUDA(cudaFuncSetAttribute((const void*)multi_score_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured[device & 63] = true;
  }
  const int64_t tiles = (n + kMT - 1) / kMT;
  int grid = sm_count(device);
  if (tiles < grid) grid = (int)tiles;
  multi_score_tc<<<grid, kMultiThreads, smem, st>>>(mx, mw, n, d, n_cls, out);
  OTF_LAUNCH_CHECK("multi_score_tc");
  return OTF_OK;
}

}  // namespace otf
