// otf_internal.h — internal launchers shared between the .cu translation units.
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include "otf_b200.h"

namespace otf {

// RAII device selection
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// NVTX ranges around the public entry points (nvtx3 is header-only: a no-op unless a profiler
// such as Nsight Systems injects itself), so a timeline shows which library call each kernel,
// copy and synchronisation belongs to.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define OTF_NVTX(name) ::otf::NvtxRange _otf_nvtx_range(name)

// SMs the persistent rank kernels size their grids for (all but the reserved ones)
int rank_sms(int device);
int reserved_sms(int device);

// a handle created over a borrowed device payload takes ownership of it (file loaders)
void repo_own_payload(otf_repo* r);

// Scoring launchers take the float64 model on the device and (optionally) a kHistBins-entry
// histogram (zero on entry) that receives the coarse score histogram for launch_topk.

// dense (otf_dense.cu)
// cmax (nullable): per-chunk maximum score bins for the top-k gather; *clog is set to log2 of
// the chunk size when the kernel wrote them, else left at -1.
// claim (nullable): 10 zeroed words; the last quarter of the rows is then handed out dynamically
// (dense_score_fast), and the words are left zero
int launch_dense_score(const float* X, int64_t n, int32_t d, const double* w, float* out,
                       uint32_t* hist, int device, cudaStream_t st, uint16_t* cmax = nullptr,
                       int* clog = nullptr, unsigned int* claim = nullptr);

// fused dense rank (score + exact top-k, one cooperative launch; otf_dense.cu dense_rank_cut).
// dense_cut_plan returns false when the path does not apply (unaligned / unsupported d, large k,
// a repository too small for the sample); then score + launch_topk run as before.
struct TopkWs;
struct DenseCutPlan {
  int grid = 0;  // CTAs (all co-resident)
  int sit = 0;   // sample groups per warp
  int r = 0;     // sample rank of the threshold
};
bool dense_cut_plan(int32_t d, const float* X, int64_t n, int64_t k_eff, int device, DenseCutPlan* pl);
int launch_dense_rank_cut(const float* X, int64_t n, int32_t d, const double* w, const int64_t* ids,
                          int64_t id_base, int64_t k_eff, const DenseCutPlan& pl, TopkWs* ws, float* scratch,
                          int64_t* out_ids, double* out_scores, int64_t* out_rows, cudaStream_t st);

// pq (otf_pq.cu)
int launch_pq_lut(const float* cents, int M, int K, int Q, const double* w, double* lut,
                  cudaStream_t st, int replicas = 1);
constexpr int kCutLutReplicas = 8;  // LUT copies the cut path's CTAs spread their reads over
// pq_encode (pq.py:206-230): X (n, M*Q) f32, cents (M,K,Q) f32 -> codes (n, M) u8.
size_t pq_encode_scratch_bytes(int M, int K);
int launch_pq_encode(const float* X, int64_t n, int M, int K, int Q, const float* cents, void* scratch,
                     uint8_t* codes, int device, cudaStream_t st);
int launch_pq_check(const uint8_t* codes, int64_t total, int K, unsigned int* bad, int device,
                    cudaStream_t st);
bool pq_fast_path(int M, const uint8_t* codes);
// M == 16 fast path can emit 16-bit score bins instead of float64 scores (rank path).
bool pq_bins_path(int M, const uint8_t* codes);
int launch_pq_scan_bins(const uint8_t* codes, int64_t n, const double* lut, int K, uint16_t* bins,
                        uint32_t* hist, int device, cudaStream_t st, uint16_t* cmax = nullptr,
                        int* clog = nullptr);
// fast path builds the LUT in-kernel from (cents, w); the generic path reads `lut`.
int launch_pq_scan(const uint8_t* codes, int64_t n, int M, const float* cents, const double* w,
                   const double* lut, int K, int Q, double* out, uint32_t* hist, int device,
                   cudaStream_t st);

// binary (otf_binary.cu)
// byte-table fast path for rows of whole 128-byte slices; needs `scratch` (n doubles) when a
// row has more than one slice (> 1024 bits); otherwise the generic kernel runs.
bool bin_bytes_path(int n_bits, const uint8_t* codes);
int launch_bin_score(const uint8_t* codes, int64_t n, int n_bits, const double* w, float* out,
                     uint32_t* hist, double* scratch, int device, cudaStream_t st,
                     uint16_t* cmax = nullptr, int* clog = nullptr);
int launch_bin_unpack(const uint8_t* codes, int64_t n, int n_bits, float* out, int device,
                      cudaStream_t st);
int launch_binarize(const double* U, const float* mu, int m, int n_bits, const double* X,
                    int64_t n, uint8_t* out, int device, cudaStream_t st);
int launch_hamming(const uint8_t* a, const uint8_t* b, int64_t n, int width, int64_t* out,
                   int device, cudaStream_t st);

// top-k (otf_topk.cu)
struct TopkWs {
  uint32_t* hist = nullptr;       // kHistBins coarse histogram (zero between calls)
  uint32_t* rhist = nullptr;      // 3 x 256 rotating radix histograms (zero between calls)
  unsigned int* bar = nullptr;    // grid barrier {count, generation}
  unsigned int* count = nullptr;  // candidate counter (zero between calls)
  uint64_t* key = nullptr;        // candidate order keys      (cap entries)
  uint64_t* inv = nullptr;        // candidate ~id             (cap entries)
  int64_t* row = nullptr;         // candidate row             (cap entries)
  int64_t cap = 0;                // power of two >= max(k_eff, kCandCap), per segment
  int n_seg = 0;                  // segments the counters are laid out for
  size_t slots = 0;               // allocated candidate slots (n_seg * cap)
  // chunk maxima (optional, single segment): cmax[c] = max bin of rows [c << clog, (c+1) << clog),
  // written by the scoring kernel of the same query; clog < 0: not available
  uint16_t* cmax = nullptr;
  size_t cmax_cap = 0;
  int clog = -1;
  // PQ cut path (pq_scan16_cut -> topk_cut_kernel): the scan appends only the rows that can
  // reach a sampled threshold. cut_word[0] = candidate count, [1] = the threshold's bin (both
  // zero between calls); cut_smax: per-CTA sample maxima of the LUT/sample kernel.
  uint64_t* cut_key = nullptr;    // (exact score order key, ~id) record per candidate (2 x cut_cap)
  int64_t* cut_row = nullptr;     // row of each candidate
  unsigned int* cut_word = nullptr;
  uint32_t* cut_smax = nullptr;   // kCutSmaxCap entries (two sample maxima per CTA / warp)
  int64_t cut_cap = 0;
};
// candidate slots of the PQ cut path (16 B each); more candidates -> exact fallback
constexpr int64_t kCutCap = 1 << 16;
constexpr int kCutSampleCtasMax = 1024;
constexpr int kCutSmaxCap = 16384;
// cut_word: [0..15] the fused selections' counters and barrier words, [16..25] the dynamic tail
// of dense_score_fast (launch_dense_score's claim), [64 + 32 c] dense_rank_cut's tail counter c
// (one 128-byte line each, c < 16), all zero between launches
constexpr int kCutWords = 64 + 16 * 32;
constexpr int kCutClaimWord = 16;
int topk_cut_alloc(TopkWs* ws);
// ensures ws->cmax holds the chunk maxima of n rows for chunks of >= 8 rows (zero padded)
int topk_cmax_ensure(TopkWs* ws, int64_t n);
int topk_ws_alloc(TopkWs* ws, int64_t k_eff, int n_seg = 1);
void topk_ws_free(TopkWs* ws);
// scores: float32 (dtype 0) or float64 (dtype 1), n entries on device. If hist_ready, ws->hist
// already holds the coarse histogram of these scores (fused into the scoring kernel).
int launch_topk(const void* scores, int dtype, int64_t n, const int64_t* ids, int64_t id_base,
                int64_t k_eff, TopkWs* ws, bool hist_ready, int64_t* out_ids, double* out_scores,
                int64_t* out_rows, int device, cudaStream_t st);
// PQ rank path: per-row bins (+ fused histogram) from launch_pq_scan_bins; exact float64 scores
// of candidates recomputed from codes + lut. scratch: n float64 (used only on the rare path).
// n_seg independent top-k selections over consecutive float32 score arrays (scores + s*n) in one
// cooperative launch (gridDim.x / n_seg CTAs each); outputs at out_ids/out_scores + s*k_eff.
// The same selections by a sampled threshold per segment (otf_topk.cu topk_seg_cut_kernel): one
// pass over the scores instead of a histogram pass and a gather pass; the plan returns false when
// it does not apply (> 64 segments, small n, large k).
bool topk_seg_cut_plan(int n_seg, int64_t n, int64_t k_eff, int device, int* r);
int launch_topk_seg_cut(const float* scores, int n_seg, int64_t n, const int64_t* ids, int64_t id_base, int64_t k_eff,
                        int r, TopkWs* ws, int64_t* out_ids, double* out_scores, int device, cudaStream_t st);
int launch_topk_segments(const float* scores, int n_seg, int64_t n, const int64_t* ids, int64_t id_base,
                         int64_t k_eff, TopkWs* ws, int64_t* out_ids, double* out_scores, int device,
                         cudaStream_t st);
// PQ cut path (M == 16, large n): a sample kernel (the float64 LUT and its replicas in `lut`,
// a sampled threshold), then one cooperative kernel that streams the codes emitting only the
// rows that reach the threshold and selects the exact top-k among them (or falls back to an
// exact select over every row); see otf_pq.cu pq_rank_cut_kernel. pq_cut_plan returns r (the
// sample rank of the threshold) or false when the path does not apply (small n or large k).
bool pq_cut_plan(int M, const uint8_t* codes, int64_t n, int64_t k_eff, int device, int* r);
int launch_pq_rank_cut(const float* cents, int K, int Q, const double* w, double* lut, const uint8_t* codes,
                       int64_t n, const int64_t* ids, int64_t id_base, int64_t k_eff, int r, TopkWs* ws,
                       double* scratch, int64_t* out_ids, double* out_scores, int64_t* out_rows, int device,
                       cudaStream_t st);
int launch_topk_pq_bins(const uint16_t* bins, const uint8_t* codes, int M, const double* lut, int K,
                        int64_t n, const int64_t* ids, int64_t id_base, int64_t k_eff, TopkWs* ws,
                        double* scratch, int64_t* out_ids, double* out_scores, int64_t* out_rows,
                        int device, cudaStream_t st);

// Pegasos (otf_train.cu)
int launch_pegasos(double* w, int d, const void* pos, int pos_dtype, int64_t n_pos,
                   const void* neg, int neg_dtype, int64_t n_neg, const int64_t* pos_idx,
                   const int64_t* neg_idx, int half, double shrink, double eta_over_b,
                   int project, double radius, cudaStream_t st);

// fixed-set training (otf_batch.cu); X: (n, d) float32/float64, rows < n_pos labelled +1
int launch_batch_train(const void* X, int dt, int64_t n_pos, int64_t n, int d, const int64_t* idx,
                       int64_t total, int bs, int64_t spe, int64_t tail_start, int64_t tail_len,
                       double lam, int project, double* w_out, double* obj_hist, cudaStream_t st);
int launch_hinge_objective(const void* X, int dt, int64_t n_pos, int64_t n, int d, const double* w,
                           double lam, double* out, cudaStream_t st);

// k-means (otf_kmeans.cu)
int kmeans_row_norms(const double* X, int64_t n, int Q, double* xx, cudaStream_t st);
int kmeans_step(const double* X, const double* xx, int64_t n, int Q, int K, double* C, double* cc, int32_t* assign,
                double* best, unsigned long long* counts, double* objective, int device, cudaStream_t st);

// multi-GPU group (otf_group.cu)
int group_unique_id(unsigned char* out128);
int group_comm_create(int n_ranks, int rank, const unsigned char* id128, void** comm);
void group_comm_destroy(void* comm);
int group_broadcast_f64(void* comm, double* buf, int64_t n, int root, cudaStream_t st);
int group_allgather_candidates(void* comm, const double* sc, const int64_t* ids, const int64_t* rows, int64_t k,
                               double* sc_all, int64_t* ids_all, int64_t* rows_all, cudaStream_t st);
int launch_group_finalize(double* sc, int64_t* ids, int64_t* rows, int64_t k_loc, int64_t k, int64_t row_offset,
                          int64_t pad_base, cudaStream_t st);

// misc
int launch_gather_rows(const uint8_t* src, int64_t row_bytes, const int64_t* rows, int64_t n,
                       uint8_t* dst, int device, cudaStream_t st);
int launch_gather_i64(const int64_t* src, const int64_t* rows, int64_t n, int64_t base_if_null,
                      int64_t* dst, cudaStream_t st);

}  // namespace otf

namespace otf {
// many classifiers (otf_multi.cu): tcgen05 TF32x3 scoring, out (n_cls x n float32)
bool multi_tc_supported(int d, const float* X);
// float32 scratch launch_multi_score needs for the split, pre-tiled classifier matrix
inline size_t multi_ws_floats(int d) { return (size_t)3 * 64 * (size_t)d + 64; }
// x_exp: the data scale exponent from multi_x_exponent (INT_MIN: TF32x3 form), see otf_multi.cu
int launch_multi_score(const float* X, int64_t n, int d, const double* W, int n_cls, float* ws, float* out,
                       int device, cudaStream_t st, int x_exp);
// one pass over X (synchronises st): ex with max|x| 2^ex in [2^14, 2^15), or INT_MIN if X holds
// inf/NaN or an extreme magnitude
int multi_x_exponent(const float* X, int64_t n, int d, int device, cudaStream_t st, int* ex);
}  // namespace otf
