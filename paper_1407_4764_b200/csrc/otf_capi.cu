// otf_capi.cu — the extern "C" boundary (include/otf_b200.h): handles, memory ownership,
// host<->device staging, error mapping. All compute is in the kernels of the other units.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "otf_b200.h"
#include "otf_common.cuh"
#include "otf_internal.h"

namespace otf {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  return OTF_ERR_CUDA;
}
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int sm_count(int device) {
  static int cache[64] = {0};
  int d = device & 63;
  if (cache[d] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    cache[d] = v > 0 ? v : 1;
  }
  return cache[d];
}


// SMs the persistent rank kernels may use: all but `reserved` (otf_set_reserved_sms), so a
// concurrent trainer's CTA always finds a free SM
static std::atomic<int> g_reserved[64];
int rank_sms(int device) {
  const int n = sm_count(device) - g_reserved[device & 63].load(std::memory_order_relaxed);
  return n > 1 ? n : 1;
}
int reserved_sms(int device) { return g_reserved[device & 63].load(std::memory_order_relaxed); }

// Simple device/pinned buffers ---------------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t b) {
    if (b <= bytes && p) return OTF_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (b == 0) return OTF_OK;
    cudaError_t e = cudaMalloc(&p, b);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    bytes = b;
    return OTF_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};
struct HostBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t b) {
    if (b <= bytes && p) return OTF_OK;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    if (b == 0) return OTF_OK;
    cudaError_t e = cudaMallocHost(&p, b);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocHost");
    bytes = b;
    return OTF_OK;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
  }
};

}  // namespace otf

using namespace otf;



struct otf_repo {
  int device = 0;
  int kind = OTF_KIND_DENSE;
  int64_t n = 0;
  int32_t model_dim = 0;   // d (dense), M*Q (pq), n_bits (binary)
  int32_t M = 0, K = 0, Q = 0;
  int64_t row_bytes = 0;
  const void* payload = nullptr;  // device
  bool owns_payload = false;
  int64_t* ids = nullptr;          // device, nullable
  int64_t id_base = 0;
  float* cents = nullptr;          // pq centroids (device)
  cudaStream_t stream = nullptr;
  std::mutex mu;                   // one call at a time per handle
  DevBuf w, w32, lut, scores, bins, outbuf, multi;  // multi: (<=64, n) float32 classifier scores
  DevBuf wpub;  // the ranker's copy of the trainer's w (otf_trainer_publish)
  HostBuf h_w, h_out;
  TopkWs topk;
  TopkWs mtopk;  // segment workspace of rank_many (kept apart: graphs capture topk's pointers)
  bool x_exp_ready = false;  // the FP16 data scale of score_many (dense payload is immutable)
  int x_exp = 0;
  // graph cache for otf_repo_rank_graph
  // cached CUDA graphs of rank (otf_repo_rank_graph and host-memory otf_repo_rank): keyed by k
  // and EVERY pointer a replay touches (w, outputs, stream and the handle's workspaces), so a
  // workspace that grew (e.g. a larger k) can never be replayed through a stale graph
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    const void* key[16] = {};
    int64_t k = -1;
    int kernels = 0;  // kernels in the graph (launch accounting of each replay)
    int reserved = 0;  // reserved SMs when captured (grid sizes depend on it)
    uint64_t used = 0;
  };
  std::vector<GraphEntry> graphs;  // <= kGraphCache entries, least recently used replaced
  uint64_t graph_clock = 0;
  // Cross-stream ordering of the handle's workspaces (scores, bins, lut, histogram, barrier word,
  // candidate slots): every call records `last` on the stream it used, and a call on a different
  // stream waits for it first, so two calls on two streams never share a workspace on the GPU.
  cudaEvent_t last = nullptr;
  cudaStream_t last_stream = nullptr;
  bool used = false;
};

struct otf_trainer {
  int device = 0;
  int32_t dim = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  DevBuf w, neg, pos_pool, pos_stage, idx;
  HostBuf h_stage, h_idx;
  int neg_dtype = OTF_F32;
  int64_t n_neg = 0;
  int64_t n_pos = 0, pos_cap = 0;
  DevBuf wsnap;                     // the published snapshot of w (otf_trainer_publish)
  cudaEvent_t published = nullptr;  // recorded after each snapshot copy (otf_trainer_publish)
  cudaEvent_t consumed = nullptr;   // recorded after a ranker copied wsnap (otf_repo_rank_published)
};

namespace {

cudaStream_t pick_stream(cudaStream_t own, void* user) {
  (void)own;  // device-memory calls run on the caller's stream (NULL = legacy default stream)
  return static_cast<cudaStream_t>(user);
}

// Orders a call on stream st after the handle's previous call (whatever stream that used).
int repo_enter(otf_repo* r, cudaStream_t st) {
  if (r->used && r->last_stream != st) OTF_CUDA(cudaStreamWaitEvent(st, r->last, 0));
  return OTF_OK;
}
// Records the end of this call's work on st (the next call on another stream waits for it).
int repo_leave(otf_repo* r, cudaStream_t st) {
  if (!r->last) OTF_CUDA(cudaEventCreateWithFlags(&r->last, cudaEventDisableTiming));
  OTF_CUDA(cudaEventRecord(r->last, st));
  r->last_stream = st;
  r->used = true;
  return OTF_OK;
}
// enter + body + leave (leave runs even when the body failed after enqueueing work)
template <typename F>
int repo_ordered(otf_repo* r, cudaStream_t st, F&& body) {
  int rc = repo_enter(r, st);
  if (rc) return rc;
  rc = body();
  const int rc2 = repo_leave(r, st);
  return rc ? rc : rc2;
}

int make_stream(cudaStream_t* s, bool high_priority) {
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  OTF_CUDA(cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, high_priority ? hi : lo));
  return OTF_OK;
}

int copy_in(void* dst, const void* src, size_t bytes, int mem, cudaStream_t st) {
  if (bytes == 0) return OTF_OK;
  OTF_CUDA(cudaMemcpyAsync(dst, src, bytes,
                           mem == OTF_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                           st));
  return OTF_OK;
}

int repo_common(otf_repo* r, int device, int64_t n, const int64_t* ids, int64_t id_base,
                int mem) {
  r->device = device;
  r->n = n;
  r->id_base = id_base;
  int rc = make_stream(&r->stream, false);
  if (rc) return rc;
  if (ids) {
    // ids may be host or device memory whatever `mem` says of the payload (from_device adopts a
    // device payload with host ids): the pointer decides
    cudaPointerAttributes pa;
    const bool dev_ids = cudaPointerGetAttributes(&pa, ids) == cudaSuccess &&
                         (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged);
    cudaGetLastError();  // clear a failed query
    const int ids_mem = dev_ids ? OTF_MEM_DEVICE : OTF_MEM_HOST;
    OTF_CUDA(cudaMalloc(&r->ids, (size_t)(n > 0 ? n : 1) * sizeof(int64_t)));
    rc = copy_in(r->ids, ids, (size_t)n * sizeof(int64_t), ids_mem, r->stream);
    if (rc) return rc;
  }
  return OTF_OK;
}

int take_payload(otf_repo* r, const void* data, size_t bytes, int mem, int borrow) {
  // a device payload may still be being written by the caller's work on any stream (e.g. torch's
  // legacy default stream, which the handle's non-blocking stream does not wait for): finish it
  if (mem == OTF_MEM_DEVICE) OTF_CUDA(cudaDeviceSynchronize());
  if (mem == OTF_MEM_DEVICE && borrow) {
    r->payload = data;
    r->owns_payload = false;
    return OTF_OK;
  }
  void* p = nullptr;
  OTF_CUDA(cudaMalloc(&p, bytes > 0 ? bytes : 16));
  r->payload = p;
  r->owns_payload = true;
  return copy_in(p, data, bytes, mem, r->stream);
}

}  // namespace
void otf::repo_own_payload(otf_repo* r) { r->owns_payload = true; }
namespace {
void repo_free(otf_repo* r) {
  if (!r) return;
  DeviceGuard g(r->device);
  if (r->stream) cudaStreamSynchronize(r->stream);
  for (auto& ge : r->graphs)
    if (ge.exec) cudaGraphExecDestroy(ge.exec);
  if (r->owns_payload && r->payload) cudaFree(const_cast<void*>(r->payload));
  if (r->ids) cudaFree(r->ids);
  if (r->cents) cudaFree(r->cents);
  if (r->last) cudaEventDestroy(r->last);
  r->w.release(); r->w32.release(); r->lut.release(); r->scores.release(); r->bins.release(); r->outbuf.release();
  r->multi.release(); r->wpub.release();
  r->h_w.release(); r->h_out.release();
  topk_ws_free(&r->topk);
  topk_ws_free(&r->mtopk);
  if (r->stream) cudaStreamDestroy(r->stream);
  delete r;
}

// Uploads w (host or device) into r->w; returns device pointer.
int stage_w(otf_repo* r, const double* w, int mem, cudaStream_t st, const double** dw) {
  const size_t bytes = (size_t)r->model_dim * sizeof(double);
  if (mem == OTF_MEM_DEVICE) {
    *dw = w;
    return OTF_OK;
  }
  int rc = r->w.ensure(bytes);
  if (rc) return rc;
  rc = r->h_w.ensure(bytes);
  if (rc) return rc;
  std::memcpy(r->h_w.p, w, bytes);
  OTF_CUDA(cudaMemcpyAsync(r->w.p, r->h_w.p, bytes, cudaMemcpyHostToDevice, st));
  *dw = static_cast<const double*>(r->w.p);
  return OTF_OK;
}

// Scores every row of r into `out` (device). hist (nullable) receives the coarse histogram.
int score_into(otf_repo* r, const double* dw, void* out, uint32_t* hist, cudaStream_t st,
               uint16_t* cmax = nullptr, int* clog = nullptr) {
  int rc = OTF_OK;
  if (r->kind == OTF_KIND_DENSE) {
    // the rank path (hist) hands the scan's tail out dynamically (counters in the cut words)
    unsigned int* claim = nullptr;
    if (hist) {
      if ((rc = topk_cut_alloc(&r->topk))) return rc;
      claim = r->topk.cut_word + kCutClaimWord;
    }
    return launch_dense_score(static_cast<const float*>(r->payload), r->n, r->model_dim, dw,
                              static_cast<float*>(out), hist, r->device, st, cmax, clog, claim);
  }
  if (r->kind == OTF_KIND_PQ) {
    // the (M, K) float64 LUT is built once per query (one thread per entry), then every scan
    // CTA copies it into shared memory instead of re-deriving it
    const uint8_t* codes = static_cast<const uint8_t*>(r->payload);
    if ((rc = r->lut.ensure((size_t)r->M * r->K * sizeof(double)))) return rc;
    if ((rc = launch_pq_lut(r->cents, r->M, r->K, r->Q, dw, static_cast<double*>(r->lut.p), st)))
      return rc;
    return launch_pq_scan(codes, r->n, r->M, nullptr, nullptr, static_cast<const double*>(r->lut.p),
                          r->K, r->Q, static_cast<double*>(out), hist, r->device, st);
  }
  // multi-slice byte-table path chains a float64 partial per row
  if ((rc = r->bins.ensure((size_t)(r->n > 0 ? r->n : 1) * sizeof(double)))) return rc;
  // (a dynamic tail as the dense scans' measured no faster here: the byte-table scan is LSU-bound,
  // not unbalanced — C5a 5.94-5.99 vs 5.91-5.97 ms on the same box)
  return launch_bin_score(static_cast<const uint8_t*>(r->payload), r->n, r->model_dim, dw,
                          static_cast<float*>(out), hist, static_cast<double*>(r->bins.p), r->device,
                          st, cmax, clog);
}

int score_dtype(const otf_repo* r) { return r->kind == OTF_KIND_PQ ? OTF_F64 : OTF_F32; }

// One query on device: scoring kernel (+ fused histogram) then the top-k kernel.
int rank_device(otf_repo* r, const double* dw, int64_t k_eff, int64_t* ids, double* scores,
                int64_t* rows, cudaStream_t st) {
  const size_t es = score_dtype(r) == OTF_F64 ? 8 : 4;
  int rc = r->scores.ensure((size_t)(r->n > 0 ? r->n : 1) * es);
  if (rc) return rc;
  if ((rc = topk_ws_alloc(&r->topk, k_eff))) return rc;
  const uint8_t* codes = static_cast<const uint8_t*>(r->payload);
  int cut_r = 0;
  if (r->kind == OTF_KIND_PQ && pq_cut_plan(r->M, codes, r->n, k_eff, r->device, &cut_r)) {
    // PQ cut path: the sample kernel (LUT + sampled threshold), then one cooperative kernel that
    // streams the codes emitting only the rows that reach the threshold and selects among them
    if ((rc = r->lut.ensure((size_t)r->M * r->K * sizeof(double) * kCutLutReplicas))) return rc;
    if ((rc = topk_cut_alloc(&r->topk))) return rc;
    return launch_pq_rank_cut(r->cents, r->K, r->Q, dw, static_cast<double*>(r->lut.p), codes, r->n, r->ids,
                              r->id_base, k_eff, cut_r, &r->topk, static_cast<double*>(r->scores.p), ids, scores, rows,
                              r->device, st);
  }
  if (r->kind == OTF_KIND_PQ && pq_bins_path(r->M, codes)) {
    // PQ: the scan writes 2-byte bins, the top-k recomputes the candidates' exact scores
    if ((rc = r->bins.ensure((size_t)(r->n > 0 ? r->n : 1) * sizeof(uint16_t)))) return rc;
    if ((rc = r->lut.ensure((size_t)r->M * r->K * sizeof(double)))) return rc;
    if ((rc = launch_pq_lut(r->cents, r->M, r->K, r->Q, dw, static_cast<double*>(r->lut.p), st)))
      return rc;
    if ((rc = topk_cmax_ensure(&r->topk, r->n))) return rc;
    int clog = -1;
    if ((rc = launch_pq_scan_bins(codes, r->n, static_cast<const double*>(r->lut.p), r->K,
                                  static_cast<uint16_t*>(r->bins.p), r->topk.hist, r->device, st,
                                  r->topk.cmax, &clog)))
      return rc;
    r->topk.clog = clog;
    rc = launch_topk_pq_bins(static_cast<const uint16_t*>(r->bins.p), codes, r->M,
                             static_cast<const double*>(r->lut.p), r->K, r->n, r->ids, r->id_base,
                             k_eff, &r->topk, static_cast<double*>(r->scores.p), ids, scores, rows,
                             r->device, st);
    r->topk.clog = -1;
    return rc;
  }
  DenseCutPlan dpl;
  if (r->kind == OTF_KIND_DENSE && k_eff < r->n &&
      dense_cut_plan(r->model_dim, static_cast<const float*>(r->payload), r->n, k_eff, r->device, &dpl)) {
    // dense cut path: one cooperative kernel scores, samples a threshold, emits the rows that
    // reach it and selects the exact top-k among them (otf_dense.cu dense_rank_cut)
    if ((rc = topk_cut_alloc(&r->topk))) return rc;
    return launch_dense_rank_cut(static_cast<const float*>(r->payload), r->n, r->model_dim, dw, r->ids, r->id_base,
                                 k_eff, dpl, &r->topk, static_cast<float*>(r->scores.p), ids, scores, rows, st);
  }
  const bool fuse = k_eff < r->n;
  int clog = -1;
  if (fuse && (rc = topk_cmax_ensure(&r->topk, r->n))) return rc;
  if ((rc = score_into(r, dw, r->scores.p, fuse ? r->topk.hist : nullptr, st, fuse ? r->topk.cmax : nullptr,
                       &clog)))
    return rc;
  r->topk.clog = clog;
  rc = launch_topk(r->scores.p, score_dtype(r), r->n, r->ids, r->id_base, k_eff, &r->topk, fuse, ids, scores,
                   rows, r->device, st);
  r->topk.clog = -1;
  return rc;
}

}  // namespace

extern "C" {

const char* otf_last_error(void) { return g_last_error.c_str(); }
int otf_abi_version(void) { return 1; }
int64_t otf_launch_count(void) { return g_launches.load(); }

const char* otf_kernel_names(void) {
  return "dense_score_fast;dense_score_generic;pq_build_lut_kernel;pq_scan_fast;pq_scan16_xor;"
         "pq_scan_generic;pq_scan16_f32bins;pq_encode_mma;pq_check_codes;bin_score_bytes;bin_score_generic;bin_unpack;bin_binarize;"
         "bin_hamming;split_w_half_kernel;absmax_kernel;topk_coop_kernel;pegasos_kernel;batch_train_kernel;hinge_objective_kernel;"
         "split_w_kernel;multi_score_tc;gather_rows_kernel;gather_i64_kernel;group_finalize_local;pq_rank_cut_kernel;dense_rank_cut;"
         "km_sqnorms;km_assign;km_objective;km_means;pq_cent_norms_kernel;pq_block_bounds_kernel;pq_encode_kernel";
}

int otf_set_reserved_sms(int device, int32_t n) {
  if (n < 0 || n >= sm_count(device)) return fail(OTF_ERR_CONFIG, "reserved SMs must be in [0, SM count)");
  g_reserved[device & 63].store(n, std::memory_order_relaxed);
  return OTF_OK;
}

int otf_device_count(int* out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *out = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  *out = n;
  return OTF_OK;
}

int otf_repo_create_dense(int device, const float* data, int64_t n, int32_t dim,
                          const int64_t* ids, int64_t id_base, int mem, int borrow,
                          otf_repo** out) {
  *out = nullptr;
  if (dim <= 0 || n < 0) return fail(OTF_ERR_CONFIG, "dense repository needs dim > 0 and n >= 0");
  DeviceGuard g(device);
  otf_repo* r = new otf_repo();
  r->kind = OTF_KIND_DENSE;
  r->model_dim = dim;
  r->row_bytes = (int64_t)dim * 4;
  int rc = repo_common(r, device, n, ids, id_base, mem);
  if (!rc) rc = take_payload(r, data, (size_t)n * dim * sizeof(float), mem, borrow);
  if (!rc && cudaStreamSynchronize(r->stream) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "create_dense");
  if (rc) { repo_free(r); return rc; }
  *out = r;
  return OTF_OK;
}

int otf_repo_create_pq(int device, const uint8_t* codes, int64_t n, const float* centroids,
                       int32_t num_blocks, int32_t num_centroids, int32_t subdim,
                       const int64_t* ids, int64_t id_base, int mem, int borrow,
                       otf_repo** out) {
  *out = nullptr;
  if (num_blocks <= 0 || subdim <= 0 || num_centroids <= 0 || num_centroids > 256 || n < 0)
    return fail(OTF_ERR_CONFIG, "pq repository needs blocks, subdim > 0 and 1 <= centroids <= 256");
  DeviceGuard g(device);
  otf_repo* r = new otf_repo();
  r->kind = OTF_KIND_PQ;
  r->M = num_blocks; r->K = num_centroids; r->Q = subdim;
  r->model_dim = num_blocks * subdim;
  r->row_bytes = num_blocks;
  int rc = repo_common(r, device, n, ids, id_base, mem);
  if (!rc) rc = take_payload(r, codes, (size_t)n * num_blocks, mem, borrow);
  const size_t cb = (size_t)num_blocks * num_centroids * subdim * sizeof(float);
  if (!rc && cudaMalloc(&r->cents, cb) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "cudaMalloc centroids");
  if (!rc) rc = copy_in(r->cents, centroids, cb, OTF_MEM_HOST, r->stream);
  // codes must index the codebook (pq.py:240-241 / load_pq_codes :326-329)
  unsigned int* bad = nullptr;
  if (!rc && num_centroids < 256) {
    if (cudaMalloc(&bad, sizeof(unsigned int)) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "cudaMalloc");
    if (!rc) { cudaMemsetAsync(bad, 0, sizeof(unsigned int), r->stream);
      rc = launch_pq_check(static_cast<const uint8_t*>(r->payload), n * num_blocks, num_centroids, bad, device, r->stream); }
  }
  if (!rc && cudaStreamSynchronize(r->stream) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "create_pq");
  if (!rc && bad) {
    unsigned int hb = 0;
    cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost);
    if (hb) rc = fail(OTF_ERR_CORRUPTION, "code value out of range for " + std::to_string(num_centroids) + " centroids");
  }
  if (bad) cudaFree(bad);
  if (rc) { repo_free(r); return rc; }
  *out = r;
  return OTF_OK;
}

int otf_repo_create_binary(int device, const uint8_t* codes, int64_t n, int32_t output_bits,
                           const int64_t* ids, int64_t id_base, int mem, int borrow,
                           otf_repo** out) {
  *out = nullptr;
  if (output_bits <= 0 || n < 0) return fail(OTF_ERR_CONFIG, "binary repository needs output_bits > 0");
  DeviceGuard g(device);
  otf_repo* r = new otf_repo();
  r->kind = OTF_KIND_BINARY;
  r->model_dim = output_bits;
  r->row_bytes = (output_bits + 7) / 8;
  int rc = repo_common(r, device, n, ids, id_base, mem);
  if (!rc) rc = take_payload(r, codes, (size_t)n * r->row_bytes, mem, borrow);
  if (!rc && cudaStreamSynchronize(r->stream) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "create_binary");
  if (rc) { repo_free(r); return rc; }
  *out = r;
  return OTF_OK;
}

int otf_repo_subset(const otf_repo* src_c, const int64_t* rows, int64_t n_keep, otf_repo** out) {
  *out = nullptr;
  otf_repo* src = const_cast<otf_repo*>(src_c);
  std::lock_guard<std::mutex> lk(src->mu);
  DeviceGuard g(src->device);
  for (int64_t i = 0; i < n_keep; ++i)
    if (rows[i] < 0 || rows[i] >= src->n) return fail(OTF_ERR_CONFIG, "subset row out of range");
  otf_repo* r = new otf_repo();
  r->device = src->device; r->kind = src->kind; r->n = n_keep; r->model_dim = src->model_dim;
  r->M = src->M; r->K = src->K; r->Q = src->Q; r->row_bytes = src->row_bytes;
  r->id_base = 0;
  int rc = make_stream(&r->stream, false);
  DevBuf d_rows;
  if (!rc) rc = d_rows.ensure((size_t)(n_keep > 0 ? n_keep : 1) * sizeof(int64_t));
  if (!rc) rc = copy_in(d_rows.p, rows, (size_t)n_keep * sizeof(int64_t), OTF_MEM_HOST, r->stream);
  void* p = nullptr;
  if (!rc && cudaMalloc(&p, (size_t)(n_keep > 0 ? n_keep : 1) * r->row_bytes) != cudaSuccess)
    rc = cuda_fail(cudaGetLastError(), "cudaMalloc subset");
  if (!rc) { r->payload = p; r->owns_payload = true; }
  if (!rc && cudaMalloc(&r->ids, (size_t)(n_keep > 0 ? n_keep : 1) * sizeof(int64_t)) != cudaSuccess)
    rc = cuda_fail(cudaGetLastError(), "cudaMalloc subset ids");
  // order the subset after any pending work on the source stream
  if (!rc) rc = repo_enter(src, r->stream);
  if (!rc) rc = launch_gather_rows(static_cast<const uint8_t*>(src->payload), r->row_bytes,
                                   static_cast<const int64_t*>(d_rows.p), n_keep,
                                   static_cast<uint8_t*>(p), r->device, r->stream);
  if (!rc) rc = launch_gather_i64(src->ids, static_cast<const int64_t*>(d_rows.p), n_keep,
                                  src->id_base, r->ids, r->stream);
  if (!rc && src->cents) {
    const size_t cb = (size_t)src->M * src->K * src->Q * sizeof(float);
    if (cudaMalloc(&r->cents, cb) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "cudaMalloc cents");
    if (!rc) rc = copy_in(r->cents, src->cents, cb, OTF_MEM_DEVICE, r->stream);
  }
  if (!rc) rc = repo_leave(src, r->stream);
  if (!rc && cudaStreamSynchronize(r->stream) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "subset");
  d_rows.release();
  if (rc) { repo_free(r); return rc; }
  *out = r;
  return OTF_OK;
}

int otf_repo_destroy(otf_repo* repo) {
  repo_free(repo);
  return OTF_OK;
}

int otf_repo_info(const otf_repo* r, int32_t* kind, int64_t* count, int32_t* model_dim,
                  int64_t* payload_bytes, int32_t* device) {
  if (kind) *kind = r->kind;
  if (count) *count = r->n;
  if (model_dim) *model_dim = r->model_dim;
  if (payload_bytes) *payload_bytes = r->n * r->row_bytes;
  if (device) *device = r->device;
  return OTF_OK;
}

int otf_repo_score(otf_repo* r, const double* w, void* out, int mem, void* stream) {
  OTF_NVTX("otf_repo_score");
  std::lock_guard<std::mutex> lk(r->mu);
  DeviceGuard g(r->device);
  cudaStream_t st = mem == OTF_MEM_DEVICE ? pick_stream(r->stream, stream) : r->stream;
  int rc = repo_ordered(r, st, [&]() -> int {
    const double* dw = nullptr;
    int rc = stage_w(r, w, mem, st, &dw);
    if (rc) return rc;
    const size_t es = score_dtype(r) == OTF_F64 ? 8 : 4;
    if (mem == OTF_MEM_DEVICE) return score_into(r, dw, out, nullptr, st);
    if ((rc = r->scores.ensure((size_t)(r->n > 0 ? r->n : 1) * es))) return rc;
    if ((rc = score_into(r, dw, r->scores.p, nullptr, st))) return rc;
    OTF_CUDA(cudaMemcpyAsync(out, r->scores.p, (size_t)r->n * es, cudaMemcpyDeviceToHost, st));
    return OTF_OK;
  });
  if (!rc && mem == OTF_MEM_HOST) OTF_CUDA(cudaStreamSynchronize(st));
  return rc;
}

int otf_repo_cut_fallbacks(otf_repo* r, int64_t* out) {
  if (!r || !out) return fail(OTF_ERR_CONFIG, "repository or out is NULL");
  std::lock_guard<std::mutex> lk(r->mu);
  DeviceGuard g(r->device);
  *out = 0;
  if (r->used) OTF_CUDA(cudaEventSynchronize(r->last));
  // the single-list cut paths (dense, PQ) and the many-classifier sampled-threshold selection
  for (const TopkWs* ws : {&r->topk, &r->mtopk}) {
    if (!ws->cut_word) continue;
    unsigned int w = 0;
    OTF_CUDA(cudaMemcpy(&w, ws->cut_word + 3, sizeof(w), cudaMemcpyDeviceToHost));
    *out += w;
  }
  return OTF_OK;
}

int otf_repo_time_rank_scan(otf_repo* r, const double* w_dev, int64_t k, float* ms, void* stream) {
  std::lock_guard<std::mutex> lk(r->mu);
  DeviceGuard g(r->device);
  if (!ms) return fail(OTF_ERR_CONFIG, "ms must not be NULL");
  cudaStream_t st = pick_stream(r->stream, stream);
  const size_t es = score_dtype(r) == OTF_F64 ? 8 : 4;
  int rc = repo_enter(r, st);
  if (!rc) rc = r->scores.ensure((size_t)(r->n > 0 ? r->n : 1) * es);
  if (!rc) rc = topk_ws_alloc(&r->topk, 1);
  if (!rc) rc = topk_cmax_ensure(&r->topk, r->n);
  const uint8_t* codes = static_cast<const uint8_t*>(r->payload);
  const int64_t k_eff = k < 0 ? 0 : (k > r->n ? r->n : k);
  int cut_r = 0;
  DenseCutPlan dpl;
  const bool dcut = r->kind == OTF_KIND_DENSE && k_eff > 0 && k_eff < r->n &&
                    dense_cut_plan(r->model_dim, static_cast<const float*>(r->payload), r->n, k_eff, r->device, &dpl);
  const bool cut = dcut || (r->kind == OTF_KIND_PQ && pq_cut_plan(r->M, codes, r->n, k_eff, r->device, &cut_r));
  const bool bins = !cut && r->kind == OTF_KIND_PQ && pq_bins_path(r->M, codes);
  if (!rc && cut && !dcut) rc = r->lut.ensure((size_t)r->M * r->K * sizeof(double) * kCutLutReplicas);
  if (!rc && cut) rc = topk_cut_alloc(&r->topk);
  if (!rc && cut) rc = topk_ws_alloc(&r->topk, k_eff);
  if (!rc && cut) rc = r->outbuf.ensure((size_t)(k_eff > 0 ? k_eff : 1) * 24);
  if (!rc && bins) rc = r->bins.ensure((size_t)(r->n > 0 ? r->n : 1) * sizeof(uint16_t));
  if (!rc && bins) rc = r->lut.ensure((size_t)r->M * r->K * sizeof(double));
  if (!rc && bins) rc = launch_pq_lut(r->cents, r->M, r->K, r->Q, w_dev, static_cast<double*>(r->lut.p), st);
  if (rc) return rc;
  cudaEvent_t e0, e1;
  OTF_CUDA(cudaEventCreate(&e0));
  OTF_CUDA(cudaEventCreate(&e1));
  int clog = -1;
  cudaEventRecord(e0, st);
  if (dcut) {
    int64_t* d_ids = static_cast<int64_t*>(r->outbuf.p);
    rc = launch_dense_rank_cut(static_cast<const float*>(r->payload), r->n, r->model_dim, w_dev, r->ids, r->id_base,
                               k_eff, dpl, &r->topk, static_cast<float*>(r->scores.p), d_ids,
                               reinterpret_cast<double*>(d_ids + k_eff), d_ids + 2 * k_eff, st);
  } else if (cut) {
    // the PQ cut path's two kernels (sample + LUT, scan + selection) are the rank path's scan
    int64_t* d_ids = static_cast<int64_t*>(r->outbuf.p);
    rc = launch_pq_rank_cut(r->cents, r->K, r->Q, w_dev, static_cast<double*>(r->lut.p), codes, r->n, r->ids,
                            r->id_base, k_eff, cut_r, &r->topk, static_cast<double*>(r->scores.p), d_ids,
                            reinterpret_cast<double*>(d_ids + k_eff), d_ids + 2 * k_eff, r->device, st);
  } else if (bins)
    rc = launch_pq_scan_bins(codes, r->n, static_cast<const double*>(r->lut.p), r->K,
                             static_cast<uint16_t*>(r->bins.p), r->topk.hist, r->device, st, r->topk.cmax, &clog);
  else
    rc = score_into(r, w_dev, r->scores.p, r->topk.hist, st, r->topk.cmax, &clog);
  cudaEventRecord(e1, st);
  if (!rc && !cut) rc = cudaMemsetAsync(r->topk.hist, 0, kHistBinsMax * sizeof(uint32_t), st) == cudaSuccess
                    ? OTF_OK : cuda_fail(cudaGetLastError(), "cudaMemsetAsync");
  const int rc_leave = repo_leave(r, st);
  if (!rc) rc = rc_leave;
  cudaError_t e = cudaEventSynchronize(e1);
  if (!rc && e == cudaSuccess) e = cudaEventElapsedTime(ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (!rc && e != cudaSuccess) rc = cuda_fail(e, "otf_repo_time_rank_scan");
  return rc;
}

namespace {
int rank_graph_locked(otf_repo* r, const double* w_dev, int64_t k_eff, int64_t* ids_dev, double* scores_dev,
                      int64_t* rows_dev, cudaStream_t st, const void* h_in = nullptr, void* h_out = nullptr);
}  // namespace

int otf_repo_rank(otf_repo* r, const double* w, int64_t k, int64_t* out_ids, double* out_scores,
                  int64_t* out_rows, int64_t* out_n, int mem, void* stream) {
  OTF_NVTX("otf_repo_rank");
  std::lock_guard<std::mutex> lk(r->mu);
  DeviceGuard g(r->device);
  int64_t k_eff = k < 0 ? 0 : (k > r->n ? r->n : k);
  if (out_n) *out_n = k_eff;
  if (k_eff == 0) return OTF_OK;
  cudaStream_t st = mem == OTF_MEM_DEVICE ? pick_stream(r->stream, stream) : r->stream;
  if (mem == OTF_MEM_DEVICE)
    return repo_ordered(r, st, [&]() -> int {
      const double* dw = nullptr;
      int rc = stage_w(r, w, mem, st, &dw);
      return rc ? rc : rank_device(r, dw, k_eff, out_ids, out_scores, out_rows, st);
    });
  int rc = repo_enter(r, st);  // host mode: r->stream, synchronised below
  if (rc) return rc;
  const size_t wbytes = (size_t)r->model_dim * sizeof(double);
  const size_t bytes = (size_t)k_eff * 24;
  if ((rc = r->w.ensure(wbytes))) return rc;
  if ((rc = r->h_w.ensure(wbytes))) return rc;
  if ((rc = r->outbuf.ensure(bytes))) return rc;
  if ((rc = r->h_out.ensure(bytes))) return rc;
  std::memcpy(r->h_w.p, w, wbytes);  // the previous host call synchronised: the staging is free
  // the selection writes the (ids, scores, rows) block straight into the pinned host buffer
  // (mapped into the device address space): no D2H copy after the kernels
  static const bool d2h_copy = getenv("OTF_HOST_D2H_COPY") != nullptr;  // A/B switch (tools/)
  int64_t* d_ids = static_cast<int64_t*>(d2h_copy ? r->outbuf.p : r->h_out.p);
  double* d_sc = reinterpret_cast<double*>(d_ids + k_eff);
  int64_t* d_rows = reinterpret_cast<int64_t*>(d_sc + k_eff);
  // host calls replay the repository's cached graph of the whole query: H2D of w from the
  // pinned staging, the kernels (staging and output buffers are the handle's own, so the graph
  // is reused by every host-memory rank of this k)
  rc = rank_graph_locked(r, static_cast<const double*>(r->w.p), k_eff, d_ids, d_sc, d_rows, st, r->h_w.p,
                         d2h_copy ? r->h_out.p : nullptr);
  if (rc) {
    repo_leave(r, st);
    cudaStreamSynchronize(st);
    return rc;
  }
  OTF_CUDA(cudaStreamSynchronize(st));
  // the stream is drained: nothing of this call is pending, so a later call on another stream
  // has nothing to wait for (no event record on the per-query host path)
  r->used = false;
  r->last_stream = st;
  const int64_t* h_ids = static_cast<const int64_t*>(r->h_out.p);
  std::memcpy(out_ids, h_ids, (size_t)k_eff * 8);
  std::memcpy(out_scores, h_ids + k_eff, (size_t)k_eff * 8);
  if (out_rows) std::memcpy(out_rows, h_ids + 2 * k_eff, (size_t)k_eff * 8);
  return OTF_OK;
}

// ---- many classifiers (C5b): tensor-core scoring of a dense repository ----------------------------
namespace {
// host W (n_cls x dim float64) -> pinned staging -> r->w (device), on st
int stage_many(otf_repo* r, const double* W, int n_cls, cudaStream_t st, const double** dw) {
  const size_t bytes = (size_t)n_cls * r->model_dim * sizeof(double);
  int rc = r->h_w.ensure(bytes);
  if (!rc) rc = r->w.ensure(bytes);
  if (rc) return rc;
  cudaStreamSynchronize(st);  // the staging buffer may still feed an earlier upload
  std::memcpy(r->h_w.p, W, bytes);
  OTF_CUDA(cudaMemcpyAsync(r->w.p, r->h_w.p, bytes, cudaMemcpyHostToDevice, st));
  *dw = static_cast<const double*>(r->w.p);
  return OTF_OK;
}
// scores for classifiers [c0, c0 + cn) into out (cn x n float32, classifier-major); W host/device.
int multi_score_group(otf_repo* r, const double* dW, int cn, float* out, cudaStream_t st) {
  int rc = r->w32.ensure((size_t)multi_ws_floats(r->model_dim) * sizeof(float));
  if (rc) return rc;
  if (!r->x_exp_ready) {  // one pass over the repository, on the first multi-classifier call
    if ((rc = multi_x_exponent(static_cast<const float*>(r->payload), r->n, r->model_dim, r->device, st,
                               &r->x_exp)))
      return rc;
    r->x_exp_ready = true;
  }
  return launch_multi_score(static_cast<const float*>(r->payload), r->n, r->model_dim, dW, cn,
                            static_cast<float*>(r->w32.p), out, r->device, st, r->x_exp);
}
}  // namespace

int otf_repo_score_many(otf_repo* r, const double* W, int32_t n_cls, float* out, int mem, void* stream) {
  OTF_NVTX("otf_repo_score_many");
  std::lock_guard<std::mutex> lk(r->mu);
  DeviceGuard g(r->device);
  if (r->kind != OTF_KIND_DENSE) return fail(OTF_ERR_CONFIG, "multi-classifier scoring needs a dense repository");
  if (n_cls < 1) return fail(OTF_ERR_CONFIG, "n_cls must be positive");
  if (!multi_tc_supported(r->model_dim, static_cast<const float*>(r->payload)))
    return fail(OTF_ERR_CONFIG, "multi-classifier scoring needs dim % 32 == 0");
  cudaStream_t st = mem == OTF_MEM_DEVICE ? pick_stream(r->stream, stream) : r->stream;
  const double* wp = W;
  int rc = repo_enter(r, st);
  if (rc) return rc;
  if (mem == OTF_MEM_HOST && (rc = stage_many(r, W, n_cls, st, &wp))) return rc;
  if (mem == OTF_MEM_HOST &&
      (rc = r->multi.ensure((size_t)std::min<int32_t>(n_cls, 64) * (r->n > 0 ? r->n : 1) * sizeof(float))))
    return rc;
  for (int c0 = 0; c0 < n_cls && !rc; c0 += 64) {
    const int cn = std::min(64, n_cls - c0);
    float* o = mem == OTF_MEM_HOST ? static_cast<float*>(r->multi.p) : out + (size_t)c0 * r->n;
    rc = multi_score_group(r, wp + (size_t)c0 * r->model_dim, cn, o, st);
    if (!rc && mem == OTF_MEM_HOST) {
      cudaError_t e = cudaMemcpyAsync(out + (size_t)c0 * r->n, o, (size_t)cn * r->n * sizeof(float),
                                      cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) rc = cuda_fail(e, "cudaMemcpyAsync");
    }
  }
  if (const int rc2 = repo_leave(r, st)) rc = rc ? rc : rc2;
  if (mem == OTF_MEM_HOST || rc) cudaStreamSynchronize(st);
  return rc;
}

int otf_repo_rank_many(otf_repo* r, const double* W, int32_t n_cls, int64_t k, int64_t* out_ids,
                       double* out_scores, int64_t* out_n, int mem, void* stream) {
  OTF_NVTX("otf_repo_rank_many");
  std::lock_guard<std::mutex> lk(r->mu);
  DeviceGuard g(r->device);
  if (r->kind != OTF_KIND_DENSE) return fail(OTF_ERR_CONFIG, "multi-classifier ranking needs a dense repository");
  if (n_cls < 1) return fail(OTF_ERR_CONFIG, "n_cls must be positive");
  if (!multi_tc_supported(r->model_dim, static_cast<const float*>(r->payload)))
    return fail(OTF_ERR_CONFIG, "multi-classifier ranking needs dim % 32 == 0");
  const int64_t k_eff = k < 0 ? 0 : (k > r->n ? r->n : k);
  if (out_n) *out_n = k_eff;
  if (k_eff == 0) return OTF_OK;
  cudaStream_t st = mem == OTF_MEM_DEVICE ? pick_stream(r->stream, stream) : r->stream;
  const double* wp = W;
  int rc = repo_enter(r, st);
  if (rc) return rc;
  const size_t lbytes = (size_t)n_cls * k_eff * 8;  // ids (int64) and scores (float64) per list entry
  if (mem == OTF_MEM_HOST) {
    if ((rc = stage_many(r, W, n_cls, st, &wp))) return rc;
    if ((rc = r->outbuf.ensure(2 * lbytes)) || (rc = r->h_out.ensure(2 * lbytes))) return rc;
  }
  int64_t* ids = mem == OTF_MEM_HOST ? static_cast<int64_t*>(r->outbuf.p) : out_ids;
  double* sc = mem == OTF_MEM_HOST ? reinterpret_cast<double*>(static_cast<char*>(r->outbuf.p) + lbytes) : out_scores;
  // the (<= 64, n) score buffer is cached on the handle (2.56 GB for 64 x 10M rows)
  if ((rc = r->multi.ensure((size_t)std::min<int32_t>(n_cls, 64) * (r->n > 0 ? r->n : 1) * sizeof(float)))) return rc;
  float* sbuf = static_cast<float*>(r->multi.p);
  for (int c0 = 0; c0 < n_cls && !rc; c0 += 64) {
    const int cn = std::min(64, n_cls - c0);
    rc = multi_score_group(r, wp + (size_t)c0 * r->model_dim, cn, sbuf, st);
    // all cn selections in one cooperative launch (a few SMs each) when the GPU has an SM pair
    // per classifier; otherwise one launch per classifier over the whole GPU
    int seg_r = 0;
    if (!rc && topk_seg_cut_plan(cn, r->n, k_eff, r->device, &seg_r))
      rc = launch_topk_seg_cut(sbuf, cn, r->n, r->ids, r->id_base, k_eff, seg_r, &r->mtopk, ids + (size_t)c0 * k_eff,
                               sc + (size_t)c0 * k_eff, r->device, st);
    else if (!rc && sm_count(r->device) >= 2 * cn)
      rc = launch_topk_segments(sbuf, cn, r->n, r->ids, r->id_base, k_eff, &r->mtopk,
                                ids + (size_t)c0 * k_eff, sc + (size_t)c0 * k_eff, r->device, st);
    else
      for (int c = 0; c < cn && !rc; ++c)
        rc = launch_topk(sbuf + (size_t)c * r->n, OTF_F32, r->n, r->ids, r->id_base, k_eff, &r->topk, false,
                         ids + (size_t)(c0 + c) * k_eff, sc + (size_t)(c0 + c) * k_eff, nullptr, r->device, st);
  }
  if (const int rc2 = repo_leave(r, st)) rc = rc ? rc : rc2;
  if (!rc && mem == OTF_MEM_HOST) {
    // one D2H of both arrays into pinned staging, then plain copies into the caller's buffers
    cudaError_t e = cudaMemcpyAsync(r->h_out.p, r->outbuf.p, 2 * lbytes, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync");
    std::memcpy(out_ids, r->h_out.p, lbytes);
    std::memcpy(out_scores, static_cast<char*>(r->h_out.p) + lbytes, lbytes);
    return OTF_OK;
  }
  if (rc) cudaStreamSynchronize(st);
  return rc;
}

namespace {
// rank(k) for a device w through the repository's cached CUDA graph (captured on the first call
// for a given (w, outputs, stream, k), replayed afterwards). Caller holds r->mu.
// h_in / h_out (host-memory rank): the graph also holds the H2D copy of w from the pinned
// staging buffer h_in and the D2H copy of the (ids, scores, rows) block to h_out, so a host query
// is ONE graph launch (no separate copy calls between the kernels).
int rank_graph_locked(otf_repo* r, const double* w_dev, int64_t k_eff, int64_t* ids_dev, double* scores_dev,
                      int64_t* rows_dev, cudaStream_t st, const void* h_in, void* h_out) {
  constexpr size_t kGraphCache = 4;
  // allocate everything outside capture (no-ops once the workspaces are large enough)
  const size_t es = score_dtype(r) == OTF_F64 ? 8 : 4;
  int rc = r->scores.ensure((size_t)(r->n > 0 ? r->n : 1) * es);
  if (!rc) rc = topk_ws_alloc(&r->topk, k_eff);
  if (!rc && (r->kind == OTF_KIND_PQ)) rc = r->lut.ensure((size_t)r->M * r->K * sizeof(double) * kCutLutReplicas);
  if (!rc && (r->kind == OTF_KIND_PQ)) rc = r->bins.ensure((size_t)(r->n > 0 ? r->n : 1) * 2);
  if (!rc && (r->kind == OTF_KIND_BINARY)) rc = r->bins.ensure((size_t)(r->n > 0 ? r->n : 1) * 8);
  if (!rc) rc = topk_cmax_ensure(&r->topk, r->n);
  if (!rc) rc = topk_cut_alloc(&r->topk);  // (every kind: the fused paths' words, the scans' dynamic tails)
  if (rc) return rc;
  if (r->kind == OTF_KIND_DENSE) {  // the plan's one-time kernel attributes, outside the capture
    DenseCutPlan dpl;
    dense_cut_plan(r->model_dim, static_cast<const float*>(r->payload), r->n, k_eff, r->device, &dpl);
  }
  const void* key[16] = {w_dev, ids_dev, scores_dev, rows_dev, st, r->scores.p, r->lut.p, r->bins.p,
                         r->topk.hist, r->topk.key, r->topk.inv, r->topk.row, r->topk.cmax, r->topk.cut_key,
                         h_in, h_out};
  otf_repo::GraphEntry* hit = nullptr;
  for (auto& ge : r->graphs) {
    bool same = ge.exec && ge.k == k_eff && ge.reserved == reserved_sms(r->device);
    for (int i = 0; i < 16 && same; ++i) same = ge.key[i] == key[i];
    if (same) { hit = &ge; break; }
  }
  if (!hit) {
    OTF_CUDA(cudaStreamSynchronize(st));  // allocations above must not race the capture
    cudaStream_t cap;
    OTF_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    OTF_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    const int64_t l0 = g_launches.load();
    if (h_in && cudaMemcpyAsync(const_cast<double*>(w_dev), h_in, (size_t)r->model_dim * sizeof(double),
                                cudaMemcpyHostToDevice, cap) != cudaSuccess)
      rc = cuda_fail(cudaGetLastError(), "cudaMemcpyAsync (graph H2D)");
    // (a one-CTA kernel reading w through the pinned buffer's device mapping instead of this copy
    // node measured the same: C1 host query 108.9 vs 108.8 us)
    if (!rc) rc = rank_device(r, w_dev, k_eff, ids_dev, scores_dev, rows_dev, cap);
    if (!rc && h_out && cudaMemcpyAsync(h_out, ids_dev, (size_t)k_eff * 24, cudaMemcpyDeviceToHost, cap) != cudaSuccess)
      rc = cuda_fail(cudaGetLastError(), "cudaMemcpyAsync (graph D2H)");
    const int kernels = (int)(g_launches.load() - l0);
    g_launches.fetch_sub(kernels);  // captured, not launched
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(cap, &graph);
    cudaStreamDestroy(cap);
    if (rc) { if (graph) cudaGraphDestroy(graph); return rc; }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
    if (r->graphs.size() < kGraphCache) {
      r->graphs.emplace_back();
      hit = &r->graphs.back();
    } else {
      hit = &r->graphs[0];
      for (auto& ge : r->graphs)
        if (ge.used < hit->used) hit = &ge;
      cudaGraphExecDestroy(hit->exec);
    }
    hit->exec = exec;
    for (int i = 0; i < 16; ++i) hit->key[i] = key[i];
    hit->k = k_eff;
    hit->kernels = kernels;
    hit->reserved = reserved_sms(r->device);
  }
  hit->used = ++r->graph_clock;
  OTF_CUDA(cudaGraphLaunch(hit->exec, st));
  count_launch(hit->kernels);
  return OTF_OK;
}
}  // namespace

int otf_repo_rank_graph(otf_repo* r, const double* w_dev, int64_t k, int64_t* ids_dev,
                        double* scores_dev, int64_t* rows_dev, void* stream) {
  OTF_NVTX("otf_repo_rank_graph");
  std::lock_guard<std::mutex> lk(r->mu);
  DeviceGuard g(r->device);
  int64_t k_eff = k < 0 ? 0 : (k > r->n ? r->n : k);
  if (k_eff == 0) return OTF_OK;
  cudaStream_t st = pick_stream(r->stream, stream);
  return repo_ordered(r, st, [&]() { return rank_graph_locked(r, w_dev, k_eff, ids_dev, scores_dev, rows_dev, st); });
}

// ---- stateless primitives ----------------------------------------------------------------------
namespace {
struct Scratch {
  std::vector<DevBuf> bufs;
  cudaStream_t st = nullptr;
  int device = 0;
  ~Scratch() {
    if (st) { cudaStreamSynchronize(st); cudaStreamDestroy(st); }
    for (auto& b : bufs) b.release();
  }
  int init(int dev) {
    device = dev;
    OTF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    return OTF_OK;
  }
  // device copy of a host input (or pass-through for device memory)
  int in(const void* src, size_t bytes, int mem, const void** dptr) {
    if (mem == OTF_MEM_DEVICE) { *dptr = src; return OTF_OK; }
    bufs.emplace_back();
    int rc = bufs.back().ensure(bytes > 0 ? bytes : 16);
    if (rc) return rc;
    if (bytes) OTF_CUDA(cudaMemcpyAsync(bufs.back().p, src, bytes, cudaMemcpyHostToDevice, st));
    *dptr = bufs.back().p;
    return OTF_OK;
  }
  int outbuf(void* user, size_t bytes, int mem, void** dptr) {
    if (mem == OTF_MEM_DEVICE) { *dptr = user; return OTF_OK; }
    bufs.emplace_back();
    int rc = bufs.back().ensure(bytes > 0 ? bytes : 16);
    if (rc) return rc;
    *dptr = bufs.back().p;
    return OTF_OK;
  }
  // device scratch in either mode (released, after the work completes, by cudaFree)
  int tmp(size_t bytes, void** dptr) {
    bufs.emplace_back();
    int rc = bufs.back().ensure(bytes > 0 ? bytes : 16);
    if (rc) return rc;
    *dptr = bufs.back().p;
    return OTF_OK;
  }
  int out(void* user, const void* dptr, size_t bytes, int mem) {
    if (mem == OTF_MEM_DEVICE) return OTF_OK;
    if (bytes) OTF_CUDA(cudaMemcpyAsync(user, dptr, bytes, cudaMemcpyDeviceToHost, st));
    OTF_CUDA(cudaStreamSynchronize(st));
    return OTF_OK;
  }
};
}  // namespace

#define STATELESS_BEGIN(device, mem, stream)                                    \
  DeviceGuard _g(device);                                                       \
  Scratch S;                                                                    \
  cudaStream_t st;                                                              \
  if (mem == OTF_MEM_DEVICE) { st = static_cast<cudaStream_t>(stream); S.device = device; } \
  else { int _rc = S.init(device); if (_rc) return _rc; st = S.st; }              \
  int rc = OTF_OK;

int otf_score_dense(int device, const float* X, int64_t n, int32_t dim, const double* w, float* out,
                    int mem, void* stream) {
  if (dim <= 0) return fail(OTF_ERR_CONFIG, "dim must be positive");
  STATELESS_BEGIN(device, mem, stream)
  const void *dX, *dw; void* dout;
  if ((rc = S.in(X, (size_t)n * dim * 4, mem, &dX))) return rc;
  if ((rc = S.in(w, (size_t)dim * 8, mem, &dw))) return rc;
  if ((rc = S.outbuf(out, (size_t)n * 4, mem, &dout))) return rc;
  if ((rc = launch_dense_score(static_cast<const float*>(dX), n, dim, static_cast<const double*>(dw),
                               static_cast<float*>(dout), nullptr, device, st))) return rc;
  return S.out(out, dout, (size_t)n * 4, mem);
}

int otf_pq_build_lut(int device, const float* centroids, int32_t M, int32_t K, int32_t Q,
                     const double* w, double* lut, int mem, void* stream) {
  if (M <= 0 || K <= 0 || Q <= 0) return fail(OTF_ERR_CONFIG, "bad codebook shape");
  STATELESS_BEGIN(device, mem, stream)
  const void *dc, *dw; void* dl;
  if ((rc = S.in(centroids, (size_t)M * K * Q * 4, mem, &dc))) return rc;
  if ((rc = S.in(w, (size_t)M * Q * 8, mem, &dw))) return rc;
  if ((rc = S.outbuf(lut, (size_t)M * K * 8, mem, &dl))) return rc;
  if ((rc = launch_pq_lut(static_cast<const float*>(dc), M, K, Q, static_cast<const double*>(dw),
                          static_cast<double*>(dl), st))) return rc;
  return S.out(lut, dl, (size_t)M * K * 8, mem);
}

int otf_pq_score_codes(int device, const double* lut, int32_t M, int32_t K, const uint8_t* codes,
                       int64_t n, double* out, int mem, void* stream) {
  if (M <= 0 || K <= 0) return fail(OTF_ERR_CONFIG, "bad LUT shape");
  STATELESS_BEGIN(device, mem, stream)
  const void *dl, *dc; void* dout; DevBuf bad;
  if ((rc = S.in(lut, (size_t)M * K * 8, mem, &dl))) return rc;
  if ((rc = S.in(codes, (size_t)n * M, mem, &dc))) return rc;
  if ((rc = S.outbuf(out, (size_t)n * 8, mem, &dout))) return rc;
  if (K < 256) {
    if ((rc = bad.ensure(sizeof(unsigned int)))) return rc;
    OTF_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned int), st));
    if ((rc = launch_pq_check(static_cast<const uint8_t*>(dc), n * M, K, static_cast<unsigned int*>(bad.p),
                              device, st))) return rc;
    unsigned int hb = 0;
    OTF_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(hb), cudaMemcpyDeviceToHost, st));
    OTF_CUDA(cudaStreamSynchronize(st));
    bad.release();
    if (hb) return fail(OTF_ERR_CORRUPTION, "code value out of range for " + std::to_string(K) + " centroids");
  }
  if ((rc = launch_pq_scan(static_cast<const uint8_t*>(dc), n, M, nullptr, nullptr,
                           static_cast<const double*>(dl), K, 0, static_cast<double*>(dout), nullptr,
                           device, st))) return rc;
  return S.out(out, dout, (size_t)n * 8, mem);
}

int otf_score_binary(int device, const uint8_t* codes, int64_t n, int32_t output_bits,
                     const double* w, float* out, int mem, void* stream) {
  OTF_NVTX("otf_score_binary");
  if (output_bits <= 0) return fail(OTF_ERR_CONFIG, "output_bits must be positive");
  STATELESS_BEGIN(device, mem, stream)
  const int row_bytes = (output_bits + 7) / 8;
  const void *dc, *dw; void* dout;
  if ((rc = S.in(codes, (size_t)n * row_bytes, mem, &dc))) return rc;
  if ((rc = S.in(w, (size_t)output_bits * 8, mem, &dw))) return rc;
  if ((rc = S.outbuf(out, (size_t)n * 4, mem, &dout))) return rc;
  DevBuf scratch;
  if ((rc = scratch.ensure((size_t)(n > 0 ? n : 1) * sizeof(double)))) return rc;
  rc = launch_bin_score(static_cast<const uint8_t*>(dc), n, output_bits, static_cast<const double*>(dw),
                        static_cast<float*>(dout), nullptr, static_cast<double*>(scratch.p), device, st);
  if (!rc) rc = S.out(out, dout, (size_t)n * 4, mem);
  cudaStreamSynchronize(st);  // scratch is freed on return
  scratch.release();
  return rc;
}

int otf_unpack_bits(int device, const uint8_t* codes, int64_t n, int32_t output_bits, float* out,
                    int mem, void* stream) {
  if (output_bits <= 0) return fail(OTF_ERR_CONFIG, "output_bits must be positive");
  STATELESS_BEGIN(device, mem, stream)
  const int row_bytes = (output_bits + 7) / 8;
  const void* dc; void* dout;
  if ((rc = S.in(codes, (size_t)n * row_bytes, mem, &dc))) return rc;
  if ((rc = S.outbuf(out, (size_t)n * output_bits * 4, mem, &dout))) return rc;
  if ((rc = launch_bin_unpack(static_cast<const uint8_t*>(dc), n, output_bits, static_cast<float*>(dout),
                              device, st))) return rc;
  return S.out(out, dout, (size_t)n * output_bits * 4, mem);
}

int otf_binarize(int device, const double* frame, const float* centering, int32_t input_dim,
                 int32_t output_bits, const double* X, int64_t n, uint8_t* out, int mem,
                 void* stream) {
  if (input_dim <= 0 || output_bits <= 0) return fail(OTF_ERR_CONFIG, "bad frame shape");
  STATELESS_BEGIN(device, mem, stream)
  const int row_bytes = (output_bits + 7) / 8;
  const void *dU, *dmu, *dX; void* dout;
  if ((rc = S.in(frame, (size_t)output_bits * input_dim * 8, mem, &dU))) return rc;
  if ((rc = S.in(centering, (size_t)input_dim * 4, mem, &dmu))) return rc;
  if ((rc = S.in(X, (size_t)n * input_dim * 8, mem, &dX))) return rc;
  if ((rc = S.outbuf(out, (size_t)n * row_bytes, mem, &dout))) return rc;
  if ((rc = launch_binarize(static_cast<const double*>(dU), static_cast<const float*>(dmu), input_dim,
                            output_bits, static_cast<const double*>(dX), n, static_cast<uint8_t*>(dout),
                            device, st))) return rc;
  return S.out(out, dout, (size_t)n * row_bytes, mem);
}

namespace {
// per-thread, per-device scratch of the stateless calls, ordered by an event: no cudaMalloc /
// cudaFree (an implicit device synchronisation, and occasionally tens of ms of host time) per call
struct CachedScratchBuf {
  DevBuf buf;
  cudaEvent_t done = nullptr;
  int device = 0;
  ~CachedScratchBuf() {
    if (done) {
      cudaSetDevice(device);
      cudaEventSynchronize(done);
      cudaEventDestroy(done);
    }
    buf.release();
  }
  // a buffer of >= bytes usable on st once the previous call's work is done
  int acquire(size_t bytes, cudaStream_t st, void** p) {
    if (done && cudaStreamWaitEvent(st, done, 0) != cudaSuccess) return cuda_fail(cudaGetLastError(), "wait");
    if (int rc = buf.ensure(bytes > 0 ? bytes : 16)) return rc;  // growing frees the old one (synchronises)
    *p = buf.p;
    return OTF_OK;
  }
  int release(cudaStream_t st) {
    if (!done && cudaEventCreateWithFlags(&done, cudaEventDisableTiming) != cudaSuccess)
      return cuda_fail(cudaGetLastError(), "cudaEventCreate");
    cudaEventRecord(done, st);
    return OTF_OK;
  }
};
CachedScratchBuf& cached_scratch(int device) {
  static thread_local std::map<int, CachedScratchBuf> per_device;
  CachedScratchBuf& c = per_device[device];
  c.device = device;
  return c;
}
}  // namespace

int otf_pq_encode(int device, const float* vectors, int64_t n, int32_t dim, const float* centroids,
                  int32_t num_blocks, int32_t num_centroids, int32_t subdim, uint8_t* out_codes, int mem,
                  void* stream) {
  OTF_NVTX("otf_pq_encode");
  if (num_blocks <= 0 || num_centroids <= 0 || subdim <= 0) return fail(OTF_ERR_CONFIG, "bad codebook shape");
  if (num_centroids > 256) return fail(OTF_ERR_CONFIG, "num_centroids must fit a byte (<= 256)");
  if ((int64_t)dim != (int64_t)num_blocks * subdim)
    return fail(OTF_ERR_CONFIG, "vector dim " + std::to_string(dim) + " does not match codebook dim " +
                                    std::to_string((int64_t)num_blocks * subdim));
  if (n < 0) return fail(OTF_ERR_CONFIG, "n must be >= 0");
  if (n == 0) return OTF_OK;
  STATELESS_BEGIN(device, mem, stream)
  const void *dX, *dc;
  void *dout, *dnorm;
  const size_t cb = (size_t)num_blocks * num_centroids * subdim * 4;
  if ((rc = S.in(vectors, (size_t)n * dim * 4, mem, &dX))) return rc;
  if ((rc = S.in(centroids, cb, mem, &dc))) return rc;
  if ((rc = S.outbuf(out_codes, (size_t)n * num_blocks, mem, &dout))) return rc;
  CachedScratchBuf& cs = cached_scratch(device);
  if ((rc = cs.acquire(pq_encode_scratch_bytes(num_blocks, num_centroids), st, &dnorm))) return rc;
  rc = launch_pq_encode(static_cast<const float*>(dX), n, num_blocks, num_centroids, subdim,
                        static_cast<const float*>(dc), dnorm, static_cast<uint8_t*>(dout), device, st);
  if (int rc2 = cs.release(st)) return rc ? rc : rc2;
  if (rc) return rc;
  return S.out(out_codes, dout, (size_t)n * num_blocks, mem);
}

int otf_hamming(int device, const uint8_t* a, const uint8_t* b, int64_t n, int32_t width,
                int64_t* out, int mem, void* stream) {
  STATELESS_BEGIN(device, mem, stream)
  const void *da, *db; void* dout;
  if ((rc = S.in(a, (size_t)n * width, mem, &da))) return rc;
  if ((rc = S.in(b, (size_t)n * width, mem, &db))) return rc;
  if ((rc = S.outbuf(out, (size_t)n * 8, mem, &dout))) return rc;
  if ((rc = launch_hamming(static_cast<const uint8_t*>(da), static_cast<const uint8_t*>(db), n, width,
                           static_cast<int64_t*>(dout), device, st))) return rc;
  return S.out(out, dout, (size_t)n * 8, mem);
}

namespace {
struct CachedTopkWs {
  TopkWs ws;
  cudaEvent_t done = nullptr;
  int device = 0;
  ~CachedTopkWs() {
    if (done) {
      cudaSetDevice(device);
      cudaEventSynchronize(done);
      cudaEventDestroy(done);
    }
    topk_ws_free(&ws);
  }
};
CachedTopkWs& cached_topk_ws(int device) {
  static thread_local std::map<int, CachedTopkWs> per_device;
  CachedTopkWs& c = per_device[device];
  c.device = device;
  return c;
}
}  // namespace

int otf_top_k(int device, const void* scores, int32_t dtype, int64_t n, const int64_t* ids, int64_t k,
              int64_t* out_ids, double* out_scores, int64_t* out_rows, int64_t* out_n, int mem,
              void* stream) {
  OTF_NVTX("otf_top_k");
  const int64_t k_eff = k < 0 ? 0 : (k > n ? n : k);
  if (out_n) *out_n = k_eff;
  if (k_eff == 0) return OTF_OK;
  STATELESS_BEGIN(device, mem, stream)
  const size_t es = dtype == OTF_F64 ? 8 : 4;
  const void *ds, *di = nullptr;
  void *d_ids, *d_sc, *d_rows = nullptr;
  // the calling thread's cached workspace for this device (the multi-GPU merge calls this once
  // per query: no allocation, no host synchronisation in device mode); a call waits for the
  // previous call's kernel before reusing it, whatever stream that ran on
  CachedTopkWs& cw = cached_topk_ws(device);
  TopkWs& ws = cw.ws;
  if (cw.done && (rc = cudaStreamWaitEvent(st, cw.done, 0) == cudaSuccess ? OTF_OK
                                                                      : cuda_fail(cudaGetLastError(), "wait")))
    return rc;
  if ((rc = S.in(scores, (size_t)n * es, mem, &ds))) return rc;
  if (ids && (rc = S.in(ids, (size_t)n * 8, mem, &di))) return rc;
  if ((rc = S.outbuf(out_ids, (size_t)k_eff * 8, mem, &d_ids))) return rc;
  if ((rc = S.outbuf(out_scores, (size_t)k_eff * 8, mem, &d_sc))) return rc;
  if (out_rows && (rc = S.outbuf(out_rows, (size_t)k_eff * 8, mem, &d_rows))) return rc;
  rc = launch_topk(ds, dtype, n, static_cast<const int64_t*>(di), 0, k_eff, &ws, false,
                   static_cast<int64_t*>(d_ids), static_cast<double*>(d_sc),
                   static_cast<int64_t*>(d_rows), device, st);
  if (!rc) {
    if (!cw.done) rc = cudaEventCreateWithFlags(&cw.done, cudaEventDisableTiming) == cudaSuccess
                           ? OTF_OK : cuda_fail(cudaGetLastError(), "cudaEventCreate");
    if (!rc) cudaEventRecord(cw.done, st);
  }
  if (!rc) rc = S.out(out_ids, d_ids, (size_t)k_eff * 8, mem);
  if (!rc) rc = S.out(out_scores, d_sc, (size_t)k_eff * 8, mem);
  if (!rc && out_rows) rc = S.out(out_rows, d_rows, (size_t)k_eff * 8, mem);
  if (rc) cudaStreamSynchronize(st);
  return rc;
}

// ---- Pegasos -------------------------------------------------------------------------------------
int otf_pegasos_update(int device, double* w, int32_t d, const void* pos, int32_t pos_dtype,
                       int64_t n_pos, const void* neg, int32_t neg_dtype, int64_t n_neg,
                       const int64_t* pos_idx, const int64_t* neg_idx, int32_t half,
                       double shrink, double eta_over_b, int project, double radius,
                       void* stream) {
  if (d <= 0 || half <= 0) return fail(OTF_ERR_CONFIG, "bad pegasos shape");
  if (n_pos <= 0) return fail(OTF_ERR_NOT_READY, "no positives available yet");
  if (n_neg <= 0) return fail(OTF_ERR_INSUFFICIENT, "negative pool is empty");
  DeviceGuard g(device);
  return launch_pegasos(w, d, pos, pos_dtype, n_pos, neg, neg_dtype, n_neg, pos_idx, neg_idx, half,
                        shrink, eta_over_b, project, radius, static_cast<cudaStream_t>(stream));
}

int otf_pegasos_step_host(int device, double* w, int32_t d, const double* batch, int32_t half,
                          double shrink, double eta_over_b, int project, double radius) {
  if (d <= 0 || half <= 0) return fail(OTF_ERR_CONFIG, "bad pegasos shape");
  STATELESS_BEGIN(device, OTF_MEM_HOST, nullptr)
  const size_t bb = (size_t)2 * half * d * 8;
  DevBuf buf, idx;
  if ((rc = buf.ensure(bb + (size_t)d * 8))) return rc;
  if ((rc = idx.ensure((size_t)2 * half * 8))) return rc;
  std::vector<int64_t> hidx(2 * half);
  for (int i = 0; i < half; ++i) { hidx[i] = i; hidx[half + i] = half + i; }
  double* dw = static_cast<double*>(buf.p);
  const double* dbatch = dw + d;
  OTF_CUDA(cudaMemcpyAsync(dw, w, (size_t)d * 8, cudaMemcpyHostToDevice, st));
  OTF_CUDA(cudaMemcpyAsync(const_cast<double*>(dbatch), batch, bb, cudaMemcpyHostToDevice, st));
  OTF_CUDA(cudaMemcpyAsync(idx.p, hidx.data(), (size_t)2 * half * 8, cudaMemcpyHostToDevice, st));
  const int64_t* di = static_cast<const int64_t*>(idx.p);
  // positives and negatives both index the one uploaded batch (rows 0..half-1, half..2h-1)
  rc = launch_pegasos(dw, d, dbatch, OTF_F64, 2 * half, dbatch, OTF_F64, 2 * half, di, di + half, half,
                      shrink, eta_over_b, project, radius, st);
  if (rc) return rc;
  OTF_CUDA(cudaMemcpyAsync(w, dw, (size_t)d * 8, cudaMemcpyDeviceToHost, st));
  OTF_CUDA(cudaStreamSynchronize(st));
  buf.release(); idx.release();
  return OTF_OK;
}

int otf_train_batch(int device, const void* features, int32_t dtype, int64_t n_pos, int64_t n,
                    int32_t d, const int64_t* idx, int64_t total, int32_t bs, int64_t spe,
                    int64_t tail_start, int64_t tail_len, double lam, int project, double* w_out,
                    double* obj_hist, int mem, void* stream) {
  OTF_NVTX("otf_train_batch");
  if (n <= 0 || n_pos <= 0 || n_pos >= n) return fail(OTF_ERR_INSUFFICIENT, "both classes need at least one example");
  if (d <= 0 || bs <= 0 || spe <= 0 || total <= 0) return fail(OTF_ERR_CONFIG, "bad train_batch shape");
  STATELESS_BEGIN(device, mem, stream)
  const size_t es = dtype == OTF_F64 ? 8 : 4;
  const int64_t n_hist = total / spe + 1;
  const void *dX, *di; void *dw, *dh = nullptr;
  if ((rc = S.in(features, (size_t)n * d * es, mem, &dX))) return rc;
  if ((rc = S.in(idx, (size_t)total * bs * 8, mem, &di))) return rc;
  if ((rc = S.outbuf(w_out, (size_t)d * 8, mem, &dw))) return rc;
  if (obj_hist && (rc = S.outbuf(obj_hist, (size_t)n_hist * 8, mem, &dh))) return rc;
  if ((rc = launch_batch_train(dX, dtype, n_pos, n, d, static_cast<const int64_t*>(di), total, bs, spe, tail_start,
                               tail_len, lam, project, static_cast<double*>(dw), static_cast<double*>(dh), st)))
    return rc;
  if ((rc = S.out(w_out, dw, (size_t)d * 8, mem))) return rc;
  if (obj_hist) rc = S.out(obj_hist, dh, (size_t)n_hist * 8, mem);
  return rc;
}

int otf_hinge_objective(int device, const void* features, int32_t dtype, int64_t n_pos, int64_t n,
                        int32_t d, const double* w, double lam, double* out, int mem, void* stream) {
  if (n <= 0 || d <= 0) return fail(OTF_ERR_CONFIG, "bad hinge_objective shape");
  STATELESS_BEGIN(device, mem, stream)
  const size_t es = dtype == OTF_F64 ? 8 : 4;
  const void *dX, *dw; void* dout;
  if ((rc = S.in(features, (size_t)n * d * es, mem, &dX))) return rc;
  if ((rc = S.in(w, (size_t)d * 8, mem, &dw))) return rc;
  if ((rc = S.outbuf(out, 8, mem, &dout))) return rc;
  if ((rc = launch_hinge_objective(dX, dtype, n_pos, n, d, static_cast<const double*>(dw), lam,
                                   static_cast<double*>(dout), st))) return rc;
  return S.out(out, dout, 8, mem);
}

int otf_trainer_create(int device, int32_t dim, const void* negatives, int32_t neg_dtype, int64_t n_neg,
                       int mem, otf_trainer** out) {
  *out = nullptr;
  if (n_neg <= 0) return fail(OTF_ERR_INSUFFICIENT, "negative pool must be a non-empty 2-D array");
  if (dim <= 0) return fail(OTF_ERR_CONFIG, "dim must be positive");
  DeviceGuard g(device);
  otf_trainer* t = new otf_trainer();
  t->device = device; t->dim = dim; t->neg_dtype = neg_dtype; t->n_neg = n_neg;
  int rc = make_stream(&t->stream, true);
  const size_t es = neg_dtype == OTF_F64 ? 8 : 4;
  if (!rc) rc = t->neg.ensure((size_t)n_neg * dim * es);
  if (!rc) rc = copy_in(t->neg.p, negatives, (size_t)n_neg * dim * es, mem, t->stream);
  if (!rc) rc = t->w.ensure((size_t)dim * 8);
  if (!rc) { cudaError_t e = cudaMemsetAsync(t->w.p, 0, (size_t)dim * 8, t->stream); if (e) rc = cuda_fail(e, "memset w"); }
  if (!rc) { cudaError_t e = cudaStreamSynchronize(t->stream); if (e) rc = cuda_fail(e, "trainer_create"); }
  if (rc) { otf_trainer_destroy(t); return rc; }
  *out = t;
  return OTF_OK;
}

int otf_trainer_destroy(otf_trainer* t) {
  if (!t) return OTF_OK;
  DeviceGuard g(t->device);
  if (t->stream) cudaStreamSynchronize(t->stream);
  t->w.release(); t->neg.release(); t->pos_pool.release(); t->pos_stage.release(); t->idx.release();
  t->wsnap.release();
  t->h_stage.release(); t->h_idx.release();
  if (t->published) cudaEventDestroy(t->published);
  if (t->consumed) cudaEventDestroy(t->consumed);
  if (t->stream) cudaStreamDestroy(t->stream);
  delete t;
  return OTF_OK;
}

int otf_trainer_append_positives(otf_trainer* t, const void* rows, int32_t dtype, int64_t n_rows, int mem) {
  std::lock_guard<std::mutex> lk(t->mu);
  DeviceGuard g(t->device);
  if (n_rows <= 0) return OTF_OK;
  const size_t rb = (size_t)t->dim * 4;  // device pool is float32 (session.py:70 PositivePool)
  if (dtype != OTF_F32) return fail(OTF_ERR_CONFIG, "device positive pool stores float32 rows");
  if (t->n_pos + n_rows > t->pos_cap) {
    int64_t cap = t->pos_cap > 0 ? t->pos_cap : 64;
    while (cap < t->n_pos + n_rows) cap *= 2;
    DevBuf grown;
    int rc = grown.ensure((size_t)cap * rb);
    if (rc) return rc;
    if (t->n_pos) OTF_CUDA(cudaMemcpyAsync(grown.p, t->pos_pool.p, (size_t)t->n_pos * rb, cudaMemcpyDeviceToDevice, t->stream));
    OTF_CUDA(cudaStreamSynchronize(t->stream));
    t->pos_pool.release();
    t->pos_pool = grown;
    grown.p = nullptr;
    t->pos_cap = cap;
  }
  int rc = copy_in(static_cast<uint8_t*>(t->pos_pool.p) + (size_t)t->n_pos * rb, rows, (size_t)n_rows * rb, mem, t->stream);
  if (rc) return rc;
  OTF_CUDA(cudaStreamSynchronize(t->stream));
  t->n_pos += n_rows;
  return OTF_OK;
}

int otf_trainer_pool_size(const otf_trainer* t, int64_t* n_pos) {
  *n_pos = t->n_pos;
  return OTF_OK;
}

int otf_trainer_step(otf_trainer* t, const void* positives, int32_t pos_dtype, int64_t n_pos,
                     const int64_t* pos_idx, const int64_t* neg_idx, int32_t half, double shrink,
                     double eta_over_b, int project, double radius) {
  OTF_NVTX("otf_trainer_step");
  std::lock_guard<std::mutex> lk(t->mu);
  DeviceGuard g(t->device);
  const int64_t pool = positives ? n_pos : t->n_pos;
  if (pool <= 0) return fail(OTF_ERR_NOT_READY, "no positives available yet");
  if (half <= 0) return fail(OTF_ERR_CONFIG, "batch half must be positive");
  const size_t es = pos_dtype == OTF_F64 ? 8 : 4;
  const size_t rb = (size_t)t->dim * es;
  // host staging: [pos rows (if host pool)] [pos_idx] [neg_idx]
  const size_t idx_bytes = (size_t)2 * half * 8;
  const size_t rows_bytes = positives ? (size_t)half * rb : 0;
  int rc = t->h_stage.ensure(rows_bytes + idx_bytes);
  if (!rc) rc = t->pos_stage.ensure(rows_bytes + idx_bytes);
  if (rc) return rc;
  // the previous step's copies out of h_stage must have completed before we overwrite it
  OTF_CUDA(cudaStreamSynchronize(t->stream));
  uint8_t* hs = static_cast<uint8_t*>(t->h_stage.p);
  int64_t* hidx = reinterpret_cast<int64_t*>(hs + rows_bytes);
  for (int i = 0; i < half; ++i) {
    if (pos_idx[i] < 0 || pos_idx[i] >= pool) return fail(OTF_ERR_CONFIG, "positive index out of range");
    if (neg_idx[i] < 0 || neg_idx[i] >= t->n_neg) return fail(OTF_ERR_CONFIG, "negative index out of range");
    if (positives) {
      std::memcpy(hs + (size_t)i * rb, static_cast<const uint8_t*>(positives) + (size_t)pos_idx[i] * rb, rb);
      hidx[i] = i;
    } else {
      hidx[i] = pos_idx[i];
    }
    hidx[half + i] = neg_idx[i];
  }
  OTF_CUDA(cudaMemcpyAsync(t->pos_stage.p, hs, rows_bytes + idx_bytes, cudaMemcpyHostToDevice, t->stream));
  uint8_t* ds = static_cast<uint8_t*>(t->pos_stage.p);
  const int64_t* d_pidx = reinterpret_cast<const int64_t*>(ds + rows_bytes);
  const void* pos_src = positives ? static_cast<const void*>(ds) : t->pos_pool.p;
  const int pdt = positives ? pos_dtype : OTF_F32;
  return launch_pegasos(static_cast<double*>(t->w.p), t->dim, pos_src, pdt, pool, t->neg.p, t->neg_dtype,
                        t->n_neg, d_pidx, d_pidx + half, half, shrink, eta_over_b, project, radius, t->stream);
}

int otf_trainer_weights(otf_trainer* t, double* out, int mem) {
  std::lock_guard<std::mutex> lk(t->mu);
  DeviceGuard g(t->device);
  OTF_CUDA(cudaMemcpyAsync(out, t->w.p, (size_t)t->dim * 8,
                           mem == OTF_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, t->stream));
  OTF_CUDA(cudaStreamSynchronize(t->stream));
  return OTF_OK;
}

int otf_trainer_set_weights(otf_trainer* t, const double* w, int mem) {
  std::lock_guard<std::mutex> lk(t->mu);
  DeviceGuard g(t->device);
  int rc = copy_in(t->w.p, w, (size_t)t->dim * 8, mem, t->stream);
  if (rc) return rc;
  OTF_CUDA(cudaStreamSynchronize(t->stream));
  return OTF_OK;
}

int otf_trainer_weights_ptr(otf_trainer* t, const double** out) {
  *out = static_cast<const double*>(t->w.p);
  return OTF_OK;
}

int otf_trainer_stream(otf_trainer* t, void** out) {
  *out = t->stream;
  return OTF_OK;
}

}  // extern "C"

// ---- multi-GPU group (otf_group.cu) ---------------------------------------------------------------
struct otf_group {
  int device = 0;
  int n_ranks = 1, rank = 0;
  void* comm = nullptr;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  DevBuf w, loc, all, outbuf;  // w (dim f64); local k x (sc, id, row); gathered; merged output
  HostBuf h_w, h_out;
  TopkWs topk;
};

int otf_group_unique_id(unsigned char id[128]) { return group_unique_id(id); }

int otf_group_create(int device, int32_t n_ranks, int32_t rank, const unsigned char id[128], otf_group** out) {
  if (!out) return fail(OTF_ERR_CONFIG, "out is NULL");
  *out = nullptr;
  if (n_ranks < 1 || rank < 0 || rank >= n_ranks) return fail(OTF_ERR_CONFIG, "rank out of range");
  int ndev = 0;
  int rc = otf_device_count(&ndev);
  if (rc) return rc;
  if (device < 0 || device >= ndev) return fail(OTF_ERR_CONFIG, "device out of range");
  DeviceGuard g(device);
  otf_group* grp = new otf_group();
  grp->device = device;
  grp->n_ranks = n_ranks;
  grp->rank = rank;
  if ((rc = group_comm_create(n_ranks, rank, id, &grp->comm))) { delete grp; return rc; }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (cudaStreamCreateWithPriority(&grp->stream, cudaStreamNonBlocking, lo) != cudaSuccess) {
    group_comm_destroy(grp->comm);
    delete grp;
    return fail(OTF_ERR_CUDA, "cudaStreamCreate failed");
  }
  *out = grp;
  return OTF_OK;
}

int otf_group_destroy(otf_group* g) {
  if (!g) return OTF_OK;
  DeviceGuard dg(g->device);
  if (g->stream) cudaStreamSynchronize(g->stream);
  group_comm_destroy(g->comm);
  g->w.release(); g->loc.release(); g->all.release(); g->outbuf.release();
  g->h_w.release(); g->h_out.release();
  topk_ws_free(&g->topk);
  if (g->stream) cudaStreamDestroy(g->stream);
  delete g;
  return OTF_OK;
}

int otf_group_rank(otf_group* g, otf_repo* r, const double* w, int32_t root, int64_t row_offset, int64_t total_rows,
                   int64_t k, int64_t* out_ids, double* out_scores, int64_t* out_rows, int64_t* out_n, int mem,
                   void* stream) {
  OTF_NVTX("otf_group_rank");
  if (!g || !r) return fail(OTF_ERR_CONFIG, "group or shard is NULL");
  if (r->device != g->device) return fail(OTF_ERR_CONFIG, "shard and group are on different devices");
  if (root < 0 || root >= g->n_ranks) return fail(OTF_ERR_CONFIG, "root out of range");
  std::lock_guard<std::mutex> lg(g->mu);
  std::lock_guard<std::mutex> lk(r->mu);
  DeviceGuard dg(g->device);
  const int64_t k_eff = k < 0 ? 0 : (k > total_rows ? total_rows : k);
  if (out_n) *out_n = k_eff;
  if (k_eff == 0) return OTF_OK;
  cudaStream_t st = mem == OTF_MEM_DEVICE ? pick_stream(g->stream, stream) : g->stream;
  const int64_t d = r->model_dim, P = g->n_ranks;
  int rc = OTF_OK;
  if ((rc = g->w.ensure((size_t)d * 8)) || (rc = g->loc.ensure((size_t)k_eff * 24)) ||
      (rc = g->all.ensure((size_t)P * k_eff * 24)) || (rc = g->outbuf.ensure((size_t)k_eff * 32)))
    return rc;
  double* dw = static_cast<double*>(g->w.p);
  // 1. broadcast w from root
  if (g->rank == root) {
    if (mem == OTF_MEM_HOST) {
      if ((rc = g->h_w.ensure((size_t)d * 8))) return rc;
      std::memcpy(g->h_w.p, w, (size_t)d * 8);
      OTF_CUDA(cudaMemcpyAsync(dw, g->h_w.p, (size_t)d * 8, cudaMemcpyHostToDevice, st));
    } else {
      OTF_CUDA(cudaMemcpyAsync(dw, w, (size_t)d * 8, cudaMemcpyDeviceToDevice, st));
    }
  }
  if ((rc = group_broadcast_f64(g->comm, dw, d, root, st))) return rc;
  // 2. local exact top-k of the shard, in exchange format (global rows, pads)
  double* lsc = static_cast<double*>(g->loc.p);
  int64_t* lid = reinterpret_cast<int64_t*>(lsc + k_eff);
  int64_t* lrow = lid + k_eff;
  const int64_t k_loc = std::min<int64_t>(k_eff, r->n);
  if (k_loc > 0 && (rc = repo_enter(r, st))) return rc;
  if (k_loc > 0 && (rc = rank_device(r, dw, k_loc, lid, lsc, lrow, st))) { repo_leave(r, st); return rc; }
  if (k_loc > 0 && (rc = repo_leave(r, st))) return rc;
  if ((rc = launch_group_finalize(lsc, lid, lrow, k_loc, k_eff, row_offset,
                                  (int64_t(1) << 62) + (int64_t)g->rank * k_eff, st)))
    return rc;
  // 3. allgather the candidates of every rank
  double* asc = static_cast<double*>(g->all.p);
  int64_t* aid = reinterpret_cast<int64_t*>(asc + P * k_eff);
  int64_t* arow = aid + P * k_eff;
  if ((rc = group_allgather_candidates(g->comm, lsc, lid, lrow, k_eff, asc, aid, arow, st))) return rc;
  // 4. exact merge: top-k by (-score, id) of the P*k candidates, then their global rows
  int64_t* mids = static_cast<int64_t*>(g->outbuf.p);
  double* msc = reinterpret_cast<double*>(mids + k_eff);
  int64_t* mpos = reinterpret_cast<int64_t*>(msc + k_eff);
  int64_t* mrow = mpos + k_eff;
  const bool dev = mem == OTF_MEM_DEVICE;
  if ((rc = launch_topk(asc, OTF_F64, P * k_eff, aid, 0, k_eff, &g->topk, false, dev ? out_ids : mids,
                        dev ? out_scores : msc, mpos, g->device, st)))
    return rc;
  if ((rc = launch_gather_i64(arow, mpos, k_eff, 0, dev ? (out_rows ? out_rows : mrow) : mrow, st))) return rc;
  if (dev) return OTF_OK;
  if ((rc = g->h_out.ensure((size_t)k_eff * 32))) return rc;
  OTF_CUDA(cudaMemcpyAsync(g->h_out.p, g->outbuf.p, (size_t)k_eff * 32, cudaMemcpyDeviceToHost, st));
  OTF_CUDA(cudaStreamSynchronize(st));
  const int64_t* h = static_cast<const int64_t*>(g->h_out.p);
  std::memcpy(out_ids, h, (size_t)k_eff * 8);
  std::memcpy(out_scores, h + k_eff, (size_t)k_eff * 8);
  if (out_rows) std::memcpy(out_rows, h + 3 * k_eff, (size_t)k_eff * 8);
  return OTF_OK;
}

// ---- k-means for PQ codebook learning (otf_kmeans.cu) ----------------------------------------
struct otf_kmeans {
  int device = 0;
  int64_t n = 0;
  int dim = 0, k = 0;
  cudaStream_t stream = nullptr;
  DevBuf X, xx, C, cc, assign, best, counts, obj;
  HostBuf h;  // staging for one step's outputs
};

int otf_kmeans_create(int device, const double* data, int64_t n, int32_t dim, int32_t k, otf_kmeans** out) {
  if (!out) return fail(OTF_ERR_CONFIG, "out is NULL");
  *out = nullptr;
  if (n <= 0 || dim <= 0 || k <= 0 || k > 256) return fail(OTF_ERR_CONFIG, "k-means needs n > 0, dim > 0, 1 <= k <= 256");
  DeviceGuard g(device);
  otf_kmeans* h = new otf_kmeans();
  h->device = device; h->n = n; h->dim = dim; h->k = k;
  int rc = OTF_OK;
  if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) rc = fail(OTF_ERR_CUDA, "cudaStreamCreate");
  const size_t xb = (size_t)n * dim * 8;
  if (!rc) rc = h->X.ensure(xb);
  if (!rc) rc = h->xx.ensure((size_t)n * 8);
  if (!rc) rc = h->C.ensure((size_t)k * dim * 8);
  if (!rc) rc = h->cc.ensure((size_t)k * 8);
  if (!rc) rc = h->assign.ensure((size_t)n * 4);
  if (!rc) rc = h->best.ensure((size_t)n * 8);
  if (!rc) rc = h->counts.ensure((size_t)k * 8);
  if (!rc) rc = h->obj.ensure(8);
  if (!rc) rc = h->h.ensure((size_t)n * 4 + (size_t)k * 8 + (size_t)k * dim * 8 + 8);
  if (!rc && cudaMemcpyAsync(h->X.p, data, xb, cudaMemcpyHostToDevice, h->stream) != cudaSuccess)
    rc = fail(OTF_ERR_CUDA, "k-means data upload");
  if (!rc) rc = kmeans_row_norms(static_cast<const double*>(h->X.p), n, dim, static_cast<double*>(h->xx.p), h->stream);
  if (!rc && cudaStreamSynchronize(h->stream) != cudaSuccess) rc = fail(OTF_ERR_CUDA, "k-means setup");
  if (rc) { otf_kmeans_destroy(h); return rc; }
  *out = h;
  return OTF_OK;
}

int otf_kmeans_load(otf_kmeans* h, const double* data) {
  if (!h) return fail(OTF_ERR_CONFIG, "k-means handle is NULL");
  DeviceGuard g(h->device);
  OTF_CUDA(cudaMemcpyAsync(h->X.p, data, (size_t)h->n * h->dim * 8, cudaMemcpyHostToDevice, h->stream));
  int rc = kmeans_row_norms(static_cast<const double*>(h->X.p), h->n, h->dim, static_cast<double*>(h->xx.p),
                            h->stream);
  if (rc) return rc;
  OTF_CUDA(cudaStreamSynchronize(h->stream));
  return OTF_OK;
}

int otf_kmeans_destroy(otf_kmeans* h) {
  if (!h) return OTF_OK;
  DeviceGuard g(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  h->X.release(); h->xx.release(); h->C.release(); h->cc.release(); h->assign.release(); h->best.release();
  h->counts.release(); h->obj.release(); h->h.release();
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return OTF_OK;
}

int otf_kmeans_step(otf_kmeans* h, double* centroids, int32_t* assign, int64_t* counts, double* objective) {
  OTF_NVTX("otf_kmeans_step");
  if (!h) return fail(OTF_ERR_CONFIG, "k-means handle is NULL");
  DeviceGuard g(h->device);
  const size_t cb = (size_t)h->k * h->dim * 8;
  OTF_CUDA(cudaMemcpyAsync(h->C.p, centroids, cb, cudaMemcpyHostToDevice, h->stream));
  int rc = kmeans_step(static_cast<const double*>(h->X.p), static_cast<const double*>(h->xx.p), h->n, h->dim, h->k,
                       static_cast<double*>(h->C.p), static_cast<double*>(h->cc.p), static_cast<int32_t*>(h->assign.p),
                       static_cast<double*>(h->best.p), static_cast<unsigned long long*>(h->counts.p),
                       static_cast<double*>(h->obj.p), h->device, h->stream);
  if (rc) return rc;
  char* hs = static_cast<char*>(h->h.p);
  const size_t ab = (size_t)h->n * 4, kb = (size_t)h->k * 8;
  OTF_CUDA(cudaMemcpyAsync(hs, h->assign.p, ab, cudaMemcpyDeviceToHost, h->stream));
  OTF_CUDA(cudaMemcpyAsync(hs + ab, h->counts.p, kb, cudaMemcpyDeviceToHost, h->stream));
  OTF_CUDA(cudaMemcpyAsync(hs + ab + kb, h->C.p, cb, cudaMemcpyDeviceToHost, h->stream));
  OTF_CUDA(cudaMemcpyAsync(hs + ab + kb + cb, h->obj.p, 8, cudaMemcpyDeviceToHost, h->stream));
  OTF_CUDA(cudaStreamSynchronize(h->stream));
  std::memcpy(assign, hs, ab);
  std::memcpy(counts, hs + ab, kb);
  std::memcpy(centroids, hs + ab + kb, cb);
  std::memcpy(objective, hs + ab + kb + cb, 8);
  return OTF_OK;
}

// ---- snapshot publication: trainer w -> ranker buffer on the device (SURVEY.md §8b threading) ----
// The snapshot lives in the TRAINER (t->wsnap), not in the repository: many sessions share one
// repository (reference service.py:91, one WallRunner per session), so a publication must not be
// overwritable by another session between its publish and its rank.
int otf_trainer_publish(otf_trainer* t, otf_repo* r) {
  OTF_NVTX("otf_trainer_publish");
  if (!t || !r) return fail(OTF_ERR_CONFIG, "trainer or repository is NULL");
  if (t->device != r->device) return fail(OTF_ERR_CONFIG, "trainer and repository are on different devices");
  if (t->dim != r->model_dim)
    return fail(OTF_ERR_CONFIG, "store dim " + std::to_string(r->model_dim) + " does not match model dim " +
                                    std::to_string(t->dim));
  std::lock_guard<std::mutex> lt(t->mu);
  DeviceGuard g(t->device);
  int rc = t->wsnap.ensure((size_t)t->dim * 8);
  if (rc) return rc;
  if (!t->published) OTF_CUDA(cudaEventCreateWithFlags(&t->published, cudaEventDisableTiming));
  // the copy is ordered after every step already enqueued on the trainer stream and before any
  // later one, and after the last ranker's read of the previous snapshot (no host round trip)
  if (t->consumed) OTF_CUDA(cudaStreamWaitEvent(t->stream, t->consumed, 0));
  OTF_CUDA(cudaMemcpyAsync(t->wsnap.p, t->w.p, (size_t)t->dim * 8, cudaMemcpyDeviceToDevice, t->stream));
  OTF_CUDA(cudaEventRecord(t->published, t->stream));
  return OTF_OK;
}

int otf_repo_rank_published(otf_repo* r, otf_trainer* t, int64_t k, int64_t* out_ids, double* out_scores,
                            int64_t* out_rows, int64_t* out_n) {
  OTF_NVTX("otf_repo_rank_published");
  if (!r || !t) return fail(OTF_ERR_CONFIG, "repository or trainer is NULL");
  if (t->device != r->device) return fail(OTF_ERR_CONFIG, "trainer and repository are on different devices");
  if (t->dim != r->model_dim)
    return fail(OTF_ERR_CONFIG, "store dim " + std::to_string(r->model_dim) + " does not match model dim " +
                                    std::to_string(t->dim));
  std::lock_guard<std::mutex> lk(r->mu);
  DeviceGuard g(r->device);
  int64_t k_eff = k < 0 ? 0 : (k > r->n ? r->n : k);
  if (out_n) *out_n = k_eff;
  cudaStream_t st = r->stream;
  const size_t bytes = (size_t)k_eff * 24;
  int rc = r->wpub.ensure((size_t)r->model_dim * 8);
  if (!rc) rc = r->outbuf.ensure(bytes > 0 ? bytes : 8);
  if (!rc) rc = r->h_out.ensure(bytes > 0 ? bytes : 8);
  if (rc) return rc;
  {
    std::lock_guard<std::mutex> lt(t->mu);
    if (!t->published) return fail(OTF_ERR_NOT_READY, "no snapshot published yet");
    if (k_eff == 0) return OTF_OK;
    // this trainer's snapshot -> the repository's ranking buffer, on the ranker's stream
    if ((rc = repo_enter(r, st))) return rc;
    OTF_CUDA(cudaStreamWaitEvent(st, t->published, 0));
    OTF_CUDA(cudaMemcpyAsync(r->wpub.p, t->wsnap.p, (size_t)t->dim * 8, cudaMemcpyDeviceToDevice, st));
    if (!t->consumed) OTF_CUDA(cudaEventCreateWithFlags(&t->consumed, cudaEventDisableTiming));
    OTF_CUDA(cudaEventRecord(t->consumed, st));
  }
  int64_t* d_ids = static_cast<int64_t*>(r->outbuf.p);
  double* d_sc = reinterpret_cast<double*>(d_ids + k_eff);
  int64_t* d_rows = reinterpret_cast<int64_t*>(d_sc + k_eff);
  // the live ranker re-ranks every tau with a new w in the same buffer: one graph replay per tick
  rc = rank_graph_locked(r, static_cast<const double*>(r->wpub.p), k_eff, d_ids, d_sc, d_rows, st);
  if (!rc && cudaMemcpyAsync(r->h_out.p, r->outbuf.p, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    rc = cuda_fail(cudaGetLastError(), "cudaMemcpyAsync");
  if (const int rc2 = repo_leave(r, st)) rc = rc ? rc : rc2;
  if (rc) { cudaStreamSynchronize(st); return rc; }
  OTF_CUDA(cudaStreamSynchronize(st));
  const int64_t* h = static_cast<const int64_t*>(r->h_out.p);
  std::memcpy(out_ids, h, (size_t)k_eff * 8);
  std::memcpy(out_scores, h + k_eff, (size_t)k_eff * 8);
  if (out_rows) std::memcpy(out_rows, h + 2 * k_eff, (size_t)k_eff * 8);
  return OTF_OK;
}
