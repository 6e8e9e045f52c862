/*
 * otf_b200.h — C ABI of the B200 (sm_100a) on-the-fly retrieval hot path.
 *
 * This is the drop-in boundary for the reference's scoring / ranking / Pegasos path
 * (arXiv 1407.4764 reference package, /root/reference/pkg/src/otf_retrieval). The reference
 * is pure Python + numpy; its "FFI" for this path is the set of Python functions listed next
 * to each entry point below. The Python host package (paper_1407_4764_b200) binds these
 * symbols with ctypes and keeps the reference's names, argument meaning and error types.
 *
 * Conventions
 *   - Every entry point returns an int status (OTF_OK == 0). On failure, otf_last_error()
 *     returns a thread-local, NUL-terminated message describing the last error of the
 *     calling thread. Status codes map 1:1 onto the reference's exception hierarchy
 *     (errors.py:10-51): see OTF_ERR_*.
 *   - `mem` arguments say where caller pointers live: OTF_MEM_HOST (pageable or pinned host
 *     memory; the call is synchronous and copies in/out) or OTF_MEM_DEVICE (device pointers on
 *     the handle's device; the call is asynchronous on `stream`, a cudaStream_t passed as
 *     void*; NULL is the legacy default stream, as everywhere in CUDA).
 *   - A repository handle serialises its calls (one lock per handle) and orders them on the
 *     GPU: a call on a different stream than the handle's previous call waits (CUDA event) for
 *     that call's work, so the handle's shared workspaces are never used by two streams at once.
 *   - Scores are computed with the semantics of the reference: dense/binary scores are
 *     float32 of <x, float32(w)> (ranker.py:69, :89-93), PQ scores are float64 of the
 *     float64 LUT sum (pq.py:248-276). Ranked lists order by (-score, id) with ties toward
 *     the smallest id (ranker.py:97-143) and report scores as float64.
 *   - No torch types, no C++ types: plain pointers and sizes only.
 */
#ifndef OTF_B200_H
#define OTF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (reference exception it maps to) ---------------------------------- */
#define OTF_OK 0
#define OTF_ERR_CONFIG 1       /* ConfigError            errors.py:30 */
#define OTF_ERR_NOT_READY 2    /* NotReadyError          errors.py:38 */
#define OTF_ERR_INSUFFICIENT 3 /* InsufficientDataError  errors.py:34 */
#define OTF_ERR_CORRUPTION 4   /* CorruptionError        errors.py:18 */
#define OTF_ERR_EMPTY 5        /* EmptyStoreError        errors.py:22 */
#define OTF_ERR_CUDA 6         /* RetrievalError         errors.py:10 (CUDA failure) */
#define OTF_ERR_NCCL 7         /* RetrievalError         errors.py:10 (collective)   */
#define OTF_ERR_FORMAT 8       /* FormatError            errors.py:14 (magic / version) */
#define OTF_ERR_DEGENERATE 9   /* DegenerateInputError   errors.py:26 (zero-norm row) */
#define OTF_ERR_IO 10          /* OSError (open / read of a repository file)           */

#define OTF_MEM_HOST 0
#define OTF_MEM_DEVICE 1

#define OTF_KIND_DENSE 0
#define OTF_KIND_PQ 1
#define OTF_KIND_BINARY 2

#define OTF_F32 0
#define OTF_F64 1

/* ---- library ------------------------------------------------------------------------- */
const char* otf_last_error(void);
int otf_abi_version(void);
int otf_device_count(int* out);
/* Leave n SMs of `device` to other work (a concurrent trainer): the persistent rank kernels
 * (fused dense / PQ selections) size their grids for the remaining SMs. 0 (default) = all.
 * No reference counterpart (the reference trains and ranks on the host). */
int otf_set_reserved_sms(int device, int32_t n);
/* Names of the kernels this build contains, ';'-separated (for launch accounting). */
const char* otf_kernel_names(void);
/* Number of kernel launches issued by this process since load (all devices). */
int64_t otf_launch_count(void);

/* ---- repositories: ranker.py:146-281 (Repository) ------------------------------------ */
typedef struct otf_repo otf_repo;

/* Repository.dense(store) — ranker.py:176-178. data is (n, dim) float32 row-major.
 * ids: n int64 (NULL = id_base + row), in host or device memory (detected from the pointer,
 * independently of mem). If mem == OTF_MEM_DEVICE and borrow != 0 the handle reads `data` in
 * place (caller keeps it alive); otherwise it copies into its own HBM. A device payload is
 * adopted after a device synchronisation (the caller's writes to it, on any stream, are done). */
int otf_repo_create_dense(int device, const float* data, int64_t n, int32_t dim,
                          const int64_t* ids, int64_t id_base, int mem, int borrow,
                          otf_repo** out);

/* Repository.quantized(codebook, codes, ids, names) — ranker.py:180-192.
 * codes (n, num_blocks) uint8; centroids (num_blocks, num_centroids, subdim) float32 host. */
int otf_repo_create_pq(int device, const uint8_t* codes, int64_t n, const float* centroids,
                       int32_t num_blocks, int32_t num_centroids, int32_t subdim,
                       const int64_t* ids, int64_t id_base, int mem, int borrow,
                       otf_repo** out);

/* Repository.binary(codec, codes, ids, names) — ranker.py:194-209.
 * codes (n, ceil(output_bits/8)) uint8, LSB-first bit order (binary.py:106,119). */
int otf_repo_create_binary(int device, const uint8_t* codes, int64_t n, int32_t output_bits,
                           const int64_t* ids, int64_t id_base, int mem, int borrow,
                           otf_repo** out);

/* Repository.without_ids(excluded) — ranker.py:254-270: new handle holding rows `rows`
 * (host int64 row positions, ascending) of `src`, ids preserved, payload gathered on device. */
int otf_repo_subset(const otf_repo* src, const int64_t* rows, int64_t n_keep, otf_repo** out);

int otf_repo_destroy(otf_repo* repo);

/* ---- repository files straight into HBM (§8 f3) --------------------------------------- *
 * The reference loads a file into a host numpy array and then builds the Repository; these read
 * the file in chunks into pinned staging buffers and copy each chunk to the repository's HBM
 * while the next is read (no host-side array of the payload). Header checks and errors follow
 * formats.py: bad magic / version -> OTF_ERR_FORMAT, short file -> OTF_ERR_CORRUPTION ("truncated
 * file ..."), trailing bytes -> OTF_ERR_CORRUPTION, open/read failure -> OTF_ERR_IO.
 * load_features(path, normalize) + Repository.dense — store.py:139-163, ranker.py:176-178:
 * an empty store -> OTF_ERR_EMPTY; normalize != 0 L2-normalises every row on the device exactly as
 * normalize_rows (store.py:32-53); a zero row -> OTF_ERR_DEGENERATE. ids are 0..count-1. */
int otf_repo_load_dense(int device, const char* path, int normalize, otf_repo** out);
/* load_pq_codes(path, num_centroids) + Repository.quantized — pq.py:318-330, ranker.py:180-192.
 * centroids (num_blocks, num_centroids, subdim) float32 host; ids: count int64 or NULL. */
int otf_repo_load_pq(int device, const char* path, const float* centroids, int32_t num_blocks,
                     int32_t num_centroids, int32_t subdim, const int64_t* ids, otf_repo** out);
/* load_binary_codes(path) + Repository.binary — binary.py:176-187, ranker.py:194-209.
 * code_bytes: the codec's ceil(output_bits / 8) (0: any); out_bits receives the file's
 * output_bits; nonzero padding bits -> OTF_ERR_CORRUPTION. */
int otf_repo_load_binary(int device, const char* path, int32_t code_bytes, const int64_t* ids,
                         otf_repo** out, int32_t* out_bits);
/* The loaders' chunked, multi-threaded reads of bytes [offset, EOF) with no device copy: the
 * host read bandwidth the loaders are measured against. */
int otf_file_read_bench(const char* path, int64_t offset, double* seconds, int64_t* bytes_read);

/* count / model_dim / payload_bytes / kind — ranker.py:213-231. */
int otf_repo_info(const otf_repo* repo, int32_t* kind, int64_t* count, int32_t* model_dim,
                  int64_t* payload_bytes, int32_t* device);

/* Repository.score(model) — ranker.py:233-240. w: model_dim float64.
 * out: count float32 (dense, binary) or float64 (pq). */
int otf_repo_score(otf_repo* repo, const double* w, void* out, int mem, void* stream);

/* Repository.rank(model, k) — ranker.py:272-281 (score + top_k, ranker.py:97-143).
 * Writes n_out = min(max(k,0), count) entries: ids (int64), scores (float64), and
 * optionally rows (int64 row positions, for names; may be NULL). If out_n is non-NULL it
 * receives n_out. With mem == OTF_MEM_DEVICE everything is asynchronous on `stream`. */
int otf_repo_rank(otf_repo* repo, const double* w, int64_t k, int64_t* out_ids,
                  double* out_scores, int64_t* out_rows, int64_t* out_n, int mem,
                  void* stream);

/* Many classifiers over one dense repository (C5b; no single reference call — the reference
 * needs n_cls separate score_dense calls, ranker.py:63-69). W: (n_cls, model_dim) float64.
 * Scores on the tcgen05 tensor cores with 3 split products (float32-level accuracy): FP16
 * (kind::f16) by default, TF32 for data holding inf/NaN or extreme magnitudes;
 * requires model_dim % 32 == 0. out: (n_cls, count) float32, classifier-major.
 * The FP16 form scales the data by a power of two derived from max |x| in ONE pass on the first
 * call (cached in the handle): the payload must not change afterwards (a borrowed buffer that is
 * rewritten needs a new handle). */
int otf_repo_score_many(otf_repo* repo, const double* W, int32_t n_cls, float* out, int mem,
                        void* stream);
/* ... and the exact top-k of each classifier: out_ids / out_scores (n_cls, n_out). */
int otf_repo_rank_many(otf_repo* repo, const double* W, int32_t n_cls, int64_t k, int64_t* out_ids,
                       double* out_scores, int64_t* out_n, int mem, void* stream);

/* Diagnostics (no reference counterpart): how many PQ rank queries of this handle took the
 * cut path's exact fallback (sampled threshold too high, or too many tied candidates). */
int otf_repo_cut_fallbacks(otf_repo* repo, int64_t* out);
/* Measurement hook (no reference counterpart; used by bench.py for the roofline): runs the
 * scoring kernel of otf_repo_rank(k) exactly as rank does (PQ: the cut scan for large n, else the
 * float32-screening bins scan; with the fused histogram and chunk maxima) for a device-resident
 * w on `stream`, times that kernel
 * with CUDA events recorded around its launch(es) on the same stream, and returns the elapsed
 * milliseconds in *ms (synchronises the stream; leaves the rank workspace clean). */
int otf_repo_time_rank_scan(otf_repo* repo, const double* w_dev, int64_t k, float* ms, void* stream);

/* Capture repo's rank(k) for a device-resident w into a CUDA graph and replay it
 * (the live ranker re-ranks every tau with a new w in the same buffer). Device memory only. */
int otf_repo_rank_graph(otf_repo* repo, const double* w_dev, int64_t k, int64_t* ids_dev,
                        double* scores_dev, int64_t* rows_dev, void* stream);

/* ---- stateless primitives (module functions) ------------------------------------------ */
/* score_dense(model, X) — ranker.py:63-69 */
int otf_score_dense(int device, const float* X, int64_t n, int32_t dim, const double* w,
                    float* out, int mem, void* stream);
/* build_score_lut(w, codebook) — pq.py:248-259: lut (M, K) float64 in numpy einsum order. */
int otf_pq_build_lut(int device, const float* centroids, int32_t num_blocks,
                     int32_t num_centroids, int32_t subdim, const double* w, double* lut,
                     int mem, void* stream);
/* score_codes(lut, codes) — pq.py:262-276: float64 numpy pairwise sum over blocks.
 * A code >= num_centroids is reported as OTF_ERR_CORRUPTION (the reference raises a numpy
 * IndexError only when the code is >= the LUT width; documented deviation). */
int otf_pq_score_codes(int device, const double* lut, int32_t num_blocks,
                       int32_t num_centroids, const uint8_t* codes, int64_t n, double* out,
                       int mem, void* stream);
/* score_binary(model, codes, output_bits) — ranker.py:78-94 */
int otf_score_binary(int device, const uint8_t* codes, int64_t n, int32_t output_bits,
                     const double* w, float* out, int mem, void* stream);
/* unpack_bits(codes, output_bits) — binary.py:110-120: (n, output_bits) float32 {0,1}. */
int otf_unpack_bits(int device, const uint8_t* codes, int64_t n, int32_t output_bits,
                    float* out, int mem, void* stream);
/* binarize(codec, X) — binary.py:86-107: frame (output_bits, input_dim) float64 row-major,
 * centering (input_dim) float32, X (n, input_dim) float64 -> (n, ceil(output_bits/8)) u8. */
int otf_binarize(int device, const double* frame, const float* centering, int32_t input_dim,
                 int32_t output_bits, const double* X, int64_t n, uint8_t* out, int mem,
                 void* stream);
/* pq_encode(codebook, vectors) — pq.py:206-230 (ingest): vectors (n, dim) float32, centroids
 * (num_blocks, num_centroids, subdim) float32 -> codes (n, num_blocks) uint8, nearest centroid
 * per block in float64 (argmin_j |c_j|^2 - 2 x.c_j, first minimum). dim != num_blocks*subdim ->
 * OTF_ERR_CONFIG (pq.py:218-219). */
int otf_pq_encode(int device, const float* vectors, int64_t n, int32_t dim, const float* centroids,
                  int32_t num_blocks, int32_t num_centroids, int32_t subdim, uint8_t* out_codes, int mem,
                  void* stream);
/* hamming_distance(a, b) — binary.py:123-128 (row-wise, equal widths). */
int otf_hamming(int device, const uint8_t* a, const uint8_t* b, int64_t n, int32_t width,
                int64_t* out, int mem, void* stream);
/* top_k(scores, k, ids) — ranker.py:97-143. scores float32 (dtype OTF_F32) or float64;
 * ids n int64 or NULL (0..n-1). Output as otf_repo_rank. */
int otf_top_k(int device, const void* scores, int32_t dtype, int64_t n, const int64_t* ids,
              int64_t k, int64_t* out_ids, double* out_scores, int64_t* out_rows,
              int64_t* out_n, int mem, void* stream);

/* ---- Pegasos trainer: trainer.py:51-173 ------------------------------------------------ */
/* _apply_update + pegasos_step gather — trainer.py:51-71, :100-106. Device pointers only.
 * w (d) float64 updated in place; pos (n_pos, d), neg (n_neg, d) of dtype pos_dtype /
 * neg_dtype (OTF_F32 | OTF_F64); pos_idx, neg_idx: `half` device int64 indices each.
 * eta_lam_shrink = 1 - eta*lam and eta_over_b = eta / batch_size are computed by the caller
 * exactly as the reference does in Python doubles; radius = 1/sqrt(lam) (project != 0). */
int otf_pegasos_update(int device, double* w, int32_t d, const void* pos, int32_t pos_dtype,
                       int64_t n_pos, const void* neg, int32_t neg_dtype, int64_t n_neg,
                       const int64_t* pos_idx, const int64_t* neg_idx, int32_t half,
                       double shrink, double eta_over_b, int project, double radius,
                       void* stream);

/* _apply_update on a host batch (trainer.py:51-71): batch (2*half, d) float64 host rows,
 * positives first; w (d) float64 host, updated in place. Stateless pegasos_step primitive. */
int otf_pegasos_step_host(int device, double* w, int32_t d, const double* batch, int32_t half,
                          double shrink, double eta_over_b, int project, double radius);

/* train_batch(positives, negatives, cfg) — trainer.py:204-257. features (n, d): the n_pos
 * positive rows then the negatives, dtype OTF_F32 | OTF_F64; idx: total*bs row indices drawn by
 * the caller exactly as the reference draws them (rng.integers(0, n, size=bs) per step);
 * spe = steps per epoch, tail_start/tail_len as trainer.py:236-238, lam = 1/(c n).
 * w_out: d float64 (the returned model); obj_hist (nullable): total/spe epoch objectives
 * followed by the tail-average objective. Host or device memory per `mem`. */
int otf_train_batch(int device, const void* features, int32_t dtype, int64_t n_pos, int64_t n,
                    int32_t d, const int64_t* idx, int64_t total, int32_t bs, int64_t spe,
                    int64_t tail_start, int64_t tail_len, double lam, int project, double* w_out,
                    double* obj_hist, int mem, void* stream);
/* hinge_objective(w, features, labels, lam) — trainer.py:197-201 (labels: n_pos +1 then -1). */
int otf_hinge_objective(int device, const void* features, int32_t dtype, int64_t n_pos, int64_t n,
                        int32_t d, const double* w, double lam, double* out, int mem, void* stream);

typedef struct otf_trainer otf_trainer;
/* OnlineTrainer(dim, negatives, cfg) — trainer.py:109-143; negatives copied to HBM once. */
int otf_trainer_create(int device, int32_t dim, const void* negatives, int32_t neg_dtype,
                       int64_t n_neg, int mem, otf_trainer** out);
int otf_trainer_destroy(otf_trainer* tr);
/* Append positives to the trainer's device pool (session.py:62-93 PositivePool.append). */
int otf_trainer_append_positives(otf_trainer* tr, const void* rows, int32_t dtype,
                                 int64_t n_rows, int mem);
int otf_trainer_pool_size(const otf_trainer* tr, int64_t* n_pos);
/* One step (trainer.py:145-159) with host-sampled indices (numpy PCG64 stream, as the
 * reference draws them). If `positives` is non-NULL the B/2 sampled rows are taken from
 * that host array (any pool the caller holds); otherwise from the device pool. */
int otf_trainer_step(otf_trainer* tr, const void* positives, int32_t pos_dtype, int64_t n_pos,
                     const int64_t* pos_idx, const int64_t* neg_idx, int32_t half,
                     double shrink, double eta_over_b, int project, double radius);
/* Snapshot copy of w (trainer.py:161-173): host float64 (mem HOST) or device. */
int otf_trainer_weights(otf_trainer* tr, double* out, int mem);
int otf_trainer_set_weights(otf_trainer* tr, const double* w, int mem);
/* Device pointer of w (float64, dim) for zero-copy ranking on the same device. */
int otf_trainer_weights_ptr(otf_trainer* tr, const double** out);
/* The trainer's CUDA stream (high priority; runs concurrently with ranking). */
int otf_trainer_stream(otf_trainer* tr, void** out);
/* Snapshot publication without a host round trip (SURVEY.md §8b threading; the device side of
 * trainer.py:161-173): copy the trainer's current w into the TRAINER's snapshot buffer on the
 * trainer stream (ordered after every step already enqueued) and record an event. `repo` is only
 * checked for device and dim. The trainer keeps stepping on its own buffer meanwhile. */
int otf_trainer_publish(otf_trainer* tr, otf_repo* repo);
/* rank(k) under `tr`'s last published snapshot (ranker.py:272-281, session.py:197-218), host
 * outputs: the repository's stream waits for the publication, copies it into the repository's
 * ranking buffer and ranks, all under the repository's lock — sessions sharing one repository
 * (service.py:91) never rank under each other's weights. NOT_READY before the first publish. */
int otf_repo_rank_published(otf_repo* repo, otf_trainer* tr, int64_t k, int64_t* out_ids, double* out_scores,
                            int64_t* out_rows, int64_t* out_n);

/* ---- PQ codebook learning (learn_pq_codebook / _lloyd, pq.py:116-203) --------------------------
 * A handle keeps one block's float64 training sub-vectors (n, dim) on the device. Each step is
 * _assign (pq.py:100-113) + the plain mean update (pq.py:155-162): on return, assign (n) and
 * counts (k) describe the assignment to the centroids passed in, *objective = sum of the clamped
 * best distances (the history entry), and centroids (k*dim, in/out) hold the means of the
 * clusters with members (others unchanged). The caller runs the convergence test and the
 * empty-cluster re-seeding (pq.py:146-171) on these host copies. */
typedef struct otf_kmeans otf_kmeans;
int otf_kmeans_create(int device, const double* data, int64_t n, int32_t dim, int32_t k, otf_kmeans** out);
/* Replace the training sub-vectors (same n and dim): the next block of learn_pq_codebook. */
int otf_kmeans_load(otf_kmeans* h, const double* data);
int otf_kmeans_destroy(otf_kmeans* h);
int otf_kmeans_step(otf_kmeans* h, double* centroids, int32_t* assign, int64_t* counts, double* objective);

/* ---- multi-GPU group (one process per GPU, shards by image) ------------
 * A native NCCL communicator over the ranks' shard handles. NCCL is loaded at run time
 * (libnccl.so.2, the one torch already mapped if any), so the library itself has no link-time
 * NCCL dependency. Per query: ncclBroadcast of w from `root`, the local exact top-k of this
 * rank's shard (otf_repo_rank), ncclAllGather of k x (float64 score, int64 id, int64 global row)
 * (ranks with fewer than k rows pad with (-inf, 2^62 + rank*k + slot, -1)), then the exact
 * (-score, id) top-k of the gathered candidates on every rank. Ids must be unique across ranks;
 * row scores do not depend on the shard, so results equal a single-GPU rank of all rows.
 * Replaces: the single-process Repository.rank (ranker.py:272-281) at 1/2/4/8 GPUs. */
typedef struct otf_group otf_group;
/* 128-byte ncclUniqueId of a new communicator (rank 0 creates it, the caller distributes it). */
int otf_group_unique_id(unsigned char id[128]);
int otf_group_create(int device, int32_t n_ranks, int32_t rank, const unsigned char id[128], otf_group** out);
int otf_group_destroy(otf_group* g);
/* w: model_dim float64 on `root` (host or device per mem; ignored elsewhere). shard: this rank's
 * repository, its rows are global rows row_offset .. row_offset + count - 1. total_rows: the sum
 * of all shards (k_eff = min(k, total_rows)). Outputs (k_eff entries, every rank): ids, float64
 * scores, global rows (nullable). */
int otf_group_rank(otf_group* g, otf_repo* shard, const double* w, int32_t root, int64_t row_offset,
                   int64_t total_rows, int64_t k, int64_t* out_ids, double* out_scores, int64_t* out_rows,
                   int64_t* out_n, int mem, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* OTF_B200_H */
