// otf_ingest.cu — §8(f3): the reference's repository file loaders, straight into HBM.
//
//   OTFR features   load_features      store.py:139-163 (+ Repository.dense,     ranker.py:176-178)
//   OTFC PQ codes   load_pq_codes      pq.py:318-330    (+ Repository.quantized, ranker.py:180-192)
//   OTFH bit codes  load_binary_codes  binary.py:176-187 (+ Repository.binary,   ranker.py:194-209)
//
// Layout (formats.py): 4-byte magic, u32 version (1), the format's header fields, then the
// payload, nothing after it. Header checks, error classes and messages follow formats.py:
// bad magic / version -> FormatError; a short header or payload -> CorruptionError("truncated
// file: expected N bytes of <what>, got M"); trailing bytes -> CorruptionError; an empty feature
// store -> EmptyStoreError.
//
// The payload never passes through a host-side array: worker threads pread() 16 MB chunks of
// the file into pinned staging buffers (two per worker) and each chunk goes to its place in the
// repository's HBM by cudaMemcpyAsync on the worker's stream while the worker reads its next
// chunk, so disk / page-cache reads and PCIe transfers overlap. The checks the reference makes
// on the loaded arrays run on the device afterwards: code values < num_centroids (pq.py:326-329,
// the existing pq_check_codes kernel), zero padding bits in the last byte of each code
// (binary.py:131-140) and the L2 row normalisation of load_features (store.py:32-53,
// normalize_rows: float64 norms in numpy's pairwise order, float64 division, float32 rounding —
// bit-identical to numpy; a zero row -> DegenerateInputError naming the first such row).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <climits>
#include <cstdio>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "otf_common.cuh"
#include "otf_internal.h"
#include "otf_pairwise.cuh"

namespace otf {

// ---- device checks ---------------------------------------------------------------------------
// store.py normalize_rows: x / sqrt(sum x^2) per row in float64 (np.linalg.norm along axis 1 =
// sqrt(add.reduce(x * x)), a pairwise sum per contiguous row), then astype(float32).
__global__ void ingest_normalize_rows(float* __restrict__ X, int64_t n, int d, unsigned long long* first_zero) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    float* x = X + r * d;
    auto sq = [x](int i) { const double v = (double)x[i]; return __dmul_rn(v, v); };
    const double nrm = __dsqrt_rn(pairwise_sum(sq, 0, d));
    if (nrm == 0.0) {
      atomicMin(first_zero, (unsigned long long)r);
      continue;
    }
    for (int i = 0; i < d; ++i) x[i] = __double2float_rn(__ddiv_rn((double)x[i], nrm));
  }
}

// binary.py:131-140: the unused high bits of the final code byte must be zero.
__global__ void ingest_check_padding(const uint8_t* __restrict__ codes, int64_t n, int row_bytes, unsigned mask,
                                     unsigned int* bad) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    if (codes[r * row_bytes + row_bytes - 1] & mask) *bad = 1u;
}

namespace {

// ---- file header (formats.py) -------------------------------------------------------------------
struct File {
  int fd = -1;
  int64_t size = 0;
  std::string path;
  ~File() {
    if (fd >= 0) close(fd);
  }
};

int open_file(const char* path, File* f) {
  f->path = path ? path : "";
  f->fd = open(f->path.c_str(), O_RDONLY | O_CLOEXEC);
  if (f->fd < 0) return fail(OTF_ERR_IO, f->path + ": " + std::strerror(errno));
  struct stat st;
  if (fstat(f->fd, &st) != 0) return fail(OTF_ERR_IO, f->path + ": " + std::strerror(errno));
  f->size = (int64_t)st.st_size;
  return OTF_OK;
}

// read_exact (formats.py:27-32): n bytes at off, or CorruptionError naming what is missing
int read_exact(const File& f, int64_t off, void* buf, size_t n, const char* what) {
  size_t got = 0;
  while (got < n) {
    const ssize_t k = pread(f.fd, static_cast<char*>(buf) + got, n - got, off + (int64_t)got);
    if (k < 0 && errno == EINTR) continue;
    if (k < 0) return fail(OTF_ERR_IO, f.path + ": " + std::strerror(errno));
    if (k == 0) break;
    got += (size_t)k;
  }
  if (got != n)
    return fail(OTF_ERR_CORRUPTION, "truncated file: expected " + std::to_string(n) + " bytes of " + what + ", got " +
                                        std::to_string(got));
  return OTF_OK;
}

// check_magic (formats.py:40-47)
int check_magic(const File& f, const char magic[4]) {
  char got[4];
  int rc = read_exact(f, 0, got, 4, "magic");
  if (rc) return rc;
  if (std::memcmp(got, magic, 4) != 0) {
    std::string g;
    for (char c : got) g += (c >= 32 && c < 127) ? std::string(1, c) : "\\x" + std::to_string((unsigned char)c);
    return fail(OTF_ERR_FORMAT, "bad magic b'" + g + "', expected b'" + std::string(magic, 4) + "'");
  }
  uint32_t version = 0;
  if ((rc = read_exact(f, 4, &version, 4, "format version"))) return rc;
  if (version != 1)
    return fail(OTF_ERR_FORMAT, "unsupported format version " + std::to_string(version) + ", expected 1");
  return OTF_OK;
}

// rows x width bytes, or -1 when that does not fit in an int64 (a corrupt header: "truncated")
int64_t payload_bytes(uint64_t rows, uint64_t width) {
  if (width != 0 && rows > (uint64_t)INT64_MAX / width) return -1;
  return (int64_t)(rows * width);
}

// the payload is the rest of the file: shorter -> truncated, longer -> trailing bytes
int check_payload(const File& f, int64_t off, int64_t bytes, const char* what) {
  if (bytes < 0)
    return fail(OTF_ERR_CORRUPTION, std::string("truncated file: the header's ") + what + " does not fit in a file");
  const int64_t have = std::max<int64_t>(0, f.size - off);
  if (have < bytes)
    return fail(OTF_ERR_CORRUPTION, "truncated file: expected " + std::to_string(bytes) + " bytes of " + what +
                                        ", got " + std::to_string(have));
  if (have > bytes) return fail(OTF_ERR_CORRUPTION, f.path + ": trailing bytes after payload");
  return OTF_OK;
}

// ---- the pipelined file -> HBM copy -------------------------------------------------------------
constexpr size_t kChunk = 16u << 20;

struct Staging {  // pinned buffers, kept for the next load (the allocation costs more than a chunk)
  std::mutex mu;
  std::vector<void*> bufs;
} g_staging;

int get_buffers(size_t count, std::vector<void*>* out) {
  std::lock_guard<std::mutex> lk(g_staging.mu);
  while (g_staging.bufs.size() < count) {
    void* p = nullptr;
    OTF_CUDA(cudaHostAlloc(&p, kChunk, cudaHostAllocDefault));
    g_staging.bufs.push_back(p);
  }
  out->assign(g_staging.bufs.begin(), g_staging.bufs.begin() + count);
  return OTF_OK;
}

int worker_count(int64_t bytes) {
  const char* e = getenv("OTF_INGEST_THREADS");
  int t = e ? std::atoi(e) : 4;
  t = std::max(1, std::min(t, 16));
  const int64_t chunks = (bytes + (int64_t)kChunk - 1) / (int64_t)kChunk;
  return (int)std::max<int64_t>(1, std::min<int64_t>(t, chunks));
}

// bytes [off, off + bytes) of the file -> dst (device memory, or host memory when dst_host)
// (one load at a time: the pinned staging buffers are shared)
std::mutex g_load_mu;

int stream_file(const File& f, int64_t off, int64_t bytes, void* dst, bool dst_host, int device,
                double* t_read = nullptr) {
  if (bytes <= 0) return OTF_OK;
  std::lock_guard<std::mutex> lk(g_load_mu);
  const int T = worker_count(bytes);
  std::vector<void*> bufs;
  int rc = dst_host ? OTF_OK : get_buffers((size_t)2 * T, &bufs);
  if (rc) return rc;
  const int64_t nchunks = (bytes + (int64_t)kChunk - 1) / (int64_t)kChunk;
  std::vector<std::vector<char>> scratch(dst_host ? T : 0);
  for (auto& v : scratch) v.assign(2 * kChunk, 0);  // touched before the timed reads
  std::vector<int> rcs(T, OTF_OK);
  std::vector<std::string> errs(T);
  auto work = [&](int t) {
    cudaStream_t st = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    bool used[2] = {false, false};
    int r = OTF_OK;
    if (!dst_host) {
      cudaSetDevice(device);
      if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming) != cudaSuccess)
        r = cuda_fail(cudaGetLastError(), "ingest stream");
    }
    for (int64_t c = t, j = 0; c < nchunks && !r; c += T, ++j) {
      const int b = (int)(j & 1);
      const int64_t o = c * (int64_t)kChunk;
      const size_t len = (size_t)std::min<int64_t>((int64_t)kChunk, bytes - o);
      if (dst_host) {  // (the read-bandwidth reference: the same reads, no device copy)
        r = read_exact(f, off + o, scratch[t].data() + (size_t)b * kChunk, len, "payload");
        continue;
      }
      void* buf = bufs[(size_t)2 * t + b];
      if (used[b] && cudaEventSynchronize(ev[b]) != cudaSuccess) { r = cuda_fail(cudaGetLastError(), "ingest"); break; }
      if ((r = read_exact(f, off + o, buf, len, "payload"))) break;
      if (cudaMemcpyAsync(static_cast<char*>(dst) + o, buf, len, cudaMemcpyHostToDevice, st) != cudaSuccess ||
          cudaEventRecord(ev[b], st) != cudaSuccess) {
        r = cuda_fail(cudaGetLastError(), "ingest H2D");
        break;
      }
      used[b] = true;
    }
    if (st) {
      if (cudaStreamSynchronize(st) != cudaSuccess && !r) r = cuda_fail(cudaGetLastError(), "ingest H2D");
      cudaEventDestroy(ev[0]);
      cudaEventDestroy(ev[1]);
      cudaStreamDestroy(st);
    }
    rcs[t] = r;
    if (r) errs[t] = otf_last_error();
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  if (t_read) *t_read = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (int t = 0; t < T; ++t)
    if (rcs[t]) return fail(rcs[t], errs[t]);
  return OTF_OK;
}

// OTF_INGEST_TRACE=1: phase times of each load on stderr (tools/ingest_bench.py)
struct Phase {
  bool on = getenv("OTF_INGEST_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[ingest] %-14s %8.2f ms\n", what, std::chrono::duration<double>(now - t).count() * 1e3);
    t = now;
  }
};

int launch_grid(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4096)); }

}  // namespace
}  // namespace otf

using namespace otf;

extern "C" {

int otf_repo_load_dense(int device, const char* path, int normalize, otf_repo** out) {
  OTF_NVTX("otf_repo_load_dense");
  *out = nullptr;
  DeviceGuard g(device);
  File f;
  int rc = open_file(path, &f);
  if (!rc) rc = check_magic(f, "OTFR");
  uint32_t dim = 0;
  uint64_t count = 0;
  if (!rc) rc = read_exact(f, 8, &dim, 4, "dim");
  if (!rc) rc = read_exact(f, 12, &count, 8, "count");
  if (rc) return rc;
  if (dim == 0 || count == 0)
    return fail(OTF_ERR_EMPTY, f.path + ": empty store (count=" + std::to_string(count) + ", dim=" + std::to_string(dim) + ")");
  const int64_t bytes = payload_bytes(count, (uint64_t)dim * 4);
  if ((rc = check_payload(f, 20, bytes, "feature payload"))) return rc;
  float* x = nullptr;
  OTF_CUDA(cudaMalloc(&x, (size_t)bytes));
  rc = stream_file(f, 20, bytes, x, false, device);
  if (!rc && normalize) {
    unsigned long long* fz = nullptr;
    unsigned long long hz = ~0ull;
    if (cudaMalloc(&fz, sizeof(*fz)) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "cudaMalloc");
    if (!rc) {
      cudaMemcpy(fz, &hz, sizeof(hz), cudaMemcpyHostToDevice);
      ingest_normalize_rows<<<launch_grid((int64_t)count), 256>>>(x, (int64_t)count, (int)dim, fz);
      count_launch();
      if (cudaMemcpy(&hz, fz, sizeof(hz), cudaMemcpyDeviceToHost) != cudaSuccess)
        rc = cuda_fail(cudaGetLastError(), "ingest_normalize_rows");
      else if (hz != ~0ull)
        rc = fail(OTF_ERR_DEGENERATE, "row " + std::to_string(hz) + " has zero norm and cannot be normalized");
    }
    if (fz) cudaFree(fz);
  }
  if (!rc) rc = otf_repo_create_dense(device, x, (int64_t)count, (int32_t)dim, nullptr, 0, OTF_MEM_DEVICE, 1, out);
  if (!rc) {
    repo_own_payload(*out);  // the handle frees the loaded payload
  } else {
    cudaFree(x);
  }
  return rc;
}

int otf_repo_load_pq(int device, const char* path, const float* centroids, int32_t num_blocks, int32_t num_centroids,
                     int32_t subdim, const int64_t* ids, otf_repo** out) {
  OTF_NVTX("otf_repo_load_pq");
  *out = nullptr;
  DeviceGuard g(device);
  File f;
  int rc = open_file(path, &f);
  if (!rc) rc = check_magic(f, "OTFC");
  uint64_t count = 0;
  uint32_t blocks = 0;
  if (!rc) rc = read_exact(f, 8, &count, 8, "count");
  if (!rc) rc = read_exact(f, 16, &blocks, 4, "num_blocks");
  if (rc) return rc;
  const int64_t bytes = payload_bytes(count, blocks);
  if ((rc = check_payload(f, 20, bytes, "code payload"))) return rc;
  // Repository.quantized: the codes must have the codebook's block count (ranker.py:188-189)
  if ((int64_t)blocks != (int64_t)num_blocks)
    return fail(OTF_ERR_CONFIG, "codes shape (" + std::to_string(count) + ", " + std::to_string(blocks) +
                                    ") does not match " + std::to_string(num_blocks) + " blocks");
  Phase ph;
  uint8_t* codes = nullptr;
  OTF_CUDA(cudaMalloc(&codes, (size_t)std::max<int64_t>(bytes, 16)));
  ph.mark("cudaMalloc");
  rc = stream_file(f, 20, bytes, codes, false, device);
  ph.mark("file -> HBM");
  // (create_pq checks every code against num_centroids on the device, pq.py:326-329)
  if (!rc)
    rc = otf_repo_create_pq(device, codes, (int64_t)count, centroids, num_blocks, num_centroids, subdim, ids, 0,
                            OTF_MEM_DEVICE, 1, out);
  ph.mark("create + check");
  if (!rc) {
    repo_own_payload(*out);
  } else {
    cudaFree(codes);
  }
  return rc;
}

int otf_repo_load_binary(int device, const char* path, int32_t code_bytes, const int64_t* ids, otf_repo** out,
                         int32_t* out_bits) {
  OTF_NVTX("otf_repo_load_binary");
  *out = nullptr;
  DeviceGuard g(device);
  File f;
  int rc = open_file(path, &f);
  if (!rc) rc = check_magic(f, "OTFH");
  uint64_t count = 0;
  uint32_t bits = 0;
  if (!rc) rc = read_exact(f, 8, &count, 8, "count");
  if (!rc) rc = read_exact(f, 16, &bits, 4, "output_bits");
  if (rc) return rc;
  const int row_bytes = (int)((bits + 7) / 8);
  const int64_t bytes = payload_bytes(count, (uint64_t)row_bytes);
  if ((rc = check_payload(f, 20, bytes, "code payload"))) return rc;
  if (out_bits) *out_bits = (int32_t)bits;
  // Repository.binary: the codes must have the codec's row width (ranker.py:205-206)
  if (code_bytes > 0 && row_bytes != code_bytes)
    return fail(OTF_ERR_CONFIG, "codes shape (" + std::to_string(count) + ", " + std::to_string(row_bytes) +
                                    ") does not match the codec's " + std::to_string(code_bytes) + " code bytes");
  if (bits == 0) return fail(OTF_ERR_CONFIG, "binary repository needs output_bits > 0");
  uint8_t* codes = nullptr;
  OTF_CUDA(cudaMalloc(&codes, (size_t)std::max<int64_t>(bytes, 16)));
  rc = stream_file(f, 20, bytes, codes, false, device);
  const unsigned mask = (bits % 8) ? (0xFFu << (bits % 8)) & 0xFFu : 0u;
  if (!rc && mask && count) {
    unsigned int* bad = nullptr;
    unsigned int hb = 0;
    if (cudaMalloc(&bad, sizeof(*bad)) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "cudaMalloc");
    if (!rc) {
      cudaMemset(bad, 0, sizeof(*bad));
      ingest_check_padding<<<launch_grid((int64_t)count), 256>>>(codes, (int64_t)count, row_bytes, mask, bad);
      count_launch();
      if (cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost) != cudaSuccess)
        rc = cuda_fail(cudaGetLastError(), "ingest_check_padding");
      else if (hb)
        rc = fail(OTF_ERR_CORRUPTION, "nonzero padding bits in final code byte");
    }
    if (bad) cudaFree(bad);
  }
  if (!rc) rc = otf_repo_create_binary(device, codes, (int64_t)count, (int32_t)bits, ids, 0, OTF_MEM_DEVICE, 1, out);
  if (!rc) {
    repo_own_payload(*out);
  } else {
    cudaFree(codes);
  }
  return rc;
}

int otf_file_read_bench(const char* path, int64_t offset, double* seconds, int64_t* bytes_read) {
  File f;
  int rc = open_file(path, &f);
  if (rc) return rc;
  const int64_t bytes = std::max<int64_t>(0, f.size - offset);
  double t = 0.0;
  rc = stream_file(f, offset, bytes, nullptr, true, 0, &t);
  if (seconds) *seconds = t;
  if (bytes_read) *bytes_read = bytes;
  return rc;
}

}  // extern "C"
