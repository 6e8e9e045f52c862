// otf_group.cu — multi-GPU plumbing of the ranking path: a native NCCL
// communicator, loaded at run time, plus the two small kernels around the exchange.
//
// The reference is single-process (Repository.rank, ranker.py:272-281). Across GPUs the dataset
// shards by image; a query is broadcast(w) -> local exact top-k -> allgather of k candidates per
// rank -> exact top-k of the gathered candidates (a total order on (-score, id), so the merge of
// per-shard top-k lists is the global top-k). The C-ABI entry points are in otf_capi.cu.
//
// NCCL is dlopen'ed (libnccl.so.2): the process that already mapped torch's NCCL reuses it,
// and the library keeps no link-time NCCL dependency (a missing NCCL fails otf_group_* loudly,
// nothing else).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "otf_common.cuh"
#include "otf_internal.h"

namespace otf {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

static const NcclApi* nccl_api() {
  static NcclApi api;
  static int state = 0;  // 0 untried, 1 ok, -1 unavailable
  if (state == 0) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    state = -1;
    if (h) {
      api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
      api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
      api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
      api.broadcast = reinterpret_cast<decltype(api.broadcast)>(dlsym(h, "ncclBroadcast"));
      api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
      api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
      api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
      api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
      if (api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.broadcast && api.all_gather &&
          api.group_start && api.group_end && api.error_string)
        state = 1;
    }
  }
  return state == 1 ? &api : nullptr;
}

static int nccl_fail(const NcclApi* a, ncclResult_t r, const char* what) {
  return fail(OTF_ERR_NCCL, std::string(what) + ": " + (a ? a->error_string(r) : "NCCL unavailable"));
}

#define OTF_NCCL(api, call, what)                         \
  do {                                                    \
    ncclResult_t _r = (call);                             \
    if (_r != ncclSuccess) return nccl_fail(api, _r, what); \
  } while (0)

int group_unique_id(unsigned char* out128) {
  const NcclApi* a = nccl_api();
  if (!a) return fail(OTF_ERR_NCCL, "libnccl.so.2 could not be loaded");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  OTF_NCCL(a, a->get_unique_id(&id), "ncclGetUniqueId");
  memcpy(out128, &id, 128);
  return OTF_OK;
}

int group_comm_create(int n_ranks, int rank, const unsigned char* id128, void** comm) {
  const NcclApi* a = nccl_api();
  if (!a) return fail(OTF_ERR_NCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  memcpy(&id, id128, 128);
  ncclComm_t c = nullptr;
  OTF_NCCL(a, a->comm_init_rank(&c, n_ranks, id, rank), "ncclCommInitRank");
  *comm = c;
  return OTF_OK;
}

void group_comm_destroy(void* comm) {
  const NcclApi* a = nccl_api();
  if (a && comm) a->comm_destroy(static_cast<ncclComm_t>(comm));
}

int group_broadcast_f64(void* comm, double* buf, int64_t n, int root, cudaStream_t st) {
  const NcclApi* a = nccl_api();
  OTF_NCCL(a, a->broadcast(buf, buf, (size_t)n, ncclFloat64, root, static_cast<ncclComm_t>(comm), st),
           "ncclBroadcast");
  return OTF_OK;
}

// The three candidate arrays of every rank in one NCCL group (k entries each per rank).
int group_allgather_candidates(void* comm, const double* sc, const int64_t* ids, const int64_t* rows, int64_t k,
                               double* sc_all, int64_t* ids_all, int64_t* rows_all, cudaStream_t st) {
  const NcclApi* a = nccl_api();
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  OTF_NCCL(a, a->group_start(), "ncclGroupStart");
  ncclResult_t r1 = a->all_gather(sc, sc_all, (size_t)k, ncclFloat64, c, st);
  ncclResult_t r2 = a->all_gather(ids, ids_all, (size_t)k, ncclInt64, c, st);
  ncclResult_t r3 = a->all_gather(rows, rows_all, (size_t)k, ncclInt64, c, st);
  ncclResult_t r4 = a->group_end();
  if (r1 != ncclSuccess) return nccl_fail(a, r1, "ncclAllGather(scores)");
  if (r2 != ncclSuccess) return nccl_fail(a, r2, "ncclAllGather(ids)");
  if (r3 != ncclSuccess) return nccl_fail(a, r3, "ncclAllGather(rows)");
  if (r4 != ncclSuccess) return nccl_fail(a, r4, "ncclGroupEnd");
  return OTF_OK;
}

// Local candidates -> exchange format: rows [0, k_loc) get the shard's global row offset,
// slots [k_loc, k) become pads (-inf, pad_base + slot, -1) that sort after every real entry.
__global__ void group_finalize_local(double* sc, int64_t* ids, int64_t* rows, int64_t k_loc, int64_t k,
                                     int64_t row_offset, int64_t pad_base) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < k_loc) {
      rows[i] += row_offset;
    } else {
      sc[i] = -__longlong_as_double(0x7ff0000000000000LL);  // -inf
      ids[i] = pad_base + i;
      rows[i] = -1;
    }
  }
}

int launch_group_finalize(double* sc, int64_t* ids, int64_t* rows, int64_t k_loc, int64_t k, int64_t row_offset,
                          int64_t pad_base, cudaStream_t st) {
  if (k <= 0) return OTF_OK;
  int64_t grid = (k + 255) / 256;
  if (grid > 1024) grid = 1024;
  group_finalize_local<<<(int)grid, 256, 0, st>>>(sc, ids, rows, k_loc, k, row_offset, pad_base);
  OTF_LAUNCH_CHECK("group_finalize_local");
  return OTF_OK;
}

}  // namespace otf
