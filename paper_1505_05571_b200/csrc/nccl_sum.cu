// nccl_sum.cu — multi-GPU exact sum over NCCL.
//
// Replaces parallel_exact_sum (vector_ops.cpp:172-186): split (vector_ops.cpp:37-49)
// -> per-part sum (sum_segment, :51-62) -> merge_partials (:64-70) -> round.
// Here a part is a GPU's shard.  Per rank, stream-ordered:
//   1. exsum_cuda_sum(shard)   -> this rank's 592-byte exsum_partial record
//                                 (canonical chunks + global first indices of
//                                 +Inf/-Inf/NaN), written into the workspace;
//   2. ncclAllGather            -> nranks records, rank order (NVLink/NVSwitch);
//   3. exsum_cuda_merge         -> chunkwise sum, canonicalise, index-ordered
//                                 specials, round: identical bits on every rank.
// The payload is nranks x 592 B, so the exchange is latency-bound (NCCL picks
// its LL protocol); the three steps are graph-capturable.
//
// NCCL is resolved at run time with dlopen: when torch (or any host program) has
// already loaded a libnccl.so.2, that copy is reused (RTLD_NOLOAD), so this
// library never pins a second NCCL version into the process.

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "exsum_b200.h"
#include "exsum_nvtx.h"

namespace {

struct NcclApi {
  ncclResult_t (*GetVersion)(int *);
  ncclResult_t (*GetUniqueId)(ncclUniqueId *);
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommCount)(const ncclComm_t, int *);
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t);
  bool ok;
};

NcclApi g_api{};
std::once_flag g_once;

void load_nccl() {
  void *h = nullptr;
  const char *env = getenv("EXSUM_NCCL_LIB");
  if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return;
  g_api.GetVersion = reinterpret_cast<decltype(g_api.GetVersion)>(dlsym(h, "ncclGetVersion"));
  g_api.GetUniqueId = reinterpret_cast<decltype(g_api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
  g_api.CommInitRank =
      reinterpret_cast<decltype(g_api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
  g_api.CommDestroy = reinterpret_cast<decltype(g_api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
  g_api.CommCount = reinterpret_cast<decltype(g_api.CommCount)>(dlsym(h, "ncclCommCount"));
  g_api.AllGather = reinterpret_cast<decltype(g_api.AllGather)>(dlsym(h, "ncclAllGather"));
  g_api.ok = g_api.GetVersion && g_api.GetUniqueId && g_api.CommInitRank && g_api.CommDestroy &&
             g_api.CommCount && g_api.AllGather;
}

const NcclApi *nccl() {
  std::call_once(g_once, load_nccl);
  return g_api.ok ? &g_api : nullptr;
}

constexpr size_t kAlign = 256;
size_t align_up(size_t v) { return (v + kAlign - 1) & ~(kAlign - 1); }

// Workspace layout: [sum workspace | own record | nranks gathered records].
size_t record_offset() { return align_up(exsum_cuda_workspace_bytes()); }
size_t gather_offset() { return align_up(record_offset() + sizeof(exsum_partial)); }

}  // namespace

extern "C" {

int exsum_shard_bounds(uint64_t n, int nranks, int rank, uint64_t *begin, uint64_t *end) {
  if (nranks < 1 || rank < 0 || rank >= nranks || !begin || !end) return EXSUM_EINVAL;
  const uint64_t p = static_cast<uint64_t>(nranks), r = static_cast<uint64_t>(rank);
  const uint64_t base = n / p, extra = n % p;
  *begin = r * base + (r < extra ? r : extra);
  *end = *begin + base + (r < extra ? 1 : 0);
  return EXSUM_OK;
}

int exsum_nccl_available(int *version) {
  const NcclApi *api = nccl();
  if (!api) return 0;
  if (version) {
    int v = 0;
    if (api->GetVersion(&v) != ncclSuccess) return 0;
    *version = v;
  }
  return 1;
}

int exsum_nccl_get_unique_id(void *id) {
  if (!id) return EXSUM_EINVAL;
  const NcclApi *api = nccl();
  if (!api) return EXSUM_ENCCL;
  ncclUniqueId u;
  if (api->GetUniqueId(&u) != ncclSuccess) return EXSUM_ENCCL;
  memcpy(id, &u, sizeof u);
  return EXSUM_OK;
}

int exsum_nccl_comm_init(void **comm, int nranks, const void *id, int rank) {
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) return EXSUM_EINVAL;
  const NcclApi *api = nccl();
  if (!api) return EXSUM_ENCCL;
  ncclUniqueId u;
  memcpy(&u, id, sizeof u);
  ncclComm_t c = nullptr;
  if (api->CommInitRank(&c, nranks, u, rank) != ncclSuccess) return EXSUM_ENCCL;
  *comm = c;
  return EXSUM_OK;
}

int exsum_nccl_comm_destroy(void *comm) {
  if (!comm) return EXSUM_EINVAL;
  const NcclApi *api = nccl();
  if (!api) return EXSUM_ENCCL;
  return api->CommDestroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? EXSUM_OK : EXSUM_ENCCL;
}

size_t exsum_nccl_workspace_bytes(int nranks) {
  if (nranks < 1) return 0;
  return gather_offset() + static_cast<size_t>(nranks) * sizeof(exsum_partial);
}

int exsum_nccl_sum(const double *d_shard, size_t n, uint64_t base_index, void *comm,
                   double *d_result, exsum_partial *d_partial, void *d_ws, size_t ws_bytes,
                   void *stream, unsigned flags) {
  EXSUM_NVTX("exsum_nccl_sum");
  if (!comm || !d_ws || (n && !d_shard)) return EXSUM_EINVAL;
  const NcclApi *api = nccl();
  if (!api) return EXSUM_ENCCL;
  int nranks = 0;
  if (api->CommCount(static_cast<ncclComm_t>(comm), &nranks) != ncclSuccess || nranks < 1)
    return EXSUM_ENCCL;
  if (ws_bytes < exsum_nccl_workspace_bytes(nranks)) return EXSUM_ENOMEM;
  unsigned char *ws = static_cast<unsigned char *>(d_ws);
  exsum_partial *rec = reinterpret_cast<exsum_partial *>(ws + record_offset());
  exsum_partial *gathered = reinterpret_cast<exsum_partial *>(ws + gather_offset());
  int st = exsum_cuda_sum_ex(d_shard, n, base_index, nullptr, rec, d_ws, record_offset(), stream,
                             flags);
  if (st != EXSUM_OK) return st;
  if (api->AllGather(rec, gathered, sizeof(exsum_partial), ncclUint8,
                     static_cast<ncclComm_t>(comm),
                     static_cast<cudaStream_t>(stream)) != ncclSuccess)
    return EXSUM_ENCCL;
  return exsum_cuda_merge(gathered, static_cast<size_t>(nranks), d_result, d_partial, stream);
}

}  // extern "C"
