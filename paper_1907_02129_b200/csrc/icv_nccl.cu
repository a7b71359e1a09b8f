// Filter replication for the batch-sharded convolution (SURVEY.md §8(b),
// §8(e)): the operator shards by image (reference indirect.py:112-125), so
// its only collective is one broadcast of the packed filter from the source
// rank, once per model load, over NVLink 5 / NVSwitch.  NCCL is opened at
// run time (dlopen of libnccl.so.2: the copy torch already loaded, else the
// system one), so libicv.so has no link-time NCCL dependency and the
// single-GPU entry points work where NCCL is absent.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "icv_internal.h"

namespace icv {
namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

const NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      return fn != nullptr;
    };
    a.ok = sym(a.GetUniqueId, "ncclGetUniqueId") && sym(a.CommInitRank, "ncclCommInitRank") &&
           sym(a.CommInitAll, "ncclCommInitAll") && sym(a.Broadcast, "ncclBroadcast") &&
           sym(a.CommDestroy, "ncclCommDestroy") && sym(a.CommCount, "ncclCommCount") &&
           sym(a.GetVersion, "ncclGetVersion") && sym(a.GetErrorString, "ncclGetErrorString");
    if (!a.ok) a.why = "libnccl.so.2 lacks an expected symbol";
  });
  return a;
}

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return ICV_OK;
  return fail(ICV_ERR_CUDA, std::string(what) + ": " + api().GetErrorString(r));
}

int need_api() {
  if (!api().ok) return fail(ICV_ERR_UNSUPPORTED, "NCCL unavailable: " + api().why);
  return ICV_OK;
}

}  // namespace
}  // namespace icv

using namespace icv;

extern "C" {

ICV_API int icv_nccl_version(int32_t* version) {
  if (int s = need_api()) return s;
  int v = 0;
  if (int s = nccl_check(api().GetVersion(&v), "ncclGetVersion")) return s;
  if (version) *version = v;
  return ICV_OK;
}

ICV_API int icv_nccl_unique_id(void* id_out) {
  if (!id_out) return fail(ICV_ERR_ARG, "icv_nccl_unique_id: null output");
  if (int s = need_api()) return s;
  ncclUniqueId id;
  if (int s = nccl_check(api().GetUniqueId(&id), "ncclGetUniqueId")) return s;
  std::memcpy(id_out, &id, sizeof(id));
  return ICV_OK;
}

ICV_API int icv_nccl_init_rank(void** comm, int32_t nranks, const void* unique_id, int32_t rank) {
  if (!comm || !unique_id) return fail(ICV_ERR_ARG, "icv_nccl_init_rank: null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(ICV_ERR_ARG, "icv_nccl_init_rank: bad rank / nranks");
  if (int s = need_api()) return s;
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclComm_t c = nullptr;
  if (int s = nccl_check(api().CommInitRank(&c, nranks, id, rank), "ncclCommInitRank")) return s;
  *comm = c;
  return ICV_OK;
}

ICV_API int icv_nccl_init_all(void** comms, int32_t ndev, const int32_t* devices) {
  if (!comms || ndev < 1) return fail(ICV_ERR_ARG, "icv_nccl_init_all: null output or ndev < 1");
  if (int s = need_api()) return s;
  static_assert(sizeof(ncclComm_t) == sizeof(void*), "communicator handle is a pointer");
  return nccl_check(api().CommInitAll(reinterpret_cast<ncclComm_t*>(comms), ndev, devices), "ncclCommInitAll");
}

ICV_API int icv_nccl_comm_size(void* comm, int32_t* nranks) {
  if (!comm || !nranks) return fail(ICV_ERR_ARG, "icv_nccl_comm_size: null argument");
  if (int s = need_api()) return s;
  int n = 0;
  if (int s = nccl_check(api().CommCount(static_cast<ncclComm_t>(comm), &n), "ncclCommCount")) return s;
  *nranks = n;
  return ICV_OK;
}

ICV_API int icv_nccl_broadcast(const void* sendbuf, void* recvbuf, int64_t bytes, int32_t root, void* comm,
                               void* stream) {
  if (!recvbuf || !comm || bytes < 0) return fail(ICV_ERR_ARG, "icv_nccl_broadcast: bad argument");
  if (int s = need_api()) return s;
  return nccl_check(api().Broadcast(sendbuf ? sendbuf : recvbuf, recvbuf, (size_t)bytes, ncclUint8, root,
                                    static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream)),
                    "ncclBroadcast");
}

ICV_API int icv_nccl_destroy(void* comm) {
  if (!comm) return ICV_OK;
  if (int s = need_api()) return s;
  return nccl_check(api().CommDestroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
}

}  // extern "C"
