// knng_nccl.cu -- NCCL loaded at run time (dlopen) for the multi-GPU insert (knng_nccl.h).
#include <dlfcn.h>
#include <stdio.h>
#include <string.h>

#include <mutex>

#include "knng_nccl.h"

namespace knng {

namespace {
struct NcclApi {
  void *so = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char *(*getErrorString)(ncclResult_t) = nullptr;
  const char *err = nullptr;
};

NcclApi &api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    // the process's NCCL when one is loaded (torch), else the system's
    a.so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!a.so) a.so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.so) a.so = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!a.so) {
      a.err = "libnccl.so.2 not found";
      return;
    }
#define SYM(f, n) *(void **)&a.f = dlsym(a.so, n)
    SYM(getUniqueId, "ncclGetUniqueId");
    SYM(commInitRank, "ncclCommInitRank");
    SYM(commDestroy, "ncclCommDestroy");
    SYM(allGather, "ncclAllGather");
    SYM(allReduce, "ncclAllReduce");
    SYM(groupStart, "ncclGroupStart");
    SYM(groupEnd, "ncclGroupEnd");
    SYM(getErrorString, "ncclGetErrorString");
#undef SYM
    if (!a.getUniqueId || !a.commInitRank || !a.commDestroy || !a.allGather || !a.allReduce || !a.groupStart ||
        !a.groupEnd)
      a.err = "libnccl.so.2 lacks an entry point";
  });
  return a;
}

const char *check(ncclResult_t r) {
  if (r == ncclSuccess) return nullptr;
  static thread_local char buf[256];
  snprintf(buf, sizeof buf, "NCCL error %d: %s", (int)r, api().getErrorString ? api().getErrorString(r) : "?");
  return buf;
}
}  // namespace

const char *nccl_get_unique_id(void *id128) {
  if (api().err) return api().err;
  return check(api().getUniqueId((ncclUniqueId *)id128));
}

const char *nccl_comm_init(void **comm, int world, const void *id128, int rank) {
  if (api().err) return api().err;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof id);
  return check(api().commInitRank((ncclComm_t *)comm, world, id, rank));
}

void nccl_comm_destroy(void *comm) {
  if (comm && !api().err) api().commDestroy((ncclComm_t)comm);
}

const char *nccl_allgather(const void *send, void *recv, size_t count, ncclDataType_t dt, void *comm, cudaStream_t s) {
  if (api().err) return api().err;
  return check(api().allGather(send, recv, count, dt, (ncclComm_t)comm, s));
}

const char *nccl_allreduce_sum(const void *send, void *recv, size_t count, ncclDataType_t dt, void *comm,
                               cudaStream_t s) {
  if (api().err) return api().err;
  return check(api().allReduce(send, recv, count, dt, ncclSum, (ncclComm_t)comm, s));
}

const char *nccl_group_start() {
  if (api().err) return api().err;
  return check(api().groupStart());
}
const char *nccl_group_end() {
  if (api().err) return api().err;
  return check(api().groupEnd());
}

}  // namespace knng
