// knng_nccl.h -- the library's NCCL data plane (multi-GPU insert, Alg. 3 + Alg. 5): NCCL is loaded at
// run time (dlopen of libnccl.so.2 -- the copy torch already loaded when there is one), so the
// library itself runs on one GPU without it.  Internal, not part of the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <stddef.h>

namespace knng {

// NULL on success, else a message (NCCL missing or a call failed)
const char *nccl_get_unique_id(void *id128);
const char *nccl_comm_init(void **comm, int world, const void *id128, int rank);
void nccl_comm_destroy(void *comm);
const char *nccl_allgather(const void *send, void *recv, size_t count, ncclDataType_t dt, void *comm, cudaStream_t s);
const char *nccl_allreduce_sum(const void *send, void *recv, size_t count, ncclDataType_t dt, void *comm, cudaStream_t s);
const char *nccl_group_start();
const char *nccl_group_end();

}  // namespace knng
