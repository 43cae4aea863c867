// fcoo_comm.cu — multi-GPU combine: the only cross-GPU step of the
// path is a per-mode sum all-reduce of the partial MTTKRP output over NVLink/NVSwitch (NCCL picks
// NVLS in-switch reduction where available).  One process per GPU; the 128-byte NCCL unique id
// is broadcast by the caller (torch.distributed in the Python binding).
#include <nccl.h>
#include <string.h>

#include "fcoo_internal.cuh"

struct fcoo_comm_s {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
};

namespace fcoo {

fcoo_status comm_allreduce(fcoo_comm_t c, float* buf, size_t count, cudaStream_t s) {
  if (!c || !c->comm) return FCOO_OK;
  ncclResult_t r = ncclAllReduce(buf, buf, count, ncclFloat, ncclSum, c->comm, s);
  if (r != ncclSuccess) return fail(FCOO_ERR_NCCL, "ncclAllReduce: %s", ncclGetErrorString(r));
  count_launch();
  return FCOO_OK;
}

fcoo_status comm_allreduce_f64(fcoo_comm_t c, double* buf, size_t count, cudaStream_t s) {
  if (!c || !c->comm) return FCOO_OK;
  ncclResult_t r = ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, c->comm, s);
  if (r != ncclSuccess) return fail(FCOO_ERR_NCCL, "ncclAllReduce(f64): %s", ncclGetErrorString(r));
  count_launch();
  return FCOO_OK;
}

void comm_rank_size(fcoo_comm_t c, int* rank, int* nranks) {
  *rank = c ? c->rank : 0;
  *nranks = c ? c->nranks : 1;
}

}  // namespace fcoo

extern "C" {

fcoo_status fcoo_comm_unique_id(void* out128) {
  if (!out128) return fcoo::fail(FCOO_ERR_ARG, "NULL out");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fcoo::fail(FCOO_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  memcpy(out128, &id, sizeof(id));
  return FCOO_OK;
}

fcoo_status fcoo_comm_init(int rank, int nranks, const void* uid128, fcoo_comm_t* out) {
  if (!out || !uid128 || nranks < 1 || rank < 0 || rank >= nranks) return fcoo::fail(FCOO_ERR_ARG, "bad comm args");
  fcoo_comm_s* c = new fcoo_comm_s();
  c->rank = rank;
  c->nranks = nranks;
  // a 1-rank communicator is a real NCCL communicator too (the handles never attach it: sharding
  // into one shard drops the comm), so the NCCL path can be exercised on a single GPU
  {
    ncclUniqueId id;
    memcpy(&id, uid128, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      delete c;
      return fcoo::fail(FCOO_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
  }
  *out = c;
  return FCOO_OK;
}

fcoo_status fcoo_comm_destroy(fcoo_comm_t c) {
  if (!c) return FCOO_OK;
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
  return FCOO_OK;
}

fcoo_status fcoo_allreduce_sum(fcoo_comm_t c, float* buf, size_t count, void* stream) {
  if (!c || !buf) return fcoo::fail(FCOO_ERR_ARG, "NULL comm/buf");
  return fcoo::comm_allreduce(c, buf, count, (cudaStream_t)stream);
}

}  // extern "C"
