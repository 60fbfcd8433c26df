// crossover_nccl.cu -- the bucket collective (C1) over NVLink 5 / NVSwitch.
//
// Replaces the reference's priced collective: comm.comm_time_allreduce
// (comm.py:87-99) is an alpha-beta formula; here the fused bucket is actually
// summed across ranks with ncclAllReduce on the caller's comm stream.  One
// communicator per process; the unique id travels over torch.distributed's store.
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <cstring>

#include "crossover.h"
#include "crossover_internal.h"

namespace {
int nccl_status(ncclResult_t r, const char* where) {
  if (r == ncclSuccess || r == ncclInProgress) return 0;
  return cs::set_error(CS_ERR_NCCL_BASE + (int)r, "%s: %s", where, ncclGetErrorString(r));
}
}  // namespace

static_assert(sizeof(ncclUniqueId) == CS_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size changed");

extern "C" {

int cs_nccl_version(void) {
  int v = 0;
  if (ncclGetVersion(&v) != ncclSuccess) return -1;
  return v;
}

int cs_nccl_get_unique_id(uint8_t* out) {
  if (out == nullptr) return cs::set_error(CS_ERR_ARG, "cs_nccl_get_unique_id: out is NULL");
  ncclUniqueId id;
  int rc = nccl_status(ncclGetUniqueId(&id), "ncclGetUniqueId");
  if (rc) return rc;
  std::memcpy(out, &id, sizeof(id));
  return 0;
}

int cs_nccl_init(void** comm, int nranks, int rank, const uint8_t* id, int min_ctas,
                 int max_ctas) {
  if (comm == nullptr || id == nullptr || nranks < 1 || rank < 0 || rank >= nranks)
    return cs::set_error(CS_ERR_ARG, "cs_nccl_init: invalid arguments (nranks=%d rank=%d)",
                         nranks, rank);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.blocking = 1;
  if (min_ctas > 0) cfg.minCTAs = min_ctas;
  if (max_ctas > 0) cfg.maxCTAs = max_ctas;
  ncclComm_t c = nullptr;
  int rc = nccl_status(ncclCommInitRankConfig(&c, nranks, uid, rank, &cfg),
                       "ncclCommInitRankConfig");
  if (rc) return rc;
  *comm = (void*)c;
  return 0;
}

int cs_nccl_allreduce_sum_f32(void* comm, const float* send, float* recv, size_t count,
                              void* stream) {
  if (comm == nullptr) return cs::set_error(CS_ERR_ARG, "cs_nccl_allreduce_sum_f32: comm is NULL");
  return nccl_status(ncclAllReduce(send, recv, count, ncclFloat32, ncclSum, (ncclComm_t)comm,
                                   (cudaStream_t)stream),
                     "ncclAllReduce");
}

int cs_nccl_reduce_scatter_sum_f32(void* comm, const float* send, float* recv,
                                   size_t recv_count, void* stream) {
  if (comm == nullptr) return cs::set_error(CS_ERR_ARG, "cs_nccl_reduce_scatter: comm is NULL");
  return nccl_status(ncclReduceScatter(send, recv, recv_count, ncclFloat32, ncclSum,
                                       (ncclComm_t)comm, (cudaStream_t)stream),
                     "ncclReduceScatter");
}

int cs_nccl_all_gather_f32(void* comm, const float* send, float* recv, size_t send_count,
                           void* stream) {
  if (comm == nullptr) return cs::set_error(CS_ERR_ARG, "cs_nccl_all_gather: comm is NULL");
  return nccl_status(ncclAllGather(send, recv, send_count, ncclFloat32, (ncclComm_t)comm,
                                   (cudaStream_t)stream),
                     "ncclAllGather");
}

int cs_nccl_async_error(void* comm) {
  if (comm == nullptr) return cs::set_error(CS_ERR_ARG, "cs_nccl_async_error: comm is NULL");
  ncclResult_t r = ncclSuccess;
  int rc = nccl_status(ncclCommGetAsyncError((ncclComm_t)comm, &r), "ncclCommGetAsyncError");
  if (rc) return rc;
  return nccl_status(r, "NCCL async error");
}

int cs_nccl_abort(void* comm) {
  if (comm == nullptr) return 0;
  return nccl_status(ncclCommAbort((ncclComm_t)comm), "ncclCommAbort");
}

int cs_nccl_destroy(void* comm) {
  if (comm == nullptr) return 0;
  return nccl_status(ncclCommDestroy((ncclComm_t)comm), "ncclCommDestroy");
}

}  // extern "C"
