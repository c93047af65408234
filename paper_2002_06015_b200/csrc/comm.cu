// Collectives of the hybrid schedule (Algorithm 3) over NCCL on NVLink/NVSwitch:
// reduce_scatter_v (src/dist.cpp:181-220) as ncclReduceScatter with ncclAvg
// over an owner-major padded buffer, all_gather_v (src/dist.cpp:222-237) as
// ncclAllGather.  One communicator per context (one process per GPU).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <vector>

#include "ctx.cuh"

using namespace spngd;

#define SPNGD_NCCL_TRY(expr)                                                                   \
  do {                                                                                         \
    ncclResult_t _r = (expr);                                                                  \
    if (_r != ncclSuccess) return fail(SPNGD_ERR_NCCL, "NCCL %s in %s", ncclGetErrorString(_r), #expr); \
  } while (0)

namespace spngd {
// Grouped ncclReduce(avg) of variable segments to their owners: the
// ReduceScatterV of a partial (stale-gated) statistic set, dist.cpp:510-537.
int comm_reduce_to_owners(spngd_ctx* ctx, const std::vector<OwnerReduce>& ops) {
  if (ops.empty()) return SPNGD_OK;
  if (ctx->world == 1) {
    for (const OwnerReduce& r : ops)
      if (r.send != r.recv && r.count > 0)
        SPNGD_CUDA_TRY(cudaMemcpyAsync(r.recv, r.send, r.count * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
    return SPNGD_OK;
  }
  if (!ctx->comm) return fail(SPNGD_ERR_NCCL, "reduce_to_owners: communicator not initialised");
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(ctx->comm);
  SPNGD_NCCL_TRY(ncclGroupStart());
  for (const OwnerReduce& r : ops)
    SPNGD_NCCL_TRY(ncclReduce(r.send, r.recv, size_t(r.count), ncclFloat, ncclAvg, r.root, comm, ctx->stream));
  SPNGD_NCCL_TRY(ncclGroupEnd());
  return SPNGD_OK;
}

int comm_allreduce_sum_f64(spngd_ctx* ctx, double* buf, int64_t count) {
  if (ctx->world == 1 || count <= 0) return SPNGD_OK;
  if (!ctx->comm) return fail(SPNGD_ERR_NCCL, "allreduce: communicator not initialised");
  SPNGD_NCCL_TRY(ncclAllReduce(buf, buf, size_t(count), ncclDouble, ncclSum, reinterpret_cast<ncclComm_t>(ctx->comm),
                               ctx->stream));
  return SPNGD_OK;
}

void comm_destroy(spngd_ctx* ctx) {
  if (ctx && ctx->comm) {
    ncclCommDestroy(reinterpret_cast<ncclComm_t>(ctx->comm));
    ctx->comm = nullptr;
  }
}
}  // namespace spngd

extern "C" {

int spngd_nccl_unique_id(void* out128) {
  if (!out128) return fail(SPNGD_ERR_INVALID, "spngd_nccl_unique_id: null");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  SPNGD_NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  return SPNGD_OK;
}

int spngd_ctx_init_comm(spngd_ctx* ctx, int world, int rank, const void* id128) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx || !id128 || world < 1 || rank < 0 || rank >= world)
    return fail(SPNGD_ERR_INVALID, "spngd_ctx_init_comm: bad argument");
  ctx->world = world;
  ctx->rank = rank;
  if (world == 1) return SPNGD_OK;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  SPNGD_CUDA_TRY(cudaSetDevice(ctx->device));
  ncclComm_t comm;
  SPNGD_NCCL_TRY(ncclCommInitRank(&comm, world, id, rank));
  ctx->comm = reinterpret_cast<ncclComm*>(comm);
  return SPNGD_OK;
}

int spngd_reduce_scatter_mean(spngd_ctx* ctx, const float* send, float* recv, int64_t count) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx) return fail(SPNGD_ERR_INVALID, "reduce_scatter: ctx is NULL");
  if (ctx->world == 1) {
    if (send != recv && count > 0)
      SPNGD_CUDA_TRY(cudaMemcpyAsync(recv, send, count * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
    return SPNGD_OK;
  }
  if (!ctx->comm) return fail(SPNGD_ERR_NCCL, "reduce_scatter: communicator not initialised");
  SPNGD_NCCL_TRY(ncclReduceScatter(send, recv, size_t(count), ncclFloat, ncclAvg,
                                   reinterpret_cast<ncclComm_t>(ctx->comm), ctx->stream));
  return SPNGD_OK;
}

int spngd_all_gather(spngd_ctx* ctx, const float* send, float* recv, int64_t count) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx) return fail(SPNGD_ERR_INVALID, "all_gather: ctx is NULL");
  if (ctx->world == 1) {
    if (send != recv && count > 0)
      SPNGD_CUDA_TRY(cudaMemcpyAsync(recv, send, count * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
    return SPNGD_OK;
  }
  if (!ctx->comm) return fail(SPNGD_ERR_NCCL, "all_gather: communicator not initialised");
  SPNGD_NCCL_TRY(ncclAllGather(send, recv, size_t(count), ncclFloat, reinterpret_cast<ncclComm_t>(ctx->comm),
                               ctx->stream));
  return SPNGD_OK;
}

}  // extern "C"
