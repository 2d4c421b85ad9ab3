// comm.cpp -- data-parallel communication over NCCL (NVLink 5 / NVSwitch).
// Replaces the reference's CommGroup ring allreduce (src/comm.cpp:288-315,
// called at src/trainer.cpp:240-242 for the loss and :251 for the gradients).
// One communicator per rank; collectives are issued on the caller's stream so
// they order against the backward kernels through CUDA events, not host syncs.
#include <nccl.h>

#include <cstring>
#include <string>

#include "ctx.h"
#include "sdb_internal.h"

namespace sdb {

int comm_unique_id(void* out128) {
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return 6;
    std::memcpy(out128, &id, sizeof(id));
    return 0;
}

int comm_init(Ctx* c, const void* id128) {
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm;
    if (ncclCommInitRank(&comm, c->world, id, c->rank) != ncclSuccess) return 6;
    c->nccl = comm;
    return 0;
}

void comm_destroy(Ctx* c) {
    if (c->nccl) {
        ncclCommDestroy(static_cast<ncclComm_t>(c->nccl));
        c->nccl = nullptr;
    }
}

// in-place SUM allreduce (the reference's allreduce_sum contract)
cudaError_t comm_allreduce_sum(Ctx* c, void* buf, int64_t n, int dtype, cudaStream_t st) {
    if (c->world == 1 || n == 0) return cudaSuccess;
    // dtype: kF32, kF16, 2 = int32, 3 = float64
    const ncclDataType_t t = dtype == kF16 ? ncclFloat16
                             : dtype == kF32 ? ncclFloat32
                             : dtype == 3 ? ncclFloat64 : ncclInt32;
    const ncclResult_t r =
        ncclAllReduce(buf, buf, static_cast<size_t>(n), t, ncclSum, static_cast<ncclComm_t>(c->nccl), st);
    return r == ncclSuccess ? cudaSuccess : cudaErrorUnknown;
}

}  // namespace sdb
