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

namespace {
constexpr int SDB_COLLECTIVE_CODE = 6;  // SDB_COLLECTIVE (include/sdb.h)
}

namespace sdb {

int comm_unique_id(void* out128) {
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return SDB_COLLECTIVE_CODE;
    std::memcpy(out128, &id, sizeof(id));
    return 0;
}

int comm_init(Ctx* c, const void* id128) {
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm;
    const ncclResult_t r = ncclCommInitRank(&comm, c->world, id, c->rank);
    if (r != ncclSuccess) {
        set_error(SDB_COLLECTIVE_CODE, (std::string("ncclCommInitRank: ") + ncclGetErrorString(r)).c_str());
        return SDB_COLLECTIVE_CODE;
    }
    c->nccl = comm;
    return 0;
}

void comm_destroy(Ctx* c) {
    if (c->nccl) {
        ncclCommDestroy(static_cast<ncclComm_t>(c->nccl));
        c->nccl = nullptr;
    }
}

// in-place allreduce on `st` (the reference's allreduce_sum contract,
// src/comm.cpp:288-315).  avg = 2: ncclMax (flags); avg = 1: ncclAvg, which NCCL implements for floating
// types as a pre-multiply of every rank's values by 1/K followed by the sum --
// used for the fp16 gradient buckets so the reduced value cannot overflow when
// no rank's value does.  A no-op without a communicator; with a forced 1-rank
// communicator the call is issued (and captured) like at K > 1.
cudaError_t comm_allreduce(Ctx* c, void* buf, int64_t n, int dtype, int avg, cudaStream_t st) {
    if (!c->nccl || n == 0) return cudaSuccess;
    // dtype: kF32, kF16, 2 = int32, 3 = float64
    const ncclDataType_t t = dtype == kF16 ? ncclFloat16
                             : dtype == kF32 ? ncclFloat32
                             : dtype == 3 ? ncclFloat64 : ncclInt32;
    const ncclRedOp_t op = avg == 2 ? ncclMax : (avg ? ncclAvg : ncclSum);
    const ncclResult_t r = ncclAllReduce(buf, buf, static_cast<size_t>(n), t, op, static_cast<ncclComm_t>(c->nccl), st);
    if (r != ncclSuccess) {
        set_error(SDB_COLLECTIVE_CODE, (std::string("ncclAllReduce: ") + ncclGetErrorString(r) + " / " +
                                        ncclGetLastError(static_cast<ncclComm_t>(c->nccl))).c_str());
        c->last_nccl_error = static_cast<int>(r);
        return cudaErrorUnknown;
    }
    return cudaSuccess;
}

static ncclDataType_t nccl_type(int dtype) {
    return dtype == kF16 ? ncclFloat16 : dtype == kF32 ? ncclFloat32 : dtype == 3 ? ncclFloat64 : ncclInt32;
}

static cudaError_t nccl_status(Ctx* c, ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return cudaSuccess;
    set_error(SDB_COLLECTIVE_CODE, (std::string(what) + ": " + ncclGetErrorString(r) + " / " +
                                    ncclGetLastError(static_cast<ncclComm_t>(c->nccl))).c_str());
    c->last_nccl_error = static_cast<int>(r);
    return cudaErrorUnknown;
}

// in-place reduce-scatter of buf[0, K*cnt): this rank's averaged (avg = 1) or
// summed chunk lands at buf + rank*cnt -- the first half of the reference's
// ring allreduce (src/comm.cpp:294-304)
cudaError_t comm_reduce_scatter(Ctx* c, void* buf, int64_t cnt, int dtype, int avg, cudaStream_t st) {
    if (!c->nccl || cnt == 0) return cudaSuccess;
    const size_t es = dtype == kF16 ? 2 : (dtype == 3 ? 8 : 4);
    void* mine = static_cast<uint8_t*>(buf) + static_cast<size_t>(c->rank) * cnt * es;
    return nccl_status(c, ncclReduceScatter(buf, mine, static_cast<size_t>(cnt), nccl_type(dtype), avg ? ncclAvg : ncclSum,
                                            static_cast<ncclComm_t>(c->nccl), st),
                       "ncclReduceScatter");
}

// in-place all-gather: every rank's chunk buf + r*cnt to all ranks (the second
// half of the ring allreduce, src/comm.cpp:305-314)
cudaError_t comm_all_gather(Ctx* c, void* buf, int64_t cnt, int dtype, cudaStream_t st) {
    if (!c->nccl || cnt == 0) return cudaSuccess;
    const size_t es = dtype == kF16 ? 2 : (dtype == 3 ? 8 : 4);
    const void* mine = static_cast<const uint8_t*>(buf) + static_cast<size_t>(c->rank) * cnt * es;
    return nccl_status(c, ncclAllGather(mine, buf, static_cast<size_t>(cnt), nccl_type(dtype),
                                        static_cast<ncclComm_t>(c->nccl), st),
                       "ncclAllGather");
}

cudaError_t comm_allreduce_sum(Ctx* c, void* buf, int64_t n, int dtype, cudaStream_t st) {
    return comm_allreduce(c, buf, n, dtype, 0, st);
}

// asynchronous communicator errors (a peer died, a network failure): the
// watchdog half of the reference's CollectiveError path (src/comm.cpp:270-282)
int comm_async_error(Ctx* c) {
    if (!c->nccl) return 0;
    ncclResult_t a = ncclSuccess;
    if (ncclCommGetAsyncError(static_cast<ncclComm_t>(c->nccl), &a) != ncclSuccess) return 1;
    return a == ncclSuccess || a == ncclInProgress ? 0 : 1;
}

}  // namespace sdb
