// ctx.h -- the per-GPU/per-rank context behind the opaque sdb_ctx handle.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

struct sdb_ctx {
    int device = 0, rank = 0, world = 1;
    cudaStream_t stream = nullptr;
    void* ws = nullptr;  // grow-only scratch (sized during warm-up, stable afterwards)
    size_t ws_bytes = 0;
    void* nccl = nullptr;  // ncclComm_t when world > 1 (or a forced 1-rank communicator)
    int last_nccl_error = 0;
    void* scratch(size_t bytes);
};

namespace sdb {
using Ctx = ::sdb_ctx;
int comm_unique_id(void* out128);
int comm_init(Ctx* c, const void* id128);
void comm_destroy(Ctx* c);
cudaError_t comm_allreduce(Ctx* c, void* buf, int64_t n, int dtype, int avg, cudaStream_t st);
cudaError_t comm_allreduce_sum(Ctx* c, void* buf, int64_t n, int dtype, cudaStream_t st);
int comm_async_error(Ctx* c);
cudaError_t comm_reduce_scatter(Ctx* c, void* buf, int64_t cnt, int dtype, int avg, cudaStream_t st);
cudaError_t comm_all_gather(Ctx* c, void* buf, int64_t cnt, int dtype, cudaStream_t st);
}  // namespace sdb
