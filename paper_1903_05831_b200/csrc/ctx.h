// ctx.h -- the per-GPU/per-rank context behind the opaque sdb_ctx handle.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

struct sdb_ctx {
    int device = 0, rank = 0, world = 1;
    cudaStream_t stream = nullptr;
    void* ws = nullptr;  // grow-only scratch (sized during warm-up, stable afterwards)
    size_t ws_bytes = 0;
    void* nccl = nullptr;  // ncclComm_t when world > 1
    void* scratch(size_t bytes);
};

namespace sdb {
using Ctx = ::sdb_ctx;
int comm_unique_id(void* out128);
int comm_init(Ctx* c, const void* id128);
void comm_destroy(Ctx* c);
}  // namespace sdb
