/* sdb.h -- C ABI of libsdb, the B200-native (sm_100a) SimpleDet Faster R-CNN
 * C4 training-step library.  This is the drop-in boundary for the hot path of
 * the reference engine `simdet` (/root/reference/proj): every entry point
 * below replaces one reference interface, cited as file:line.
 *
 * Conventions
 *   - plain C types only: device pointers (caller-owned), sizes, a stream
 *     handle (cudaStream_t passed as void*; NULL = the context's stream);
 *   - activations NHWC, conv filters KRSC ([out][kh][kw][in]); the reference is
 *     NCHW/OIHW (tensor.hpp:18) -- layout conversion belongs to the caller's
 *     shim;
 *   - dtype: SDB_F32 or SDB_F16 storage; arithmetic always accumulates in
 *     fp32 (conv/matmul) or fp64 (statistics, losses) exactly like the
 *     reference's fp16 contract (src/tensor.cpp:79-82, src/syncbn.cpp:29-39);
 *   - every function returns an sdb_status; the numeric codes mirror the
 *     reference exception taxonomy (include/simdet/errors.hpp:9-40) and
 *     sdb_last_error() returns the message (thread-local);
 *   - no exceptions cross the ABI; one context per GPU/rank, used by one host
 *     thread at a time (the reference's one-CommGroup-per-thread rule,
 *     src/comm.cpp:242-245,451-471).
 */
#ifndef SDB_H_
#define SDB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SDB_OK = 0,
    SDB_SHAPE = 1,          /* simdet::ShapeError            errors.hpp:13  */
    SDB_CONTRACT = 2,       /* simdet::ContractError         errors.hpp:17  */
    SDB_DEGENERATE = 3,     /* simdet::DegenerateBatchError  errors.hpp:23  */
    SDB_NONINVERTIBLE = 4,  /* simdet::NonInvertibleError    errors.hpp:25  */
    SDB_PARAM = 5,          /* simdet::ParamError            errors.hpp:35  */
    SDB_COLLECTIVE = 6,     /* simdet::CollectiveError       errors.hpp:31  */
    SDB_CUDA = 7,           /* CUDA runtime / launch failure                */
    SDB_UNSUPPORTED = 8     /* shape outside the kernels' envelope          */
} sdb_status;

typedef enum { SDB_F32 = 0, SDB_F16 = 1 } sdb_dtype;

typedef struct sdb_ctx sdb_ctx;

const char* sdb_last_error(void);
int sdb_version(void);

/* ---- context: replaces run_workers + CommGroup (src/comm.cpp:242-245,451-471).
 * nccl_id: 128-byte ncclUniqueId shared by all ranks (NULL when world == 1). */
int sdb_ctx_create(int device, int rank, int world, const void* nccl_id, sdb_ctx** out);
int sdb_ctx_destroy(sdb_ctx* ctx);
void* sdb_ctx_stream(sdb_ctx* ctx);
int sdb_get_nccl_unique_id(void* out128);
int sdb_synchronize(sdb_ctx* ctx);

/* ---- convolution: simdet::conv2d (src/tensor.cpp:169-196) and
 * Tape::conv2d backward (src/autograd.cpp:290-320).
 * x [N,H,W,C], w [K,R,S,C], y [N,Ho,Wo,K]; single stride/pad, no bias. */
int sdb_conv_fprop(sdb_ctx* ctx, int dtype, const void* x, const void* w, void* y, int N, int H, int W, int C, int K,
                   int R, int S, int stride, int pad, void* stream);
/* dx (=|+=) conv^T(dy, w); accumulate=1 adds into dx (residual fan-in) */
int sdb_conv_dgrad(sdb_ctx* ctx, int dtype, const void* dy, const void* w, void* dx, int N, int H, int W, int C, int K,
                   int R, int S, int stride, int pad, int accumulate, void* stream);
/* dw = sum over pixels dy (x) im2col(x); deterministic split-K (no atomics) */
int sdb_conv_wgrad(sdb_ctx* ctx, int dtype, const void* x, const void* dy, void* dw, int N, int H, int W, int C, int K,
                   int R, int S, int stride, int pad, void* stream);

/* ---- BatchNorm: syncbn_forward/backward with group == nullptr
 * (src/syncbn.cpp:21-117).  rows = N*H*W; relu=1 fuses the ReLU that follows
 * BN in the reference chain (src/model.cpp:238-245). */
int sdb_bn_fwd(sdb_ctx* ctx, int dtype, const void* x, const float* gamma, const float* beta, void* y, float* mean,
               float* invstd, int64_t rows, int C, float eps, int relu, void* stream);
/* y_relu: the stored BN+ReLU output when relu was fused, else NULL */
int sdb_bn_bwd(sdb_ctx* ctx, int dtype, const void* dy, const void* x, const void* y_relu, const float* gamma,
               const float* mean, const float* invstd, void* dx, float* dgamma, float* dbeta, int64_t rows, int C,
               void* stream);

/* ---- InPlace-ABN: iabn_forward / iabn_backward (src/memopt.cpp:226-327).
 * Backward recomputes from the OUTPUT y only. */
int sdb_iabn_fwd(sdb_ctx* ctx, int dtype, const void* x, const float* gamma, const float* beta, void* y, float* mean,
                 float* invstd, int64_t rows, int C, float eps, float slope, void* stream);
int sdb_iabn_bwd(sdb_ctx* ctx, int dtype, const void* dy, const void* y, const float* gamma, const float* beta,
                 const float* mean, const float* invstd, void* dx, float* dgamma, float* dbeta, int64_t rows, int C,
                 float slope, void* stream);

/* ---- loss-scaled optimizer: has_nonfinite + apply_sgd + fp16 shadow cast
 * (src/trainer.cpp:78-94, 222-227) and update_scale (src/precision.cpp:45-56).
 * flag: device int, OR-accumulated (zero it before the first check).
 * scale: device double (the live loss scale) or NULL for 1.0;
 * denom = (*scale) * denom_mult (denom_mult = K, the world size). */
int sdb_nonfinite(sdb_ctx* ctx, int dtype, const void* g, int64_t n, int* flag, void* stream);
int sdb_fused_sgd(sdb_ctx* ctx, int gdtype, const void* gsum, float* w, float* v, void* w16, int64_t n, float lr,
                  float momentum, const double* scale, double denom_mult, const int* flag, void* stream);
int sdb_update_scale(sdb_ctx* ctx, double* scale, int64_t* good_steps, const int* flag, int dynamic,
                     int64_t growth_interval, double growth, double backoff, double min_scale, double max_scale,
                     void* stream);
/* binary16 RNE round trip / casts (src/half.cpp:9-71) */
int sdb_cast(sdb_ctx* ctx, int src_dtype, const void* src, int dst_dtype, void* dst, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SDB_H_ */
