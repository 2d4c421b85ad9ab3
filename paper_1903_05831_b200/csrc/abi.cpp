// abi.cpp -- the extern "C" boundary (include/sdb.h): argument validation with
// the reference's error taxonomy, context/workspace management, dispatch to
// the sm_100a kernels.  No compute happens on the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sdb.h"
#include "ctx.h"
#include "detect.h"
#include "sdb_internal.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return SDB_OK;
    return fail(SDB_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

cudaStream_t pick(sdb_ctx* ctx, void* stream) {
    return stream ? static_cast<cudaStream_t>(stream) : (ctx ? ctx->stream : nullptr);
}

int check_dtype(int d) { return (d == SDB_F32 || d == SDB_F16) ? SDB_OK : fail(SDB_PARAM, "unknown dtype"); }

// conv2d_out_shape's checks, src/tensor.cpp:157-167
int check_conv(int N, int H, int W, int C, int K, int R, int S, int stride, int pad) {
    if (N < 1 || H < 1 || W < 1 || C < 1 || K < 1 || R < 1 || S < 1)
        return fail(SDB_SHAPE, "conv2d: dims must be >= 1");
    if (stride < 1 || pad < 0) return fail(SDB_SHAPE, "conv2d: stride >= 1, pad >= 0 required");
    if (H + 2 * pad < R || W + 2 * pad < S) return fail(SDB_SHAPE, "conv2d: kernel larger than padded input");
    return SDB_OK;
}

}  // namespace

namespace sdb {
int set_error(int code, const char* msg) { return fail(code, msg); }
}  // namespace sdb

// Grow-only scratch shared by the ABI ops of one context.  Ops that take
// workspace must be issued on ONE stream per context (or be serialised by the
// caller): two streams would race on its contents.  Growing waits for the
// whole device, so a caller stream still reading the old buffer is covered.
void* sdb_ctx::scratch(size_t bytes) {
    if (bytes <= ws_bytes) return ws;
    if (ws) {
        cudaDeviceSynchronize();
        cudaFree(ws);
    }
    ws_bytes = std::max(bytes, ws_bytes * 2);
    if (cudaMalloc(&ws, ws_bytes) != cudaSuccess) {
        ws = nullptr;
        ws_bytes = 0;
    }
    return ws;
}

extern "C" {

const char* sdb_last_error(void) { return g_err.c_str(); }

int sdb_debug_set(int key, int value) {
    if (key == 1) {
        sdb::conv_set_force_simt(value != 0);
        return SDB_OK;
    }
    return fail(SDB_PARAM, "unknown debug key");
}
int sdb_version(void) { return 1; }

int sdb_ctx_create(int device, int rank, int world, const void* nccl_id, sdb_ctx** out) {
    if (!out) return fail(SDB_PARAM, "null out");
    if (world < 1 || rank < 0 || rank >= world) return fail(SDB_PARAM, "invalid rank/world");
    if (int rc = cuda_status(cudaSetDevice(device), "cudaSetDevice")) return rc;
    auto* c = new sdb_ctx();
    c->device = device;
    c->rank = rank;
    c->world = world;
    // the step's critical chain runs on this stream: above the side stream that
    // carries the overlapped wgrads (least priority), below the comm stream
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    const int prio = std::getenv("SDB_FLAT_PRIORITY") ? 0 : (hi < lo ? hi + 1 : hi);
    if (int rc = cuda_status(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio), "stream")) {
        delete c;
        return rc;
    }
    // world > 1 needs the shared id; world == 1 with an id builds a 1-rank
    // communicator, so the data-parallel code path (bucket allreduces inside
    // the captured step, the loss/BN-gradient allreduces) runs on one GPU
    if (world > 1 && !nccl_id) {
        cudaStreamDestroy(c->stream);
        delete c;
        return fail(SDB_PARAM, "world > 1 requires an nccl unique id");
    }
    if (nccl_id) {
        if (int rc = sdb::comm_init(c, nccl_id)) {
            cudaStreamDestroy(c->stream);
            delete c;
            return rc;
        }
    }
    *out = c;
    return SDB_OK;
}

int sdb_ctx_destroy(sdb_ctx* ctx) {
    if (!ctx) return SDB_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    sdb::comm_destroy(ctx);
    if (ctx->ws) cudaFree(ctx->ws);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
    return SDB_OK;
}

void* sdb_ctx_stream(sdb_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

int sdb_synchronize(sdb_ctx* ctx) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    return cuda_status(cudaStreamSynchronize(ctx->stream), "synchronize");
}

int sdb_get_nccl_unique_id(void* out128) { return sdb::comm_unique_id(out128); }

int sdb_device_alloc(sdb_ctx* ctx, size_t bytes, void** out) {
    if (!ctx || !out) return fail(SDB_PARAM, "null argument");
    *out = nullptr;
    if (int rc = cuda_status(cudaSetDevice(ctx->device), "cudaSetDevice")) return rc;
    return cuda_status(cudaMalloc(out, std::max<size_t>(bytes, 16)), "cudaMalloc");
}

int sdb_device_free(sdb_ctx* ctx, void* p) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (int rc = cuda_status(cudaStreamSynchronize(ctx->stream), "synchronize")) return rc;
    return cuda_status(cudaFree(p), "cudaFree");
}

int sdb_copy_to_device(sdb_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (int rc = cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream), "copy h2d"))
        return rc;
    return cuda_status(cudaStreamSynchronize(ctx->stream), "copy h2d");
}

int sdb_copy_to_host(sdb_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (int rc = cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream), "copy d2h"))
        return rc;
    return cuda_status(cudaStreamSynchronize(ctx->stream), "copy d2h");
}

int sdb_conv_fprop(sdb_ctx* ctx, int dtype, const void* x, const void* w, void* y, int N, int H, int W, int C, int K,
                   int R, int S, int stride, int pad, void* stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (int rc = check_conv(N, H, W, C, K, R, S, stride, pad)) return rc;
    const sdb::ConvShape g{N, H, W, C, K, R, S, stride, pad};
    return cuda_status(sdb::conv_fprop(g, dtype, x, w, y, pick(ctx, stream)), "conv_fprop");
}

int sdb_conv_dgrad(sdb_ctx* ctx, int dtype, const void* dy, const void* w, void* dx, int N, int H, int W, int C, int K,
                   int R, int S, int stride, int pad, int accumulate, void* stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (int rc = check_conv(N, H, W, C, K, R, S, stride, pad)) return rc;
    const sdb::ConvShape g{N, H, W, C, K, R, S, stride, pad};
    return cuda_status(sdb::conv_dgrad(g, dtype, dy, w, dx, accumulate, pick(ctx, stream)), "conv_dgrad");
}

int sdb_conv_dgrad_act(sdb_ctx* ctx, int dtype, const void* dy, const void* w, void* dx, int N, int H, int W, int C,
                       int K, int R, int S, int stride, int pad, const void* addend, const void* y, float neg,
                       const void* y_bits, void* stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (int rc = check_conv(N, H, W, C, K, R, S, stride, pad)) return rc;
    if (!y) return fail(SDB_PARAM, "conv_dgrad_act: null activation y");
    const sdb::ConvShape g{N, H, W, C, K, R, S, stride, pad};
    return cuda_status(sdb::conv_dgrad(g, dtype, dy, w, dx, 1, pick(ctx, stream), addend, y, neg,
                                       static_cast<const uint8_t*>(y_bits)),
                       "conv_dgrad_act");
}

int sdb_conv_fprop_stats(sdb_ctx* ctx, int dtype, const void* x, const void* w, void* y, int N, int H, int W, int C,
                         int K, int R, int S, int stride, int pad, float eps, int iabn, float* mean, float* invstd,
                         int* fused, void* stream) {
    if (!ctx) return fail(SDB_PARAM, "conv_fprop_stats needs a context (workspace)");
    if (int rc = check_dtype(dtype)) return rc;
    if (int rc = check_conv(N, H, W, C, K, R, S, stride, pad)) return rc;
    const sdb::ConvShape g{N, H, W, C, K, R, S, stride, pad};
    const int64_t rows = static_cast<int64_t>(N) * g.Ho() * g.Wo();
    if (rows < 2) return fail(SDB_DEGENERATE, "batch norm needs at least 2 values per channel");
    if (!sdb::norm_channels_ok(K)) return fail(SDB_UNSUPPORTED, "norm kernels need C % 8 == 0, C <= 2048, C | 2048");
    const size_t cap = static_cast<size_t>(2 * 148) * 4 * 2 * 256 * sizeof(double);
    const size_t nws = sdb::norm_workspace_bytes(rows, K);
    uint8_t* ws = static_cast<uint8_t*>(ctx->scratch(cap + nws + 256));
    if (!ws) return fail(SDB_CUDA, "workspace allocation failed");
    cudaStream_t st = pick(ctx, stream);
    sdb::ConvStats cs{reinterpret_cast<double*>(ws), cap, 0, 0, 0, 0};
    if (int rc = cuda_status(sdb::conv_fprop(g, dtype, x, w, y, st, &cs), "conv_fprop")) return rc;
    if (fused) *fused = cs.produced;
    const int act = iabn ? 2 : 0;
    if (cs.produced)
        return cuda_status(sdb::bn_forward_conv_stats(dtype, y, nullptr, nullptr, nullptr, mean, invstd, rows, K, eps, act,
                                                      1.0f, cs, st),
                           "conv stats finalize");
    return cuda_status(sdb::bn_forward_stats(dtype, y, mean, invstd, rows, K, eps, act, ws + cap + 256, st),
                       "norm stats");
}

int sdb_conv_dgrad_iabn_bwd(sdb_ctx* ctx, int dtype, const void* dy, const void* w, void* dy_iabn, int N, int H, int W,
                            int C, int K, int R, int S, int pad, const void* y, const float* gamma, const float* beta,
                            const float* invstd, float slope, void* dz, float* dgamma, float* dbeta, int* fused,
                            void* stream) {
    if (!ctx) return fail(SDB_PARAM, "conv_dgrad_iabn_bwd needs a context (workspace)");
    if (int rc = check_dtype(dtype)) return rc;
    if (int rc = check_conv(N, H, W, C, K, R, S, 1, pad)) return rc;
    const int64_t rows = static_cast<int64_t>(N) * H * W;
    if (rows < 2) return fail(SDB_DEGENERATE, "batch norm needs at least 2 values per channel");
    if (!sdb::norm_channels_ok(C)) return fail(SDB_UNSUPPORTED, "norm kernels need C % 8 == 0, C <= 2048, C | 2048");
    if (!(slope > 0.0f)) return fail(SDB_NONINVERTIBLE, "iabn requires a strictly positive leaky slope");
    const sdb::ConvShape g{N, H, W, C, K, R, S, 1, pad};
    const size_t cap = static_cast<size_t>(2 * 148) * 4 * 2 * 256 * sizeof(double);
    const size_t nws = sdb::norm_workspace_bytes(rows, C);
    uint8_t* ws = static_cast<uint8_t*>(ctx->scratch(cap + nws + 2 * C * sizeof(float) + 512));
    if (!ws) return fail(SDB_CUDA, "workspace allocation failed");
    cudaStream_t st = pick(ctx, stream);
    sdb::ConvStats cs{reinterpret_cast<double*>(ws), cap, 0, 0, 0, 0};
    cs.bs_y = y;
    cs.bs_gamma = gamma;
    cs.bs_beta = beta;
    cs.bs_slope = slope;
    if (int rc = cuda_status(sdb::conv_dgrad(g, dtype, dy, w, dy_iabn, 0, st, nullptr, nullptr, 0.f, nullptr, &cs),
                             "conv_dgrad"))
        return rc;
    if (fused) *fused = cs.produced;
    if (cs.produced) {
        float* coef = reinterpret_cast<float*>(ws + cap + 256);
        return cuda_status(sdb::iabn_backward_conv_stats(dtype, dy_iabn, y, gamma, beta, invstd, dz, dgamma, dbeta, rows,
                                                         C, slope, cs, coef, st),
                           "iabn_bwd (fused statistics)");
    }
    return cuda_status(sdb::iabn_backward(dtype, dy_iabn, y, gamma, beta, nullptr, invstd, dz, dgamma, dbeta, rows, C,
                                          slope, ws + cap + 256, st),
                       "iabn_bwd");
}

int sdb_conv_wgrad(sdb_ctx* ctx, int dtype, const void* x, const void* dy, void* dw, int N, int H, int W, int C, int K,
                   int R, int S, int stride, int pad, void* stream) {
    if (!ctx) return fail(SDB_PARAM, "conv_wgrad needs a context (workspace)");
    if (int rc = check_dtype(dtype)) return rc;
    if (int rc = check_conv(N, H, W, C, K, R, S, stride, pad)) return rc;
    const sdb::ConvShape g{N, H, W, C, K, R, S, stride, pad};
    const size_t wsb = sdb::conv_wgrad_workspace(g, dtype);
    void* ws = ctx->scratch(wsb);
    if (!ws) return fail(SDB_CUDA, "workspace allocation failed");
    return cuda_status(sdb::conv_wgrad(g, dtype, x, dy, dw, ws, wsb, pick(ctx, stream)), "conv_wgrad");
}

static int check_norm(int dtype, int64_t rows, int C) {
    if (int rc = check_dtype(dtype)) return rc;
    if (rows < 2) return fail(SDB_DEGENERATE, "batch norm needs at least 2 values per channel");
    if (!sdb::norm_channels_ok(C)) return fail(SDB_UNSUPPORTED, "norm kernels need C % 8 == 0, C <= 2048, C | 2048");
    return SDB_OK;
}

int sdb_bn_fwd(sdb_ctx* ctx, int dtype, const void* x, const float* gamma, const float* beta, void* y, float* mean,
               float* invstd, int64_t rows, int C, float eps, int relu, void* stream) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (int rc = check_norm(dtype, rows, C)) return rc;
    void* ws = ctx->scratch(sdb::norm_workspace_bytes(rows, C));
    return cuda_status(sdb::bn_forward(dtype, x, gamma, beta, y, mean, invstd, rows, C, eps, relu ? 1 : 0, 1.0f, ws,
                                       pick(ctx, stream)),
                       "bn_fwd");
}

int sdb_bn_bwd(sdb_ctx* ctx, int dtype, const void* dy, const void* x, const void* y_relu, const float* gamma,
               const float* mean, const float* invstd, void* dx, float* dgamma, float* dbeta, int64_t rows, int C,
               void* stream) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (int rc = check_norm(dtype, rows, C)) return rc;
    void* ws = ctx->scratch(sdb::norm_workspace_bytes(rows, C));
    return cuda_status(sdb::bn_backward(dtype, dy, x, y_relu, gamma, mean, invstd, dx, dgamma, dbeta, rows, C, ws,
                                        pick(ctx, stream)),
                       "bn_bwd");
}

// SyncBN over the context's ranks: local fp64 sums -> float buffer -> one fp32
// SUM allreduce (NCCL, on the op's stream) -> statistics from the global sums
int sdb_syncbn_fwd(sdb_ctx* ctx, int dtype, const void* x, const float* gamma, const float* beta, void* y,
                   float* mean, float* invstd, float* agg, int64_t rows, int C, float eps, int relu, void* stream) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (!agg) return fail(SDB_PARAM, "syncbn_fwd: null reduction buffer");
    if (int rc = check_dtype(dtype)) return rc;
    // src/syncbn.cpp:47: the GLOBAL count must be >= 2 (ranks hold equal shards)
    if (rows * ctx->world < 2) return fail(SDB_DEGENERATE, "syncbn: global batch count < 2 per channel");
    if (rows < 1 || !sdb::norm_channels_ok(C))
        return fail(SDB_UNSUPPORTED, "norm kernels need C % 8 == 0, C <= 2048, C | 2048 and rows >= 1");
    cudaStream_t st = pick(ctx, stream);
    void* ws = ctx->scratch(sdb::norm_workspace_bytes(rows, C));
    if (int rc = cuda_status(sdb::syncbn_local_sums(dtype, x, rows, C, agg, ws, st), "syncbn_fwd")) return rc;
    if (int rc = cuda_status(sdb::comm_allreduce_sum(ctx, agg, 2 * static_cast<int64_t>(C) + 1, sdb::kF32, st),
                             "syncbn_fwd allreduce"))
        return rc;
    return cuda_status(
        sdb::syncbn_forward_finish(dtype, x, gamma, beta, y, mean, invstd, agg, rows, C, eps, relu ? 1 : 0, st),
        "syncbn_fwd");
}

int sdb_syncbn_bwd(sdb_ctx* ctx, int dtype, const void* dy, const void* x, const void* y_relu, const float* gamma,
                   const float* mean, const float* invstd, const float* agg_fwd, float* red, void* dx, float* dgamma,
                   float* dbeta, int64_t rows, int C, void* stream) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (!agg_fwd || !red) return fail(SDB_PARAM, "syncbn_bwd: null forward statistics / reduction buffer");
    if (int rc = check_dtype(dtype)) return rc;
    if (rows < 1 || !sdb::norm_channels_ok(C))
        return fail(SDB_UNSUPPORTED, "norm kernels need C % 8 == 0, C <= 2048, C | 2048 and rows >= 1");
    cudaStream_t st = pick(ctx, stream);
    void* ws = ctx->scratch(sdb::norm_workspace_bytes(rows, C));
    if (int rc = cuda_status(
            sdb::syncbn_backward_local_sums(dtype, dy, x, y_relu, mean, invstd, red, rows, C, ws, st), "syncbn_bwd"))
        return rc;
    if (int rc = cuda_status(sdb::comm_allreduce_sum(ctx, red, 2 * static_cast<int64_t>(C), sdb::kF32, st),
                             "syncbn_bwd allreduce"))
        return rc;
    return cuda_status(sdb::syncbn_backward_finish(dtype, dy, x, y_relu, gamma, mean, invstd, red, agg_fwd, dx,
                                                   dgamma, dbeta, rows, C, ws, st),
                       "syncbn_bwd");
}

// iabn_forward's contract checks, src/memopt.cpp:229-235
static int check_iabn_params(sdb_ctx* ctx, const float* gamma, int C, float slope, cudaStream_t st) {
    if (!(slope > 0.0f)) return fail(SDB_NONINVERTIBLE, "iabn requires a strictly positive leaky slope");
    std::vector<float> g(static_cast<size_t>(C));
    if (int rc = cuda_status(cudaMemcpyAsync(g.data(), gamma, C * sizeof(float), cudaMemcpyDeviceToHost, st), "gamma"))
        return rc;
    if (int rc = cuda_status(cudaStreamSynchronize(st), "gamma sync")) return rc;
    for (float v : g)
        if (v == 0.0f) return fail(SDB_NONINVERTIBLE, "iabn requires gamma != 0 in every channel");
    (void)ctx;
    return SDB_OK;
}

int sdb_iabn_fwd(sdb_ctx* ctx, int dtype, const void* x, const float* gamma, const float* beta, void* y, float* mean,
                 float* invstd, int64_t rows, int C, float eps, float slope, void* stream) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (int rc = check_norm(dtype, rows, C)) return rc;
    if (int rc = check_iabn_params(ctx, gamma, C, slope, pick(ctx, stream))) return rc;
    void* ws = ctx->scratch(sdb::norm_workspace_bytes(rows, C));
    return cuda_status(
        sdb::bn_forward(dtype, x, gamma, beta, y, mean, invstd, rows, C, eps, 2, slope, ws, pick(ctx, stream)),
        "iabn_fwd");
}

int sdb_iabn_bwd(sdb_ctx* ctx, int dtype, const void* dy, const void* y, const float* gamma, const float* beta,
                 const float* mean, const float* invstd, void* dx, float* dgamma, float* dbeta, int64_t rows, int C,
                 float slope, void* stream) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (int rc = check_norm(dtype, rows, C)) return rc;
    if (!(slope > 0.0f)) return fail(SDB_NONINVERTIBLE, "iabn requires a strictly positive leaky slope");
    void* ws = ctx->scratch(sdb::norm_workspace_bytes(rows, C));
    return cuda_status(sdb::iabn_backward(dtype, dy, y, gamma, beta, mean, invstd, dx, dgamma, dbeta, rows, C, slope,
                                          ws, pick(ctx, stream)),
                       "iabn_bwd");
}

int sdb_nonfinite(sdb_ctx* ctx, int dtype, const void* g, int64_t n, int* flag, void* stream) {
    if (int rc = check_dtype(dtype)) return rc;
    return cuda_status(sdb::nonfinite_check(dtype, g, n, flag, pick(ctx, stream)), "nonfinite");
}

int sdb_fused_sgd(sdb_ctx* ctx, int gdtype, const void* gsum, float* w, float* v, void* w16, int64_t n, float lr,
                  float momentum, const double* scale, double denom_mult, const int* flag, void* stream) {
    if (int rc = check_dtype(gdtype)) return rc;
    if (n < 0) return fail(SDB_CONTRACT, "negative parameter count");
    return cuda_status(sdb::fused_sgd(gdtype, gsum, w, v, static_cast<__half*>(w16), n, lr, momentum, scale,
                                      denom_mult, flag, pick(ctx, stream)),
                       "fused_sgd");
}

int sdb_update_scale(sdb_ctx* ctx, double* scale, int64_t* good_steps, const int* flag, int dynamic,
                     int64_t growth_interval, double growth, double backoff, double min_scale, double max_scale,
                     void* stream) {
    // LossScaleState::validate's policy checks, src/precision.cpp:20-30
    if (growth_interval < 1 || growth <= 1.0 || backoff <= 0.0 || backoff >= 1.0)
        return fail(SDB_CONTRACT, "invalid loss scale policy parameters");
    return cuda_status(sdb::update_scale_device(scale, good_steps, flag, dynamic, growth_interval, growth, backoff,
                                                min_scale, max_scale, pick(ctx, stream)),
                       "update_scale");
}

int sdb_make_anchors(sdb_ctx* ctx, int H, int W, float stride, const float* scales, int n_scales, const float* ratios,
                     int n_ratios, float* out, void* stream) {
    if (H < 1 || W < 1 || n_scales < 1 || n_scales > 8 || n_ratios < 1 || n_ratios > 8)
        return fail(SDB_PARAM, "anchors: bad grid or scale/ratio count (1..8)");
    sdb::AnchorCfg c{};
    c.H = H; c.W = W; c.stride = stride; c.ns = n_scales; c.nr = n_ratios;
    for (int i = 0; i < n_scales; ++i) c.scales[i] = scales[i];
    for (int i = 0; i < n_ratios; ++i) c.ratios[i] = ratios[i];
    return cuda_status(sdb::make_anchors(c, out, pick(ctx, stream)), "make_anchors");
}

int sdb_rpn_proposal(sdb_ctx* ctx, int dtype, const void* logits, const void* deltas, const float* anchors, int n_img,
                     int n_loc, int A, int A_pad, int pre_k, double iou, int post_k, float img_h, float img_w,
                     float* rois, float* roi_scores, int32_t* count, int32_t* topk_order, void* stream) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (int rc = check_dtype(dtype)) return rc;
    if (iou < 0.0 || iou > 1.0) return fail(SDB_PARAM, "iou threshold outside [0,1]");  // postproc.cpp:48
    if (n_img < 1 || n_loc < 1 || A < 1 || A_pad < A || pre_k < 1 || post_k < 1)
        return fail(SDB_SHAPE, "rpn_proposal: bad sizes");
    if (std::min<int64_t>(pre_k, static_cast<int64_t>(n_loc) * A) > 16384)
        return fail(SDB_UNSUPPORTED, "rpn_proposal: pre_k > 16384");
    const size_t wsb = sdb::proposal_workspace_bytes(n_img, n_loc * A, pre_k);
    // one scratch region: the proposal workspace, then the keep positions
    void* ws2 = ctx->scratch(wsb + static_cast<size_t>(n_img) * post_k * 4 + 256);
    if (!ws2) return fail(SDB_CUDA, "workspace allocation failed");
    sdb::ProposalArgs p{};
    p.logits = logits; p.deltas = deltas; p.dtype = dtype; p.anchors = anchors;
    p.n_img = n_img; p.n_loc = n_loc; p.A = A; p.A_pad = A_pad; p.pre_k = pre_k; p.post_k = post_k;
    p.iou_thr = iou; p.img_h = img_h; p.img_w = img_w; p.clip_dw = static_cast<float>(std::log(1000.0 / 16.0));
    p.rois = rois; p.roi_scores = roi_scores; p.count = count; p.topk_order_out = topk_order;
    p.keep_pos = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ws2) + ((wsb + 255) & ~size_t(255)));
    return cuda_status(sdb::rpn_proposals(p, ws2, pick(ctx, stream)), "rpn_proposal");
}

int sdb_roialign_fwd(sdb_ctx* ctx, int dtype, const void* feat, int N, int H, int W, int C, const float* rois, int R,
                     int P, float spatial_scale, int sampling_ratio, void* out, void* stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (C % 8 || P < 1 || sampling_ratio < 1 || R < 0) return fail(SDB_UNSUPPORTED, "roialign: C % 8, P, ratio");
    return cuda_status(sdb::roialign_fwd(dtype, feat, N, H, W, C, rois, R, P, spatial_scale, sampling_ratio, out,
                                         pick(ctx, stream)),
                       "roialign_fwd");
}

int sdb_roialign_bwd(sdb_ctx* ctx, int dtype, const void* dy, int N, int H, int W, int C, const float* rois, int R,
                     int P, float spatial_scale, int sampling_ratio, void* dfeat, void* stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (C % 8 || P < 1 || P > 16 || sampling_ratio < 1 || R < 0)
        return fail(SDB_UNSUPPORTED, "roialign: C % 8, P <= 16, ratio");
    if (!ctx) return fail(SDB_PARAM, "roialign_bwd needs a context (workspace)");
    const size_t wsb = sdb::roialign_bwd_workspace(R, H, W, P, 1, N);
    void* ws = ctx->scratch(wsb);
    if (!ws) return fail(SDB_CUDA, "workspace allocation failed");
    return cuda_status(sdb::roialign_bwd(dtype, dy, N, H, W, C, rois, R, P, spatial_scale, sampling_ratio, dfeat, ws,
                                         wsb, pick(ctx, stream)),
                       "roialign_bwd");
}

int sdb_roialign_fwd_folded(sdb_ctx* ctx, int dtype, const void* feat, int N, int H, int W, int C, const float* rois,
                            int R, int P, float spatial_scale, int sampling_ratio, int bin_step, void* out,
                            void* stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (C % 8 || P < 1 || sampling_ratio < 1 || R < 0 || bin_step < 1)
        return fail(SDB_UNSUPPORTED, "roialign: C % 8, P, ratio, bin_step");
    return cuda_status(sdb::roialign_fwd(dtype, feat, N, H, W, C, rois, R, P, spatial_scale, sampling_ratio, out,
                                         pick(ctx, stream), bin_step),
                       "roialign_fwd");
}

int sdb_roialign_bwd_folded(sdb_ctx* ctx, int dtype, const void* dy, int N, int H, int W, int C, const float* rois,
                            int R, int P, float spatial_scale, int sampling_ratio, int bin_step, void* dfeat,
                            void* stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (!ctx) return fail(SDB_PARAM, "roialign_bwd needs a context (workspace)");
    if (C % 8 || P < 1 || bin_step < 1 || (P + bin_step - 1) / bin_step > 16 || sampling_ratio < 1 || R < 0)
        return fail(SDB_UNSUPPORTED, "roialign: C % 8, pooled bins <= 16, ratio, bin_step");
    const size_t wsb = sdb::roialign_bwd_workspace(R, H, W, P, bin_step, N);
    void* ws = ctx->scratch(wsb);
    if (!ws) return fail(SDB_CUDA, "workspace allocation failed");
    return cuda_status(sdb::roialign_bwd(dtype, dy, N, H, W, C, rois, R, P, spatial_scale, sampling_ratio, dfeat, ws,
                                         wsb, pick(ctx, stream), bin_step),
                       "roialign_bwd");
}

int sdb_softmax_ce(sdb_ctx* ctx, int dtype, const void* logits, int R, int ncls, int ld, const int32_t* labels,
                   const double* grad_scale, double* loss, void* dlogits, void* stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (R < 1 || ncls < 1 || ld < ncls) return fail(SDB_SHAPE, "cross-entropy expects [batch, classes] logits");
    sdb::LossArgs la{grad_scale, loss, 0};
    return cuda_status(sdb::softmax_ce(dtype, logits, R, ncls, ld, labels, dlogits, la, nullptr, pick(ctx, stream)),
                       "softmax_ce");
}

// ---- losses and targets of the detection step (no reference implementation;
// semantics of the restated oracle, oracle/restate.cpp orc_* -- the same
// kernels the training step runs)

static size_t loss_scratch(int64_t rows) {
    return std::max(sdb::loss_workspace_bytes(rows), static_cast<size_t>(rows + 2) * sizeof(double)) + 256;
}

int sdb_rpn_bce(sdb_ctx* ctx, int dtype, const void* logits, int64_t n_loc, int A, int A_pad, const int8_t* labels,
                const double* grad_scale, double* loss, void* dlogits, void* stream) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (int rc = check_dtype(dtype)) return rc;
    if (n_loc < 1 || A < 1 || A_pad < A) return fail(SDB_SHAPE, "rpn_bce: bad sizes");
    void* ws = ctx->scratch(loss_scratch(n_loc * A));
    if (!ws) return fail(SDB_CUDA, "workspace allocation failed");
    sdb::LossArgs la{grad_scale, loss, 0};
    return cuda_status(sdb::sigmoid_bce(dtype, logits, n_loc, A, A_pad, labels, dlogits, la, ws, pick(ctx, stream)),
                       "rpn_bce");
}

int sdb_rpn_smoothl1(sdb_ctx* ctx, int dtype, const void* deltas, int64_t n_loc, int A, int A_pad,
                     const int8_t* labels, const float* targets, double beta, double norm, const double* grad_scale,
                     double* loss, void* ddeltas, void* stream) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (int rc = check_dtype(dtype)) return rc;
    if (n_loc < 1 || A < 1 || A_pad < A) return fail(SDB_SHAPE, "rpn_smoothl1: bad sizes");
    if (!(beta > 0.0) || !(norm > 0.0)) return fail(SDB_PARAM, "rpn_smoothl1: beta and norm must be > 0");
    void* ws = ctx->scratch(loss_scratch(n_loc * A));
    if (!ws) return fail(SDB_CUDA, "workspace allocation failed");
    sdb::LossArgs la{grad_scale, loss, 0};
    return cuda_status(sdb::rpn_smooth_l1(dtype, deltas, n_loc, A, A_pad, labels, targets, beta, norm, ddeltas, la,
                                          ws, pick(ctx, stream)),
                       "rpn_smoothl1");
}

int sdb_smoothl1(sdb_ctx* ctx, int dtype, const void* pred, int R, int ld, const int32_t* labels,
                 const float* targets, double beta, const double* grad_scale, double* loss, void* dpred,
                 void* stream) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (int rc = check_dtype(dtype)) return rc;
    if (R < 1 || ld < 8) return fail(SDB_SHAPE, "smoothl1: bad sizes");
    if (!(beta > 0.0)) return fail(SDB_PARAM, "smoothl1: beta must be > 0");
    void* ws = ctx->scratch(loss_scratch(R));
    if (!ws) return fail(SDB_CUDA, "workspace allocation failed");
    sdb::LossArgs la{grad_scale, loss, 0};
    return cuda_status(sdb::rcnn_smooth_l1(dtype, pred, R, ld, labels, targets, beta, dpred, la, ws,
                                           pick(ctx, stream)),
                       "smoothl1");
}

int sdb_anchor_targets(sdb_ctx* ctx, const float* anchors, int nA, int n_img, const float* gt, int gt_stride,
                       const int32_t* gt_count, float img_h, float img_w, const uint64_t* keys, double fg_thr,
                       double bg_thr, int batch, double fg_frac, int8_t* labels, float* targets, void* stream) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (nA < 1 || n_img < 1 || gt_stride < 1 || batch < 1) return fail(SDB_SHAPE, "anchor_targets: bad sizes");
    if (!(fg_frac >= 0.0 && fg_frac <= 1.0) || bg_thr > fg_thr)
        return fail(SDB_PARAM, "anchor_targets: fg fraction in [0,1], bg threshold <= fg threshold");
    void* ws = ctx->scratch(sdb::anchor_target_workspace_bytes(n_img, nA, gt_stride));
    if (!ws) return fail(SDB_CUDA, "workspace allocation failed");
    sdb::AnchorTargetArgs a{};
    a.anchors = anchors; a.nA = nA; a.n_img = n_img; a.gt = gt; a.gt_stride = gt_stride; a.gt_count = gt_count;
    a.img_h = img_h; a.img_w = img_w; a.keys = keys; a.fg_thr = fg_thr; a.bg_thr = bg_thr; a.batch = batch;
    a.fg_cap = static_cast<int>(fg_frac * batch); a.labels = labels; a.targets = targets;
    return cuda_status(sdb::anchor_targets(a, ws, pick(ctx, stream)), "anchor_targets");
}

int sdb_proposal_targets(sdb_ctx* ctx, const float* proposals, int prop_stride, const int32_t* prop_count,
                         const float* gt, const int32_t* gt_cls, int gt_stride, const int32_t* gt_count, int n_img,
                         const uint64_t* keys, double fg_thr, double bg_hi, double bg_lo, int batch, double fg_frac,
                         float* out_rois, int32_t* out_labels, float* out_targets, int32_t* out_count,
                         void* stream) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (prop_stride < 1 || gt_stride < 1 || n_img < 1 || batch < 1)
        return fail(SDB_SHAPE, "proposal_targets: bad sizes");
    if (!(fg_frac >= 0.0 && fg_frac <= 1.0) || bg_lo > bg_hi)
        return fail(SDB_PARAM, "proposal_targets: fg fraction in [0,1], bg_lo <= bg_hi");
    const int stride = prop_stride + gt_stride;
    const size_t flag_bytes = (static_cast<size_t>(n_img) * stride + 255) & ~size_t(255);
    void* ws = ctx->scratch(flag_bytes + static_cast<size_t>(n_img) * stride * 4);
    if (!ws) return fail(SDB_CUDA, "workspace allocation failed");
    sdb::ProposalTargetArgs a{};
    a.proposals = proposals; a.prop_stride = prop_stride; a.prop_count = prop_count; a.gt = gt; a.gt_cls = gt_cls;
    a.gt_stride = gt_stride; a.gt_count = gt_count; a.keys = keys; a.fg_thr = fg_thr; a.bg_hi = bg_hi;
    a.bg_lo = bg_lo; a.batch = batch; a.fg_cap = static_cast<int>(std::llround(fg_frac * batch)); a.n_img = n_img;
    a.work_flag = static_cast<int8_t*>(ws);
    a.work_arg = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ws) + flag_bytes);
    a.work_stride = stride;
    a.out_rois = out_rois; a.out_labels = out_labels; a.out_targets = out_targets; a.out_src = nullptr;
    a.out_count = out_count;
    return cuda_status(sdb::proposal_targets(a, pick(ctx, stream)), "proposal_targets");
}

// ---- collectives: CommGroup::allreduce_sum (src/comm.cpp:288-315)
int sdb_allreduce_sum(sdb_ctx* ctx, int dtype, void* buf, int64_t n, void* stream) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (dtype != SDB_F32 && dtype != SDB_F16 && dtype != SDB_F64) return fail(SDB_PARAM, "allreduce: dtype");
    if (n < 0) return fail(SDB_SHAPE, "allreduce: negative length");
    const int d = dtype == SDB_F64 ? 3 : dtype;
    if (sdb::comm_allreduce(ctx, buf, n, d, 0, pick(ctx, stream)) != cudaSuccess) return SDB_COLLECTIVE;
    return SDB_OK;
}

int sdb_comm_check(sdb_ctx* ctx) {
    if (!ctx) return fail(SDB_PARAM, "null ctx");
    if (sdb::comm_async_error(ctx)) return fail(SDB_COLLECTIVE, "communicator reported an asynchronous error");
    return SDB_OK;
}

int sdb_cast(sdb_ctx* ctx, int src_dtype, const void* src, int dst_dtype, void* dst, int64_t n, void* stream) {
    cudaStream_t st = pick(ctx, stream);
    if (src_dtype == SDB_F32 && dst_dtype == SDB_F16)
        return cuda_status(sdb::cast_f32_f16(static_cast<const float*>(src), static_cast<__half*>(dst), n, st), "cast");
    if (src_dtype == SDB_F16 && dst_dtype == SDB_F32)
        return cuda_status(sdb::cast_f16_f32(static_cast<const __half*>(src), static_cast<float*>(dst), n, st), "cast");
    return fail(SDB_PARAM, "unsupported cast");
}

}  // extern "C"
