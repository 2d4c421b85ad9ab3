// sdb_internal.h -- internal host-side declarations shared by the kernel
// translation units, the C ABI (abi.cpp) and the step driver (detector.cpp).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace sdb {

enum DType { kF32 = 0, kF16 = 1 };

// records the thread-local message returned by sdb_last_error(); returns code
int set_error(int code, const char* msg);

struct ConvShape {
    int N, H, W, C;  // input activation (NHWC)
    int K, R, S;     // filter KRSC
    int stride, pad;
    int Ho() const { return (H + 2 * pad - R) / stride + 1; }
    int Wo() const { return (W + 2 * pad - S) / stride + 1; }
};

// ---- conv.cu
// optional fused output statistics of an fprop (see ConvArgs::stats): when
// `produced`, buf holds [ctas][4][sum | sumsq][bn] fp64 for finalize_conv_stats
struct ConvStats {
    double* buf;
    size_t cap_bytes;
    int produced, ctas, tiles_n, bn;
    // dgrad only: the InPlace-ABN layer whose backward statistics the epilogue
    // reduces ([sum dz | sum dz*xhat] per column, src/memopt.cpp:305-314)
    const void* bs_y = nullptr;
    const float* bs_gamma = nullptr;
    const float* bs_beta = nullptr;
    float bs_slope = 1.0f;
};
cudaError_t conv_fprop(const ConvShape& g, int dtype, const void* x, const void* w, void* y, cudaStream_t st,
                       ConvStats* stats = nullptr);
// accumulate: dx = conv^T(dy, w) + addend (addend = dx itself when null)
// mask (optional): dx = round(dx) * (mask > 0 ? 1 : mask_neg), the backward of
// the ReLU / leaky that produced this layer's input, fused into the epilogue
// mask_bits (optional): sign bitmap of `mask` (bit c%8 of byte [row][c/8] = mask > 0),
// used by the stride-1 residual epilogue instead of the fp16 mask when present
// bstats (optional, fp16 stride-1 dgrads without addend/mask): the output
// feeds an InPlace-ABN backward; its statistics are reduced in the epilogue
// (bstats->produced reports it) for iabn_backward_conv_stats
cudaError_t conv_dgrad(const ConvShape& g, int dtype, const void* dy, const void* w, void* dx, int accumulate,
                       cudaStream_t st, const void* addend = nullptr, const void* mask = nullptr,
                       float mask_neg = 0.0f, const uint8_t* mask_bits = nullptr, ConvStats* bstats = nullptr);
size_t conv_wgrad_workspace(const ConvShape& g, int dtype);
cudaError_t conv_wgrad(const ConvShape& g, int dtype, const void* x, const void* dy, void* dw, void* ws,
                       size_t ws_bytes, cudaStream_t st);
// split-K wgrad whose reduction is deferred: the fp32 partials stay in `ws`
// (which must then not be reused before the batched reduce runs) and the job
// is described for wgrad_reduce_batched (fp16 gradients only)
struct WgradJob {
    const float* ws;
    void* dw;
    int splits, rows, cols;  // partials [splits][rows][cols]
    int transposed;          // 1: rows = R*S*C, cols = K, dw[K][R*S*C] written transposed
};
cudaError_t conv_wgrad_deferred(const ConvShape& g, int dtype, const void* x, const void* dy, void* dw, void* ws,
                                size_t ws_bytes, cudaStream_t st, WgradJob* job);
// nonfinite (optional): OR-ed with 1 when any fp16 gradient written is inf/NaN
cudaError_t wgrad_reduce_batched(const WgradJob* jobs_dev, const int* tile_start_dev, int njobs, int total_tiles,
                                 cudaStream_t st, int* nonfinite = nullptr);
int wgrad_job_tiles(const WgradJob& j);
bool conv_force_simt();
void conv_set_force_simt(bool v);

// ---- norm.cu  (rows = N*H*W, channels innermost)
// workspace: norm_workspace_bytes(rows, C)
size_t norm_workspace_bytes(int64_t rows, int C);
// act: 0 = BN, 1 = BN + ReLU, 2 = IABN (leaky `slope`; slope == 1 -> identity)
cudaError_t bn_forward(int dtype, const void* x, const float* gamma, const float* beta, void* y, float* mean,
                       float* invstd, int64_t rows, int C, float eps, int act, float slope, void* ws,
                       cudaStream_t st);
// the two halves of bn_forward, for an IABN layer whose apply is fused with the
// residual add + activation that follows it: out = act2(round(y) + shortcut)
// (act2: 0 none, 1 relu, 2 leaky slope2); y is still written (IABN backward
// recomputes from it)
cudaError_t bn_forward_stats(int dtype, const void* x, float* mean, float* invstd, int64_t rows, int C, float eps,
                             int act, void* ws, cudaStream_t st);
// bn_apply_add_act closing the RoI head (C == 2048 fp16 / the CTA width x 8):
// the block output is average-pooled per pool_hw rows in the same pass and
// only its sign bitmap is stored (avgpool_fwd's arithmetic, bit-identical)
cudaError_t bn_apply_add_act_pool(int dtype, const void* x, const float* gamma, const float* beta, const float* mean,
                                  const float* invstd, void* y, const void* shortcut, void* pooled, int pool_hw,
                                  int64_t rows, int C, float slope, int act2, float slope2, cudaStream_t st,
                                  uint8_t* out_bits);
cudaError_t bn_apply_add_act(int dtype, const void* x, const float* gamma, const float* beta, const float* mean,
                             const float* invstd, void* y, const void* shortcut, void* out, int64_t rows, int C,
                             float slope, int act2, float slope2, cudaStream_t st, uint8_t* out_bits = nullptr);
// y_mask: stored BN+ReLU output (relu mask) or null for plain BN
cudaError_t bn_backward(int dtype, const void* dy, const void* x, const void* y_mask, const float* gamma,
                        const float* mean, const float* invstd, void* dx, float* dgamma, float* dbeta, int64_t rows,
                        int C, void* ws, cudaStream_t st);
bool norm_channels_ok(int C);
// BN/IABN forward whose statistics came fused out of the producing fprop
// (ConvStats.produced); y == nullptr: statistics only (the fused bn3 apply)
cudaError_t bn_forward_conv_stats(int dtype, const void* x, const float* gamma, const float* beta, void* y,
                                  float* mean, float* invstd, int64_t rows, int C, float eps, int act, float slope,
                                  const ConvStats& cs, cudaStream_t st);
// SyncBN (src/syncbn.cpp:21-117 with a group): the per-rank float sums go to
// agg [2C+1] (forward: sum, sumsq, count) / red [2C] (backward: sum dy, sum
// dy*xhat); the caller all-reduces them between the two halves
cudaError_t syncbn_local_sums(int dtype, const void* x, int64_t rows, int C, float* agg, void* ws, cudaStream_t st);
cudaError_t syncbn_forward_finish(int dtype, const void* x, const float* gamma, const float* beta, void* y,
                                  float* mean, float* invstd, const float* agg, int64_t rows, int C, float eps,
                                  int act, cudaStream_t st);
cudaError_t syncbn_backward_local_sums(int dtype, const void* dy, const void* x, const void* y_mask,
                                       const float* mean, const float* invstd, float* red, int64_t rows, int C,
                                       void* ws, cudaStream_t st);
cudaError_t syncbn_backward_finish(int dtype, const void* dy, const void* x, const void* y_mask, const float* gamma,
                                   const float* mean, const float* invstd, const float* red, const float* agg_fwd,
                                   void* dx, float* dgamma, float* dbeta, int64_t rows, int C, void* ws,
                                   cudaStream_t st);
// iabn_backward from the statistics a dgrad epilogue reduced (ConvStats with
// bs_y): finalize into dgamma/dbeta and the coefficients (coef: 2C floats of
// workspace), then the apply pass dx = f(dy, y)
cudaError_t iabn_backward_conv_stats(int dtype, const void* dy, const void* y, const float* gamma, const float* beta,
                                     const float* invstd, void* dx, float* dgamma, float* dbeta, int64_t rows, int C,
                                     float slope, const ConvStats& cs, float* coef, cudaStream_t st);
// iabn_backward of the layer whose dy is the masked average-pool backward
// (the last RoI-head block's bn3 when its output was pooled in place): dy is
// formed from the pooled gradient and the output's sign bitmap inside the
// statistics pass (written once to dy_out for the residual consumer) and again
// inside the apply pass, never read back as a tensor
cudaError_t iabn_backward_pooled(int dtype, const void* pooled, const uint8_t* bits, int pool_hw, float neg,
                                 const void* y, const float* gamma, const float* beta, const float* invstd,
                                 void* dy_out, void* dx, float* dgamma, float* dbeta, int64_t rows, int C, float slope,
                                 void* ws, cudaStream_t st);
cudaError_t iabn_backward(int dtype, const void* dy, const void* y, const float* gamma, const float* beta,
                          const float* mean, const float* invstd, void* dx, float* dgamma, float* dbeta,
                          int64_t rows, int C, float slope, void* ws, cudaStream_t st);

// ---- optim.cu
cudaError_t nonfinite_check(int gdtype, const void* g, int64_t n, int* flag, cudaStream_t st);
cudaError_t fused_sgd(int gdtype, const void* gsum, float* w, float* v, __half* w16, int64_t n, float lr, float mu,
                      const double* scale, double denom_mult, const int* flag, cudaStream_t st);
cudaError_t update_scale_device(double* scale, int64_t* good_steps, const int* flag, int dynamic,
                                int64_t growth_interval, double growth, double backoff, double min_scale,
                                double max_scale, cudaStream_t st);
cudaError_t cast_f32_f16(const float* in, __half* out, int64_t n, cudaStream_t st);
cudaError_t cast_f16_f32(const __half* in, float* out, int64_t n, cudaStream_t st);

}  // namespace sdb
