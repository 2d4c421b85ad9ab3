// detect.h -- argument blocks for the detection kernels (proposal.cu, roi.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sdb {

struct AnchorCfg {
    int H, W;        // feature grid
    float stride;
    int ns, nr;      // scales, ratios (anchor a = i*ns + j: ratio-major)
    float scales[8];
    float ratios[8];
};

struct ProposalArgs {
    const void* logits;  // [n_img][n_loc][A_pad]
    const void* deltas;  // [n_img][n_loc][4*A_pad]
    int dtype;
    const float* anchors;  // [n_loc*A][4]
    int n_img, n_loc, A, A_pad;
    int pre_k, post_k;
    double iou_thr;
    float img_h, img_w, clip_dw;
    float* rois;          // [n_img][post_k][4]
    float* roi_scores;    // [n_img][post_k] (optional)
    int32_t* keep_pos;    // [n_img][post_k] positions in the top-k order
    int32_t* count;       // [n_img]
    int32_t* topk_order_out;  // optional [n_img][k]
};

struct AnchorTargetArgs {
    const float* anchors;
    int nA, n_img;
    const float* gt;         // [n_img][gt_stride][4]
    int gt_stride;
    const int32_t* gt_count; // [n_img]
    float img_h, img_w;
    const uint64_t* keys;    // [n_img] sampling keys
    double fg_thr, bg_thr;
    int batch, fg_cap;
    int8_t* labels;          // [n_img][nA]
    float* targets;          // [n_img][nA][4]
};

struct ProposalTargetArgs {
    const float* proposals;  // [n_img][prop_stride][4]
    int prop_stride;
    const int32_t* prop_count;
    const float* gt;
    const int32_t* gt_cls;
    int gt_stride;
    const int32_t* gt_count;
    const uint64_t* keys;
    double fg_thr, bg_hi, bg_lo;
    int batch, fg_cap, n_img;
    int8_t* work_flag;       // [n_img][work_stride]
    int32_t* work_arg;       // [n_img][work_stride]
    int work_stride;         // >= prop_stride + gt_stride
    float* out_rois;         // [n_img*batch][5] (batch idx, x1, y1, x2, y2); padded slots idx -1
    int32_t* out_labels;     // [n_img*batch] class (0 bg) or -1 padding
    float* out_targets;      // [n_img*batch][4]
    int32_t* out_src;        // optional [n_img*batch] candidate index
    int32_t* out_count;      // [n_img]
};

#ifdef __CUDACC__
// orc_encode (oracle/restate.cpp) with weights (wx, wy, ww, wh)
__device__ __forceinline__ void encode_box(const float* e, const float* g, float wx, float wy, float ww, float wh,
                                          float* t) {
    const float ew = __fsub_rn(e[2], e[0]), eh = __fsub_rn(e[3], e[1]);
    const float ecx = __fadd_rn(e[0], __fmul_rn(0.5f, ew)), ecy = __fadd_rn(e[1], __fmul_rn(0.5f, eh));
    const float gw = __fsub_rn(g[2], g[0]), gh = __fsub_rn(g[3], g[1]);
    const float gcx = __fadd_rn(g[0], __fmul_rn(0.5f, gw)), gcy = __fadd_rn(g[1], __fmul_rn(0.5f, gh));
    t[0] = __fdiv_rn(__fmul_rn(wx, __fsub_rn(gcx, ecx)), ew);
    t[1] = __fdiv_rn(__fmul_rn(wy, __fsub_rn(gcy, ecy)), eh);
    t[2] = __fmul_rn(ww, logf(__fdiv_rn(gw, ew)));
    t[3] = __fmul_rn(wh, logf(__fdiv_rn(gh, eh)));
}
#endif

cudaError_t make_anchors(const AnchorCfg& cfg, float* out, cudaStream_t st);
size_t proposal_workspace_bytes(int n_img, int n_anchors, int pre_k);
cudaError_t rpn_proposals(const ProposalArgs& p, void* ws, cudaStream_t st);
size_t anchor_target_workspace_bytes(int n_img, int nA, int gt_stride);
cudaError_t anchor_targets(const AnchorTargetArgs& a, void* ws, cudaStream_t st);
cudaError_t proposal_targets(const ProposalTargetArgs& a, cudaStream_t st);

// ---- roi.cu
// RoIAlign (aligned, fixed sampling ratio), NHWC features, rois [R][5].
// step > 1 computes only every step-th bin of the P x P grid (output
// ceil(P/step)^2 bins): exactly the values a following 1x1 stride-`step`
// convolution reads, so the stride folds into the pooling.
cudaError_t roialign_fwd(int dtype, const void* feat, int N, int H, int W, int C, const float* rois, int R, int P,
                         float scale, int sr, void* out, cudaStream_t st, int step = 1);
// backward workspace: per-RoI separable weight tables, boxes and per-pixel-block RoI lists
size_t roialign_bwd_workspace(int R, int H, int W, int P, int step = 1, int N = 1);
cudaError_t roialign_bwd(int dtype, const void* dy, int N, int H, int W, int C, const float* rois, int R, int P,
                         float scale, int sr, void* dfeat, void* ws, size_t ws_bytes, cudaStream_t st, int step = 1);
// [n][3][H][W] (the reference image layout) -> NHWC with Cp channels (zero padded)
cudaError_t nchw3_to_nhwc(int dtype, const void* in, int n, int H, int W, int Cp, void* out, cudaStream_t st);
// the 7x7 stem as a 1x1 GEMM over its im2col matrix X' [pixels][192] (fp16):
// stem_im2col builds X'; stem_weights packs W [K][7][7][Cs] -> W' [K][192]
// (fold = 1: dW' -> dW, zeros for the padded channels)
cudaError_t stem_im2col(const void* x, int N, int H, int W, int Cs, int Ho, int Wo, int stride, int pad, void* out,
                        cudaStream_t st);
cudaError_t stem_weights(const void* w, int K, int Cs, void* w2, int fold, cudaStream_t st);
cudaError_t maxpool_fwd(int dtype, const void* x, int N, int H, int W, int C, int k, int s, int p, void* y,
                        uint8_t* argmax, cudaStream_t st);
cudaError_t maxpool_bwd(int dtype, const void* dy, const uint8_t* argmax, int N, int H, int W, int C, int k, int s,
                        int p, void* dx, cudaStream_t st);
cudaError_t avgpool_fwd(int dtype, const void* x, int N, int HW, int C, void* y, cudaStream_t st);
// act_y (optional): fuse the backward of the activation that produced the pooled
// tensor (out = act_y > 0 ? g : neg * g on the rounded pooling gradient);
// act_bits (optional, instead of act_y): its sign bitmap (bit j of byte
// [pixel][c/8] = act_y > 0)
cudaError_t avgpool_bwd(int dtype, const void* dy, int N, int HW, int C, void* dx, cudaStream_t st,
                        const void* act_y = nullptr, float neg = 0.0f, const uint8_t* act_bits = nullptr);
// out = act(a + b); act: 0 none, 1 relu, 2 leaky(slope)
cudaError_t add_act(int dtype, const void* a, const void* b, void* out, int64_t n, int act, float slope,
                    cudaStream_t st);
// dx = dy * (y > 0 ? 1 : neg_slope)  (relu: neg_slope = 0); may be in place
cudaError_t act_bwd(int dtype, const void* dy, const void* y, void* dx, int64_t n, float neg_slope, cudaStream_t st);
cudaError_t relu_fwd(int dtype, const void* x, void* y, int64_t n, cudaStream_t st);
cudaError_t add_inplace(int dtype, void* acc, const void* b, int64_t n, cudaStream_t st);
// losses: results (double) written to loss_out[slot]; gradients (dtype) scaled by *scale
struct LossArgs {
    const double* scale;  // device loss scale (null -> 1)
    double* loss_out;
    int slot;
};
size_t loss_workspace_bytes(int64_t rows);
cudaError_t softmax_ce(int dtype, const void* logits, int R, int ncls, int ld, const int32_t* labels, void* dlogits,
                       const LossArgs& la, void* ws, cudaStream_t st);
cudaError_t sigmoid_bce(int dtype, const void* logits, int64_t n_loc, int A, int A_pad, const int8_t* labels,
                        void* dlogits, const LossArgs& la, void* ws, cudaStream_t st);
// smooth-L1 on RPN deltas: deltas [n_loc][4*A_pad], targets [n_loc*A][4], weight = (label==1)
cudaError_t rpn_smooth_l1(int dtype, const void* deltas, int64_t n_loc, int A, int A_pad, const int8_t* labels,
                          const float* targets, double beta, double norm, void* ddeltas, const LossArgs& la, void* ws,
                          cudaStream_t st);
// smooth-L1 on class-specific RCNN box regression: pred [R][ld], targets [R][4] at slot 4*label
cudaError_t rcnn_smooth_l1(int dtype, const void* pred, int R, int ld, const int32_t* labels, const float* targets,
                           double beta, void* dpred, const LossArgs& la, void* ws, cudaStream_t st);
// synthetic N(0,1) images (NHWC, C_pad channels, channels >= 3 zero) keyed by (seed, slot, element)
cudaError_t synth_images(int dtype, void* out, int n, int H, int W, int C_pad, uint64_t seed,
                         const int64_t* slots_dev, int64_t slot0, cudaStream_t st);

}  // namespace sdb
