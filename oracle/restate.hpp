// oracle/restate.hpp -- TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the operators on the SimpleDet Faster R-CNN C4 training
// step that the reference `simdet` engine (/root/reference/proj) either keeps
// in an anonymous namespace (softmax-CE, apply_sgd) or does not implement at
// all (anchors, RPN proposal layer, RoIAlign, max-pool, detection losses,
// anchor/proposal target assignment).  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline leg may load this code, and only as the checker.
//
// Parity status:
//   * apply_sgd, softmax-CE, update_scale, iou, nms_greedy, binary16 RNE:
//     restatements pinned against the compiled reference (oracle/_ref) and the
//     reference's own golden vectors (tests/test_oracle_pins.py).
//   * anchors / decode / proposal / targets / RoIAlign / max-pool / BCE /
//     smooth-L1: the reference has no implementation -> "parity unpinned by
//     the reference"; pinned instead by self-authored known-answer tests and,
//     for RoIAlign, by torchvision.ops.roi_align as an independent check.
//
// Conventions follow the reference (file:line under /root/reference/proj):
//   - boxes are continuous corners, no +1 (src/postproc.cpp:20-26, postproc.hpp:12-21)
//   - IoU in FP64, 0 when the union is 0 (src/postproc.cpp:20-26)
//   - ordering is (score desc, index asc) (src/postproc.cpp:41-43)
//   - suppression iff IoU > t strictly (src/postproc.cpp:58)
//   - counter RNG is the reference's mix64 (src/dataset.cpp:11-17)
//   - FP32 accumulation for conv-like loops, FP64 for statistics/losses
//     (src/tensor.cpp:178-194, src/syncbn.cpp:29-39, src/model.cpp:117-128)
// Build with -ffp-contract=off: several outputs are compared bit-exactly.
#pragma once
#include <cstdint>

extern "C" {

// ---- numerics ----
float orc_half_round(float f);                       // RNE through binary16 (src/half.cpp:9-50)
void orc_half_round_n(const float* in, float* out, int64_t n);
float orc_expf(float x);                             // portable exp, bit-identical to the CUDA path
uint64_t orc_mix64(uint64_t a, uint64_t b);          // src/dataset.cpp:11-17

// ---- optimizer / loss scale (src/trainer.cpp:78-94, src/precision.cpp:45-56) ----
int orc_has_nonfinite(const float* g, int64_t n);
void orc_apply_sgd(float* w, float* v, const float* gsum, int64_t n, float lr, float mu, double denom);
void orc_update_scale(double* scale, int64_t* good_steps, int dynamic, int64_t growth_interval,
                      double growth, double backoff, double min_scale, double max_scale, int overflow);

// ---- losses (loss scale folded into backward, src/model.cpp:132-150) ----
// softmax CE over rows, mean over B; returns loss, writes dx (may be null)
double orc_softmax_ce(const float* logits, int64_t B, int64_t C, const int32_t* labels, double dy,
                      double grad_scale, float* dx);
// sigmoid BCE over elements with label >= 0, normalised by `norm`
double orc_sigmoid_bce(const float* logits, const int8_t* labels, int64_t n, double norm,
                       double grad_scale, float* dx);
// smooth-L1 over rows with weight[i] != 0 (4 coords per row), normalised by `norm`
double orc_smooth_l1(const float* pred, const float* target, const float* weight, int64_t rows,
                     double beta, double norm, double grad_scale, float* dpred);

// ---- boxes ----
double orc_iou(const float* a, const float* b);      // float corners widened to double
void orc_anchors(int H, int W, float stride, const float* scales, int ns, const float* ratios, int nr,
                 float* out);                        // [(H*W*A), 4], a = (y*W+x)*A + i*ns + j
void orc_decode(const float* anchors, const float* deltas, int64_t n, const float* weights4,
                float clip_dw, float img_h, float img_w, float* boxes);
void orc_encode(const float* ex, const float* gt, int64_t n, const float* weights4, float* targets);
// (score desc, index asc) order of the best k (NaN ranks below -inf)
void orc_topk_order(const float* scores, int64_t n, int64_t k, int32_t* order);
// greedy NMS over boxes already in priority order; returns kept positions
int64_t orc_nms_sorted(const float* boxes, int64_t n, double thresh, int64_t max_keep, int32_t* keep);
// full RPN proposal layer for one image
int64_t orc_proposals(const float* logits, const float* deltas, const float* anchors, int64_t n_anchors,
                      float img_h, float img_w, int64_t pre_k, double iou, int64_t post_k,
                      float* rois, float* roi_scores, int32_t* topk_order);
// RPN anchor targets for one image. labels: -1 ignore, 0 bg, 1 fg.
void orc_anchor_targets(const float* anchors, int64_t nA, const float* gt, int64_t G, float img_h,
                        float img_w, uint64_t key, double fg_thr, double bg_thr, int64_t batch,
                        double fg_frac, int8_t* labels, float* bbox_targets);
// RCNN proposal targets for one image. Returns the sampled count S.
int64_t orc_proposal_targets(const float* rois, int64_t R, const float* gt, const int32_t* gt_cls,
                             int64_t G, uint64_t key, double fg_thr, double bg_hi, double bg_lo,
                             int64_t batch, double fg_frac, float* out_rois, int32_t* out_labels,
                             float* out_targets, int32_t* out_src_index);

// ---- feature ops, NCHW, fp32 math ----
void orc_roialign_fwd(const float* feat, int N, int C, int H, int W, const float* rois, int64_t R,
                      int P, float spatial_scale, int sr, int aligned, float* out);
void orc_roialign_bwd(const float* dy, int N, int C, int H, int W, const float* rois, int64_t R,
                      int P, float spatial_scale, int sr, int aligned, float* dfeat);
void orc_maxpool_fwd(const float* x, int N, int C, int H, int W, int k, int s, int p, float* y);
void orc_maxpool_bwd(const float* x, const float* dy, int N, int C, int H, int W, int k, int s, int p,
                     float* dx);
void orc_avgpool_fwd(const float* x, int N, int C, int H, int W, float* y);
void orc_avgpool_bwd(const float* dy, int N, int C, int H, int W, float* dx);

}  // extern "C"
