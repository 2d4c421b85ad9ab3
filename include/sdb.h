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
    SDB_UNSUPPORTED = 8,    /* shape outside the kernels' envelope          */
    SDB_FORMAT = 9          /* simdet::FormatError           errors.hpp:40  */
} sdb_status;

typedef enum { SDB_F32 = 0, SDB_F16 = 1, SDB_F64 = 2 /* collectives only */ } sdb_dtype;

typedef struct sdb_ctx sdb_ctx;

const char* sdb_last_error(void);
int sdb_version(void);

/* ---- context: replaces run_workers + CommGroup (src/comm.cpp:242-245,451-471).
 * nccl_id: 128-byte ncclUniqueId shared by all ranks (required when world > 1).
 * world == 1 with an id builds a 1-rank NCCL communicator: every collective of
 * the data-parallel step is then issued (and captured) as at world > 1.
 * Ops that take context workspace (conv wgrad, norms, proposal/targets,
 * losses) must be issued on one stream per context. */
int sdb_ctx_create(int device, int rank, int world, const void* nccl_id, sdb_ctx** out);
int sdb_ctx_destroy(sdb_ctx* ctx);
void* sdb_ctx_stream(sdb_ctx* ctx);
int sdb_get_nccl_unique_id(void* out128);
int sdb_synchronize(sdb_ctx* ctx);
/* ---- device memory for hosts without a CUDA runtime of their own (the
 * reference is a pure C++ CPU library; its shim stages Tensors through these).
 * Copies are ordered on the context's stream and complete before returning. */
int sdb_device_alloc(sdb_ctx* ctx, size_t bytes, void** out);
int sdb_device_free(sdb_ctx* ctx, void* p);
int sdb_copy_to_device(sdb_ctx* ctx, void* dst, const void* src, size_t bytes);
int sdb_copy_to_host(sdb_ctx* ctx, void* dst, const void* src, size_t bytes);
/* in-place SUM over the context's ranks: CommGroup::allreduce_sum
 * (src/comm.cpp:288-315), NCCL on `stream`; dtype SDB_F32 / SDB_F16 / SDB_F64;
 * identity without a communicator.  Issue order must agree on every rank (the
 * reference's sequence check, src/comm.cpp:268-278). */
int sdb_allreduce_sum(sdb_ctx* ctx, int dtype, void* buf, int64_t n, void* stream);
/* watchdog: SDB_COLLECTIVE when the communicator reported an asynchronous
 * error (ncclCommGetAsyncError) -- the CollectiveError path of
 * src/comm.cpp:270-282 for failures that surface after the call returned */
int sdb_comm_check(sdb_ctx* ctx);

/* ---- convolution: simdet::conv2d (src/tensor.cpp:169-196) and
 * Tape::conv2d backward (src/autograd.cpp:290-320).
 * x [N,H,W,C], w [K,R,S,C], y [N,Ho,Wo,K]; single stride/pad, no bias. */
int sdb_conv_fprop(sdb_ctx* ctx, int dtype, const void* x, const void* w, void* y, int N, int H, int W, int C, int K,
                   int R, int S, int stride, int pad, void* stream);
/* dx (=|+=) conv^T(dy, w); accumulate=1 adds into dx (residual fan-in) */
int sdb_conv_dgrad(sdb_ctx* ctx, int dtype, const void* dy, const void* w, void* dx, int N, int H, int W, int C, int K,
                   int R, int S, int stride, int pad, int accumulate, void* stream);
/* dw = sum over pixels dy (x) im2col(x); deterministic split-K (no atomics) */
/* fused residual fan-in + activation backward of the training step (tests and
 * tools): dx = act'(y) * rn16(conv^T(dy, w) + addend), act' = 1 where y > 0
 * else neg (the Tape's add + leaky/relu backward, src/autograd.cpp:340-351,
 * folded into the dgrad epilogue).  y_bits (optional) = sign bitmap of y, bit
 * c%8 of byte [pixel][c/8]; results are identical with and without it. */
int sdb_conv_dgrad_act(sdb_ctx* ctx, int dtype, const void* dy, const void* w, void* dx, int N, int H, int W, int C,
                       int K, int R, int S, int stride, int pad, const void* addend, const void* y, float neg,
                       const void* y_bits, void* stream);
int sdb_conv_wgrad(sdb_ctx* ctx, int dtype, const void* x, const void* dy, void* dw, int N, int H, int W, int C, int K,
                   int R, int S, int stride, int pad, void* stream);
/* conv2d followed by the BN / IABN forward statistics of its output (what the
 * training step runs before every norm layer): on the tcgen05 TMA-store path
 * the per-channel fp64 sums are reduced inside the fprop epilogue (no extra
 * read of y); elsewhere a separate statistics pass runs.  mean/invstd [K] as
 * syncbn_forward / iabn_forward compute them (src/syncbn.cpp:27-56,
 * src/memopt.cpp:247-259); iabn selects the IABN variant; *fused (optional)
 * reports which path ran. */
int sdb_conv_fprop_stats(sdb_ctx* ctx, int dtype, const void* x, const void* w, void* y, int N, int H, int W, int C,
                         int K, int R, int S, int stride, int pad, float eps, int iabn, float* mean, float* invstd,
                         int* fused, void* stream);
/* the backward twin: a stride-1 dgrad whose output dy_iabn is the gradient of
 * an InPlace-ABN output y (the conv's input), followed by that layer's
 * iabn_backward (src/memopt.cpp:278-327) -> dz, dgamma, dbeta.  On the
 * tcgen05 path the IABN backward sums (sum dz, sum dz*xhat) are reduced in the
 * dgrad epilogue from the staged dy box and a TMA-loaded y box, so the norm
 * backward is one apply pass; *fused (optional) reports which path ran.
 * H, W, C: the conv input (= y) dims; K, R, S, pad: the filter. */
int sdb_conv_dgrad_iabn_bwd(sdb_ctx* ctx, int dtype, const void* dy, const void* w, void* dy_iabn, int N, int H, int W,
                            int C, int K, int R, int S, int pad, const void* y, const float* gamma, const float* beta,
                            const float* invstd, float slope, void* dz, float* dgamma, float* dbeta, int* fused,
                            void* stream);

/* ---- BatchNorm: syncbn_forward/backward with group == nullptr
 * (src/syncbn.cpp:21-117).  rows = N*H*W; relu=1 fuses the ReLU that follows
 * BN in the reference chain (src/model.cpp:238-245). */
int sdb_bn_fwd(sdb_ctx* ctx, int dtype, const void* x, const float* gamma, const float* beta, void* y, float* mean,
               float* invstd, int64_t rows, int C, float eps, int relu, void* stream);
/* y_relu: the stored BN+ReLU output when relu was fused, else NULL */
int sdb_bn_bwd(sdb_ctx* ctx, int dtype, const void* dy, const void* x, const void* y_relu, const float* gamma,
               const float* mean, const float* invstd, void* dx, float* dgamma, float* dbeta, int64_t rows, int C,
               void* stream);

/* ---- SyncBN across the context's ranks: syncbn_forward/backward with a group
 * (src/syncbn.cpp:21-117).  Forward: per-rank FP64 sums rounded to float into
 * agg[2C+1] = [sum, sumsq, count] (device, caller-owned; keep it for the
 * backward), one fp32 SUM allreduce over the ranks (NCCL on `stream`; identity
 * at world 1), mean/invstd from the global sums.  Backward: red[2C] = [sum dy,
 * sum dy*xhat] allreduced the same way; dgamma/dbeta are the GLOBAL sums, as in
 * the reference -- a caller must not allreduce them again (the reference
 * trainer does). rows = this rank's N*H*W. */
int sdb_syncbn_fwd(sdb_ctx* ctx, int dtype, const void* x, const float* gamma, const float* beta, void* y,
                   float* mean, float* invstd, float* agg, int64_t rows, int C, float eps, int relu, void* stream);
int sdb_syncbn_bwd(sdb_ctx* ctx, int dtype, const void* dy, const void* x, const void* y_relu, const float* gamma,
                   const float* mean, const float* invstd, const float* agg_fwd, float* red, void* dx, float* dgamma,
                   float* dbeta, int64_t rows, int C, void* stream);
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
/* debug switches (tests only): key 1 = force the CUDA-core conv path instead
 * of tcgen05 (a second, independently ordered implementation of the same GEMM
 * views -- used to measure the fp16 accumulation-order noise floor). */
int sdb_debug_set(int key, int value);
/* binary16 RNE round trip / casts (src/half.cpp:9-71) */
int sdb_cast(sdb_ctx* ctx, int src_dtype, const void* src, int dst_dtype, void* dst, int64_t n, void* stream);

/* ---- detection operators (no reference implementation exists; semantics of
 * the restated oracle, boxes/IoU/ordering per src/postproc.cpp:20-63). ---- */
/* RPN proposal layer per image: top pre_k by (score desc, index asc), decode,
 * clip, greedy bitmask NMS (IoU > iou in FP64), first post_k kept.
 * logits [n_img][n_loc][A_pad], deltas [n_img][n_loc][4*A_pad] (dtype),
 * anchors [n_loc*A][4] fp32; outputs rois [n_img][post_k][4], count [n_img]. */
int sdb_rpn_proposal(sdb_ctx* ctx, int dtype, const void* logits, const void* deltas, const float* anchors, int n_img,
                     int n_loc, int A, int A_pad, int pre_k, double iou, int post_k, float img_h, float img_w,
                     float* rois, float* roi_scores, int32_t* count, int32_t* topk_order, void* stream);
/* anchors [H*W*A][4] for scales x ratios (anchor a = ratio_i * n_scales + scale_j) */
int sdb_make_anchors(sdb_ctx* ctx, int H, int W, float stride, const float* scales, int n_scales,
                     const float* ratios, int n_ratios, float* out, void* stream);
/* RoIAlign (aligned, fixed sampling ratio): feat [N,H,W,C], rois [R][5] =
 * (batch, x1, y1, x2, y2); out [R,P,P,C].  Backward is an atomics-free gather. */
int sdb_roialign_fwd(sdb_ctx* ctx, int dtype, const void* feat, int N, int H, int W, int C, const float* rois, int R,
                     int P, float spatial_scale, int sampling_ratio, void* out, void* stream);
int sdb_roialign_bwd(sdb_ctx* ctx, int dtype, const void* dy, int N, int H, int W, int C, const float* rois, int R,
                     int P, float spatial_scale, int sampling_ratio, void* dfeat, void* stream);
/* the same with the bin subsampling of the training step folded in: only every
 * bin_step-th bin of the P x P grid is pooled (out/dy [R][Po][Po][C], Po =
 * ceil(P / bin_step)) -- exactly the values a following 1x1 stride-bin_step
 * convolution reads (the res5 entry block of the C4 head) */
int sdb_roialign_fwd_folded(sdb_ctx* ctx, int dtype, const void* feat, int N, int H, int W, int C, const float* rois,
                            int R, int P, float spatial_scale, int sampling_ratio, int bin_step, void* out,
                            void* stream);
int sdb_roialign_bwd_folded(sdb_ctx* ctx, int dtype, const void* dy, int N, int H, int W, int C, const float* rois,
                            int R, int P, float spatial_scale, int sampling_ratio, int bin_step, void* dfeat,
                            void* stream);
/* softmax cross-entropy, the reference CE op (src/model.cpp:101-151): mean over
 * rows with label >= 0, backward scaled by *grad_scale (device double or NULL).
 * logits/dlogits [R][ld] (first ncls columns valid); loss written to *loss. */
int sdb_softmax_ce(sdb_ctx* ctx, int dtype, const void* logits, int R, int ncls, int ld, const int32_t* labels,
                   const double* grad_scale, double* loss, void* dlogits, void* stream);

/* losses of the detection step (scale folded into the backward like the CE op,
 * src/model.cpp:139; loss values are unscaled, written as double to *loss).
 * RPN objectness: sigmoid BCE, mean over anchors labelled 0/1 (label -1 =
 * ignored); logits [n_loc][A_pad], labels [n_loc*A] int8. */
int sdb_rpn_bce(sdb_ctx* ctx, int dtype, const void* logits, int64_t n_loc, int A, int A_pad, const int8_t* labels,
                const double* grad_scale, double* loss, void* dlogits, void* stream);
/* RPN box regression: smooth-L1 (beta) over anchors labelled 1, summed and
 * divided by norm; deltas [n_loc][4*A_pad], targets [n_loc*A][4] fp32 */
int sdb_rpn_smoothl1(sdb_ctx* ctx, int dtype, const void* deltas, int64_t n_loc, int A, int A_pad,
                     const int8_t* labels, const float* targets, double beta, double norm, const double* grad_scale,
                     double* loss, void* ddeltas, void* stream);
/* RCNN class-specific box regression: smooth-L1 (beta) of pred[r][4*label ..
 * 4*label+3] against targets[r] for foreground RoIs (label > 0), summed and
 * divided by the number of RoIs with label >= 0; pred [R][ld] */
int sdb_smoothl1(sdb_ctx* ctx, int dtype, const void* pred, int R, int ld, const int32_t* labels,
                 const float* targets, double beta, const double* grad_scale, double* loss, void* dpred,
                 void* stream);
/* RPN anchor targets per image: IoU of every anchor with the GT (FP64,
 * src/postproc.cpp:20-26 convention), fg = best IoU >= fg_thr or the best
 * anchor of a GT box, bg = best IoU < bg_thr, anchors crossing the image
 * ignored, then keyed random subsampling to batch anchors with at most
 * fg_frac*batch foreground (keys [n_img], splitmix64 of the slot);
 * labels [n_img][nA] (1 fg, 0 bg, -1 ignored), targets [n_img][nA][4]. */
int sdb_anchor_targets(sdb_ctx* ctx, const float* anchors, int nA, int n_img, const float* gt, int gt_stride,
                       const int32_t* gt_count, float img_h, float img_w, const uint64_t* keys, double fg_thr,
                       double bg_thr, int batch, double fg_frac, int8_t* labels, float* targets, void* stream);
/* RCNN proposal targets per image: candidates = proposals + GT boxes, fg =
 * IoU >= fg_thr, bg = IoU in [bg_lo, bg_hi), keyed sampling of batch RoIs with
 * at most round(fg_frac*batch) fg; out_rois [n_img*batch][5] (image, box),
 * labels (class, 0 bg, -1 padding), targets [..][4], count [n_img] */
int sdb_proposal_targets(sdb_ctx* ctx, const float* proposals, int prop_stride, const int32_t* prop_count,
                         const float* gt, const int32_t* gt_cls, int gt_stride, const int32_t* gt_count, int n_img,
                         const uint64_t* keys, double fg_thr, double bg_hi, double bg_lo, int batch, double fg_frac,
                         float* out_rois, int32_t* out_labels, float* out_targets, int32_t* out_count,
                         void* stream);

/* ---- the data-parallel Faster R-CNN C4 training step (src/trainer.cpp:217-271) ---- */
typedef struct {
    int mode;            /* 0: fp32 + BN+ReLU (config C1); 1: fp16 + InPlace-ABN, fp32 masters;
                            2: fp32 + InPlace-ABN (isolates fp16 rounding in parity tests) */
    int batch;           /* images per GPU */
    int img_h, img_w;
    int blocks[4];       /* bottlenecks in res2..res5 (res5 == 0: RoIAlign -> avgpool -> fc head) */
    int num_classes;     /* foreground classes (background added) */
    int rpn_channels;
    int n_scales, n_ratios;
    float scales[8], ratios[8];
    int pre_nms, post_nms;
    double nms_iou;
    int rpn_batch;
    double rpn_fg_frac, rpn_fg_thr, rpn_bg_thr;
    int roi_batch;
    double roi_fg_frac, roi_fg_thr, roi_bg_hi, roi_bg_lo;
    int pool, sampling_ratio;
    float lr, momentum, eps, slope;
    int dynamic_scale;
    double scale_init;
    int64_t growth_interval;
    double growth, backoff, min_scale, max_scale;
    uint64_t seed;
    int max_gt;
    double bucket_mb;    /* fp16 gradient bucket size for the NCCL allreduce */
    int shard_optimizer; /* fp16 with a communicator: reduce-scatter each bucket, update this
                            rank's 1/K shard of the fp32 masters, all-gather the fp16 shadows
                            (instead of allreduce + a replicated update) */
    int sync_bn;         /* mode 0 only: cross-GPU SyncBN (bn.mode "sync", src/model.cpp:204):
                            every BN layer's float [sum, sumsq, count] and backward [sum dy,
                            sum dy*xhat] are summed over the ranks (src/syncbn.cpp:21-117);
                            dgamma/dbeta are then global and, as in the reference trainer
                            (src/trainer.cpp:251), summed again with the other gradients */
    int checkpoint;      /* memory.checkpoint (src/trainer.cpp:233): sqrt(L) activation
                            checkpointing of the backbone's L bottleneck blocks with the
                            reference's segment plan (src/memopt.cpp:76-89); only segment
                            boundary outputs persist, each segment is recomputed from its
                            boundary in backward (src/memopt.cpp:150-210); bit-identical */
} sdb_det_config;

typedef struct sdb_det sdb_det;

int sdb_det_create(sdb_ctx* ctx, const sdb_det_config* cfg, sdb_det** out);
int sdb_det_destroy(sdb_det* det);
/* parameter registry, in the reference's flat pack order (src/model.cpp:155-167 style) */
int sdb_det_num_params(sdb_det* det, int* n_tensors, int64_t* n_conv_fc, int64_t* n_bn);
/* kind: 0 conv [O,C,kh,kw], 1 fc [in,out], 2 bn gamma [C], 3 bn beta [C] (reference layouts) */
int sdb_det_param_info(sdb_det* det, int idx, char* name, int name_len, int64_t* shape4, int* ndim, int* kind);
int sdb_det_get_param(sdb_det* det, int idx, float* host);  /* fp32 master, reference layout */
int sdb_det_set_param(sdb_det* det, int idx, const float* host);
int sdb_det_get_grad(sdb_det* det, int idx, float* host);   /* last step's summed gradient (scaled) */
int sdb_det_get_velocity(sdb_det* det, int idx, float* host);       /* SGD momentum buffer */
/* Training state in the reference's SDCK v1 format (src/checkpoint.cpp:47-128):
 * fp32 masters in pack order and reference layouts, the flat velocity, the
 * loss-scale state; no running-stat blocks (IABN keeps none).  A run resumed
 * from it continues bit-identically (tests/test_trainer.cpp:203-290).  Load
 * checks magic/version/truncation (SDB_FORMAT) and that names and shapes match
 * this detector (SDB_CONTRACT); step and config digest are returned. */
int sdb_det_save_checkpoint(sdb_det* det, const char* path, uint64_t config_digest, int64_t step);
int sdb_det_load_checkpoint(sdb_det* det, const char* path, uint64_t* config_digest, int64_t* step);
int sdb_det_set_velocity(sdb_det* det, int idx, const float* host);
/* feed one batch: images NHWC with C padded to 8 (dtype of the mode), on host
 * (pinned, copied H2D on the step stream) or device; GT arrays on host
 * ([batch][max_gt][4], [batch][max_gt], [batch]); slots = global batch slots
 * (src/dataset.cpp:94) keying the sampling RNG. */
int sdb_det_set_batch(sdb_det* det, const void* images, int images_on_host, const float* gt_boxes,
                      const int32_t* gt_cls, const int32_t* gt_count, const int64_t* slots);
/* synthesize the batch's images on device from the slots (N(0,1) pixels) */
int sdb_det_synth_images(sdb_det* det, const int64_t* slots);
int sdb_det_step(sdb_det* det);
/* blocks until the step finished; losses[0..3] = rpn_cls, rpn_box, rcnn_cls,
 * rcnn_box (allreduced /K), losses[4] = total; scale_used; overflow flag */
int sdb_det_read_losses(sdb_det* det, double* losses5, double* scale_used, int* overflow);
/* end-to-end call with HOST buffers: H2D of images+GT, the step, D2H of losses */
int sdb_det_train_step_host(sdb_det* det, const void* images_host, const float* gt_boxes, const int32_t* gt_cls,
                            const int32_t* gt_count, const int64_t* slots, double* losses5);
/* the same with images in the reference layout [batch][3][H][W] (Tensor NCHW,
 * src/tensor.cpp; dtype of the detector): only the 3 real channels cross PCIe,
 * the 8-channel NHWC padding is done on device */
int sdb_det_train_step_host_nchw(sdb_det* det, const void* images_nchw_host, const float* gt_boxes,
                                 const int32_t* gt_cls, const int32_t* gt_count, const int64_t* slots,
                                 double* losses5);
/* debug/parity exports of the last step's discrete decisions & intermediates.
 * what: 0 anchor labels (int8 [batch][nA]), 1 anchor targets (f32 [batch][nA][4]),
 * 2 proposals (f32 [batch][post][4]), 3 proposal counts (i32 [batch]),
 * 4 sampled rois (f32 [batch*roi_batch][5]), 5 roi labels (i32), 6 roi targets (f32 [..][4]),
 * 7 rpn logits (dtype [batch][n_loc][A_pad]), 8 rpn deltas (dtype [batch][n_loc][4*A_pad]),
 * 9 anchors (f32 [nA][4]), 10 C4 feature (dtype NHWC), 11 images (dtype NHWC8),
 * 12 loss-scale state (f64 scale, then i64 good_steps), 13 stem conv output (dtype NHWC),
 * 14 max-pool output (dtype NHWC), 15 stem im2col matrix (f16 [pixels][192], fp16 mode),
 * 16 fp16 weight shadows (flat, driver layout), 17 fp32 masters (flat, driver layout),
 * 18 RoIAlign output (dtype [R][Po][Po][1024], Po = the pooled bins the head reads),
 * 19 RoI-head output (dtype NHWC), 20 pooled head features (dtype [R][feat]),
 * 21 class logits (dtype [R][ncls_pad]), 22 box regression (dtype [R][4*(ncls) padded]).
 * Returns bytes in *bytes. */
int sdb_det_export(sdb_det* det, int what, void* host, int64_t capacity, int64_t* bytes);
int sdb_det_dims(sdb_det* det, int* feat_h, int* feat_w, int* n_anchor_per_loc, int* a_pad);
/* launches of libsdb kernels per step (counted at the first step) */
int sdb_det_kernel_launches(sdb_det* det, int64_t* n);
/* the checkpoint segment plan for L layers (host logic, no GPU): starts[0..S]
 * = segment starts then L; returns S (= ceil(sqrt(L)) segments, the reference's
 * plan_checkpoints, src/memopt.cpp:76-89), or < 0 (SDB_PARAM for L < 1) */
int sdb_plan_checkpoints(int L, int* starts, int cap);
/* device memory: bytes of backbone activations (persistent tensors + the
 * checkpoint arena), all device bytes the detector allocated, and the
 * checkpoint segment count (0: checkpointing off) -- the MemoryTrace "act"
 * peak of tests/test_memopt.cpp:139-150 for this static schedule */
int sdb_det_memory(sdb_det* det, int64_t* backbone_act_bytes, int64_t* device_bytes, int* segments);
/* the gradient-bucket plan of the data-parallel allreduce (host logic, no GPU):
 * offsets = start of every conv/fc gradient slice in the flat buffer (pack
 * order), total = buffer length; buckets are emitted in issue order (from the
 * end).  Returns the bucket count; out_lo_hi gets [lo, hi) pairs. */
int sdb_plan_buckets(const int64_t* offsets, int n, int64_t total, int64_t cap_elems, int64_t* out_lo_hi, int cap_out);
/* one eager, CUDA-event-instrumented step on the current batch: per category
 * (0 conv fprop, 1 dgrad, 2 wgrad, 3 norm fwd, 4 norm bwd, 5 elementwise,
 * 6 pooling, 7 targets, 8 proposal, 9 roialign fwd, 10 roialign bwd, 11 losses,
 * 12 optimizer, 13 comm) device ms, algorithmic FLOPs, algorithmic bytes, launches */
int sdb_det_profile(sdb_det* det, double* ms, double* flops, double* bytes, int64_t* launches, int ncat);
/* the last profiled step's labelled records (every conv: "fprop|dgrad|wgrad N H W
 * C K R S st"; norms with SDB_PROFILE_VERBOSE): k < 0 returns the count, else
 * record k's category, label, device ms, algorithmic FLOPs and bytes */
int sdb_det_profile_record(sdb_det* det, int k, int* cat, char* label, int cap, double* ms, double* flops,
                           double* bytes);

#ifdef __cplusplus
}
#endif
#endif /* SDB_H_ */
